#!/bin/bash
O=gpurun_out/g6; mkdir -p $O; rm -f $O/trace.ndjson
timeout 600 python tools/tc_trace.py run $O/trace.ndjson > $O/run.log 2>&1
python tools/tc_trace.py show $O/trace.ndjson > $O/show.txt 2>&1
