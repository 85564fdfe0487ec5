#!/bin/bash
O=gpurun_out/g9; mkdir -p $O; rm -f $O/serve.ndjson
timeout 900 python tools/serve_trace.py hetero --seed 0 --out $O/serve.ndjson > $O/hetero.log 2>&1
timeout 600 python tools/serve_trace.py cfg1 --out $O/serve.ndjson > $O/cfg1.log 2>&1
timeout 600 python tools/serve_trace.py cfg4-analog --cv 4 --out $O/serve.ndjson > $O/cfg4.log 2>&1
timeout 600 python tools/serve_trace.py cfg4-analog --cv 1 --out $O/serve.ndjson > $O/cfg4b.log 2>&1
