#!/bin/bash
# Serving traces (p50/p99) and the cfg5 bandwidth sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/serve.ndjson
timeout 300 python tools/serve_trace.py cfg1 --out gpurun_out/serve.ndjson
timeout 300 python tools/serve_trace.py cfg2 --out gpurun_out/serve.ndjson
timeout 300 python tools/serve_trace.py cfg2-t1 --out gpurun_out/serve.ndjson
for cv in 0.25 1 4; do timeout 300 python tools/serve_trace.py cfg4-analog --cv $cv --out gpurun_out/serve.ndjson; done
timeout 1200 python tools/sweep_cfg5.py --out gpurun_out/cfg5.ndjson > gpurun_out/cfg5.log 2>&1
