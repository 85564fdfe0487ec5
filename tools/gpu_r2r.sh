#!/bin/bash
set -x
O=gpurun_out/r2r
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
GT_M=2,64,128,256 timeout 1200 python tools/gemm_tune.py large > $O/gemm_large.ndjson 2>&1
for v in 1 2; do MPSW_TC_VW=$v timeout 600 python tools/tc_trace.py run $O/trace_vw$v.ndjson; python tools/tc_trace.py show $O/trace_vw$v.ndjson > $O/trace_vw$v.txt 2>&1; done
