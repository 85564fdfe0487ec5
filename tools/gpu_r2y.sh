#!/bin/bash
set -x
O=gpurun_out/r2y
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none --csv --log-file $O/launches_gemm64.csv python tools/gemm_one.py 64 20480 5120 2 5 > $O/ncu_l64.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gemm256.csv python tools/gemm_one.py 256 20480 5120 2 5 > $O/ncu_l256.log 2>&1
for m in opt-13b opt-1.3b; do timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,2x8,8x8,16x8,32x8 >> $O/fwd.ndjson 2>&1; done
GT_M=2,16,64,256 timeout 600 python tools/gemm_tune.py default > $O/gemm_default.ndjson 2>&1
