#!/bin/bash
O=gpurun_out/g7; mkdir -p $O; rm -f $O/trace.ndjson
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_forward.py -q -x > $O/pytest.txt 2>&1
timeout 900 python tools/gemm_tune.py l2pf > $O/tune.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-13b tc > $O/fwd13.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-1.3b tc > $O/fwd13b.txt 2>&1
timeout 600 python tools/tc_trace.py run $O/trace.ndjson > $O/run.log 2>&1
python tools/tc_trace.py show $O/trace.ndjson > $O/show.txt 2>&1
