#!/bin/bash
set -x
O=gpurun_out/r2i
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for m in opt-13b opt-1.3b opt-125m; do timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,32x8 >> $O/fwd.ndjson 2>&1; done
timeout 600 python tools/gemm_tune.py default > $O/gemm.ndjson 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_forward.py tests/test_gpu_layers.py -q -x --tb=short > $O/pytest.txt 2>&1
