#!/bin/bash
# Sibling fix-up for tile-aligned splits: correctness (bits vs the fix-up grid) and forward A/B.
set -x
O=gpurun_out/r3c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
timeout 800 python -m pytest tests/test_gpu_gemm_modes.py -q -x --tb=short > $O/pytest_modes.txt 2>&1
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1500 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_shape_fuzz.py tests/test_gpu_graphs.py tests/test_gpu_engine.py -q -x --tb=short -k "not full_size" > $O/pytest_fwd.txt 2>&1
for v in "MPSW_TC_SIB=0" "MPSW_TC_SIB=1"; do
  for m in opt-13b opt-1.3b opt-125m; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,16x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/fwd.ndjson 2>&1; done
  env $v GT_M=2,64,256 timeout 600 python tools/gemm_tune.py default | sed "s/^{/{\"variant\": \"$v\", /" >> $O/gemm.ndjson 2>&1
done
