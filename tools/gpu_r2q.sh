#!/bin/bash
# Pair split executed on independent CTAs (small M) or CTA pairs with two workers each (large M):
# GEMM correctness (bits across executions), per-shape timing vs the single split, forward A/B.
set -x
O=gpurun_out/r2q
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
timeout 900 python tools/gemm_tune.py split > $O/gemm_split.ndjson 2>&1
for sp in 1 2; do
  for m in opt-13b opt-1.3b opt-125m; do MPSW_TC_SPLIT=$sp timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,16x8,32x8 | sed "s/^{/{\"split\": $sp, /" >> $O/fwd_split.ndjson 2>&1; done
done
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1500 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_shape_fuzz.py -q -x --tb=short -k "not full_size" > $O/pytest_fwd.txt 2>&1
