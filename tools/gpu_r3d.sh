#!/bin/bash
# Fix-up grid shape: tokens per CTA (16 / 8), trigger before the wait; forward A/B.
set -x
O=gpurun_out/r3d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
MPSW_TC_FIX_TOK=8 MPSW_TC_FIX_EARLY=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm_tok8.txt 2>&1
GT_M=64,128,256 timeout 1200 python tools/gemm_tune.py fixup > $O/gemm_fixup.ndjson 2>&1
for v in "MPSW_TC_FIX_TOK=16" "MPSW_TC_FIX_TOK=8" "MPSW_TC_FIX_EARLY=1" "MPSW_TC_FIX_TOK=8 MPSW_TC_FIX_EARLY=1"; do
  for m in opt-13b opt-1.3b; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=8x8,16x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/fwd.ndjson 2>&1; done
done
