#!/bin/bash
# Lean reduce_ln (2 CTAs / SM at >= 16 rows), fix-up with 4 runs x 16 tokens of loads in flight:
# correctness, forward A/B, launch list at M = 256.
set -x
O=gpurun_out/r2u
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1500 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_shape_fuzz.py tests/test_gpu_allreduce.py -q -x --tb=short -k "not full_size" > $O/pytest_fwd.txt 2>&1
for v in "MPSW_TC_SPLIT=1" "MPSW_TC_SPLIT=2" "MPSW_TC_SPLIT=2 MPSW_LN_LEAN_MIN=100000" "MPSW_TC_SPLIT=2 MPSW_DEV_NOOP_FIXUP=1" "MPSW_TC_SPLIT=2 MPSW_DEV_NOOP_LN=1" "MPSW_TC_SPLIT=2 MPSW_TC_EXT_MIN=32" "MPSW_TC_SPLIT=2 MPSW_TC_EXT_MIN=100000"; do
  for m in opt-13b opt-1.3b; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,2x8,4x8,8x8,16x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/fwd.ndjson 2>&1; done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/launches_m256.csv python tools/fwd_one.py opt-13b 32 8 2 2 > $O/ncu_m256.log 2>&1
python tools/ncu_summary.py $O/launches_m256.csv > $O/launches_m256_summary.ndjson 2>&1
