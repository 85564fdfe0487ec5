#!/bin/bash
# Dirty-cache hypothesis for slow small copy-engine swaps (flush on / off), dynamic-run GEMM
# bring-up (correctness + timing vs static stream-K).
set -x
O=gpurun_out/r2f
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/ce_lib_probe.py 1 4 16 64 > $O/ce_lib_flush.ndjson 2>&1
MPSW_NO_FLUSH=1 timeout 300 python tools/ce_lib_probe.py 1 4 16 64 > $O/ce_lib_noflush.ndjson 2>&1
MPSW_TC_DYN=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm_dyn.txt 2>&1
MPSW_TC_DYN=1 MPSW_PARITY_LOG=$O/parity_dyn.ndjson timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_shape_fuzz.py tests/test_gpu_graphs.py -q -x --tb=short > $O/pytest_fwd_dyn.txt 2>&1
for q in 2 3 4 6; do MPSW_TC_DYN=1 MPSW_TC_DYN_Q=$q timeout 600 python tools/gemm_tune.py default >> $O/gemm_dyn.ndjson 2>&1; done
timeout 600 python tools/gemm_tune.py default >> $O/gemm_dyn.ndjson 2>&1
for d in 0 1; do
  MPSW_TC_DYN=$d timeout 900 python tools/fwd_bench.py opt-13b tc shapes=1x2,8x8,32x8 >> $O/fwd_dyn.ndjson 2>&1
  MPSW_TC_DYN=$d timeout 600 python tools/fwd_bench.py opt-1.3b tc shapes=1x2,8x8,32x8 >> $O/fwd_dyn.ndjson 2>&1
  MPSW_TC_DYN=$d timeout 600 python tools/fwd_bench.py opt-125m tc shapes=1x2,8x8 >> $O/fwd_dyn.ndjson 2>&1
done
