#!/bin/bash
# CTA-pair GEMM (cta_group::2) bring-up: correctness under MPSW_TC_PAIR=1, then GEMM and forward
# timings of both modes, the new PP / runtime tests, the AUTO-table measurement.
set -x
O=gpurun_out/pair
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_TC_PAIR=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm_pair.txt 2>&1
MPSW_TC_PAIR=1 MPSW_PARITY_LOG=$O/parity_pair.ndjson timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_shape_fuzz.py -q -x --tb=short > $O/pytest_fwd_pair.txt 2>&1
timeout 900 python tools/gemm_tune.py pair > $O/gemm_pair.ndjson 2>&1
for p in 0 1; do
  MPSW_TC_PAIR=$p timeout 900 python tools/fwd_bench.py opt-13b tc shapes=1x2,8x8,32x8 >> $O/fwd_pair.ndjson 2>&1
  MPSW_TC_PAIR=$p timeout 600 python tools/fwd_bench.py opt-1.3b tc shapes=1x2,8x8,32x8 >> $O/fwd_pair.ndjson 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_pp.py tests/test_gpu_runtime.py -q --tb=short > $O/pytest_pp_runtime.txt 2>&1
timeout 1500 python tools/auto_table.py --out $O/auto_table.ndjson > $O/auto_table.log 2>&1
timeout 300 python -m pytest tests/test_gpu_numa.py -q > $O/pytest_numa.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_allreduce.py -q --tb=short > $O/pytest_allreduce.txt 2>&1
for rs in 1152921504606846976 0; do
  MPSW_RS_MIN_BYTES=$rs timeout 900 python tools/fwd_tp.py opt-30b 8 32 8 >> $O/fwd_tp_rs.txt 2>&1
  MPSW_RS_MIN_BYTES=$rs timeout 900 python tools/fwd_tp.py opt-13b 8 32 8 >> $O/fwd_tp_rs.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q --tb=short -k test_process_group > $O/pytest_mp_rs.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_graphs.py -q --tb=short > $O/pytest_graphs.txt 2>&1
for g in 0 1; do
  for m in opt-125m opt-1.3b opt-13b; do MPSW_GRAPHS=$g timeout 900 python tools/fwd_bench.py $m tc shapes=1x2,8x8 >> $O/fwd_graphs.ndjson 2>&1; done
done
