#!/bin/bash
# Reduce-scatter all-reduce, CUDA graphs, pipelined PP, AUTO table.
set -x
O=gpurun_out/r2c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_graphs.py tests/test_gpu_pp.py -q --tb=short > $O/pytest_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q --tb=short -k test_process_group > $O/pytest_mp_rs.txt 2>&1
for rs in 1152921504606846976 0; do
  MPSW_RS_MIN_BYTES=$rs timeout 900 python tools/fwd_tp.py opt-30b 8 32 8 >> $O/fwd_tp_rs.ndjson 2>&1
  MPSW_RS_MIN_BYTES=$rs timeout 900 python tools/fwd_tp.py opt-30b 8 1 2 >> $O/fwd_tp_rs.ndjson 2>&1
  MPSW_RS_MIN_BYTES=$rs timeout 900 python tools/fwd_tp.py opt-13b 4 8 8 >> $O/fwd_tp_rs.ndjson 2>&1
done
for g in 0 1; do
  for m in opt-125m opt-1.3b opt-13b; do MPSW_GRAPHS=$g timeout 900 python tools/fwd_bench.py $m tc shapes=1x2,8x8 >> $O/fwd_graphs.ndjson 2>&1; done
done
timeout 1800 python tools/auto_table.py --out $O/auto_table.ndjson > $O/auto_table.log 2>&1
