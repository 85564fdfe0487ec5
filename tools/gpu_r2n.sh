#!/bin/bash
# Session-3 re-validation of the tree as restored: full GPU tests, smoke, bench, and the
# critical-path experiments of the last session (empty-kernel stand-ins, cluster LN).
set -x
O=gpurun_out/r2n
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi -q | grep -iE 'product name|link (gen|width)' | head -8 > $O/box.txt
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1500 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for v in "MPSW_LN_CLUSTER=0" "MPSW_DEV_NOOP_LN=1" "MPSW_DEV_NOOP_ATTN=1" "MPSW_DEV_NOOP_LN=1 MPSW_DEV_NOOP_ATTN=1" "MPSW_LN_CLUSTER=1"; do
  for m in opt-13b opt-1.3b opt-125m; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/noop.ndjson 2>&1; done
done
MPSW_LN_CLUSTER=1 MPSW_PARITY_LOG=$O/parity_cluster.ndjson timeout 1200 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_allreduce.py -q -x --tb=short -k "not full_size" > $O/pytest_cluster.txt 2>&1
