#!/bin/bash
set -x
O=gpurun_out/r2m
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for v in "MPSW_LN_CLUSTER=0" "MPSW_DEV_NOOP_LN=1" "MPSW_DEV_NOOP_ATTN=1" "MPSW_DEV_NOOP_LN=1 MPSW_DEV_NOOP_ATTN=1" "MPSW_LN_CLUSTER=1"; do
  for m in opt-13b opt-1.3b opt-125m; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/noop.ndjson 2>&1; done
done
MPSW_LN_CLUSTER=1 MPSW_PARITY_LOG=$O/parity_cluster.ndjson timeout 1500 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_allreduce.py tests/test_gpu_shape_fuzz.py -q -x --tb=short -k "not full_size" > $O/pytest_cluster.txt 2>&1
