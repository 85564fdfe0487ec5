#!/bin/bash
set -x
O=gpurun_out/r2m
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for v in "" "MPSW_DEV_NOOP_LN=1" "MPSW_DEV_NOOP_ATTN=1" "MPSW_DEV_NOOP_LN=1 MPSW_DEV_NOOP_ATTN=1"; do
  for m in opt-13b opt-1.3b opt-125m; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2 | sed "s/^{/{\"noop\": \"$v\", /" >> $O/noop.ndjson 2>&1; done
done
