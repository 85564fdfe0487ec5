#!/bin/bash
set -x
O=gpurun_out/r2z
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
GT_M=2,16,64,128,256 timeout 2400 python tools/gemm_tune.py knobs2 > $O/gemm_knobs2.ndjson 2>&1
for v in "MPSW_TC_EXT_MIN=64" "MPSW_DEV_NOOP_FIXUP=1"; do
  for m in opt-13b opt-1.3b; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,16x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/fwd.ndjson 2>&1; done
done
