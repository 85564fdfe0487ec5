#!/bin/bash
set -x
O=gpurun_out/r2j
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for a in 0 1; do
  MPSW_TC_ALIGN60=$a timeout 600 python tools/gemm_shapes_ab.py 3584x7168 7168x3584 5120x5120 >> $O/ab.ndjson 2>&1
  MPSW_TC_ALIGN60=$a timeout 900 python tools/fwd_tp.py opt-30b 8 1 8 >> $O/fwd_tp.ndjson 2>&1
  MPSW_TC_ALIGN60=$a timeout 900 python tools/fwd_tp.py opt-30b 8 32 8 >> $O/fwd_tp.ndjson 2>&1
done
