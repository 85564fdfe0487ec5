#!/bin/bash
# Forward at serving batch sizes: split A/B, fixup stand-in, launch lists at M = 64 / 256.
set -x
O=gpurun_out/r2t
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for v in "MPSW_TC_SPLIT=1" "MPSW_TC_SPLIT=2" "MPSW_TC_SPLIT=2 MPSW_DEV_NOOP_FIXUP=1" "MPSW_TC_SPLIT=2 MPSW_DEV_NOOP_LN=1"; do
  for m in opt-13b opt-1.3b; do env $v timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8,16x8,32x8 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/fwd.ndjson 2>&1; done
done
for bl in "32 8" "8 8"; do
  set -- $bl
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/launches_m$(( $1 * $2 )).csv python tools/fwd_one.py opt-13b $1 $2 2 2 > $O/ncu_m$(( $1 * $2 )).log 2>&1
  python tools/ncu_summary.py $O/launches_m$(( $1 * $2 )).csv > $O/launches_m$(( $1 * $2 ))_summary.ndjson 2>&1
done
