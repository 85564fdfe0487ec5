#!/bin/bash
# Large-M GEMM diagnosis: single vs CTA-pair at M = 64 / 128 / 256 (OPT-13B shapes), per-CTA phase
# stamps, and one ncu --set full capture of fc1 at M = 256 in each mode.
set -x
O=gpurun_out/r2o
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for p in 0 1; do
  for m in 64 128 256; do
    for s in "15360 5120" "5120 5120" "20480 5120" "5120 20480"; do
      echo "pair=$p $(MPSW_TC_PAIR=$p python tools/gemm_one.py $m $s 2 20)" >> $O/gemm.txt
    done
  done
  MPSW_TC_PAIR=$p timeout 600 python tools/tc_trace.py run $O/trace_pair$p.ndjson
  python tools/tc_trace.py show $O/trace_pair$p.ndjson > $O/trace_pair$p.txt 2>&1
done
for p in 0 1; do
  MPSW_TC_PAIR=$p timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $O/fc1_m256_pair$p python tools/gemm_one.py 256 20480 5120 2 1 > $O/ncu_pair$p.log 2>&1
  MPSW_TC_PAIR=$p timeout 900 ncu --set full --clock-control none -k regex:tc_fixup -s 3 -c 1 -o $O/fixup_m256_pair$p python tools/gemm_one.py 256 20480 5120 2 1 > $O/ncu_fix_pair$p.log 2>&1
done
