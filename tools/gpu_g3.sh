#!/bin/bash
# ncu captures (with source) of the tcgen05 GEMM after the fix-up rework + forward bench.
O=gpurun_out/g3; mkdir -p $O
i=0
for s in "256 5120 20480" "256 15360 5120" "2 15360 5120"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -f -o $O/tc_$i \
     python tools/gemm_one.py $s 2 1 > $O/tc_$i.log 2>&1
done
timeout 600 python tools/fwd_bench.py opt-13b tc > $O/fwd13.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-1.3b tc > $O/fwd13b.txt 2>&1
