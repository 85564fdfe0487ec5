#!/bin/bash
O=gpurun_out/g12; mkdir -p $O
timeout 900 python tools/gemm_tune.py smem > $O/tune.txt 2>&1
for kb in 72 104; do
  MPSW_TC_SMEM_KB=$kb timeout 600 python tools/fwd_bench.py opt-13b tc > $O/fwd13_$kb.txt 2>&1
  MPSW_TC_SMEM_KB=$kb timeout 600 python tools/fwd_bench.py opt-1.3b tc > $O/fwd13b_$kb.txt 2>&1
done
