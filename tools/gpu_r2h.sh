#!/bin/bash
# Knob sweep of the tcgen05 split / ring with CUDA graphs on (forward device time).
set -x
O=gpurun_out/r2h
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for mu in 4 8 16; do for kb in 88 104 112; do for m in opt-13b opt-1.3b; do
  MPSW_TC_MINU=$mu MPSW_TC_SMEM_KB=$kb timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8 | sed "s/^{/{\"minu\": $mu, \"smem_kb\": $kb, /" >> $O/knobs.ndjson 2>&1
done; done; done
for a in 0 1; do for m in opt-13b opt-1.3b; do
  MPSW_TC_ALIGN=$a timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,8x8 | sed "s/^{/{\"align\": $a, /" >> $O/knobs.ndjson 2>&1
done; done
