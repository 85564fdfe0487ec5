#!/bin/bash
set -x
O=gpurun_out/r2x
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_fixup -s 3 -c 1 -o $O/fixup_m64 python tools/gemm_one.py 64 20480 5120 2 1 > $O/ncu_fix64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_fixup -s 3 -c 1 -o $O/fixup_m256 python tools/gemm_one.py 256 20480 5120 2 1 > $O/ncu_fix256.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gemm64.csv python tools/gemm_one.py 64 20480 5120 2 5 > $O/ncu_l64.log 2>&1
