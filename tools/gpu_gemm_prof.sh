#!/bin/bash
# GPU round: test suite on HEAD + ncu captures of the tcgen05 GEMM at M = 64 / 256.
O=gpurun_out/gprof; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
for s in "256 15360 5120" "256 5120 20480" "64 15360 5120" "64 5120 20480"; do
  timeout 120 python tools/gemm_one.py $s 2 10 >> $O/gemm_one.txt 2>&1
done
i=0
for s in "256 15360 5120" "256 5120 20480" "64 5120 20480"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -f -o $O/tc_$i \
     python tools/gemm_one.py $s 2 1 > $O/tc_$i.log 2>&1
done
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
