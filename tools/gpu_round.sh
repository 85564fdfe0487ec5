#!/bin/bash
# One GPU round: build, GPU tests, smoke, bench, ncu launch list + tcgen05 GEMM capture.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -rf --tb=short > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --n-models 2 > gpurun_out/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o gpurun_out/prof_tc \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --n-models 2 > gpurun_out/prof_tc.log 2>&1
