set -x
O=gpurun_out/s3w; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --writeback 1 --no-cpu-baseline > $O/bench_wb.json 2> $O/bench_wb.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --n-models 2 > $O/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o $O/prof_tc \
    python tools/fwd_one.py opt-13b 1 2 2 2 > $O/prof_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_ln -s 40 -c 1 -f -o $O/prof_ln \
    python tools/fwd_one.py opt-13b 1 2 2 2 > $O/prof_ln.log 2>&1
