O=gpurun_out/s3z; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python tools/fwd_bench.py opt-13b tc > $O/fwd_bench.txt 2>&1
MPSW_TC_ALIGN=0 timeout 900 python tools/fwd_bench.py opt-13b impls=2 shapes=32x8 > $O/fwd_noalign_256.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-1.3b tc >> $O/fwd_bench.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-125m impls=2 shapes=1x2,8x8,32x8 >> $O/fwd_bench.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
