O=gpurun_out/g2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_forward.py -q -x > $O/pytest.txt 2>&1
timeout 600 python tools/gemm_tune.py ext > $O/tune.txt 2>&1
timeout 600 python tools/fwd_bench.py > $O/fwd.txt 2>&1
