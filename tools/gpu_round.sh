#!/bin/bash
# One GPU round: build, GPU tests, smoke, bench N=1, N=2 code path on one GPU (numbers meaningless).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -rf --tb=short -k "not full_size" > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
MPSW_BENCH_DEVICE0=1 MPSW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 1 --model opt-1.3b \
   > gpurun_out/bench_n2_dev0.json 2> gpurun_out/bench_n2_dev0.err
