#!/bin/bash
# Copy-engine small-swap probe; M>256 chunks; writeback chunk sweep; GPU tests touched by the
# fused-kernel removal.
set -x
O=gpurun_out/r2d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/ce_reg_probe.py > $O/ce_reg_probe.ndjson 2> $O/ce_reg_probe.err
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_gemm.py -q --tb=short > $O/pytest_fwd.txt 2>&1
for ch in 16 32 128; do
  timeout 900 python bench.py --steps 4 --warmup 3 --wb-steps 4 --chunk-mb $ch --no-cpu-baseline --no-parity > $O/bench_chunk$ch.json 2> $O/bench_chunk$ch.err
done
