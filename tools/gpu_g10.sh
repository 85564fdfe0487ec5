#!/bin/bash
O=gpurun_out/g10; mkdir -p $O; rm -f $O/serve.ndjson
timeout 900 python -m pytest tests/test_gpu_hetero.py tests/test_gpu_engine.py tests/test_gpu_swap.py -q -x > $O/pytest.txt 2>&1
for pf in 0 1; do
  for seed in 0 1; do
    timeout 900 python tools/serve_trace.py hetero --seed $seed --prefetch $pf --check-logits 0 --out $O/serve.ndjson > $O/hetero_${pf}_${seed}.log 2>&1
  done
done
