#!/bin/bash
set -x
O=gpurun_out/r2e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_SWAP_DEBUG=1 timeout 300 python tools/ce_lib_probe.py 1 4 16 64 > $O/ce_lib_probe.ndjson 2> $O/ce_lib_probe.err
timeout 900 python -m pytest tests/test_gpu_hetero.py tests/test_gpu_swap.py -q --tb=short > $O/pytest_hetero_swap.txt 2>&1
