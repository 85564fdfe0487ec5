#!/bin/bash
set -x
O=gpurun_out/r2k
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1800 python -m pytest tests/test_gpu_layers.py tests/test_gpu_allreduce.py tests/test_gpu_graphs.py -q -rf --tb=short > $O/pytest.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
