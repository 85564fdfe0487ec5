#!/bin/bash
set -x
O=gpurun_out/r2g
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --no-cpu-baseline --no-parity > $O/bench_default.json 2> $O/bench_default.err
MPSW_NO_FLUSH=1 timeout 900 python bench.py --no-cpu-baseline --no-parity > $O/bench_noflush.json 2> $O/bench_noflush.err
MPSW_GRAPHS=0 timeout 900 python bench.py --no-cpu-baseline --no-parity > $O/bench_nographs.json 2> $O/bench_nographs.err
timeout 1200 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_engine_fuzz.py tests/test_gpu_graphs.py -q --tb=short > $O/pytest_debug.txt 2>&1
