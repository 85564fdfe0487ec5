#!/bin/bash
# Round-2 session-4 check of HEAD on a B200: full GPU tests with parity logs, smoke, bench and
# the reference arm (the code last changed after session 3's evidence run: the cluster reduce_ln
# removal).
set -x
O=${OUT:-gpurun_out/final_s4}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 2000 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
