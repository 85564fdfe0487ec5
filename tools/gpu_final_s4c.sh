#!/bin/bash
# Full GPU suite and smoke on the final session-4 tree (after the fuzz-test changes).
set -x
O=${OUT:-gpurun_out/final_s4c}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 1300 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
