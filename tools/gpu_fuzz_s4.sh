#!/bin/bash
# Session-4 extended shape-fuzz campaign on a B200: the default seeds of tests/test_gpu_shape_fuzz.py
# (incl. the new large-batch cases: one batch of up to 640 rows), then MPSW_FUZZ_SEEDS=16:80, i.e.
# 64 more seeded shapes per test (bf16 vs the emulating oracle, fp32 vs exact, large batches).
set -x
O=${OUT:-gpurun_out/fuzz_s4}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity_default.ndjson timeout 900 python -m pytest tests/test_gpu_shape_fuzz.py -m gpu -q -rf --tb=short > $O/pytest_default.txt 2>&1
MPSW_FUZZ_SEEDS=16:80 MPSW_PARITY_LOG=$O/parity_ext.ndjson timeout 2400 python -m pytest tests/test_gpu_shape_fuzz.py -m gpu -q -rf --tb=short > $O/pytest_ext.txt 2>&1
