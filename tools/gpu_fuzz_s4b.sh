#!/bin/bash
# Session-4 larger fuzz campaign: shape fuzz seeds 80:600 (bf16, fp32, large batches), engine
# serving fuzz seeds 8:40 (plain, pipeline, fp32; the long run once).
set -x
O=${OUT:-gpurun_out/fuzz_s4b}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_FUZZ_SEEDS=80:600 MPSW_PARITY_LOG=$O/parity_shape.ndjson timeout 1000 python -m pytest tests/test_gpu_shape_fuzz.py -m gpu -q -rf --tb=short > $O/pytest_shape.txt 2>&1
MPSW_FUZZ_SEEDS=8:40 MPSW_PARITY_LOG=$O/parity_engine.ndjson timeout 1300 python -m pytest tests/test_gpu_engine_fuzz.py -m gpu -q -rf --tb=short > $O/pytest_engine.txt 2>&1
