#!/bin/bash
# Decoupled weight / token rings, staged partial stores: correctness, then the knob sweep.
set -x
O=gpurun_out/r2s
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm.txt 2>&1
MPSW_TC_STAGE_MIN=16 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm_stage.txt 2>&1
MPSW_TC_VW=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short > $O/pytest_gemm_vw1.txt 2>&1
GT_M=2,16,64,128,256 timeout 1500 python tools/gemm_tune.py rings > $O/gemm_rings.ndjson 2>&1
