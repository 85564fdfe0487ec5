#!/bin/bash
# Quick health round: build, GPU tests, smoke, default bench.
set -x
O=gpurun_out/base
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
nproc > $O/host.txt; lscpu >> $O/host.txt; free -g >> $O/host.txt; ulimit -l >> $O/host.txt; which nsys >> $O/host.txt 2>&1; nvidia-smi topo -m >> $O/host.txt 2>&1
