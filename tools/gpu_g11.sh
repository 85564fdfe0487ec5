#!/bin/bash
O=gpurun_out/g11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
