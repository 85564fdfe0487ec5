#!/bin/bash
O=gpurun_out/g8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --writeback 1 > $O/bench_wb.json 2> $O/bench_wb.err
