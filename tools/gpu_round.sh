#!/bin/bash
# One GPU round: build, GPU tests (incl. full size), smoke, bench, ncu launch list + tcgen05 GEMM capture.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -rf --tb=short > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --writeback 1 --no-cpu-baseline > gpurun_out/bench_wb.json 2> gpurun_out/bench_wb.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --n-models 2 > gpurun_out/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o gpurun_out/prof_tc \
    python tools/fwd_one.py opt-13b 1 2 2 2 > gpurun_out/prof_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_ln -s 40 -c 1 -f -o gpurun_out/prof_ln \
    python tools/fwd_one.py opt-13b 1 2 2 2 > gpurun_out/prof_ln.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zero_copy -c 1 -f -o gpurun_out/prof_zc \
    python tools/zc_one.py > gpurun_out/prof_zc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:checksum -c 1 -f -o gpurun_out/prof_ck \
    python -c "
import sys; sys.path.insert(0,'.')
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims
from oracle import layout
d=opt_dims('opt-1.3b'); S=layout.shard_bytes(d,1)
with M.Ctx(device_ids=(0,), budget=S+4096) as c:
    m=c.register_model(d); c.synth_fill(m,1); c.wait(c.swap_in(m)); print(hex(c.checksum(m,0)))
" > gpurun_out/prof_ck.log 2>&1
