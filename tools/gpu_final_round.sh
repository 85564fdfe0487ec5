#!/bin/bash
# Full evidence round (one gpurun call): tests, smoke, bench (clean / writeback / reference arm),
# launch list, ncu captures of the tcgen05 GEMM (M = 2 in the forward, M = 256 alone), per-CTA
# phase trace, forward bench (OPT-13B, OPT-1.3B), GEMM sweep, serving traces (3 seeds, hetero
# with prefetch off / on), cfg5 sweep.
set -x
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --writeback 1 --no-cpu-baseline > $O/bench_wb.json 2> $O/bench_wb.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --n-models 2 > $O/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o $O/prof_tc \
    python tools/fwd_one.py opt-13b 1 2 2 2 > $O/prof_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -f -o $O/prof_tc_m256 \
    python tools/gemm_one.py 256 5120 20480 2 1 > $O/prof_tc_m256.log 2>&1
rm -f $O/tc_trace.ndjson
timeout 600 python tools/tc_trace.py run $O/tc_trace.ndjson > /dev/null 2>&1
python tools/tc_trace.py show $O/tc_trace.ndjson > $O/tc_trace.txt 2>&1
timeout 900 python tools/fwd_bench.py opt-13b > $O/fwd_bench.txt 2>&1
timeout 600 python tools/fwd_bench.py opt-1.3b tc >> $O/fwd_bench.txt 2>&1
timeout 900 python tools/gemm_tune.py grid > $O/gemm_tune.txt 2>&1
timeout 1500 python tools/gemm_tune.py align > $O/gemm_align.txt 2>&1
for cfg in "opt-13b 2 1 2" "opt-13b 8 1 2" "opt-1.3b 8 1 2"; do timeout 600 python tools/fwd_tp.py $cfg >> $O/fwd_tp.txt 2>&1; done
rm -f $O/serve.ndjson
timeout 300 python tools/serve_trace.py cfg1 --out $O/serve.ndjson
for seed in 0 1 2; do
  timeout 300 python tools/serve_trace.py cfg2-t1 --seed $seed --out $O/serve.ndjson
  for cv in 0.25 1 4; do timeout 300 python tools/serve_trace.py cfg4-analog --cv $cv --seed $seed --out $O/serve.ndjson; done
done
timeout 300 python tools/serve_trace.py cfg2 --out $O/serve.ndjson
for pf in 0 1; do
  timeout 900 python tools/serve_trace.py hetero --prefetch $pf --out $O/serve.ndjson
done
timeout 1500 python tools/sweep_cfg5.py --out $O/cfg5.ndjson > $O/cfg5.log 2>&1
