#!/bin/bash
# Round-2 final evidence (one gpurun call): full GPU tests with parity logs, smoke, bench (clean +
# writeback leg + parity + oracle baseline), reference arm, ncu launch list of the bench command,
# ncu --set full of the tcgen05 GEMM in the OPT-13B forward (M = 2) and of the reduce-scatter
# all-reduce, serving traces (cfg1, cfg2, cfg2-t1 x3, cfg4-analog CV x3 seeds, hetero victim
# policy 0/1, cfg4-slice), AUTO table.
set -x
O=gpurun_out/final2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 2700 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --wb-steps 0 --n-models 2 > $O/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o $O/prof_tc \
    python tools/fwd_one.py opt-13b 1 2 2 2 > $O/prof_tc.log 2>&1
MPSW_RS_MIN_BYTES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_ln -s 64 -c 2 -f -o $O/prof_ln_rs \
    python tools/fwd_tp.py opt-30b 8 32 8 > $O/prof_ln_rs.log 2>&1
for f in prof_tc prof_ln_rs; do
  ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
  ncu -i $O/$f.ncu-rep --page details --csv > $O/${f}_details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
timeout 300 python tools/serve_trace.py cfg1 --out $O/serve.ndjson > /dev/null 2>&1
timeout 400 python tools/serve_trace.py cfg2 --out $O/serve.ndjson > /dev/null 2>&1
for seed in 0 1 2; do
  timeout 300 python tools/serve_trace.py cfg2-t1 --seed $seed --out $O/serve.ndjson > /dev/null 2>&1
  for cv in 0.25 1 4; do timeout 300 python tools/serve_trace.py cfg4-analog --cv $cv --seed $seed --out $O/serve.ndjson > /dev/null 2>&1; done
done
for vp in 0 1; do timeout 900 python tools/serve_trace.py hetero --victim-policy $vp --out $O/serve.ndjson > /dev/null 2>&1; done
timeout 1500 python tools/serve_trace.py cfg4-slice --check-logits 1 --out $O/serve.ndjson > /dev/null 2>&1
timeout 1800 python tools/auto_table.py --out $O/auto_table.ndjson > $O/auto_table.log 2>&1
