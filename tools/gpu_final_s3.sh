#!/bin/bash
# Round-2 session-3 evidence on the final GEMM (pair split, L2 hints, 32-bit split math): full GPU
# tests with parity logs, smoke, bench + reference arm, launch list of the bench command, ncu
# --set full of the tcgen05 GEMM at M = 2 and M = 256, forward table, TP8 virtual-rank forward,
# serving traces (cfg1, cfg4-slice with logits), sanitizers.
set -x
O=${OUT:-gpurun_out/final_s3}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 2400 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --wb-steps 0 --n-models 2 > $O/bench_under_ncu.json 2>&1
python tools/ncu_summary.py $O/launches_bench.csv > $O/launches_bench_summary.ndjson 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 120 -c 4 -f -o $O/prof_tc \
    python tools/fwd_one.py opt-13b 1 2 2 2 > $O/prof_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -f -o $O/prof_tc_m256 \
    python tools/gemm_one.py 256 20480 5120 2 1 > $O/prof_tc_m256.log 2>&1
for f in prof_tc prof_tc_m256; do
  ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
  ncu -i $O/$f.ncu-rep --page details --csv > $O/${f}_details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
for m in opt-13b opt-1.3b opt-125m; do timeout 600 python tools/fwd_bench.py $m tc shapes=1x2,2x8,4x8,8x8,16x8,32x8 >> $O/fwd.ndjson 2>&1; done
GT_M=2,16,64,128,256 timeout 600 python tools/gemm_tune.py default > $O/gemm_default.ndjson 2>&1
timeout 900 python tools/fwd_tp.py opt-30b 8 32 8 > $O/fwd_tp8.txt 2>&1
timeout 900 python tools/fwd_tp.py opt-30b 8 1 2 >> $O/fwd_tp8.txt 2>&1
timeout 300 python tools/serve_trace.py cfg1 --out $O/serve.ndjson > /dev/null 2>&1
timeout 1500 python tools/serve_trace.py cfg4-slice --check-logits 2 --out $O/serve.ndjson > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  MPSW_DEBUG_CHECKS=1 MPSW_RS_MIN_BYTES=0 timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$t.txt 2>&1
done
