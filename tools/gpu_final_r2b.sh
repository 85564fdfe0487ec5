#!/bin/bash
# Last validation round on the final code: full GPU tests, smoke, bench, reference arm, serving
# traces with logits samples (cfg2 at TP2, cfg4 slice with golden resident checksums),
# compute-sanitizer over every kernel (incl. the stamps, RS all-reduce and graphs).
set -x
O=gpurun_out/final3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 2700 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python tools/serve_trace.py cfg2 --check-logits 8 --out $O/serve.ndjson > /dev/null 2>&1
timeout 1800 python tools/serve_trace.py cfg4-slice --check-logits 2 --out $O/serve.ndjson > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  MPSW_DEBUG_CHECKS=1 MPSW_RS_MIN_BYTES=0 timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$t.txt 2>&1
done
