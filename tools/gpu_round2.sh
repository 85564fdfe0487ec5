#!/bin/bash
# Round-2 evidence run: build, full GPU tests (parity log), smoke, default bench (clean + writeback
# leg + parity + oracle baseline), reference arm, driver-form --gpus 2 bench on one GPU.
set -x
O=gpurun_out/r2a
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 2400 python -m pytest tests -m gpu -q -rf --tb=short > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python tools/serve_trace.py cfg1 --out $O/serve.ndjson > $O/serve_cfg1.log 2>&1
timeout 1500 python tools/serve_trace.py cfg4-slice --check-logits 1 --out $O/serve.ndjson > $O/serve_cfg4slice.log 2>&1
timeout 200 python tools/serve_trace.py cfg4 --out $O/serve.ndjson > $O/serve_cfg4.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$t.txt 2>&1
done
