#!/bin/bash
# cfg4 slice: 3 seeds (p99 pooled over ~800 requests), 16 sampled logits vs the fp64 / emulating
# oracle on seed 0, resident shards vs golden hashes.
set -x
O=gpurun_out/r2l
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 3600 python tools/serve_trace.py cfg4-slice --seed 0 --check-logits 16 --out $O/serve.ndjson > $O/s0.log 2>&1
for s in 1 2; do timeout 1200 python tools/serve_trace.py cfg4-slice --seed $s --check-logits 0 --out $O/serve.ndjson > $O/s$s.log 2>&1; done
