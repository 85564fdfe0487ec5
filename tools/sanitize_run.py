"""Short workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of the
library on a small model — zero-copy and copy-engine swaps with writeback, TP 2 forward (GEMMs at
M = 2 and M = 64 with both fix-up paths, attention, fused all-reduce + LN, embedding, lm_head),
checksums — through the C-ABI. Prints one line; sanitizer reports go to stderr/log."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2306_13835_b200 import mpsw as M  # noqa: E402
from synth import opt_dims, request_tokens  # noqa: E402
from oracle import layout  # noqa: E402

d = opt_dims(sys.argv[1] if len(sys.argv) > 1 else "small")
tp = 2
S_ = layout.shard_bytes(d, tp)
for mode in (M.SWAP_ZERO_COPY, M.SWAP_COPY_ENGINE):
    with M.Ctx(device_ids=(0,) * tp, budget=(S_ + 4095) // 4096 * 4096, swap_mode=mode, writeback=1,
               chunk_bytes=1 << 20, max_batch=8, max_tokens=8) as ctx:
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.synth_fill(a, 1)
        ctx.synth_fill(b, 2)
        for m in (a, b, a):
            rids = [ctx.request(m, request_tokens(5, m, i, 8, d.vocab)) for i in range(8)]
            for rid, _ in rids:
                ctx.wait_request(rid, 600)
            rid, _ = ctx.request(m, request_tokens(6, m, 0, 2, d.vocab))
            ctx.wait_request(rid, 600)
        print("checksums", [hex(ctx.checksum(a, r)) for r in range(tp)], "launches", ctx.stats()["kernel_launches"])

# TP 1: the forward is captured into a CUDA graph on a shape's second batch and replayed after
S1 = layout.shard_bytes(d, 1)
with M.Ctx(device_ids=(0,), budget=(S1 + 4095) // 4096 * 4096, max_batch=4, max_tokens=8) as ctx:
    a, b = ctx.register_model(d), ctx.register_model(d)
    ctx.synth_fill(a, 1)
    ctx.synth_fill(b, 2)
    for it in range(4):
        for m in (a, b):
            rid, _ = ctx.request(m, request_tokens(7, m, it, 8, d.vocab))
            ctx.wait_request(rid, 600)
    print("tp1 graphs: launches", ctx.stats()["kernel_launches"])
