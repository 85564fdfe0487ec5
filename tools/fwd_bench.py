"""Steady-state forward timing through the C-ABI (dev tool): one resident model, back-to-back
blocking batches, per-batch device time from the library's CUDA events.
impl: 0 auto (= 2 for bf16), 1 SIMT, 2 per-op tcgen05.
usage: python tools/fwd_bench.py [model=opt-13b] [tc | impls=0,2] [shapes=1x2,4x8]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims, request_tokens
from oracle import layout

name = sys.argv[1] if len(sys.argv) > 1 else "opt-13b"
d = opt_dims(name)
S = layout.shard_bytes(d, 1)
impls = (1, 2)
shapes = [(1, 2), (8, 8), (32, 8)]
for a in sys.argv[2:]:
    if a == "tc":
        impls = (2,)
    elif a.startswith("impls="):
        impls = tuple(int(x) for x in a[6:].split(","))
    elif a.startswith("shapes="):
        shapes = [tuple(int(v) for v in x.split("x")) for x in a[7:].split(",")]
for B, L in shapes:
    for impl in impls:
        with M.Ctx(device_ids=(0,), budget=S + 4096, max_batch=B, max_tokens=L, gemm_impl=impl) as ctx:
            m = ctx.register_model(d)
            ctx.synth_fill(m, 1)
            ctx.wait(ctx.swap_in(m))
            toks = [request_tokens(0, 0, i, L, d.vocab) for i in range(B)]
            outs = [[np.empty(d.vocab, np.float32) for _ in range(B)] for _ in range(2)]

            def submit(k):
                return [ctx.request(m, t, o)[0] for t, o in zip(toks, outs[k % 2])]

            # pipelined: round i+1 is queued while round i's batch runs, so after the first round
            # every batch holds exactly B requests (D = 1 dynamic batching)
            warm, n = 3, 10
            pending = submit(0)
            for it in range(warm + n):
                nxt = submit(it + 1)
                for r in pending:
                    ctx.wait_request(r, 60)
                pending = nxt
                if it == warm - 1:
                    s0 = ctx.stats()
                    t0 = time.perf_counter()
            for r in pending:
                ctx.wait_request(r, 60)
            wall = (time.perf_counter() - t0) / n
            s1 = ctx.stats()
            nb = s1["fwd_gpu_n"] - s0["fwd_gpu_n"]
            ms = (s1["fwd_gpu_us_sum"] - s0["fwd_gpu_us_sum"]) / 1e3 / max(1, nb)
            import os
            print(json.dumps({"graphs": os.environ.get("MPSW_GRAPHS", "1"), "pair": os.environ.get("MPSW_TC_PAIR", "0"), "model": name, "B": B, "L": L, "impl": ["auto", "simt", "tcgen05"][impl], "batches": nb, "batch_rows": B * L,
                              "fwd_ms_device": ms, "GBps": S / (ms / 1e3) / 1e9, "wall_ms_per_round": wall * 1e3}),
                  flush=True)
