"""A few forwards of one resident model (target for ncu launch lists of the forward)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims, request_tokens
from oracle import layout

name = sys.argv[1] if len(sys.argv) > 1 else "opt-13b"
B, L, impl, n = (int(x) for x in (sys.argv[2:6] if len(sys.argv) > 5 else (1, 2, 2, 3)))
d = opt_dims(name)
S = layout.shard_bytes(d, 1)
with M.Ctx(device_ids=(0,), budget=S + 4096, max_batch=B, max_tokens=L, gemm_impl=impl) as ctx:
    m = ctx.register_model(d)
    ctx.synth_fill(m, 1)
    ctx.wait(ctx.swap_in(m))
    toks = [request_tokens(0, 0, i, L, d.vocab) for i in range(B)]
    for it in range(n):
        rids = [ctx.request(m, t)[0] for t in toks]
        for r in rids:
            ctx.wait_request(r, 120)
    st = ctx.stats()
    print("fwd_ms", st["fwd_gpu_us_sum"] / 1e3 / st["fwd_gpu_n"])
