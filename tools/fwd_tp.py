"""Forward device time of one resident model on TP virtual ranks sharing cuda:0 (dev tool: the
all-reduce reads go to local HBM, not NVLink, so this checks the code path, not TP scaling).
usage: python tools/fwd_tp.py model tp B L"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims, request_tokens
from oracle import layout

name, tp, B, L = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
d = opt_dims(name)
S = layout.shard_bytes(d, tp)
with M.Ctx(device_ids=(0,) * tp, budget=S + 4096, max_batch=B, max_tokens=L) as ctx:
    m = ctx.register_model(d)
    ctx.synth_fill(m, 1)
    ctx.wait(ctx.swap_in(m))
    toks = [request_tokens(0, 0, i, L, d.vocab) for i in range(B)]
    for it in range(8):
        if it == 3:
            s0 = ctx.stats()
        rids = [ctx.request(m, t)[0] for t in toks]
        for r in rids:
            ctx.wait_request(r, 120)
    s1 = ctx.stats()
    n = s1["fwd_gpu_n"] - s0["fwd_gpu_n"]
    import os
    print(json.dumps({"model": name, "tp": tp, "B": B, "L": L, "rs_min_bytes": os.environ.get("MPSW_RS_MIN_BYTES"),
                      "fwd_ms_device": (s1["fwd_gpu_us_sum"] - s0["fwd_gpu_us_sum"]) / 1e3 / max(1, n)}), flush=True)
