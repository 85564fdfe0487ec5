"""Swap-path probe through the C-ABI (development tool): swap-in GB/s per mode and size, and the
paired (writeback) swap window via alternating blocking requests."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims
from oracle import layout

res = []
for name in sys.argv[1:] or ["small", "opt-125m", "opt-1.3b"]:
    d = opt_dims(name)
    S = layout.shard_bytes(d, 1)
    for mode, ctas in [(1, 0), (2, 16), (2, 32), (2, 64), (2, 148)]:
        for wb in (1, 0):
            with M.Ctx(device_ids=(0,), budget=S + (2 << 20), swap_mode=mode, zc_ctas=ctas, writeback=wb,
                       max_batch=1, max_tokens=2) as ctx:
                a, b = ctx.register_model(d), ctx.register_model(d)
                ctx.synth_fill(a, 1); ctx.synth_fill(b, 2)
                ctx.wait(ctx.swap_in(a))
                lat, gms = [], []
                for i in range(6):
                    ctx.wait(ctx.swap_out(a if i % 2 == 0 else b))
                    t = ctx.swap_in(b if i % 2 == 0 else a)
                    ts, td = ctx.wait(t)
                    lat.append(td[0] - ts)
                    gms.append(ctx.entry_gpu_ms(t)[2][0])
                # paired swaps through requests (alternating blocking)
                tok = np.array([5, 7], np.int32)
                pl = []
                for i in range(6):
                    t0 = time.perf_counter()
                    rid, _ = ctx.request(a if i % 2 == 0 else b, tok)
                    ctx.wait_request(rid, 60)
                    pl.append(time.perf_counter() - t0)
                r = dict(model=name, S=S, mode=mode, ctas=ctas, writeback=wb,
                         swapin_ms_med=1e3 * float(np.median(lat[1:])), gpu_ms_med=float(np.median(gms[1:])),
                         GBps_host=S / np.median(lat[1:]) / 1e9, GBps_gpu=S / (np.median(gms[1:]) / 1e3) / 1e9,
                         request_swap_ms_med=1e3 * float(np.median(pl[1:])))
                print(json.dumps(r), flush=True)
                res.append(r)
json.dump(res, open("gpurun_out/swap_probe.json", "w"), indent=1)
