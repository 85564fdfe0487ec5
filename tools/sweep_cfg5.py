"""BASELINE cfg5: per-rank shard swap bandwidth, 1 MB .. 8 GB, through the C-ABI (one GPU).

For each target size a synthetic OPT-shaped model whose per-rank arena is ~that size is
registered twice (budget = one slot); swap-in device time (CUDA events on the H2D stream) and
host-observed latency are measured for the copy-engine and zero-copy paths, clean eviction and
writeback (paired chunk pipeline); with writeback also the D2H of the swap-out alone. Also the paper's alpha-beta ablation: T separate
per-tensor copies vs one flat copy of the same bytes (torch copy engine), fitting alpha.

usage: python tools/sweep_cfg5.py [--max-gb 8] [--out gpurun_out/cfg5.ndjson]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_13835_b200 import mpsw as M
from synth.models import OptDims
from synth import opt_dims
from oracle import layout


def dims_for(target):
    """An OPT-shaped model (valid for the kernels) whose TP1 arena is close to `target` bytes."""
    for h, L in reversed([(128, 1), (256, 1), (512, 1), (1024, 1), (1024, 4), (2048, 4), (4096, 4), (4096, 12),
                          (4096, 20)]):
        per_layer = 2 * (12 * h * h + 13 * h)
        fixed = 2 * (18 * h + 2 * h)
        rem = target - L * per_layer - fixed
        if L * per_layer <= 0.75 * target and rem >= 2 * h * 64:
            V = max(64, (rem // (2 * h)) // 8 * 8)
            return OptDims(L, h, max(1, h // 64), 4 * h, vocab=V, max_pos=16)
    return OptDims(1, 128, 2, 512, vocab=64, max_pos=16)


def measure(d, mode, writeback, zc_ctas=0, reps=5):
    S = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=(S + 4095) // 4096 * 4096, swap_mode=mode, writeback=writeback,
               zc_ctas=zc_ctas, max_batch=1, max_tokens=2) as ctx:
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.synth_fill(a, 1)
        ctx.synth_fill(b, 2)
        ctx.wait(ctx.swap_in(a))
        dev, host, d2h = [], [], []
        cur, other = a, b
        for _ in range(reps + 1):
            to = ctx.swap_out(cur)
            ctx.wait(to)
            d2h.append(ctx.entry_gpu_ms(to)[2][0])     # D2H alone (writeback) / gate only (clean)
            t = ctx.swap_in(other)
            ts, td = ctx.wait(t)
            dev.append(ctx.entry_gpu_ms(t)[2][0])
            host.append((td[0] - ts) * 1e3)
            cur, other = other, cur
        # paired (offload + load in one step) via a request: the paper's swap window
        pair = []
        tok = np.array([1, 2], np.int32)
        for i in range(reps):
            t0 = time.perf_counter()
            rid, _ = ctx.request(a if i % 2 == 0 else b, tok)
            ctx.wait_request(rid, 120)
            pair.append((time.perf_counter() - t0) * 1e3)
    dev, host, d2h = dev[1:], host[1:], d2h[1:]
    return S, float(np.median(dev)), float(np.median(host)), float(np.median(pair[1:])), float(np.median(d2h))


def alpha_ablation(n_tensors_list=(1, 196, 644, 2000), total=1 << 30):
    """Per-message cost of the copy engine: T copies of total/T bytes vs one copy."""
    import torch
    h = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    dv = torch.empty(total, dtype=torch.uint8, device=0)
    s = torch.cuda.Stream()
    out = []
    for T in n_tensors_list:
        step = total // T // 256 * 256
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for i in range(T):
                    dv[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
                e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out.append({"T": T, "bytes": step * T, "ms": best, "GBps": step * T / (best / 1e3) / 1e9})
    # alpha = (t_T - t_1 * bytes_T / bytes_1) / (T - 1) for the largest T
    t1 = out[0]["ms"] / out[0]["bytes"]
    for o in out[1:]:
        o["alpha_us"] = (o["ms"] - t1 * o["bytes"]) / (o["T"] - 1) * 1e3
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gb", type=float, default=8)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    sizes = [1 << p for p in range(20, 34) if (1 << p) <= args.max_gb * (1 << 30)]
    for target in sizes:
        d = dims_for(target)
        for mode, zc, wb in [(1, 0, 0), (2, 32, 0), (2, 148, 0), (1, 0, 1)]:
            if mode == 2 and target > (1 << 31):
                continue
            S, dev_ms, host_ms, pair_ms, d2h_ms = measure(d, mode, wb, zc)
            r = {"target": target, "S_r": S, "mode": ["", "copy_engine", "zero_copy"][mode], "zc_ctas": zc,
                 "writeback": wb, "swapin_dev_ms": dev_ms, "swapin_host_ms": host_ms,
                 "GBps_dev": S / (dev_ms / 1e3) / 1e9, "GBps_host": S / (host_ms / 1e3) / 1e9,
                 "frac_of_64": S / (dev_ms / 1e3) / 1e9 / 64.0, "request_with_swap_ms": pair_ms}
            if wb:
                r["swapout_dev_ms"] = d2h_ms
                r["GBps_d2h"] = S / (d2h_ms / 1e3) / 1e9
            print(json.dumps(r), flush=True)
            rows.append(r)
    ab = alpha_ablation()
    print(json.dumps({"alpha_ablation": ab}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
            f.write(json.dumps({"alpha_ablation": ab}) + "\n")


if __name__ == "__main__":
    main()
