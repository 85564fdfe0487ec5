"""Measures the copy-engine vs zero-copy swap-in per shard-size bucket, alone and under a
concurrent forward, for the AUTO swap mode's table (north star: "the faster of the two kept per
shard size"; csrc/swap.cpp kAutoTable). Prints NDJSON rows and a summary line per bucket.

Per bucket (1 MiB .. 1 GiB, x4 steps): two OPT-shaped models A, B of ~that shard size alternate
in one range (explicit swap_out A / swap_in B, clean eviction), device time of the load entry
from its CUDA events; "busy" repeats it while a third model (OPT-1.3B, resident in its own range)
serves back-to-back batches of 8 x 8 tokens on the compute stream, so the zero-copy kernel
competes with the forward for SMs (and the forward with the swap for HBM).

usage: python tools/auto_table.py [--out FILE] [--reps 7]"""
import argparse
import json
import os
import statistics
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_13835_b200 import mpsw as M  # noqa: E402
from synth import opt_dims, request_tokens  # noqa: E402
from synth.models import OptDims  # noqa: E402
from tools.sweep_cfg5 import dims_for  # noqa: E402


def dmax(a, b):
    return OptDims(max(a.n_layers, b.n_layers), max(a.hidden, b.hidden), max(a.heads, b.heads), max(a.ffn, b.ffn),
                   vocab=max(a.vocab, b.vocab), max_pos=max(a.max_pos, b.max_pos))


def raw_ce(nbytes, reps):
    """The copy engine alone (torch, pinned -> device, CUDA events): DMA cost without the library."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=0)
    s = torch.cuda.Stream()
    ts = []
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[2:]), min(ts[2:])


def run(target, mode, zc_ctas, busy, reps):
    d = dims_for(target)
    big = opt_dims("opt-1.3b")
    S = M.shard_layout(d, 1)[1]
    Sb = M.shard_layout(big, 1)[1]
    rnd = lambda x: (x + 4095) // 4096 * 4096
    with M.Ctx(device_ids=(0,), budget=rnd(S) + (rnd(Sb) if busy else 0), swap_mode=mode, zc_ctas=zc_ctas,
               writeback=0, max_batch=8, max_tokens=8, max_dims=dmax(big, d) if busy else None) as ctx:
        if busy:
            c = ctx.register_model(big)
            ctx.synth_fill(c, 3)
            ctx.wait(ctx.swap_in(c))
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.synth_fill(a, 1)
        ctx.synth_fill(b, 2)
        stop = threading.Event()

        def serve():
            i = 0
            while not stop.is_set():
                rids = [ctx.request(c, request_tokens(9, 0, i * 8 + j, 8, big.vocab))[0] for j in range(8)]
                for r in rids:
                    ctx.wait_request(r, 600)
                i += 1

        th = threading.Thread(target=serve, daemon=True) if busy else None
        if th:
            th.start()
        ctx.wait(ctx.swap_in(a))
        cur, other = a, b
        dev = []
        for _ in range(reps + 2):
            ctx.wait(ctx.swap_out(cur))
            t = ctx.swap_in(other)
            ctx.wait(t)
            dev.append(ctx.entry_gpu_ms(t)[2][0])
            cur, other = other, cur
        stop.set()
        if th:
            th.join()
    dev = dev[2:]
    med = statistics.median(dev)
    return {"target": target, "S_r": S, "mode": {1: "copy_engine", 2: "zero_copy"}[mode], "zc_ctas": zc_ctas,
            "busy": busy, "dev_ms_median": med, "dev_ms_min": min(dev), "GBps": S / (med / 1e3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    rows = []
    for p in range(20, 31, 2):
        target = 1 << p
        for busy in (False, True):
            cand = []
            for mode, zc in ((1, 0), (2, 32), (2, 148)):
                r = run(target, mode, zc, busy, args.reps)
                print(json.dumps(r), flush=True)
                rows.append(r)
                cand.append(r)
            best = min(cand, key=lambda x: x["dev_ms_median"])
            if not busy:
                med, mn = raw_ce(cand[0]["S_r"], args.reps)
                print(json.dumps({"target": target, "raw_ce_torch_ms_median": med, "raw_ce_torch_ms_min": mn,
                                  "raw_ce_GBps": cand[0]["S_r"] / (med / 1e3) / 1e9}), flush=True)
            s = {"summary": True, "target": target, "busy": busy, "winner": best["mode"], "zc_ctas": best["zc_ctas"],
                 "ce_ms": cand[0]["dev_ms_median"], "zc32_ms": cand[1]["dev_ms_median"], "zc148_ms": cand[2]["dev_ms_median"]}
            print(json.dumps(s), flush=True)
            rows.append(s)
    if args.out:
        with open(args.out, "a") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
