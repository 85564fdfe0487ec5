"""Open-loop serving runs through the C-ABI (BASELINE cfg1/cfg2/cfg4-shaped traces on one GPU).

For a named preset: registers the models, fills them with the C0 weights, injects a Gamma /
Zipf / alternating trace at its arrival times (real time), and reports nearest-rank p50/p99/mean
request latency, swap counts and swap-in GB/s; then replays the engine's recorded event
log through the oracle scheduler (decisions must be identical) and checks the logits of sampled
requests against the oracle forward when the model is small enough for the oracle.

usage: python tools/serve_trace.py PRESET [--cv 4] [--seed 0] [--out results.json]
presets: cfg1 | cfg2 | cfg2-t1 | cfg4 | cfg4-slice | cfg4-analog | hetero
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
from synth import opt_dims, gamma_trace, alternating_blocking, zipf_rates
from oracle import layout, forward, metrics, scheduler as S

PRESETS = {
    # 2 x OPT-125M, TP1, budget 1 model, 20 alternating blocking requests, L=2
    "cfg1": dict(model="opt-125m", n=2, tp=1, k=1, max_batch=1, L=2, kind="alternating", n_req=20),
    # 4 x OPT-1.3B, TP2 (two virtual ranks on one GPU: they share ONE PCIe link), budget 2 models,
    # uniform rates 2 req/s, Gamma CV=1, 30 s, L=8, max batch 8
    "cfg2": dict(model="opt-1.3b", n=4, tp=2, k=2, max_batch=8, L=8, kind="gamma", rates=[2.0] * 4, duration=30.0),
    "cfg2-t1": dict(model="opt-1.3b", n=4, tp=1, k=2, max_batch=8, L=8, kind="gamma", rates=[2.0] * 4, duration=30.0),
    # cfg4's trace shape (6 models, 4 resident, Zipf lambda_i = 10/i, CV=4, max batch 32, L=8) on
    # OPT-1.3B-shaped models at TP1 (one GPU / 196 GB host cannot hold 6 x OPT-30B)
    "cfg4-analog": dict(model="opt-1.3b", n=6, tp=1, k=4, max_batch=32, L=8, kind="gamma",
                        rates=zipf_rates(6, 10.0, 1.0), duration=30.0),
    # cfg4 at its real shape: 6 x OPT-30B, TP8 (one GPU per rank), 4 resident,
    # Zipf lambda_i = 10/i, Gamma CV=4, max batch 32, L=8, 30 s. Needs 8 GPUs and
    # 6 x 60.2 GB = 361 GB of pinned host memory: the preflight reports what is missing.
    "cfg4": dict(model="opt-30b", n=6, tp=8, k=4, max_batch=32, L=8, kind="gamma",
                 rates=zipf_rates(6, 10.0, 1.0), duration=30.0, gpus=8),
    # the largest slice of cfg4 one B200 + 196 GB host holds: cfg4's per-rank shapes (OPT-30B at
    # TP8, 7.5 GB per rank, 8 virtual ranks on cuda:0 sharing its one PCIe link), 2 models with
    # the first two Zipf rates (10, 5 req/s), budget 1 model, CV=4, max batch 32, L=8, 20 s
    "cfg4-slice": dict(model="opt-30b", n=2, tp=8, k=1, max_batch=32, L=8, kind="gamma",
                       rates=zipf_rates(6, 10.0, 1.0)[:2], duration=20.0, gpus=1, seed0=3000),
    # NEXT-4 (§6): models of different sizes in one 30 GB region (first-fit placement):
    # 1 x OPT-13B, 3 x OPT-1.3B, 2 x OPT-125M; Gamma CV=1, 30 s, L=8, max batch 8
    "hetero": dict(models=["opt-13b", "opt-1.3b", "opt-1.3b", "opt-1.3b", "opt-125m", "opt-125m"], tp=1,
                   budget=30 * 10**9, max_batch=8, L=8, kind="gamma", rates=[0.5, 3.0, 3.0, 3.0, 6.0, 6.0],
                   duration=30.0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("preset")
    ap.add_argument("--cv", type=float, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--check-logits", type=int, default=-1, help="requests to check vs the oracle (-1 = auto)")
    ap.add_argument("--prefetch", type=int, default=0, help="1 = NEXT-3 prefetch policy (reading #29)")
    ap.add_argument("--victim-policy", type=int, default=0, help="1 = minimum-cost window (reading #30)")
    args = ap.parse_args()
    P = dict(PRESETS[args.preset])
    names = P.get("models") or [P["model"]] * P["n"]
    P["n"] = len(names)
    dims = [opt_dims(nm) for nm in names]
    d = max(dims, key=lambda x: layout.shard_bytes(x, P["tp"]))     # workspace dims (max_dims)
    tp = P["tp"]
    S_r = layout.shard_bytes(dims[0], tp)
    sizes_r = [layout.shard_bytes(x, tp) for x in dims]
    cv = args.cv if args.cv is not None else (4.0 if "cfg4" in args.preset else 1.0)
    if P["kind"] == "alternating":
        trace = alternating_blocking(P["n_req"], args.seed, P["L"], min(x.vocab for x in dims))
    else:
        trace = gamma_trace(P["rates"], cv, P["duration"], args.seed, P["L"], min(x.vocab for x in dims))
    budget = P["budget"] if "budget" in P else P["k"] * ((S_r + 4095) // 4096 * 4096)
    # preflight: GPUs and pinned host memory (all ranks' shards of every model) before pinning
    gpus = P.get("gpus", 1)
    host_need = sum(tp * sz for sz in sizes_r)
    avail = None
    for l in open("/proc/meminfo"):
        if l.startswith("MemAvailable:"):
            avail = int(l.split()[1]) * 1024
    import torch
    ngpu = torch.cuda.device_count()
    if ngpu < gpus or (avail is not None and host_need > 0.95 * avail):
        print(json.dumps({"preset": args.preset, "runnable": False, "needs": {
            "gpus": gpus, "gpus_present": ngpu, "pinned_host_bytes": host_need, "host_bytes_available": avail,
            "device_param_bytes_per_gpu": budget, "models": names, "tp": tp}}))
        sys.exit(2)
    device_ids = tuple(range(tp)) if gpus >= tp else (0,) * tp
    res = {"preset": args.preset, "prefetch": args.prefetch, "victim_policy": args.victim_policy, "models": names, "tp": tp, "k": P.get("k"), "budget": budget, "cv": cv,
           "seed": args.seed, "requests": len(trace), "shard_bytes": sizes_r}
    t_setup = time.perf_counter()
    with M.Ctx(device_ids=device_ids, budget=budget, max_batch=P["max_batch"], max_tokens=P["L"], trace=1,
               writeback=0, max_dims=d, prefetch=args.prefetch, victim_policy=args.victim_policy) as ctx:
        ids = [ctx.register_model(x) for x in dims]
        for m in ids:
            ctx.synth_fill(m, P.get("seed0", 7000) + m)
        res["setup_s"] = time.perf_counter() - t_setup
        outs = []
        t0 = time.perf_counter()
        for r in trace:
            if P["kind"] == "gamma" and not r.warmup:
                dt = r.t_arr - (time.perf_counter() - t0)
                if dt > 0:
                    time.sleep(dt)
            rid, out = ctx.request(ids[r.model], r.tokens)
            outs.append((rid, r, out))
            if r.warmup or P["kind"] == "alternating":
                ctx.wait_request(rid, 600)
        lat, lat_by = [], {}
        for rid, r, out in outs:
            ta, td = ctx.wait_request(rid, 600)
            if not r.warmup:
                lat.append(td - ta)
                lat_by.setdefault(names[r.model], []).append(td - ta)
        # resident shards vs the oracle's hashes of their C0 images, where tests/golden has them
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c0_shard_hashes.json")))
        checks = []
        for mi, m in enumerate(ids):
            if ctx.residency(m) != M.RESIDENT:
                continue
            for r in range(tp):
                k = f"{names[mi]}/tp{tp}/r{r}/seed{P.get('seed0', 7000) + mi}/bf16"
                if k in gold:
                    checks.append(ctx.checksum(m, r) == int(gold[k], 16))
        if checks:
            res["resident_checksums_equal_oracle"] = all(checks)
            res["resident_checksums_checked"] = len(checks)
        tpath = "/tmp/serve_trace.ndjson"
        ctx.trace_dump(tpath)
        ctx.timeline_dump("/tmp/serve_timeline.ndjson")
        st = ctx.stats()
        loads = [json.loads(l) for l in open(tpath) if '"dec":"load"' in l]
        h2d = []   # host-observed swap-in latency (submit -> last rank's ack), ms: virtual ranks share
        for ld in loads:  # one GPU and one link, so per-rank device spans would overlap-count
            ts, td = ctx.wait(ld["id"])
            h2d.append(((max(td) - ts) * 1e3, sizes_r[ld["model"]]))
    if P["kind"] == "alternating":
        lat = lat[1:]                       # cold first load reported separately
    res["latency_s"] = metrics.summary(lat)
    res["swaps_in"] = st["swaps_in"]
    res["h2d_bytes"] = st["h2d_bytes"]
    res["prefetches"] = st["prefetches"]
    res["swap_in_GBps_median"] = float(np.median([tp * n / (ms / 1e3) / 1e9 for ms, n in h2d])) if h2d else None
    if len(set(names)) > 1:
        res["latency_by_model_s"] = {k: metrics.summary(v) for k, v in lat_by.items()}
        res["swaps_in_by_model"] = {k: sum(1 for ld in loads if names[ld["model"]] == k) for k in set(names)}
    res["batches"] = st["batches"]
    res["fwd_ms_mean"] = st["fwd_gpu_us_sum"] / 1e3 / max(1, st["fwd_gpu_n"])
    # device timeline: how much forward time ran while a swap-in was streaming on the same GPU
    # ("a later batch entry [proceeds] without waiting for a previous load entry")
    spans = [json.loads(l) for l in open("/tmp/serve_timeline.ndjson")]
    loads = sorted((s_["t0_ms"], s_["t1_ms"]) for s_ in spans if s_["kind"] == "load")
    fwd = [(s_["t0_ms"], s_["t1_ms"]) for s_ in spans if s_["kind"] == "batch"]
    merged = []
    for a, b in loads:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    ov = sum(max(0.0, min(b, y) - max(a, x)) for a, b in fwd for x, y in merged)
    tot = sum(b - a for a, b in fwd)
    res["fwd_ms_total"] = tot
    res["fwd_overlapped_with_swapin_frac"] = ov / tot if tot else 0.0
    # replay parity of the engine's decisions (oracle C1)
    rcfg, evs, decs = S.read_trace(tpath)
    rdecs, _ = S.replay(rcfg, evs)
    res["replay_identical"] = rdecs == decs
    # logits parity on sampled requests (oracle C5, bf16-emulating) where the oracle is fast enough
    # (OPT-125M requests by default; --check-logits N samples N requests of any model, the large
    # ones through the oracle's layer-by-layer C0 weights)
    small = [(rid, r, out) for rid, r, out in outs if names[r.model] == "opt-125m"]
    n_check = args.check_logits if args.check_logits >= 0 else (len(small) if args.preset == "cfg1" else min(8, len(small)))
    pool = small if args.check_logits < 0 or small else [(rid, r, out) for rid, r, out in outs if not r.warmup]
    if n_check and pool:
        errs, errs_ex, maxabs = [], [], []
        Ws = {}
        for rid, r, out in pool[:: max(1, len(pool) // n_check)][:n_check]:
            if r.model not in Ws:
                big = layout.shard_bytes(dims[r.model], 1) > 2**31
                Ws[r.model] = (layout.LazyFull if big else layout.full_tensors)(dims[r.model], P.get("seed0", 7000) + r.model)
            ref = forward.forward_bf16_emulated(dims[r.model], Ws[r.model], r.tokens[None])[0]
            ex = forward.forward_exact(dims[r.model], Ws[r.model], r.tokens[None])[0]
            errs.append(forward.rel_l2(out, ref))
            errs_ex.append(forward.rel_l2(out, ex))
            maxabs.append(float(np.abs(out - ex).max() / np.abs(ex).max()))
        res["logits_checked"] = len(errs)
        res["logits_max_rel_l2"] = max(errs)
        res["logits_max_rel_l2_vs_exact"] = max(errs_ex)
        res["logits_max_elementwise_vs_exact"] = max(maxabs)
    print(json.dumps(res), flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
