"""bench.py — the swap-dominated serving step of Computron (arXiv 2306.13835) on B200.

One STEP = one blocking request that forces a model swap (§5.1: "alternating
blocking requests ... forces the worst case scenario where each request must perform a swap"):
the engine picks the LRU victim, offloads it, swaps the requested model's shard into the freed
slot over PCIe (a2/a3), joins the ranks' acks (a4), batches the request (a5), runs the TP
forward (a6) and returns the logits (a7).  Timed through the public C-ABI (mpsw_request).

Default workload (N = 1): BASELINE cfg3 at t = 1 — three OPT-13B-shaped bf16 models (25.7 GB
each), budget of one model, round-robin blocking requests A, B, C, input length 2.
Metric: model swap-in aggregate H2D GB/s (and swap-in latency; p50/p99 request latency).
  value  = sum over ranks of S_r / swap-in time, swap-in time from CUDA events on each rank's
           load (H2D) stream (device-timed; max over ranks; summed over the K timed steps)
  e2e    = the same bytes / wall time of the K blocking mpsw_request calls (host tokens in,
           host logits out; includes offload gating, scheduling, forward and D2H)
Inputs are larger than L2 (a 25.7 GB shard per step), so no L2 flush is needed.

`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

PCIE_GEN5_X16_GBPS = 64.0        # nominal per direction per GPU (north star roofline)


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0                # B200_PROFILING.md fallback


HBM_PEAK = _hbm_peak()


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=9)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="opt-13b")
    p.add_argument("--n-models", type=int, default=3)
    p.add_argument("--tokens", type=int, default=2)
    p.add_argument("--writeback", type=int, default=0)
    p.add_argument("--swap-mode", type=int, default=0)
    p.add_argument("--chunk-mb", type=int, default=64)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--trace", default="")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev=0):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ce_peak_h2d(dev=0, nbytes=1 << 30):
    """Raw copy-engine pinned H2D bandwidth (torch, CUDA events) — context for the roofline."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del h, d
    return best


# ----------------------------------------------------------------------------- CPU oracle arm
def cpu_oracle_step(model, sample_bytes, layer_W, tokens, d):
    """One oracle step on a bounded sample: the C3 swap semantics (paired chunked copy of the
    victim back to its arena, then the requested model's arena into the slot) over
    `sample_bytes`, plus the C5 forward of ONE decoder layer (fp64) scaled by the layer count."""
    from oracle import swap as OS, forward as OF
    t0 = time.perf_counter()
    model.paired(0, 1 if model.owner[0] == 0 else 0)
    t_swap = time.perf_counter() - t0
    t1 = time.perf_counter()
    x = layer_W["x"]
    p = "decoder.layers.0."
    a = OF.layer_norm(x, layer_W[p + "self_attn_layer_norm.weight"], layer_W[p + "self_attn_layer_norm.bias"], np.float64)
    hd = d.hidden // d.heads
    q = (a @ layer_W[p + "self_attn.q_proj.weight"].T + layer_W[p + "self_attn.q_proj.bias"]) * hd ** -0.5
    k = a @ layer_W[p + "self_attn.k_proj.weight"].T + layer_W[p + "self_attn.k_proj.bias"]
    v = a @ layer_W[p + "self_attn.v_proj.weight"].T + layer_W[p + "self_attn.v_proj.bias"]
    o = OF._attention(q, k, v, d.heads, np.float64)
    h = x + o @ layer_W[p + "self_attn.out_proj.weight"].T + layer_W[p + "self_attn.out_proj.bias"]
    f = OF.layer_norm(h, layer_W[p + "final_layer_norm.weight"], layer_W[p + "final_layer_norm.bias"], np.float64)
    h = h + np.maximum(f @ layer_W[p + "fc1.weight"].T + layer_W[p + "fc1.bias"], 0) @ layer_W[p + "fc2.weight"].T
    t_layer = time.perf_counter() - t1
    return t_swap, t_layer


def oracle_setup(d, tokens, sample_bytes):
    from oracle import swap as OS, layout as OL
    from oracle import weights as OW
    rng = np.random.default_rng(0)
    imgs = {m: [rng.integers(0, 256, sample_bytes, dtype=np.uint8)] for m in range(2)}
    model = OS.SwapModel(imgs, 1, 64 << 20, writeback=True)
    model.load(0, 0)
    # one decoder layer's weights of the full-width model (C0 values, fp64)
    specs = [s for s in OL.canonical_tensors(d) if s.name.startswith("decoder.layers.0.")]
    W = {}
    for s in specs:
        n = int(np.prod(s.shape))
        W[s.name] = OW.round_bf16(OW.fp32_values(1, s.tid, np.arange(n), s.ln_gamma)).astype(np.float64).reshape(s.shape)
    W["x"] = rng.standard_normal((1, tokens, d.hidden)) * 0.02
    return model, W


def run_cpu_baseline(d, S_r, tokens, steps, sample_bytes=1 << 30):
    model, W = oracle_setup(d, tokens, sample_bytes)
    ts, tl = [], []
    for _ in range(steps):
        a, b = cpu_oracle_step(model, sample_bytes, W, tokens, d)
        ts.append(a)
        tl.append(b)
    t_step_full = statistics.median(ts) * (S_r / sample_bytes) + statistics.median(tl) * d.n_layers
    return {"value": S_r / t_step_full / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": (f"oracle C3 paired swap over a {sample_bytes >> 20} MiB sample of the {S_r/1e9:.2f} GB shard "
                       f"+ C5 fp64 forward of 1 of {d.n_layers} decoder layers (L={tokens}); step time scaled to the "
                       f"full shard and all layers; {steps} steps, median"),
            "seconds_per_step_scaled": t_step_full}


# ----------------------------------------------------------------------------- our arm
def bench_device():
    """One GPU per rank (LOCAL_RANK). MPSW_BENCH_DEVICE0=1 maps every rank to cuda:0 — only to
    exercise the N > 1 code path on a one-GPU box (numbers are then meaningless)."""
    return 0 if os.environ.get("MPSW_BENCH_DEVICE0") == "1" else int(os.environ.get("LOCAL_RANK", 0))


def run_ours(args, rank, world):
    """N = 1: one process, TP = 1. N > 1 (torchrun): one process per GPU forming ONE TP group of
    t = N ranks (library multi-process mode): every request swaps the next model's t shards in
    concurrently, one per GPU over its own PCIe link."""
    import torch
    import torch.distributed as dist
    from paper_2306_13835_b200 import mpsw as M
    from synth import opt_dims, round_robin_blocking
    from oracle import layout as OL_sizes   # sizes only, for reporting (no oracle compute)

    dev = bench_device()
    torch.cuda.set_device(dev)
    d = opt_dims(args.model)
    tp = world
    M.lib()
    ce_peak = ce_peak_h2d(dev)
    S_r = OL_sizes.shard_bytes(d, tp)
    t_setup = time.perf_counter()
    kw = dict(budget=(S_r + 4095) // 4096 * 4096, max_batch=1, max_tokens=max(8, args.tokens),
              writeback=args.writeback, swap_mode=args.swap_mode, chunk_bytes=args.chunk_mb << 20, trace=1)
    if world > 1:
        from paper_2306_13835_b200.group import open_group_ctx
        ctx = open_group_ctx(dev, **kw)
    else:
        ctx = M.Ctx(device_ids=(dev,), **kw)
    ids = [ctx.register_model(d) for _ in range(args.n_models)]
    t_reg = time.perf_counter() - t_setup
    for i, m in enumerate(ids):
        ctx.synth_fill(m, 1000 + i)
    t_fill = time.perf_counter() - t_setup - t_reg
    reqs = round_robin_blocking(args.warmup + args.steps, seed=0, token_len=args.tokens, vocab=d.vocab,
                                models=tuple(range(args.n_models)))
    out = np.empty(d.vocab, np.float32)

    def one(r):
        rid, _ = ctx.request(ids[r.model], r.tokens, out)
        return rid, ctx.wait_request(rid, 600)

    # CPU (gloo) barriers for the long waits of the followers: an NCCL barrier would park a
    # spinning kernel on every follower GPU while rank 0 drives the requests
    cpu_group = dist.new_group(backend="gloo") if world > 1 else None
    if rank == 0:
        for r in reqs[:args.warmup]:
            one(r)
    if world > 1:
        dist.barrier(group=cpu_group)
    torch.cuda.synchronize()
    st0 = ctx.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        e0.record()
        w0 = time.perf_counter()
        if rank == 0:
            for r in reqs[args.warmup:]:
                _, (ta, td) = one(r)
                lat.append(td - ta)
        if world > 1:
            dist.barrier(group=cpu_group)
        wall = time.perf_counter() - w0
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    st1 = ctx.stats()
    dev_s = e0.elapsed_time(e1) / 1e3
    timed = [None]
    if rank == 0:
        tpath = args.trace or "/tmp/mpsw_bench_trace.ndjson"
        ctx.trace_dump(tpath)
        loads = [json.loads(l) for l in open(tpath) if '"dec":"load"' in l]
        timed = [[ld["id"] for ld in loads[-args.steps:]]]
    if world > 1:
        dist.broadcast_object_list(timed, src=0)
    h2d_ms, swapin_lat = [], []
    for lid in timed[0]:
        ts, tdone = ctx.wait(lid, 600)
        _, _, ms = ctx.entry_gpu_ms(lid)
        h2d_ms.append(ms[rank])
        swapin_lat.append(max(tdone) - ts)
    if world > 1:
        from paper_2306_13835_b200.group import max_over_ranks
        tdev = "cuda" if dist.get_backend() == "nccl" else None
        h2d_ms = max_over_ranks(h2d_ms, device=tdev)
        dev_s = max_over_ranks([dev_s], device=tdev)[0]
        dist.barrier(group=cpu_group)
    ctx.close()
    return {
        "h2d_ms": h2d_ms, "swapin_lat_s": swapin_lat, "req_lat_s": lat, "dev_s": dev_s, "wall_s": wall,
        "launches": st1["kernel_launches"] - st0["kernel_launches"], "S_r": S_r, "tp": tp,
        "fwd_ms": (st1["fwd_gpu_us_sum"] - st0["fwd_gpu_us_sum"]) / 1e3 / max(1, st1["fwd_gpu_n"] - st0["fwd_gpu_n"]),
        "ce_peak": ce_peak, "clocks": clk.summary(), "setup": {"register_pin_s": t_reg, "synth_fill_s": t_fill},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(bench_device())
        dist.init_process_group(os.environ.get("MPSW_BENCH_BACKEND", "nccl"))

    from synth import opt_dims
    from oracle import layout as OL_sizes
    d = opt_dims(args.model)
    S_r = OL_sizes.shard_bytes(d, world)
    config = {"workload": f"cfg3-t{world}: {args.n_models}x {args.model.upper()}-shaped bf16, ONE TP={world} group "
                          f"(one process per GPU), budget 1 model per GPU, round-robin blocking requests (every "
                          f"request swaps), L={args.tokens}, B=1",
              "model": args.model, "n_models": args.n_models, "tp": world, "shard_bytes_per_rank": S_r,
              "writeback": bool(args.writeback), "swap_mode": ["auto", "copy_engine", "zero_copy"][args.swap_mode],
              "chunk_mb": args.chunk_mb, "l2": "inputs larger than L2 (one >=25.7 GB shard per step); no flush needed",
              "global_batch": 1, "seq_len": args.tokens, "parallelism": f"tp{world}"}
    metric = "model swap-in aggregate H2D GB/s (all TP ranks' shards over PCIe Gen5), OPT-13B cfg3"

    if args.impl == "reference":
        if rank != 0:
            return
        cb = run_cpu_baseline(d, S_r, args.tokens, args.warmup + args.steps)
        print(json.dumps({"impl": "reference", "metric": metric, "value": cb["value"], "unit": "GB/s",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": cb["seconds_per_step_scaled"] * 1e3, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "u8 (swap) / f64 (forward)",
                          "data": "synthetic", "config": config,
                          "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                          "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    r = run_ours(args, rank, world)
    if rank != 0:
        return
    steps = len(r["h2d_ms"])
    tp = r["tp"]
    achieved = tp * r["S_r"] / (statistics.median(r["h2d_ms"]) / 1e3) / 1e9
    value = tp * r["S_r"] * steps / (sum(r["h2d_ms"]) / 1e3) / 1e9
    e2e = tp * r["S_r"] * steps / r["dev_s"] / 1e9
    dev_s_max = r["dev_s"]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cb = run_cpu_baseline(d, r["S_r"], args.tokens, 5)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    from oracle import metrics as OM
    line = {
        "metric": metric, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_s_max / steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8 (bf16 weights moved as bytes); forward bf16/fp32-acc",
        "data": "synthetic (counter-based random-init OPT weights, DESIGN.md §Inputs)", "config": config,
        "swap_in_latency_ms": {"p50": 1e3 * OM.nearest_rank(r["swapin_lat_s"], 50),
                               "p99": 1e3 * OM.nearest_rank(r["swapin_lat_s"], 99),
                               "device_h2d_p50": OM.nearest_rank(r["h2d_ms"], 50)},
        "request_latency_ms": {"p50": 1e3 * OM.nearest_rank(r["req_lat_s"], 50),
                               "p99": 1e3 * OM.nearest_rank(r["req_lat_s"], 99)},
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": tp * r["S_r"] + 4 * args.tokens * tp,
                "d2h_bytes_per_step": (tp * r["S_r"] if args.writeback else 0) + 4 * d.vocab},
        "roofline": {"bound": "pcie", "achieved": achieved, "peak": PCIE_GEN5_X16_GBPS * tp, "unit": "GB/s",
                     "frac": achieved / (PCIE_GEN5_X16_GBPS * tp), "traffic": None,
                     "peak_source": "nominal PCIe Gen5 x16 per direction (north star); MEASURED_PEAKS.json has no PCIe entry",
                     "measured_ce_peak_GBps_per_gpu": r["ce_peak"], "frac_of_measured_ce_peak": achieved / (tp * r["ce_peak"]),
                     "kernel": "swap-in H2D (copy engine cudaMemcpyAsync chunks; not an SM kernel, so ncu dram traffic is n/a)"},
        "forward": {"ms_per_batch_device": r["fwd_ms"], "weight_bytes_per_rank": r["S_r"],
                    "achieved_hbm_GBps": r["S_r"] / (r["fwd_ms"] / 1e3) / 1e9 if r["fwd_ms"] > 0 else None,
                    "peak_hbm_GBps": HBM_PEAK, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "frac": (r["S_r"] / (r["fwd_ms"] / 1e3) / 1e9) / HBM_PEAK if r["fwd_ms"] > 0 else None,
                    "note": "TP forward of the swapped-in model (a6): weight-streaming, HBM-bound at M=B*L=2"},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "setup_s": r["setup"],
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line))


if __name__ == "__main__":
    main()
