"""bench.py — the swap-dominated serving step of Computron (arXiv 2306.13835) on B200.

One STEP = one blocking request that forces a model swap (§5.1: "alternating
blocking requests ... forces the worst case scenario where each request must perform a swap"):
the engine picks the LRU victim, offloads it, swaps the requested model's shards into the freed
range over PCIe (a2/a3), joins the ranks' acks (a4), batches the request (a5), runs the TP
forward (a6) and returns the logits (a7). Timed through the public C-ABI (mpsw_request).

Default workload (N = 1): BASELINE cfg3 at t = 1 — three OPT-13B-shaped bf16 models (25.7 GB
each), budget of one model, round-robin blocking requests A, B, C, input length 2.
`--gpus N` (N > 1) runs ONE TP = N group, one process per GPU (re-launched under
torch.distributed.run when WORLD_SIZE is not set): cfg3 at t = N.

Metric: model swap-in aggregate H2D GB/s (and swap-in latency; p50/p99 request latency).
  value  = K * sum_r S_r / sum of the K swap-in latencies; swap-in latency =
           last rank's load ack - load submit, both on the engine's clock (rank 0's process)
  e2e    = the same bytes / device time of the K blocking mpsw_request calls (host tokens in,
           host logits out; includes offload gating, scheduling, forward and D2H), max over ranks
  roofline.achieved = sum_r S_r / median over steps of the max-over-ranks CUDA-event span of the
           load (H2D) stream: the DMA itself, against PCIe Gen5 x16 (64 GB/s per GPU)
  writeback = a second timed leg with the paper-faithful offload (D2H writeback chunk-paired with
           the load): H2D GB/s, the paper's swap window (offload submit -> both done)
  parity = device checksums of the resident shards and host checksums of the written-back arenas
           against the oracle's hashes (tests/golden/c0_shard_hashes.json, oracle-generated)
Inputs are larger than L2 (a >= 3.2 GB shard per step), so no L2 flush is needed.

`--impl reference` times the CPU oracle (oracle/) on slices of the same workload (see
run_reference); the default run's cpu_baseline times it once at full size.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

PCIE_GEN5_X16_GBPS = 64.0        # nominal per direction per GPU (north star roofline)
SWAP_MODES = {0: "auto", 1: "copy_engine", 2: "zero_copy", 3: "hybrid"}
GOLDEN = os.path.join(ROOT, "tests", "golden", "c0_shard_hashes.json")
SEED0 = 1000                     # model i of the bench has C0 seed SEED0 + i


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
    p.add_argument("--writeback", type=int, default=0, choices=[0, 1])
    p.add_argument("--wb-steps", type=int, default=6, help="timed steps of the writeback leg (0: skip)")
    p.add_argument("--swap-mode", type=int, default=0, choices=sorted(SWAP_MODES))
    p.add_argument("--chunk-mb", type=int, default=64)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--trace", default="")
    return p.parse_args()


def nearest_rank(xs, q):
    """Nearest-rank percentile."""
    s = sorted(xs)
    if not s:
        return float("nan")
    k = max(1, int(np.ceil(q / 100.0 * len(s))))
    return s[k - 1]


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


def ce_peaks(dev=0, nbytes=1 << 30):
    """Raw copy-engine pinned bandwidth of this GPU's link (torch, CUDA events): H2D alone and
    H2D + D2H concurrently on two streams (the ceiling of the paper's paired swap)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best_h2d = best_bi = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s1):
            e0.record(s1)
            d.copy_(h, non_blocking=True)
            e1.record(s1)
        e1.synchronize()
        best_h2d = max(best_h2d, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(dev)
        best_bi = max(best_bi, 2 * nbytes / (time.perf_counter() - t0) / 1e9)
    del h, h2, d, d2
    return best_h2d, best_bi


def pcie_link(dev=0):
    """PCIe generation and width of the GPU's link (nvidia-smi): the roofline's assumption, checked."""
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(dev), "--query-gpu=pcie.link.gen.current,pcie.link.width.current,"
                              "pcie.link.gen.max,pcie.link.width.max", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=30).stdout.strip().split(",")
        g, w, gm, wm = (int(x.strip()) for x in out[:4])
        return {"gen": g, "width": w, "gen_max": gm, "width_max": wm}
    except Exception:
        return None


def host_info():
    model = ""
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                model = l.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0))}


def mem_available():
    try:
        for l in open("/proc/meminfo"):
            if l.startswith("MemAvailable:"):
                return int(l.split()[1]) * 1024
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------- CPU oracle
# Only this leg (and --impl reference) imports oracle/: the oracle as it stands, timed on the
# host cores. "Full" = one complete oracle step of the workload; "slice" = 1/L_m of it.
def _oracle_layer_forward(d, W, h, i, dt=np.float64):
    """C5 layer i (oracle/forward.py layer_ops, fp64) on the residual stream h [1, L, hidden]."""
    from oracle import forward as OF
    op = OF.layer_ops(d, W, i, dt)
    xm = op["attn_block"](h, op["attn"](op["qkv"](op["ln1"](h)), d.heads))
    return op["mlp_block"](xm, op["fc1"](op["ln2"](xm)))


def oracle_step(d, arenas, slot, sm, tokens, layers, W, h, hash_threads):
    """One oracle step over `arenas` (C3 paired swap via oracle/swap.py SwapModel: victim written
    back chunk by chunk, requested arena copied in), the C4 hash of the new slot (invariant
    (iii) check), and the C5 forward of `layers` (embedding before layer 0, final LN + lm_head
    after the last layer). Returns (t_swap, t_hash, t_fwd, h)."""
    from oracle import checksum as OC, forward as OF
    m = 1 if sm.owner[0] == 0 else 0
    t0 = time.perf_counter()
    sm.paired(0, m)
    t1 = time.perf_counter()
    if hash_threads == 1:
        OC.checksum(sm.slot[0][0])
    else:
        OC.checksum_parallel(sm.slot[0][0], threads=hash_threads)
    t2 = time.perf_counter()
    L = tokens.shape[1]
    for i in layers:
        if i == 0:
            h = (W["decoder.embed_tokens.weight"].astype(np.float64)[tokens]
                 + W["decoder.embed_positions.weight"].astype(np.float64)[np.arange(L) + 2])
        h = _oracle_layer_forward(d, W, h, i)
        if i == d.n_layers - 1:
            op = OF.layer_ops(d, W, d.n_layers, np.float64)
            op["lm_head"](op["lnf"](h[:, L - 1]))
    t3 = time.perf_counter()
    return t1 - t0, t2 - t1, t3 - t2, h


def _oracle_arenas(nbytes, chunk):
    """Two model arenas + one slot of nbytes (the oracle's C3 state at TP 1, k = 1). Contents
    are arbitrary bytes: the swap's cost does not depend on them."""
    from oracle import swap as OS
    blk = np.random.default_rng(0).integers(0, 256, min(nbytes, 1 << 26), dtype=np.uint8)
    imgs = {}
    for m in range(2):
        a = np.empty(nbytes, np.uint8)
        for o in range(0, nbytes, blk.size):
            n = min(blk.size, nbytes - o)
            a[o:o + n] = blk[:n]
            a[o] = m
        imgs[m] = [a]
    # SwapModel copies the images it is given; at full size (2 x 25.7 GB) that would double the
    # host memory, so it is built on placeholders and handed the arenas afterwards (its copy
    # loop, the part that is timed, is used as it stands)
    sm = OS.SwapModel({m: [np.zeros(8, np.uint8)] for m in range(2)}, 1, chunk, writeback=True)
    sm.host, sm.S = imgs, nbytes
    sm.slot = [[np.empty(nbytes, np.uint8)]]
    sm.load(0, 0)                    # also faults the slot's pages in, outside the timed step
    return sm


def _limits(n):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(n)
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def run_cpu_baseline(d, S_r, tokens_len, chunk):
    """The oracle timed on the box's host cores, no extrapolation:
    * full: ONE complete oracle step at full size, all cores for the hash and the fp64 BLAS
      (oracle/swap.py's copy loop is single-threaded as it stands): paired swap of the whole
      S_r-byte shard, its C4 hash, the 40-layer fp64 forward with weights generated from C0;
    * one_thread: one 1/L_m slice of that step (S_r/L_m bytes swapped + hashed, one layer) on a
      single thread;
    * cfg1: BASELINE cfg1 end to end on the oracle (2 x OPT-125M, 20 alternating blocking
      requests): decision log (virtual-time DES) + 19 paired swaps + hashes + 20 bf16-emulated
      forwards. value/unit: swap-in GB/s of the full step (the metric's oracle analogue)."""
    from oracle import layout as OL
    info = host_info()
    tok = np.zeros((1, tokens_len), np.int64) + np.arange(tokens_len) * 7 + 3
    W = OL.LazyFull(d, SEED0)
    res = {"kind": "oracle", "unit": "GB/s", **info}
    with _limits(info["cores"]):
        sm = _oracle_arenas(S_r, chunk)
        ts, th, tf, _ = oracle_step(d, None, None, sm, tok, range(d.n_layers), W, None, info["cores"])
        del sm
    full = ts + th + tf
    res.update(value=S_r / ts / 1e9, e2e_value=S_r / full / 1e9, seconds_per_step=full,
               parts_s={"paired_swap": ts, "hash": th, "forward_40_layers": tf})
    sl = (S_r // d.n_layers) // 4096 * 4096
    with _limits(1):
        sm = _oracle_arenas(sl, chunk)
        ts1, th1, tf1, _ = oracle_step(d, None, None, sm, tok, [d.n_layers // 2], W,
                                       np.zeros((1, tokens_len, d.hidden)) + 0.01, 1)
        del sm
    res["one_thread"] = {"value": sl / ts1 / 1e9, "e2e_value": sl / (ts1 + th1 + tf1) / 1e9, "slice_bytes": sl,
                         "parts_s": {"paired_swap": ts1, "hash": th1, "forward_1_layer": tf1}}
    res["cfg1_oracle_e2e_s"] = cfg1_oracle_seconds(info["cores"])
    res["sample"] = (f"full: one complete oracle step of cfg3-t1 (paired swap of the {S_r / 1e9:.2f} GB shard via "
                     f"oracle/swap.py, its C4 hash on {info['cores']} threads, fp64 forward of all {d.n_layers} "
                     f"layers with C0 weights, BLAS on {info['cores']} threads; copy loop single-threaded as it "
                     f"stands); one_thread: a 1/{d.n_layers} slice on 1 thread; cfg1: BASELINE cfg1 end to end")
    return res


def cfg1_oracle_seconds(threads):
    """BASELINE cfg1 end to end on the oracle: 2 x OPT-125M (budget 1 model), 20 alternating
    blocking requests. The scheduler's virtual-time DES (oracle/scheduler.py, 55 GB/s
    links) decides every swap and batch; oracle/swap.py applies the decisions to the byte images
    (paired writeback swaps); the final resident image and both arenas are C4-hashed against the
    C0 images; every request's logits come from the bf16-emulating C5 forward."""
    from oracle import scheduler as OSch, layout as OL, forward as OF, checksum as OC, swap as OSW
    from synth import opt_dims, round_robin_blocking
    d = opt_dims("opt-125m")
    t0 = time.perf_counter()
    imgs = {m: [OL.shard_image(d, 1, 0, 1 + m)] for m in range(2)}
    Ws = {m: OL.full_tensors(d, 1 + m) for m in range(2)}
    t_gen = time.perf_counter() - t0
    reqs = round_robin_blocking(20, seed=0, token_len=2, vocab=d.vocab, models=(0, 1))
    S = OL.shard_bytes(d, 1)
    t1 = time.perf_counter()
    with _limits(threads):
        _, decisions, t_done, _ = OSch.simulate(OSch.EngineConfig(2, 1, 1, 1), OSch.Costs(S, 55e9, 55e9),
                                                [(r.rid, r.model) for r in reqs], token_len=2, blocking=True)
        sm = OSW.SwapModel(imgs, 1, 64 << 20, writeback=True)
        sm.apply(decisions)
        ok = all(OC.checksum(sm.host[m][0]) == OC.checksum(imgs[m][0]) for m in range(2))
        ok = ok and OC.checksum(sm.slot[0][0]) == OC.checksum(imgs[reqs[-1].model][0])
        for r in reqs:
            OF.forward_bf16_emulated(d, Ws[r.model], r.tokens[None])
    swaps = sum(1 for x in decisions if x["dec"] == "load")
    return {"seconds": time.perf_counter() - t1, "weights_and_images_s": t_gen, "requests": len(t_done),
            "loads": swaps, "hashes_equal": ok}


def run_reference(args, d, S_r, config, metric):
    """--impl reference: the oracle as it stands on this host, each step = 1/L_m of one full
    oracle step of the workload (S_r/L_m bytes paired-swapped + C4-hashed, one decoder layer of
    the fp64 forward, the layer index cycling so L_m steps cover one full request), all cores.
    value = swapped bytes / swap time; e2e = swapped bytes / step time (intensive rates: a slice
    has the full step's rates; ms_per_step is the slice's own measured time)."""
    from oracle import layout as OL
    info = host_info()
    sl = (S_r // d.n_layers) // 4096 * 4096
    tok = np.zeros((1, args.tokens), np.int64) + np.arange(args.tokens) * 7 + 3
    W = OL.LazyFull(d, SEED0)
    times = []
    with _limits(info["cores"]):
        sm = _oracle_arenas(sl, args.chunk_mb << 20)
        h = None
        for s in range(args.warmup + args.steps):
            layer = s % d.n_layers
            ts, th, tf, h = oracle_step(d, None, None, sm, tok, [layer], W, h, info["cores"])
            if s >= args.warmup:
                times.append((ts, th, tf))
    swap_s = sum(t[0] for t in times)
    step_s = sum(sum(t) for t in times)
    value = sl * len(times) / swap_s / 1e9
    e2e = sl * len(times) / step_s / 1e9
    print(json.dumps({"impl": "reference", "metric": metric, "value": value, "unit": "GB/s",
                      "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": step_s / len(times) * 1e3, "higher_is_better": True, "scaling": "strong",
                      "vs_baseline": None, "dtype": "u8 (swap) / f64 (forward)", "data": "synthetic",
                      "config": config,
                      "cpu_baseline": {"value": value, "unit": "GB/s", "cores": info["cores"], "kind": "oracle",
                                       "cpu_model": info["cpu_model"],
                                       "sample": (f"each step = 1/{d.n_layers} of one full oracle step: {sl >> 20} MiB "
                                                  f"paired swap (oracle/swap.py) + C4 hash on {info['cores']} threads "
                                                  f"+ one fp64 decoder layer (C0 weights, BLAS on {info['cores']} "
                                                  f"threads)")},
                      "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                      "parts_ms_per_step": {k: 1e3 * sum(t[i] for t in times) / len(times)
                                            for i, k in enumerate(("paired_swap", "hash", "forward_layer"))}}))


# ----------------------------------------------------------------------------- our arm
def bench_device():
    """One GPU per rank (LOCAL_RANK). MPSW_BENCH_DEVICE0=1 maps every rank to cuda:0 — only to
    exercise the N > 1 code path on a one-GPU box (numbers are then meaningless)."""
    return 0 if os.environ.get("MPSW_BENCH_DEVICE0") == "1" else int(os.environ.get("LOCAL_RANK", 0))


def golden_hashes():
    try:
        return json.load(open(GOLDEN))
    except (OSError, ValueError):
        return {}


def swap_records(ctx, trace_path, load_ids):
    """Per timed load: C7 swap-in latency (engine clock), the paired offload's paper window
    (offload submit -> both offload and load complete, on the engine's clock) and this
    process's device H2D span."""
    offs = {}
    prev = None
    for l in open(trace_path):
        o = json.loads(l)
        if o.get("dec") == "offload":
            prev = o
        elif o.get("dec") == "load":
            offs[o["id"]] = prev if prev is not None and prev["off"] == o["off"] else None
            prev = None
    out = []
    for lid in load_ids:
        ts, tdone = ctx.wait(lid, 600)
        _, _, ms = ctx.entry_gpu_ms(lid)
        rec = {"swapin_s": max(tdone) - ts, "h2d_ms": ms, "paper_window_s": None}
        off = offs.get(lid)
        if off is not None:
            to, to_done = ctx.wait(off["id"], 600)
            rec["paper_window_s"] = max(max(tdone), max(to_done)) - to
        out.append(rec)
    return out


def timed_requests(ctx, ids, reqs, out, rank, world, cpu_group, dev):
    import torch
    import torch.distributed as dist
    lat = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = ctx.stats()
    torch.cuda.synchronize()
    e0.record()
    if rank == 0:
        for r in reqs:
            rid, _ = ctx.request(ids[r.model], r.tokens, out)
            ta, td = ctx.wait_request(rid, 600)
            lat.append(td - ta)
    if world > 1:
        dist.barrier(group=cpu_group)
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    st1 = ctx.stats()
    return lat, e0.elapsed_time(e1) / 1e3, st0, st1


def run_ours(args, rank, world):
    """N = 1: one process, TP = 1. N > 1 (torchrun): one process per GPU forming ONE TP group of
    t = N ranks (library multi-process mode): every request swaps the next model's t shards in
    concurrently, one per GPU over its own PCIe link."""
    import torch
    import torch.distributed as dist
    from paper_2306_13835_b200 import mpsw as M
    from synth import opt_dims, round_robin_blocking

    dev = bench_device()
    torch.cuda.set_device(dev)
    d = opt_dims(args.model)
    tp = world
    M.lib()
    S_r = M.shard_layout(d, tp, rank)[1]                 # the library's own layout (C2)
    need = args.n_models * S_r * (world if os.environ.get("MPSW_BENCH_DEVICE0") == "1" else 1)
    avail = mem_available()
    if avail is not None and need > avail:
        raise SystemExit(f"bench: {args.n_models} models x {S_r / 1e9:.2f} GB pinned per rank need "
                         f"{need / 1e9:.1f} GB of host RAM, {avail / 1e9:.1f} GB available (ENOMEM)")
    ce_peak, ce_bidir = ce_peaks(dev)
    link = pcie_link(dev)
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
        ctx.synth_fill(m, SEED0 + i)
    t_fill = time.perf_counter() - t_setup - t_reg
    n_wb = args.wb_steps if not args.writeback else 0
    reqs = round_robin_blocking(args.warmup + args.steps + (2 + n_wb if n_wb else 0), seed=0,
                                token_len=args.tokens, vocab=d.vocab, models=tuple(range(args.n_models)))
    out = np.empty(d.vocab, np.float32)
    # CPU (gloo) barriers for the long waits of the followers: an NCCL barrier would park a
    # spinning kernel on every follower GPU while rank 0 drives the requests
    cpu_group = dist.new_group(backend="gloo") if world > 1 else None
    if rank == 0:
        for r in reqs[:args.warmup]:
            rid, _ = ctx.request(ids[r.model], r.tokens, out)
            ctx.wait_request(rid, 600)
    if world > 1:
        dist.barrier(group=cpu_group)
    main_reqs = reqs[args.warmup:args.warmup + args.steps]
    with Clocks(dev) as clk:
        lat, dev_s, st0, st1 = timed_requests(ctx, ids, main_reqs, out, rank, world, cpu_group, dev)
    tpath = args.trace or f"/tmp/mpsw_bench_trace_{os.getpid()}.ndjson"

    def last_loads(n):
        ids_ = [None]
        if rank == 0:
            ctx.trace_dump(tpath)
            loads = [json.loads(l)["id"] for l in open(tpath) if '"dec":"load"' in l]
            ids_ = [loads[-n:]]
        if world > 1:
            dist.broadcast_object_list(ids_, src=0)
        return ids_[0]

    main_ids = last_loads(args.steps)
    recs = swap_records(ctx, tpath, main_ids) if rank == 0 else [
        {"swapin_s": 0.0, "h2d_ms": ctx.entry_gpu_ms(l)[2], "paper_window_s": None} for l in main_ids]
    wb = None
    if n_wb:
        # the paper-faithful leg: offloads write the victim back (D2H chunk-paired with the load)
        if rank == 0:
            ctx.set_writeback(1)
            for r in reqs[args.warmup + args.steps:args.warmup + args.steps + 2]:
                rid, _ = ctx.request(ids[r.model], r.tokens, out)
                ctx.wait_request(rid, 600)
        if world > 1:
            dist.barrier(group=cpu_group)
        wlat, wdev_s, w0, w1 = timed_requests(ctx, ids, reqs[args.warmup + args.steps + 2:], out, rank, world,
                                              cpu_group, dev)
        wids = last_loads(n_wb)
        wrecs = swap_records(ctx, tpath, wids) if rank == 0 else [
            {"swapin_s": 0.0, "h2d_ms": ctx.entry_gpu_ms(l)[2], "paper_window_s": None} for l in wids]
        wb = {"recs": wrecs, "req_lat_s": wlat, "dev_s": wdev_s, "d2h_bytes": w1["d2h_bytes"] - w0["d2h_bytes"]}
    parity = None
    if not args.no_parity:
        parity = check_parity(ctx, ids, args, d, tp, rank, world, cpu_group)
    h2d_local = [r["h2d_ms"][rank] for r in recs]
    wb_h2d_local = [r["h2d_ms"][rank] for r in wb["recs"]] if wb else []
    if world > 1:
        from paper_2306_13835_b200.group import max_over_ranks
        tdev = "cuda" if dist.get_backend() == "nccl" else None
        h2d_local = max_over_ranks(h2d_local, device=tdev)
        dev_s = max_over_ranks([dev_s], device=tdev)[0]
        if wb:
            wb_h2d_local = max_over_ranks(wb_h2d_local, device=tdev)
            wb["dev_s"] = max_over_ranks([wb["dev_s"]], device=tdev)[0]
        dist.barrier(group=cpu_group)
    ctx.close()
    return {
        "recs": recs, "h2d_ms_max": h2d_local, "req_lat_s": lat, "dev_s": dev_s, "S_r": S_r, "tp": tp,
        "launches": st1["kernel_launches"] - st0["kernel_launches"],
        "fwd_ms": (st1["fwd_gpu_us_sum"] - st0["fwd_gpu_us_sum"]) / 1e3 / max(1, st1["fwd_gpu_n"] - st0["fwd_gpu_n"]),
        "ce_peak": ce_peak, "ce_bidir": ce_bidir, "clocks": clk.summary(),
        "setup": {"register_pin_s": t_reg, "synth_fill_s": t_fill}, "wb": wb, "wb_h2d_ms_max": wb_h2d_local,
        "parity": parity, "link": link,
    }


def check_parity(ctx, ids, args, d, tp, rank, world, cpu_group):
    """Bytes the bench moved, checked against the oracle's hashes of the C0 images: every
    RESIDENT model's device range on this rank, and every non-resident model's host arena
    (after the writeback leg these arenas have made a D2H round trip: invariant (iv))."""
    import torch.distributed as dist
    from paper_2306_13835_b200 import mpsw as M
    gold = golden_hashes()
    res = {"device": [], "host": [], "missing_golden": 0}
    for i, m in enumerate(ids):
        k = f"{args.model}/tp{tp}/r{rank}/seed{SEED0 + i}/bf16"
        want = gold.get(k)
        if want is None:
            res["missing_golden"] += 1
            continue
        want = int(want, 16)
        if ctx.residency(m) == M.RESIDENT:
            res["device"].append(ctx.checksum(m, rank) == want)
        else:
            res["host"].append(ctx.checksum(m, rank, on_device=False) == want)
    allres = [res]
    if world > 1:
        allres = [None] * world
        dist.all_gather_object(allres, res, group=cpu_group)
    dv = [x for r in allres for x in r["device"]]
    hs = [x for r in allres for x in r["host"]]
    return {"resident_device_checksums_equal_oracle": (all(dv) if dv else None), "n_device": len(dv),
            "host_arena_checksums_equal_oracle": (all(hs) if hs else None), "n_host": len(hs),
            "missing_golden": sum(r["missing_golden"] for r in allres),
            "golden": "tests/golden/c0_shard_hashes.json (tools/gen_golden_hashes.py, oracle only)"}


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` without a torchrun environment: re-exec this command under
    torch.distributed.run with N processes (one per GPU) on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl == "ours" and args.gpus > 1 and world == 0:
        sys.exit(relaunch_under_torchrun(args))
    world = max(world, 1)
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    from synth import opt_dims
    d = opt_dims(args.model)
    t = world if args.impl == "ours" else args.gpus
    from paper_2306_13835_b200 import mpsw as M
    S_r = M.shard_layout(d, t, 0)[1]
    config = {"workload": f"cfg3-t{t}: {args.n_models}x {args.model.upper()}-shaped bf16, ONE TP={t} group "
                          f"(one process per GPU), budget 1 model per GPU, round-robin blocking requests (every "
                          f"request swaps), L={args.tokens}, B=1",
              "model": args.model, "n_models": args.n_models, "tp": t, "shard_bytes_per_rank": S_r,
              "writeback": bool(args.writeback), "swap_mode": SWAP_MODES[args.swap_mode],
              "chunk_mb": args.chunk_mb, "l2": "inputs larger than L2 (one >= 3.2 GB shard per rank per step); no flush",
              "global_batch": 1, "seq_len": args.tokens, "parallelism": f"tp{t}"}
    metric = "model swap-in aggregate H2D GB/s (all TP ranks' shards over PCIe Gen5), OPT-13B cfg3"

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, d, S_r, config, metric)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(bench_device())
        dist.init_process_group(os.environ.get("MPSW_BENCH_BACKEND", "nccl"))
    r = run_ours(args, rank, world)
    if rank != 0:
        return
    tp = r["tp"]
    total = tp * r["S_r"]
    K = len(r["recs"])
    swapin = [x["swapin_s"] for x in r["recs"]]
    value = total * K / sum(swapin) / 1e9
    achieved = total / (statistics.median(r["h2d_ms_max"]) / 1e3) / 1e9
    e2e = total * K / r["dev_s"] / 1e9
    peak = PCIE_GEN5_X16_GBPS * tp
    line = {
        "metric": metric, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["dev_s"] / K * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8 (bf16 weights moved as bytes); forward bf16/fp32-acc",
        "data": "synthetic (counter-based random-init OPT weights, DESIGN.md §Inputs)", "config": config,
        "swap_in_latency_ms": {"p50": 1e3 * nearest_rank(swapin, 50), "p99": 1e3 * nearest_rank(swapin, 99),
                               "mean": 1e3 * statistics.mean(swapin),
                               "definition": "last rank's load ack - load submit, engine clock (C7)",
                               "device_h2d_p50_max_over_ranks": nearest_rank(r["h2d_ms_max"], 50)},
        "request_latency_ms": {"p50": 1e3 * nearest_rank(r["req_lat_s"], 50),
                               "p99": 1e3 * nearest_rank(r["req_lat_s"], 99)},
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": total + 4 * args.tokens * tp,
                "d2h_bytes_per_step": (total if args.writeback else 0) + 4 * d.vocab},
        "roofline": {"bound": "pcie", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "peak_source": "nominal PCIe Gen5 x16 per direction per GPU (north star); MEASURED_PEAKS.json has no PCIe entry",
                     "measured_ce_peak_GBps_per_gpu": r["ce_peak"], "frac_of_measured_ce_peak": achieved / (tp * r["ce_peak"]),
                     "measured_ce_bidir_GBps_per_gpu": r["ce_bidir"], "pcie_link": r["link"],
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
    if r["wb"]:
        w = r["wb"]
        ws = [x["swapin_s"] for x in w["recs"]]
        win = [x["paper_window_s"] for x in w["recs"] if x["paper_window_s"] is not None]
        h2d = total * len(ws) / sum(ws) / 1e9
        dev_h2d = total / (statistics.median(r["wb_h2d_ms_max"]) / 1e3) / 1e9
        line["writeback"] = {
            "steps": len(ws), "h2d_GBps": h2d, "frac_of_64": h2d / peak,
            "device_h2d_GBps": dev_h2d,
            "link_GBps_both_directions": 2 * total / statistics.median(win) / 1e9 if win else None,
            "frac_of_measured_bidir_ceiling": (2 * total / statistics.median(win) / 1e9) / (tp * r["ce_bidir"]) if win else None,
            "swap_in_latency_ms": {"p50": 1e3 * nearest_rank(ws, 50), "p99": 1e3 * nearest_rank(ws, 99)},
            "paper_window_ms": {"p50": 1e3 * nearest_rank(win, 50), "p99": 1e3 * nearest_rank(win, 99),
                                "definition": "offload submit -> offload and load both complete (P:129, C7)"},
            "request_latency_ms_p50": 1e3 * nearest_rank(w["req_lat_s"], 50),
            "d2h_bytes": w["d2h_bytes"],
        }
    if r["parity"]:
        line["parity"] = r["parity"]
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = run_cpu_baseline(d, r["S_r"], args.tokens, args.chunk_mb << 20)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
