"""Seeded fuzz of the whole serving path on the GPU (a0-a8 together): random sets of 3-5 OPT-like
models of different sizes in one region, TP 1/2/4 virtual ranks, D = 1/2 batches in flight,
writeback or clean eviction, copy-engine / zero-copy / auto swaps, chunk sizes, prefetch on/off,
and bursts of ragged requests. Per seed the checks are the north star's:
  * the engine's event log replays through the oracle scheduler to identical decisions;
  * every request is served, in per-model FIFO order;
  * after every burst each resident model is bit-exact on every rank (checksum vs the oracle
    image), and the byte-level oracle (RegionSwapModel) predicts every resident hash;
  * host arenas round-trip unchanged; sampled logits match the oracle forward at 1e-2."""
import json
import random

import numpy as np
import pytest

from oracle import checksum, forward, layout, scheduler as S
from oracle.swap import RegionSwapModel
from synth import request_tokens
from synth.models import OptDims
from tests.gpu_util import need_gpu, fuzz_seeds
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def placement_bytes(d, tp):
    return (layout.shard_bytes(d, tp) + 4095) // 4096 * 4096


def random_setup(seed):
    rnd = random.Random(seed)
    tp = rnd.choice([1, 2, 4])
    dims = []
    for _ in range(rnd.randint(3, 5)):
        hd = rnd.choice([32, 64])
        heads = tp * rnd.randint(1, 8 // tp + 1)
        h = heads * hd
        dims.append(OptDims(rnd.randint(1, 3), h, heads, 4 * h, vocab=tp * rnd.randint(100 // tp, 3000 // tp),
                            max_pos=16))
    big = max(dims, key=lambda d: d.hidden)
    dmax = OptDims(1, big.hidden, big.heads, max(d.ffn for d in dims), vocab=max(d.vocab for d in dims),
                   max_pos=16)
    opts = dict(tp=tp, D=rnd.choice([1, 2]), writeback=rnd.choice([0, 1]), mode=rnd.choice([0, 1, 2]),
                chunk=rnd.choice([1 << 18, 1 << 20, 4 << 20]), prefetch=rnd.choice([0, 1]))
    return rnd, dims, dmax, opts


@pytest.mark.parametrize("seed", fuzz_seeds(8))
def test_engine_fuzz(tmp_path, seed):
    M = need_gpu()
    rnd, dims, dmax, o = random_setup(seed)
    tp = o["tp"]
    sizes = [placement_bytes(d, tp) for d in dims]
    # room for the largest model plus about half of the rest: every burst can be served, and
    # most requests for an evicted model force placement traffic
    budget = max(sizes) + sum(sorted(sizes)[:-1]) // 2 + 4096
    seeds = [7000 + 10 * seed + i for i in range(len(dims))]
    imgs = {m: [layout.shard_image(d, tp, r, seeds[m]) for r in range(tp)] for m, d in enumerate(dims)}
    ref = {m: [checksum.checksum(a) for a in v] for m, v in imgs.items()}
    outs = []
    with M.Ctx(device_ids=(0,) * tp, budget=budget, max_batch=4, max_tokens=8, trace=1, max_inflight=o["D"],
               writeback=o["writeback"], swap_mode=o["mode"], chunk_bytes=o["chunk"], max_dims=dmax,
               prefetch=o["prefetch"], debug_checks=1) as ctx:     # residency stamps checked in every forward
        ids = [ctx.register_model(d) for d in dims]
        for m in ids:
            ctx.synth_fill(m, seeds[m])
        for step in range(25):
            pend = []
            for j in range(rnd.choice([1, 2, 3, 5])):
                m = rnd.randrange(len(dims))
                tok = request_tokens(8000 + seed, m, 10 * step + j, rnd.randint(1, 8), dims[m].vocab)
                rid, out = ctx.request(ids[m], tok)
                pend.append((rid, m, tok, out))
            for rid, m, tok, out in pend:
                ctx.wait_request(rid, 120)
                outs.append((m, tok, out.copy()))
            for mm in range(len(dims)):
                if ctx.residency(ids[mm]) == M.RESIDENT:
                    for r in range(tp):
                        assert ctx.checksum(ids[mm], r) == ref[mm][r], (step, mm, r, o)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        st = ctx.stats()
        final_dev = {m: [ctx.checksum(ids[m], r) for r in range(tp)]
                     for m in range(len(dims)) if ctx.residency(ids[m]) == M.RESIDENT}
        host = {m: [ctx.checksum(ids[m], r, on_device=False) for r in range(tp)] for m in range(len(dims))}
    cfg, evs, decs = S.read_trace(p)
    assert cfg.sizes == sizes and cfg.tp == tp and cfg.max_inflight == o["D"]
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs, o
    served, arrived = {}, {}
    for line in open(p):
        x = json.loads(line)
        if x.get("dec") == "batch":
            served.setdefault(x["model"], []).extend(x["rids"])
    for e in evs:
        if e["ev"] == "arrival":
            arrived.setdefault(e["model"], []).append(e["rid"])
    assert served == arrived                                       # all served, per-model FIFO
    assert st["swaps_in"] >= len({m for m, _, _ in outs})
    sm = RegionSwapModel(imgs, cfg.cap, writeback=bool(o["writeback"]))
    sm.apply(decs)
    assert sm.expected_resident_hashes() == final_dev
    assert host == ref
    Ws = {}
    for m, tok, out in outs[::4]:
        if m not in Ws:
            Ws[m] = layout.full_tensors(dims[m], seeds[m])
        refl = forward.forward_bf16_emulated(dims[m], Ws[m], tok[None])[0]
        PU.assert_logits(out, refl, tag=f"fuzz m{m}")


@pytest.mark.parametrize("tp", [2, 4])
def test_inflight_batches_allreduce_buffers(tp):
    """Regression (found by seed 7 above): with D > 1 batches in flight a fast TP peer starts its
    next batch while a slower one still reads its last all-reduce partial. A batch has an odd
    number of all-reduce points, so the partial double buffer must alternate across batch
    boundaries too. 160 one-request batches of a 1-layer model (the fastest forward, the widest
    race window) with D = 3 must equal the D = 1 run bit for bit, and the oracle. The race needs
    the ranks' streams to drift apart, so this stress run may pass on broken code; the fuzz case
    above (seed 7, with swaps in flight) is the one that failed on it."""
    M = need_gpu()
    d = OptDims(1, 64 * tp, 2 * tp, 256 * tp, vocab=500 * tp, max_pos=16)
    S_ = layout.shard_bytes(d, tp)
    toks = [request_tokens(9000, 0, i, 1 + i % 8, d.vocab) for i in range(160)]
    res = {}
    for D in (1, 3):
        with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), max_batch=1, max_tokens=8, max_inflight=D) as ctx:
            m = ctx.register_model(d)
            ctx.synth_fill(m, 9100)
            ctx.wait(ctx.swap_in(m))
            rids = [ctx.request(m, t) for t in toks]           # all queued at once: D batches in flight
            for rid, _ in rids:
                ctx.wait_request(rid, 120)
            res[D] = [out for _, out in rids]
    for a, b in zip(res[1], res[3]):
        assert np.array_equal(a, b)
    W = layout.full_tensors(d, 9100)
    for t, y in list(zip(toks, res[3]))[::20]:
        PU.assert_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], tag="fuzz")


@pytest.mark.parametrize("seed", fuzz_seeds(4, 300_000))
def test_engine_fuzz_pipeline(tmp_path, seed):
    """The same checks with pipeline parallelism (NEXT-1, reading #27): tp x pp ranks (pp 2-4),
    models of different depths and widths whose stage shards differ in size, D = 1."""
    M = need_gpu()
    rnd = random.Random(100 + seed)
    tp, pp = rnd.choice([(1, 2), (2, 2), (1, 3), (1, 4), (2, 4)])
    nr = tp * pp
    dims = []
    for _ in range(rnd.randint(2, 4)):
        hd = rnd.choice([32, 64])
        heads = tp * rnd.randint(1, 4)
        h = heads * hd
        dims.append(OptDims(pp * rnd.randint(1, 2), h, heads, 4 * h, vocab=tp * rnd.randint(100, 1500), max_pos=16))
    big = max(dims, key=lambda d: d.hidden)
    dmax = OptDims(pp, big.hidden, big.heads, max(d.ffn for d in dims), vocab=max(d.vocab for d in dims), max_pos=16)
    wb, mode = rnd.choice([0, 1]), rnd.choice([0, 1, 2])

    def img(d, g, s):
        return layout.shard_image(d, tp, g % tp, s, "bf16", pp, g // tp)

    sizes = [max((layout.shard_bytes(d, tp, "bf16", pp, st) + 4095) // 4096 * 4096 for st in range(pp)) for d in dims]
    budget = max(sizes) + sum(sorted(sizes)[:-1]) // 2 + 4096
    seeds = [7500 + 10 * seed + i for i in range(len(dims))]
    imgs = {m: [img(d, g, seeds[m]) for g in range(nr)] for m, d in enumerate(dims)}
    ref = {m: [checksum.checksum(a) for a in v] for m, v in imgs.items()}
    outs = []
    with M.Ctx(device_ids=(0,) * nr, pp=pp, budget=budget, max_batch=4, max_tokens=8, trace=1, writeback=wb,
               swap_mode=mode, chunk_bytes=1 << 20, max_dims=dmax, debug_checks=1) as ctx:
        ids = [ctx.register_model(d) for d in dims]
        for m in ids:
            ctx.synth_fill(m, seeds[m])
        for step in range(15):
            pend = []
            for j in range(rnd.choice([1, 2, 4])):
                m = rnd.randrange(len(dims))
                tok = request_tokens(8500 + seed, m, 10 * step + j, rnd.randint(1, 8), dims[m].vocab)
                rid, out = ctx.request(ids[m], tok)
                pend.append((rid, m, tok, out))
            for rid, m, tok, out in pend:
                ctx.wait_request(rid, 120)
                outs.append((m, tok, out.copy()))
            for mm in range(len(dims)):
                if ctx.residency(ids[mm]) == M.RESIDENT:
                    for g in range(nr):
                        assert ctx.checksum(ids[mm], g) == ref[mm][g], (step, mm, g, tp, pp)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        final_dev = {m: [ctx.checksum(ids[m], g) for g in range(nr)]
                     for m in range(len(dims)) if ctx.residency(ids[m]) == M.RESIDENT}
        host = {m: [ctx.checksum(ids[m], g, on_device=False) for g in range(nr)] for m in range(len(dims))}
    cfg, evs, decs = S.read_trace(p)
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs, (tp, pp)
    sm = RegionSwapModel(imgs, cfg.cap, writeback=bool(wb))
    sm.apply(decs)
    assert sm.expected_resident_hashes() == final_dev
    assert host == ref
    Ws = {}
    for m, tok, out in outs[::3]:
        if m not in Ws:
            Ws[m] = layout.full_tensors(dims[m], seeds[m])
        refl = forward.forward_bf16_emulated(dims[m], Ws[m], tok[None])[0]
        PU.assert_logits(out, refl, tag=f"fuzz-pp m{m} tp{tp} pp{pp}")


@pytest.mark.parametrize("seed", fuzz_seeds(3, 400_000))
def test_engine_fuzz_fp32(tmp_path, seed):
    """fp32 weights (the SIMT parity path, true fp32 FMA) under the same serving fuzz: replay
    identity, per-burst checksums and logits against the exact oracle at the fp32 bar 1e-5."""
    M = need_gpu()
    rnd, dims, dmax, o = random_setup(200 + seed)
    tp = o["tp"]
    sizes = [(layout.shard_bytes(d, tp, "fp32") + 4095) // 4096 * 4096 for d in dims]
    budget = max(sizes) + sum(sorted(sizes)[:-1]) // 2 + 4096
    seeds = [7700 + 10 * seed + i for i in range(len(dims))]
    ref = {m: [checksum.checksum(layout.shard_image(d, tp, r, seeds[m], "fp32")) for r in range(tp)]
           for m, d in enumerate(dims)}
    outs = []
    with M.Ctx(device_ids=(0,) * tp, budget=budget, dtype=M.FP32, max_batch=4, max_tokens=8, trace=1,
               max_inflight=o["D"], writeback=o["writeback"], swap_mode=o["mode"], chunk_bytes=o["chunk"],
               max_dims=dmax, prefetch=o["prefetch"]) as ctx:
        ids = [ctx.register_model(d) for d in dims]
        for m in ids:
            ctx.synth_fill(m, seeds[m])
        for step in range(12):
            pend = []
            for j in range(rnd.choice([1, 2, 3])):
                m = rnd.randrange(len(dims))
                tok = request_tokens(8700 + seed, m, 10 * step + j, rnd.randint(1, 8), dims[m].vocab)
                rid, out = ctx.request(ids[m], tok)
                pend.append((rid, m, tok, out))
            for rid, m, tok, out in pend:
                ctx.wait_request(rid, 120)
                outs.append((m, tok, out.copy()))
            for mm in range(len(dims)):
                if ctx.residency(ids[mm]) == M.RESIDENT:
                    for r in range(tp):
                        assert ctx.checksum(ids[mm], r) == ref[mm][r], (step, mm, r, o)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
    cfg, evs, decs = S.read_trace(p)
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs, o
    Ws = {}
    for m, tok, out in outs[::3]:
        if m not in Ws:
            Ws[m] = layout.full_tensors(dims[m], seeds[m], "fp32")
        ex = forward.forward_exact(dims[m], Ws[m], tok[None])[0]
        PU.assert_logits(out, None, ex, tol=PU.FP32_LOGITS_TOL, tag=f"fuzz-fp32 m{m}")


def test_long_run_many_swaps(tmp_path):
    """3000 requests round-robin over 3 models with room for one, 8 outstanding (batches of two
    form, so about every fourth request swaps), TP 2, D = 2, writeback: no resource runs out
    (events, staging ring, request ids, ack slots), every request completes, the decisions
    replay, and the last resident model is bit-exact on device and in its host arena."""
    M = need_gpu()
    d = OptDims(1, 128, 2, 512, vocab=512, max_pos=16)
    tp = 2
    S_ = placement_bytes(d, tp)
    seeds = [9300 + i for i in range(3)]
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + 4096, max_batch=2, max_tokens=4, trace=1, max_inflight=2,
               writeback=1, chunk_bytes=1 << 20, debug_checks=1) as ctx:
        ids = [ctx.register_model(d) for _ in range(3)]
        for m in ids:
            ctx.synth_fill(m, seeds[m])
        pend = []
        for i in range(3000):
            pend.append(ctx.request(ids[i % 3], np.array([1 + i % 7, 2, 3], np.int32))[0])
            if len(pend) >= 8:
                ctx.wait_request(pend.pop(0), 120)
        for rid in pend:
            ctx.wait_request(rid, 120)
        st = ctx.stats()
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        res = [m for m in range(3) if ctx.residency(ids[m]) == M.RESIDENT]
        assert len(res) == 1
        m = res[0]
        for r in range(tp):
            assert ctx.checksum(ids[m], r) == checksum.checksum(layout.shard_image(d, tp, r, seeds[m]))
            assert ctx.checksum(ids[m], r, on_device=False) == checksum.checksum(layout.shard_image(d, tp, r, seeds[m]))
    assert st["swaps_in"] >= 500
    cfg, evs, decs = S.read_trace(p)
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs
