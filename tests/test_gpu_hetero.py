"""NEXT-4: models of different sizes share one region per rank, placed
first-fit (reading #28), with and without the NEXT-3 prefetch policy (reading #29).
On the GPU: decisions replay identically through the oracle scheduler, every resident model's
range is bit-exact on every rank after arbitrary swap traffic, the byte-level oracle
(RegionSwapModel) predicts every resident hash, host arenas round-trip, and logits match the
oracle forward."""
import random

import numpy as np
import pytest

from oracle import checksum, forward, layout, scheduler as S
from oracle.swap import RegionSwapModel
from synth import opt_dims, request_tokens
from synth.models import OptDims
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu

DIMS = [opt_dims("mid"), opt_dims("small"), OptDims(2, 256, 4, 1024, vocab=1000, max_pos=64),
        opt_dims("small"), opt_dims("mid"), OptDims(2, 384, 6, 1536, vocab=2048, max_pos=64)]


def placement_bytes(d, tp):
    return (layout.shard_bytes(d, tp) + 4095) // 4096 * 4096


# vp: victim_policy (0: LRU prefix + first fit, reading #28; 1: minimum-cost window, reading #30)
@pytest.mark.parametrize("tp,writeback,mode,prefetch,vp", [(1, 0, 0, 0, 0), (1, 1, 1, 1, 0), (2, 1, 1, 0, 0),
                                                           (2, 0, 2, 1, 0), (1, 0, 0, 1, 0), (1, 1, 1, 0, 1),
                                                           (2, 0, 0, 1, 1)])
def test_heterogeneous_models(tmp_path, tp, writeback, mode, prefetch, vp):
    M = need_gpu()
    sizes = [placement_bytes(d, tp) for d in DIMS]
    budget = sizes[0] + sizes[1] + sizes[5] + 3 * 4096        # one mid + two smaller ones
    seeds = [900 + i for i in range(len(DIMS))]
    imgs = {m: [layout.shard_image(d, tp, r, seeds[m]) for r in range(tp)] for m, d in enumerate(DIMS)}
    ref = {m: [checksum.checksum(a) for a in v] for m, v in imgs.items()}
    rnd = random.Random(tp * 100 + writeback * 10 + mode)
    outs = []
    with M.Ctx(device_ids=(0,) * tp, budget=budget, max_batch=4, max_tokens=8, trace=1, writeback=writeback,
               swap_mode=mode, chunk_bytes=1 << 20, max_dims=opt_dims("mid"), prefetch=prefetch,
               victim_policy=vp) as ctx:
        ids = [ctx.register_model(d) for d in DIMS]
        for m in ids:
            ctx.synth_fill(m, seeds[m])
        for step in range(40):
            burst = [rnd.randrange(len(DIMS)) for _ in range(rnd.choice([1, 1, 3]))]
            pend = []
            for j, m in enumerate(burst):
                L = rnd.choice([2, 5, 8])
                tok = request_tokens(step, m, j, L, DIMS[m].vocab)
                rid, out = ctx.request(ids[m], tok)
                pend.append((rid, m, tok, out))
            for rid, m, tok, out in pend:
                ctx.wait_request(rid, 120)
                outs.append((m, tok, out.copy()))
            for mm in range(len(DIMS)):
                if ctx.residency(ids[mm]) == M.RESIDENT:
                    for r in range(tp):
                        assert ctx.checksum(ids[mm], r) == ref[mm][r], (step, mm, r)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        st = ctx.stats()
        final_dev = {m: [ctx.checksum(ids[m], r) for r in range(tp)]
                     for m in range(len(DIMS)) if ctx.residency(ids[m]) == M.RESIDENT}
        host = {m: [ctx.checksum(ids[m], r, on_device=False) for r in range(tp)] for m in range(len(DIMS))}
    cfg, evs, decs = S.read_trace(p)
    assert cfg.sizes == sizes and cfg.cap == budget // 4096 * 4096 and st["region_bytes"] == cfg.cap
    assert cfg.prefetch == bool(prefetch) and cfg.victim_policy == vp
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs
    n_pf = sum(1 for d in decs if d.get("prefetch"))
    assert n_pf == st["prefetches"] and (n_pf > 0) == bool(prefetch)
    offs = {d["off"] for d in decs if d["dec"] == "load"}
    assert len(offs) > 1 and st["swaps_in"] > len(DIMS)          # real placement traffic
    # byte-level oracle: the decisions applied to the images predict every resident hash
    sm = RegionSwapModel(imgs, cfg.cap, writeback=bool(writeback))
    sm.apply(decs)
    assert sm.expected_resident_hashes() == final_dev
    assert host == ref                                            # (iv) round trip
    Ws = {}
    for m, tok, out in outs[::5]:
        if m not in Ws:
            Ws[m] = layout.full_tensors(DIMS[m], seeds[m])
        refl = forward.forward_bf16_emulated(DIMS[m], Ws[m], tok[None])[0]
        assert out.shape[0] == DIMS[m].vocab
        PU.assert_logits(out, refl, tag="hetero")


def test_heterogeneous_limits():
    M = need_gpu()
    small, mid = opt_dims("small"), opt_dims("mid")
    # without max_dims the first model fixes the workspace: a wider model is rejected
    with M.Ctx(device_ids=(0,), budget=64 << 20, max_batch=2, max_tokens=4) as ctx:
        ctx.register_model(small)
        with pytest.raises(M.MpswError) as e:
            ctx.register_model(mid)
        assert e.value.status == M.EINVAL
    # a model larger than the whole region: ENOMEM; the smaller one still works
    with M.Ctx(device_ids=(0,), budget=placement_bytes(small, 1) + 4096, max_batch=2, max_tokens=4,
               max_dims=mid) as ctx:
        a = ctx.register_model(small)
        with pytest.raises(M.MpswError) as e:
            ctx.register_model(mid)
        assert e.value.status == M.ENOMEM
        ctx.synth_fill(a, 3)
        rid, out = ctx.request(a, np.array([1, 2, 3], np.int32))
        ctx.wait_request(rid, 60)
        ref = forward.forward_bf16_emulated(small, layout.full_tensors(small, 3), np.array([[1, 2, 3]]))[0]
        PU.assert_logits(out, ref, tag="hetero")
