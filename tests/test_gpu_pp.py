"""Pipeline parallelism (NEXT-1, P:72 TP x PP workers; P:105 entries pipelined stage to stage,
load entries forwarded without waiting for their copy, complete when every worker acked):
per-(stage, TP rank) shard parity, logits vs the oracle for pp = 2 / 3 / 4 with tp = 1 / 2
(virtual ranks on one GPU) with D = 1 / 2 / 3 batches in flight (batches overlap across stages),
bitwise equality with pp = 1, engine replay parity, and the broadcast ablation."""
import json

import numpy as np
import pytest

from synth import opt_dims, request_tokens, alternating_blocking
from oracle import layout, checksum, forward, scheduler as S
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def budget_for(d, tp, pp, k=1):
    return k * max((layout.shard_bytes(d, tp, "bf16", pp, st) + 4095) // 4096 * 4096 for st in range(pp))


@pytest.mark.parametrize("tp,pp,name,D", [(1, 2, "mid", 1), (2, 2, "mid", 2), (1, 3, "small", 3), (1, 4, "mid", 2),
                                         (2, 2, "tiny", 1)])
def test_pp_swap_and_logits(tp, pp, name, D):
    M = need_gpu()
    d = opt_dims(name)
    with M.Ctx(device_ids=(0,) * (tp * pp), pp=pp, budget=budget_for(d, tp, pp), max_batch=4 if D == 1 else 1,
               max_tokens=8, max_inflight=D) as ctx:
        assert ctx.tp == tp and ctx.nr == tp * pp
        m = ctx.register_model(d)
        ctx.synth_fill(m, 61)
        ctx.wait(ctx.swap_in(m))
        for g in range(tp * pp):
            img = layout.shard_image(d, tp, g % tp, 61, "bf16", pp, g // tp)
            assert ctx.checksum(m, g) == checksum.checksum(img)
        toks = [request_tokens(6, 0, i, L, d.vocab) for i, L in enumerate([8, 3, 8, 1])]
        outs = []
        for t in toks:
            rid, out = ctx.request(m, t)
            outs.append((rid, out))
        for rid, _ in outs:
            ctx.wait_request(rid, 120)
    W = layout.full_tensors(d, 61)
    for t, (_, y) in zip(toks, outs):
        ref = forward.forward_bf16_emulated(d, W, t[None])[0]
        PU.assert_logits(y, ref, tag="pp")


@pytest.mark.parametrize("D,broadcast", [(1, 0), (3, 0), (1, 1)])
def test_pp_matches_no_pp_bitwise(D, broadcast):
    """PP only moves the residual stream between stages (an exact copy): logits are bitwise equal
    to the single-stage run with the same TP degree, also with D = 3 batches pipelined across
    the stages (12 requests of one token count each, max batch 1: 12 batches through 3 hop slots)
    and in the broadcast ablation."""
    M = need_gpu()
    d = opt_dims("small")
    toks = [request_tokens(7, 0, i, 8, d.vocab) for i in range(12)]
    res = []
    for pp in (1, 3):
        with M.Ctx(device_ids=(0,) * pp, pp=pp, budget=budget_for(d, 1, pp), max_batch=1, max_tokens=8,
                   max_inflight=D if pp > 1 else 1, pp_broadcast=broadcast if pp > 1 else 0) as ctx:
            m = ctx.register_model(d)
            ctx.synth_fill(m, 62)
            rids = [ctx.request(m, t) for t in toks]
            for rid, _ in rids:
                ctx.wait_request(rid, 120)
            res.append([out.copy() for _, out in rids])
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("D", [1, 2])
def test_pp_engine_replay(tmp_path, D):
    M = need_gpu()
    d = opt_dims("mid")
    tp, pp = 2, 2
    reqs = alternating_blocking(8, 0, 4, d.vocab)
    with M.Ctx(device_ids=(0,) * 4, pp=pp, budget=budget_for(d, tp, pp), max_batch=2, max_tokens=8, trace=1,
               max_inflight=D) as ctx:
        ids = [ctx.register_model(d), ctx.register_model(d)]
        for m in ids:
            ctx.synth_fill(m, 70 + m)
        for r in reqs:
            rid, out = ctx.request(ids[r.model], r.tokens)
            ctx.wait_request(rid, 120)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        st = ctx.stats()
    cfg, evs, decs = S.read_trace(p)
    assert cfg.tp == tp * pp and cfg.cap // cfg.sizes[0] == st["k_slots"]
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs
    assert sum(1 for e in evs if e["ev"] == "ack") == tp * pp * (st["swaps_in"] + st["swaps_out"])


def test_pp_config_errors():
    M = need_gpu()
    with pytest.raises(M.MpswError):
        M.Ctx(device_ids=(0, 0, 0), pp=2)                 # tp * pp != n_gpus
    with pytest.raises(M.MpswError):
        M.Ctx(device_ids=(0, 0), pp=2, max_inflight=2, pp_broadcast=1)   # the broadcast ablation needs D = 1
    with M.Ctx(device_ids=(0, 0), pp=2, max_inflight=2):                 # pipelined entries allow D > 1
        pass
