"""GPU engine parity: the CUDA engine's recorded ordered event log, replayed through the oracle
scheduler (C1), yields identical decisions; request outcomes (logits) match the oracle forward;
per-model FIFO and load-before-batch hold in the trace."""
import json

import numpy as np
import pytest

from synth import opt_dims, gamma_trace, alternating_blocking
from oracle import layout, forward, scheduler as S
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def replay_check(path, nm, k, tp, mb, D):
    """Replay the engine's trace through the oracle scheduler, configured from the trace header
    (region bytes, placement bytes per model); equal-size models: cap // size == k slots."""
    cfg, events, decisions = S.read_trace(path)
    assert (cfg.n_models, cfg.tp, cfg.max_batch, cfg.max_inflight) == (nm, tp, mb, D)
    assert cfg.cap // cfg.sizes[0] == k
    rdecs, eng = S.replay(cfg, events)
    assert rdecs == decisions
    # per-model FIFO and load-before-batch (in the engine's own order)
    resident = set()
    served = {}
    for line in open(path):
        o = json.loads(line)
        if o.get("dec") == "batch":
            served.setdefault(o["model"], []).extend(o["rids"])
    arrived = {}
    for e in events:
        if e["ev"] == "arrival":
            arrived.setdefault(e["model"], []).append(e["rid"])
    assert served == arrived
    return events, decisions


@pytest.mark.parametrize("tp,D", [(1, 1), (2, 1), (2, 2)])
def test_gamma_trace_replay_and_outcomes(tmp_path, tp, D):
    M = need_gpu()
    d = opt_dims("small")
    nm, k, mb = 3, 2, 4
    S_ = layout.shard_bytes(d, tp)
    trace = gamma_trace([20, 5, 5], cv=4.0, duration=0.5, seed=1, token_len=8, vocab=d.vocab)
    import time
    with M.Ctx(device_ids=(0,) * tp, budget=k * ((S_ + 4095) // 4096 * 4096), max_batch=mb,
               max_tokens=8, trace=1, max_inflight=D) as ctx:
        ids = [ctx.register_model(d) for _ in range(nm)]
        for m in ids:
            ctx.synth_fill(m, 500 + m)
        t0 = time.perf_counter()
        outs = []
        for r in trace:
            if not r.warmup:
                dt = r.t_arr - (time.perf_counter() - t0)
                if dt > 0:
                    time.sleep(dt)
            rid, out = ctx.request(ids[r.model], r.tokens)
            outs.append((rid, r, out))
            if r.warmup:
                ctx.wait_request(rid, 120)
        for rid, r, out in outs:
            ctx.wait_request(rid, 120)
        p = str(tmp_path / "trace.ndjson")
        ctx.trace_dump(p)
        tl = str(tmp_path / "timeline.ndjson")
        ctx.timeline_dump(tl)
        st = ctx.stats()
    assert st["k_slots"] == k
    spans = [json.loads(l) for l in open(tl)]
    assert spans and all(s["t1_ms"] >= s["t0_ms"] >= 0 for s in spans)
    by_entry = {}
    for s in spans:
        by_entry.setdefault((s["kind"], s["id"]), set()).add(s["rank"])
    assert all(r == set(range(tp)) for r in by_entry.values())      # every rank's span recorded
    assert sum(1 for k_ in by_entry if k_[0] == "load") == st["swaps_in"]
    replay_check(p, nm, k, tp, mb, D)
    assert st["swaps_in"] >= nm
    Ws = {m: layout.full_tensors(d, 500 + m) for m in range(nm)}
    for rid, r, out in outs[:: max(1, len(outs) // 12)]:
        ref = forward.forward_bf16_emulated(d, Ws[r.model], r.tokens[None])[0]
        PU.assert_logits(out, ref, tag="engine")          # north-star bf16 tolerance


def test_alternating_blocking_every_request_swaps(tmp_path):
    """capacity 1, alternating blocking requests -> every request after the first swaps."""
    M = need_gpu()
    d = opt_dims("small")
    S_ = layout.shard_bytes(d, 1)
    reqs = alternating_blocking(10, 0, 2, d.vocab)
    with M.Ctx(device_ids=(0,), budget=S_ + (2 << 20), trace=1) as ctx:
        ids = [ctx.register_model(d), ctx.register_model(d)]
        for m in ids:
            ctx.synth_fill(m, 40 + m)
        for r in reqs:
            rid, out = ctx.request(ids[r.model], r.tokens)
            ctx.wait_request(rid, 60)
        p = str(tmp_path / "t.ndjson")
        ctx.trace_dump(p)
        st = ctx.stats()
    events, decisions = replay_check(p, 2, 1, 1, 8, 1)
    assert st["swaps_in"] == 10 and st["swaps_out"] == 9
    assert sum(1 for x in decisions if x["dec"] == "offload") == 9


def test_request_id_released_after_ok():
    """mpsw_poll / mpsw_wait_request release the id after the first OK (include/mpsw.h)."""
    import ctypes as C
    M = need_gpu()
    d = opt_dims("small")
    with M.Ctx(device_ids=(0,), budget=layout.shard_bytes(d, 1) + 4096) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 1)
        rid, out = ctx.request(m, np.array([3, 4], np.int32))
        ctx.wait_request(rid, 60)
        a, b = C.c_double(), C.c_double()
        assert M.lib().mpsw_poll(ctx.h, rid, C.byref(a), C.byref(b)) == M.ENOENT
        assert ctx.poll(rid) is not None          # the binding keeps the observed result
        with pytest.raises(M.MpswError) as e:
            ctx.wait(123456)
        assert e.value.status == M.ENOENT
