"""Pins for oracle/scheduler.py (C1): SPEC worked examples, textbook-LRU brute force,
closed forms (P:129's 0.75 s), invariants on random traces, exhaustive interleavings."""
import itertools
import json
import os
import random

import pytest

from oracle import scheduler as S
from oracle import costmodel, metrics

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ev(kind, t, **kw):
    return dict(ev=kind, t=t, **kw)


def make(n=2, k=1, tp=1, mb=8, D=1):
    return S.Engine(S.EngineConfig(n, k, tp, mb, D))


def load_resident(e, m, t=0.0, rid=1000):
    """Bring m resident via an explicit swap_in + acks."""
    out = e.step(ev("cmd_swap_in", t, model=m))
    ld = [d for d in out if d["dec"] == "load"][0]
    for r in range(e.cfg.tp):
        e.step(ev("ack", t, entry=ld["id"], rank=r))


def test_arrival_to_resident_idle_batches_at_once():
    e = make(1, 1)
    load_resident(e, 0)
    out = e.step(ev("arrival", 1.0, rid=0, model=0))
    assert [d["dec"] for d in out] == ["batch"] and out[0]["rids"] == [0]


def test_two_arrivals_packed_when_engine_busy():               # S:259 (D = 1 reading #26)
    e = make(1, 1)
    out = e.step(ev("arrival", 0.0, rid=0, model=0))
    assert out[0]["dec"] == "load"                             # load issued, batch deferred
    assert e.step(ev("arrival", 1.0, rid=1, model=0)) == []
    out = e.step(ev("ack", 2.0, entry=out[0]["id"], rank=0))
    assert [d["dec"] for d in out] == ["batch"] and out[0]["rids"] == [0, 1]


def test_d1_gating_then_pack():
    e = make(1, 1)
    load_resident(e, 0)
    b0 = e.step(ev("arrival", 1.0, rid=0, model=0))[0]
    assert e.step(ev("arrival", 1.1, rid=1, model=0)) == []
    assert e.step(ev("arrival", 1.2, rid=2, model=0)) == []
    out = e.step(ev("batch_done", 2.0, batch=b0["id"]))
    assert out[0]["dec"] == "complete" and out[1]["rids"] == [1, 2]


def test_oldest_head_first():
    e = make(2, 2, D=S.INF_D)
    load_resident(e, 0); load_resident(e, 1)
    e.cfg.max_inflight = 0                                       # hold dispatch while queuing
    e.step(ev("arrival", 0.5, rid=0, model=0))
    e.step(ev("arrival", 0.2, rid=1, model=1))
    e.cfg.max_inflight = S.INF_D
    out = e.step(ev("arrival", 0.9, rid=2, model=0))
    assert [(d["model"], d["rids"]) for d in out if d["dec"] == "batch"] == [(1, [1]), (0, [0, 2])]


def test_capacity1_swap_order():
    e = make(2, 1)
    load_resident(e, 0)
    out = e.step(ev("arrival", 1.0, rid=0, model=1))
    assert [d["dec"] for d in out] == ["offload", "load"]
    assert out[0]["model"] == 0 and out[1]["model"] == 1 and out[0]["off"] == out[1]["off"]
    assert e.step(ev("ack", 1.5, entry=out[0]["id"], rank=0)) == []
    b = e.step(ev("ack", 1.6, entry=out[1]["id"], rank=0))
    assert [d["dec"] for d in b] == ["batch"] and b[0]["model"] == 1


def test_lru_victim():
    e = make(3, 2, D=S.INF_D)
    load_resident(e, 0); load_resident(e, 1)
    b = e.step(ev("arrival", 1.0, rid=0, model=0))[0]; e.step(ev("batch_done", 1.0, batch=b["id"]))
    b = e.step(ev("arrival", 3.0, rid=1, model=1))[0]; e.step(ev("batch_done", 3.0, batch=b["id"]))
    out = e.step(ev("arrival", 4.0, rid=2, model=2))
    assert out[0]["dec"] == "offload" and out[0]["model"] == 0


def test_acks_all_ranks_any_order():
    e = make(1, 1, tp=4)
    ld = e.step(ev("cmd_swap_in", 0.0, model=0))[0]
    for i, r in enumerate([2, 0, 3]):
        e.step(ev("ack", 0.1 * i, entry=ld["id"], rank=r))
        assert e.state[0] == S.LOADING
    e.step(ev("ack", 1.0, entry=ld["id"], rank=1))
    assert e.state[0] == S.RESIDENT
    with pytest.raises(S.InvariantViolation):
        e.step(ev("ack", 1.0, entry=ld["id"], rank=1))


def test_no_eviction_under_inflight_batch():
    e = make(2, 1)
    load_resident(e, 0)
    b = e.step(ev("arrival", 1.0, rid=0, model=0))
    assert b[0]["dec"] == "batch"
    assert e.step(ev("arrival", 1.1, rid=1, model=1)) == []      # deferred
    out = e.step(ev("batch_done", 2.0, batch=b[0]["id"]))
    assert [d["dec"] for d in out] == ["complete", "offload", "load"]


def test_manual_swaps():
    e = make(2, 1)
    assert e.step(ev("cmd_swap_in", 0, model=0))[0]["dec"] == "load"
    assert e.step(ev("cmd_swap_in", 0, model=0))[0]["dec"] == "noop"
    assert e.step(ev("cmd_swap_in", 0, model=1))[0] == {"dec": "reject", "model": 1, "status": "ENOMEM"}
    assert e.step(ev("cmd_swap_out", 0, model=0))[0]["status"] == "EBUSY"     # still loading
    e.step(ev("ack", 0, entry=0, rank=0))
    b = e.step(ev("arrival", 1, rid=0, model=0))[0]
    assert e.step(ev("cmd_swap_out", 1, model=0))[0]["status"] == "EBUSY"     # in-flight batch
    e.step(ev("batch_done", 2, batch=b["id"]))
    assert e.step(ev("cmd_swap_out", 2, model=0))[0]["dec"] == "offload"
    assert e.step(ev("cmd_swap_out", 2, model=0))[0]["dec"] == "noop"
    assert e.step(ev("arrival", 3, rid=1, model=9))[0]["status"] == "ENOENT"


def test_textbook_lru_equivalence_blocking():                    # S:296, S:513 criterion 9
    rnd = random.Random(0)
    for trial in range(1000):
        n = rnd.randint(2, 20)
        k = rnd.randint(1, min(5, n))
        acc = [rnd.randrange(n) for _ in range(rnd.randint(1, 40))]
        e = make(n, k)
        evicted, t = [], 0.0
        for rid, m in enumerate(acc):
            t += 1.0
            pend = e.step(ev("arrival", t, rid=rid, model=m))
            while True:
                nxt = []
                for d in pend:
                    if d["dec"] == "offload":
                        evicted.append(d["model"])
                    if d["dec"] in ("offload", "load"):
                        nxt.append(ev("ack", t, entry=d["id"], rank=0))
                    if d["dec"] == "batch":
                        nxt.append(ev("batch_done", t, batch=d["id"]))
                if not nxt:
                    break
                pend = []
                for x in nxt:
                    pend += e.step(x)
        assert evicted == S.textbook_lru_evictions(acc, k), (trial, acc, k)


def test_closed_form_lower_bound_paper():
    """24 GB over a 32 GB/s link = 0.75 s; SPEC S:114/S:399/S:401; workers divide it."""
    gold = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for c in gold["transfer_time"]:
        assert costmodel.transfer_time(c["bytes"], c["msgs"], c["B"], c["alpha"]) == pytest.approx(c["expect"], abs=1e-12)
    for c in gold["swap_latency_ideal"]:
        # alternating blocking, clean eviction, alpha = 0: every measured swap = S/(w B)
        cfg = S.EngineConfig(2, 1, c["workers"], 8, 1)
        costs = S.Costs(int(c["S"] / c["workers"]), c["B"], c["B"], 0.0, chunk=1 << 62, writeback=False)
        evs, decs, tdone, log = S.simulate(cfg, costs, [(i, i % 2) for i in range(6)], 2, blocking=True)
        loads = [v for v in log.values() if v["kind"] == "load"]
        assert len(loads) == 6                                    # every request swaps
        for ld in loads[1:]:
            assert metrics.swap_in_latency(ld["submit"], list(ld["done"].values())) == pytest.approx(c["expect"], abs=1e-9)
    paper = json.load(open(os.path.join(GOLD, "paper_numbers.json")))
    assert paper["opt13b_footprint_GB"]["value"] / paper["link_bandwidth_GBps"]["value"] == paper["swap_lower_bound_s"]["value"]


def test_paired_swap_closed_form():
    """Writeback + load pipelined per chunk, alpha = 0, equal bandwidth: the load lags the
    offload by exactly one chunk: load_done = c/B + S/B; window = max(...) - submit."""
    S_, c, B = 1 << 30, 1 << 26, 50e9
    cfg = S.EngineConfig(2, 1, 1, 8, 1)
    costs = S.Costs(S_, B, B, 0.0, chunk=c, writeback=True)
    evs, decs, tdone, log = S.simulate(cfg, costs, [(i, i % 2) for i in range(4)], 2, blocking=True)
    offs = [v for v in log.values() if v["kind"] == "offload"]
    loads = [v for v in log.values() if v["kind"] == "load"]
    for off, ld in zip(offs, loads[1:]):
        assert ld["submit"] == off["submit"]
        assert off["done"][0] - off["submit"] == pytest.approx(S_ / B, rel=1e-12)
        assert ld["done"][0] - ld["submit"] == pytest.approx(c / B + S_ / B, rel=1e-12)
        assert metrics.swap_latency(off["submit"], off["done"][0], ld["done"][0]) == pytest.approx(c / B + S_ / B, rel=1e-12)


def test_sublinear_tp_with_alpha():                              # S:507 criterion 3
    lat = []
    for tp in (1, 2, 4):
        cfg = S.EngineConfig(2, 1, tp, 8, 1)
        costs = S.Costs(int(24e9 / tp), 32e9, 32e9, alpha=1e-3, chunk=int(24e9 / tp / 1000) + 1, writeback=False)
        _, _, _, log = S.simulate(cfg, costs, [(i, i % 2) for i in range(4)], 2, blocking=True)
        ld = [v for v in log.values() if v["kind"] == "load"][-1]
        lat.append(max(ld["done"].values()) - ld["submit"])
    assert lat[0] > lat[1] > lat[2] and lat[2] > lat[0] / 4


def _check_trace(decisions, events, n):
    """Post-hoc invariants: load-before-batch, per-model FIFO,
    every request completes, batches only for resident models (engine.check is online)."""
    resident = set()
    pend = {}
    served = {m: [] for m in range(n)}
    arrived = {m: [] for m in range(n)}
    for e in events:
        if e["ev"] == "arrival":
            arrived[e["model"]].append(e["rid"])
    for d in decisions:
        if d["dec"] == "batch":
            served[d["model"]] += d["rids"]
    for m in range(n):
        assert served[m] == arrived[m]                            # FIFO + work conservation


def test_random_traces_invariants():
    rnd = random.Random(5)
    for trial in range(300):
        n = rnd.randint(1, 6)
        k = rnd.randint(1, n)
        tp = rnd.choice([1, 2, 4, 8])
        D = rnd.choice([1, 2, S.INF_D])
        mb = rnd.choice([1, 2, 8, 32])
        cfg = S.EngineConfig(n, k, tp, mb, D)
        arr = sorted((rnd.uniform(0, 2.0), rnd.randrange(n)) for _ in range(rnd.randint(0, 40)))
        arr = [(i, m, t) for i, (t, m) in enumerate(arr)]
        costs = S.Costs(rnd.choice([1 << 20, 1 << 28]), 50e9, 55e9, rnd.choice([0, 1e-5]), 1 << 24,
                        1e-3, 1e-4, rnd.random() < 0.5, tuple(rnd.uniform(0, 1e-3) for _ in range(tp)))
        evs, decs, tdone, log = S.simulate(cfg, costs, arr, 8)
        assert set(tdone) == {a[0] for a in arr}
        _check_trace(decs, evs, n)
        # replay of the recorded event order reproduces every decision (replay mode C1)
        rdecs, _ = S.replay(cfg, evs)
        assert rdecs == decs


def test_exhaustive_interleavings_tiny():
    """All orders of arrival / ack / batch_done events on tiny systems keep the invariants
    (engine.check raises on violation), drain every request and keep per-model FIFO."""
    import copy
    total = 0
    for n, k, tp, seq in [(2, 1, 1, [0, 1, 0, 1]), (3, 2, 1, [0, 1, 2]), (2, 1, 2, [0, 1]),
                          (3, 1, 1, [2, 0, 1]), (2, 2, 1, [1, 0, 1])]:
        arrivals = [ev("arrival", float(i), rid=i, model=m) for i, m in enumerate(seq)]

        def explore(eng, pending, next_arr, served):
            nonlocal total
            if next_arr >= len(arrivals) and not pending:
                assert all(not q for q in eng.queue)
                for m in range(n):
                    assert served.get(m, []) == [a["rid"] for a in arrivals if a["model"] == m]
                total += 1
                return
            opts = list(range(len(pending)))
            if next_arr < len(arrivals):
                opts.append(-1)
            for o in opts:
                e2 = copy.deepcopy(eng)
                if o == -1:
                    x, newp, na = arrivals[next_arr], list(pending), next_arr + 1
                else:
                    x, newp, na = pending[o], pending[:o] + pending[o + 1:], next_arr
                sv = {m: list(v) for m, v in served.items()}
                for d in e2.step(x):
                    if d["dec"] in ("load", "offload"):
                        newp += [ev("ack", 0.0, entry=d["id"], rank=r) for r in range(tp)]
                    if d["dec"] == "batch":
                        newp.append(ev("batch_done", 0.0, batch=d["id"]))
                        sv.setdefault(d["model"], []).extend(d["rids"])
                explore(e2, newp, na, sv)

        explore(make(n, k, tp, mb=2), [], 0, {})
    assert total > 100
    print('leaves', total)
