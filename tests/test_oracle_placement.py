"""Oracle pins for placement of models of different sizes (reading #28, SURVEY §8(f)
NEXT-4, §6 "models of different sizes"): worked examples, a brute-force placement checker
(unit bitmap scan, independent of the engine's interval sweep), reduction to the k-slot scheme for
equal sizes (pinned to textbook LRU), invariants under random traces, and byte-level swap
semantics (RegionSwapModel)."""
import random

import numpy as np
import pytest

from oracle import scheduler as S
from oracle.checksum import checksum
from oracle.swap import RegionSwapModel


def ev(kind, t, **kw):
    return dict(ev=kind, t=t, **kw)


def cfg(sizes, cap, mb=4, D=1, tp=1):
    return S.EngineConfig(len(sizes), 0, tp, mb, D, cap=cap, sizes=list(sizes))


def drive_resident(e, m, t):
    """Request model m once and complete everything it causes; returns the decisions."""
    out = e.step(ev("arrival", t, rid=int(t * 1000), model=m))
    allout = list(out)
    pend = [d for d in out if d["dec"] in ("load", "offload", "batch")]
    while pend:
        d = pend.pop(0)
        if d["dec"] == "batch":
            o2 = e.step(ev("batch_done", t, batch=d["id"]))
        else:
            o2 = []
            for r in range(e.cfg.tp):
                o2 += e.step(ev("ack", t, entry=d["id"], rank=r))
        allout += o2
        pend += [x for x in o2 if x["dec"] in ("load", "offload", "batch")]
    return allout


def swaps(decs):
    return [(d["dec"], d["model"], d["off"]) for d in decs if d["dec"] in ("load", "offload")]


def test_worked_example_first_fit_and_lru_prefix():
    # cap 10: A(4) -> 0, B(4) -> 4; C(6) needs both A and B out (LRU A, then B); A(4) then fits
    # in the free tail [6, 10) without any eviction
    e = S.Engine(cfg([4, 4, 6], 10))
    assert swaps(drive_resident(e, 0, 1.0)) == [("load", 0, 0)]
    assert swaps(drive_resident(e, 1, 2.0)) == [("load", 1, 4)]
    assert swaps(drive_resident(e, 2, 3.0)) == [("offload", 0, 0), ("offload", 1, 4), ("load", 2, 0)]
    assert swaps(drive_resident(e, 0, 4.0)) == [("load", 0, 6)]


def test_worked_example_only_overlapping_victims():
    # A(3) at 0, B(3) at 3, D(3) at 6, cap 10. Victim order A, D, B (LRU). C(4): removing A leaves
    # [0,3)+[9,10) (no fit); removing D too gives [6,10) -> fit at 6: only D is evicted, A stays.
    e = S.Engine(cfg([3, 3, 3, 4], 10))
    for t, m in ((1.0, 0), (2.0, 1), (3.0, 2)):
        drive_resident(e, m, t)
    drive_resident(e, 1, 4.0)       # B used last -> LRU order A (1.0), D (3.0), B (4.0)
    assert swaps(drive_resident(e, 3, 5.0)) == [("offload", 2, 6), ("load", 3, 6)]
    assert e.state[0] == S.RESIDENT and e.off_of[0] == 0


def test_worked_example_defer_when_victim_busy():
    # A(6) resident with a batch in flight; B(6) cannot fit and A is not evictable -> B defers,
    # nothing is offloaded; after A's batch completes, A is evicted and B loads at 0
    e = S.Engine(cfg([6, 6], 10))
    drive_resident(e, 0, 1.0)
    out = e.step(ev("arrival", 2.0, rid=1, model=0))
    b = [d for d in out if d["dec"] == "batch"][0]
    out = e.step(ev("arrival", 2.5, rid=2, model=1))
    assert swaps(out) == []
    out = e.step(ev("batch_done", 3.0, batch=b["id"]))
    assert swaps(out) == [("offload", 0, 0), ("load", 1, 0)]


def test_model_larger_than_free_space_but_fits_region():
    e = S.Engine(cfg([2, 9], 10))
    drive_resident(e, 0, 1.0)
    assert swaps(drive_resident(e, 1, 2.0)) == [("offload", 0, 0), ("load", 1, 0)]


def brute_check(before_off, sizes, cap, decs_group, victims_in_order, m):
    """Independent check of one scheduling step for requester m: `before_off` = owned ranges
    before the step (model -> off), `victims_in_order` = eligible victims in victim-key order.
    Uses a unit bitmap: the load offset must be the lowest free one after removing the smallest
    victim prefix that admits a fit, and the offloads exactly the prefix members overlapping it."""
    def free_offsets(removed):
        used = np.zeros(cap, bool)
        for w, o in before_off.items():
            if w not in removed:
                used[o:o + sizes[w]] = True
        return [o for o in range(cap - sizes[m] + 1) if not used[o:o + sizes[m]].any()]

    fits = free_offsets(set())
    if fits:
        return [("load", m, fits[0])]
    for j in range(1, len(victims_in_order) + 1):
        pre = victims_in_order[:j]
        fits = free_offsets(set(pre))
        if fits:
            o = fits[0]
            out = [("offload", w, before_off[w]) for w in pre
                   if before_off[w] < o + sizes[m] and o < before_off[w] + sizes[w]]
            return out + [("load", m, o)]
    return []


@pytest.mark.parametrize("seed", range(40))
def test_random_blocking_vs_brute_force(seed):
    """Blocking requests (all queues empty at decision time): every placement decision equals
    the brute-force bitmap answer; invariants hold after every event."""
    rng = random.Random(seed)
    n = rng.randint(2, 6)
    sizes = [rng.randint(1, 5) for _ in range(n)]
    cap = rng.randint(max(sizes), 12)
    e = S.Engine(cfg(sizes, cap))
    t = 0.0
    for _ in range(30):
        m = rng.randrange(n)
        t += 1.0
        if e.state[m] == S.RESIDENT:
            drive_resident(e, m, t)
            continue
        before = {w: e.off_of[w] for w in range(n) if e.off_of[w] is not None}
        vics = sorted((w for w in range(n) if e.state[w] == S.RESIDENT and e.outstanding[w] == 0),
                      key=lambda w: (0, e.last_use[w], w))
        expect = brute_check(before, sizes, cap, None, vics, m)
        got = swaps(drive_resident(e, m, t))
        assert got[:len(expect)] == expect, (sizes, cap, before, got, expect)
        assert e.state[m] == S.RESIDENT


@pytest.mark.parametrize("seed", range(30))
def test_equal_sizes_reduce_to_textbook_lru(seed):
    """Equal sizes with a residue (cap = k*size + r, r < size): blocking accesses evict exactly
    the textbook-LRU victims, and offsets are slot multiples."""
    rng = random.Random(1000 + seed)
    n, k = rng.randint(2, 8), rng.randint(1, 4)
    size = rng.randint(2, 7)
    cap = k * size + rng.randrange(size)
    e = S.Engine(cfg([size] * n, cap))
    acc = [rng.randrange(n) for _ in range(60)]
    evicted = []
    for i, m in enumerate(acc):
        for d in drive_resident(e, m, float(i + 1)):
            if d["dec"] in ("load", "offload"):
                assert d["off"] % size == 0 and d["off"] + size <= k * size
            if d["dec"] == "offload":
                evicted.append(d["model"])
    assert evicted == S.textbook_lru_evictions(acc, k)


@pytest.mark.parametrize("seed", range(25))
def test_random_open_loop_invariants_and_completion(seed):
    """Open-loop arrivals, random ack / completion interleaving on heterogeneous sizes: invariants
    hold at every step (Engine.check), per-model FIFO, and every request completes."""
    rng = random.Random(77 + seed)
    n = rng.randint(2, 5)
    sizes = [rng.randint(1, 6) for _ in range(n)]
    cap = rng.randint(max(sizes), 14)
    tp = rng.choice([1, 2])
    e = S.Engine(cfg(sizes, cap, mb=rng.choice([1, 2, 4]), D=rng.choice([1, 2]), tp=tp))
    arrivals = sorted((rng.uniform(0, 10), rng.randrange(n)) for _ in range(25))
    rid_model, done, pend = {}, [], []
    t = 0.0
    ai = 0
    while ai < len(arrivals) or pend:
        if ai < len(arrivals) and (not pend or rng.random() < 0.5):
            t = max(t, arrivals[ai][0])
            rid_model[ai] = arrivals[ai][1]
            out = e.step(ev("arrival", t, rid=ai, model=arrivals[ai][1]))
            ai += 1
        else:
            # acks in any order; batches finish in submission order (one compute stream per
            # rank executes them serially, SURVEY §8(c) finding on D > 1)
            i = rng.randrange(len(pend))
            if pend[i]["dec"] == "batch":
                i = next(j for j, x in enumerate(pend) if x["dec"] == "batch")
            d = pend.pop(i)
            t += 0.01
            if d["dec"] == "batch":
                out = e.step(ev("batch_done", t, batch=d["id"]))
            else:
                out = []
                for r in range(tp):
                    out += e.step(ev("ack", t, entry=d["id"], rank=r))
        for d in out:
            if d["dec"] in ("load", "offload", "batch"):
                pend.append(d)
            if d["dec"] == "complete":
                done += d["rids"]
    assert sorted(done) == list(range(len(arrivals)))
    for m in range(n):                                    # per-model FIFO
        mine = [r for r in done if rid_model[r] == m]
        assert mine == sorted(mine)


@pytest.mark.parametrize("writeback", [True, False])
def test_region_swap_bytes(writeback):
    """Byte level: after random heterogeneous traffic, every resident model's range holds its
    image bit-exactly on every rank, and (writeback) host arenas round-trip unchanged."""
    rng = np.random.default_rng(5)
    sizes_b = {0: 3000, 1: 5000, 2: 1504, 3: 7000}
    tp = 2
    images = {m: [rng.integers(0, 256, n, dtype=np.uint8) for _ in range(tp)] for m, n in sizes_b.items()}
    place = [(n + 255) // 256 * 256 for n in sizes_b.values()]
    cap = 10240
    e = S.Engine(cfg(place, cap, tp=tp))
    sm = RegionSwapModel(images, cap, writeback=writeback)
    pyr = random.Random(9)
    for i in range(40):
        decs = drive_resident(e, pyr.randrange(4), float(i + 1))
        sm.apply(decs)
        for m, hs in sm.expected_resident_hashes().items():
            assert hs == [checksum(a) for a in images[m]]
    for m, ims in sm.host.items():
        for r in range(tp):
            assert np.array_equal(ims[r], images[m][r])


# ---- prefetch (NEXT-3, reading #29) --------------------------------------------------------
def test_prefetch_worked_example():
    # cap 10: B(3)@0, C(3)@3; A(7) evicts both (LRU prefix B, C) and loads at 0; once every swap
    # is acked, the policy prefetches C (same count as B, later arrival) into the free [7, 10);
    # the next request for C then needs no swap
    for pf in (False, True):
        e = S.Engine(S.EngineConfig(3, 0, 1, 4, 1, cap=10, sizes=[7, 3, 3], prefetch=pf))
        assert swaps(drive_resident(e, 1, 1.0)) == [("load", 1, 0)]
        assert swaps(drive_resident(e, 2, 2.0)) == [("load", 2, 3)]
        decs = drive_resident(e, 0, 3.0)
        got = swaps(decs)
        assert got[:3] == [("offload", 1, 0), ("offload", 2, 3), ("load", 0, 0)]
        if pf:
            assert got[3:] == [("load", 2, 7)]
            assert [(d["model"], d["off"]) for d in decs if d.get("prefetch")] == [(2, 7)]
            assert swaps(drive_resident(e, 2, 4.0)) == []              # prefetched: no swap
        else:
            assert got[3:] == []
            assert swaps(drive_resident(e, 2, 4.0)) == [("load", 2, 7)]


def test_prefetch_skips_candidates_that_do_not_fit():
    # the most frequent evicted model (A, 8) does not fit the free space; the next one (B, 2) does
    e = S.Engine(S.EngineConfig(3, 0, 1, 4, 1, cap=10, sizes=[8, 2, 9], prefetch=True))
    drive_resident(e, 0, 1.0)
    drive_resident(e, 0, 1.5)
    drive_resident(e, 1, 2.0)          # B(2) fits beside A at 8
    decs = drive_resident(e, 2, 3.0)   # C(9) evicts A and B; free [9, 10) is too small for anyone
    assert swaps(decs) == [("offload", 0, 0), ("offload", 1, 8), ("load", 2, 0)]
    assert not any(d.get("prefetch") for d in decs)


@pytest.mark.parametrize("seed", range(25))
def test_prefetch_random_traces(seed):
    """With prefetch on: invariants, completion and per-model FIFO hold; a prefetch load is the
    only swap decision of its step (the link was idle) and never comes with an eviction."""
    rng = random.Random(500 + seed)
    n = rng.randint(2, 6)
    sizes = [rng.randint(1, 5) for _ in range(n)]
    cap = rng.randint(max(sizes), 14)
    tp = rng.choice([1, 2])
    e = S.Engine(S.EngineConfig(n, 0, tp, rng.choice([1, 2, 4]), rng.choice([1, 2]), cap=cap, sizes=sizes,
                                prefetch=True))
    arrivals = sorted((rng.uniform(0, 10), rng.choices(range(n), weights=[i + 1 for i in range(n)])[0])
                      for _ in range(30))
    rid_model, done, pend, n_pf = {}, [], [], 0
    t, ai = 0.0, 0
    while ai < len(arrivals) or pend:
        if ai < len(arrivals) and (not pend or rng.random() < 0.5):
            t = max(t, arrivals[ai][0])
            rid_model[ai] = arrivals[ai][1]
            out = e.step(ev("arrival", t, rid=ai, model=arrivals[ai][1]))
            ai += 1
        else:
            i = rng.randrange(len(pend))
            if pend[i]["dec"] == "batch":
                i = next(j for j, x in enumerate(pend) if x["dec"] == "batch")
            d = pend.pop(i)
            t += 0.01
            if d["dec"] == "batch":
                out = e.step(ev("batch_done", t, batch=d["id"]))
            else:
                out = []
                for r in range(tp):
                    out += e.step(ev("ack", t, entry=d["id"], rank=r))
        sw = [d for d in out if d["dec"] in ("load", "offload")]
        if any(d.get("prefetch") for d in sw):
            n_pf += 1
            assert len(sw) == 1
        for d in out:
            if d["dec"] in ("load", "offload", "batch"):
                pend.append(d)
            if d["dec"] == "complete":
                done += d["rids"]
    assert sorted(done) == list(range(len(arrivals)))
    for m in range(n):
        mine = [r for r in done if rid_model[r] == m]
        assert mine == sorted(mine)


# ---- reading #30: victim_policy 1, the minimum-cost window (NEXT-4 knapsack) -------------------
def cfg1(sizes, cap, mb=4, D=1, tp=1):
    return S.EngineConfig(len(sizes), 0, tp, mb, D, cap=cap, sizes=list(sizes), victim_policy=1)


def test_min_cost_window_worked_example():
    # cap 10: A(4) loads at 0, C(4) at 4, B(2) at 8 (first fit), LRU order A, C, B. D(2) finds no
    # free range: the LRU-prefix policy (#28) evicts A (the oldest, 4 bytes) and loads D at 0; the
    # min-cost window (#30) evicts only B (2 bytes) and loads D at 8
    for pol, want in ((0, [("offload", 0, 0), ("load", 3, 0)]), (1, [("offload", 1, 8), ("load", 3, 8)])):
        e = S.Engine(S.EngineConfig(4, 0, 1, 4, 1, cap=10, sizes=[4, 2, 4, 2], victim_policy=pol))
        for t, m in ((1.0, 0), (2.0, 2), (3.0, 1)):
            drive_resident(e, m, t)
        assert (e.off_of[0], e.off_of[2], e.off_of[1]) == (0, 4, 8)
        assert swaps(drive_resident(e, 3, 4.0)) == want, pol


def brute_window(before_off, sizes, cap, m, eligible, key):
    """Every integer offset o (not only the candidate starts): the feasible window with the least
    (bytes evicted, victims, newest victim key, o)."""
    best = None
    for o in range(cap - sizes[m] + 1):
        over = [w for w, lo in before_off.items() if lo < o + sizes[m] and o < lo + sizes[w]]
        if any(w not in eligible for w in over):
            continue
        cost = (sum(sizes[w] for w in over), len(over), max((key(w) for w in over), default=()), o)
        if best is None or cost < best[0]:
            best = (cost, o, over)
    return best


@pytest.mark.parametrize("seed", range(60))
def test_min_cost_window_vs_brute_force(seed):
    """Blocking requests over random heterogeneous sizes: every decision of victim_policy 1 equals
    the brute force over all integer offsets (so the candidate-start restriction loses nothing),
    offloads in victim-key order, invariants after every event."""
    rng = random.Random(7000 + seed)
    n = rng.randint(2, 6)
    sizes = [rng.randint(1, 5) for _ in range(n)]
    cap = rng.randint(max(sizes), 14)
    e = S.Engine(cfg1(sizes, cap))
    t = 0.0
    for _ in range(30):
        m = rng.randrange(n)
        t += 1.0
        if e.state[m] == S.RESIDENT:
            drive_resident(e, m, t)
            continue
        before = {w: e.off_of[w] for w in range(n) if e.off_of[w] is not None}
        key = lambda w: (0, e.last_use[w], w)
        elig = {w for w in range(n) if e.state[w] == S.RESIDENT and e.outstanding[w] == 0}
        got = swaps(drive_resident(e, m, t))
        free = brute_window(before, sizes, cap, m, set(), key)
        if free is not None:                      # a free range exists: plain first fit
            assert got[0] == ("load", m, free[1]), (got, free)
            continue
        best = brute_window(before, sizes, cap, m, elig, key)
        assert best is not None
        want = [("offload", w, before[w]) for w in sorted(best[2], key=key)] + [("load", m, best[1])]
        assert got[:len(want)] == want, (sizes, cap, before, got, want)


@pytest.mark.parametrize("seed", range(20))
def test_min_cost_window_equal_sizes_is_textbook_lru(seed):
    """Equal sizes: every window costs one model, the newest-key tie-break picks the LRU victim,
    so victim_policy 1 reduces to textbook LRU exactly like policy 0."""
    rng = random.Random(9000 + seed)
    n, k = rng.randint(2, 8), rng.randint(1, 4)
    size = rng.randint(2, 7)
    cap = k * size + rng.randrange(size)
    e = S.Engine(cfg1([size] * n, cap))
    acc = [rng.randrange(n) for _ in range(60)]
    evicted = []
    for i, m in enumerate(acc):
        for d in drive_resident(e, m, float(i + 1)):
            if d["dec"] == "offload":
                evicted.append(d["model"])
    assert evicted == S.textbook_lru_evictions(acc, k)


@pytest.mark.parametrize("seed", range(15))
def test_min_cost_window_open_loop_invariants(seed):
    """Open-loop arrivals with random ack / completion interleaving under victim_policy 1:
    Engine.check invariants at every step and every request completes (replay of its own
    event log reproduces the decisions)."""
    rng = random.Random(11000 + seed)
    n = rng.randint(3, 6)
    sizes = [rng.randint(1, 5) for _ in range(n)]
    cap = rng.randint(max(sizes) + 1, 14)
    c = cfg1(sizes, cap, mb=rng.randint(1, 3), D=rng.randint(1, 2))
    arrivals = sorted((rng.uniform(0, 5), rid, rng.randrange(n)) for rid in range(40))
    events, decisions, t_done, _ = S.simulate(c, S.Costs(1, 1e9, 1e9, alpha=1e-3, gamma0=2e-3),
                                              [(rid, m, t) for t, rid, m in arrivals], token_len=2)
    assert len(t_done) == 40
    rdecs, _ = S.replay(c, events)
    assert rdecs == decisions
