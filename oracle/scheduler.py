"""C1 — engine scheduling semantics (oracle side): per-model FIFO queues, oldest-head batch
scheduling, LRU replacement with load/offload entries, ack-based completion.

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

Paper: P:74 (per-model queues with timestamps; "repeatedly picks a queue to pop oldest request
objects, then packs and submits them ... as a single batch entry"), P:94 (load entries load or
offload one instance), P:105 (async load entries; "completed when every worker finishes ...
and sends a response back"; batches submitted "only after that model has been fully loaded";
later batches for other models proceed), P:114 ("scheduled in batches based on the oldest
timestamp", "LRU replacement policy"), P:129 (offload submitted first, overlapped with load).
Readings: #1 global oldest head, ties by registration order; #2 take what is
queued up to max_batch; #3 last_use = batch submission time; #4 victim eligibility; #5
chunk-paired in-place swap (victim's range handed to the requester at once); #7 concurrent swaps
allowed when space permits; #21 tie-breaks by registration order; #24 requests for a LOADING
model queue; #26 at most D batches in flight per TP group (default 1); #28 placement of models
of different sizes (NEXT-4, §6): each rank's region holds `cap` bytes, model m occupies
[off, off + size[m]) on every rank, loads go to the lowest-address free range that fits (first
fit); with no fit, eligible victims are removed in victim-key order until a first fit exists and
only the victims overlapping that range are offloaded. Equal sizes reduce to k slots
(cap = k, size 1: off is the slot index); #29 prefetch (NEXT-3, "more sophisticated
fetching algorithms"): when enabled and no load/offload is pending, after SCHEDULE the EVICTED
model with an empty queue that appears most often among the last 32 arrivals (ties: latest
arrival, then registration order) is loaded into the lowest free range that fits it; it never
evicts, and candidates that do not fit are skipped.

`Engine` is a deterministic state machine.  `step(event)` applies one event and returns the
decisions it caused.  Two drivers use it:
  * `replay(events)`: feed the CUDA engine's recorded ordered event log and compare decisions;
  * `simulate(...)`: a virtual-time discrete-event simulation with alpha-beta durations.
"""
import heapq
from collections import deque
from dataclasses import dataclass, field

EVICTED, LOADING, RESIDENT, OFFLOADING = 0, 1, 2, 3
STATE_NAMES = {EVICTED: "EVICTED", LOADING: "LOADING", RESIDENT: "RESIDENT", OFFLOADING: "OFFLOADING"}
INF_D = 1 << 30


@dataclass
class EngineConfig:
    n_models: int
    k_slots: int
    tp: int
    max_batch: int
    max_inflight: int = 1       # D (reading #26)
    cap: int = None             # region bytes per rank (reading #28); None: k_slots unit slots
    sizes: list = None          # placement bytes per model; None: 1 each
    prefetch: bool = False      # reading #29
    victim_policy: int = 0      # reading #28 (0: LRU prefix, first fit) or #30 (1: min-cost window)

    def region(self):
        return self.k_slots if self.cap is None else self.cap

    def size(self, m):
        return 1 if self.sizes is None else self.sizes[m]


def config_from_trace(cfg):
    """EngineConfig from the {"cfg": ...} header line of the engine's trace (mpsw_trace_dump)."""
    c = cfg["cfg"]
    return EngineConfig(len(c["sizes"]), 0, c["acks"], c["max_batch"], c["D"], cap=c["cap"], sizes=list(c["sizes"]),
                        prefetch=bool(c.get("prefetch", False)), victim_policy=int(c.get("victim_policy", 0)))


def read_trace(path):
    """(EngineConfig, events, decisions) of an engine trace file."""
    import json
    cfg, evs, decs = None, [], []
    for line in open(path):
        o = json.loads(line)
        if "cfg" in o:
            cfg = config_from_trace(o)
        elif "ev" in o:
            evs.append(o)
        else:
            decs.append(o)
    return cfg, evs, decs


class InvariantViolation(Exception):
    pass


@dataclass
class Engine:
    cfg: EngineConfig
    queue: list = field(init=False)
    state: list = field(init=False)
    last_use: list = field(init=False)
    outstanding: list = field(init=False)
    off_of: list = field(init=False)         # model -> offset of its range, None if it owns none
    pending: dict = field(init=False)        # entry id -> [kind, model, acks left, set(ranks acked)]
    batches: dict = field(init=False)        # batch id -> (model, rids)
    inflight: int = 0
    next_id: int = 0
    HISTORY = 32                             # arrivals remembered by the prefetch policy

    def __post_init__(self):
        n = self.cfg.n_models
        self.recent = deque(maxlen=self.HISTORY)
        self.last_arrival = [float("-inf")] * n
        self.queue = [deque() for _ in range(n)]
        self.state = [EVICTED] * n
        self.last_use = [float("-inf")] * n
        self.outstanding = [0] * n
        self.off_of = [None] * n
        self.pending = {}
        self.batches = {}

    # ---- helpers -------------------------------------------------------------------------
    def _eid(self):
        e = self.next_id
        self.next_id += 1
        return e

    def _head_key(self, m):
        return (self.queue[m][0][1], m)

    def _load(self, m, off, out):
        e = self._eid()
        self.off_of[m] = off
        self.state[m] = LOADING
        self.pending[e] = ["load", m, self.cfg.tp, set()]
        out.append({"dec": "load", "id": e, "model": m, "off": off})

    def _offload(self, v, out):
        e = self._eid()
        off = self.off_of[v]
        self.off_of[v] = None
        self.state[v] = OFFLOADING
        self.pending[e] = ["offload", v, self.cfg.tp, set()]
        out.append({"dec": "offload", "id": e, "model": v, "off": off})

    def _first_fit(self, need, without=()):
        """Lowest offset o such that [o, o + need) lies in the region and overlaps no range
        owned by a model outside `without`; None if there is none."""
        owned = sorted((self.off_of[m], self.off_of[m] + self.cfg.size(m)) for m in range(self.cfg.n_models)
                       if self.off_of[m] is not None and m not in without)
        o = 0
        for lo, hi in owned:
            if lo - o >= need:
                return o
            o = max(o, hi)
        return o if self.cfg.region() - o >= need else None

    def _min_cost_window(self, need, vics):
        """Reading #30 (victim_policy 1): among windows [o, o + need) inside the region whose
        every overlapping model is an eligible victim, the one minimising (bytes evicted, number
        of victims, the newest victim key, o); a victim key is (queue non-empty, last_use, model).
        Windows starting at 0 or at the end of an owned range suffice: sliding any feasible
        window left to the nearest such start only drops overlapped ranges. None if no window is
        feasible. Returns (o, set of victims)."""
        key = lambda v: (1 if self.queue[v] else 0, self.last_use[v], v)
        owned = [(self.off_of[v], self.off_of[v] + self.cfg.size(v), v) for v in range(self.cfg.n_models)
                 if self.off_of[v] is not None]
        best = None
        for o in sorted({0} | {hi for _, hi, _ in owned}):
            if o + need > self.cfg.region():
                continue
            over = [v for lo, hi, v in owned if lo < o + need and o < hi]
            if any(v not in vics for v in over):
                continue
            cost = (sum(self.cfg.size(v) for v in over), len(over), max(key(v) for v in over) if over else (), o)
            if best is None or cost < best[0]:
                best = (cost, o, set(over))
        return None if best is None else (best[1], best[2])

    # ---- SCHEDULE ----------------------------------------------------------
    def schedule(self, now, out):
        blocked = set()
        while True:
            cands = [m for m in range(self.cfg.n_models) if self.queue[m] and m not in blocked]
            if not cands:
                self._prefetch(out)
                return
            m = min(cands, key=self._head_key)
            st = self.state[m]
            if st == RESIDENT:
                if self.inflight < self.cfg.max_inflight:
                    n = min(self.cfg.max_batch, len(self.queue[m]))
                    rids = [self.queue[m].popleft()[0] for _ in range(n)]
                    e = self._eid()
                    self.batches[e] = (m, rids)
                    self.last_use[m] = now
                    self.outstanding[m] += 1
                    self.inflight += 1
                    out.append({"dec": "batch", "id": e, "model": m, "rids": rids})
                else:
                    blocked.add(m)
            elif st in (LOADING, OFFLOADING):
                blocked.add(m)
            else:  # EVICTED
                need = self.cfg.size(m)
                o = self._first_fit(need)
                if o is not None:
                    self._load(m, o, out)
                else:
                    hk = self._head_key(m)
                    vics = sorted((v for v in range(self.cfg.n_models)
                                   if self.state[v] == RESIDENT and self.outstanding[v] == 0
                                   and (not self.queue[v] or self._head_key(v) > hk)),
                                  key=lambda v: (1 if self.queue[v] else 0, self.last_use[v], v))
                    if self.cfg.victim_policy == 1:
                        w = self._min_cost_window(need, vics)
                        if w is not None:
                            o, ws = w
                            for v in vics:                       # evicted in victim-key order
                                if v in ws:
                                    self._offload(v, out)
                            self._load(m, o, out)
                        blocked.add(m)
                        continue
                    for j in range(1, len(vics) + 1):
                        o = self._first_fit(need, set(vics[:j]))
                        if o is None:
                            continue
                        for w in vics[:j]:
                            lo = self.off_of[w]
                            if lo < o + need and o < lo + self.cfg.size(w):
                                self._offload(w, out)
                        self._load(m, o, out)
                        break
                blocked.add(m)

    def _prefetch(self, out):
        """Reading #29: one prefetch load into free space when the link is idle."""
        if not self.cfg.prefetch or self.pending:
            return
        count = {}
        for m in self.recent:
            count[m] = count.get(m, 0) + 1
        cands = [m for m in count if self.state[m] == EVICTED and not self.queue[m]]
        for m in sorted(cands, key=lambda m: (-count[m], -self.last_arrival[m], m)):
            o = self._first_fit(self.cfg.size(m))
            if o is not None:
                self._load(m, o, out)
                out[-1]["prefetch"] = True
                return

    # ---- events ----------------------------------------------------------------------------
    def step(self, ev):
        """Apply one event dict; return the list of decision dicts it caused."""
        out = []
        kind = ev["ev"]
        now = ev["t"]
        if kind == "arrival":
            m = ev["model"]
            if not 0 <= m < self.cfg.n_models:
                out.append({"dec": "reject", "rid": ev["rid"], "status": "ENOENT"})
                return out
            self.queue[m].append((ev["rid"], now))
            self.recent.append(m)
            self.last_arrival[m] = now
        elif kind == "ack":
            e, r = ev["entry"], ev["rank"]
            if e not in self.pending:
                raise InvariantViolation(f"ack for unknown entry {e}")
            p = self.pending[e]
            if r in p[3]:
                raise InvariantViolation(f"duplicate ack entry {e} rank {r}")
            p[3].add(r)
            p[2] -= 1
            if p[2] == 0:
                del self.pending[e]
                self.state[p[1]] = RESIDENT if p[0] == "load" else EVICTED
        elif kind == "batch_done":
            b = ev["batch"]
            if b not in self.batches:
                raise InvariantViolation(f"unknown batch {b}")
            m, rids = self.batches.pop(b)
            self.outstanding[m] -= 1
            self.inflight -= 1
            out.append({"dec": "complete", "id": b, "rids": rids})
        elif kind == "cmd_swap_in":
            m = ev["model"]
            st = self.state[m]
            if st in (RESIDENT, LOADING):
                out.append({"dec": "noop", "model": m})
            elif st == OFFLOADING:
                out.append({"dec": "reject", "model": m, "status": "EBUSY"})
            else:
                o = self._first_fit(self.cfg.size(m))
                if o is None:
                    out.append({"dec": "reject", "model": m, "status": "ENOMEM"})
                else:
                    self._load(m, o, out)
        elif kind == "cmd_swap_out":
            m = ev["model"]
            st = self.state[m]
            if st in (EVICTED, OFFLOADING):
                out.append({"dec": "noop", "model": m})
            elif st == LOADING or self.outstanding[m] > 0:
                out.append({"dec": "reject", "model": m, "status": "EBUSY"})
            else:
                self._offload(m, out)
        else:
            raise ValueError(kind)
        self.schedule(now, out)
        self.check()
        return out

    def check(self):
        """Invariants: owned ranges lie inside the region and never overlap (so bytes held per
        rank <= cap <= budget), LOADING/RESIDENT models and only they own a range, a model with
        in-flight batches is RESIDENT, inflight <= D."""
        ranges = []
        for m in range(self.cfg.n_models):
            if self.outstanding[m] > 0 and self.state[m] != RESIDENT:
                raise InvariantViolation(f"model {m} has in-flight batches but is {STATE_NAMES[self.state[m]]}")
            owns = self.state[m] in (LOADING, RESIDENT)
            if owns != (self.off_of[m] is not None):
                raise InvariantViolation("range ownership")
            if owns:
                ranges.append((self.off_of[m], self.off_of[m] + self.cfg.size(m)))
        ranges.sort()
        for i, (lo, hi) in enumerate(ranges):
            if lo < 0 or hi > self.cfg.region():
                raise InvariantViolation("range outside the region")
            if i and lo < ranges[i - 1][1]:
                raise InvariantViolation("overlapping ranges")
        if self.inflight > self.cfg.max_inflight:
            raise InvariantViolation("D exceeded")


def replay(cfg: EngineConfig, events):
    """Feed a recorded ordered event log; returns the flat decision list."""
    eng = Engine(cfg)
    decisions = []
    for ev in events:
        decisions.extend(eng.step(ev))
    return decisions, eng


# ------------------------------------------------------------------------------------------
# Virtual-time discrete-event simulation (alpha-beta durations; S:21-74 ordering by (t, seq)).
# ------------------------------------------------------------------------------------------
@dataclass
class Costs:
    shard_bytes: int
    b_in: float
    b_out: float
    alpha: float = 0.0          # per chunk
    chunk: int = 64 << 20
    gamma0: float = 0.0         # forward = gamma0 + gamma1 * B * L
    gamma1: float = 0.0
    writeback: bool = True
    rank_delay: tuple = ()      # optional extra per-rank copy delay (fault injection)


def simulate(cfg: EngineConfig, costs: Costs, arrivals, token_len: int, blocking=False):
    """arrivals: list of (rid, model, t_arr) (open loop) or, with blocking=True, a list of
    (rid, model) issued one after the previous completes (P:127 alternating blocking).
    Returns (events, decisions, t_done dict, entry_log) with events in processing order.
    Models are equal-size here (one shard_bytes): the chunk gates are keyed by range offset."""
    eng = Engine(cfg)
    pq, seq = [], 0

    def push(t, ev):
        nonlocal seq
        heapq.heappush(pq, (t, seq, ev))
        seq += 1

    tp = cfg.tp
    h2d_free = [0.0] * tp
    d2h_free = [0.0] * tp
    comp_free = 0.0
    slot_chunk_free = {}        # (rank, slot) -> list of times chunk i may be overwritten
    entry_log = {}
    from .costmodel import chunk_sizes
    sizes = chunk_sizes(costs.shard_bytes, costs.chunk)
    t_done = {}
    bl = list(arrivals)
    if blocking:
        if bl:
            rid, m = bl.pop(0)
            push(0.0, {"ev": "arrival", "rid": rid, "model": m})
    else:
        for rid, m, t in arrivals:
            push(t, {"ev": "arrival", "rid": rid, "model": m})
    events, decisions = [], []
    while pq:
        t, _, ev = heapq.heappop(pq)
        ev = dict(ev, t=t)
        events.append(ev)
        decs = eng.step(ev)
        decisions.extend(decs)
        for dcs in decs:
            k = dcs["dec"]
            if k == "offload":
                entry_log[dcs["id"]] = {"kind": "offload", "submit": t, "done": {}}
                for r in range(tp):
                    extra = costs.rank_delay[r] if r < len(costs.rank_delay) else 0.0
                    if costs.writeback:
                        tt = max(t, d2h_free[r]) + extra
                        times = []
                        for c in sizes:
                            tt += costs.alpha + c / costs.b_out
                            times.append(tt)
                        d2h_free[r] = tt
                    else:                       # clean eviction: nothing to copy
                        tt, times = t, [t] * len(sizes)
                    slot_chunk_free[(r, dcs["off"])] = times
                    entry_log[dcs["id"]]["done"][r] = tt
                    push(tt, {"ev": "ack", "entry": dcs["id"], "rank": r})
            elif k == "load":
                entry_log[dcs["id"]] = {"kind": "load", "submit": t, "done": {}}
                for r in range(tp):
                    extra = costs.rank_delay[r] if r < len(costs.rank_delay) else 0.0
                    tt = max(t, h2d_free[r]) + extra
                    gate = slot_chunk_free.get((r, dcs["off"]), [])
                    for i, c in enumerate(sizes):
                        if i < len(gate):
                            tt = max(tt, gate[i])
                        tt += costs.alpha + c / costs.b_in
                    h2d_free[r] = tt
                    slot_chunk_free[(r, dcs["off"])] = []
                    entry_log[dcs["id"]]["done"][r] = tt
                    push(tt, {"ev": "ack", "entry": dcs["id"], "rank": r})
            elif k == "batch":
                start = max(t, comp_free)
                dur = costs.gamma0 + costs.gamma1 * len(dcs["rids"]) * token_len
                comp_free = start + dur
                push(comp_free, {"ev": "batch_done", "batch": dcs["id"]})
            elif k == "complete":
                for rid in dcs["rids"]:
                    t_done[rid] = t
                if blocking and bl:
                    rid, m = bl.pop(0)
                    push(t, {"ev": "arrival", "rid": rid, "model": m})
    return events, decisions, t_done, entry_log


def textbook_lru_evictions(accesses, k):
    """Brute-force textbook LRU (the S:296 oracle): returns the list of evicted keys."""
    cache, ev = [], []
    for a in accesses:
        if a in cache:
            cache.remove(a)
            cache.append(a)
            continue
        if len(cache) >= k:
            ev.append(cache.pop(0))
        cache.append(a)
    return ev
