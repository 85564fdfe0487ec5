"""C3 — swap data semantics at byte/chunk level, and the memory budget (oracle side).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

P:94: a load entry loads or offloads "the parameters of an instance"; loading and
offloading run concurrently on two extra streams; offloaded parameters stay in pinned
host memory (the host copy is the master); "our asynchronous implementation overlaps
the two [offload and load]".  North star: "eviction never races an in-flight request", and a
per-GPU memory budget.  DESIGN.md reading #5: chunk-paired in-place swap.

Per rank, the parameter region is k slots of S_r bytes, each split into chunks of c bytes.
  load(m -> s):            slot[s][i] := arena[m][i]                      for every chunk i
  paired swap(v -> m, s):  for i in order: arena[v][i] := slot[s][i] (writeback) THEN
                                           slot[s][i] := arena[m][i]
  offload(v):              arena[v] := slot[s] (writeback) or untouched (clean eviction)
Budget: every byte held by any model lives inside one of the k slots, so bytes held <= k*S_r
<= budget at every instant (stricter than SPEC's slot count).

`SwapModel` takes decisions of unit-size scheduler configs (off = slot index).
`RegionSwapModel` is the byte-level version for models of different sizes (reading #28): the
region of each rank is `cap` bytes and a model's shard lives at [off, off + S_m,r).
"""
import numpy as np

from .checksum import checksum


class SwapModel:
    def __init__(self, images, k_slots, chunk, writeback=True):
        """images: dict model -> list (per rank) of uint8 arrays (the C0 shard images)."""
        self.host = {m: [im.copy() for im in ims] for m, ims in images.items()}
        m0 = next(iter(images))
        self.tp = len(images[m0])
        self.S = images[m0][0].size
        self.k = k_slots
        self.chunk = chunk
        self.writeback = writeback
        self.slot = [[np.zeros(self.S, np.uint8) for _ in range(k_slots)] for _ in range(self.tp)]
        self.owner = [None] * k_slots
        self.peak_bytes_held = 0

    def _held(self):
        return sum(self.S for o in self.owner if o is not None)

    def load(self, m, s):
        assert self.owner[s] is None, "load into an occupied slot"
        self.owner[s] = m
        for r in range(self.tp):
            for i in range(0, self.S, self.chunk):
                self.slot[r][s][i:i + self.chunk] = self.host[m][r][i:i + self.chunk]
        self.peak_bytes_held = max(self.peak_bytes_held, self._held())

    def offload(self, s):
        v = self.owner[s]
        assert v is not None
        if self.writeback:
            for r in range(self.tp):
                self.host[v][r][:] = self.slot[r][s]
        self.owner[s] = None

    def paired(self, s, m):
        v = self.owner[s]
        assert v is not None
        for r in range(self.tp):
            for i in range(0, self.S, self.chunk):
                if self.writeback:
                    self.host[v][r][i:i + self.chunk] = self.slot[r][s][i:i + self.chunk]
                self.slot[r][s][i:i + self.chunk] = self.host[m][r][i:i + self.chunk]
        self.owner[s] = m
        self.peak_bytes_held = max(self.peak_bytes_held, self._held())

    def apply(self, decisions):
        """Apply engine decisions (oracle.scheduler format) in order; a load that directly
        follows an offload of the same slot is the paired swap."""
        i = 0
        while i < len(decisions):
            d = decisions[i]
            if d["dec"] == "offload":
                nxt = decisions[i + 1] if i + 1 < len(decisions) else None
                if nxt and nxt["dec"] == "load" and nxt["off"] == d["off"]:
                    self.paired(d["off"], nxt["model"])
                    i += 2
                    continue
                self.offload(d["off"])
            elif d["dec"] == "load":
                self.load(d["model"], d["off"])
            i += 1

    def expected_slot_hashes(self):
        """{model: [hash per rank]} for every model resident in a slot."""
        return {m: [checksum(self.slot[r][s]) for r in range(self.tp)]
                for s, m in enumerate(self.owner) if m is not None}

    def expected_host_hashes(self):
        return {m: [checksum(a) for a in ims] for m, ims in self.host.items()}


class RegionSwapModel:
    """C3 for models of different sizes (reading #28, NEXT-4). Per rank: one region of
    `cap` bytes; a resident model m occupies [off_m, off_m + S_m,r). Decisions apply in engine
    order: offload(v) writes v's bytes back to its arena (writeback) or leaves the arena
    untouched (clean eviction) and frees the range; load(m, off) copies m's arena into
    [off, off + S_m,r). The engine overlaps an offload with the loads that reuse its bytes
    chunk by chunk, gating every load chunk on the D2H of the bytes it overwrites, which gives
    exactly this sequential result."""

    def __init__(self, images, cap, writeback=True):
        """images: dict model -> list (per rank) of uint8 arrays (the C0 shard images)."""
        self.host = {m: [im.copy() for im in ims] for m, ims in images.items()}
        self.tp = len(next(iter(images.values())))
        self.cap = cap
        self.writeback = writeback
        self.region = [np.zeros(cap, np.uint8) for _ in range(self.tp)]
        self.off = {}

    def apply(self, decisions):
        for d in decisions:
            m = d.get("model")
            if d["dec"] == "offload":
                o = self.off.pop(m)
                assert o == d["off"], "offload of a range the model does not own"
                if self.writeback:
                    for r in range(self.tp):
                        n = self.host[m][r].size
                        self.host[m][r][:] = self.region[r][o:o + n]
            elif d["dec"] == "load":
                o = d["off"]
                for r in range(self.tp):
                    n = self.host[m][r].size
                    assert o + n <= self.cap, "range beyond the region"
                    for w, ow in self.off.items():     # never overwrite a resident model
                        nw = self.host[w][r].size
                        assert ow + nw <= o or o + n <= ow, "load overlaps a resident model"
                    self.region[r][o:o + n] = self.host[m][r]
                self.off[m] = o

    def expected_resident_hashes(self):
        """{model: [hash per rank]} of every model the decisions left resident."""
        return {m: [checksum(self.region[r][o:o + self.host[m][r].size]) for r in range(self.tp)]
                for m, o in self.off.items()}
