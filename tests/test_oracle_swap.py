"""Pins for oracle/swap.py (C3): invariants (i)-(iv) by brute force on tiny images and all
swap/request sequences of length <= 4 over 3 tiny models, k in {1, 2}."""
import itertools

import numpy as np
import pytest

from synth import opt_dims
from oracle import layout, swap, checksum
from oracle import scheduler as S


def images(nm, tp, dtype="bf16"):
    d = opt_dims("tiny")
    return {m: [layout.shard_image(d, tp, r, 100 + m, dtype) for r in range(tp)] for m in range(nm)}


@pytest.mark.parametrize("writeback", [True, False])
def test_paired_swap_roundtrip(writeback):
    ims = images(2, 2)
    sm = swap.SwapModel(ims, 1, chunk=1000, writeback=writeback)
    sm.load(0, 0)
    for r in range(2):
        assert np.array_equal(sm.slot[r][0], ims[0][r])
    sm.paired(0, 1)
    for r in range(2):
        assert np.array_equal(sm.slot[r][0], ims[1][r])          # (iii) resident == image
        assert np.array_equal(sm.host[0][r], ims[0][r])          # (iv) writeback round trip
    assert sm.peak_bytes_held <= 1 * sm.S                        # (i) budget


def test_exhaustive_sequences():
    ims = images(3, 1)
    ref = {m: [checksum.checksum(a) for a in v] for m, v in ims.items()}
    ops = [("req", 0), ("req", 1), ("req", 2), ("out", 0), ("out", 1), ("in", 2)]
    n_seq = 0
    for k in (1, 2):
        for L in range(1, 5):
            for seq in itertools.product(ops, repeat=L):
                eng = S.Engine(S.EngineConfig(3, k, 1, 4, 1))
                sm = swap.SwapModel(ims, k, chunk=777, writeback=True)
                t = 0.0
                for rid, (op, m) in enumerate(seq):
                    t += 1
                    evs = [{"ev": {"req": "arrival", "out": "cmd_swap_out", "in": "cmd_swap_in"}[op],
                            "t": t, "model": m, "rid": rid}]
                    while evs:
                        decs = eng.step(evs.pop(0))
                        sm.apply(decs)
                        for d in decs:
                            if d["dec"] in ("load", "offload"):
                                evs.append({"ev": "ack", "t": t, "entry": d["id"], "rank": 0})
                            elif d["dec"] == "batch":
                                # a batch runs only on a fully resident, bit-exact model
                                assert sm.owner[eng.off_of[d["model"]]] == d["model"]
                                assert checksum.checksum(sm.slot[0][eng.off_of[d["model"]]]) == ref[d["model"]][0]
                                evs.append({"ev": "batch_done", "t": t, "batch": d["id"]})
                    assert sum(o is not None for o in sm.owner) <= k
                for m, hs in sm.expected_slot_hashes().items():
                    assert hs == ref[m]
                assert sm.expected_host_hashes() == ref
                n_seq += 1
    assert n_seq > 2000
