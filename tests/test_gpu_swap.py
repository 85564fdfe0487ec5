"""GPU parity of the swap path (a2/a3/a8): resident bytes are bit-exact with the oracle's C0
image (checksum C4 + sampled element reads), writeback leaves host arenas unchanged, random
swap sequences match oracle/swap.py, every swap mode and chunk size."""
import json
import os
import random

import numpy as np
import pytest

from synth import opt_dims
from oracle import layout, checksum
from oracle import scheduler as S
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("tp", [1, 2])
def test_fill_and_swap_in_bit_exact(mode, tp):
    M = need_gpu()
    d = opt_dims("small")
    S_ = layout.shard_bytes(d, tp)
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + 4096, swap_mode=mode, chunk_bytes=1 << 20) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 77)
        for r in range(tp):
            img = layout.shard_image(d, tp, r, 77)
            assert np.array_equal(ctx.model_arena(m, r), img)       # product C0 == oracle C0
        ctx.wait(ctx.swap_in(m))
        assert ctx.residency(m) == M.RESIDENT
        for r in range(tp):
            img = layout.shard_image(d, tp, r, 77)
            assert ctx.checksum(m, r) == checksum.checksum(img)
            assert ctx.checksum(m, r, on_device=False) == checksum.checksum(img)
            assert np.array_equal(ctx.peek(m, r, 0, S_), img)


def test_register_with_caller_shards_and_fp32():
    M = need_gpu()
    d = opt_dims("tiny")
    imgs = [layout.shard_image(d, 2, r, 5, "fp32") for r in range(2)]
    with M.Ctx(device_ids=(0, 0), budget=imgs[0].size + 4096, dtype=M.FP32) as ctx:
        m = ctx.register_model(d, shards=imgs)
        ctx.wait(ctx.swap_in(m))
        for r in range(2):
            assert ctx.checksum(m, r) == checksum.checksum(imgs[r])


@pytest.mark.parametrize("writeback", [1, 0])
@pytest.mark.parametrize("mode", [1, 2])
def test_random_swap_sequences_match_oracle(writeback, mode, tmp_path):
    """60 random requests / explicit swap-ins / swap-outs over 4 models with room for 2: after
    every step each RESIDENT range equals its C0 image; at the end the engine's recorded decisions
    are applied to the oracle's byte-level swap model (oracle/swap.py RegionSwapModel), whose
    predicted resident and host-arena hashes must equal the device / host checksums."""
    M = need_gpu()
    from oracle.swap import RegionSwapModel
    d = opt_dims("tiny")
    tp, nm, k = 2, 4, 2
    S_ = layout.shard_bytes(d, tp)
    imgs = {m: [layout.shard_image(d, tp, r, 300 + m) for r in range(tp)] for m in range(nm)}
    ref = {m: [checksum.checksum(a) for a in v] for m, v in imgs.items()}
    rnd = random.Random(writeback * 10 + mode)
    with M.Ctx(device_ids=(0,) * tp, budget=k * ((S_ + 4095) // 4096 * 4096), swap_mode=mode, chunk_bytes=4096,
               writeback=writeback, max_batch=2, max_tokens=4, trace=1) as ctx:
        ids = [ctx.register_model(d, shards=imgs[m]) for m in range(nm)]
        for step in range(60):
            m = rnd.randrange(nm)
            if rnd.random() < 0.6:
                rid, out = ctx.request(ids[m], np.array([1, 2, 3], np.int32))   # LRU swap if needed
                ctx.wait_request(rid, 60)
            elif rnd.random() < 0.5:
                try:
                    ctx.wait(ctx.swap_out(ids[m]))
                except M.MpswError as e:
                    assert e.status == M.EBUSY
            else:
                try:
                    ctx.wait(ctx.swap_in(ids[m]))
                except M.MpswError as e:
                    assert e.status in (M.ENOMEM, M.EBUSY)
            for mm in range(nm):
                if ctx.residency(ids[mm]) == M.RESIDENT:
                    for r in range(tp):
                        assert ctx.checksum(ids[mm], r) == ref[mm][r], (step, mm, r)
        for mm in range(nm):
            for r in range(tp):
                assert ctx.checksum(ids[mm], r, on_device=False) == ref[mm][r]     # (iv) writeback identity
        st = ctx.stats()
        assert st["k_slots"] == k
        p = str(tmp_path / "trace.ndjson")
        ctx.trace_dump(p)
        cfg, _, decs = S.read_trace(p)
        sm = RegionSwapModel(imgs, cfg.cap, writeback=bool(writeback))
        sm.apply(decs)
        pred = sm.expected_resident_hashes()
        assert pred, "no model resident at the end"
        for mm, hs in pred.items():
            assert ctx.residency(ids[mm]) == M.RESIDENT
            assert [ctx.checksum(ids[mm], r) for r in range(tp)] == hs
        for mm in range(nm):
            assert [checksum.checksum(a) for a in sm.host[mm]] == [ctx.checksum(ids[mm], r, on_device=False)
                                                                 for r in range(tp)]


def test_budget_errors():
    M = need_gpu()
    d = opt_dims("small")
    with M.Ctx(device_ids=(0,), budget=1 << 20) as ctx:
        with pytest.raises(M.MpswError) as e:
            ctx.register_model(d)
        assert e.value.status == M.ENOMEM
    with M.Ctx(device_ids=(0,), budget=layout.shard_bytes(d, 1) + (2 << 20)) as ctx:
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.wait(ctx.swap_in(a))
        assert ctx.swap_in(a) == M.NOOP_TICKET
        with pytest.raises(M.MpswError) as e:
            ctx.swap_in(b)
        assert e.value.status == M.ENOMEM
        with pytest.raises(M.MpswError) as e:
            ctx.request(7, np.array([1], np.int32))
        assert e.value.status == M.ENOENT
        with pytest.raises(M.MpswError) as e:
            ctx.request(a, np.array([d.vocab], np.int32))
        assert e.value.status == M.EINVAL
        with pytest.raises(M.MpswError) as e:
            ctx.request(a, np.zeros(0, np.int32))
        assert e.value.status == M.EINVAL
        assert ctx.stats()["rejected"] == 1


@pytest.mark.slow
def test_full_size_opt13b_tp1_sampled_and_checksum():
    """BASELINE cfg3 at t=1: a 25.7 GB shard, swap-in through the bench's launch config; sampled
    elements vs the oracle one by one; device checksum == oracle checksum of the host arena."""
    M = need_gpu()
    d = opt_dims("opt-13b")
    S_ = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=S_ + (2 << 20), swap_mode=M.SWAP_COPY_ENGINE) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 9)
        ctx.wait(ctx.swap_in(m))
        rng = np.random.default_rng(0)
        for off in rng.integers(0, S_ // 2, 64) * 2:
            got = ctx.peek(m, 0, int(off), 2).view(np.uint16)[0]
            exp = layout.element_at(d, 1, 0, 9, int(off))
            assert (exp is None and got == 0) or int(exp) == int(got)
        host = ctx.model_arena(m, 0)
        assert ctx.checksum(m, 0) == checksum.checksum_parallel(host)
        # the full-size image's hash from the oracle alone (tests/golden, tools/gen_golden_hashes.py)
        gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c0_shard_hashes.json")))
        assert ctx.checksum(m, 0) == int(gold["opt-13b/tp1/r0/seed9/bf16"], 16)
