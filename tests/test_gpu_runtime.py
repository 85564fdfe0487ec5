"""Runtime robustness (GPU): a rank failing inside a TP batch poisons the ctx without hanging its
peers (SpinBarrier poison check) and shutdown returns; offload semantics switch at run time
(mpsw_set_writeback) with the D2H bytes to match; the completed-ticket history is bounded;
a failed init frees its parameter budget (a retry of the same size succeeds)."""
import threading
import time

import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, checksum
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tp", [2, 4])
def test_rank_fault_mid_batch_poisons_and_shutdown_returns(tp):
    M = need_gpu()
    d = opt_dims("small")
    ctx = M.Ctx(device_ids=(0,) * tp, budget=layout.shard_bytes(d, tp) + (2 << 20), max_batch=1, max_tokens=8)
    m = ctx.register_model(d)
    ctx.synth_fill(m, 3)
    ctx.wait(ctx.swap_in(m))
    rid, _ = ctx.request(m, request_tokens(0, 0, 0, 8, d.vocab))
    ctx.wait_request(rid, 60)                       # healthy first
    ctx.inject_fault(tp - 1)
    rid, _ = ctx.request(m, request_tokens(0, 0, 1, 8, d.vocab))
    with pytest.raises(M.MpswError) as e:
        ctx.wait_request(rid, 60)
    assert e.value.status == M.ECUDA and "injected" in str(e.value)
    done = threading.Event()
    th = threading.Thread(target=lambda: (ctx.close(), done.set()), daemon=True)
    th.start()
    assert done.wait(60), "mpsw_shutdown hung after a rank failure"
    with pytest.raises(M.MpswError):                # a new ctx is unaffected
        with M.Ctx(device_ids=(0,), budget=1 << 20) as c2:
            c2.register_model(d)                    # ENOMEM: budget below one shard


def test_set_writeback_switches_offload_semantics():
    M = need_gpu()
    d = opt_dims("tiny")
    S_ = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=(S_ + 4095) // 4096 * 4096, writeback=0, chunk_bytes=4096, max_batch=1,
               max_tokens=4) as ctx:
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.synth_fill(a, 1)
        ctx.synth_fill(b, 2)
        tok = np.array([1, 2], np.int32)
        for m in (a, b, a):                          # clean eviction: no D2H
            ctx.wait_request(ctx.request(m, tok)[0], 60)
        assert ctx.stats()["d2h_bytes"] == 0
        ctx.set_writeback(1)
        for m in (b, a):                             # writeback: one shard D2H per swap
            ctx.wait_request(ctx.request(m, tok)[0], 60)
        assert ctx.stats()["d2h_bytes"] == 2 * S_
        for m, seed in ((a, 1), (b, 2)):             # (iv) round trip identity
            assert ctx.checksum(m, 0, on_device=False) == checksum.checksum(layout.shard_image(d, 1, 0, seed))


def test_ticket_history_is_bounded():
    M = need_gpu()
    d = opt_dims("tiny")
    S_ = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=(S_ + 4095) // 4096 * 4096, writeback=0) as ctx:
        m = ctx.register_model(d)
        first = ctx.swap_in(m)
        ctx.wait(first)
        ctx.wait(ctx.swap_out(m))
        last = None
        for _ in range(2100):                        # 4200 more completed swap entries
            last = ctx.swap_in(m)
            ctx.wait(last)
            ctx.wait(ctx.swap_out(m))
        with pytest.raises(M.MpswError) as e:
            ctx.wait(first, 1)
        assert e.value.status == M.ENOENT
        ctx.wait(last, 1)                            # recent tickets stay queryable
        assert ctx.entry_gpu_ms(last)[0] == 0


def test_failed_init_frees_the_budget():
    """An init that fails after allocating must not leak the parameter budget: two ranks on one
    GPU with a budget of ~60 % of free HBM each -> the second cudaMalloc fails (ENOMEM) after the
    first succeeded; three such failures in a row, then one rank with the same budget succeeds
    (it would not if the first rank's region had leaked)."""
    M = need_gpu()
    import torch
    free, _ = torch.cuda.mem_get_info(0)
    big = int(free * 0.6) // 4096 * 4096
    for _ in range(3):
        with pytest.raises(M.MpswError) as e:
            M.Ctx(device_ids=(0, 0), budget=big)
        assert e.value.status == M.ENOMEM
    with M.Ctx(device_ids=(0,), budget=big) as ctx:
        d = opt_dims("tiny")
        ctx.wait(ctx.swap_in(ctx.register_model(d)))


@pytest.mark.parametrize("tp,writeback", [(1, 1), (2, 0)])
def test_debug_checks_silent_on_correct_runs(tp, writeback):
    """Residency stamps on (debug_checks): 30 alternating blocking requests over 3 models with room
    for one — every request swaps, every forward checks the stamp of the load it was gated on —
    and no check trips; logits still match the oracle."""
    M = need_gpu()
    from oracle import forward
    from tests import parity_util as PU
    d = opt_dims("small")
    S_ = layout.shard_bytes(d, tp)
    with M.Ctx(device_ids=(0,) * tp, budget=(S_ + 4095) // 4096 * 4096, max_batch=2, max_tokens=8,
               writeback=writeback, debug_checks=1) as ctx:
        ids = [ctx.register_model(d) for _ in range(3)]
        for i, m in enumerate(ids):
            ctx.synth_fill(m, 40 + i)
        outs = []
        for i in range(30):
            m = ids[i % 3]
            tok = request_tokens(8, m, i, 8, d.vocab)
            rid, y = ctx.request(m, tok)
            ctx.wait_request(rid, 120)
            outs.append((m, tok, y.copy()))
        assert ctx.stats()["swaps_in"] == 30
    W = layout.full_tensors(d, 40 + outs[-1][0])
    PU.assert_logits(outs[-1][2], forward.forward_bf16_emulated(d, W, outs[-1][1][None])[0], tag="debug checks")


def test_debug_checks_detect_a_forward_on_a_non_resident_range():
    """The detector fires: corrupt a resident model's stamp (as a load that never finished, or an
    eviction racing the forward, would leave it); its next request poisons the ctx with
    EINVARIANT naming the residency stamp, and shutdown still returns."""
    M = need_gpu()
    d = opt_dims("small")
    ctx = M.Ctx(device_ids=(0, 0), budget=layout.shard_bytes(d, 2) + (2 << 20), max_batch=1, max_tokens=8,
                debug_checks=1)
    m = ctx.register_model(d)
    ctx.synth_fill(m, 3)
    rid, _ = ctx.request(m, request_tokens(0, 0, 0, 8, d.vocab))
    ctx.wait_request(rid, 60)
    ctx.corrupt_stamp(m)
    rid, _ = ctx.request(m, request_tokens(0, 0, 1, 8, d.vocab))
    with pytest.raises(M.MpswError) as e:
        ctx.wait_request(rid, 60)
    assert "residency stamp" in str(e.value)
    done = threading.Event()
    threading.Thread(target=lambda: (ctx.close(), done.set()), daemon=True).start()
    assert done.wait(60)
