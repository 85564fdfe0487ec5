"""GPU parity of the TP forward (a6/a7): logits vs the oracle (bf16-emulating at 1e-2 — expected
far below — and fp64-exact), fp32 mode at 1e-5, TP = 1/2/4 virtual ranks, ragged batches, and
bitwise batch invariance."""
import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, forward
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def run_requests(M, d, tp, dtype, seed, token_lists, max_batch=8, hold=True):
    S_ = layout.shard_bytes(d, tp, "bf16" if dtype == M.BF16 else "fp32")
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), dtype=dtype, max_batch=max_batch,
               max_tokens=max(len(t) for t in token_lists)) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, seed)
        ctx.wait(ctx.swap_in(m))
        rids = [ctx.request(m, t) for t in token_lists]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
        return [out for _, out in rids], ctx.stats()


@pytest.mark.parametrize("tp", [1, 2, 4])
@pytest.mark.parametrize("name", ["tiny", "small"])
def test_bf16_logits_parity(tp, name):
    M = need_gpu()
    d = opt_dims(name)
    toks = [request_tokens(1, 0, i, L, d.vocab) for i, L in enumerate([8, 8, 3, 1, 8, 5])]
    outs, st = run_requests(M, d, tp, M.BF16, 21, toks)
    W = layout.full_tensors(d, 21, "bf16")
    for t, y in zip(toks, outs):
        em = forward.forward_bf16_emulated(d, W, t[None])[0]
        ex = forward.forward_exact(d, W, t[None])[0]
        # north-star bar 1e-2 against both oracles; per-stage element-wise parity is
        # tests/test_gpu_layers.py (the free-running emulation decorrelates after a layer)
        PU.assert_logits(y, em, ex, tag=f"{name} tp{tp}")
    assert st["batches"] >= 1


# Per-rank q/k/v widths that are not whole 128-row tiles: small at TP 8 (one 32-wide head per
# rank) and OPT-125M at TP 4 (hl = 192). The QKV GEMM tiles each segment on its own, so it has
# more tiles and stream-K CTAs than 3 * hl suggests; the split-K workspace must be sized for that
# (a regression: it was not, and the partials overran it, giving all-zero logits).
@pytest.mark.parametrize("name,tp", [("small", 8), ("opt-125m", 4)])
def test_bf16_parity_ragged_head_tiles(name, tp):
    M = need_gpu()
    d = opt_dims(name)
    toks = [request_tokens(6, 0, i, L, d.vocab) for i, L in enumerate([8, 3, 1, 8])]
    outs, _ = run_requests(M, d, tp, M.BF16, 23, toks, max_batch=4)
    W = layout.full_tensors(d, 23, "bf16")
    for t, y in zip(toks, outs):
        em = forward.forward_bf16_emulated(d, W, t[None])[0]
        PU.assert_logits(y, em, forward.forward_exact(d, W, t[None])[0], tag=f"{name} tp{tp} ragged tiles")


@pytest.mark.parametrize("tp", [1, 2, 4])
def test_fp32_logits_parity(tp):
    M = need_gpu()
    d = opt_dims("small")
    toks = [request_tokens(2, 0, i, 8, d.vocab) for i in range(4)]
    outs, _ = run_requests(M, d, tp, M.FP32, 22, toks)
    W = layout.full_tensors(d, 22, "fp32")
    for t, y in zip(toks, outs):
        ex = forward.forward_exact(d, W, t[None])[0]
        PU.assert_logits(y, None, ex, tol=PU.FP32_LOGITS_TOL, tag=f"fp32 tp{tp}")


def test_batch_invariance_bitwise():
    M = need_gpu()
    d = opt_dims("small")
    base = request_tokens(3, 0, 0, 8, d.vocab)
    others = [request_tokens(3, 0, i, 8, d.vocab) for i in range(1, 8)]
    alone, _ = run_requests(M, d, 2, M.BF16, 5, [base], max_batch=1)
    batched, _ = run_requests(M, d, 2, M.BF16, 5, others[:3] + [base] + others[3:], max_batch=8)
    assert np.array_equal(alone[0], batched[3])


def test_mid_model_tp2_parity():
    M = need_gpu()
    d = opt_dims("mid")
    toks = [request_tokens(4, 0, i, 8, d.vocab) for i in range(3)]
    outs, _ = run_requests(M, d, 2, M.BF16, 23, toks)
    W = layout.full_tensors(d, 23, "bf16")
    for t, y in zip(toks, outs):
        PU.assert_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], forward.forward_exact(d, W, t[None])[0],
                         tag="mid tp2")


@pytest.mark.slow
def test_full_size_opt13b_logits_parity():
    """cfg3 at full size (OPT-13B, TP1, the bench's launch configuration): request logits vs the
    oracle's bf16-emulating forward computed layer by layer from the C0 spec."""
    M = need_gpu()
    d = opt_dims("opt-13b")
    toks = [request_tokens(9, 0, i, 2, d.vocab) for i in range(2)]
    outs, st = run_requests(M, d, 1, M.BF16, 1000, toks, max_batch=1)
    W = layout.LazyFull(d, 1000)
    for t, y in zip(toks, outs):
        PU.assert_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], forward.forward_exact(d, W, t[None])[0],
                         tag="opt-13b tp1 full size")


@pytest.mark.slow
def test_full_size_opt13b_tp2_batch_invariance():
    """Property at full size: OPT-13B TP2 (virtual ranks) is bitwise batch-invariant and agrees
    with TP1 within the bf16 tolerance."""
    M = need_gpu()
    d = opt_dims("opt-13b")
    toks = [request_tokens(8, 0, i, 2, d.vocab) for i in range(3)]
    tp2_batched, _ = run_requests(M, d, 2, M.BF16, 1001, toks, max_batch=4)
    tp2_alone, _ = run_requests(M, d, 2, M.BF16, 1001, toks[1:2], max_batch=1)
    assert np.array_equal(tp2_alone[0], tp2_batched[1])
    tp1, _ = run_requests(M, d, 1, M.BF16, 1001, toks, max_batch=4)
    for a, b in zip(tp1, tp2_batched):
        assert forward.rel_l2(b, a) < 1e-2
    W = layout.LazyFull(d, 1001)
    PU.assert_logits(tp2_batched[0], None, forward.forward_exact(d, W, toks[0][None])[0], tag="opt-13b tp2 full size")


def test_max_tokens_and_max_rows():
    """Edge sizes: L = 128 (attention maximum) and a full 32 x 8 batch (M = 256: the MMA N = 256
    single-buffered-accumulator path), logits vs the oracle."""
    M = need_gpu()
    d = opt_dims("mid")
    long_tok = [request_tokens(11, 0, 0, 128, d.vocab)]
    outs, _ = run_requests(M, d, 1, M.BF16, 31, long_tok, max_batch=1)
    W = layout.full_tensors(d, 31)
    ref = forward.forward_bf16_emulated(d, W, long_tok[0][None])[0]
    PU.assert_logits(outs[0], ref, forward.forward_exact(d, W, long_tok[0][None])[0], tag="mid L128")
    toks = [request_tokens(12, 0, i, 8, d.vocab) for i in range(32)]
    S_ = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=S_ + 4096, max_batch=32, max_tokens=8) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 31)
        ctx.wait(ctx.swap_in(m))
        rids = [ctx.request(m, t) for t in toks]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
        st = ctx.stats()
    assert st["batches"] <= 3                       # most requests share one M = 248..256 batch
    for t, (_, y) in list(zip(toks, rids))[::5]:
        ref = forward.forward_bf16_emulated(d, W, t[None])[0]
        PU.assert_logits(y, ref, tag="mid M256")


@pytest.mark.slow
def test_full_size_opt30b_tp8_logits_parity():
    """cfg4's model at its TP degree (OPT-30B, TP8 as 8 virtual ranks on one B200; 7.5 GB per
    rank): request logits vs the oracle streamed layer by layer."""
    M = need_gpu()
    d = opt_dims("opt-30b")
    toks = [request_tokens(13, 0, 0, 8, d.vocab)]
    outs, _ = run_requests(M, d, 8, M.BF16, 2000, toks, max_batch=1)
    W = layout.LazyFull(d, 2000)
    PU.assert_logits(outs[0], forward.forward_bf16_emulated(d, W, toks[0][None])[0],
                     forward.forward_exact(d, W, toks[0][None])[0], tag="opt-30b tp8 full size")


@pytest.mark.slow
def test_full_size_opt1_3b_tp2_vs_oracle():
    """cfg2 at full size (OPT-1.3B TP2 (virtual ranks): logits vs the oracle."""
    M = need_gpu()
    d = opt_dims("opt-1.3b")
    toks = [request_tokens(14, 0, i, 8, d.vocab) for i in range(4)]
    outs, _ = run_requests(M, d, 2, M.BF16, 2001, toks, max_batch=8)
    W = layout.LazyFull(d, 2001)
    for t, y in zip(toks, outs):
        PU.assert_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], forward.forward_exact(d, W, t[None])[0],
                         tag="opt-1.3b tp2 full size")


def test_rows_beyond_256_run_in_tcgen05_chunks():
    """M > 256 token rows (40 requests x 8 tokens = 320 in one batch) run through the tcgen05
    kernel in 256-row chunks (no SIMT fallback): logits vs both oracles, and a request whose rows
    fall in the second chunk is bitwise equal to the same request run alone (batch invariance
    across chunk boundaries)."""
    M = need_gpu()
    d = opt_dims("mid")
    toks = [request_tokens(15, 0, i, 8, d.vocab) for i in range(40)]
    S_ = layout.shard_bytes(d, 1)
    # 4 KiB copy-engine chunks make the implicit swap-in take tens of ms, so all 40 requests queue
    # behind the LOADING model and leave as ONE batch of 320 rows
    with M.Ctx(device_ids=(0,), budget=S_ + 4096, max_batch=40, max_tokens=8, chunk_bytes=4096,
               swap_mode=M.SWAP_COPY_ENGINE) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 33)
        rids = [ctx.request(m, t) for t in toks]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
        st = ctx.stats()
        outs = [y for _, y in rids]
        rid, alone = ctx.request(m, toks[37])
        ctx.wait_request(rid, 120)
    assert st["batches"] == 1                        # M = 320 > 256: two tcgen05 chunks per GEMM
    assert np.array_equal(alone, outs[37])
    W = layout.full_tensors(d, 33)
    for i in (1, 20, 33, 39):
        PU.assert_logits(outs[i], forward.forward_bf16_emulated(d, W, toks[i][None])[0],
                         forward.forward_exact(d, W, toks[i][None])[0], tag="mid M>256")
