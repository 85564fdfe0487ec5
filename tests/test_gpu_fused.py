"""GPU parity of the fused persistent layers kernel (csrc/fwd_fused.cu): every decoder layer of a
TP = 1 bf16 forward at M <= 48 in one launch (opt-in, gemm_impl = 3). It must give the same bits
as the per-op kernels (gemm_impl = 2), so logits stay batch-invariant across the M = 48 routing boundary, and match
the oracle's bf16-emulating forward (north-star bar 1e-2)."""
import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, forward
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def serve(M, d, seed, token_lists, gemm_impl, max_batch=8, one_by_one=False):
    S_ = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=S_ + (2 << 20), max_batch=max_batch,
               max_tokens=max(len(t) for t in token_lists), gemm_impl=gemm_impl) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, seed)
        ctx.wait(ctx.swap_in(m))
        outs = []
        if one_by_one:
            for t in token_lists:
                rid, out = ctx.request(m, t)
                ctx.wait_request(rid, 120)
                outs.append(out)
        else:
            rids = [ctx.request(m, t) for t in token_lists]
            for rid, _ in rids:
                ctx.wait_request(rid, 120)
            outs = [out for _, out in rids]
        return outs, ctx.stats()


@pytest.mark.parametrize("name", ["tiny", "small", "mid", "opt-125m"])
def test_fused_bitwise_equals_per_op(name):
    """Ragged batches of up to 48 tokens (several tiles, ragged tails, stream-K splits; OPT-125M's
    QKV has fewer units than CTAs): fused == per-op bit for bit, and fewer kernel launches."""
    M = need_gpu()
    d = opt_dims(name)
    L = min(8, d.max_pos)
    lens = [L, 3, 1, L, 5, 2, L, 7]
    toks = [request_tokens(41, 0, i, n, d.vocab) for i, n in enumerate(lens)]
    fused, st_f = serve(M, d, 51, toks, 3, max_batch=8)
    per_op, st_p = serve(M, d, 51, toks, 2, max_batch=8)
    for a, b in zip(fused, per_op):
        assert np.array_equal(a, b)
    assert st_f["kernel_launches"] < st_p["kernel_launches"]


def test_fused_vs_oracle_opt125m():
    M = need_gpu()
    d = opt_dims("opt-125m")
    toks = [request_tokens(42, 0, i, n, d.vocab) for i, n in enumerate([2, 8, 8, 1])]
    outs, _ = serve(M, d, 52, toks, 3, max_batch=4)
    W = layout.full_tensors(d, 52)
    for t, y in zip(toks, outs):
        ref = forward.forward_bf16_emulated(d, W, t[None])[0]
        PU.assert_logits(y, ref, tag="fused")
        assert int(np.argmax(y)) == int(np.argmax(ref))


def test_batch_invariance_across_fused_boundary():
    """A request alone (M = 8: fused kernel) and inside a 64-token batch (per-op kernels): same bits."""
    M = need_gpu()
    d = opt_dims("small")
    toks = [request_tokens(43, 0, i, 8, d.vocab) for i in range(8)]
    alone, _ = serve(M, d, 53, toks[3:4], 3, max_batch=1)
    batched, st = serve(M, d, 53, toks, 3, max_batch=8)
    assert st["batches"] < len(toks)            # at least one batch above the fused limit
    assert np.array_equal(alone[0], batched[3])


def test_fused_many_launches():
    """The phase counters are monotonic across launches (per-forward epoch): 40 back-to-back
    forwards on one ctx stay equal to the per-op path."""
    M = need_gpu()
    d = opt_dims("small")
    toks = [request_tokens(44, 0, i, 1 + i % 8, d.vocab) for i in range(40)]
    fused, _ = serve(M, d, 54, toks, 3, max_batch=1, one_by_one=True)
    per_op, _ = serve(M, d, 54, toks, 2, max_batch=1, one_by_one=True)
    for a, b in zip(fused, per_op):
        assert np.array_equal(a, b)


@pytest.mark.slow
def test_full_size_opt13b_fused_bitwise():
    """cfg3's launch configuration (OPT-13B, TP1, B = 1, L = 2): fused == per-op bit for bit."""
    M = need_gpu()
    d = opt_dims("opt-13b")
    toks = [request_tokens(45, 0, i, 2, d.vocab) for i in range(2)]
    fused, _ = serve(M, d, 1000, toks, 3, max_batch=1, one_by_one=True)
    per_op, _ = serve(M, d, 1000, toks, 2, max_batch=1, one_by_one=True)
    for a, b in zip(fused, per_op):
        assert np.array_equal(a, b)


def test_fused_models_of_different_depths():
    """Two models of different depth and width in one region (reading #28), requests alternating:
    the phase counters are reset at kernel exit, so a deeper model after a shallower one still
    synchronises (no stale counts); logits equal the per-op path bit for bit."""
    M = need_gpu()
    big, small = opt_dims("mid"), opt_dims("small")          # 4 and 3 layers
    budget = layout.shard_bytes(big, 1) + layout.shard_bytes(small, 1) + (4 << 20)
    toks = [request_tokens(46, 0, i, 1 + i % 8, small.vocab) for i in range(12)]
    res = {}
    for impl in (3, 2):
        with M.Ctx(device_ids=(0,), budget=budget, max_batch=1, max_tokens=8, gemm_impl=impl) as ctx:
            a = ctx.register_model(big)
            b = ctx.register_model(small)
            ctx.synth_fill(a, 61)
            ctx.synth_fill(b, 62)
            outs = []
            for i, t in enumerate(toks):
                rid, out = ctx.request(a if i % 2 == 0 else b, t)
                ctx.wait_request(rid, 120)
                outs.append(out)
            res[impl] = outs
    for x, y in zip(res[3], res[2]):
        assert np.array_equal(x, y)
