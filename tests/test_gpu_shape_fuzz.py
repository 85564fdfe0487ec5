"""Seeded shape fuzz of the TP forward (a6/a7) against the oracle: random OPT-like dims inside the
library's documented limits (head_dim a multiple of 8 up to 128, hidden/tp and ffn/tp multiples of
8, vocab/tp of any parity), TP 1/2/4/8 virtual ranks, ragged batches whose token count spans both
split-K fix-up regimes of the tcgen05 GEMM (Mp < 64 in-kernel, >= 64 external). Per-rank q/k/v
widths that are not whole 128-row tiles found a real workspace-sizing bug (tests/test_gpu_forward.py
`test_bf16_parity_ragged_head_tiles`); this sweeps the neighbourhood."""
import numpy as np
import pytest

from synth import request_tokens
from synth.models import OptDims
from oracle import layout, forward
from tests.gpu_util import need_gpu, fuzz_seeds as seeds
from tests import parity_util as PU

pytestmark = pytest.mark.gpu


def random_case(seed):
    rng = np.random.default_rng(seed)
    tp = int(rng.choice([1, 2, 4, 8]))
    hd = int(rng.choice([8, 16, 24, 32, 40, 64, 72, 96, 128]))
    heads = tp * int(rng.integers(1, max(2, 512 // (hd * tp)) + 1))
    ffn = 8 * tp * int(rng.integers(1, 256 // tp + 1))
    vocab = tp * int(rng.integers(max(1, 40 // tp), 2000 // tp))
    d = OptDims(int(rng.integers(1, 4)), heads * hd, heads, ffn, vocab=vocab, max_pos=32)
    B = int(rng.integers(1, 7))
    lens = [int(x) for x in rng.integers(1, 17, size=B)]
    return d, tp, lens


def large_batch_case(seed):
    """One batch of 12..40 requests x 1..16 tokens (M up to 640 rows): spans the in-kernel and
    grid fix-ups, the CTA-pair execution from 192 padded tokens and the 256-row tcgen05 chunks."""
    d, tp, _ = random_case(seed)
    rng = np.random.default_rng(10_000 + seed)
    B = int(rng.integers(12, 41))
    lens = [int(x) for x in rng.integers(1, 17, size=B)]
    return d, tp, lens


def check_logits(y, ref, tol):
    """rel-L2 and element-wise bars, argmax where the oracle's margin is clear (parity_util)."""
    if tol >= PU.BF16_LOGITS_TOL:
        PU.assert_logits(y, ref, tol=tol, tag="shape-fuzz")
    else:
        PU.assert_logits(y, None, ref, tol=tol, tag="shape-fuzz-fp32")


@pytest.mark.parametrize("seed", seeds(16))
def test_random_shapes_bf16_vs_oracle(seed):
    M = need_gpu()
    d, tp, lens = random_case(seed)
    S_ = layout.shard_bytes(d, tp)
    toks = [request_tokens(300 + seed, 0, i, n, d.vocab) for i, n in enumerate(lens)]
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), max_batch=len(lens), max_tokens=16) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 400 + seed)
        ctx.wait(ctx.swap_in(m))
        rids = [ctx.request(m, t) for t in toks]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
    W = layout.full_tensors(d, 400 + seed, "bf16")
    for t, (_, y) in zip(toks, rids):
        check_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], 1e-2)


@pytest.mark.parametrize("seed", seeds(4, 100_000))
def test_random_shapes_fp32_vs_exact(seed):
    M = need_gpu()
    d, tp, lens = random_case(1000 + seed)
    S_ = layout.shard_bytes(d, tp, "fp32")
    toks = [request_tokens(500 + seed, 0, i, n, d.vocab) for i, n in enumerate(lens)]
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), dtype=M.FP32, max_batch=len(lens), max_tokens=16) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 600 + seed)
        ctx.wait(ctx.swap_in(m))
        rids = [ctx.request(m, t) for t in toks]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
    W = layout.full_tensors(d, 600 + seed, "fp32")
    for t, (_, y) in zip(toks, rids):
        check_logits(y, forward.forward_exact(d, W, t[None])[0], 1e-5)


@pytest.mark.parametrize("seed", seeds(6, 200_000))
def test_random_shapes_large_batch_bf16_vs_oracle(seed):
    """Random shapes with one large ragged batch (M up to 640 rows): every request's logits vs the
    emulating oracle, and one request rerun alone is bitwise equal (batch invariance across the
    fix-up regimes, the CTA-pair switch and the 256-row chunks)."""
    M = need_gpu()
    d, tp, lens = large_batch_case(seed)
    S_ = layout.shard_bytes(d, tp)
    toks = [request_tokens(700 + seed, 0, i, n, d.vocab) for i, n in enumerate(lens)]
    # Every request must queue behind m's LOADING so they all leave as ONE batch: 4 KiB copy-engine
    # chunks, and m's load sits behind the loads of `nb` same-shaped blocker models on each rank's
    # H2D stream (>= ~2000 chunks per rank ahead of it, tens of ms).
    nb = int(min(64, max(2, -(-2000 * 4096 // S_))))
    with M.Ctx(device_ids=(0,) * tp, budget=(nb + 1) * (S_ + 4096) + (2 << 20), max_batch=len(lens), max_tokens=16,
               chunk_bytes=4096, swap_mode=M.SWAP_COPY_ENGINE) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, 800 + seed)
        blockers = [ctx.register_model(d) for _ in range(nb)]
        tickets = [ctx.swap_in(b) for b in blockers]
        rids = [ctx.request(m, t) for t in toks]
        for rid, _ in rids:
            ctx.wait_request(rid, 120)
        for tk in tickets:
            ctx.wait(tk, 120)
        st = ctx.stats()
        j = len(toks) - 1
        rid, alone = ctx.request(m, toks[j])
        ctx.wait_request(rid, 120)
    assert st["batches"] == 1, st
    assert np.array_equal(alone, rids[j][1])
    W = layout.full_tensors(d, 800 + seed, "bf16")
    for t, (_, y) in zip(toks, rids):
        check_logits(y, forward.forward_bf16_emulated(d, W, t[None])[0], 1e-2)
