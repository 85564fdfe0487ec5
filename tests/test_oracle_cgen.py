"""Pin of oracle/c/c0gen.c (the C transcription of C0) against oracle/weights.py (numpy)."""
import numpy as np
import pytest

from oracle import cgen, weights


@pytest.mark.parametrize("gamma", [False, True])
@pytest.mark.parametrize("bf16", [False, True])
def test_c_matches_numpy(gamma, bf16):
    for seed, tid, start, n in [(7, 3, 0, 5000), (123456789, 600, 10**9, 4096), (2**63 + 5, 1, 77, 1000)]:
        c = cgen.values(seed, tid, start, n, gamma, bf16)
        ref = weights.fp32_values(seed, tid, np.arange(start, start + n, dtype=np.int64), gamma)
        if bf16:
            ref = weights.round_bf16(ref)
        assert np.array_equal(c, ref)


def test_lazy_full_equals_full_tensors():
    from synth import opt_dims
    from oracle import layout
    d = opt_dims("small")
    full = layout.full_tensors(d, 42)
    lazy = layout.LazyFull(d, 42)
    for k in full:
        assert np.array_equal(full[k], lazy[k])


def test_forward_with_lazy_weights():
    from synth import opt_dims, request_tokens
    from oracle import layout, forward
    d = opt_dims("tiny")
    tok = request_tokens(0, 0, 0, 8, d.vocab)[None]
    a = forward.forward_bf16_emulated(d, layout.full_tensors(d, 3), tok)
    b = forward.forward_bf16_emulated(d, layout.LazyFull(d, 3), tok)
    assert np.array_equal(a, b)
