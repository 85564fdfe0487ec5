"""Pins for oracle/weights.py (C0) and its bf16 rounding — against published SplitMix64
vectors, closed forms, brute force, and an independent library rounding (torch)."""
import os
import numpy as np
import pytest

from oracle import weights

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_vectors():
    vals = [int(l, 16) for l in open(os.path.join(GOLD, "splitmix64_seed0.txt")) if l.startswith("0x")]
    # stateful generator: the i-th output is the mix of state (i+1)*gamma, i.e. splitmix64(i*gamma)
    g = 0x9E3779B97F4A7C15
    for i, v in enumerate(vals):
        assert weights.splitmix64_scalar((i * g) & weights.MASK64) == v
        assert int(weights.splitmix64(np.array([(i * g) & weights.MASK64], np.uint64))[0]) == v


def test_vectorised_equals_scalar_bruteforce():
    rng = np.random.default_rng(1)
    z = rng.integers(0, 2**63, size=2000, dtype=np.int64).astype(np.uint64) * np.uint64(3)
    v = weights.splitmix64(z)
    for a, b in zip(z[:300], v[:300]):
        assert weights.splitmix64_scalar(int(a)) == int(b)


def test_w_closed_form_and_range():
    seed, tid = 12345, 7
    idx = np.arange(0, 5000, dtype=np.int64)
    w = weights.raw_w(seed, tid, idx)
    # brute force recompute of each index from the spec text
    for i in [0, 1, 17, 4999]:
        x = weights.splitmix64_scalar(seed ^ (tid << 40) ^ i)
        assert w[i] == ((x >> 40) - 2**23) * 2.0**-28
    assert w.min() >= -2.0**-5 and w.max() < 2.0**-5
    # exact in fp32 (24-bit integer times a power of two)
    assert np.all(w.astype(np.float32).astype(np.float64) == w)


def test_w_statistics():
    w = weights.raw_w(3, 1, np.arange(10**6))
    assert abs(w.std() / (2.0**-5 / np.sqrt(3)) - 1) < 0.01
    assert abs(w.mean()) < 1e-4


def test_bf16_rne_special_cases():
    # 1 + 2^-8 is exactly halfway between 1 and 1 + 2^-7 -> ties to even (1.0)
    x = np.array([1.0, 1 + 2.0**-8, 1 + 3 * 2.0**-8, -1 - 2.0**-8, 2.0**-30, 1 + 2.0**-7], np.float32)
    r = weights.round_bf16(x)
    assert list(r) == [1.0, 1.0, 1 + 2.0**-6, -1.0, 2.0**-30, 1 + 2.0**-7]


def test_bf16_rne_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(200000) * rng.choice([1e-3, 1, 1e3], 200000)).astype(np.float32)
    ours = weights.round_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(ours, ref)


def test_ln_gamma_is_one_plus_w():
    idx = np.arange(64)
    g = weights.fp32_values(9, 3, idx, True)
    w = weights.raw_w(9, 3, idx)
    assert np.array_equal(g, (1.0 + w).astype(np.float32))
