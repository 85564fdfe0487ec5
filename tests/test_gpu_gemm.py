"""GEMM kernels in isolation (include/mpsw_testing.h): the tcgen05/TMA kernel and the SIMT
kernel vs a float64 reference of the same bf16/fp32 values, ragged N/K tails, M up to 256,
bias/scale/ReLU epilogues, split-K determinism and bitwise batch invariance."""
import numpy as np
import pytest

from oracle.weights import bf16_bits_from_fp32, bf16_bits_to_fp32
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

SHAPES = [(1, 300, 64), (2, 1280, 5120), (8, 640, 896), (16, 129, 72), (33, 256, 128), (64, 2048, 2048),
          (256, 512, 1024), (2, 3840, 5120), (5, 20480, 512),
          # few tiles x long K: every tile split over ~70 CTAs (stream-K fix-up, both reducers)
          (2, 512, 16384), (64, 512, 16384), (256, 520, 16384)]


def rand_bf16(shape, rng, scale=0.05):
    return bf16_bits_from_fp32((rng.standard_normal(shape) * scale).astype(np.float32))


@pytest.mark.parametrize("impl", [2, 1])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_vs_fp64(impl, M, N, K):
    M_ = need_gpu()
    rng = np.random.default_rng(M * 7 + N + K)
    W, X, b = rand_bf16((N, K), rng), rand_bf16((M, K), rng, 1.0), rand_bf16((N,), rng)
    Wf, Xf, bf = (bf16_bits_to_fp32(a).astype(np.float64) for a in (W, X, b))
    ref = (Xf @ Wf.T + bf) * 0.125
    out = M_.test_gemm(W, X, b, impl=impl, epi=0, scale=0.125)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < 2e-6, err
    relu = M_.test_gemm(W, X, b, impl=impl, epi=1)
    ref2 = bf16_bits_to_fp32(bf16_bits_from_fp32(np.maximum(Xf @ Wf.T + bf, 0).astype(np.float32)))
    # bf16 output: equal up to one bf16 ulp where fp32 summation order flips the rounding (and
    # pre-activations within fp32 rounding of 0 may land on either side of the ReLU)
    assert np.all(np.abs(relu - ref2) <= np.abs(ref2) * 2 ** -7 + 1e-5 * np.abs(ref2).max())


def test_fp32_simt_vs_fp64():
    M_ = need_gpu()
    rng = np.random.default_rng(3)
    W = (rng.standard_normal((700, 1024)) * 0.05).astype(np.float32)
    X = rng.standard_normal((3, 1024)).astype(np.float32)
    out = M_.test_gemm(W, X, None, impl=1, dtype=M_.FP32)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    assert np.abs(out - ref).max() / np.abs(ref).max() < 1e-6


@pytest.mark.parametrize("impl", [2, 1])
def test_batch_invariance_and_determinism(impl):
    M_ = need_gpu()
    rng = np.random.default_rng(11)
    W = rand_bf16((2560, 4096), rng)
    X = rand_bf16((256, 4096), rng, 1.0)
    full = M_.test_gemm(W, X, impl=impl)
    again = M_.test_gemm(W, X, impl=impl)
    assert np.array_equal(full, again)
    # small M reduces split tiles in-kernel, large M in tc_fixup_kernel: same bits either way
    for m in (1, 2, 7, 17, 48, 64, 100, 200):
        part = M_.test_gemm(W, X[:m], impl=impl)
        assert np.array_equal(part, full[:m])
