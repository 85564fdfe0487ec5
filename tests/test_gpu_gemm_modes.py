"""The tcgen05 GEMM's execution choices against each other ("Pair split, two
executions"). The split knobs are read once per process, so each configuration runs in its own
subprocess on the same seeded operands:
* the pair split on independent CTAs and on CTA pairs (cta_group::2) must give the same bits at
  every M, because the runs of a tile and their summation order are the same;
* the fix-up done in-kernel by the last-arriving CTA or by the separate grid: same bits;
* the round-1 single split: also vs the float64 reference, and bitwise batch-invariant."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(2, 3840, 5120), (64, 2048, 2048), (100, 2560, 4096), (208, 640, 896), (256, 2560, 4096), (256, 520, 16384),
          (48, 5120, 20480), (2, 2560, 4096)]

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, ROOT)
from paper_2306_13835_b200 import mpsw as M_
from oracle.weights import bf16_bits_from_fp32
out = {}
for (M, N, K) in SHAPES:
    rng = np.random.default_rng(N + K)          # same operands for every M of an (N, K)
    W = bf16_bits_from_fp32((rng.standard_normal((N, K)) * 0.05).astype(np.float32))
    X = bf16_bits_from_fp32(rng.standard_normal((256, K)).astype(np.float32))[:M]
    y = M_.test_gemm(W, X, impl=2)
    np.save(f"{OUT}_{M}_{N}_{K}.npy", y)
"""


def run_mode(tmp_path, tag, env):
    out = str(tmp_path / tag)
    code = CHILD.replace("ROOT", repr(ROOT)).replace("SHAPES", repr(SHAPES)).replace("{OUT}", out)
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return {s: np.load(f"{out}_{s[0]}_{s[1]}_{s[2]}.npy") for s in SHAPES}


def test_pair_split_executions_bitwise_equal(tmp_path):
    need_gpu()
    indep = run_mode(tmp_path, "indep", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "100000"})
    pairs = run_mode(tmp_path, "pairs", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "16"})
    pairs_vw2 = run_mode(tmp_path, "pairs_vw2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "16", "MPSW_TC_VW": "2"})
    for s in SHAPES:
        assert np.array_equal(indep[s], pairs[s]), s
        assert np.array_equal(indep[s], pairs_vw2[s]), s


def test_fixup_reducers_bitwise_equal(tmp_path):
    need_gpu()
    in_kernel = run_mode(tmp_path, "ink", {"MPSW_TC_EXT_MIN": "100000"})
    ext = run_mode(tmp_path, "ext", {"MPSW_TC_EXT_MIN": "16"})
    hints_off = run_mode(tmp_path, "nohint", {"MPSW_TC_L2HINT": "0"})
    for s in SHAPES:
        assert np.array_equal(in_kernel[s], ext[s]), s
        assert np.array_equal(in_kernel[s], hints_off[s]), s


def test_single_split_vs_fp64_and_invariant(tmp_path):
    need_gpu()
    from oracle.weights import bf16_bits_from_fp32, bf16_bits_to_fp32
    single = run_mode(tmp_path, "single", {"MPSW_TC_SPLIT": "1"})
    for (M, N, K), y in single.items():
        rng = np.random.default_rng(N + K)
        W = bf16_bits_from_fp32((rng.standard_normal((N, K)) * 0.05).astype(np.float32))
        X = bf16_bits_from_fp32(rng.standard_normal((256, K)).astype(np.float32))[:M]
        ref = bf16_bits_to_fp32(X).astype(np.float64) @ bf16_bits_to_fp32(W).astype(np.float64).T
        # fp32 accumulation over K = 20480 terms: ~3e-6 of max|ref| (test_gpu_gemm's 2e-6 is for
        # K <= 16384)
        assert np.abs(y - ref).max() / np.abs(ref).max() < 5e-6, (M, N, K)
    # batch invariance of the single split: M = 2 / 100 rows equal the first rows at M = 256
    full = single[(256, 2560, 4096)]
    assert np.array_equal(single[(100, 2560, 4096)], full[:100])
    assert np.array_equal(single[(2, 2560, 4096)], full[:2])


def test_pair_split_batch_invariant_across_executions(tmp_path):
    need_gpu()
    y = run_mode(tmp_path, "dflt", {})             # default: CTA pairs from 192 padded tokens
    full = y[(256, 2560, 4096)]                    # CTA pairs
    assert np.array_equal(y[(100, 2560, 4096)], full[:100])   # independent CTAs, in-kernel / grid fix-up
    assert np.array_equal(y[(2, 2560, 4096)], full[:2])
