"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mpsw.h declares,
and its pure host function mpsw_shard_layout agrees with the oracle's layout (C2)."""
import os
import re

import pytest

from synth import opt_dims
from oracle import layout as OL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def M():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2306_13835_b200 import mpsw
    return mpsw


def test_exports_every_declared_symbol(M):
    hdr = open(os.path.join(ROOT, "include", "mpsw.h")).read() + open(os.path.join(ROOT, "include", "mpsw_testing.h")).read()
    names = set(re.findall(r"^(?:mpsw_status|const char\*)\s+(mpsw_[a-z_]+)\s*\(", hdr, re.M))
    assert len(names) >= 19 and "mpsw_test_gemm" in names
    L = M.lib()
    for n in names:
        assert hasattr(L, n), n


@pytest.mark.parametrize("name,tp,pp", [("tiny", 1, 1), ("tiny", 2, 1), ("tiny", 4, 1), ("opt-125m", 2, 1),
                                        ("opt-13b", 4, 1), ("opt-30b", 8, 1), ("opt-1.3b", 2, 1), ("tiny", 2, 2),
                                        ("opt-13b", 2, 4), ("opt-125m", 1, 3)])
@pytest.mark.parametrize("dtype", [0, 1])
def test_layout_matches_oracle(M, name, tp, pp, dtype):
    d = opt_dims(name)
    for stage in range(pp):
        ours, sb = M.shard_layout(d, tp, tp - 1, dtype, pp, stage)
        placed, total = OL.arena_layout(d, tp, tp - 1, "bf16" if dtype == 0 else "fp32", pp, stage)
        assert sb == total
        assert len(ours) == len(placed)
        for (nm, off, nb, rows, cols, split, tid), p in zip(ours, placed):
            assert nm == p.spec.name and off == p.offset and nb == p.nbytes and split == p.spec.split
            assert tid == p.spec.tid
            assert (rows, cols) == (p.shape if len(p.shape) == 2 else (p.shape[0], 1))


def test_layout_errors(M):
    with pytest.raises(M.MpswError) as e:
        M.shard_layout(opt_dims("opt-125m"), 8)
    assert e.value.status == M.EINVAL
    with pytest.raises(M.MpswError):
        M.shard_layout(opt_dims("tiny"), 2, rank=2)
    with pytest.raises(M.MpswError):
        M.shard_layout(opt_dims("opt-13b"), 1, pp=3)      # 40 layers
    with pytest.raises(M.MpswError):
        M.shard_layout(opt_dims("tiny"), 1, pp=2, stage=2)


def test_init_without_gpu_fails_cleanly(M):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(M.MpswError) as e:
        M.Ctx()
    assert e.value.status in (M.ECUDA, M.EINVAL)


def _gemm_shapes(name, tp):
    d = opt_dims(name)
    hl = d.heads // tp * d.head_dim
    qkv = 3 * ((hl + 127) // 128 * 128)
    return [(qkv, d.hidden), (d.hidden, hl), (d.ffn // tp, d.hidden), (d.hidden, d.ffn // tp),
            ((d.vocab + tp - 1) // tp, d.hidden)]


@pytest.mark.parametrize("name,tp", [("opt-125m", 1), ("opt-1.3b", 1), ("opt-1.3b", 2), ("opt-13b", 1), ("opt-13b", 2),
                                     ("opt-13b", 8), ("opt-30b", 8), ("small", 4)])
def test_tc_plan_split_is_m_independent_and_fits(M, name, tp):
    """The tcgen05 GEMM's launch plan (host arithmetic) for every forward GEMM of the
    model at every batch size: the stream-K split (workers, unit tiles, k-blocks) never depends on
    M (bitwise batch invariance); every CTA of the persistent grid is resident at once (smem,
    TMEM columns, CTAs per SM on 148 SMs); CTA pairs only from 192 padded tokens; the 32-bit
    split arithmetic cannot overflow."""
    for N, K in _gemm_shapes(name, tp):
        split = None
        for m in (1, 2, 15, 16, 17, 48, 64, 100, 128, 176, 192, 200, 256):
            p = M.tc_plan(N, K, m)
            key = (p["workers"], p["tiles_per_unit"], p["unit_tiles"], p["kblocks"])
            split = split or key
            assert key == split, (N, K, m, key, split)
            units = p["unit_tiles"] * p["kblocks"]
            assert 1 <= p["workers"] <= units and units * p["workers"] < 2 ** 32
            assert p["workers"] * p["tiles_per_unit"] <= 2 * 148
            assert p["ctas"] <= p["ctas_per_sm"] * 148, p            # one resident wave
            assert p["smem_bytes"] * p["ctas_per_sm"] + 1024 * p["ctas_per_sm"] <= 233472, p
            assert p["tmem_cols"] * p["ctas_per_sm"] <= 512, p
            assert p["stages"] >= 2
            assert p["cta_pairs"] == (1 if p["mp"] >= 192 else 0)
            assert p["fixup_grid"] == (1 if p["mp"] >= 64 else 0)
            assert p["mp"] % 16 == 0 and p["mp"] >= m


def test_tc_plan_rejects_bad_shapes(M):
    for args in [(0, 64, 2), (128, 7, 2), (128, 64, 0), (128, 64, 257)]:
        with pytest.raises(M.MpswError):
            M.tc_plan(*args)
