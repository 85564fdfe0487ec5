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
