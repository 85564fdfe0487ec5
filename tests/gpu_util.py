import os

import pytest


def fuzz_seeds(default_n, offset=0):
    """Seeds of a seeded fuzz test: range(default_n), or MPSW_FUZZ_SEEDS="a:b" for an extended
    campaign (the same case generators, more seeds; each test adds its own offset so the
    campaigns of different tests never share a seed)."""
    e = os.environ.get("MPSW_FUZZ_SEEDS")
    if not e:
        return range(default_n)
    a, b = (int(x) for x in e.split(":"))
    return range(a + offset, b + offset)


def need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2306_13835_b200 import mpsw
    return mpsw
