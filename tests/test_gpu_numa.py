"""NUMA-affine shard store (a0): with a NUMA node for the GPU (forced to node 0 through
MPSW_NUMA_NODE on a one-node box), every pinned arena is mbind-bound to it, its pages are verified
resident there (move_pages on sampled pages), and swaps stay bit-exact."""
import json
import os
import subprocess
import sys

import pytest

from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims
from oracle import layout, checksum
d = opt_dims("small")
S = layout.shard_bytes(d, 2)
with M.Ctx(device_ids=(0, 0), budget=S + 4096) as ctx:
    a, b = ctx.register_model(d), ctx.register_model(d)
    ctx.synth_fill(a, 5); ctx.synth_fill(b, 6)
    ctx.wait(ctx.swap_in(a))
    ok = all(ctx.checksum(a, r) == checksum.checksum(layout.shard_image(d, 2, r, 5)) for r in range(2))
    st = ctx.stats()
print(json.dumps({"ok": ok, "req": st["numa_requested"], "ver": st["numa_verified"]}))
'''


def test_numa_bound_arenas():
    need_gpu()
    env = dict(os.environ, MPSW_NUMA_NODE="0")
    p = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    o = json.loads(p.stdout.strip().splitlines()[-1])
    assert o["ok"] and o["req"] == 4 and o["ver"] == 4, o
