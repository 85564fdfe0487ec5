"""CUDA-graph replay of the TP = 1 forward (batch.cpp: the first batch of a (model, range offset,
M, B) runs eagerly, the second is captured, later ones replay the graph): logits are bitwise equal
to the eager path (MPSW_GRAPHS=0) over repeated shapes, two models swapping through one range
(same offset, different weights), ragged batches, and the engine's launch accounting counts the
graph's kernels."""
import os
import subprocess
import sys

import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, forward
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json
import numpy as np
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims, request_tokens
from oracle import layout
out = sys.argv[1]
d = opt_dims("small")
S = layout.shard_bytes(d, 1)
res = []
with M.Ctx(device_ids=(0,), budget=(S + 4095) // 4096 * 4096, max_batch=4, max_tokens=8) as ctx:
    a, b = ctx.register_model(d), ctx.register_model(d)
    ctx.synth_fill(a, 31); ctx.synth_fill(b, 32)
    for it in range(5):
        for m in (a, b, a):                      # every request swaps: same offset, other weights
            rid, y = ctx.request(m, request_tokens(3, m, it, 8, d.vocab))
            ctx.wait_request(rid, 120)
            res.append(y.copy())
        rids = [ctx.request(a, request_tokens(4, 0, it * 4 + j, L, d.vocab)) for j, L in enumerate((8, 3, 5))]
        for rid, y in rids:
            ctx.wait_request(rid, 120)
            res.append(y.copy())
    st = ctx.stats()
np.save(out, np.stack(res))
print(json.dumps({"launches": st["kernel_launches"], "batches": st["batches"]}))
'''


def test_graph_replay_bitwise_equals_eager(tmp_path):
    need_gpu()
    outs, meta = {}, {}
    for g in ("0", "1"):
        p = subprocess.run([sys.executable, "-c", CHILD, str(tmp_path / f"g{g}.npy")], cwd=ROOT,
                           env=dict(os.environ, MPSW_GRAPHS=g), capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-3000:]
        outs[g] = np.load(str(tmp_path / f"g{g}.npy"))
        meta[g] = p.stdout.strip().splitlines()[-1]
    assert np.array_equal(outs["0"], outs["1"])
    assert meta["0"] == meta["1"]                 # same kernels counted with and without graphs
    d = opt_dims("small")
    W = layout.full_tensors(d, 31)
    PU.assert_logits(outs["1"][-3], forward.forward_bf16_emulated(d, W, request_tokens(4, 0, 16, 8, d.vocab)[None])[0],
                     tag="graphs")
