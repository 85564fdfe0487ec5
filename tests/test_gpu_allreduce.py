"""The reduce-scatter all-reduce (each TP rank reduces + normalises its slice of the rows and
writes the bf16 LN rows into every rank's A operand) is bitwise identical to the direct mode
(every rank reduces every row): same adds in the same order per element, same LN code. Checked
end to end on logits for TP 2/4/8 (virtual ranks), ragged row counts (M not a multiple of t),
D = 2 batches in flight, and against the oracle. Each mode runs in its own process
(MPSW_RS_MIN_BYTES is read once)."""
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
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims, request_tokens
from oracle import layout
name, tp, D, out, dt = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
d = opt_dims(name)
lens = [8, 3, 8, 1, 7, 8, 5, 2, 8, 8, 6, 4]
toks = [request_tokens(77, 0, i, L, d.vocab) for i, L in enumerate(lens)]
with M.Ctx(device_ids=(0,) * tp, budget=layout.shard_bytes(d, tp, dt) + (2 << 20), max_batch=6, max_tokens=8,
           max_inflight=D, dtype=M.BF16 if dt == "bf16" else M.FP32) as ctx:
    m = ctx.register_model(d)
    ctx.synth_fill(m, 12)
    ctx.wait(ctx.swap_in(m))
    rids = [ctx.request(m, t) for t in toks]
    for rid, _ in rids:
        ctx.wait_request(rid, 120)
    np.save(out, np.stack([o for _, o in rids]))
'''


def _run(tmp_path, name, tp, D, rs_min, dt="bf16"):
    out = str(tmp_path / f"{name}_{tp}_{D}_{rs_min}_{dt}.npy")
    env = dict(os.environ, MPSW_RS_MIN_BYTES=str(rs_min))
    p = subprocess.run([sys.executable, "-c", CHILD, name, str(tp), str(D), out, dt], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("name,tp,D,dt", [("small", 2, 1, "bf16"), ("small", 4, 2, "bf16"), ("small", 8, 1, "bf16"),
                                         ("mid", 4, 1, "bf16"), ("small", 4, 1, "fp32")])
def test_reduce_scatter_bitwise_equals_direct(tmp_path, name, tp, D, dt):
    need_gpu()
    direct = _run(tmp_path, name, tp, D, 1 << 62, dt)
    rs = _run(tmp_path, name, tp, D, 0, dt)
    assert np.array_equal(direct, rs)
    d = opt_dims(name)
    W = layout.full_tensors(d, 12, dt)
    lens = [8, 3, 8, 1, 7, 8, 5, 2, 8, 8, 6, 4]
    for i in (0, 3, 11):
        t = request_tokens(77, 0, i, lens[i], d.vocab)
        ex = forward.forward_exact(d, W, t[None])[0]
        if dt == "bf16":
            PU.assert_logits(rs[i], forward.forward_bf16_emulated(d, W, t[None])[0], ex, tag=f"rs {name} tp{tp}")
        else:
            PU.assert_logits(rs[i], None, ex, tol=PU.FP32_LOGITS_TOL, tag=f"rs fp32 tp{tp}")
