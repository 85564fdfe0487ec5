"""Teacher-forced element-wise parity of every stage of the TP forward (a6), through the tap hook
(include/mpsw_testing.h): embedding (bitwise), LN1, q/k/v, attention, out_proj + all-reduce +
bias + residual, LN2, fc1 + ReLU, fc2 + all-reduce + bias + residual, final LN and lm_head, each
checked on the GPU's own inputs to that stage against the fp64 oracle step (tests/layer_taps.py
states the bars and why a free-running comparison cannot be element-wise)."""
import json
import os

import pytest

from synth import opt_dims, request_tokens
from oracle import layout
from tests import layer_taps as LT
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

LOG = os.environ.get("MPSW_PARITY_LOG")


def _run(name, tp, L, seed, dtype="bf16", layers=None):
    M = need_gpu()
    d = opt_dims(name)
    tok = request_tokens(seed, 0, 0, L, d.vocab)
    # weights regenerated per access by the oracle's C transcription of C0 for the OPT shapes
    W = layout.LazyFull(d, seed, dtype) if name.startswith("opt-") else layout.full_tensors(d, seed, dtype)
    dt = M.BF16 if dtype == "bf16" else M.FP32
    with M.Ctx(device_ids=(0,) * tp, budget=layout.shard_bytes(d, tp, dtype) + (2 << 20), max_batch=1,
               max_tokens=L, dtype=dt) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, seed)
        ctx.wait(ctx.swap_in(m))
        recs = LT.teacher_forced(M, ctx, m, d, tp, W, tok, layers or sorted({0, 1, d.n_layers - 1}),
                                 bf16=dtype == "bf16")
    if LOG:
        with open(LOG, "a") as f:
            for r in recs:
                f.write(json.dumps({"model": name, "tp": tp, "L": L, "dtype": dtype, **r}) + "\n")
    bad = [r for r in recs if not r["ok"]]
    assert not bad, bad
    return recs


@pytest.mark.parametrize("name,tp", [("small", 1), ("small", 2), ("small", 4), ("small", 8), ("opt-125m", 1),
                                     ("opt-125m", 4)])
def test_stages_bf16(name, tp):
    _run(name, tp, 8, 31 + tp)


@pytest.mark.parametrize("L", [1, 2, 17])
def test_stages_bf16_lengths(L):
    _run("small", 2, L, 40 + L)


def test_stages_bf16_opt1_3b_tp2():
    """OPT-1.3B at TP 2 (cfg2's shapes: K = 2048 / 4096, 16 heads per rank)."""
    _run("opt-1.3b", 2, 8, 7, layers=[0, 23])


def test_stages_bf16_opt13b_full_size():
    """Full-size OPT-13B (cfg3's model, 25.7 GB shard at TP 1): first and last layer, final LN and
    lm_head, teacher-forced against the fp64 oracle."""
    _run("opt-13b", 1, 2, 3, layers=[0, 39])


@pytest.mark.parametrize("tp", [1, 2])
def test_stages_fp32(tp):
    _run("small", tp, 8, 50 + tp, dtype="fp32")


@pytest.mark.slow
@pytest.mark.parametrize("name,tp,layers", [("opt-13b", 8, [0, 39]), ("opt-30b", 8, [0, 47])])
def test_stages_bf16_full_size_tp8(name, tp, layers):
    """cfg3 at t = 8 and cfg4's model at its TP degree (8 virtual ranks on one B200): every stage of
    the first and last layer, the final LN and lm_head, teacher-forced against the fp64 oracle —
    per-rank slices of q/k/v, attention and ReLU on all 8 ranks, the 8-way all-reduce blocks."""
    _run(name, tp, 8, 5, layers=layers)
