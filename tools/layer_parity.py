"""Per-layer element-wise parity of the GPU forward vs the oracle (diagnostic; prints NDJSON).

usage: python tools/layer_parity.py MODEL TP [L] [SEED] [--free]
Teacher-forced records of every stage (tests/layer_taps.py) of layers 0, 1 and the last one;
with --free, also the free-running comparison (GPU residual after every layer vs the emulating
and exact oracles), which shows the rounding-flip cascade that makes teacher forcing necessary."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2306_13835_b200 import mpsw as M  # noqa: E402
from synth import opt_dims, request_tokens  # noqa: E402
from oracle import layout, forward  # noqa: E402
from tests import layer_taps as LT  # noqa: E402
from tests.parity_util import logits_stats, f32_stats  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name, tp = args[0], int(args[1])
    L = int(args[2]) if len(args) > 2 else 8
    seed = int(args[3]) if len(args) > 3 else 31
    d = opt_dims(name)
    tok = request_tokens(seed, 0, 0, L, d.vocab)
    S_ = layout.shard_bytes(d, tp)
    W = layout.full_tensors(d, seed)
    tag = {"model": name, "tp": tp, "L": L}
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), max_batch=1, max_tokens=L) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, seed)
        ctx.wait(ctx.swap_in(m))
        for r in LT.teacher_forced(M, ctx, m, d, tp, W, tok, sorted({0, 1, d.n_layers - 1})):
            print(json.dumps({**tag, "mode": "teacher_forced", **r}), flush=True)
        if "--free" in sys.argv:
            em, ex = {}, {}
            forward.forward_bf16_emulated(d, W, tok[None], taps=em)
            forward.forward_exact(d, W, tok[None], taps=ex)
            for l in range(d.n_layers + 1):
                g = LT._tap(M, ctx, m, tok, l, M.TAP_X, 0, d.hidden, 4)
                e1, r1 = f32_stats(g, em[("x", l)][0])
                e2, r2 = f32_stats(g, ex[("x", l)][0])
                e3, r3 = f32_stats(em[("x", l)][0], ex[("x", l)][0])
                print(json.dumps({**tag, "mode": "free", "stage": "x", "layer": l, "rel_l2_gpu_em": r1,
                                  "rel_l2_gpu_ex": r2, "rel_l2_em_ex": r3}), flush=True)
        rid, y = ctx.request(m, tok)
        ctx.wait_request(rid, 120)
    yem = forward.forward_bf16_emulated(d, W, tok[None])[0]
    yex = forward.forward_exact(d, W, tok[None])[0]
    print(json.dumps({**tag, "mode": "logits", **logits_stats(y, yem, yex), "em_vs_ex": forward.rel_l2(yem, yex)}))


if __name__ == "__main__":
    main()
