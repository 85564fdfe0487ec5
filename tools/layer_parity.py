"""Per-layer element-wise parity of the GPU forward vs the oracle (diagnostic; prints NDJSON).

usage: python tools/layer_parity.py MODEL TP [L] [SEED] [--all-layers]
Every tap point of tests/layer_taps.py, plus (with --all-layers) the residual after every layer."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2306_13835_b200 import mpsw as M  # noqa: E402
from synth import opt_dims, request_tokens  # noqa: E402
from oracle import layout, forward  # noqa: E402
from tests import layer_taps as LT  # noqa: E402
from tests.parity_util import logits_stats  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name, tp = args[0], int(args[1])
    L = int(args[2]) if len(args) > 2 else 8
    seed = int(args[3]) if len(args) > 3 else 31
    d = opt_dims(name)
    tok = request_tokens(seed, 0, 0, L, d.vocab)
    pts = LT.tap_points(d.n_layers)
    if "--all-layers" in sys.argv:
        pts += [("x", l) for l in range(3, d.n_layers) if ("x", l) not in pts]
    S_ = layout.shard_bytes(d, tp)
    W = layout.full_tensors(d, seed)
    em, ex = LT.oracle_taps(d, W, tok, d.n_layers)
    with M.Ctx(device_ids=(0,) * tp, budget=S_ + (2 << 20), max_batch=1, max_tokens=L) as ctx:
        m = ctx.register_model(d)
        ctx.synth_fill(m, seed)
        ctx.wait(ctx.swap_in(m))
        g = LT.gpu_taps(M, ctx, m, d, tp, tok, pts)
        rid, y = ctx.request(m, tok)
        ctx.wait_request(rid, 120)
    for r in LT.compare(d, tp, g, em, ex):
        print(json.dumps({"model": name, "tp": tp, "L": L, **r}))
    yem = forward.forward_bf16_emulated(d, W, tok[None])[0]
    yex = forward.forward_exact(d, W, tok[None])[0]
    print(json.dumps({"model": name, "tp": tp, "L": L, "what": "logits", **logits_stats(y, yem, yex),
                      "em_vs_ex": forward.rel_l2(yem, yex)}))


if __name__ == "__main__":
    main()
