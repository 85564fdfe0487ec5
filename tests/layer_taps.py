"""Per-layer tap comparison of the GPU forward against the bf16-emulating oracle (shared by
tests/test_gpu_layers.py and tools/layer_parity.py; test infrastructure).

`gpu_taps` runs the library forward through the one-shot tap hook (include/mpsw_testing.h,
mpsw_test_tap) and `compare` lines every tapped buffer up with the oracle's value of the same
quantity (oracle/forward.py `taps`), element by element."""
import numpy as np

from oracle import forward
from tests.parity_util import bf16_bits_of_f32, ulp_stats, f32_stats


def tap_points(n_layers):
    """(what, layer) pairs: the embedding, every intermediate of layers 0 and 1, the residual and
    LN output after layers 1, 2 and all of them."""
    pts = [("x", 0), ("a", 0), ("qkv", 0), ("o", 0), ("r", 0), ("x", 1), ("a", 1)]
    if n_layers > 1:
        pts += [("qkv", 1), ("o", 1), ("r", 1), ("x", 2), ("a", 2)]
    pts += [("x", n_layers), ("a", n_layers)]
    out = []
    for p in pts:
        if p not in out and p[1] <= n_layers:
            out.append(p)
    return out


def gpu_taps(M, ctx, model, d, tp, tokens, points, dtype_bf16=True):
    """{(what, layer, rank): array} from the GPU; tokens: [L] int32 (one request per batch)."""
    what_id = {"x": M.TAP_X, "a": M.TAP_A, "qkv": M.TAP_QKV, "o": M.TAP_O, "r": M.TAP_R}
    Lt = len(tokens)
    hl = d.hidden // tp
    ffl = d.ffn // tp
    es = 2 if dtype_bf16 else 4
    out = {}
    for what, l in points:
        ranks = range(tp) if what in ("qkv", "o", "r") else [0]
        for r in ranks:
            cols = {"x": d.hidden, "a": d.hidden, "qkv": 3 * hl, "o": hl, "r": ffl}[what]
            nb = Lt * cols * (4 if what in ("x", "qkv") else es)
            buf = ctx.tap(l, what_id[what], r, nb)
            rid, _ = ctx.request(model, tokens)
            ctx.wait_request(rid, 120)
            if what in ("x", "qkv") or not dtype_bf16:
                out[(what, l, r)] = buf.view(np.float32).reshape(Lt, cols).copy()
            else:
                out[(what, l, r)] = buf.view(np.uint16).reshape(Lt, cols).copy()
    return out


def oracle_slice(d, tp, what, r, v):
    """Rank r's columns of an oracle tap value [L, ...] (Megatron layout, oracle/layout.py)."""
    hl = d.hidden // tp
    if what == "qkv":
        h = d.hidden
        return np.concatenate([v[:, r * hl:(r + 1) * hl], v[:, h + r * hl:h + (r + 1) * hl],
                               v[:, 2 * h + r * hl:2 * h + (r + 1) * hl]], axis=1)
    if what == "o":
        return v[:, r * hl:(r + 1) * hl]
    if what == "r":
        f = d.ffn // tp
        return v[:, r * f:(r + 1) * f]
    return v


def oracle_taps(d, W, tokens, max_layer):
    em, ex = {}, {}
    forward.forward_bf16_emulated(d, W, tokens[None], taps=em, n_layers=None if max_layer >= d.n_layers else max_layer)
    forward.forward_exact(d, W, tokens[None], taps=ex, n_layers=None if max_layer >= d.n_layers else max_layer)
    return em, ex


def compare(d, tp, gpu, em, ex, dtype_bf16=True):
    """One record per tapped buffer: bf16 buffers -> fraction of elements off by >= 1 ulp and the
    max ulp vs the emulating oracle; fp32 buffers -> max |diff| / max |ref| and rel-L2 vs the
    emulating oracle; every buffer also vs the exact (fp64) oracle."""
    recs = []
    for (what, l, r), g in sorted(gpu.items(), key=lambda kv: (kv[0][1], kv[0][0], kv[0][2])):
        ref = oracle_slice(d, tp, what, r, em[(what, l)][0])
        rex = oracle_slice(d, tp, what, r, ex[(what, l)][0])
        rec = {"what": what, "layer": l, "rank": r}
        if g.dtype == np.uint16:
            frac, mx = ulp_stats(g, bf16_bits_of_f32(ref))
            rec.update(ulp_frac=frac, ulp_max=mx)
            gv = (g.astype(np.uint32) << 16).view(np.float32)
        else:
            gv = g
            rec["maxabs_em"], rec["rel_l2_em"] = f32_stats(gv, ref)
        rec["maxabs_ex"], rec["rel_l2_ex"] = f32_stats(gv, rex)
        recs.append(rec)
    return recs
