"""Teacher-forced, element-by-element parity of every stage of the GPU forward (shared by
tests/test_gpu_layers.py and tools/layer_parity.py; test infrastructure).

Why teacher forcing. Comparing the GPU's intermediate values with a free-running bf16-emulating
oracle works only for the first few stages: the two compute each fp32 sum in a different order,
so about 1 in 10^4 bf16 roundings goes the other way, and each such flip perturbs the next
LayerNorm output by ~1/30 of a bf16 ulp, which flips a few % of THOSE roundings; after one layer
the two rounding sequences are decorrelated (measured: profiles/r02_layer_parity_free.ndjson,
where GPU-vs-emulation drifts to the emulation-vs-fp64 distance by layer 2). So instead every
stage is checked on the GPU's OWN inputs to that stage: the oracle's step (oracle/forward.py
`layer_ops`, fp64) is applied to the tapped GPU input and compared with the tapped GPU output.
A local bug anywhere (a dropped bias, a wrong scale, a transposed slice, a bad tile) shows up at
the stage that has it, undiluted.

Bars (derived in DESIGN.md §4):
  * fp32 outputs (q/k/v, residual after each block, logits):  max|gpu - ref| <= 1e-5 * max|ref|;
  * bf16 outputs (LN1, attention, LN2, ReLU): every element is a bf16 neighbour of the fp64
    value (|gpu - ref| <= 1 ulp(ref) + 1e-5 * max|ref|) and at most 1 % of the elements differ
    from RNE(ref) (the fp32 accumulation sits within ~1e-6 of ref, so few roundings can flip);
  * the embedding sum is exact (bitwise)."""
import numpy as np

from oracle import forward
from oracle.weights import round_bf16

FP32_BAR = 1e-5
BF16_FLIP_BAR = 0.01


def _ulp_bf16(v):
    """Spacing of bf16 numbers at |v| (8 significant bits): 2^(floor(log2|v|) - 7)."""
    a = np.abs(v)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, np.exp2(e - 7), 0.0)


def check_fp32(stage, layer, rank, g, ref):
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    den = float(np.abs(ref).max()) or 1.0
    err = float(np.abs(g - ref).max()) / den
    return {"stage": stage, "layer": layer, "rank": rank, "kind": "fp32", "maxabs_rel": err,
            "rel_l2": float(np.linalg.norm(g - ref) / (np.linalg.norm(ref) or 1.0)), "ok": err <= FP32_BAR}


def check_bf16(stage, layer, rank, g_bits, ref):
    ref = np.asarray(ref, np.float64)
    g = (np.asarray(g_bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rne = round_bf16(ref.astype(np.float32)).astype(np.float64)
    slack = 1e-5 * (float(np.abs(ref).max()) or 1.0)
    excess = np.abs(g - ref) - (_ulp_bf16(ref) + slack)
    flips = float(np.mean(g != rne))
    return {"stage": stage, "layer": layer, "rank": rank, "kind": "bf16", "flip_frac": flips,
            "max_excess_over_1ulp": float(max(excess.max(initial=-1.0), 0.0)),
            "ok": bool(np.all(excess <= 0)) and flips <= BF16_FLIP_BAR}


def _tap(M, ctx, model, tokens, layer, what, rank, cols, es):
    buf = ctx.tap(layer, what, rank, len(tokens) * cols * es)
    rid, _ = ctx.request(model, tokens)
    ctx.wait_request(rid, 120)
    dt = np.float32 if es == 4 else np.uint16
    return buf.view(dt).reshape(len(tokens), cols).copy()


def teacher_forced(M, ctx, model, d, tp, W, tokens, layers, bf16=True):
    """Records of every stage of the given layers (+ embedding, final LN and logits). bf16=False:
    the fp32 parity mode, where every stage is an fp32 output (FP32_BAR)."""
    L = len(tokens)
    hl, ffl, h = d.hidden // tp, d.ffn // tp, d.hidden
    nloc = d.heads // tp
    T = lambda l, what, r, cols, es: _tap(M, ctx, model, tokens, l, what, r, cols, es)
    recs = []
    # embedding (C5 step 1): exact
    x0 = T(0, M.TAP_X, 0, h, 4)
    # one fp32 addition of two stored weight values, as in the emulating oracle's step 1
    ref0 = (W["decoder.embed_tokens.weight"].astype(np.float32)[tokens]
            + W["decoder.embed_positions.weight"].astype(np.float32)[np.arange(L) + 2])
    recs.append({"stage": "embed", "layer": 0, "rank": 0, "kind": "exact",
                 "ok": bool(np.array_equal(x0, ref0))})
    es = 2 if bf16 else 4
    if bf16:
        f32 = lambda bits: (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        check_rnd = check_bf16
    else:
        f32 = lambda v: np.asarray(v, np.float64)
        check_rnd = check_fp32
    for l in layers:
        op = forward.layer_ops(d, W, l, np.float64)
        x = T(l, M.TAP_X, 0, h, 4).astype(np.float64)
        a = T(l, M.TAP_A, 0, h, es)
        recs.append(check_rnd("ln1", l, 0, a, op["ln1"](x)))
        full_q = op["qkv"](f32(a))                       # [L, 3h]
        os_ = []
        for r in range(tp):
            qkv_r = T(l, M.TAP_QKV, r, 3 * hl, 4)
            ref = np.concatenate([full_q[:, r * hl:(r + 1) * hl], full_q[:, h + r * hl:h + (r + 1) * hl],
                                  full_q[:, 2 * h + r * hl:2 * h + (r + 1) * hl]], axis=1)
            recs.append(check_fp32("qkv", l, r, qkv_r, ref))
            o_r = T(l, M.TAP_O, r, hl, es)
            recs.append(check_rnd("attn", l, r, o_r, op["attn"](qkv_r.astype(np.float64)[None], nloc)[0]))
            os_.append(f32(o_r))
        xm = T(l, M.TAP_XM, 0, h, 4)
        recs.append(check_fp32("attn_block", l, 0, xm, op["attn_block"](x, np.concatenate(os_, axis=1))))
        f = T(l, M.TAP_F, 0, h, es)
        recs.append(check_rnd("ln2", l, 0, f, op["ln2"](xm.astype(np.float64))))
        full_r = op["fc1"](f32(f))
        rs = []
        for r in range(tp):
            r_r = T(l, M.TAP_R, r, ffl, es)
            recs.append(check_rnd("fc1_relu", l, r, r_r, full_r[:, r * ffl:(r + 1) * ffl]))
            rs.append(f32(r_r))
        xn = T(l + 1, M.TAP_X, 0, h, 4)
        recs.append(check_fp32("mlp_block", l, 0, xn, op["mlp_block"](xm.astype(np.float64), np.concatenate(rs, axis=1))))
    # final LN + lm_head on the GPU's own inputs
    op = forward.layer_ops(d, W, d.n_layers, np.float64)
    xL = T(d.n_layers, M.TAP_X, 0, h, 4).astype(np.float64)
    aL = T(d.n_layers, M.TAP_A, 0, h, es)
    recs.append(check_rnd("lnf", d.n_layers, 0, aL, op["lnf"](xL)))
    rid, y = ctx.request(model, tokens)
    ctx.wait_request(rid, 120)
    recs.append(check_fp32("lm_head", d.n_layers, 0, y, op["lm_head"](f32(aL)[L - 1])))
    return recs
