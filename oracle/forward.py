"""C5 — OPT forward pass (oracle side), plain definition.

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

The paper serves OPT-13B and never restates the architecture; the external pin is
HF `OPTForCausalLM` (transformers 5.5: modeling_opt.py) with do_layer_norm_before=True,
ReLU, LayerNorm eps 1e-5 (biased variance), learned positions with offset 2, tied lm_head,
no KV cache (a request is one forward over its L tokens; reading #9).

    h0 = E_tok[x] + E_pos[arange(L) + 2]
    per layer:  a = LN1(h); q = (a Wq^T + bq) * hd^-0.5; k = a Wk^T + bk; v = a Wv^T + bv
                o = concat_heads softmax(q k^T + causal) v;   h = h + o Wo^T + bo
                f = LN2(h);  h = h + relu(f W1^T + b1) W2^T + b2
    logits = LNf(h)[:, L-1] E_tok^T                                       (fp32 out, [B, V])

Two precision modes (reading #20):
  * `forward_exact`: float64 math on the stored weight values, no intermediate rounding.
  * `forward_bf16_emulated`: float32 math, rounding to bf16 (RNE) exactly at the GPU path's
    documented storage points = GEMM A-operands: LN1/LN2/LNf outputs, the attention output o
    and the ReLU output.  Residual stream, q/k/v, softmax and all-reduce partials stay fp32.
`forward_tp_simulated` runs the Megatron-sharded computation rank by rank (summing partials)
to pin that the TP layout of oracle.layout computes the same function.
"""
import numpy as np

from .weights import round_bf16

EPS = 1e-5


def layer_norm(x, g, b, dt):
    x = x.astype(dt)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return ((x - mu) / np.sqrt(var + dt(EPS))) * g.astype(dt) + b.astype(dt)


def _attention(q, k, v, heads, dt):
    """q,k,v: [B, L, n*hd] (n local heads) -> o [B, L, n*hd]; fp32/fp64 softmax."""
    B, L, H = q.shape
    hd = H // heads
    q = q.reshape(B, L, heads, hd).transpose(0, 2, 1, 3)
    k = k.reshape(B, L, heads, hd).transpose(0, 2, 1, 3)
    v = v.reshape(B, L, heads, hd).transpose(0, 2, 1, 3)
    s = q @ k.transpose(0, 1, 3, 2)                               # [B, n, L, L]
    mask = np.triu(np.ones((L, L), dtype=bool), k=1)
    s = np.where(mask, dt(-np.inf), s)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    o = p @ v
    return o.transpose(0, 2, 1, 3).reshape(B, L, H).astype(dt)


def _run(d, W, tokens, dt, rnd, taps=None, n_layers=None):
    """taps: optional dict filled with the intermediate values, keyed (name, layer):
    ("x", l) residual stream after l layers [B, L, h]; ("a", l) the LN output feeding layer l
    (l = L_m: the final LN over all positions); ("qkv", l) = [q | k | v] [B, L, 3h] (q scaled);
    ("o", l) attention output [B, L, h]; ("r", l) ReLU output [B, L, ff]. Recording only: the
    arithmetic is the same with or without it. n_layers: stop after that many layers (returns
    None; for taps)."""
    tokens = np.asarray(tokens)
    B, L = tokens.shape
    hd = d.hidden // d.heads
    g = lambda n: W[n].astype(dt)
    rec = (lambda k, l, v: taps.__setitem__((k, l), v)) if taps is not None else (lambda k, l, v: None)
    h = g("decoder.embed_tokens.weight")[tokens] + g("decoder.embed_positions.weight")[np.arange(L) + 2][None]
    rec("x", 0, h)
    scale = dt(hd ** -0.5)
    for i in range(d.n_layers if n_layers is None else n_layers):
        p = f"decoder.layers.{i}."
        a = rnd(layer_norm(h, W[p + "self_attn_layer_norm.weight"], W[p + "self_attn_layer_norm.bias"], dt))
        rec("a", i, a)
        q = (a @ g(p + "self_attn.q_proj.weight").T + g(p + "self_attn.q_proj.bias")) * scale
        k = a @ g(p + "self_attn.k_proj.weight").T + g(p + "self_attn.k_proj.bias")
        v = a @ g(p + "self_attn.v_proj.weight").T + g(p + "self_attn.v_proj.bias")
        rec("qkv", i, np.concatenate([q, k, v], axis=-1))
        o = rnd(_attention(q, k, v, d.heads, dt))
        rec("o", i, o)
        h = h + (o @ g(p + "self_attn.out_proj.weight").T + g(p + "self_attn.out_proj.bias"))
        f = rnd(layer_norm(h, W[p + "final_layer_norm.weight"], W[p + "final_layer_norm.bias"], dt))
        r = rnd(np.maximum(f @ g(p + "fc1.weight").T + g(p + "fc1.bias"), dt(0)))
        rec("r", i, r)
        h = h + (r @ g(p + "fc2.weight").T + g(p + "fc2.bias"))
        rec("x", i + 1, h)
    if n_layers is not None and n_layers < d.n_layers:
        return None
    if taps is not None:
        rec("a", d.n_layers, rnd(layer_norm(h, W["decoder.final_layer_norm.weight"], W["decoder.final_layer_norm.bias"], dt)))
    x = rnd(layer_norm(h[:, L - 1], W["decoder.final_layer_norm.weight"], W["decoder.final_layer_norm.bias"], dt))
    return x @ g("decoder.embed_tokens.weight").T


def forward_exact(d, W, tokens, taps=None, n_layers=None):
    """float64 logits [B, V] of the last position.  W: dict name -> full tensor values."""
    return _run(d, W, tokens, np.float64, lambda x: x, taps, n_layers)


def forward_bf16_emulated(d, W, tokens, taps=None, n_layers=None):
    """float32 logits [B, V], bf16 rounding at the GEMM A-operand storage points."""
    return _run(d, W, tokens, np.float32, lambda x: round_bf16(x.astype(np.float32)), taps, n_layers)


def layer_ops(d, W, i, dt=np.float64, rnd=lambda x: x):
    """The steps of C5 for decoder layer i (i = d.n_layers: the final LN / lm_head) as separate
    functions, each computing ONE step from given inputs, in the order and arithmetic of `_run`
    (composing them in that order reproduces forward_exact / forward_bf16_emulated exactly,
    tests/test_oracle_forward.py). Used for teacher-forced parity: each GPU stage is checked
    against this step applied to the GPU's own inputs of that stage.
      ln1(x) -> a;  qkv(a) -> [q|k|v];  attn(qkv, heads) -> o;  attn_block(x, o) -> xm;
      ln2(xm) -> f;  fc1(f) -> r;  mlp_block(xm, r) -> x';  lnf(x) -> a_f;  lm_head(a_f) -> logits.
    Arrays are [..., features]; attn takes [B, L, 3*n*hd] with n local heads."""
    g = lambda n: W[n].astype(dt)
    p = f"decoder.layers.{i}."
    hd = d.hidden // d.heads
    scale = dt(hd ** -0.5)
    ops = {}
    if i < d.n_layers:
        def qkv(a):
            q = (a @ g(p + "self_attn.q_proj.weight").T + g(p + "self_attn.q_proj.bias")) * scale
            k = a @ g(p + "self_attn.k_proj.weight").T + g(p + "self_attn.k_proj.bias")
            v = a @ g(p + "self_attn.v_proj.weight").T + g(p + "self_attn.v_proj.bias")
            return np.concatenate([q, k, v], axis=-1)

        def attn(qkv_, heads):
            n = qkv_.shape[-1] // 3
            return rnd(_attention(qkv_[..., :n], qkv_[..., n:2 * n], qkv_[..., 2 * n:], heads, dt))

        ops["ln1"] = lambda x: rnd(layer_norm(x, W[p + "self_attn_layer_norm.weight"], W[p + "self_attn_layer_norm.bias"], dt))
        ops["qkv"] = qkv
        ops["attn"] = attn
        ops["attn_block"] = lambda x, o: x + (o @ g(p + "self_attn.out_proj.weight").T + g(p + "self_attn.out_proj.bias"))
        ops["ln2"] = lambda xm: rnd(layer_norm(xm, W[p + "final_layer_norm.weight"], W[p + "final_layer_norm.bias"], dt))
        ops["fc1"] = lambda f: rnd(np.maximum(f @ g(p + "fc1.weight").T + g(p + "fc1.bias"), dt(0)))
        ops["mlp_block"] = lambda xm, r: xm + (r @ g(p + "fc2.weight").T + g(p + "fc2.bias"))
    else:
        ops["lnf"] = lambda x: rnd(layer_norm(x, W["decoder.final_layer_norm.weight"], W["decoder.final_layer_norm.bias"], dt))
        ops["lm_head"] = lambda a: a @ g("decoder.embed_tokens.weight").T
    return ops


def forward_tp_simulated(d, shards, tokens, dt=np.float64):
    """Megatron-sharded forward: shards[r] = dict name -> rank-r shard values.
    Partials of row-parallel GEMMs (and of the vocab-parallel embedding) are summed
    across ranks (the TP all-reduce, "distributed collectives"); replicated biases
    added once after the sum; logits = concatenation of the ranks' vocab slices."""
    tp = len(shards)
    tokens = np.asarray(tokens)
    B, L = tokens.shape
    hd = d.hidden // d.heads
    nloc = d.heads // tp
    Vl = d.vocab // tp
    S0 = shards[0]
    g = lambda r, n: shards[r][n].astype(dt)
    emb = np.zeros((B, L, d.hidden), dt)
    for r in range(tp):
        lo = r * Vl
        inr = (tokens >= lo) & (tokens < lo + Vl)
        part = g(r, "decoder.embed_tokens.weight")[np.where(inr, tokens - lo, 0)]
        emb += np.where(inr[..., None], part, dt(0))
    h = emb + g(0, "decoder.embed_positions.weight")[np.arange(L) + 2][None]
    scale = dt(hd ** -0.5)
    for i in range(d.n_layers):
        p = f"decoder.layers.{i}."
        a = layer_norm(h, S0[p + "self_attn_layer_norm.weight"], S0[p + "self_attn_layer_norm.bias"], dt)
        acc = np.zeros_like(h)
        for r in range(tp):
            q = (a @ g(r, p + "self_attn.q_proj.weight").T + g(r, p + "self_attn.q_proj.bias")) * scale
            k = a @ g(r, p + "self_attn.k_proj.weight").T + g(r, p + "self_attn.k_proj.bias")
            v = a @ g(r, p + "self_attn.v_proj.weight").T + g(r, p + "self_attn.v_proj.bias")
            o = _attention(q, k, v, nloc, dt)
            acc += o @ g(r, p + "self_attn.out_proj.weight").T
        h = h + acc + g(0, p + "self_attn.out_proj.bias")
        f = layer_norm(h, S0[p + "final_layer_norm.weight"], S0[p + "final_layer_norm.bias"], dt)
        acc = np.zeros_like(h)
        for r in range(tp):
            acc += np.maximum(f @ g(r, p + "fc1.weight").T + g(r, p + "fc1.bias"), dt(0)) @ g(r, p + "fc2.weight").T
        h = h + acc + g(0, p + "fc2.bias")
    x = layer_norm(h[:, L - 1], S0["decoder.final_layer_norm.weight"], S0["decoder.final_layer_norm.bias"], dt)
    return np.concatenate([x @ g(r, "decoder.embed_tokens.weight").T for r in range(tp)], axis=-1)


def rel_l2(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
