"""Pins for oracle/forward.py (C5): HF OPTForCausalLM (library routine, independent code) in
float64 with the same weights; TP-sharded == unsharded; bf16 emulation close to exact."""
import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, forward


def _hf_model(d, W, dtype):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    cfg = tr.OPTConfig(vocab_size=d.vocab, hidden_size=d.hidden, num_hidden_layers=d.n_layers,
                       ffn_dim=d.ffn, num_attention_heads=d.heads, max_position_embeddings=d.max_pos,
                       word_embed_proj_dim=d.hidden, dropout=0.0, attention_dropout=0.0,
                       pad_token_id=1, attn_implementation="eager")
    m = tr.OPTForCausalLM(cfg).to(dtype).eval()
    npdt = np.float64 if dtype == torch.float64 else np.float32
    sd = {"model." + k: torch.from_numpy(np.asarray(v, npdt)) for k, v in W.items()}
    sd["lm_head.weight"] = sd["model.decoder.embed_tokens.weight"]
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("lm_head" in k for k in missing)
    return m


def _hf_logits(d, W, tokens):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    cfg = tr.OPTConfig(vocab_size=d.vocab, hidden_size=d.hidden, num_hidden_layers=d.n_layers,
                       ffn_dim=d.ffn, num_attention_heads=d.heads, max_position_embeddings=d.max_pos,
                       word_embed_proj_dim=d.hidden, dropout=0.0, attention_dropout=0.0,
                       pad_token_id=1)
    m = tr.OPTForCausalLM(cfg).double().eval()
    sd = {"model." + k: torch.from_numpy(np.asarray(v, np.float64)) for k, v in W.items()}
    sd["lm_head.weight"] = sd["model.decoder.embed_tokens.weight"]
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("lm_head" in k for k in missing)
    with torch.no_grad():
        out = m(input_ids=torch.from_numpy(np.asarray(tokens, np.int64)),
                attention_mask=torch.ones(tokens.shape, dtype=torch.long))
    return out.logits[:, -1].numpy()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_exact_matches_hf_fp64(dtype):
    d = opt_dims("tiny")
    W = layout.full_tensors(d, 11, dtype)
    tok = np.stack([request_tokens(0, 0, i, 8, d.vocab) for i in range(3)])
    ours = forward.forward_exact(d, W, tok)
    ref = _hf_logits(d, W, tok)
    assert forward.rel_l2(ours, ref) < 1e-12
    assert np.array_equal(ours.argmax(-1), ref.argmax(-1))


def test_exact_matches_hf_single_token_and_len2():
    d = opt_dims("tiny")
    W = layout.full_tensors(d, 2)
    for L in (1, 2):
        tok = np.stack([request_tokens(1, 0, i, L, d.vocab) for i in range(2)])
        assert forward.rel_l2(forward.forward_exact(d, W, tok), _hf_logits(d, W, tok)) < 1e-12


@pytest.mark.parametrize("tp", [1, 2, 4])
def test_tp_sharded_equals_unsharded(tp):
    d = opt_dims("tiny")
    W = layout.full_tensors(d, 4)
    shards = [layout.shard_tensors(d, tp, r, 4) for r in range(tp)]
    tok = np.stack([request_tokens(2, 0, i, 8, d.vocab) for i in range(2)])
    a = forward.forward_exact(d, W, tok)
    b = forward.forward_tp_simulated(d, shards, tok)
    assert forward.rel_l2(b, a) < 1e-12


def test_bf16_emulated_near_exact_and_rounds():
    d = opt_dims("small")
    W = layout.full_tensors(d, 6)
    tok = np.stack([request_tokens(3, 0, i, 8, d.vocab) for i in range(2)])
    ex = forward.forward_exact(d, W, tok)
    em = forward.forward_bf16_emulated(d, W, tok)
    err = forward.rel_l2(em, ex)
    # rounding at the A-operands is visible but bounded (SURVEY §8(c) C5 measured ~5e-3)
    assert 1e-5 < err < 1e-2
    assert em.dtype == np.float32


def test_causality():
    """Changing a later token cannot change earlier positions: the last-position logits of a
    length-3 prefix equal those of the 3-token request itself."""
    d = opt_dims("tiny")
    W = layout.full_tensors(d, 8)
    tok = request_tokens(4, 0, 0, 6, d.vocab)[None]
    a = forward.forward_exact(d, W, tok[:, :3])
    tok2 = tok.copy(); tok2[0, 4] = (tok2[0, 4] + 1) % d.vocab
    b = forward.forward_exact(d, W, tok2[:, :3])
    assert np.array_equal(a, b)


def _hf_bf16_at_linear_inputs(d, W, tokens, skip_in=(), extra_out_round=()):
    """HF OPTForCausalLM in float32 with a forward-pre-hook on EVERY nn.Linear that rounds the
    Linear's input to bf16 (torch's own RNE conversion): the plain definition of "bf16 rounding
    exactly at the GEMM A-operands" (reading #20) written with library code. The
    residual stream, LayerNorm statistics, q/k/v, softmax and partial sums stay float32.
    Mutations: skip_in = Linear names whose input is NOT rounded; extra_out_round = Linear names
    whose OUTPUT is also rounded."""
    torch = pytest.importorskip("torch")
    m = _hf_model(d, W, torch.float32)
    rb = lambda t: t.to(torch.bfloat16).to(torch.float32)
    for name, mod in m.named_modules():
        if isinstance(mod, torch.nn.Linear):
            if not any(name.endswith(x) for x in skip_in):
                mod.register_forward_pre_hook(lambda _m, args: (rb(args[0]),) + tuple(args[1:]))
            if any(name.endswith(x) for x in extra_out_round):
                mod.register_forward_hook(lambda _m, _a, out: rb(out))
    with torch.no_grad():
        out = m(input_ids=torch.from_numpy(np.asarray(tokens, np.int64)),
                attention_mask=torch.ones(tokens.shape, dtype=torch.long))
    return out.logits[:, -1].double().numpy()


PIN_BAR = 2e-5


def test_bf16_emulation_storage_points_match_hf_hooks():
    """Pins forward_bf16_emulated's storage points (reading #20) against an independent
    construction: HF's OPT forward with bf16 rounding hooked onto every Linear input. Only fp32
    summation order differs, so the two agree far inside PIN_BAR. Each plausible storage-point
    mistake (q/k/v rounded; attention output, ReLU output or final-LN output left unrounded; no
    rounding at all) moves the HF construction by well over PIN_BAR, so an oracle with that
    mistake would fail the first assertion."""
    d = opt_dims("small")
    W = layout.full_tensors(d, 6)
    tok = np.stack([request_tokens(3, 0, i, 8, d.vocab) for i in range(3)])
    em = forward.forward_bf16_emulated(d, W, tok)
    hf = _hf_bf16_at_linear_inputs(d, W, tok)
    err = forward.rel_l2(em, hf)
    assert err < PIN_BAR, err
    mutants = {
        "qkv rounded": dict(extra_out_round=("q_proj", "k_proj", "v_proj")),
        "o unrounded": dict(skip_in=("out_proj",)),
        "relu unrounded": dict(skip_in=("fc2",)),
        "final LN unrounded": dict(skip_in=("lm_head",)),
    }
    for what, kw in mutants.items():
        mut = _hf_bf16_at_linear_inputs(d, W, tok, **kw)
        assert forward.rel_l2(mut, em) > 5 * PIN_BAR, what
    assert forward.rel_l2(forward.forward_exact(d, W, tok), em) > 50 * PIN_BAR


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_layer_ops_compose_to_forward(mode):
    """layer_ops (the per-step functions used for teacher-forced GPU parity) composed in C5's
    order reproduce forward_exact / forward_bf16_emulated bit for bit."""
    from oracle.weights import round_bf16
    d = opt_dims("small")
    W = layout.full_tensors(d, 9)
    tok = np.stack([request_tokens(5, 0, i, 6, d.vocab) for i in range(2)])
    dt, rnd = (np.float64, lambda x: x) if mode == "exact" else (np.float32, lambda x: round_bf16(x.astype(np.float32)))
    ref = (forward.forward_exact if mode == "exact" else forward.forward_bf16_emulated)(d, W, tok)
    L = tok.shape[1]
    h = W["decoder.embed_tokens.weight"].astype(dt)[tok] + W["decoder.embed_positions.weight"].astype(dt)[np.arange(L) + 2][None]
    for i in range(d.n_layers):
        op = forward.layer_ops(d, W, i, dt, rnd)
        xm = op["attn_block"](h, op["attn"](op["qkv"](op["ln1"](h)), d.heads))
        h = op["mlp_block"](xm, op["fc1"](op["ln2"](xm)))
    op = forward.layer_ops(d, W, d.n_layers, dt, rnd)
    y = op["lm_head"](op["lnf"](h[:, L - 1]))
    assert np.array_equal(y, ref)
