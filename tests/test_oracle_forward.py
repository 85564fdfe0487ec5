"""Pins for oracle/forward.py (C5): HF OPTForCausalLM (library routine, independent code) in
float64 with the same weights; TP-sharded == unsharded; bf16 emulation close to exact."""
import numpy as np
import pytest

from synth import opt_dims, request_tokens
from oracle import layout, forward


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
