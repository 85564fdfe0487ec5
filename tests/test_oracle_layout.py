"""Pins for oracle/layout.py (C2): HF tensor order/counts, conservation, shard reconstruction."""
import numpy as np
import pytest

from synth import opt_dims, OPT_PRESETS
from oracle import layout


def _hf_names_and_count(d):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    cfg = tr.OPTConfig(vocab_size=d.vocab, hidden_size=d.hidden, num_hidden_layers=d.n_layers,
                       ffn_dim=d.ffn, num_attention_heads=d.heads, max_position_embeddings=d.max_pos,
                       word_embed_proj_dim=d.hidden)
    with torch.device("meta"):
        m = tr.OPTForCausalLM(cfg)
    names = [(n[len("model."):], tuple(p.shape)) for n, p in m.named_parameters()]
    return names, sum(p.numel() for p in m.parameters())


@pytest.mark.parametrize("name,T", [("opt-125m", 196), ("opt-1.3b", 388), ("opt-13b", 644), ("opt-30b", 772)])
def test_tensor_order_and_counts_match_hf(name, T):
    d = opt_dims(name)
    names, nparams = _hf_names_and_count(d)
    specs = layout.canonical_tensors(d)
    assert len(specs) == T == len(names)
    assert [(s.name, s.shape) for s in specs] == names
    assert sum(int(np.prod(s.shape)) for s in specs) == nparams


def test_known_param_count_125m():
    d = opt_dims("opt-125m")
    assert sum(int(np.prod(s.shape)) for s in layout.canonical_tensors(d)) == 125_239_296


@pytest.mark.parametrize("name,t", [("opt-1.3b", 2), ("opt-13b", 4), ("opt-13b", 8), ("opt-30b", 8), ("opt-125m", 2)])
def test_conservation(name, t):
    """sum_r S_r(t) = S + (t-1) S_rep when no padding is needed (adjusted)."""
    d = opt_dims(name)
    S = layout.shard_bytes(d, 1)
    S_rep = layout.replicated_bytes(d)
    assert t * layout.shard_bytes(d, t) == S + (t - 1) * S_rep


def test_survey_shard_sizes():
    assert layout.shard_bytes(opt_dims("opt-13b"), 4) == 6_444_339_200
    assert layout.shard_bytes(opt_dims("opt-30b"), 8) == 7_522_988_032
    assert layout.shard_bytes(opt_dims("opt-1.3b"), 2) == 1_320_255_488
    assert layout.shard_bytes(opt_dims("opt-125m"), 1) == 250_478_592


@pytest.mark.parametrize("tp", [1, 2, 4])
def test_shards_reconstruct_full(tp):
    d = opt_dims("tiny")
    full = layout.full_tensors(d, 5)
    shards = [layout.shard_tensors(d, tp, r, 5) for r in range(tp)]
    for s in layout.canonical_tensors(d):
        parts = [sh[s.name] for sh in shards]
        if s.split == layout.REPL:
            for p in parts:
                assert np.array_equal(p, full[s.name])
        elif s.split == layout.ROWS:
            assert np.array_equal(np.concatenate(parts, axis=0), full[s.name])
        else:
            assert np.array_equal(np.concatenate(parts, axis=1), full[s.name])


def test_alignment_and_padding_zero():
    d = opt_dims("tiny")
    placed, total = layout.arena_layout(d, 2, 1)
    assert total % 256 == 0
    img = layout.shard_image(d, 2, 1, 3)
    covered = np.zeros(total, bool)
    for p in placed:
        assert p.offset % 256 == 0
        covered[p.offset:p.offset + p.nbytes] = True
    assert np.all(img[~covered] == 0)
    # element_at agrees with the image (sampled, one by one)
    for off in [0, 2, 254, placed[5].offset + 6, total - 2]:
        e = layout.element_at(d, 2, 1, 3, off)
        got = int(img[off - off % 2:off - off % 2 + 2].view(np.uint16)[0])
        assert (e is None and got == 0) or int(e) == got


def test_invalid_tp():
    with pytest.raises(ValueError):
        layout.arena_layout(opt_dims("opt-125m"), 8, 0)   # 12 heads


@pytest.mark.parametrize("pp", [1, 2])
def test_pp_stages_partition_layers(pp):
    """Every layer tensor is held by exactly one stage; embed_tokens by the first and the last
    stage (tied lm_head), positions by the first, the final LN by the last."""
    d = opt_dims("tiny")
    holders = {}
    for st in range(pp):
        for p in layout.arena_layout(d, 1, 0, "bf16", pp, st)[0]:
            holders.setdefault(p.spec.name, []).append(st)
    for s in layout.canonical_tensors(d):
        h = holders[s.name]
        if s.name == "decoder.embed_tokens.weight":
            assert h == sorted({0, pp - 1})
        elif s.name == "decoder.embed_positions.weight":
            assert h == [0]
        elif s.name.startswith("decoder.final_layer_norm"):
            assert h == [pp - 1]
        else:
            assert len(h) == 1 and h[0] == int(s.name.split(".")[2]) // (d.n_layers // pp)
    total = sum(layout.shard_bytes(d, 1, "bf16", pp, st) for st in range(pp))
    emb = layout.arena_layout(d, 1, 0)[0][0].nbytes
    assert total == layout.shard_bytes(d, 1) + (emb if pp > 1 else 0)
