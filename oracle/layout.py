"""C2 — TP partition of an OPT model and the per-rank flat arena layout (oracle side).

PAPER.md §5.1: "Each TP shard still contains the same number of tensors as the
original model albeit smaller" -> every rank holds all T = 16*L_m + 4 tensors.
The paper does not give OPT's TP layout (reading #12); we use the Megatron 1-D
layout that Colossal-AI implements:
  * column-parallel (rows of the [out, in] weight split): q/k/v/fc1 weights and biases;
  * row-parallel (columns split, stored as a contiguous [out, in/t] slice): out_proj, fc2
    weights; their biases are replicated (added once after the all-reduce);
  * vocab-parallel: rows of embed_tokens (lm_head is tied, HF:opt.py:444);
  * replicated: embed_positions, all LayerNorm gammas/betas.
P:107 keeps parameters pinned; DESIGN.md lays each rank's shard out as ONE contiguous blob:
tensors in HF `named_parameters()` order (decoder.embed_tokens, embed_positions,
final_layer_norm, then per layer k,v,q,out_proj,self_attn_layer_norm,fc1,fc2,
final_layer_norm), each starting at a 256-byte aligned offset, zero padding between.
"""
from dataclasses import dataclass
import numpy as np

from . import weights

ALIGN = 256
REPL, ROWS, COLS = 0, 1, 2          # split kinds (same numbering as mpsw_tensor_desc.split)


@dataclass(frozen=True)
class TensorSpec:
    tid: int
    name: str
    shape: tuple          # full (unsharded) shape, [out, in] or [n]
    split: int            # REPL / ROWS / COLS
    ln_gamma: bool


def canonical_tensors(d):
    """HF OPTForCausalLM.named_parameters() order (verified against transformers 5.5)."""
    h, ff, V, P = d.hidden, d.ffn, d.vocab, d.max_pos + 2
    specs = [("decoder.embed_tokens.weight", (V, h), ROWS, False),
             ("decoder.embed_positions.weight", (P, h), REPL, False),
             ("decoder.final_layer_norm.weight", (h,), REPL, True),
             ("decoder.final_layer_norm.bias", (h,), REPL, False)]
    for i in range(d.n_layers):
        p = f"decoder.layers.{i}."
        for proj in ("k_proj", "v_proj", "q_proj"):
            specs += [(p + f"self_attn.{proj}.weight", (h, h), ROWS, False),
                      (p + f"self_attn.{proj}.bias", (h,), ROWS, False)]
        specs += [(p + "self_attn.out_proj.weight", (h, h), COLS, False),
                  (p + "self_attn.out_proj.bias", (h,), REPL, False),
                  (p + "self_attn_layer_norm.weight", (h,), REPL, True),
                  (p + "self_attn_layer_norm.bias", (h,), REPL, False),
                  (p + "fc1.weight", (ff, h), ROWS, False),
                  (p + "fc1.bias", (ff,), ROWS, False),
                  (p + "fc2.weight", (h, ff), COLS, False),
                  (p + "fc2.bias", (h,), REPL, False),
                  (p + "final_layer_norm.weight", (h,), REPL, True),
                  (p + "final_layer_norm.bias", (h,), REPL, False)]
    return [TensorSpec(i, n, s, k, g) for i, (n, s, k, g) in enumerate(specs)]


def check_tp(d, tp: int):
    if tp < 1 or d.heads % tp or d.vocab % tp or d.ffn % tp or d.hidden % tp:
        raise ValueError(f"tp={tp} does not divide heads/vocab/ffn/hidden")


def shard_shape(spec: TensorSpec, tp: int):
    s = spec.shape
    if spec.split == REPL:
        return s
    if spec.split == ROWS:
        return (s[0] // tp,) + tuple(s[1:])
    return (s[0], s[1] // tp)


def shard_flat_indices(spec: TensorSpec, tp: int, rank: int) -> np.ndarray:
    """Flat indices (into the full tensor) of rank `rank`'s shard, in the shard's own
    row-major storage order."""
    s = spec.shape
    n = int(np.prod(s))
    if spec.split == REPL:
        return np.arange(n, dtype=np.int64)
    if spec.split == ROWS:
        per = n // tp
        return np.arange(rank * per, (rank + 1) * per, dtype=np.int64)
    rows, cols = s
    c = cols // tp
    return (np.arange(rows, dtype=np.int64)[:, None] * cols
            + np.arange(rank * c, (rank + 1) * c, dtype=np.int64)[None, :]).reshape(-1)


@dataclass(frozen=True)
class Placed:
    spec: TensorSpec
    shape: tuple          # shard shape
    offset: int           # byte offset in the rank's arena
    nbytes: int


def stage_holds(d, spec: TensorSpec, pp: int, stage: int) -> bool:
    """Pipeline split (reading #27; P:72 TP and PP dimensions): stage s holds layers
    [s*L/pp, (s+1)*L/pp); stage 0 also the embeddings; the last stage the final LayerNorm and
    (for pp > 1) a copy of embed_tokens for the tied lm_head."""
    name = spec.name
    if name.startswith("decoder.layers."):
        i = int(name.split(".")[2])
        per = d.n_layers // pp
        return stage * per <= i < (stage + 1) * per
    if name == "decoder.embed_tokens.weight":
        return stage == 0 or stage == pp - 1
    if name == "decoder.embed_positions.weight":
        return stage == 0
    return stage == pp - 1                       # final_layer_norm


def arena_layout(d, tp: int, rank: int, dtype: str = "bf16", pp: int = 1, stage: int = 0):
    """Returns (list[Placed], shard_bytes) of TP rank `rank` of pipeline stage `stage`.  Sizes
    do not depend on `rank` (every TP rank has the same shard shapes)."""
    check_tp(d, tp)
    if not 0 <= rank < tp:
        raise ValueError("rank out of range")
    if pp < 1 or d.n_layers % pp or not 0 <= stage < pp:
        raise ValueError("pp must divide n_layers and 0 <= stage < pp")
    es = 2 if dtype == "bf16" else 4
    off, out = 0, []
    for spec in canonical_tensors(d):
        if not stage_holds(d, spec, pp, stage):
            continue
        shp = shard_shape(spec, tp)
        nb = int(np.prod(shp)) * es
        out.append(Placed(spec, shp, off, nb))
        off = (off + nb + ALIGN - 1) // ALIGN * ALIGN
    return out, off


def shard_bytes(d, tp: int, dtype: str = "bf16", pp: int = 1, stage: int = 0) -> int:
    return arena_layout(d, tp, 0, dtype, pp, stage)[1]


def replicated_bytes(d, dtype: str = "bf16") -> int:
    """Bytes every rank holds in full (S_rep), aligned as placed."""
    es = 2 if dtype == "bf16" else 4
    return sum(int(np.prod(p.shape)) * es for p in arena_layout(d, 1, 0, dtype)[0]
               if p.spec.split == REPL)


def shard_image(d, tp: int, rank: int, model_seed: int, dtype: str = "bf16", pp: int = 1,
                stage: int = 0) -> np.ndarray:
    """The exact bytes of (stage, TP rank)'s arena (uint8 array of shard_bytes)."""
    placed, total = arena_layout(d, tp, rank, dtype, pp, stage)
    img = np.zeros(total, dtype=np.uint8)
    for p in placed:
        idx = shard_flat_indices(p.spec, tp, rank)
        vals = weights.tensor_values(model_seed, p.spec.tid, idx, p.spec.ln_gamma, dtype)
        img[p.offset:p.offset + p.nbytes] = np.ascontiguousarray(vals).view(np.uint8)
    return img


def shard_tensors(d, tp: int, rank: int, model_seed: int, dtype: str = "bf16"):
    """dict name -> float32 array (shard shape) of the values rank `rank` stores."""
    out = {}
    for p in arena_layout(d, tp, rank, dtype)[0]:
        idx = shard_flat_indices(p.spec, tp, rank)
        v = weights.fp32_values(model_seed, p.spec.tid, idx, p.spec.ln_gamma)
        if dtype == "bf16":
            v = weights.round_bf16(v)
        out[p.spec.name] = v.reshape(p.shape)
    return out


def full_tensors(d, model_seed: int, dtype: str = "bf16"):
    """dict name -> float32 array (full shape): the unsharded model (tp = 1)."""
    return shard_tensors(d, 1, 0, model_seed, dtype)


def element_at(d, tp: int, rank: int, model_seed: int, byte_offset: int, dtype: str = "bf16"):
    """Expected storage element covering `byte_offset` of rank's arena: returns the
    (uint16 or float32) element value, or None if the byte is padding (expected zero)."""
    es = 2 if dtype == "bf16" else 4
    for p in arena_layout(d, tp, rank, dtype)[0]:
        if p.offset <= byte_offset < p.offset + p.nbytes:
            k = (byte_offset - p.offset) // es
            idx = shard_flat_indices(p.spec, tp, rank)[k:k + 1]
            return weights.tensor_values(model_seed, p.spec.tid, idx, p.spec.ln_gamma, dtype)[0]
    return None


class LazyFull:
    """Read-only mapping name -> FULL (unsharded) tensor values, generated on demand by the C
    transcription of C0 (oracle/c/c0gen.c) and never cached, so an OPT-13B/30B forward can be
    computed layer by layer in O(layer) memory (test infrastructure for full-size parity)."""

    def __init__(self, d, model_seed: int, dtype: str = "bf16"):
        self.specs = {s.name: s for s in canonical_tensors(d)}
        self.seed = model_seed
        self.bf16 = dtype == "bf16"

    def __getitem__(self, name):
        from . import cgen
        s = self.specs[name]
        n = int(np.prod(s.shape))
        return cgen.values(self.seed, s.tid, 0, n, s.ln_gamma, self.bf16).reshape(s.shape)

    def keys(self):
        return self.specs.keys()
