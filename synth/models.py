"""OPT model-shape presets (input configuration, not method arithmetic).

Values are the public OPT configurations (HF `OPTConfig` defaults and the OPT paper's
Table 1): hidden size h, layers L_m, heads nh, ffn = 4h, vocab V = 50272, 2048
positions (+2 offset rows in `embed_positions`, HF:opt.py:53).  PAPER.md §5.1
names OPT-13B; the other sizes are the BASELINE.json configs.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class OptDims:
    n_layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int = 50272
    max_pos: int = 2048          # embed_positions has max_pos + 2 rows

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


OPT_PRESETS = {
    "opt-125m": OptDims(12, 768, 12, 3072),
    "opt-1.3b": OptDims(24, 2048, 32, 8192),
    "opt-13b": OptDims(40, 5120, 40, 20480),
    "opt-30b": OptDims(48, 7168, 56, 28672),
    # tiny shapes for oracle-speed parity tests (several tiles + ragged tails)
    "tiny": OptDims(2, 64, 4, 256, vocab=100, max_pos=16),
    "small": OptDims(3, 256, 8, 1024, vocab=1000, max_pos=64),
    "mid": OptDims(4, 512, 8, 2048, vocab=4096, max_pos=128),
}


def opt_dims(name: str) -> OptDims:
    return OPT_PRESETS[name]
