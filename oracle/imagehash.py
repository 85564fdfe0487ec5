"""C4 hash of a C0 shard image computed without materialising the image (oracle side).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

The expected checksum of a full-size resident shard (north star: "resident parameters after any
swap sequence must be bit-exact with the oracle's (checksums)") is
    H(shard_image(d, tp, rank, seed))                    (oracle/checksum.py, oracle/layout.py)
For OPT-13B/30B that image is 3-26 GB, so this module streams it: each tensor's shard values
come from the oracle's C transcription of C0 (oracle/c/c0gen.c) in the layout's order, and
since H is a sum of per-word terms indexed by the word's position j,
    H(image) = sum over placed tensors of hash_words(tensor bytes, offset/8)
             + sum over zero padding words j of splitmix64(0 ^ j*K)
(the padding is 0 bytes at every BASELINE config but is handled generally). Pinned against
checksum(shard_image(...)) on small shapes (tests/test_oracle_imagehash.py).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import cgen, checksum, layout
from .weights import MASK64

_CHUNK_WORDS = 1 << 22


def _tensor_words(spec, tp, rank, seed, bf16):
    """Rank `rank`'s stored values of one tensor, as little-endian bytes (uint8)."""
    n = int(np.prod(spec.shape))
    if spec.split == layout.REPL:
        v = cgen.values(seed, spec.tid, 0, n, spec.ln_gamma, bf16)
    elif spec.split == layout.ROWS:
        per = n // tp
        v = cgen.values(seed, spec.tid, rank * per, per, spec.ln_gamma, bf16)
    else:
        rows, cols = spec.shape
        c = cols // tp
        v = np.ascontiguousarray(cgen.values(seed, spec.tid, 0, n, spec.ln_gamma, bf16)
                                 .reshape(rows, cols)[:, rank * c:(rank + 1) * c]).reshape(-1)
    if bf16:
        return (v.view(np.uint32) >> 16).astype(np.uint16).view(np.uint8)
    return v.view(np.uint8)


def _hash_at(buf_u8, first_word, threads):
    w = buf_u8.view(np.uint64)
    starts = range(0, w.size, _CHUNK_WORDS)
    with ThreadPoolExecutor(threads) as ex:
        parts = ex.map(lambda s: checksum.hash_words(w[s:s + _CHUNK_WORDS], first_word + s), starts)
        return sum(parts) & MASK64


def shard_image_hash(d, tp, rank, seed, dtype="bf16", pp=1, stage=0, threads=0):
    """H(shard_image(d, tp, rank, seed, dtype, pp, stage)) streamed tensor by tensor."""
    threads = threads or len(os.sched_getaffinity(0))
    placed, total = layout.arena_layout(d, tp, rank, dtype, pp, stage)
    bf16 = dtype == "bf16"
    h, pos = 0, 0
    for p in placed:
        if p.offset > pos:                                   # zero padding words [pos, offset)
            h = (h + _hash_at(np.zeros(p.offset - pos, np.uint8), pos // 8, threads)) & MASK64
        b = _tensor_words(p.spec, tp, rank, seed, bf16)
        pad = (-b.size) % 8                                  # tail of the last word: zero padding
        if pad:
            b = np.concatenate([b, np.zeros(pad, np.uint8)])
        h = (h + _hash_at(b, p.offset // 8, threads)) & MASK64
        pos = p.offset + b.size
    if total > pos:
        h = (h + _hash_at(np.zeros(total - pos, np.uint8), pos // 8, threads)) & MASK64
    return h
