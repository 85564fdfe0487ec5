"""C4 — order-independent, position-sensitive 64-bit hash of a byte buffer (oracle side).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

Not in the paper; fixed by DESIGN.md (north star: "resident parameters ... bit-exact ...
(checksums)"):
    H(buf) = sum_j splitmix64(word_j XOR (j * 0x9E3779B97F4A7C15))  mod 2^64
over the little-endian 64-bit words of buf (len(buf) % 8 == 0).  Addition mod 2^64 is
commutative, so any reduction order gives the same bits.
"""
import numpy as np

from .weights import splitmix64, splitmix64_scalar, MASK64

K = np.uint64(0x9E3779B97F4A7C15)


def hash_words(words: np.ndarray, first_index: int = 0) -> int:
    j = np.arange(first_index, first_index + words.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        t = splitmix64(words.astype(np.uint64) ^ (j * K))
    # exact modular sum: split into 32-bit halves to avoid float/overflow surprises
    lo = int((t & np.uint64(0xFFFFFFFF)).sum(dtype=np.uint64))
    hi = int((t >> np.uint64(32)).sum(dtype=np.uint64))
    return (lo + (hi << 32)) & MASK64


def checksum(buf: np.ndarray, chunk_words: int = 1 << 24) -> int:
    b = np.ascontiguousarray(buf).view(np.uint8)
    if b.size % 8:
        raise ValueError("buffer length must be a multiple of 8 bytes")
    w = b.view(np.uint64)
    h = 0
    for s in range(0, w.size, chunk_words):
        h = (h + hash_words(w[s:s + chunk_words], s)) & MASK64
    return h


def checksum_scalar(buf: bytes) -> int:
    """Plain loop version for pins on tiny buffers."""
    assert len(buf) % 8 == 0
    h = 0
    for j in range(len(buf) // 8):
        word = int.from_bytes(buf[8 * j:8 * j + 8], "little")
        h = (h + splitmix64_scalar(word ^ ((j * 0x9E3779B97F4A7C15) & MASK64))) & MASK64
    return h


def checksum_parallel(buf: np.ndarray, threads: int = 0, chunk_words: int = 1 << 23) -> int:
    """Same H, chunks hashed on a thread pool (numpy releases the GIL in ufuncs)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    b = np.ascontiguousarray(buf).view(np.uint8)
    w = b.view(np.uint64)
    starts = list(range(0, w.size, chunk_words))
    n = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(n) as ex:
        parts = list(ex.map(lambda s: hash_words(w[s:s + chunk_words], s), starts))
    return sum(parts) & MASK64
