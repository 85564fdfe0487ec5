"""Pins for oracle/checksum.py (C4): scalar reference on zero buffers, bit-flip sensitivity,
order independence, chunking invariance."""
import numpy as np

from oracle import checksum as C
from oracle.weights import splitmix64_scalar, MASK64


def test_zero_buffer_reference_value():
    n = 257
    ref = 0
    for j in range(n):
        ref = (ref + splitmix64_scalar((j * 0x9E3779B97F4A7C15) & MASK64)) & MASK64
    assert C.checksum(np.zeros(8 * n, np.uint8)) == ref
    assert C.checksum_scalar(bytes(8 * n)) == ref


def test_vector_matches_scalar_random():
    b = np.random.default_rng(2).integers(0, 256, 8 * 1000, dtype=np.uint8)
    assert C.checksum(b) == C.checksum_scalar(b.tobytes())


def test_single_bit_flip_changes_hash():
    rng = np.random.default_rng(3)
    b = rng.integers(0, 256, 4096, dtype=np.uint8)
    h = C.checksum(b)
    for _ in range(200):
        c = b.copy()
        i = rng.integers(0, c.size)
        c[i] ^= np.uint8(1 << rng.integers(0, 8))
        assert C.checksum(c) != h


def test_position_sensitive_swap_words():
    b = np.arange(64, dtype=np.uint64)
    c = b.copy(); c[[3, 9]] = c[[9, 3]]
    assert C.checksum(b.view(np.uint8)) != C.checksum(c.view(np.uint8))


def test_chunking_and_parallel_invariance():
    b = np.random.default_rng(4).integers(0, 256, 8 * 100003, dtype=np.uint8)
    h = C.checksum(b)
    assert C.checksum(b, chunk_words=777) == h
    assert C.checksum_parallel(b, threads=3, chunk_words=1001) == h
    # sum of per-range hashes with offsets == whole hash (commutativity of the sum)
    w = b.view(np.uint64)
    parts = [C.hash_words(w[s:s + 5000], s) for s in range(0, w.size, 5000)][::-1]
    assert sum(parts) & MASK64 == h
