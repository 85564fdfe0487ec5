"""C0 — synthetic OPT weights from a counter-based generator (oracle side).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

Not in the paper (P:127 uses trained OPT-13B; there are no weights here, so random-init
weights "of that architecture" are generated).  Spec:

    x = splitmix64(model_seed ^ (tensor_id << 40) ^ flat_index)          (uint64, wraps)
    u = x >> 40                                                          (24-bit integer)
    w = (u - 2^23) * 2^-28          exact in fp32, uniform on [-2^-5, 2^-5)
    value = 1 + w for LayerNorm gammas, w otherwise (computed exactly, then rounded
            RNE to fp32; bf16 mode then rounds that fp32 RNE to bf16)

`flat_index` indexes the FULL (unsharded) tensor in row-major [out, in] order, so
TP shards are exact slices.  `tensor_id` is the tensor's position in the canonical
order of `oracle.layout.canonical_tensors`.

The product library implements the same spec independently in C++ (csrc/synth_fill.cpp);
the two share no code.
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
MASK64 = (1 << 64) - 1


def splitmix64_scalar(z: int) -> int:
    """Textbook SplitMix64 output function (Steele, Lea, Flood 2014), pure Python ints."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """Vectorised SplitMix64 on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def raw_w(model_seed: int, tensor_id: int, flat_index: np.ndarray) -> np.ndarray:
    """w as float64 (exact) for the given flat indices."""
    key = np.uint64((model_seed ^ (tensor_id << 40)) & MASK64)
    x = splitmix64(np.asarray(flat_index, dtype=np.uint64) ^ key)
    u = (x >> np.uint64(40)).astype(np.int64)
    return (u - (1 << 23)).astype(np.float64) * 2.0 ** -28


def fp32_values(model_seed: int, tensor_id: int, flat_index, is_ln_gamma: bool) -> np.ndarray:
    w = raw_w(model_seed, tensor_id, flat_index)
    base = 1.0 + w if is_ln_gamma else w           # exact in float64
    return base.astype(np.float32)                 # RNE to fp32


def bf16_bits_from_fp32(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))
    return (b >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_fp32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest-even bf16 value, returned as fp32 (used by the bf16-emulating forward)."""
    return bf16_bits_to_fp32(bf16_bits_from_fp32(np.asarray(x, dtype=np.float32)))


def tensor_values(model_seed: int, tensor_id: int, flat_index, is_ln_gamma: bool, dtype: str):
    """Element values of one tensor at `flat_index` in storage dtype: 'bf16' -> uint16 bits,
    'fp32' -> float32."""
    v = fp32_values(model_seed, tensor_id, flat_index, is_ln_gamma)
    if dtype == "bf16":
        return bf16_bits_from_fp32(v)
    if dtype == "fp32":
        return v
    raise ValueError(dtype)
