"""Element-wise comparison helpers for the bf16 / fp32 parity tests (test infrastructure).

bf16 values are compared in units in the last place (ulp) of bf16: the distance between two
bf16 numbers is the number of representable bf16 values between them (sign-magnitude mapped
onto a monotone integer line), so 1 ulp = one rounding decision taken the other way."""
import numpy as np


def bf16_bits_of_f32(x):
    """bf16 bit patterns of float32 values that are exactly bf16 (the oracle's rounded values)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    assert not np.any(b & 0xFFFF), "value is not a bf16 number"
    return (b >> 16).astype(np.uint16)


def bf16_to_f32(bits):
    return (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32)


def _ordered(bits):
    b = np.asarray(bits, np.int64)
    return np.where(b & 0x8000, -(b & 0x7FFF), b)


def ulp_stats(gpu_bits, ref_bits):
    """(fraction of elements that differ, max ulp distance) between two bf16 bit arrays."""
    d = np.abs(_ordered(gpu_bits) - _ordered(ref_bits))
    return float(np.mean(d > 0)), int(d.max(initial=0))


def f32_stats(y, ref):
    """(max |y - ref| / max |ref|, rel-L2) for fp32 / fp64 arrays."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    den = float(np.abs(ref).max()) or 1.0
    return float(np.abs(y - ref).max() / den), float(np.linalg.norm(y - ref) / (np.linalg.norm(ref) or 1.0))


def logits_stats(y, em, ex):
    """Logits of one request vs the bf16-emulating and the exact oracle: rel-L2 to each, and the
    element-wise max |y - ref| / max |ref| to each."""
    e1, r1 = f32_stats(y, em)
    e2, r2 = f32_stats(y, ex)
    return {"rel_l2_em": r1, "rel_l2_ex": r2, "maxabs_em": e1, "maxabs_ex": e2}


BF16_LOGITS_TOL = 1e-2     # north star: bf16 outputs within 1e-2 relative
FP32_LOGITS_TOL = 1e-5     # north star: fp32 outputs within 1e-5 relative


def assert_logits(y, em, ex=None, tol=BF16_LOGITS_TOL, tag=None):
    """End-to-end logits of one request vs the oracle (north-star bars): rel-L2 < tol AND every
    element |y - ref| <= tol * max|ref|, against the emulating oracle `em` (or the exact one when
    that is the only reference) and, when given, the fp64-exact oracle `ex`; argmax equal whenever
    the reference's top-2 gap exceeds 2 * tol * max|ref| (SURVEY §8(c) C5 metric). Appends one
    NDJSON record to $MPSW_PARITY_LOG when set. Returns the record."""
    import json
    import os
    y = np.asarray(y, np.float64)
    rec = {"tag": tag, "tol": tol}
    for name, ref in (("em", em), ("ex", ex)):
        if ref is None:
            continue
        ref = np.asarray(ref, np.float64)
        mx = float(np.abs(ref).max())
        rec[f"rel_l2_{name}"] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
        rec[f"maxabs_{name}"] = float(np.abs(y - ref).max() / mx)
        top2 = np.sort(ref)[-2:]
        rec[f"argmax_checked_{name}"] = bool(top2[1] - top2[0] > 2 * tol * mx)
        rec[f"argmax_equal_{name}"] = int(np.argmax(y)) == int(np.argmax(ref))
    log = os.environ.get("MPSW_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(rec) + "\n")
    for name in ("em", "ex"):
        if f"rel_l2_{name}" in rec:
            assert rec[f"rel_l2_{name}"] < tol, rec
            assert rec[f"maxabs_{name}"] <= tol, rec
            assert rec[f"argmax_equal_{name}"] or not rec[f"argmax_checked_{name}"], rec
    return rec
