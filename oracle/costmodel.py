"""Alpha-beta transfer cost model (oracle side; virtual-time durations).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

P:129: lower bound S/B per GPU (24/32 = 0.75 s), "inversely decrease" with #GPUs.
P:138: total latency alpha + beta*n per message; TP shards keep the tensor count T, so a
per-tensor transfer costs T*alpha + S_r/B while the flat per-rank arena costs
n_chunks*alpha_c + S_r/B.
"""
import math


def transfer_time(nbytes, n_messages, bandwidth, alpha):
    if bandwidth <= 0:
        raise ValueError("bandwidth must be positive")
    return n_messages * alpha + nbytes / bandwidth


def n_chunks(nbytes, chunk):
    return max(1, math.ceil(nbytes / chunk)) if nbytes else 0


def chunk_sizes(nbytes, chunk):
    n = n_chunks(nbytes, chunk)
    return [min(chunk, nbytes - i * chunk) for i in range(n)]


def paired_swap_times(nbytes, chunk, b_in, b_out, alpha):
    """Two-stage chunk pipeline (C3): D2H chunk i on the offload stream, then H2D chunk i on
    the load stream (full-duplex link).  Returns (offload_done, load_done) relative to
    submission; each chunk costs alpha + size/B on its stream."""
    d2h_done, t = [], 0.0
    for c in chunk_sizes(nbytes, chunk):
        t += alpha + c / b_out
        d2h_done.append(t)
    h = 0.0
    for i, c in enumerate(chunk_sizes(nbytes, chunk)):
        h = max(h, d2h_done[i]) + alpha + c / b_in
    return (d2h_done[-1] if d2h_done else 0.0), h


def scaling_efficiency(s_total, s_rep, t):
    """E(t) = T_in(1) / (t * T_in(t)) with equal per-rank bandwidth: S / (S + (t-1) S_rep)."""
    return s_total / (s_total + (t - 1) * s_rep)
