"""C7 — metrics (oracle side).

TEST INFRASTRUCTURE (oracle side; see oracle/__init__.py), not product code.

* Swap latency window: "we measure from when the offload entry is submitted to
  when both offload and load entries are completed" = max(off_done, load_done) - off_submit.
* Swap-in latency: max over ranks of H2D completion - submission (north star metric).
* Nearest-rank percentiles: p-th percentile of n sorted values is the
  value at rank ceil(p/100 * n) (1-based).
"""
import math


def swap_latency(off_submit, off_done, load_done):
    return max(off_done, load_done) - off_submit


def swap_in_latency(submit, done_per_rank):
    return max(done_per_rank) - submit


def nearest_rank(values, p):
    if not values:
        raise ValueError("empty measured set")
    v = sorted(values)
    k = max(1, math.ceil(p / 100.0 * len(v)))
    return v[k - 1]


def summary(values):
    if not values:
        raise ValueError("empty measured set")
    return {"count": len(values), "mean": sum(values) / len(values),
            "p50": nearest_rank(values, 50), "p90": nearest_rank(values, 90),
            "p99": nearest_rank(values, 99), "max": max(values)}
