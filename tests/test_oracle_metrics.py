"""Pins for oracle/metrics.py (C7) and synth traces (C6): SPEC examples, Gamma statistics."""
import json
import os
import numpy as np
import pytest

from oracle import metrics
from synth import traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_percentile_examples():
    for c in json.load(open(os.path.join(GOLD, "spec_examples.json")))["percentiles"]:
        s = metrics.summary(c["values"])
        assert s["mean"] == pytest.approx(c["mean"]) and s["p50"] == c["p50"]
    with pytest.raises(ValueError):
        metrics.summary([])
    assert metrics.nearest_rank(list(range(1, 101)), 99) == 99
    assert metrics.nearest_rank(list(range(1, 101)), 100) == 100


def test_swap_latency_window():
    assert metrics.swap_latency(1.0, 1.5, 1.75) == 0.75
    assert metrics.swap_latency(1.0, 2.0, 1.25) == 1.0         # offload later -> window ends there


@pytest.mark.parametrize("lam,cv", [(1, 0.25), (1, 1), (1, 4), (10, 0.25), (10, 1), (10, 4)])
def test_gamma_statistics(lam, cv):                            # S:344, S:514 criterion 10
    g = traces.gamma_gaps(0, 0, lam, cv, 10**6)
    assert abs(g.mean() * lam - 1) < 0.02
    assert abs(g.std() / g.mean() / cv - 1) < 0.02


def test_gamma_cv1_is_exponential():
    scipy = pytest.importorskip("scipy.stats")
    g = traces.gamma_gaps(1, 0, 2.0, 1.0, 200000)
    assert scipy.kstest(g, "expon", args=(0, 0.5)).pvalue > 1e-3


def test_trace_isolation_and_determinism():
    a = traces.gamma_trace([10, 1, 1], 4.0, 5.0, 3, 8, 100)
    b = traces.gamma_trace([10, 5, 1], 4.0, 5.0, 3, 8, 100)
    c = traces.gamma_trace([10, 1, 1], 4.0, 5.0, 3, 8, 100)
    ta = [(r.t_arr, r.model) for r in a if r.model == 0 and not r.warmup]
    tb = [(r.t_arr, r.model) for r in b if r.model == 0 and not r.warmup]
    assert ta == tb
    assert [(r.t_arr, r.model, r.tokens.tolist()) for r in a] == [(r.t_arr, r.model, r.tokens.tolist()) for r in c]
    assert sum(r.warmup for r in a) == 3
    ts = [r.t_arr for r in a]
    assert ts == sorted(ts)


def test_zipf():
    assert traces.zipf_rates(6) == pytest.approx([10, 5, 10 / 3, 2.5, 2, 10 / 6])
