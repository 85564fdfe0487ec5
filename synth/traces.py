"""Request traces and token ids.

* Gamma arrivals: per model i, i.i.d. gaps ~ Gamma(k = 1/CV^2, theta = CV^2/lambda_i)
  ("random independent Gamma arrival process"; parameterisation S:339,
  DESIGN.md reading #17).  Per-model sub-seeds `[seed, i]` so model i's stream does not
  depend on other models' rates.  Arrivals beyond `duration` are dropped.
* Warm-up: `warmup_per_model` sequential requests per model before t = 0.
* Alternating / round-robin blocking drivers.
* Zipf rates lambda_i = lambda_max * i^-s (north star; reading #18).
* Tokens: uniform in [0, V) (reading #10), one int32 vector of length L per request.
"""
from dataclasses import dataclass, field
import numpy as np


@dataclass
class Request:
    rid: int
    model: int
    t_arr: float
    tokens: np.ndarray = field(repr=False)
    warmup: bool = False


def request_tokens(seed: int, model: int, index: int, length: int, vocab: int) -> np.ndarray:
    rng = np.random.default_rng([seed, 7919, model, index])
    return rng.integers(0, vocab, size=length, dtype=np.int64).astype(np.int32)


def zipf_rates(n: int, lam_max: float = 10.0, s: float = 1.0):
    return [lam_max * (i + 1) ** (-s) for i in range(n)]


def gamma_gaps(seed: int, model: int, rate: float, cv: float, n: int) -> np.ndarray:
    if rate <= 0 or cv <= 0:
        raise ValueError("rate and cv must be positive")
    rng = np.random.default_rng([seed, model])
    return rng.gamma(shape=1.0 / (cv * cv), scale=cv * cv / rate, size=n)


def gamma_trace(rates, cv: float, duration: float, seed: int, token_len: int, vocab: int,
                warmup_per_model: int = 1, warmup_spacing: float = 0.0):
    """Merged, time-sorted open-loop trace.  Warm-up requests get negative times
    (sequential, model order) and `warmup=True`."""
    reqs = []
    for i, lam in enumerate(rates):
        # draw enough gaps to cover the window (expected duration*lam, generous margin)
        n = int(duration * lam * 4 + 64)
        while True:
            gaps = gamma_gaps(seed, i, lam, cv, n)
            t = np.cumsum(gaps)
            if t[-1] > duration:
                break
            n *= 2
        for j, tj in enumerate(t[t <= duration]):
            reqs.append((float(tj), i, j))
    reqs.sort(key=lambda x: (x[0], x[1]))
    out = []
    rid = 0
    nw = warmup_per_model * len(rates)
    for w in range(nw):
        m = w % len(rates)
        out.append(Request(rid, m, -(nw - w) * warmup_spacing if warmup_spacing else -1.0 + w * 1e-9,
                           request_tokens(seed, m, 10**9 + w // len(rates), token_len, vocab), True))
        rid += 1
    for (tj, i, j) in reqs:
        out.append(Request(rid, i, tj, request_tokens(seed, i, j, token_len, vocab)))
        rid += 1
    return out


def alternating_blocking(n_requests: int, seed: int, token_len: int, vocab: int, models=(0, 1)):
    """A, B, A, B, ...: each request is issued after the previous completes."""
    return round_robin_blocking(n_requests, seed, token_len, vocab, models)


def round_robin_blocking(n_requests: int, seed: int, token_len: int, vocab: int, models=(0, 1, 2)):
    out = []
    for r in range(n_requests):
        m = models[r % len(models)]
        out.append(Request(r, m, float("nan"), request_tokens(seed, m, r, token_len, vocab)))
    return out
