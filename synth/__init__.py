"""Seeded synthetic INPUT generators shared by the oracle and the CUDA path.

This package holds no arithmetic of the method (no swap, scheduler, checksum,
layout or forward logic): only model-shape presets (HF OPT configs), request
traces (Gamma arrivals, Zipf rates, alternating blocking sequences) and token
ids.  Model WEIGHTS are not generated here: the oracle (numpy, `oracle/weights.py`)
and the product library (C++, `csrc/synth_fill.cpp`) each implement the same
counter-based generator spec.
"""
from .models import OPT_PRESETS, OptDims, opt_dims
from .traces import (Request, gamma_trace, alternating_blocking, round_robin_blocking,
                     zipf_rates, request_tokens)

__all__ = ["OPT_PRESETS", "OptDims", "opt_dims", "Request", "gamma_trace",
           "alternating_blocking", "round_robin_blocking", "zipf_rates", "request_tokens"]
