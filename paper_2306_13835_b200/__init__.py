"""paper_2306_13835_b200 — B200-native model-parallel swapping (Computron, arXiv 2306.13835).

The product is the C-ABI library `libmpsw.so` (include/mpsw.h; sources in csrc/). This package
only builds it (`build.py`) and exposes a thin ctypes binding (`mpsw.py`).
"""
from . import mpsw  # noqa: F401
