"""GEMM microbenchmark of given (N, K) shapes at M = 2 / 64 / 256 (dev; knobs from the env).
usage: python tools/gemm_shapes_ab.py N1xK1 N2xK2 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_13835_b200 import mpsw as M  # noqa: E402

for sh in sys.argv[1:]:
    N, K = (int(x) for x in sh.split("x"))
    for Mt in (2, 64, 256):
        us = M.bench_gemm(Mt, N, K, impl=2, reps=20)
        print(json.dumps({"N": N, "K": K, "M": Mt, "us": round(us, 2), "GBps": round(2 * N * K / (us * 1e3), 1),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("MPSW_TC")}}), flush=True)
