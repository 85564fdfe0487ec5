"""Per-CTA phase timeline of one tcgen05 GEMM launch (dev): MPSW_TC_TRACE stamps (%globaltimer)
of a launch that follows an identical launch back to back (PDL), summarised as percentiles
relative to the earliest CTA start.

usage: python tools/tc_trace.py run OUT.ndjson   (GPU: OPT-13B / OPT-1.3B layer shapes, M=2/256)
       python tools/tc_trace.py show OUT.ndjson"""
import json
import os
import sys

import numpy as np

PH = ["start", "prologue", "pdl_wait", "first_stage", "last_mma", "acc_ready", "drained", "done"]
SHAPES = [(15360, 5120), (5120, 5120), (20480, 5120), (5120, 20480), (6144, 2048), (2048, 2048), (8192, 2048),
          (2048, 8192)]

if sys.argv[1] == "run":
    sys.path.insert(0, ".")
    os.environ["MPSW_TC_TRACE"] = sys.argv[2]
    from paper_2306_13835_b200 import mpsw as M
    for m in (2, 256):
        for n, k in SHAPES:
            M.bench_gemm(m, n, k, impl=2, reps=5)
    sys.exit(0)

for line in open(sys.argv[2]):
    o = json.loads(line)
    t = np.array(o["t"], dtype=np.int64).reshape(o["G"], 8)
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    span = r[:, 7].max()
    mb = 2 * o["N"] * o["K"] / 1e6
    print(f"M={o['M']:3d} N={o['N']:5d} K={o['K']:5d} G={o['G']} CTAs={live.sum()} span={span:6.1f}us "
          f"({mb:.0f} MB -> {mb / span:.2f} TB/s)")
    for i, name in enumerate(PH):
        col = r[:, i]
        col = col[t[:, i] > 0]
        if len(col):
            print(f"   {name:12s} min {col.min():6.1f}  p50 {np.median(col):6.1f}  max {col.max():6.1f}")
