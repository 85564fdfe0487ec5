"""Per-phase timeline of the fused layers kernel from MPSW_FUSED_TRACE stamps (dev tool).
usage: MPSW_FUSED_TRACE=t.ndjson python tools/fwd_one.py opt-13b 1 2 0 3; python tools/fused_trace.py t.ndjson
For every phase P (7 per layer: qkv, attn, out, ln2, fc1, fc2, ln1'): when the last CTA passed
the wait for P-1 (start), when the first / last CTA arrived (done); all relative to the first
start, microseconds. Averages over layers > 0 per phase kind."""
import json
import sys

import numpy as np

names = ["qkv", "attn", "out", "ln2", "fc1", "fc2", "ln_next"]
for line in open(sys.argv[1]):
    r = json.loads(line)
    G, L = r["G"], r["L"]
    t = np.array(r["t"], dtype=np.float64).reshape(G, L * 7, 2)
    start = t[:, :, 0]
    arr = t[:, :, 1]
    t0 = start[start > 0].min()
    done = arr.max(axis=0)                      # barrier P complete
    first = arr.min(axis=0)
    prev = np.concatenate([[t0], done[:-1]])
    dur = (done - prev) / 1e3                   # phase P: barrier P-1 -> barrier P
    spread = (done - first) / 1e3
    print(f"M={r['M']} L={L} total {(done[-1] - t0) / 1e3:.1f} us, per layer {(done[-1] - t0) / 1e3 / L:.1f} us")
    for k in range(7):
        d = dur[7 + k::7] if L > 1 else dur[k::7]
        sp = spread[7 + k::7] if L > 1 else spread[k::7]
        print(f"  {names[k]:8s} {d.mean():7.2f} us (arrival spread {sp.mean():6.2f})")
