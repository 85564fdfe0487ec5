"""Writes tests/golden/c0_shard_hashes.json: the C4 hash of every C0 shard image the full-size
tests and bench.py verify against, computed by the ORACLE only (oracle/imagehash.py: the C
transcription of C0 + the numpy C4 hash, streamed tensor by tensor). Never touches the CUDA path.

usage: python tools/gen_golden_hashes.py [--only KEY_SUBSTRING]
Keys: "<model>/tp<t>/r<rank>/seed<seed>/bf16". Existing keys are kept (incremental)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import opt_dims  # noqa: E402
from oracle import imagehash  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c0_shard_hashes.json")

# (model, tp, seeds): full-size swap test (seed 9), bench cfg3 models (1000 + i) at every t of the
# sweep, the cfg4 slice (OPT-30B TP8, seeds 3000 + i)
JOBS = [("opt-1.3b", 2, [2001]), ("opt-13b", 1, [9, 1000, 1001, 1002]), ("opt-30b", 8, [3000, 3001]),
        ("opt-13b", 2, [1000, 1001, 1002]), ("opt-13b", 4, [1000, 1001, 1002]), ("opt-13b", 8, [1000, 1001, 1002])]


def key(model, tp, r, seed):
    return f"{model}/tp{tp}/r{r}/seed{seed}/bf16"


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else ""
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out.setdefault("_doc", "C4 hashes of C0 shard images (tools/gen_golden_hashes.py; oracle only)")
    for model, tp, seeds in JOBS:
        d = opt_dims(model)
        for seed in seeds:
            for r in range(tp):
                k = key(model, tp, r, seed)
                if k in out or only not in k:
                    continue
                t0 = time.time()
                out[k] = hex(imagehash.shard_image_hash(d, tp, r, seed))
                print(k, out[k], f"{time.time() - t0:.1f}s", flush=True)
                tmp = OUT + ".tmp"
                json.dump(out, open(tmp, "w"), indent=1, sort_keys=True)
                os.replace(tmp, OUT)


if __name__ == "__main__":
    main()
