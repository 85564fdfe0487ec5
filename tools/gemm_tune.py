"""GEMM microbenchmark sweep (dev): OPT-13B TP1 shapes x M, for tuning knobs given by env vars.
Each configuration runs in a fresh process (the knobs are read once)."""
import json, os, subprocess, sys
SHAPES = {"qkv": (15360, 5120), "out": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)}
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ".")
    from paper_2306_13835_b200 import mpsw as M
    impl = int(sys.argv[2])
    for Mt in (2, 16, 64, 256):
        row = {"M": Mt, "impl": impl, "env": {k: v for k, v in os.environ.items() if k.startswith("MPSW_TC")}}
        tot = 0
        for name, (N, K) in SHAPES.items():
            us = M.bench_gemm(Mt, N, K, impl=impl, reps=10)
            row[name] = round(us, 1)
            tot += us
        row["layer_us"] = round(tot, 1)
        row["GBps"] = round(sum(2 * N * K for N, K in SHAPES.values()) / (tot * 1e3), 1)
        print(json.dumps(row), flush=True)
    sys.exit(0)
configs = [("2", {})]
if len(sys.argv) > 1 and sys.argv[1] == "ext":
    configs = [("2", {"MPSW_TC_EXT_MIN": v}) for v in ("16", "32", "64", "100000")]
for impl, env in configs:
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, __file__, "child", impl], env=e)
