"""GEMM microbenchmark sweep (dev): per-layer GEMM shapes of OPT-13B / OPT-1.3B at TP1 x M, for
tuning knobs given by env vars. Each configuration runs in a fresh process (knobs are read once).

usage: python tools/gemm_tune.py [default|ext|grid|l2pf|smem|align|pair|split]"""
import json, os, subprocess, sys
MODELS = {"opt-13b": {"qkv": (15360, 5120), "out": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)},
          "opt-1.3b": {"qkv": (6144, 2048), "out": (2048, 2048), "fc1": (8192, 2048), "fc2": (2048, 8192)},
          "opt-125m": {"qkv": (2304, 768), "out": (768, 768), "fc1": (3072, 768), "fc2": (768, 3072)},
          # cfg4's per-rank shapes (OPT-30B at TP 8; QKV as one GEMM of its three 896-row segments)
          "opt-30b-tp8": {"qkv": (2688, 7168), "out": (7168, 896), "fc1": (3584, 7168), "fc2": (7168, 3584)}}
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ".")
    from paper_2306_13835_b200 import mpsw as M
    impl = int(sys.argv[2])
    for model in sys.argv[3].split(","):
        for Mt in [int(x) for x in os.environ.get("GT_M", "2,16,64,256").split(",")]:
            row = {"model": model, "M": Mt, "impl": impl,
                   "env": {k: v for k, v in os.environ.items() if k.startswith("MPSW_TC") or k.startswith("MPSW_DEV")}}
            tot = 0
            for name, (N, K) in MODELS[model].items():
                us = M.bench_gemm(Mt, N, K, impl=impl, reps=10)
                row[name] = round(us, 1)
                tot += us
            row["layer_us"] = round(tot, 1)
            row["GBps"] = round(sum(2 * N * K for N, K in MODELS[model].values()) / (tot * 1e3), 1)
            print(json.dumps(row), flush=True)
    sys.exit(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "default"
models = "opt-13b,opt-1.3b,opt-125m" if os.environ.get("MPSW_TC_DYN") or mode == "default" else "opt-13b"
configs = [("2", {})]
if mode == "ext":
    configs = [("2", {"MPSW_TC_EXT_MIN": v}) for v in ("16", "32", "64", "100000")]
elif mode == "l2pf":
    models = "opt-13b,opt-1.3b"
    configs = [("2", {"MPSW_TC_L2PF": v}) for v in ("0", "4", "8", "16", "32")]
elif mode == "smem":
    models = "opt-13b,opt-1.3b"
    configs = [("2", {"MPSW_TC_SMEM_KB": v}) for v in ("56", "72", "88", "104")]
elif mode == "align":
    models = "opt-13b,opt-1.3b,opt-125m"
    configs = [("2", {"MPSW_TC_ALIGN": v}) for v in ("0", "1")]
elif mode == "pair":
    models = "opt-13b,opt-1.3b,opt-125m"
    configs = [("2", {"MPSW_TC_PAIR": v}) for v in ("0", "1")] + [("2", {"MPSW_TC_PAIR": "1", "MPSW_TC_SMEM_KB": v})
                                                                 for v in ("88", "112")]
elif mode == "split":
    models = "opt-13b,opt-1.3b,opt-125m"
    configs = [("2", {"MPSW_TC_SPLIT": "1"}), ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "100000"}),
               ("2", {"MPSW_TC_SPLIT": "2"}), ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "64"}),
               ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "1"})]
elif mode == "large":
    models = "opt-13b,opt-1.3b"
    base = {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "1"}
    configs = [("2", dict(base))] + [("2", dict(base, MPSW_TC_L2PF=v)) for v in ("4", "8", "16")] + \
              [("2", dict(base, MPSW_TC_EXT_MIN="100000")), ("2", dict(base, MPSW_TC_CL_MIN="64")),
               ("2", dict(base, MPSW_TC_SMEM_KB="112"))]
elif mode == "rings":
    models = "opt-13b,opt-1.3b"
    configs = [("2", {"MPSW_TC_SPLIT": "1"}), ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_CL_MIN": "100000"}),
               ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "1"}), ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "2"}),
               ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "2", "MPSW_TC_STAGE_MIN": "64"}),
               ("2", {"MPSW_TC_SPLIT": "2", "MPSW_TC_VW": "1", "MPSW_TC_WPRE": "4"})]
elif mode == "knobs2":
    models = "opt-13b,opt-1.3b,opt-125m"
    configs = [("2", {})] + [("2", {"MPSW_TC_L2PF": v}) for v in ("2", "4")] + \
              [("2", {"MPSW_TC_EXT_MIN": v}) for v in ("32", "48", "128")] + \
              [("2", {"MPSW_TC_MINU": v}) for v in ("6", "12")] + [("2", {"MPSW_TC_CL_MIN": "128"})]
elif mode == "fixup":
    models = "opt-13b,opt-1.3b,opt-30b-tp8"
    configs = [("2", {}), ("2", {"MPSW_TC_FIX_TOK": "8"}), ("2", {"MPSW_TC_FIX_EARLY": "1"}),
               ("2", {"MPSW_TC_FIX_TOK": "8", "MPSW_TC_FIX_EARLY": "1"}), ("2", {"MPSW_DEV_NOOP_FIXUP": "1"})]
elif mode == "grid":
    models = "opt-13b,opt-1.3b"
    configs = [("2", {}), ("2", {"MPSW_TC_CPS": "1", "MPSW_TC_SMEM_KB": "200"}), ("1", {})]
for impl, env in configs:
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, __file__, "child", impl, models], env=e)
