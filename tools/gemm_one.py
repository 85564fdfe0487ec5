"""One GEMM shape through mpsw_bench_gemm (dev/profiling): python tools/gemm_one.py M N K [impl=2] [reps=5]"""
import sys
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M

m, n, k = (int(a) for a in sys.argv[1:4])
impl = int(sys.argv[4]) if len(sys.argv) > 4 else 2
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
us = M.bench_gemm(m, n, k, impl=impl, reps=reps)
print(f"M={m} N={n} K={k} impl={impl} us={us:.1f} GBps={2 * n * k / us / 1e3:.0f} TFLOPs={2 * m * n * k / us / 1e6:.1f}")
