"""Reference point (dev): cuBLAS bf16 (torch.matmul) on the forward's GEMM shapes, y[M,N] = x[M,K] W[N,K]^T,
weights rotated over enough copies that every launch streams them from HBM. Not on any product path.
usage: python tools/cublas_ref.py [model=opt-13b]"""
import json
import sys

import torch

SH = {"opt-13b": {"qkv": (15360, 5120), "out": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)},
      "opt-1.3b": {"qkv": (6144, 2048), "out": (2048, 2048), "fc1": (8192, 2048), "fc2": (2048, 8192)},
      "opt-30b-tp8": {"qkv": (2688, 7168), "out": (7168, 896), "fc1": (3584, 7168), "fc2": (7168, 3584)}}
model = sys.argv[1] if len(sys.argv) > 1 else "opt-13b"
dev = "cuda"
for M in (2, 16, 64, 128, 256):
    row = {"model": model, "M": M, "impl": "cublas(torch.matmul)"}
    tot = 0.0
    for name, (N, K) in SH[model].items():
        copies = max(2, int(400e6 // (N * K * 2)) + 1)
        Ws = [torch.randn(N, K, device=dev, dtype=torch.bfloat16) for _ in range(copies)]
        x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        for i in range(5):
            y = x @ Ws[i % copies].t()
        torch.cuda.synchronize()
        reps = 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            y = x @ Ws[i % copies].t()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / reps
        row[name] = round(us, 1)
        tot += us
        del Ws
    row["layer_us"] = round(tot, 1)
    print(json.dumps(row), flush=True)
