"""Does splitting an H2D transfer over 2-4 concurrent copy streams beat one stream? (dev probe)"""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=0)
for ns in (1, 2, 3, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    best = 0
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(ss):
            a, b = n * i // ns, n * (i + 1) // ns
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t) / 1e9)
    # interleaved chunks of 64 MiB across streams
    best2 = 0
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        c = 64 << 20
        for i in range(n // c):
            with torch.cuda.stream(ss[i % ns]):
                d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
        torch.cuda.synchronize()
        best2 = max(best2, n / (time.perf_counter() - t) / 1e9)
    print(f"streams={ns} split {best:.2f} GB/s  interleaved64M {best2:.2f} GB/s", flush=True)
