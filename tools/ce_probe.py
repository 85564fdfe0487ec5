"""Copy-engine bandwidth probe (pinned H2D / D2H / bidirectional) on every visible GPU.

Box discovery only. Not part of the product path.
"""
import time, torch, os

def probe(dev, nbytes, direction, reps=5):
    torch.cuda.set_device(dev)
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) if direction == "bidir" else None
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev) if direction == "bidir" else None
    s1 = torch.cuda.Stream(dev); s2 = torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        if direction == "h2d":
            with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        elif direction == "d2h":
            with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
        else:
            with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(dev)
        best = min(best, time.perf_counter() - t0)
    mult = 2 if direction == "bidir" else 1
    return nbytes * mult / best / 1e9

n = torch.cuda.device_count()
print("gpus", n)
for dev in range(n):
    for sz in [1 << 20, 16 << 20, 256 << 20, 1 << 30, 4 << 30]:
        for dr in ["h2d", "d2h", "bidir"]:
            print(f"dev{dev} size={sz>>20}MiB {dr} {probe(dev, sz, dr):.2f} GB/s", flush=True)
