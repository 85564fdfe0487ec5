"""Copy-engine H2D cost by host-buffer kind (dev probe for the AUTO table): cudaHostAlloc vs an
mmap'd range registered with cudaHostRegister (the library's arenas: Portable | Mapped, with and
without transparent huge pages, and Portable only), device time of one cudaMemcpyAsync per size
from CUDA events on a private stream. Prints NDJSON.

usage: python tools/ce_reg_probe.py"""
import ctypes
import json
import mmap
import statistics
import time

from cuda.bindings import runtime as rt

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_HUGEPAGE = 14
MAX = 64 << 20


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert err == rt.cudaError_t.cudaSuccess, err
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def host_buffer(kind):
    if kind == "cudaHostAlloc":
        return ck(rt.cudaHostAlloc(MAX, rt.cudaHostAllocPortable))
    p = libc.mmap(None, MAX, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    if kind.endswith("thp"):
        libc.madvise(p, MAX, MADV_HUGEPAGE)
    flags = rt.cudaHostRegisterPortable | (rt.cudaHostRegisterMapped if "mapped" in kind else 0)
    ck(rt.cudaHostRegister(p, MAX, flags))
    return p


def main():
    ck(rt.cudaSetDevice(0))
    dev = ck(rt.cudaMalloc(MAX))
    st = ck(rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking))
    e0, e1 = ck(rt.cudaEventCreate()), ck(rt.cudaEventCreate())
    for kind in ("cudaHostAlloc", "register_mapped_thp", "register_mapped", "register_portable_thp"):
        h = host_buffer(kind)
        ctypes.memset(h, 1, MAX)
        for sz in (1 << 20, 4 << 20, 16 << 20, 64 << 20):
            ts, hs = [], []
            for _ in range(9):
                ck(rt.cudaEventRecord(e0, st))
                t0 = time.perf_counter()
                ck(rt.cudaMemcpyAsync(dev, h, sz, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st))
                hs.append((time.perf_counter() - t0) * 1e3)
                ck(rt.cudaEventRecord(e1, st))
                ck(rt.cudaEventSynchronize(e1))
                ts.append(ck(rt.cudaEventElapsedTime(e0, e1)))
            med = statistics.median(ts[2:])
            print(json.dumps({"kind": kind, "bytes": sz, "ms_median": med, "ms_min": min(ts[2:]),
                              "host_submit_ms_median": statistics.median(hs[2:]),
                              "GBps": sz / (med / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
