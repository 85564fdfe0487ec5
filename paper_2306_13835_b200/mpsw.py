"""Thin ctypes binding of libmpsw.so (include/mpsw.h). Argument marshalling only: every step of
the hot path (swaps, scheduling, the TP forward, checksums) runs inside the C++/CUDA library.
Fails loudly if the library is missing — there is no CPU fallback.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpsw.so")

OK, EINVAL, ENOMEM, EBUSY, ENOENT, EAGAIN, ECUDA, ENCCL, EINVARIANT, ETIMEDOUT = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9
STATUS_NAMES = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "EBUSY", -4: "ENOENT", -5: "EAGAIN", -6: "ECUDA",
                -7: "ENCCL", -8: "EINVARIANT", -9: "ETIMEDOUT"}
BF16, FP32 = 0, 1
SWAP_AUTO, SWAP_COPY_ENGINE, SWAP_ZERO_COPY, SWAP_HYBRID = 0, 1, 2, 3
EVICTED, LOADING, RESIDENT, OFFLOADING = 0, 1, 2, 3
TAP_X, TAP_A, TAP_QKV, TAP_O, TAP_R, TAP_XM, TAP_F = 0, 1, 2, 3, 4, 5, 6
NOOP_TICKET = (1 << 64) - 1


class MpswError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class OptDims(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("heads", C.c_int), ("ffn", C.c_int),
                ("vocab", C.c_int), ("max_pos", C.c_int)]


class Config(C.Structure):
    _fields_ = [("n_gpus", C.c_int), ("device_ids", C.POINTER(C.c_int)), ("tp", C.c_int),
                ("param_budget_bytes_per_gpu", C.c_uint64), ("workspace_bytes_per_gpu", C.c_uint64),
                ("max_batch", C.c_int), ("max_tokens", C.c_int), ("dtype", C.c_int),
                ("max_inflight_batches", C.c_int), ("swap_mode", C.c_int), ("chunk_bytes", C.c_uint64),
                ("writeback", C.c_int), ("trace", C.c_int), ("zc_ctas", C.c_int),
                ("world_size", C.c_int), ("world_rank", C.c_int), ("shm_name", C.c_char_p),
                ("gemm_impl", C.c_int), ("pp", C.c_int), ("helper_device_ids", C.POINTER(C.c_int)),
                ("n_helpers", C.c_int), ("max_dims", OptDims), ("prefetch", C.c_int), ("pp_broadcast", C.c_int),
                ("victim_policy", C.c_int), ("debug_checks", C.c_int)]


class TensorDesc(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("offset", C.c_uint64), ("bytes", C.c_uint64), ("rows", C.c_int),
                ("cols", C.c_int), ("split", C.c_int), ("tensor_id", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("swaps_in", C.c_uint64), ("swaps_out", C.c_uint64), ("batches", C.c_uint64),
                ("requests", C.c_uint64), ("rejected", C.c_uint64), ("k_slots", C.c_int),
                ("shard_bytes", C.c_uint64), ("fwd_gpu_us_sum", C.c_uint64), ("fwd_gpu_n", C.c_uint64),
                ("region_bytes", C.c_uint64), ("prefetches", C.c_uint64), ("numa_requested", C.c_uint64),
                ("numa_verified", C.c_uint64)]


_P = C.c_void_p
_SIGS = {
    "mpsw_init": [C.POINTER(Config), C.POINTER(_P)],
    "mpsw_shutdown": [_P],
    "mpsw_shard_layout": [C.POINTER(OptDims), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(TensorDesc),
                          C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_uint64)],
    "mpsw_register_model": [_P, C.POINTER(OptDims), C.c_int, C.POINTER(_P), C.POINTER(C.c_uint64),
                            C.POINTER(C.c_int)],
    "mpsw_model_arena": [_P, C.c_int, C.c_int, C.POINTER(_P), C.POINTER(C.c_uint64)],
    "mpsw_synth_fill": [_P, C.c_int, C.c_int, C.c_uint64, C.c_int],
    "mpsw_swap_in": [_P, C.c_int, C.POINTER(C.c_uint64)],
    "mpsw_swap_out": [_P, C.c_int, C.POINTER(C.c_uint64)],
    "mpsw_wait": [_P, C.c_uint64, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "mpsw_entry_gpu_ms": [_P, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_float)],
    "mpsw_request": [_P, C.c_int, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int64)],
    "mpsw_poll": [_P, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "mpsw_wait_request": [_P, C.c_int64, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "mpsw_checksum": [_P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64)],
    "mpsw_peek": [_P, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _P],
    "mpsw_residency": [_P, C.c_int, C.POINTER(C.c_int)],
    "mpsw_trace_dump": [_P, C.c_char_p],
    "mpsw_timeline_dump": [_P, C.c_char_p],
    "mpsw_get_stats": [_P, C.POINTER(Stats)],
    "mpsw_bench_gemm": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)],
    "mpsw_tc_plan": [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)],
    "mpsw_test_gemm": [C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                       C.POINTER(C.c_float)],
    "mpsw_test_tap": [_P, C.c_int, C.c_int, C.c_int, _P, C.c_uint64],
    "mpsw_set_writeback": [_P, C.c_int],
    "mpsw_test_inject_fault": [_P, C.c_int],
    "mpsw_test_corrupt_stamp": [_P, C.c_int],
}

_lib = None


def lib():
    """Load libmpsw.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.mpsw_last_error.restype = C.c_char_p
        L.mpsw_last_error.argtypes = []
        _lib = L
    return _lib


def _check(st):
    if st != OK:
        raise MpswError(st, lib().mpsw_last_error().decode())
    return st


def test_gemm(W, X, bias=None, impl=2, epi=0, scale=1.0, dtype=BF16, device=0):
    """Verification hook (include/mpsw_testing.h): one library GEMM on host arrays.
    W [N, K], X [M, K] as uint16 bf16 bits (dtype BF16) or float32; returns float32 [M, N]."""
    W = np.ascontiguousarray(W)
    X = np.ascontiguousarray(X)
    N, K = W.shape
    M = X.shape[0]
    b = None if bias is None else np.ascontiguousarray(bias)
    out = np.empty((M, N), np.float32)
    _check(lib().mpsw_test_gemm(device, dtype, impl, W.ctypes.data, X.ctypes.data,
                                None if b is None else b.ctypes.data, M, N, K, epi, scale,
                                out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


TC_PLAN_KEYS = ("workers", "tiles_per_unit", "unit_tiles", "kblocks", "ctas", "cta_pairs", "stages", "smem_bytes",
                "tmem_cols", "fixup_grid", "ctas_per_sm", "mp")


def tc_plan(N, K, M):
    """Launch plan of one tcgen05 GEMM, host arithmetic only (include/mpsw_testing.h)."""
    out = (C.c_int64 * 12)()
    _check(lib().mpsw_tc_plan(N, K, M, out))
    return dict(zip(TC_PLAN_KEYS, (int(v) for v in out)))


def bench_gemm(M, N, K, impl=2, reps=20, device=0):
    """Average device microseconds of one library GEMM launch (include/mpsw_testing.h)."""
    us = C.c_float()
    _check(lib().mpsw_bench_gemm(device, impl, M, N, K, reps, C.byref(us)))
    return us.value


def dims_of(d):
    return OptDims(d.n_layers, d.hidden, d.heads, d.ffn, d.vocab, d.max_pos)


def shard_layout(dims, tp, rank=0, dtype=BF16, pp=1, stage=0):
    """[(name, offset, bytes, rows, cols, split, tensor_id)], shard_bytes of (stage, TP rank)."""
    od = dims_of(dims)
    n = C.c_int()
    sb = C.c_uint64()
    _check(lib().mpsw_shard_layout(C.byref(od), tp, pp, stage, rank, dtype, None, 0, C.byref(n), C.byref(sb)))
    arr = (TensorDesc * n.value)()
    _check(lib().mpsw_shard_layout(C.byref(od), tp, pp, stage, rank, dtype, arr, n.value, C.byref(n), C.byref(sb)))
    return [(t.name.decode(), t.offset, t.bytes, t.rows, t.cols, t.split, t.tensor_id) for t in arr], sb.value


class Ctx:
    """One TP group (see include/mpsw.h). Methods mirror the C-ABI names."""

    def __init__(self, device_ids=(0,), budget=1 << 30, max_batch=8, max_tokens=8, dtype=BF16,
                 max_inflight=1, swap_mode=SWAP_AUTO, chunk_bytes=0, writeback=1, trace=0, zc_ctas=0,
                 world_size=1, world_rank=0, shm_name=None, gemm_impl=0, pp=1, helper_device_ids=(),
                 max_dims=None, prefetch=0, pp_broadcast=0, victim_policy=0, debug_checks=0):
        """Single-process: one ctx over len(device_ids) = tp * pp ranks (global rank
        g = stage * tp + tp_rank). Multi-process (world_size > 1): device_ids = (this process's
        GPU,), rank world_rank of a TP group of world_size. max_dims: the largest model shape the
        forward workspace must hold when models of different sizes are registered (default:
        the first registered model). prefetch: load predicted models into free space while no
        swap is in flight (reading #29)."""
        self._ids = (C.c_int * len(device_ids))(*device_ids)
        self.world_size, self.world_rank = world_size, world_rank
        self.pp = pp
        self.nr = world_size if world_size > 1 else len(device_ids)      # ranks (workers)
        self.tp = self.nr // pp                                            # TP degree
        self.local_ranks = [world_rank] if world_size > 1 else list(range(len(device_ids)))
        self._shm = shm_name.encode() if shm_name else None
        cfg = Config(len(device_ids), self._ids, self.tp, budget, 0, max_batch, max_tokens, dtype,
                     max_inflight, swap_mode, chunk_bytes, writeback, trace, zc_ctas, world_size, world_rank,
                     self._shm, gemm_impl, pp,
                     (C.c_int * max(1, len(helper_device_ids)))(*helper_device_ids) if helper_device_ids else None,
                     len(helper_device_ids), dims_of(max_dims) if max_dims is not None else OptDims(), prefetch,
                     pp_broadcast, victim_policy, debug_checks)
        h = _P()
        _check(lib().mpsw_init(C.byref(cfg), C.byref(h)))
        self.h = h
        self.dtype = dtype
        self.vocab = None        # vocab of the last registered model
        self.vocabs = {}         # model id -> vocab (logits length)
        self._live = {}          # request id -> output array the library writes into (kept alive)
        self._done = {}          # request id -> (t_arrival, t_done); the library releases ids on OK

    def close(self):
        if self.h:
            lib().mpsw_shutdown(self.h)   # waits for in-flight work before buffers are released
            self.h = None
            self._live.clear()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def register_model(self, dims, shards=None):
        """shards: list of nr per-rank blobs in global-rank order (non-local entries may be None)."""
        od = dims_of(dims)
        mid = C.c_int()
        if shards is None:
            _check(lib().mpsw_register_model(self.h, C.byref(od), self.tp, None, None, C.byref(mid)))
        else:
            arrs = [None if s is None else np.ascontiguousarray(s) for s in shards]
            ptrs = (_P * self.nr)(*[None if a is None else a.ctypes.data for a in arrs])
            sizes = (C.c_uint64 * self.nr)(*[0 if a is None else a.nbytes for a in arrs])
            _check(lib().mpsw_register_model(self.h, C.byref(od), self.tp, ptrs, sizes, C.byref(mid)))
        self.vocab = dims.vocab
        self.vocabs[mid.value] = dims.vocab
        return mid.value

    def model_arena(self, model_id, rank):
        """numpy uint8 view of the pinned arena (library-owned memory)."""
        p = _P()
        n = C.c_uint64()
        _check(lib().mpsw_model_arena(self.h, model_id, rank, C.byref(p), C.byref(n)))
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(n.value,))

    def synth_fill(self, model_id, seed, rank=-1, threads=0):
        _check(lib().mpsw_synth_fill(self.h, model_id, rank, seed, threads))

    def swap_in(self, model_id):
        t = C.c_uint64()
        _check(lib().mpsw_swap_in(self.h, model_id, C.byref(t)))
        return t.value

    def swap_out(self, model_id):
        t = C.c_uint64()
        _check(lib().mpsw_swap_out(self.h, model_id, C.byref(t)))
        return t.value

    def wait(self, ticket, timeout=-1.0):
        """(t_submit, [t_ack per rank]); on a follower only its own rank's entry is meaningful."""
        ts = C.c_double()
        td = (C.c_double * self.nr)()
        _check(lib().mpsw_wait(self.h, ticket, timeout, C.byref(ts), td))
        return ts.value, list(td)

    def entry_gpu_ms(self, ticket):
        k, m = C.c_int(), C.c_int()
        ms = (C.c_float * self.nr)()
        _check(lib().mpsw_entry_gpu_ms(self.h, ticket, C.byref(k), C.byref(m), ms))
        return k.value, m.value, list(ms)

    def request(self, model_id, tokens, out=None):
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        V = self.vocabs.get(model_id, self.vocab or 1)
        if out is None:
            out = np.empty(V, np.float32)
        rid = C.c_int64()
        if out.dtype != np.float32 or out.size < V or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float32 array of at least vocab elements")
        _check(lib().mpsw_request(self.h, model_id, tok.ctypes.data_as(C.POINTER(C.c_int32)), tok.size,
                                  out.ctypes.data_as(C.POINTER(C.c_float)), C.byref(rid)))
        self._live[rid.value] = out    # the library writes here until the request completes
        return rid.value, out

    def poll(self, rid):
        a, d = C.c_double(), C.c_double()
        if rid in self._done:
            return self._done[rid]
        st = lib().mpsw_poll(self.h, rid, C.byref(a), C.byref(d))
        if st == EAGAIN:
            return None
        _check(st)
        self._live.pop(rid, None)
        self._done[rid] = (a.value, d.value)
        return a.value, d.value

    def wait_request(self, rid, timeout=-1.0):
        if rid in self._done:
            return self._done[rid]
        a, d = C.c_double(), C.c_double()
        _check(lib().mpsw_wait_request(self.h, rid, timeout, C.byref(a), C.byref(d)))
        self._live.pop(rid, None)
        self._done[rid] = (a.value, d.value)
        return a.value, d.value

    def tap(self, n_layers, what, rank, nbytes):
        """Arm the one-shot forward tap (include/mpsw_testing.h) and return the host buffer the
        next dispatched batch fills (uint8, nbytes); valid once that batch's request completed."""
        buf = np.zeros(nbytes, np.uint8)
        _check(lib().mpsw_test_tap(self.h, n_layers, what, rank, buf.ctypes.data, nbytes))
        self._tap_buf = buf
        return buf

    def inject_fault(self, rank):
        """Test hook (include/mpsw_testing.h): rank throws at its next all-reduce point."""
        _check(lib().mpsw_test_inject_fault(self.h, rank))

    def corrupt_stamp(self, model_id):
        """Test hook (include/mpsw_testing.h): make the model's next forward trip the debug check."""
        _check(lib().mpsw_test_corrupt_stamp(self.h, model_id))

    def set_writeback(self, writeback):
        _check(lib().mpsw_set_writeback(self.h, int(writeback)))

    @staticmethod
    def _retry(fn, tries=200):
        """Re-issue a verification read that raced a swap (EAGAIN, include/mpsw.h)."""
        import time
        for _ in range(tries):
            st = fn()
            if st != EAGAIN:
                return _check(st)
            time.sleep(0.005)
        return _check(st)

    def checksum(self, model_id, rank, on_device=True):
        h = C.c_uint64()
        self._retry(lambda: lib().mpsw_checksum(self.h, model_id, rank, int(on_device), C.byref(h)))
        return h.value

    def peek(self, model_id, rank, offset, nbytes):
        buf = np.empty(nbytes, np.uint8)
        self._retry(lambda: lib().mpsw_peek(self.h, model_id, rank, offset, nbytes, buf.ctypes.data))
        return buf

    def residency(self, model_id):
        s = C.c_int()
        _check(lib().mpsw_residency(self.h, model_id, C.byref(s)))
        return s.value

    def trace_dump(self, path):
        _check(lib().mpsw_trace_dump(self.h, path.encode()))

    def timeline_dump(self, path):
        _check(lib().mpsw_timeline_dump(self.h, path.encode()))

    def stats(self):
        s = Stats()
        _check(lib().mpsw_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}
