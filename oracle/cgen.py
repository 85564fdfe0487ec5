"""Loader of oracle/c/c0gen.c (TEST INFRASTRUCTURE): the C0 generator in plain C + OpenMP, for
full-size oracle weights. Pinned element-for-element against oracle/weights.py."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "c0gen.c")
LIB = os.path.join(HERE, "c", "libc0gen.so")
_lib = None


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", LIB, SRC], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.c0_values.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                C.POINTER(C.c_float)]
        L.c0_values.restype = None
        _lib = L
    return _lib


def values(seed, tensor_id, start, count, gamma, bf16):
    out = np.empty(count, np.float32)
    lib().c0_values(seed & ((1 << 64) - 1), tensor_id, start, count, int(gamma), int(bf16),
                    out.ctypes.data_as(C.POINTER(C.c_float)))
    return out
