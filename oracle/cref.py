"""ctypes access to oracle/_build/libftar_oracle.so (the C port of the
reference ring, ftar_ref.c) — TEST / BASELINE INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libftar_oracle.so")


def build() -> str:
    src = os.path.join(HERE, "ftar_ref.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def build_ref() -> str | None:
    """The reference's own compiled kernel (needs /root/reference; dev container only)."""
    if not os.path.exists("/root/reference/pkg/src/ftdp/_ckernels.pyx"):
        return None
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return os.path.join(HERE, "_ref")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.oracle_ring_allreduce.restype = C.c_int
        _lib.oracle_ring_allreduce.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_uint64, C.c_uint64,
                                               C.c_int, C.c_int]
        _lib.oracle_reduce_f32.restype = None
        _lib.oracle_reduce_f32.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                           C.c_void_p]
        _lib.oracle_sgd_momentum.restype = None
        _lib.oracle_sgd_momentum.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_float,
                                             C.c_float]
    return _lib


def ring_allreduce(bufs: list[np.ndarray], chunk_bytes: int, max_in_flight: int, threads_per_member: int = 1) -> int:
    """In-place reference-schedule ring all-reduce of fp32 buffers."""
    n = len(bufs)
    for b in bufs:
        assert b.dtype == np.float32 and b.flags.c_contiguous
    ptrs = (C.c_void_p * n)(*[b.ctypes.data for b in bufs])
    return lib().oracle_ring_allreduce(ptrs, n, bufs[0].size, chunk_bytes, max_in_flight, threads_per_member)


def reduce_f32(arrays: list[np.ndarray], chunk_bytes: int, max_in_flight: int) -> np.ndarray:
    n = len(arrays)
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in arrays]
    out = np.empty(arrs[0].size, dtype=np.float32)
    ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in arrs])
    lib().oracle_reduce_f32(ptrs, n, out.size, chunk_bytes, max_in_flight, out.ctypes.data)
    return out
