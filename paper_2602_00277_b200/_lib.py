"""ctypes binding of libftar_b200.so (the C-ABI in include/ftar_b200.h).

There is no fallback: if the shared library is missing or was built for
another architecture, importing this module raises.  The library is built
in-tree by ``paper_2602_00277_b200._build.build()`` (``__graft_entry__.build``).
"""

from __future__ import annotations

import ctypes as C
import os
import re

from . import _build

_HDR = os.path.join(os.path.dirname(_build.PKG), "include", "ftar_b200.h")

c_ctx_p = C.c_void_p
c_snap_p = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int
i64 = C.c_int64
vp = C.c_void_p
dbl = C.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "ftar_last_error": (C.c_char_p, []),
    "ftar_version": (C.c_char_p, []),
    "ftar_set_tuning": (i32, [i32, i32]),
    "ftar_ctx_create": (i32, [i32, u64, u64, i32, C.POINTER(c_ctx_p)]),
    "ftar_ctx_destroy": (i32, [c_ctx_p]),
    "ftar_ctx_pool": (i32, [c_ctx_p, C.POINTER(u64), C.POINTER(u64)]),
    "ftar_ctx_export": (i32, [c_ctx_p, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ftar_ctx_import": (i32, [c_ctx_p, i32, vp, C.c_size_t, u64]),
    "ftar_ctx_unmap": (i32, [c_ctx_p, i32]),
    "ftar_ctx_link_local": (i32, [c_ctx_p, i32, c_ctx_p]),
    "ftar_set_membership": (i32, [c_ctx_p, C.POINTER(i32), i32, i32, u32, u64]),
    "ftar_region_register": (i32, [c_ctx_p, vp, u64, C.POINTER(i32), vp, C.c_size_t, C.POINTER(u64)]),
    "ftar_region_unregister": (i32, [c_ctx_p, i32]),
    "ftar_region_import": (i32, [c_ctx_p, i32, i32, vp, C.c_size_t, u64, u64]),
    "ftar_allreduce_launch": (i32, [c_ctx_p, vp, i32, vp, u64, u64, i32, C.c_float, u32, vp]),
    "ftar_allreduce_sgd_launch": (i32, [c_ctx_p, vp, i32, vp, u64, u64, i32, C.c_float, u32, vp, vp, vp, vp,
                                        C.c_float, C.c_float, vp]),
    "ftar_local_allreduce_sgd_launch": (i32, [C.POINTER(c_ctx_p), i32, C.POINTER(vp), i32, C.POINTER(vp), u64, u64,
                                              i32, C.c_float, u32, u32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                              C.POINTER(vp), C.c_float, C.c_float, vp]),
    "ftar_allreduce_launch_range": (i32, [c_ctx_p, vp, i32, vp, u64, u64, u64, u64, i32, C.c_float, u32, vp]),
    "ftar_intra_launch": (i32, [c_ctx_p, i32, vp, i32, vp, u64, C.POINTER(u64), C.POINTER(u64), vp]),
    "ftar_local_intra_launch": (i32, [C.POINTER(c_ctx_p), i32, i32, C.POINTER(vp), i32, C.POINTER(vp), u64,
                                      C.POINTER(u64), C.POINTER(u64), vp]),
    "ftar_local_allreduce_launch_range": (i32, [C.POINTER(c_ctx_p), i32, C.POINTER(vp), i32, C.POINTER(vp), u64,
                                                u64, u64, u64, i32, C.c_float, u32, u32, i32, i32, vp]),
    "ftar_local_allreduce_launch": (i32, [C.POINTER(c_ctx_p), i32, C.POINTER(vp), i32,
                                          C.POINTER(vp), u64, u64, i32, C.c_float, u32, u32,
                                          i32, i32, vp]),
    "ftar_poll": (i32, [c_ctx_p, C.POINTER(i32), C.POINTER(u64)]),
    "ftar_abort": (i32, [c_ctx_p]),
    "ftar_inflight": (i32, [c_ctx_p]),
    "ftar_wait": (i32, [c_ctx_p, dbl, C.POINTER(i32)]),
    "ftar_wait_local": (i32, [C.POINTER(c_ctx_p), i32, dbl, C.POINTER(i32), C.POINTER(i32)]),
    "ftar_geometry": (i32, [u64, i32, C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)]),
    "ftar_inflight_bound": (i32, [i32, u64, i32, u64, i32, i32, C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)]),
    "ftar_probe_clock": (i32, [i32, i32, C.POINTER(C.c_int64)]),
    "ftar_snap_region": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64), C.POINTER(u64), C.POINTER(u64),
                               C.POINTER(C.c_int64)]),
    "ftar_accumulate": (i32, [vp, vp, i32, u64, vp]),
    "ftar_copy_into": (i32, [vp, vp, i32, u64, vp]),
    "ftar_snap_create": (i32, [i32, u64, i32, C.POINTER(c_snap_p)]),
    "ftar_snap_destroy": (i32, [c_snap_p]),
    "ftar_snap_export": (i32, [c_snap_p, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ftar_snap_capture": (i32, [c_snap_p, u64, vp, u64, vp, u64, vp]),
    "ftar_snap_info": (i32, [c_snap_p, C.POINTER(i64), C.POINTER(u64), C.POINTER(u64)]),
    "ftar_snap_import": (i32, [c_snap_p, i32, vp, C.c_size_t, u64]),
    "ftar_snap_unmap": (i32, [c_snap_p, i32]),
    "ftar_snap_peer_info": (i32, [c_snap_p, i32, C.POINTER(i64), C.POINTER(u64), C.POINTER(u64)]),
    "ftar_snap_pull_launch": (i32, [c_snap_p, i32, c_snap_p, u64, vp, u64, vp, u64, i32, vp]),
    "ftar_snap_pull_multi_launch": (i32, [c_snap_p, C.POINTER(i32), i32, c_snap_p, u64, vp, u64, vp, u64, i32, vp]),
    "ftar_snap_poll": (i32, [c_snap_p, C.POINTER(i32), C.POINTER(u64), C.POINTER(i64)]),
    "ftar_snap_pull_boost": (i32, [c_snap_p, i32, vp]),
    "ftar_snap_abort": (i32, [c_snap_p]),
    "ftar_snap_wait": (i32, [c_snap_p, dbl, C.POINTER(i64)]),
    "ftar_probe_copy": (i32, [vp, vp, u64, i32, vp]),
    "ftar_probe_bulk": (i32, [vp, vp, u64, i32, i32, i32, vp]),
    "ftar_peer_enable": (i32, [i32, i32]),
    "ftar_probe_fence": (i32, [vp, vp, vp, u64, i32, i32, vp, i32, vp]),
    "ftar_phase_times": (i32, [c_ctx_p, C.POINTER(u64), i32]),
    "ftar_debug_cta_times": (i32, [c_ctx_p, C.POINTER(u64), C.POINTER(u64), i32]),
    "ftar_debug_trace": (i32, [c_ctx_p, C.POINTER(u64), i32]),
    "ftar_probe_pattern": (i32, [vp, vp, vp, u64, i32, i32, i32, i32, i32, vp]),
}

DT_F32 = 0
DT_BF16 = 1
OP_RS, OP_AG = 1, 2  # ftar_intra_launch ops
F_SCALE = 1
F_PROTOCOL = 2


def header_symbols(path: str = _HDR) -> list[str]:
    """Every function the public header declares."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ftar_[a-z_]+)\s*\(", text)))


def _load() -> C.CDLL:
    path = _build.LIB_DIAG if os.environ.get("FTAR_LIB_VARIANT") == "diag" else _build.LIB
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with paper_2602_00277_b200._build.build() "
            "(the FTAR data plane has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    return (lib.ftar_last_error() or b"").decode(errors="replace")


def check(code: int, what: str = "") -> None:
    """Raise the taxonomy exception for a failing C-ABI call."""
    if code:
        from .errors import from_status
        raise from_status(code, f"{what}: {last_error()}" if what else last_error())


def version() -> str:
    return lib.ftar_version().decode()
