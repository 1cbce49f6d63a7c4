"""Build the sm_100a shared library in-tree (no JIT cache, no pip install).

``build()`` compiles ``csrc/ftar_b200.cu`` with nvcc for sm_100a only into
``paper_2602_00277_b200/_lib/libftar_b200.so``; the .so travels to the GPU box
with the repo snapshot.  -fmad=false keeps every fp32 add/multiply separately
rounded, as numpy does in the reference (SURVEY §7 hard part 8).
"""

from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libftar_b200.so")
# timing-diagnostic variant (-DFTAR_DIAGNOSTICS: FTAR_DIAG modes that skip
# stores or read local data only); built on request for tools, never loaded
# by the package unless FTAR_LIB_VARIANT=diag
LIB_DIAG = os.path.join(OUT_DIR, "libftar_b200_diag.so")
SOURCES = [os.path.join(CSRC, "ftar_b200.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "ftar_device.cuh"),
                  os.path.join(os.path.dirname(PKG), "include", "ftar_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "550",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libftar_b200.so")


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, diag: bool = False) -> str:
    lib = LIB_DIAG if diag else LIB
    if not force and up_to_date(lib):
        return lib
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DFTAR_DIAGNOSTICS"] if diag else []), "-o", tmp, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose and res.stderr:
        print(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
