"""Reduce/copy operators — drop-in for ``ftdp.kernels`` (kernels.py:16-56).

The reference selects, at import, between a compiled Cython loop
(_ckernels.pyx:9-27) and numpy; both do ``dst[i] += f32(src[i])`` in order and
``dst[:] = src``.  Here the only backend is the sm_100a library: the same two
operators on CUDA tensors, with a bf16 source upcast exactly to fp32.  There
is no CPU fallback; a missing library fails at import.
"""

from __future__ import annotations

import torch

from . import _lib

BACKEND = "sm_100a"


def _args(dst: torch.Tensor, src: torch.Tensor, op: str):
    if not (isinstance(dst, torch.Tensor) and dst.is_cuda and dst.dtype == torch.float32 and dst.is_contiguous()):
        raise ValueError(f"{op}: dst must be a contiguous float32 CUDA tensor")
    if not (isinstance(src, torch.Tensor) and src.is_cuda and src.is_contiguous()):
        raise ValueError(f"{op}: src must be a contiguous CUDA tensor")
    if src.dtype == torch.float32:
        code = _lib.DT_F32
    elif src.dtype == torch.bfloat16:
        code = _lib.DT_BF16
    else:
        raise ValueError(f"{op}: src must be float32 or bfloat16")
    if src.numel() != dst.numel():
        raise ValueError(f"{op}: src byte length does not match dst")
    return code, torch.cuda.current_stream(dst.device).cuda_stream


def accumulate(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[i] += src[i] (fp32, in order, separately rounded)."""
    code, stream = _args(dst, src, "accumulate")
    _lib.check(_lib.lib.ftar_accumulate(dst.data_ptr(), src.data_ptr(), code, dst.numel(), stream), "accumulate")


def copy_into(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[:] = src (bf16 upcast exactly)."""
    code, stream = _args(dst, src, "copy_into")
    _lib.check(_lib.lib.ftar_copy_into(dst.data_ptr(), src.data_ptr(), code, dst.numel(), stream), "copy_into")


def backends() -> dict[str, tuple]:
    """kernels.py:51-56: every available backend (one here)."""
    return {BACKEND: (accumulate, copy_into)}
