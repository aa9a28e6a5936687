"""ctypes binding of the C ABI in include/flashbias_b200.h.

This is the reference-side binding a maintainer would add:
the shared library libflashbias_b200.so is built in-tree by
``__graft_entry__.build()`` and loaded from ``paper_2505_12044_b200/_lib/``.
Non-zero status codes are mapped back onto the reference's exception
taxonomy (pkg/src/flashbias/errors.py:4-25).  There is no fallback: if the
library is missing or CUDA is unavailable, calls raise.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

from .errors import ConfigError, MaskError, ShapeError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libflashbias_b200.so")

FB_F32, FB_BF16, FB_F16, FB_F64 = 0, 1, 2, 3
MASK_CODES = {"none": 0, "causal": 1}

#: every symbol the public header declares (tests check the .so exports them)
EXPORTED_SYMBOLS = (
    "fb_attn_fwd", "fb_attn_bwd", "fb_attn_bwd_ex", "fb_bwd_workspace_bytes", "fb_prepare_factors",
    "fb_factor_rpad", "fb_factor_cols", "fb_fold_factor_grads", "fb_factor_alibi",
    "fb_factor_spatial", "fb_dense_from_factors", "fb_bwd_preprocess", "fb_last_error",
    "fb_abi_version", "fb_launch_count", "fb_mlp_factor_panels", "fb_prepare_factor_pair",
)


class FbTensor(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("shape", ctypes.c_int64 * 4),
        ("stride", ctypes.c_int64 * 4),
        ("dtype", ctypes.c_int32),
    ]


_P = ctypes.POINTER(FbTensor)
_lib: Optional[ctypes.CDLL] = None


def _declare(lib: ctypes.CDLL) -> None:
    i32, i64, f32, vp, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t
    sig = {
        "fb_attn_fwd": (i32, [_P, _P, _P, _P, _P, _P, i32, f32, _P, _P, vp]),
        "fb_attn_bwd": (i32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, i32, f32, _P, _P, _P, _P, _P, vp, sz, vp]),
        "fb_attn_bwd_ex": (i32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, i32, f32, _P, _P, _P, _P, _P, _P, i32, vp,
                                 sz, vp]),
        "fb_bwd_workspace_bytes": (sz, [_P, _P]),
        "fb_prepare_factors": (i32, [_P, i32, i32, f32, _P, vp]),
        "fb_factor_rpad": (i64, [i64, i32]),
        "fb_factor_cols": (i64, [i64, i32]),
        "fb_fold_factor_grads": (i32, [_P, i32, i32, f32, _P, vp]),
        "fb_factor_alibi": (i32, [vp, i64, i64, i64, _P, _P, vp]),
        "fb_factor_spatial": (i32, [_P, _P, _P, _P, _P, vp]),
        "fb_dense_from_factors": (i32, [_P, _P, _P, vp]),
        "fb_bwd_preprocess": (i32, [_P, _P, _P, vp]),
        "fb_last_error": (ctypes.c_char_p, []),
        "fb_abi_version": (i32, []),
        "fb_launch_count": (i64, [i32]),
        "fb_mlp_factor_panels": (i32, [_P, _P, _P, _P, _P, _P, _P, i32, i32, f32, _P, _P, vp]),
        "fb_prepare_factor_pair": (i32, [_P, _P, i32, f32, _P, _P, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"flashbias native library not built: {LIB_PATH} missing "
                "(run __graft_entry__.build()); there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        _declare(handle)
        _lib = handle
    return _lib


def check(status: int) -> None:
    """Raise the reference exception class matching a C-ABI status code."""
    if status == 0:
        return
    msg = lib().fb_last_error().decode("utf-8", "replace")
    if status == 1:
        raise ShapeError(msg)
    if status == 2:
        raise MaskError(msg)
    if status == 3:
        raise ConfigError(msg)
    if status == 4:
        raise ValidationError(msg)
    raise RuntimeError(f"flashbias CUDA error: {msg}")


def _dtype_code(t) -> int:
    import torch
    return {torch.float32: FB_F32, torch.bfloat16: FB_BF16, torch.float16: FB_F16,
            torch.float64: FB_F64}[t.dtype]


def desc(t) -> Optional[FbTensor]:
    """Describe a torch tensor of rank <= 4 as an fb_tensor ([B,H,L,D] view)."""
    if t is None:
        return None
    while t.dim() < 4:
        t = t.unsqueeze(0)
    if t.dim() != 4:
        raise ShapeError(f"expected a tensor of rank <= 4, got {t.dim()}")
    d = FbTensor()
    d.data = t.data_ptr()
    for i in range(4):
        d.shape[i] = t.shape[i]
        d.stride[i] = t.stride(i)
    d.dtype = _dtype_code(t)
    return d


def ref(d: Optional[FbTensor]):
    return None if d is None else ctypes.byref(d)


def stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
