"""Reference-side binding: what a maintainer of the numpy ``flashbias`` package
would add to route ``flashbias_attention`` (pkg/src/flashbias/attention.py:205-230)
to the B200 C ABI (include/flashbias_b200.h) — ctypes + libcudart only, no
torch.  Host numpy in, host numpy out, exactly the reference signature.

    from flashbias_ctypes_binding import flashbias_attention_b200
    o = flashbias_attention_b200(q, k, v, fq, fk, mask="causal")   # float64 numpy

fp32 device compute (the 1e-5 SIMT kernel); pass precision="bf16" for the
tcgen05 kernel (q/k/v rounded to bf16, factors split into bf16 panels).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.environ.get("FLASHBIAS_B200_LIB",
                      os.path.join(_HERE, "..", "paper_2505_12044_b200", "_lib", "libflashbias_b200.so"))


class FbTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("shape", ctypes.c_int64 * 4),
                ("stride", ctypes.c_int64 * 4), ("dtype", ctypes.c_int32)]


_fb = ctypes.CDLL(_LIB)
_cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if _cudart is None:
    import ctypes.util
    _cudart = ctypes.CDLL(ctypes.util.find_library("cudart") or "libcudart.so")
_P = ctypes.POINTER(FbTensor)
_fb.fb_attn_fwd.argtypes = [_P, _P, _P, _P, _P, _P, ctypes.c_int, ctypes.c_float, _P, _P, ctypes.c_void_p]
_fb.fb_prepare_factors.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_float, _P, ctypes.c_void_p]
_fb.fb_factor_rpad.restype = ctypes.c_int64
_fb.fb_factor_rpad.argtypes = [ctypes.c_int64, ctypes.c_int]
_fb.fb_last_error.restype = ctypes.c_char_p
_cudart.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
_cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
_cudart.cudaFree.argtypes = [ctypes.c_void_p]
_H2D, _D2H = 1, 2
_ERRORS = {1: "ShapeError", 2: "MaskError", 3: "ConfigError", 4: "ValidationError"}


def _check(rc: int) -> None:
    if rc:
        raise ValueError(f"{_ERRORS.get(rc, 'CUDA error')}: {_fb.fb_last_error().decode()}")


class _Dev:
    """A device copy of a host array viewed as [1, 1, rows, cols]."""

    def __init__(self, arr: np.ndarray, dtype_code: int):
        self.host = np.ascontiguousarray(arr)
        self.ptr = ctypes.c_void_p()
        assert _cudart.cudaMalloc(ctypes.byref(self.ptr), max(self.host.nbytes, 16)) == 0
        assert _cudart.cudaMemcpy(self.ptr, self.host.ctypes.data, self.host.nbytes, _H2D) == 0
        self.t = FbTensor()
        self.t.data = self.ptr.value
        rows, cols = self.host.shape
        for i, (s, st) in enumerate(zip((1, 1, rows, cols), (rows * cols, rows * cols, cols, 1))):
            self.t.shape[i], self.t.stride[i] = s, st
        self.t.dtype = dtype_code

    def to_host(self) -> np.ndarray:
        out = np.empty_like(self.host)
        assert _cudart.cudaMemcpy(out.ctypes.data, self.ptr, out.nbytes, _D2H) == 0
        return out

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            _cudart.cudaFree(self.ptr)


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit patterns (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def flashbias_attention_b200(q, k, v, fq, fk, mask: str = "none", precision: str = "fp32") -> np.ndarray:
    q, k, v, fq, fk = (np.asarray(x, dtype=np.float64) for x in (q, k, v, fq, fk))
    c = q.shape[1]
    root_c = math.sqrt(c)
    mcode = {"none": 0, "causal": 1}[mask]
    if precision == "fp32":
        dq, dk, dv = (_Dev(x.astype(np.float32), 0) for x in (q, k, v))
        duq, duk = _Dev((root_c * fq).astype(np.float32), 0), _Dev(fk.astype(np.float32), 0)
        do = _Dev(np.zeros((q.shape[0], v.shape[1]), np.float32), 0)
        _check(_fb.fb_attn_fwd(ctypes.byref(dq.t), ctypes.byref(dk.t), ctypes.byref(dv.t), ctypes.byref(duq.t),
                               ctypes.byref(duk.t), None, mcode, 1.0 / root_c, ctypes.byref(do.t), None, None))
        return do.to_host().astype(np.float64)
    # bf16: head dim padded to a tcgen05 size, factors split on the device
    dpad = 32 if c <= 32 else (64 if c <= 64 else 128)
    pad = lambda x: np.pad(x, ((0, 0), (0, dpad - x.shape[1])))  # noqa: E731
    dq, dk, dv = (_Dev(_bf16_bits(pad(x)), 1) for x in (q, k, v))
    split = 3 if fq.shape[1] * 6 <= (64 if dpad == 128 else 128) else (2 if fq.shape[1] * 3 <= 64 else 1)
    rpad = _fb.fb_factor_rpad(fq.shape[1], split)
    fq32, fk32 = _Dev(fq.astype(np.float32), 0), _Dev(fk.astype(np.float32), 0)
    uq = _Dev(np.zeros((q.shape[0], rpad), np.uint16), 1)
    uk = _Dev(np.zeros((k.shape[0], rpad), np.uint16), 1)
    _check(_fb.fb_prepare_factors(ctypes.byref(fq32.t), 0, split, root_c, ctypes.byref(uq.t), None))
    _check(_fb.fb_prepare_factors(ctypes.byref(fk32.t), 1, split, 1.0, ctypes.byref(uk.t), None))
    do = _Dev(np.zeros((q.shape[0], dpad), np.uint16), 1)
    _check(_fb.fb_attn_fwd(ctypes.byref(dq.t), ctypes.byref(dk.t), ctypes.byref(dv.t), ctypes.byref(uq.t),
                           ctypes.byref(uk.t), None, mcode, 1.0 / root_c, ctypes.byref(do.t), None, None))
    return _bf16_to_f64(do.to_host())[:, : v.shape[1]]
