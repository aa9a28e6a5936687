"""Attention with additive bias on B200 — drop-in for pkg/src/flashbias/attention.py.

Public names and argument meaning follow the reference:

* ``flashbias_attention(q, k, v, fq, fk, mask="none", tiles=None)``
  (attention.py:205-230): logits = q k^T / sqrt(C) + fq fk^T with C the
  ORIGINAL channel count; computed as a widened contraction inside the
  tcgen05 kernel (K1): [q | sqrt(C) fq][k | fk]^T / sqrt(C) (the reference
  order) or Q' = [q / sqrt(C), fq], K' = [k, fk] (north_star fold, chosen when
  it needs fewer bf16 split columns -- see FactorPlan).
* ``tiled_attention(q, k, v, bias=NO_BIAS, mask, tiles, scale)``
  (attention.py:140-202): NoBias / DenseBias (K3, bias tile streamed by TMA) /
  FactoredBias (K1, the factor term unscaled).
* ``reference_attention`` / ``attention_weights`` (attention.py:111-137): the
  materialised formula, evaluated on the GPU with torch (validation helper).
* ``TileConfig`` / ``choose_tile_sizes`` (attention.py:38-74): kept for API
  compatibility; on B200 the tile is fixed by UMMA (128 x 128), ``tiles`` is
  validated and otherwise advisory (outputs are tiling-invariant,
  tests/test_attention.py:143-158 of the reference).

Inputs: numpy arrays (reference style, 2-D per head, returned as float64
numpy) or torch tensors ([N, C], [H, N, C] or [B, H, N, C]) on CPU or CUDA.
Compute precision follows the input: bf16/fp16 -> tcgen05 kernels (forward and
backward, autograd-enabled); fp32/fp64 -> the fp32 SIMT kernel (forward).
Host inputs are copied to the GPU and results copied back (the e2e path).
There is no CPU fallback: without the CUDA library every call raises.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .bias import NO_BIAS, DenseBias, FactoredBias, NoBias, _is_torch
from .errors import ConfigError, MaskError, ShapeError, ValidationError

MASK_NONE = "none"
MASK_CAUSAL = "causal"
MASK_FILL = float(np.finfo(np.float64).min)
_SUPPORTED_D = (32, 64, 128)


@dataclass(frozen=True)
class TileConfig:
    """Rows per query block and per key/value block (advisory on B200)."""

    b_q: int
    b_kv: int
    sram_budget_bytes: Optional[int] = None

    def __post_init__(self):
        if self.b_q < 1 or self.b_kv < 1:
            raise ConfigError("tile sizes must be >= 1")


def choose_tile_sizes(c: int, r: int, sram_bytes: int, dtype_bytes: int) -> TileConfig:
    """Reference sizing rule b_q = floor(S / (4 e (c+r))), b_kv = min(b_q, c+r),
    rounded down to multiples of 8 (attention.py:51-74)."""
    width = c + r
    if width < 1:
        raise ConfigError("c + r must be >= 1")
    need = 4 * dtype_bytes * width
    if sram_bytes < need:
        raise ConfigError(f"sram_bytes={sram_bytes} below minimum {need} for width c+r={width}")
    b_q = sram_bytes // need
    b_kv = min(b_q, width)
    r8 = lambda x: x - x % 8 if x >= 8 else x  # noqa: E731
    return TileConfig(max(1, r8(b_q)), max(1, r8(b_kv)), sram_bytes)


# ---------------------------------------------------------------- input plumbing
class _Shape:
    """Remember how a user input was laid out so the result mirrors it."""

    def __init__(self, x):
        self.numpy = not _is_torch(x)
        self.device = None if self.numpy else x.device
        self.dtype = None if self.numpy else x.dtype
        self.ndim = np.ndim(x) if self.numpy else x.dim()


def _to_torch(x, name: str, device, dtype=None):
    import torch
    if _is_torch(x):
        t = x
        if t.dim() < 2 or t.dim() > 4:
            raise ShapeError(f"{name} must be 2-D, 3-D or 4-D, got ndim={t.dim()}")
    else:
        a = np.asarray(x, dtype=np.float64)
        if a.ndim != 2:
            raise ShapeError(f"{name} must be 2-D, got ndim={a.ndim}")
        t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if t.device != device:
        t = t.to(device, non_blocking=True)
    while t.dim() < 4:
        t = t.unsqueeze(0)
    return t


def _compute_dtype(shape: _Shape, precision: Optional[str]):
    import torch
    if precision is not None:
        return {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[precision]
    if shape.numpy or shape.dtype in (torch.float64, torch.float32):
        return torch.float32
    if shape.dtype in (torch.bfloat16, torch.float16):
        return shape.dtype
    raise ValidationError(f"unsupported dtype {shape.dtype}")


def _validate_mask(mask: str, n: int, m: int) -> None:
    if mask not in (MASK_NONE, MASK_CAUSAL):
        raise ValidationError(f"unknown mask {mask!r}")
    if mask == MASK_CAUSAL and n != m:
        raise MaskError(f"causal mask requires N == M, got {n} x {m}")


def _validate_qkv_shapes(q, k, v) -> None:
    if q.shape[-1] != k.shape[-1]:
        raise ShapeError(f"q and k channel counts differ: {q.shape[-1]} vs {k.shape[-1]}")
    if k.shape[-2] != v.shape[-2]:
        raise ShapeError(f"k and v row counts differ: {k.shape[-2]} vs {v.shape[-2]}")


def _pad_last(t, to: int):
    import torch
    if t.shape[-1] == to:
        return t.contiguous()
    out = torch.zeros(*t.shape[:-1], to, dtype=t.dtype, device=t.device)
    out[..., : t.shape[-1]] = t
    return out


def _padded_head_dim(c: int) -> int:
    for d in _SUPPORTED_D:
        if c <= d:
            return d
    raise ConfigError(f"head dim {c} > 128 is not supported by the sm_100a kernels")


_SPLIT_CACHE: dict = {}


@dataclass(frozen=True)
class FactorPlan:
    """How a factor pair enters the widened contraction (north_star fold).

    The logits are ``s * q.k + fq.fk``.  ``q_fold`` False: the reference order
    (attention.py:225-230), uq = split(fq / s) and the kernel scales the whole
    product by s.  ``q_fold`` True: Q' = [s * q, U], K' = [k, V] -- the kernel
    scale is 1, q is pre-scaled (one bf16 rounding of q) and uq = split(fq),
    so bf16-exact SVD / neural factors need no split even when 1/s = sqrt(C)
    is not a power of two.  ``split`` is the bf16 k-way split level."""

    split: int
    q_fold: bool
    premul: float
    kernel_scale: float


def _is_pow2(x: float) -> bool:
    return x > 0 and math.frexp(x)[0] == 0.5


def _part_stats(x64, x32, pdt, dims):
    """Per-rank magnitudes of the k-way split the prepare kernel builds from the
    fp32 value x32 (fb_small.cu split_part: successive residual roundings to the
    panel dtype): P[i] = max|part_i| (i < 3), Rs[k] = max|x_exact - sum_{i<k} part_i|
    (k = 1..3; includes the fp32 rounding of premul*f), X = max|x_exact|."""
    import torch
    rem = x32.clone()
    acc = torch.zeros_like(x64)
    P, Rs = [], []
    for _ in range(3):
        part = rem.to(pdt).float()
        rem = rem - part
        acc = acc + part.double()
        P.append(part.abs().amax(dim=dims))
        Rs.append((x64 - acc).abs().amax(dim=dims))
    return P, Rs, x64.abs().amax(dim=dims)


def _split_bounds(fq, fk, premuls, pdt=None):
    """One device->host read: for each premul, the worst-case |logit term error|
    (in units of premul*fq.fk) of the k-way split for k = 1, 2, 3:
      sum_r [ sum_{i,j<k, i+j>=k} P_a[i] P_b[j] + Ra[k] max|b| + (max|a| + Ra[k]) Rb[k] ]
    (a = premul*fq, b = fk; the kept columns are the part pairs i + j <= k-1)."""
    import torch
    pdt = pdt or torch.bfloat16
    dims_a = tuple(range(fq.dim() - 1))
    dims_b = tuple(range(fk.dim() - 1))
    b64 = fk.detach().double()
    Pb, Rb, Xb = _part_stats(b64, fk.detach().float(), pdt, dims_b)
    rows = []
    for pm in premuls:
        a64 = fq.detach().double() * pm
        Pa, Ra, Xa = _part_stats(a64, fq.detach().float() * pm, pdt, dims_a)
        for k in (1, 2, 3):
            t = Ra[k - 1] * Xb + (Xa + Ra[k - 1]) * Rb[k - 1]
            for i in range(k):
                for j in range(k):
                    if i + j >= k:
                        t = t + Pa[i] * Pb[j]
            rows.append(t.sum())
    vals = torch.stack(rows).cpu().tolist()
    return [vals[3 * n: 3 * n + 3] for n in range(len(premuls))]


def _split_level(bounds, logit_scale: float, r: int, tol: float, max_cols: int) -> Optional[int]:
    """Smallest k in {1,2,3} with logit_scale * bound_k <= tol and R k(k+1)/2 <= max_cols; None if none."""
    for k in (1, 2, 3):
        if r * k * (k + 1) // 2 > max_cols:
            return None
        b = bounds[k - 1] * logit_scale
        if b == b and b <= tol:  # NaN/inf (e.g. fp16 overflow) never qualifies
            return k
    return None


def choose_split(fq, fk, premul: float = 1.0, tol: float = 1e-2, max_cols: int = 64, logit_scale=None,
                 panel_dtype=None) -> int:
    """bf16 k-way split level for logical fp32 factors.

    The smallest k whose worst-case error on the logit term, logit_scale *
    |premul fq.fk - sum of the kept part products| (default logit_scale =
    1/premul: the reference fold, logits = (1/premul) * (premul fq).fk), is
    within ``tol`` with R * k(k+1)/2 <= max_cols columns.  Raises ConfigError
    when no level meets the bound inside the panel budget (it never silently
    drops below it)."""
    ls = 1.0 / premul if logit_scale is None else logit_scale
    bounds = _split_bounds(fq, fk, [premul], panel_dtype)[0]
    k = _split_level(bounds, ls, int(fq.shape[-1]), tol, max_cols)
    if k is None:
        raise ConfigError(
            f"rank-{fq.shape[-1]} factors need more than {max_cols} panel columns to stay within {tol:g} logits "
            f"(k=1..3 error bounds {[round(b * ls, 6) for b in bounds]}); pass bf16-exact factors, a lower rank, "
            f"or use the fp32 path")
    return k


def plan_factor_fold(fq, fk, scale: float, tol: float = 1e-2, max_cols: int = 64, panel_dtype=None,
                     shard_invariant: bool = False) -> FactorPlan:
    """Pick the fold and split for logits = scale*q.k + fq.fk (see FactorPlan).

    The reference order is kept whenever 1/scale is a power of two (exact) or
    it needs no more columns; otherwise Q' = [scale*q, U] avoids the
    premultiplier's rounding.  Raises ConfigError if neither meets ``tol``.

    ``shard_invariant``: the split level must not depend on WHICH heads share
    the launch (the bound is a max over them), so use the most accurate level
    that fits ``max_cols`` -- a function of R alone -- and only check ``tol``."""
    pm = 1.0 / scale
    r = int(fq.shape[-1])
    if shard_invariant:
        kfit = max([k for k in (1, 2, 3) if r * k * (k + 1) // 2 <= max_cols] or [0])
        if kfit:
            ba, bq = _split_bounds(fq, fk, [pm, 1.0], panel_dtype)
            if ba[kfit - 1] * scale <= tol:
                return FactorPlan(kfit, False, pm, scale)
            if bq[kfit - 1] <= tol:
                return FactorPlan(kfit, True, 1.0, 1.0)
        raise ConfigError(f"rank-{r} factors cannot meet {tol:g} logits within {max_cols} panel columns")
    if _is_pow2(pm):
        ba = _split_bounds(fq, fk, [pm], panel_dtype)[0]
        ka, kq, bq = _split_level(ba, scale, r, tol, max_cols), None, None
    else:
        ba, bq = _split_bounds(fq, fk, [pm, 1.0], panel_dtype)
        ka = _split_level(ba, scale, r, tol, max_cols)
        kq = _split_level(bq, 1.0, r, tol, max_cols)
    if ka is not None and (kq is None or ka <= kq):
        return FactorPlan(ka, False, pm, scale)
    if kq is not None:
        return FactorPlan(kq, True, 1.0, 1.0)
    raise ConfigError(
        f"rank-{r} factors need more than {max_cols} panel columns to stay within {tol:g} logits "
        f"(k=1..3 error bounds {[round(b * scale, 6) for b in ba]}); pass bf16-exact factors, a lower rank, "
        f"or use the fp32 path")


def _base_of(t):
    return t._base if t._base is not None else t


def plan_factor_fold_cached(fq_user, fk_user, fq, fk, scale: float, tol: float = 1e-2,
                            max_cols: int = 64, panel_dtype=None, shard_invariant: bool = False) -> FactorPlan:
    """plan_factor_fold memoised per user factor tensors (the decision needs a
    device->host read; static factors such as ALiBi/spatial pay it once).

    Identity = the base tensor OBJECT (held by weak reference) + the view
    geometry + the shared in-place version counter, so per-call views of the
    same factors (head slices) hit the cache, while a new tensor that happens
    to reuse a freed allocation never inherits a stale split level.  numpy
    inputs (a fresh device copy every call) are not cached."""
    import weakref
    if not (_is_torch(fq_user) and _is_torch(fk_user)):
        return plan_factor_fold(fq, fk, scale, tol, max_cols, panel_dtype, shard_invariant)
    bq, bk = _base_of(fq_user), _base_of(fk_user)

    def geom(t, base):
        return (id(base), base._version, t.storage_offset(), tuple(t.shape), tuple(t.stride()), t.dtype)
    key = (geom(fq_user, bq), geom(fk_user, bk), float(scale), float(tol), int(max_cols), str(panel_dtype),
           bool(shard_invariant))
    hit = _SPLIT_CACHE.get(key)
    if hit is not None and hit[0]() is bq and hit[1]() is bk:
        return hit[2]
    plan = plan_factor_fold(fq, fk, scale, tol, max_cols, panel_dtype, shard_invariant)
    if len(_SPLIT_CACHE) > 256:
        _SPLIT_CACHE.clear()
    _SPLIT_CACHE[key] = (weakref.ref(bq), weakref.ref(bk), plan)
    return plan


def prepare_factor_panels(fq, fk, premul: float, split: int, dtype):
    """Device-ready panels (fb_prepare_factors): uq = split(premul*fq), uk = split(fk)."""
    import torch
    lib = _lib.lib()
    with torch.cuda.device(fq.device):
        fq32 = fq.float().contiguous()
        fk32 = fk.float().contiguous()
        r = fq32.shape[-1]
        rpad = int(lib.fb_factor_rpad(r, split))
        uq = torch.empty(*fq32.shape[:-1], rpad, dtype=dtype, device=fq32.device)
        uk = torch.empty(*fk32.shape[:-1], rpad, dtype=dtype, device=fk32.device)
        s = _lib.stream_ptr(fq32.device)
        D, ref = _lib.desc, _lib.ref
        _lib.check(lib.fb_prepare_factor_pair(ref(D(fq32)), ref(D(fk32)), split, float(premul), ref(D(uq)),
                                              ref(D(uk)), s))
    return uq, uk


_PANEL_CACHE: dict = {}


def prepare_factor_panels_cached(fq, fk, premul: float, split: int, dtype):
    """prepare_factor_panels memoised on the factor tensors' identity (base
    object by weak reference + view geometry + in-place version counter), so
    static factors (ALiBi, spatial, offline SVD) are split into panels once,
    not every step; any in-place update (an optimizer step) re-splits."""
    import weakref
    bq, bk = _base_of(fq), _base_of(fk)

    def geom(t, base):
        return (id(base), base._version, t.storage_offset(), tuple(t.shape), tuple(t.stride()), t.dtype, t.device)
    key = (geom(fq, bq), geom(fk, bk), float(premul), int(split), dtype)
    hit = _PANEL_CACHE.get(key)
    if hit is not None and hit[0]() is bq and hit[1]() is bk:
        return hit[2]
    panels = prepare_factor_panels(fq, fk, premul, split, dtype)
    if len(_PANEL_CACHE) >= 8:
        _PANEL_CACHE.pop(next(iter(_PANEL_CACHE)))
    _PANEL_CACHE[key] = (weakref.ref(bq), weakref.ref(bk), panels)
    return panels


_F32_CACHE: dict = {}


def _fp32_factors_cached(fq, fk, scale: float):
    """The fp32 path's factor operands uq = fq / scale, uk = fk (fp32, contiguous), memoised like
    prepare_factor_panels_cached so static factors cost no per-call elementwise launch."""
    import weakref
    bq, bk = _base_of(fq), _base_of(fk)

    def geom(t, base):
        return (id(base), base._version, t.storage_offset(), tuple(t.shape), tuple(t.stride()), t.dtype, t.device)
    key = (geom(fq, bq), geom(fk, bk), float(scale))
    hit = _F32_CACHE.get(key)
    if hit is not None and hit[0]() is bq and hit[1]() is bk:
        return hit[2]
    ops = ((fq.float() / scale).contiguous(), fk.float().contiguous())
    if len(_F32_CACHE) >= 8:
        _F32_CACHE.pop(next(iter(_F32_CACHE)))
    _F32_CACHE[key] = (weakref.ref(bq), weakref.ref(bk), ops)
    return ops


def fold_factor_grads(dpanel, like, side: int, split: int, postmul: float):
    """fb_fold_factor_grads: split-panel gradients -> logical factor gradient shaped like ``like``."""
    import torch
    lib = _lib.lib()
    with torch.cuda.device(dpanel.device):
        out = torch.empty(like.shape, dtype=torch.float32, device=dpanel.device)
        _lib.check(lib.fb_fold_factor_grads(_lib.ref(_lib.desc(dpanel)), side, split, float(postmul),
                                            _lib.ref(_lib.desc(out)), _lib.stream_ptr(dpanel.device)))
    return out


# ---------------------------------------------------------------- core launches
def _fwd_launch(q, k, v, uq, uk, bias, mask_code, scale, need_lse=True):
    import torch
    lib = _lib.lib()
    B, H, N, _ = q.shape
    with torch.cuda.device(q.device):
        o = torch.empty(B, H, N, v.shape[-1], dtype=q.dtype, device=q.device)
        lse = torch.empty(B, H, N, dtype=torch.float32, device=q.device) if need_lse else None
        D = _lib.desc
        _lib.check(lib.fb_attn_fwd(_lib.ref(D(q)), _lib.ref(D(k)), _lib.ref(D(v)), _lib.ref(D(uq)), _lib.ref(D(uk)),
                                   _lib.ref(D(bias)), mask_code, float(scale), _lib.ref(D(o)), _lib.ref(D(lse)),
                                   _lib.stream_ptr(q.device)))
    return o, lse


FB_BWD_DETERMINISTIC = 1


def _bwd_launch(q, k, v, uq, uk, bias, o, lse, do, mask_code, scale, want_fgrad, deterministic=False,
                want_dbias=False):
    import torch
    lib = _lib.lib()
    D = _lib.desc
    with torch.cuda.device(q.device):
        dq = torch.empty_like(q)
        dk = torch.empty_like(k)
        dv = torch.empty_like(v)
        duq = duk = None
        if want_fgrad and uq is not None:
            B, H = q.shape[0], q.shape[1]
            duq = torch.empty(B, H, q.shape[2], uq.shape[-1], dtype=torch.float32, device=q.device)
            duk = torch.empty(B, H, k.shape[2], uk.shape[-1], dtype=torch.float32, device=q.device)
        db = None
        if want_dbias:  # [B,H,N,M] in the bias dtype, even row stride; causal blocks above the diagonal stay 0
            B, H, N, M = q.shape[0], q.shape[1], q.shape[2], k.shape[2]
            alloc = torch.zeros if mask_code == 1 else torch.empty
            db = alloc(B, H, N, M + (M & 1), dtype=bias.dtype, device=q.device)[..., :M]
        dq_d, k_d = D(q), D(k)
        ws_bytes = int(lib.fb_bwd_workspace_bytes(_lib.ref(dq_d), _lib.ref(k_d)))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
        _lib.check(lib.fb_attn_bwd_ex(_lib.ref(D(q)), _lib.ref(D(k)), _lib.ref(D(v)), _lib.ref(D(uq)),
                                      _lib.ref(D(uk)), _lib.ref(D(bias)), _lib.ref(D(o)), _lib.ref(D(lse)),
                                      _lib.ref(D(do)), mask_code, float(scale), _lib.ref(D(dq)), _lib.ref(D(dk)),
                                      _lib.ref(D(dv)), _lib.ref(D(duq)), _lib.ref(D(duk)), _lib.ref(D(db)),
                                      FB_BWD_DETERMINISTIC if deterministic else 0, ws.data_ptr(), ws_bytes,
                                      _lib.stream_ptr(q.device)))
    return dq, dk, dv, duq, duk, db


def _make_fn():
    import torch

    class FlashBiasFunction(torch.autograd.Function):
        """Autograd wrapper: forward K1/K3, backward K2/K4 (+ factor gradients)."""

        @staticmethod
        def forward(ctx, q, k, v, fq, fk, bias, mask_code, scale, premul, split, deterministic=False):
            uq = uk = None
            if fq is not None:
                uq, uk = prepare_factor_panels_cached(fq, fk, premul, split, q.dtype)
            o, lse = _fwd_launch(q, k, v, uq, uk, bias, mask_code, scale)
            ctx.save_for_backward(q, k, v, uq, uk, bias, o, lse, fq, fk)
            ctx.cfg = (mask_code, scale, premul, split, deterministic)
            return o

        @staticmethod
        def backward(ctx, do):
            q, k, v, uq, uk, bias, o, lse, fq, fk = ctx.saved_tensors
            mask_code, scale, premul, split, deterministic = ctx.cfg
            want_db = bias is not None and ctx.needs_input_grad[5]
            want_fg = fq is not None and (ctx.needs_input_grad[3] or ctx.needs_input_grad[4])
            dq, dk, dv, duq, duk, db = _bwd_launch(q, k, v, uq, uk, bias, o, lse, do.contiguous(), mask_code,
                                                   scale, want_fg, deterministic, want_db)
            if db is not None:  # learnable dense bias: sum dS over the dims the bias broadcasts
                dims = [i for i in (0, 1) if bias.shape[i] == 1 and db.shape[i] != 1]
                if dims:
                    db = db.sum(dim=dims, keepdim=True)
            dfq = dfk = None
            if want_fg:
                # the kernel's duq is d/d(uq) of scale*uq.uk; uq = premul*fq -> dfq = premul*duq
                dfq = fold_factor_grads(duq, fq, 0, split, premul).to(fq.dtype)
                dfk = fold_factor_grads(duk, fk, 1, split, 1.0).to(fk.dtype)
            return dq, dk, dv, dfq, dfk, db, None, None, None, None, None

    return FlashBiasFunction


_FN = None


def _fn():
    global _FN
    if _FN is None:
        _FN = _make_fn()
    return _FN


def _needs_grad(*ts) -> bool:
    return any(t is not None and _is_torch(t) and t.requires_grad for t in ts)


def _attention(q, k, v, *, fq=None, fk=None, bias=None, mask="none", scale=None, precision=None, split=None,
               deterministic=False):
    """Shared driver: logits = scale*q.k + fq.fk + bias (+ causal); normalise
    inputs, run the kernel, mirror the input layout."""
    import torch
    shp = _Shape(q)
    _validate_qkv_shapes(q, k, v)
    n, m, c = int(q.shape[-2]), int(k.shape[-2]), int(q.shape[-1])
    _validate_mask(mask, n, m)
    if scale is None:
        scale = 1.0 / math.sqrt(c)
    if not torch.cuda.is_available():
        raise RuntimeError("flashbias: CUDA device required (no CPU fallback)")
    device = shp.device if (shp.device is not None and shp.device.type == "cuda") else torch.device("cuda")
    cdt = _compute_dtype(shp, precision)
    with torch.cuda.device(device):
        return _attention_on_device(q, k, v, fq, fk, bias, mask, float(scale), cdt, split, shp, device, n, m, c,
                                    deterministic)


def _attention_on_device(q, k, v, fq, fk, bias, mask, scale, cdt, split, shp, device, n, m, c, deterministic):
    import torch
    qt = _to_torch(q, "q", device, cdt)
    kt = _to_torch(k, "k", device, cdt)
    vt = _to_torch(v, "v", device, cdt)
    if qt.shape[:2] != kt.shape[:2] or kt.shape[:2] != vt.shape[:2]:
        raise ShapeError("batch/head extents of q, k, v differ")
    fqt = fkt = None
    if fq is not None:
        fqt = _to_torch(fq, "fq", device)
        fkt = _to_torch(fk, "fk", device)
        if fqt.shape[-1] != fkt.shape[-1]:
            raise ShapeError(f"factor ranks differ: {fqt.shape[-1]} vs {fkt.shape[-1]}")
        if fqt.shape[-2] != n:
            raise ShapeError(f"fq rows {fqt.shape[-2]} do not match q rows {n}")
        if fkt.shape[-2] != m:
            raise ShapeError(f"fk rows {fkt.shape[-2]} do not match k rows {m}")
    bt = None
    if bias is not None:
        bt = _to_torch(bias, "bias", device)
        if tuple(bt.shape[-2:]) != (n, m):
            raise ShapeError(f"bias shape {tuple(bt.shape[-2:])} does not match logits {(n, m)}")
    mask_code = _lib.MASK_CODES[mask]
    if qt.shape[0] * qt.shape[1] == 0:  # zero heads (e.g. an empty shard): nothing to launch
        return _mirror(torch.empty(*qt.shape[:3], vt.shape[-1], dtype=qt.dtype, device=device), shp)

    if cdt == torch.float32:
        if torch.is_grad_enabled() and _needs_grad(q, k, v, fq, fk, bias):
            raise ConfigError("the fp32 path is forward-only: inputs that require grad need precision='bf16' "
                              "or 'fp16' (tcgen05 forward + backward)")
        qf, kf, vf = (t.contiguous() for t in (qt, kt, vt))
        uq = uk = None
        if fqt is not None:
            uq, uk = _fp32_factors_cached(fqt, fkt, scale)
        bf = bt.float().contiguous() if bt is not None else None
        o, _ = _fwd_launch(qf, kf, vf, uq, uk, bf, mask_code, scale, need_lse=False)
    else:
        dp = _padded_head_dim(max(c, int(vt.shape[-1])))
        qp, kp, vp = _pad_last(qt, dp), _pad_last(kt, dp), _pad_last(vt, dp)
        bp = None
        if bt is not None:
            # -inf / finfo.min entries round to -inf: the kernels treat them as masked keys
            bt = bt.to(cdt)
            if m % 8:
                store = torch.zeros(*bt.shape[:-1], (m + 7) // 8 * 8, dtype=cdt, device=device)
                store[..., :m] = bt
                bp = store[..., :m]
            else:
                bp = bt.contiguous()
        kscale, premul, sp = scale, 1.0 / scale, None
        if fqt is not None:
            max_cols = 64 if dp == 128 else 128
            if split is not None:
                plan = FactorPlan(int(split), False, 1.0 / scale, scale)
            else:
                plan = plan_factor_fold_cached(fq, fk, fqt, fkt, scale, max_cols=max_cols, panel_dtype=cdt,
                                               shard_invariant=deterministic)
            sp, premul, kscale = plan.split, plan.premul, plan.kernel_scale
            if plan.q_fold:  # Q' = [scale*q, U]: autograd carries d/dq = scale * d/dQ'
                qp = qp * scale
        o = _fn().apply(qp, kp, vp, fqt, fkt, bp, mask_code, float(kscale), float(premul), sp, bool(deterministic))
        o = o[..., : vt.shape[-1]]
    return _mirror(o, shp)


def _mirror(o, shp: _Shape):
    if shp.numpy:
        return o.reshape(o.shape[-2], o.shape[-1]).double().cpu().numpy()
    while o.dim() > shp.ndim:
        o = o.squeeze(0)
    if shp.device is not None and o.device != shp.device:
        o = o.to(shp.device)
    if o.dtype != shp.dtype:
        o = o.to(shp.dtype)
    return o


def _check_tiles(tiles) -> None:
    if tiles is not None and not isinstance(tiles, TileConfig):
        raise ValidationError("tiles must be a TileConfig")


# ---------------------------------------------------------------- public API
def flashbias_attention(q, k, v, fq, fk, mask: str = MASK_NONE, tiles: Optional[TileConfig] = None, *,
                        precision: Optional[str] = None, split: Optional[int] = None, deterministic: bool = False):
    """softmax(q k^T / sqrt(C) + fq fk^T) v without materialising the bias
    (attention.py:205-230): widened contraction [q | sqrt(C) fq][k | fk]^T with
    the original 1/sqrt(C) scale, folded into the tcgen05 kernel.

    ``deterministic``: bitwise-reproducible gradients (two-kernel backward, no
    atomics) and a factor split level that depends on the rank only, so the
    result of a head does not depend on the heads it is launched with."""
    _check_tiles(tiles)
    c = int(q.shape[-1])
    return _attention(q, k, v, fq=fq, fk=fk, mask=mask, scale=1.0 / math.sqrt(c), precision=precision,
                      split=split, deterministic=deterministic)


def tiled_attention(q, k, v, bias=NO_BIAS, mask: str = MASK_NONE, tiles: Optional[TileConfig] = None,
                    scale: Optional[float] = None, *, precision: Optional[str] = None,
                    split: Optional[int] = None, deterministic: bool = False):
    """Streaming attention with NoBias / DenseBias / FactoredBias (attention.py:140-202)."""
    _check_tiles(tiles)
    c = int(q.shape[-1])
    if scale is None:
        scale = 1.0 / math.sqrt(c)
    if isinstance(bias, NoBias):
        return _attention(q, k, v, mask=mask, scale=scale, precision=precision, deterministic=deterministic)
    if isinstance(bias, DenseBias):
        return _attention(q, k, v, bias=bias.b, mask=mask, scale=scale, precision=precision,
                          deterministic=deterministic)
    if isinstance(bias, FactoredBias):
        # the factor term is added unscaled: logits = scale*q.k + fq.fk
        return _attention(q, k, v, fq=bias.fq, fk=bias.fk, mask=mask, scale=scale, precision=precision,
                          split=split, deterministic=deterministic)
    raise ValidationError(f"unknown bias provider {type(bias).__name__}")


def _dense_of(bias, n: int, m: int):
    if isinstance(bias, NoBias):
        return None
    if isinstance(bias, DenseBias):
        b = bias.b
    elif isinstance(bias, FactoredBias):
        b = bias.dense()
    else:
        raise ValidationError(f"unknown bias provider {type(bias).__name__}")
    if tuple(b.shape[-2:]) != (n, m):
        raise ShapeError(f"bias shape {tuple(b.shape[-2:])} does not match logits {(n, m)}")
    return b


def attention_weights(q, k, bias=NO_BIAS, mask: str = MASK_NONE, scale: Optional[float] = None):
    """Row-stochastic weights of the materialised formula (attention.py:111-128), on the GPU in fp64."""
    import torch
    shp = _Shape(q)
    if q.shape[-1] != k.shape[-1]:
        raise ShapeError(f"q and k channel counts differ: {q.shape[-1]} vs {k.shape[-1]}")
    n, m = int(q.shape[-2]), int(k.shape[-2])
    _validate_mask(mask, n, m)
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[-1])
    dev = torch.device("cuda")
    qt = _to_torch(q, "q", dev, torch.float64)
    kt = _to_torch(k, "k", dev, torch.float64)
    logits = (qt @ kt.transpose(-1, -2)) * scale
    b = _dense_of(bias, n, m)
    if b is not None:
        logits = logits + _to_torch(b, "bias", dev, torch.float64)
    if mask == MASK_CAUSAL:
        upper = torch.ones(n, m, dtype=torch.bool, device=dev).triu(1)
        logits = logits.masked_fill(upper, MASK_FILL)
    w = torch.softmax(logits, dim=-1)
    return _mirror_f64(w, shp)


def reference_attention(q, k, v, bias=NO_BIAS, mask: str = MASK_NONE, scale: Optional[float] = None):
    """softmax(q k^T scale + bias + mask) v with the full logit matrix (attention.py:131-137)."""
    import torch
    _validate_qkv_shapes(q, k, v)
    shp = _Shape(q)
    w = attention_weights(q if not shp.numpy else np.asarray(q, dtype=np.float64), k, bias, mask, scale)
    wt = w if _is_torch(w) else torch.from_numpy(w).cuda()
    vt = _to_torch(v, "v", wt.device, torch.float64)
    out = wt.to(torch.float64) @ vt
    return _mirror_f64(out, shp)


def _mirror_f64(t, shp: _Shape):
    if shp.numpy:
        return t.reshape(t.shape[-2], t.shape[-1]).cpu().numpy()
    while t.dim() > shp.ndim:
        t = t.squeeze(0)
    return t
