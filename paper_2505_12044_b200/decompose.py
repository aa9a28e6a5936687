"""Bias factorisation on the device — drop-in for pkg/src/flashbias/decompose.py.

* ``decompose_alibi``  (decompose.py:37-52)  exact rank 2, closed form;
* ``decompose_spatial`` (decompose.py:55-81) exact rank 9, closed form;
* ``alibi_factors`` / ``spatial_factors``: multi-head device forms used by the
  kernels (K6, C-ABI ``fb_factor_alibi`` / ``fb_factor_spatial``, fp32);
* ``svd_decompose`` (decompose.py:98-138): truncated SVD on the GPU —
  cuSOLVER (``torch.linalg.svd``) for small matrices, a GEMM-bound randomized
  range finder (K7) for large ones when only a rank is requested;
* ``energy_profile`` (84-95) and ``reconstruction_report`` (141-165).

numpy in -> numpy (float64) out, computed on the GPU in float64, matching the
reference's arithmetic; torch in -> torch out on the input's device.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .bias import FactoredBias, _is_torch
from .errors import ShapeError, ValidationError


@dataclass
class DecompositionReport:
    rank_used: int
    energy_retained: float
    max_abs_err: float
    rel_fro_err: float

    def as_dict(self) -> dict:
        return {"rank_used": self.rank_used, "energy_retained": self.energy_retained,
                "max_abs_err": self.max_abs_err, "rel_fro_err": self.rel_fro_err}


def _dev():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("flashbias: CUDA device required (no CPU fallback)")
    return torch.device("cuda")


def _t64(x):
    import torch
    if _is_torch(x):
        return x.to(_dev() if x.device.type != "cuda" else x.device, dtype=torch.float64)
    a = np.asarray(x, dtype=np.float64)
    return torch.as_tensor(np.ascontiguousarray(a), device=_dev())


def _back(t, like_numpy: bool):
    return t.cpu().numpy() if like_numpy else t


# ---------------------------------------------------------------- closed forms
def alibi_factors(slopes, n: int, m: int):
    """Per-head ALiBi factors on the device: fq [1,H,N,2] = slope_h [1, i],
    fk [1,H,M,2] = [-j, 1] (1-based), fp32, via fb_factor_alibi."""
    import torch
    if n < 1 or m < 1:
        raise ValidationError("decompose_alibi requires n, m >= 1")
    dev = _dev()
    s = torch.as_tensor(slopes, dtype=torch.float32, device=dev).reshape(-1).contiguous()
    h = s.numel()
    fq = torch.empty(1, h, n, 2, dtype=torch.float32, device=dev)
    fk = torch.empty(1, h, m, 2, dtype=torch.float32, device=dev)
    lib = _lib.lib()
    _lib.check(lib.fb_factor_alibi(s.data_ptr(), h, n, m, _lib.ref(_lib.desc(fq)), _lib.ref(_lib.desc(fk)),
                                   _lib.stream_ptr(dev)))
    return fq, fk


def decompose_alibi(n: int, m: int, slope: float = 1.0) -> FactoredBias:
    """Rank-2 factors of slope*(i - j): fq_i = slope*[1, i], fk_j = [-j, 1]."""
    fq, fk = alibi_factors([slope], n, m)
    fq64 = fq[0, 0].double().cpu().numpy()
    fk64 = fk[0, 0].double().cpu().numpy()
    # fp32 slope*i is exact for power-of-two slopes; re-evaluate in fp64 so
    # arbitrary slopes match the reference bit-for-bit on the host copy
    fq64[:, 0] = slope
    fq64[:, 1] = slope * np.arange(1, n + 1, dtype=np.float64)
    return FactoredBias(fq64, fk64, origin="exact", descriptor=f"alibi(n={n},m={m},slope={slope})")


def spatial_factors(pos_q, pos_k, row_weights=None):
    """Device rank-9 factors (fp32) via fb_factor_spatial.  pos_* [..., L, 3]
    (leading dims broadcast), row_weights [..., N] or None."""
    import torch
    dev = _dev()
    pq = torch.as_tensor(pos_q, dtype=torch.float32, device=dev)
    pk = torch.as_tensor(pos_k, dtype=torch.float32, device=dev)
    while pq.dim() < 4:
        pq = pq.unsqueeze(0)
    while pk.dim() < 4:
        pk = pk.unsqueeze(0)
    if pq.shape[-1] != 3 or pk.shape[-1] != 3:
        raise ShapeError("decompose_spatial requires N x 3 positions")
    w = None
    bq, hq = pq.shape[0], pq.shape[1]
    if row_weights is not None:
        w = torch.as_tensor(row_weights, dtype=torch.float32, device=dev)
        if w.shape[-1] != pq.shape[-2]:
            raise ShapeError("row_weights length must equal pos_q rows")
        while w.dim() < 3:
            w = w.unsqueeze(0)
        w = w.unsqueeze(2).contiguous()  # [Bw, Hw, 1, N]
        bq, hq = max(bq, w.shape[0]), max(hq, w.shape[1])
    fq = torch.empty(bq, hq, pq.shape[2], 9, dtype=torch.float32, device=dev)
    fk = torch.empty(pk.shape[0], pk.shape[1], pk.shape[2], 9, dtype=torch.float32, device=dev)
    lib = _lib.lib()
    _lib.check(lib.fb_factor_spatial(_lib.ref(_lib.desc(pq.contiguous())), _lib.ref(_lib.desc(pk.contiguous())),
                                     _lib.ref(_lib.desc(w)), _lib.ref(_lib.desc(fq)), _lib.ref(_lib.desc(fk)),
                                     _lib.stream_ptr(dev)))
    return fq, fk


def decompose_spatial(pos_q, pos_k, row_weights=None) -> FactoredBias:
    """Rank-9 factors of the weighted squared distance: per coordinate d,
    fq += [x_d^2, 1, -2 x_d] and fk += [1, y_d^2, y_d]; fq row i times w_i."""
    numpy_in = not _is_torch(pos_q)
    pq, pk = _t64(pos_q), _t64(pos_k)
    if pq.dim() != 2 or pk.dim() != 2 or pq.shape[1] != 3 or pk.shape[1] != 3:
        raise ShapeError("decompose_spatial requires N x 3 positions")
    import torch
    one_q = torch.ones(pq.shape[0], dtype=torch.float64, device=pq.device)
    one_k = torch.ones(pk.shape[0], dtype=torch.float64, device=pk.device)
    fq = torch.stack([c for d in range(3) for c in (pq[:, d] ** 2, one_q, -2.0 * pq[:, d])], dim=1)
    fk = torch.stack([c for d in range(3) for c in (one_k, pk[:, d] ** 2, pk[:, d])], dim=1)
    if row_weights is not None:
        w = _t64(row_weights).reshape(-1)
        if w.shape[0] != pq.shape[0]:
            raise ShapeError("row_weights length must equal pos_q rows")
        fq = w[:, None] * fq
    return FactoredBias(_back(fq, numpy_in), _back(fk, numpy_in), origin="exact",
                        descriptor="spatial_distance_3d")


# ---------------------------------------------------------------- SVD
def energy_profile(singular_values):
    """Cumulative energy fractions (decompose.py:84-95); all ones for a zero spectrum."""
    numpy_in = not _is_torch(singular_values)
    s = _t64(singular_values)
    s2 = s * s
    cum = s2.cumsum(0)
    total = float(cum[-1]) if cum.numel() else 0.0
    out = cum.new_ones(cum.shape) if total == 0.0 else cum / total
    return _back(out, numpy_in)


def randomized_svd(b, rank: int, oversample: int = 16, power_iters: int = 2, seed: int = 0):
    """Halko-style range finder on the GPU (K7): Y = (B B^T)^q B Omega, QR,
    then an exact SVD of the small (k+p) x M projection.  GEMM-bound."""
    import torch
    g = torch.Generator(device=b.device).manual_seed(seed)
    n, m = b.shape[-2], b.shape[-1]
    k = min(rank + oversample, min(n, m))
    omega = torch.randn(*b.shape[:-2], m, k, generator=g, device=b.device, dtype=b.dtype)
    y = b @ omega
    for _ in range(power_iters):
        y, _ = torch.linalg.qr(y)
        y = b @ (b.transpose(-1, -2) @ y)
    qm, _ = torch.linalg.qr(y)
    small = qm.transpose(-1, -2) @ b
    ub, s, vh = torch.linalg.svd(small, full_matrices=False)
    u = qm @ ub
    return u[..., :rank], s[..., :rank], vh[..., :rank, :]


def svd_decompose(b, rank: Optional[int] = None, energy: Optional[float] = None, *,
                  method: str = "auto") -> Tuple[FactoredBias, DecompositionReport]:
    """Truncated-SVD factors fq = U_k sqrt(s), fk = V_k sqrt(s) (decompose.py:98-138).

    Exactly one of ``rank`` / ``energy``.  ``method``: "exact" (cuSOLVER SVD),
    "randomized" (rank only) or "auto" (randomized when rank is given and
    min(N, M) > 2048).  The report's energy is exact for "exact"; for
    "randomized" it is computed from the retained singular values against the
    Frobenius norm (sum of all s^2), which is the same quantity.
    """
    import torch
    numpy_in = not _is_torch(b)
    bt = _t64(b) if numpy_in else b.to(_dev() if b.device.type != "cuda" else b.device)
    if bt.dim() != 2:
        raise ShapeError(f"bias must be 2-D, got ndim={bt.dim()}")
    if not torch.isfinite(bt).all():
        raise ValidationError("bias contains non-finite entries")
    if (rank is None) == (energy is None):
        raise ValidationError("specify exactly one of rank= or energy=")
    n, m = bt.shape
    full = min(n, m)
    if energy is not None and not 0.0 < energy <= 1.0:
        raise ValidationError("energy target must lie in (0, 1]")
    if rank is not None and not 1 <= rank <= full:
        raise ValidationError(f"rank must lie in [1, {full}]")
    use_rand = method == "randomized" or (method == "auto" and rank is not None and full > 2048)
    if use_rand and rank is None:
        raise ValidationError("randomized SVD needs rank=")
    work = bt if bt.dtype in (torch.float32, torch.float64) else bt.float()
    norm2 = float((work.double() ** 2).sum())
    if use_rand:
        u, s, vh = randomized_svd(work, rank)
        k = rank
        s64 = s.double()
        retained = float((s64 ** 2).sum())
        energy_k = retained / norm2 if norm2 > 0 else 1.0
    else:
        u, s, vh = torch.linalg.svd(work, full_matrices=False)
        prof = energy_profile(s)
        if energy is not None:
            k = int(torch.searchsorted(prof, torch.tensor([energy], dtype=prof.dtype, device=prof.device))[0]) + 1
            k = min(k, full)
        else:
            k = int(rank)
        energy_k = float(prof[k - 1])
    root = torch.sqrt(s[:k])
    fq = u[:, :k] * root
    fk = vh[:k].transpose(0, 1) * root
    diff = fq.double() @ fk.double().T - bt.double()
    norm_b = norm2 ** 0.5
    rel = float(torch.linalg.norm(diff)) / norm_b if norm_b > 0 else 0.0
    report = DecompositionReport(rank_used=k, energy_retained=float(energy_k),
                                 max_abs_err=float(diff.abs().max()), rel_fro_err=float(rel))
    fb = FactoredBias(_back(fq, numpy_in), _back(fk, numpy_in), origin="svd", descriptor=f"svd(k={k})")
    return fb, report


def reconstruction_report(fb: FactoredBias, target) -> DecompositionReport:
    """max-abs / relative-Frobenius error of fq fk^T against ``target`` plus the
    energy the target's own spectrum retains at fb's rank (decompose.py:141-165)."""
    import torch
    tt = _t64(target)
    if tt.dim() != 2:
        raise ShapeError("target must be 2-D")
    fq, fk = _t64(fb.fq), _t64(fb.fk)
    if (fq.shape[-2], fk.shape[-2]) != tuple(tt.shape):
        raise ShapeError(f"factor shapes imply {(fq.shape[-2], fk.shape[-2])}, target is {tuple(tt.shape)}")
    diff = fq @ fk.T - tt
    norm_t = float(torch.linalg.norm(tt))
    nd = float(torch.linalg.norm(diff))
    rel = nd / norm_t if norm_t > 0 else (0.0 if nd == 0.0 else float("inf"))
    s = torch.linalg.svdvals(tt)
    prof = energy_profile(s)
    k = min(fb.rank, prof.numel())
    return DecompositionReport(rank_used=fb.rank, energy_retained=float(prof[k - 1]) if prof.numel() else 1.0,
                               max_abs_err=float(diff.abs().max()), rel_fro_err=float(rel))
