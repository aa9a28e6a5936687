"""Head splitting by bias rank and the mixed factored / dense attention path.

``split_heads_by_rank`` restates the reference partition (pkg/src/flashbias/
decompose.py:179-225) on the GPU: one batched float64 SVD over the head stack
(cuSOLVER through torch.linalg.svd), energy ranks from the cumulative
spectrum, the shared kernel rank rounded up to a multiple of 8, factors
U sqrt(s) / V sqrt(s) zero-padded to it.  The deployment pattern it serves
(reference test_acceptance.py:204-236) runs the
low-rank heads through the FlashBias kernel and the remaining heads through
the dense-bias kernel.  ``mixed_head_attention`` does that with one launch
per subset; with the heads permuted offline into two contiguous stacks
(``HeadSplit.permutation``/``permuted``) the subsets are views, otherwise they
are gathered and the outputs scattered back into head order.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from .attention import MASK_NONE, TileConfig, flashbias_attention, tiled_attention
from .bias import DenseBias, FactoredBias
from .errors import ShapeError, ValidationError

__all__ = ["HeadSplit", "split_heads_by_rank", "mixed_head_attention"]


@dataclass
class HeadSplit:
    """Partition of a head stack into a factored (low-rank) subset and a dense
    remainder (ref: decompose.py:170-177).  ``low_fq``/``low_fk`` hold the
    stacked device factors [H_low, N, R] / [H_low, M, R] of ``low_factors``."""

    low_indices: List[int]
    low_factors: List[FactoredBias]
    dense_indices: List[int]
    common_rank: int
    low_fq: object = field(default=None, repr=False)
    low_fk: object = field(default=None, repr=False)

    def permutation(self) -> List[int]:
        """Head order that makes both subsets contiguous (low first): apply it
        once offline to the model's heads so mixed_head_attention slices
        instead of gathering."""
        return list(self.low_indices) + list(self.dense_indices)

    def permuted(self) -> "HeadSplit":
        """The same split expressed in permutation() order."""
        nl = len(self.low_indices)
        return HeadSplit(list(range(nl)), self.low_factors, list(range(nl, nl + len(self.dense_indices))),
                         self.common_rank, self.low_fq, self.low_fk)


def _stack_heads(biases):
    import torch
    if isinstance(biases, torch.Tensor):
        if biases.dim() != 3:
            raise ShapeError(f"head stack must be [H, N, M], got shape {tuple(biases.shape)}")
        return biases.to("cuda", torch.float64)
    if len(biases) < 1:
        raise ValidationError("need at least one head")
    mats = []
    for i, b in enumerate(biases):
        t = b if isinstance(b, torch.Tensor) else torch.as_tensor(b)
        if t.dim() != 2:
            raise ShapeError(f"head {i} must be 2-D, got ndim={t.dim()}")
        mats.append(t.to("cuda", torch.float64))
    for i, t in enumerate(mats):
        if t.shape != mats[0].shape:
            raise ShapeError(f"head {i} shape {tuple(t.shape)} differs from {tuple(mats[0].shape)}")
    return torch.stack(mats)


def split_heads_by_rank(biases: Sequence, energy_threshold: float, max_rank: int) -> HeadSplit:
    """Assign each head to the factored or dense path by its energy rank (ref: decompose.py:179-225).

    A head joins the low subset when the smallest rank retaining
    ``energy_threshold`` of its energy is at most ``max_rank``.  All low heads
    share one rank (the subset maximum rounded up to a multiple of 8)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("flashbias: CUDA device required (no CPU fallback)")
    if not isinstance(biases, torch.Tensor) and len(biases) < 1:
        raise ValidationError("need at least one head")
    if not 0.0 < energy_threshold <= 1.0:
        raise ValidationError("energy threshold must lie in (0, 1]")
    b = _stack_heads(biases)
    u, s, vh = torch.linalg.svd(b, full_matrices=False)          # batched cuSOLVER, f64
    s2 = s * s
    cum = torch.cumsum(s2, dim=-1)
    tot = cum[:, -1:]
    prof = torch.where(tot > 0, cum / torch.where(tot > 0, tot, torch.ones_like(tot)), torch.ones_like(cum))
    # smallest k with prof[k-1] >= threshold == searchsorted(prof, threshold) + 1 (left side)
    thr = torch.full((prof.shape[0], 1), float(energy_threshold), dtype=prof.dtype, device=prof.device)
    ranks = (torch.searchsorted(prof.contiguous(), thr).squeeze(1) + 1).tolist()
    low = [i for i, r in enumerate(ranks) if r <= max_rank]
    dense = [i for i in range(b.shape[0]) if i not in low]
    if not low:
        return HeadSplit([], [], dense, 0)
    common = (max(ranks[i] for i in low) + 7) // 8 * 8
    k_eff = min(common, s.shape[-1])
    idx = torch.tensor(low, device=b.device)
    root = torch.sqrt(s[idx, :k_eff])
    fq = u[idx, :, :k_eff] * root[:, None, :]
    fk = vh[idx, :k_eff, :].transpose(-1, -2) * root[:, None, :]
    if k_eff < common:  # pad to the shared kernel rank
        fq = torch.nn.functional.pad(fq, (0, common - k_eff))
        fk = torch.nn.functional.pad(fk, (0, common - k_eff))
    factors = [FactoredBias(fq[j], fk[j], origin="svd", descriptor=f"head{i}(common_rank={common})")
               for j, i in enumerate(low)]
    return HeadSplit(low, factors, dense, common, low_fq=fq, low_fk=fk)


_SIDE = {}


def _side_stream(device):
    """One cached side stream per device for the concurrent subset launch."""
    import torch
    key = torch.device(device).index
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


def mixed_head_attention(q, k, v, split: HeadSplit, biases, mask: str = MASK_NONE,
                         tiles: Optional[TileConfig] = None, *, precision: Optional[str] = None):
    """Per-head attention with the split's factored heads on the FlashBias
    kernel and its dense heads on the dense-bias kernel.

    q, k, v: [B, H, L, C], [H, L, C] or 2-D (shared by every head, as in the
    reference criterion-9 test); biases: the [H, N, M] stack the split was
    computed from (only the dense heads are read; broadcast over B).  Returns
    the output in head order with q's layout."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("flashbias: CUDA device required (no CPU fallback)")
    nh = len(split.low_indices) + len(split.dense_indices)
    numpy_in = not isinstance(q, torch.Tensor)

    def heads_of(x, name):
        t = torch.as_tensor(x) if not isinstance(x, torch.Tensor) else x
        t = t.to("cuda")
        if t.dim() == 2:
            t = t.unsqueeze(0).expand(nh, -1, -1)
        if t.dim() == 3:
            t = t.unsqueeze(0)
        if t.dim() != 4 or t.shape[1] != nh:
            raise ShapeError(f"{name} must be [H, L, C] or [B, H, L, C] with H = {nh}, or 2-D")
        return t

    batched = isinstance(q, torch.Tensor) and q.dim() == 4
    qh, kh, vh = heads_of(q, "q"), heads_of(k, "k"), heads_of(v, "v")
    b = None
    if split.dense_indices:
        b = biases if (isinstance(biases, torch.Tensor) and biases.is_cuda and biases.dim() == 3) \
            else _stack_heads(biases)
        if b.shape[0] != nh:
            raise ShapeError(f"bias stack has {b.shape[0]} heads, split covers {nh}")

    def take(t, idx, dim=1):
        # heads permuted offline into contiguous stacks (split.permutation()) are plain views
        if idx == list(range(idx[0], idx[0] + len(idx))):
            return t.narrow(dim, idx[0], len(idx))
        return t.index_select(dim, torch.tensor(idx, device=t.device))

    parts = []
    # Both subsets at once: each launch alone under-fills the 148 SMs at small head counts, so the
    # FlashBias launch runs on a side stream next to the dense-bias launch (autograd runs each
    # backward on its forward's stream, so the backwards overlap too).
    both = bool(split.low_indices) and bool(split.dense_indices)
    cur = torch.cuda.current_stream(qh.device)
    side = _side_stream(qh.device) if both else cur
    if both:
        side.wait_stream(cur)
    if split.low_indices:
        li = split.low_indices
        fq = split.low_fq if split.low_fq is not None else torch.stack([torch.as_tensor(f.fq) for f in split.low_factors])
        fk = split.low_fk if split.low_fk is not None else torch.stack([torch.as_tensor(f.fk) for f in split.low_factors])
        # the low subset: one FlashBias launch over the [1, H_low, ...] stack
        with torch.cuda.stream(side):
            o_low = flashbias_attention(take(qh, li), take(kh, li), take(vh, li),
                                        fq.to("cuda").unsqueeze(0), fk.to("cuda").unsqueeze(0), mask=mask,
                                        tiles=tiles, precision=precision)
        parts.append((li, o_low))
    if split.dense_indices:
        di = split.dense_indices
        # the dense subset: one dense-bias launch
        o_dense = tiled_attention(take(qh, di), take(kh, di), take(vh, di),
                                  DenseBias(take(b, di, 0).unsqueeze(0)), mask=mask, tiles=tiles, precision=precision)
        parts.append((di, o_dense))
    if both:
        cur.wait_stream(side)
        o_low.record_stream(cur)
    if len(parts) == 2 and parts[0][0] + parts[1][0] == list(range(nh)):
        out = torch.cat([parts[0][1], parts[1][1]], 1)
    elif len(parts) == 2 and parts[1][0] + parts[0][0] == list(range(nh)):
        out = torch.cat([parts[1][1], parts[0][1]], 1)
    elif len(parts) == 1:
        out = parts[0][1]
    else:
        o0 = parts[0][1]
        out = torch.empty((o0.shape[0], nh) + tuple(o0.shape[2:]), dtype=o0.dtype, device=o0.device)
        for idx, o in parts:
            out[:, torch.tensor(idx, device=out.device)] = o
    if not batched:
        out = out.squeeze(0)
    if numpy_in:
        return out.double().cpu().numpy()
    return out
