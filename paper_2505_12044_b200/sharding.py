"""Batch x head sharding across the GPUs of one box.

Every (b, h) head is independent, so the path partitions with no data-path
collective: rank r owns a contiguous range of whole heads (head-major, all
batch rows of a head on one rank, so batch-broadcast factor gradients never
span ranks).  Inputs are generated / loaded per rank; the only collective is
the optional all-gather of outputs and gradients after the kernels (NCCL over
NVLink on GPUs, gloo in the CPU tests).  The reference has no distribution
(SPEC.md:449); this is new plumbing around the same per-head computation.
"""

from __future__ import annotations

from typing import Callable, Sequence, Tuple


def head_range(num_heads: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) head range of ``rank`` (ceil split; tail ranks may be short/empty)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    per = (num_heads + world - 1) // world
    lo = min(rank * per, num_heads)
    return lo, min(lo + per, num_heads)


def shard_heads(t, world: int, rank: int, dim: int = 1):
    """This rank's slice of a [B, H, ...] tensor along the head dim."""
    lo, hi = head_range(t.shape[dim], world, rank)
    return t.narrow(dim, lo, hi - lo)


def gather_heads(local, num_heads: int, group=None, dim: int = 1):
    """All-gather per-rank head slices back into the full [B, H, ...] tensor.

    Uniform-size collective: slices are zero-padded to ceil(H / world) heads,
    gathered with ``all_gather_into_tensor`` (one NCCL call), then trimmed."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = (num_heads + world - 1) // world
    x = local.movedim(dim, 0).contiguous()
    if x.shape[0] < per:
        pad = torch.zeros((per - x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        x = torch.cat([x, pad], 0)
    out = torch.empty((per * world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if hasattr(dist, "all_gather_into_tensor") and out.device.type == "cuda":
        dist.all_gather_into_tensor(out, x, group=group)
    else:
        parts = list(out.chunk(world, 0))
        dist.all_gather(parts, x, group=group)
        out = torch.cat(parts, 0)
    return out[:num_heads].movedim(0, dim).contiguous()


def sharded_apply(fn: Callable, tensors: Sequence, num_heads: int, group=None, gather: bool = True):
    """Run ``fn`` on this rank's head slice of every [B, H, ...] tensor and
    (optionally) gather the per-head result.  ``fn`` is the hot path (e.g. a
    ``flashbias_attention`` closure); no collective runs inside it."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = [shard_heads(t, world, rank) if t is not None and t.dim() >= 2 and t.shape[1] == num_heads else t
             for t in tensors]
    out = fn(*local)
    if not gather or world == 1:
        return out
    return gather_heads(out, num_heads, group)
