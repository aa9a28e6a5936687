"""Batch x head sharding across the GPUs of one box.

Every (b, h) head is independent, so the path partitions with no data-path
collective: rank r owns a contiguous range of whole heads (head-major, all
batch rows of a head on one rank, so batch-broadcast factor gradients never
span ranks).  Inputs are generated / loaded per rank; the only collective is
the gather of outputs and gradients after the kernels (NCCL over NVLink on
GPUs, gloo in the CPU tests).  The reference has no distribution
(SPEC.md:449); this is new plumbing around the same per-head computation.

Gather layout: results are assembled in a head-major buffer [world*per, B, ...]
(per = ceil(H / world)) and returned as the [B, H, ...] view of it, so a rank
whose slice is already head-major (``head_major_empty``) sends without a copy
and nobody copies after the collective.  ``sharded_apply(chunks=c)`` computes
the local heads in c slices and gathers slice i (one NCCL broadcast per rank,
straight into its place in the final buffer, asynchronous on the process
group's stream) while slice i+1 computes.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple


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


def head_major_empty(B: int, H: int, *rest, dtype=None, device=None):
    """An empty [B, H, *rest] tensor stored head-major ([H, B, *rest] memory):
    the kernels write any 16-byte-aligned strides, and gather_heads sends it
    without a copy."""
    import torch
    return torch.empty((H, B) + tuple(rest), dtype=dtype, device=device).transpose(0, 1)


def _head_major(x, dim: int):
    """[H_loc, ...] head-major view of ``x``; copies only if it is not already head-major."""
    y = x.movedim(dim, 0)
    return y if y.is_contiguous() else y.contiguous()


def gather_heads(local, num_heads: int, group=None, dim: int = 1):
    """Gather per-rank head slices back into the full tensor (head dim ``dim``).

    One uniform ``all_gather_into_tensor`` (ranks short of ceil(H / world)
    heads pad their send buffer); the result is a view of the head-major
    receive buffer, not a copy."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = (num_heads + world - 1) // world
    x = _head_major(local, dim)
    if x.shape[0] < per:
        pad = torch.zeros((per,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[: x.shape[0]] = x
        x = pad
    out = torch.empty((per * world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if hasattr(dist, "all_gather_into_tensor") and out.device.type == "cuda":
        dist.all_gather_into_tensor(out, x, group=group)
    else:
        dist.all_gather(list(out.chunk(world, 0)), x, group=group)
    return out[:num_heads].movedim(0, dim)


def _default_head_args(tensors, num_heads: int):
    # only [B, H, L, C] tensors are sharded by default: a 2-D [N, R] factor whose
    # rank happens to equal H must never be split by columns
    return [i for i, t in enumerate(tensors) if t is not None and hasattr(t, "dim") and t.dim() == 4
            and t.shape[1] == num_heads]


def sharded_apply(fn: Callable, tensors: Sequence, num_heads: int, group=None, gather: bool = True,
                  head_args: Optional[Sequence[int]] = None, chunks: int = 1):
    """Run ``fn`` on this rank's head slice of the tensors listed in
    ``head_args`` (indices into ``tensors``; default: every 4-D [B, H, L, C]
    tensor with H == num_heads) and optionally gather the [B, H, ...] result.

    ``fn`` is the hot path (e.g. a ``flashbias_attention`` closure); no
    collective runs inside it.  ``chunks`` > 1 splits the local heads into
    slices and overlaps the gather of each slice with the compute of the next.
    A rank whose range is empty calls ``fn`` on zero-head slices (the API
    returns empty outputs for them without a launch) and contributes padding."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    idx = set(_default_head_args(tensors, num_heads) if head_args is None else head_args)
    lo, hi = head_range(num_heads, world, rank)
    if world == 1 or not gather:
        local = [t.narrow(1, lo, hi - lo) if i in idx else t for i, t in enumerate(tensors)]
        return fn(*local)
    if chunks <= 1:
        local = [t.narrow(1, lo, hi - lo) if i in idx else t for i, t in enumerate(tensors)]
        return gather_heads(fn(*local), num_heads, group)
    return _gather_chunked(fn, tensors, idx, num_heads, world, rank, group, chunks)


def _gather_chunked(fn, tensors, idx, num_heads, world, rank, group, chunks):
    """Chunked compute + gather: slice c of every rank lands in its final place
    (head-major buffer [world, per, ...]) by one async broadcast per source rank."""
    import torch
    import torch.distributed as dist

    per = (num_heads + world - 1) // world
    bounds = [(per * c // chunks, per * (c + 1) // chunks) for c in range(chunks)]
    bounds = [(a, b) for a, b in bounds if b > a]
    buf, works = None, []
    for a, b in bounds:
        # every rank computes the same relative slice [a, b) of its own range (empty past its end)
        local = []
        for i, t in enumerate(tensors):
            if i in idx:
                lo, hi = head_range(num_heads, world, rank)
                s, e = min(lo + a, hi), min(lo + b, hi)
                t = t.narrow(1, s, e - s)
            local.append(t)
        out = fn(*local)
        x = _head_major(out, 1)
        if buf is None:
            buf = torch.empty((world, per) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        if x.shape[0]:
            buf[rank, a:a + x.shape[0]].copy_(x)
        for src in range(world):
            works.append(dist.broadcast(buf[src, a:b], src=src, group=group, async_op=True))
    for w in works:
        w.wait()
    return buf.reshape((world * per,) + tuple(buf.shape[2:]))[:num_heads].movedim(0, 1)
