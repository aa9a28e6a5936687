"""Context-parallel ring FlashBias: sequences longer than one
GPU, split into G contiguous chunks, one per rank.

Each rank keeps its query chunk (q, fq) and passes its key chunk around the
ring: at step s it holds the K/V chunk of rank (r - s) mod G, together with
that chunk's factor panel uk = split(fk) -- the bias factor travels with K for
free (Eq. 3: the bias is part of the widened K' = [K | fk]), where a
dense bias would need an N x M tile per step.  The transfer of the next chunk
is posted before the current chunk's kernels run, so NVLink traffic overlaps
the tensor-core work.

Forward: per step the FlashBias kernel (fb_attn_fwd) returns the chunk's
normalised output and log-sum-exp; partials merge exactly by
O = sum_s exp(lse_s - lse) O_s, lse = logsumexp_s lse_s (the reference's
online-softmax recurrence, attention.py:174-201, applied across chunks).
Backward: per step fb_attn_bwd runs with the GLOBAL O and LSE, which makes
its P = exp(S - lse) and D = rowsum(dO * O) exact for the chunk pair, so dQ
sums over the visited chunks locally while dK / dV / dfk (and the factor
panel gradient) travel with their chunk and return home after G hops.
Causal masks (N == M, equal chunks): the diagonal chunk is causal, chunks
from later ranks are skipped, earlier ones are unmasked.

The reference has no distribution; the per-chunk arithmetic is
the single-GPU kernels'.  Transports: ``DistRing`` (torch.distributed P2P:
NCCL over NVLink, gloo on CPU) and ``ThreadRing`` (G ranks as threads of one
process on one device: tests and single-GPU runs).
"""

from __future__ import annotations

import math
import threading
from typing import Callable, List, Optional, Sequence

from .errors import ConfigError, MaskError, ShapeError

__all__ = ["DistRing", "SoloRing", "ThreadRing", "ring_flashbias_attention", "ring_forward", "ring_backward"]


class DistRing:
    """Ring over a torch.distributed group: rotate() sends to rank + 1 and
    receives from rank - 1 with batched isend / irecv (asynchronous)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def rotate(self, tensors: Sequence):
        import torch
        dist = self.dist
        nxt = dist.get_global_rank(self.group, (self.rank + 1) % self.world) if self.group else \
            (self.rank + 1) % self.world
        prv = dist.get_global_rank(self.group, (self.rank - 1) % self.world) if self.group else \
            (self.rank - 1) % self.world
        recv = [torch.empty_like(t) for t in tensors]
        ops = []
        for t, r in zip(tensors, recv):  # even ranks send first, odd ranks receive first (no cycle stall)
            send, rcv = dist.P2POp(dist.isend, t.contiguous(), nxt, self.group), \
                dist.P2POp(dist.irecv, r, prv, self.group)
            ops += [send, rcv] if self.rank % 2 == 0 else [rcv, send]
        reqs = dist.batch_isend_irecv(ops)

        def wait():
            for q in reqs:
                q.wait()
            return recv
        return wait


class SoloRing:
    """The trivial ring of one rank (the whole sequence on this GPU)."""

    rank, world = 0, 1

    def rotate(self, tensors: Sequence):
        return lambda: list(tensors)


class ThreadRing:
    """G virtual ranks as threads of one process (one device): ``run(fn)``
    calls fn(comm) on every rank concurrently; rotate() exchanges through
    shared slots between barriers.  Same interface as DistRing."""

    def __init__(self, world: int):
        self.world = world
        self._slots: List = [None] * world
        self._barrier = threading.Barrier(world)

    def run(self, fn: Callable):
        out, err = [None] * self.world, []

        def body(r):
            try:
                out[r] = fn(_ThreadRank(self, r))
            except BaseException as e:  # noqa: BLE001 - re-raised on the caller's thread
                err.append(e)
                self._barrier.abort()
        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        return out


class _ThreadRank:
    def __init__(self, ring: ThreadRing, rank: int):
        self.ring, self.rank, self.world = ring, rank, ring.world

    def rotate(self, tensors: Sequence):
        import torch
        ring = self.ring
        if torch.cuda.is_available():
            torch.cuda.synchronize()  # producers' kernels done before a peer thread reads the tensors
        ring._barrier.wait()
        ring._slots[self.rank] = [t.clone() for t in tensors]
        ring._barrier.wait()
        recv = ring._slots[(self.rank - 1) % self.world]
        ring._barrier.wait()
        return lambda: recv


def _acc_dtype(t):
    """Accumulators: fp32 for the bf16/fp16 kernels, the input precision above that."""
    import torch
    return torch.float64 if t.dtype == torch.float64 else torch.float32


def _merge(o_acc, lse_acc, o_s, lse_s):
    """Exact merge of two normalised partial outputs by their log-sum-exps."""
    import torch
    dt = _acc_dtype(o_s)
    if o_acc is None:
        return o_s.to(dt), lse_s.to(dt)
    lse = torch.logaddexp(lse_acc, lse_s.to(dt))
    w_a = torch.exp(lse_acc - lse).nan_to_num_(0.0)
    w_s = torch.exp(lse_s.to(dt) - lse).nan_to_num_(0.0)
    return o_acc * w_a[..., None] + o_s.to(dt) * w_s[..., None], lse


def _chunk_mask(mask: str, rank: int, src: int) -> Optional[str]:
    """Mask of the (query chunk = rank, key chunk = src) pair; None = skip."""
    if mask != "causal":
        return "none"
    if src > rank:
        return None
    return "causal" if src == rank else "none"


def ring_forward(comm, q, k, v, uq, uk, mask: str, scale: float, fwd: Callable):
    """Per-rank forward: returns (O, LSE) of this rank's query chunk (fp32, or fp64 for fp64 inputs).
    fwd(q, k, v, uq, uk, mask) -> (o, lse) is the chunk kernel."""
    o_acc = lse_acc = None
    cur = [k, v] + ([uk] if uk is not None else [])
    for s in range(comm.world):
        src = (comm.rank - s) % comm.world
        pending = comm.rotate(cur) if s + 1 < comm.world else None  # next chunk in flight during this step
        m = _chunk_mask(mask, comm.rank, src)
        if m is not None:
            o_s, lse_s = fwd(q, cur[0], cur[1], uq, cur[2] if uk is not None else None, m)
            o_acc, lse_acc = _merge(o_acc, lse_acc, o_s, lse_s)
        if pending is not None:
            cur = pending()
    return o_acc, lse_acc


def ring_backward(comm, q, k, v, uq, uk, o, lse, do, mask: str, scale: float, bwd: Callable, want_fgrad: bool):
    """Per-rank backward with the global O / LSE: returns dq, dk, dv and the
    factor-panel gradients duq, duk (or None), accumulated in fp32 (fp64 inputs: fp64).  bwd(q, k, v, uq, uk,
    o, lse, do, mask, want_fgrad) -> (dq, dk, dv, duq, duk) is the chunk kernel."""
    import torch
    dt = _acc_dtype(q)
    dq = torch.zeros(q.shape, dtype=dt, device=q.device)
    duq = None
    # the K-side state that circulates: K, V (, uk) and their gradient accumulators
    acc = [torch.zeros(k.shape, dtype=dt, device=k.device), torch.zeros(v.shape, dtype=dt, device=v.device)]
    if want_fgrad and uk is not None:
        acc.append(torch.zeros(tuple(q.shape[:-2]) + (k.shape[-2], uk.shape[-1]), dtype=dt,
                               device=k.device))  # per (b, h): the kernel's panel gradients are not batch-reduced
    data = [k, v] + ([uk] if uk is not None else [])
    nd = len(data)
    for s in range(comm.world):
        src = (comm.rank - s) % comm.world
        m = _chunk_mask(mask, comm.rank, src)
        if m is not None:
            g_q, g_k, g_v, g_uq, g_uk = bwd(q, data[0], data[1], uq, data[2] if uk is not None else None,
                                           o, lse, do, m, want_fgrad)
            dq += g_q.to(dt)
            acc[0] += g_k.to(dt)
            acc[1] += g_v.to(dt)
            if want_fgrad and uk is not None:
                duq = g_uq if duq is None else duq + g_uq
                acc[2] += g_uk
        # every hop moves K/V/uk (needed next step) and the accumulators; after G hops they are home
        if comm.world > 1:
            moved = comm.rotate(data + acc)()
            data, acc = moved[:nd], moved[nd:]
    return dq, acc[0], acc[1], duq, (acc[2] if len(acc) > 2 else None)


def _kernel_fwd(scale):
    from .attention import _fwd_launch

    def fwd(q, k, v, uq, uk, m):
        return _fwd_launch(q, k, v, uq, uk, None, 1 if m == "causal" else 0, scale)
    return fwd


def _kernel_bwd(scale):
    from .attention import _bwd_launch

    def bwd(q, k, v, uq, uk, o, lse, do, m, want_fgrad):
        dq, dk, dv, duq, duk, _ = _bwd_launch(q, k, v, uq, uk, None, o, lse, do, 1 if m == "causal" else 0,
                                              scale, want_fgrad)
        return dq, dk, dv, duq, duk
    return bwd


def ring_flashbias_attention(q, k, v, fq, fk, mask: str = "none", group=None, comm=None):
    """flashbias_attention (ref attention.py:205-230) over a sequence split
    across the ranks of ``group`` (or an explicit ring ``comm``).

    Per rank: q [B,H,Nc,C] bf16/fp16 (this rank's query rows), k, v [B,H,Mc,C]
    (this rank's key rows), fq [Bf,Hf,Nc,R] / fk [Bf,Hf,Mc,R] with the factors
    of the GLOBAL positions of those rows.  Returns this rank's output rows,
    autograd-enabled (dq, dk, dv, dfq, dfk of the local chunks)."""
    import torch

    from . import attention as A
    if comm is None:
        comm = DistRing(group)
    if q.dtype not in (torch.bfloat16, torch.float16) or not q.is_cuda:
        raise ConfigError("ring_flashbias_attention runs the tcgen05 kernels: bf16/fp16 CUDA tensors")
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise ShapeError("ring_flashbias_attention takes [B, H, L, C] chunks")
    if mask not in ("none", "causal"):
        raise MaskError(f"unknown mask {mask!r}")
    if mask == "causal" and q.shape[2] != k.shape[2]:
        raise MaskError("causal ring attention needs equal query and key chunks")
    c = int(q.shape[-1])
    scale = 1.0 / math.sqrt(c)
    dp = A._padded_head_dim(c)
    # a split level that depends on R alone, so every rank builds panels of the same width
    plan = A.plan_factor_fold(fq, fk, scale, max_cols=64 if dp == 128 else 128, panel_dtype=q.dtype,
                              shard_invariant=True)
    fn = _ring_fn()
    return fn.apply(q, k, v, fq, fk, comm, mask, plan, dp)[..., :c]


_RING_FN = None


def _ring_fn():
    global _RING_FN
    if _RING_FN is not None:
        return _RING_FN
    import torch

    from . import attention as A

    class RingFunction(torch.autograd.Function):
        @staticmethod
        def forward(ctx, q, k, v, fq, fk, comm, mask, plan, dp):
            qp, kp, vp = (A._pad_last(t, dp) for t in (q, k, v))
            if plan.q_fold:
                qp = (qp * (1.0 / math.sqrt(q.shape[-1]))).to(q.dtype)
            uq, uk = A.prepare_factor_panels(fq, fk, plan.premul, plan.split, q.dtype)
            o32, lse = ring_forward(comm, qp, kp, vp, uq, uk, mask, plan.kernel_scale,
                                    _kernel_fwd(plan.kernel_scale))
            o = o32.to(q.dtype)
            ctx.save_for_backward(qp, kp, vp, uq, uk, o, lse.contiguous(), fq, fk)
            ctx.cfg = (comm, mask, plan, q.shape[-1])
            return o

        @staticmethod
        def backward(ctx, do):
            qp, kp, vp, uq, uk, o, lse, fq, fk = ctx.saved_tensors
            comm, mask, plan, c = ctx.cfg
            want_fg = ctx.needs_input_grad[3] or ctx.needs_input_grad[4]
            dop = A._pad_last(do.contiguous(), qp.shape[-1])
            dq, dk, dv, duq, duk = ring_backward(comm, qp, kp, vp, uq, uk, o, lse, dop, mask, plan.kernel_scale,
                                                 _kernel_bwd(plan.kernel_scale), want_fg)
            if plan.q_fold:  # Q' = scale * q
                dq = dq * (1.0 / math.sqrt(c))
            dfq = dfk = None
            if want_fg:
                dfq = A.fold_factor_grads(duq, fq, 0, plan.split, plan.premul).to(fq.dtype)
                dfk = A.fold_factor_grads(duk, fk, 1, plan.split, 1.0).to(fk.dtype)
            c_ = c
            return (dq[..., :c_].to(qp.dtype), dk[..., :c_].to(kp.dtype), dv[..., :c_].to(vp.dtype), dfq, dfk,
                    None, None, None, None)

    _RING_FN = RingFunction
    return _RING_FN
