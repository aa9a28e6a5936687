"""B x H sharding on 2 CPU ranks (gloo): per-rank head slices computed with the
oracle and all-gathered must equal the unsharded result bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_12044_b200.sharding import gather_heads, head_range, sharded_apply


def test_head_range_partitions():
    for h in (1, 7, 32):
        for w in (1, 2, 3, 8):
            spans = [head_range(h, w, r) for r in range(w)]
            covered = [i for lo, hi in spans for i in range(lo, hi)]
            assert covered == list(range(h))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import flashbias_oracle as orc
    g = torch.Generator().manual_seed(0)
    B, H, N, d, R = 2, 5, 40, 8, 3
    q, k, v = (torch.randn(B, H, N, d, generator=g, dtype=torch.float64) for _ in range(3))
    fq = torch.randn(1, H, N, R, generator=g, dtype=torch.float64)
    fk = torch.randn(1, H, N, R, generator=g, dtype=torch.float64)

    def hot(qs, ks, vs, fqs, fks):
        o = orc.flashbias_attention(qs.numpy(), ks.numpy(), vs.numpy(), fqs.numpy(), fks.numpy(), mask="causal")
        return torch.from_numpy(np.ascontiguousarray(o))

    full = sharded_apply(hot, [q, k, v, fq, fk], H)
    if rank == 0:
        ref = hot(q, k, v, fq, fk)
        torch.save({"eq": bool(torch.equal(full, ref)), "shape": tuple(full.shape)}, result_path)
    # gather of a ragged split (H=5 over 2 ranks -> 3 + 2 heads)
    lo, hi = head_range(H, world, rank)
    part = torch.full((B, hi - lo, 2), float(rank))
    allp = gather_heads(part, H)
    # gradients shard the same way: every rank computes dq/dk/dv/dfq/dfk of its own heads
    do = torch.randn(B, H, N, d, generator=g, dtype=torch.float64)

    def grads(qs, ks, vs, dos, fqs, fks):
        r = orc.attention_bwd(qs.numpy(), ks.numpy(), vs.numpy(), dos.numpy(), fq=fqs.numpy(), fk=fks.numpy(),
                              premul=np.sqrt(d), mask="causal")
        return torch.from_numpy(np.stack([r["dq"], r["dk"], r["dv"]], 2))  # [B, H, 3, N, d]

    gfull = sharded_apply(grads, [q, k, v, do, fq, fk], H)
    gref = grads(q, k, v, do, fq, fk)
    # chunked compute + gather (slices land in place by per-rank broadcasts) == unchunked
    chunked = sharded_apply(hot, [q, k, v, fq, fk], H, chunks=2)
    # a 2-D [N, R] factor with R == H is shared, never split by columns
    shared = torch.randn(N, H, generator=g, dtype=torch.float64)
    got2d = sharded_apply(lambda a, f: a.sum(-1, keepdim=True) + f.sum(), [q, shared], H)
    # H < world: the empty rank still takes part in the gather
    one = sharded_apply(lambda a: a * 2, [q[:, :1]], 1)
    if rank == 0:
        res = torch.load(result_path)
        res["ragged"] = allp[0, :, 0].tolist()
        res["chunked_eq"] = bool(torch.equal(chunked, full))
        res["shared_eq"] = bool(torch.equal(got2d, q.sum(-1, keepdim=True) + shared.sum()))
        res["one_eq"] = bool(torch.equal(one, q[:, :1] * 2))
        res["grads_eq"] = bool(torch.equal(gfull, gref))
        torch.save(res, result_path)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_equals_unsharded_gloo(tmp_path):
    path = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    res = torch.load(path)
    assert res["eq"] and res["shape"] == (2, 5, 40, 8)
    assert res["ragged"] == [0.0, 0.0, 0.0, 1.0, 1.0]
    assert res["chunked_eq"] and res["shared_eq"] and res["one_eq"] and res["grads_eq"]
