"""Context-parallel ring FlashBias (§8(f)-4) on CPU ranks (gloo, world 2 and 3):
the ring schedule (chunk rotation, LSE merge, travelling dK/dV/dfk
accumulators, causal chunk skipping) with the float64 oracle as the chunk
kernel must reproduce the unsharded oracle's output and gradients."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mask, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import flashbias_oracle as orc
    from paper_2505_12044_b200.ring import DistRing, ring_backward, ring_forward
    n_c, d, r = 24, 8, 3
    n = n_c * world
    g = torch.Generator().manual_seed(11)
    q, k, v, do = (torch.randn(n, d, generator=g, dtype=torch.float64) for _ in range(4))
    fq, fk = torch.randn(n, r, generator=g, dtype=torch.float64), torch.randn(n, r, generator=g, dtype=torch.float64)
    prem, scale = math.sqrt(d), 1.0 / math.sqrt(d)
    sl = slice(rank * n_c, (rank + 1) * n_c)

    def fwd(qc, kc, vc, uq, uk, m):
        o, lse = orc.streaming_attention(qc.numpy(), kc.numpy(), vc.numpy(), fq=uq.numpy(), fk=uk.numpy(),
                                         premul=1.0, mask=m, scale=scale)
        return torch.from_numpy(o), torch.from_numpy(lse)

    def bwd(qc, kc, vc, uq, uk, o, lse, doc, m, want):
        res = orc.chunk_attention_bwd(qc.numpy(), kc.numpy(), vc.numpy(), doc.numpy(), o.numpy(), lse.numpy(),
                                      fq=uq.numpy(), fk=uk.numpy(), premul=1.0, mask=m, scale=scale)
        t = {key: torch.from_numpy(np.ascontiguousarray(val)) for key, val in res.items()}
        # panel gradients: d/d(uq) and d/d(uk) of scale * uq.uk
        return t["dq"], t["dk"], t["dv"], t["dfq"], t["dfk"]

    comm = DistRing()
    o, lse = ring_forward(comm, q[sl], k[sl], v[sl], fq[sl] * prem, fk[sl], mask, scale, fwd)
    dq, dk, dv, duq, duk = ring_backward(comm, q[sl], k[sl], v[sl], fq[sl] * prem, fk[sl], o, lse, do[sl], mask,
                                         scale, bwd, True)
    ref_o, _ = orc.streaming_attention(q.numpy(), k.numpy(), v.numpy(), fq=fq.numpy(), fk=fk.numpy(), premul=prem,
                                       mask=mask, scale=scale)
    ref = orc.attention_bwd(q.numpy(), k.numpy(), v.numpy(), do.numpy(), fq=fq.numpy(), fk=fk.numpy(), premul=prem,
                            mask=mask, scale=scale)
    errs = {
        "o": orc.rel_max_err(o.numpy(), ref_o[sl]),
        "dq": orc.rel_max_err(dq.numpy(), ref["dq"][sl]),
        "dk": orc.rel_max_err(dk.numpy(), ref["dk"][sl]),
        "dv": orc.rel_max_err(dv.numpy(), ref["dv"][sl]),
        "dfq": orc.rel_max_err(duq.numpy() * prem, ref["dfq"][sl]),
        "dfk": orc.rel_max_err(duk.numpy(), ref["dfk"][sl]),
    }
    torch.save(errs, f"{path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_ring_schedule_matches_unsharded_oracle(tmp_path, world, mask):
    path = str(tmp_path / "errs")
    mp.spawn(_worker, args=(world, _free_port(), mask, path), nprocs=world, join=True)
    for r in range(world):
        errs = torch.load(f"{path}.{r}")
        assert max(errs.values()) < 1e-12, (r, errs)
