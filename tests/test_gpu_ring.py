"""Ring FlashBias (§8(f)-4) with the CUDA kernels: G virtual ranks as threads on
one B200 (ThreadRing) run the real ring schedule -- rotating K / V / factor
panels, merging partial outputs by LSE, carrying dK / dV / panel gradients
home -- against the float64 oracle of the whole sequence; and the autograd
wrapper on the one-rank ring equals the single-call API exactly."""

import math

import pytest
import torch

import paper_2505_12044_b200 as fb
from oracle import flashbias_oracle as orc
from paper_2505_12044_b200 import attention as A
from paper_2505_12044_b200.ring import SoloRing, ThreadRing, _kernel_bwd, _kernel_fwd, ring_backward, ring_forward

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _np(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("G,D,mask", [(2, 128, "causal"), (4, 128, "causal"), (2, 64, "none"), (3, 64, "causal")])
def test_thread_ring_matches_oracle(G, D, mask):
    Nc, H = 256, 2
    N = Nc * G
    g = torch.Generator(device="cuda").manual_seed(G * 10 + D)
    q, k, v, do = (torch.randn(1, H, N, D, generator=g, device="cuda").bfloat16() for _ in range(4))
    # well-conditioned learnable factors (ALiBi's position-sized factor gradients cancel to ~0 and are not a
    # meaningful bf16 parity target); each chunk keeps its own rows' factors, which travel with K
    fq = (torch.randn(1, H, N, 8, generator=g, device="cuda") * 0.4).contiguous()
    fk = (torch.randn(1, H, N, 8, generator=g, device="cuda") * 0.4).contiguous()
    scale = 1 / math.sqrt(D)
    outs = {}

    def rank_fn(comm):
        sl = slice(comm.rank * Nc, (comm.rank + 1) * Nc)
        fq_r, fk_r = fq[:, :, sl].contiguous(), fk[:, :, sl].contiguous()
        plan = A.plan_factor_fold(fq_r, fk_r, scale, max_cols=64 if D == 128 else 128, shard_invariant=True)
        uq, uk = A.prepare_factor_panels(fq_r, fk_r, plan.premul, plan.split, torch.bfloat16)
        qr, kr, vr, dor = (t[:, :, sl].contiguous() for t in (q, k, v, do))
        if plan.q_fold:
            qr = (qr * scale).to(torch.bfloat16)
        o32, lse = ring_forward(comm, qr, kr, vr, uq, uk, mask, plan.kernel_scale, _kernel_fwd(plan.kernel_scale))
        o = o32.to(torch.bfloat16)
        dq, dk, dv, duq, duk = ring_backward(comm, qr, kr, vr, uq, uk, o, lse.contiguous(), dor, mask,
                                             plan.kernel_scale, _kernel_bwd(plan.kernel_scale), True)
        if plan.q_fold:
            dq = dq * scale
        dfq = A.fold_factor_grads(duq, fq_r, 0, plan.split, plan.premul)
        dfk = A.fold_factor_grads(duk, fk_r, 1, plan.split, 1.0)
        torch.cuda.synchronize()
        outs[comm.rank] = dict(o=o, dq=dq, dk=dk, dv=dv, dfq=dfq, dfk=dfk)

    ThreadRing(G).run(rank_fn)
    fq64, fk64 = _np(fq), _np(fk)
    for h in range(H):
        ref = orc.blocked_attention_fwd_bwd(_np(q[0, h]), _np(k[0, h]), _np(v[0, h]), _np(do[0, h]),
                                            fq=fq64[0, h], fk=fk64[0, h], premul=math.sqrt(D), mask=mask,
                                            scale=scale)
        for key in ("o", "dq", "dk", "dv", "dfq", "dfk"):
            got = torch.cat([outs[r][key][0, h] for r in range(G)], 0)
            err = orc.rel_max_err(_np(got), ref[key])
            assert err < TOL, (G, D, mask, h, key, err)


def test_ring_autograd_on_one_rank_equals_single_call():
    N, H, D = 384, 2, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, do = (torch.randn(2, H, N, D, generator=g, device="cuda").bfloat16() for _ in range(4))
    fq = (torch.randn(1, H, N, 4, generator=g, device="cuda") * 0.4).contiguous()
    fk = (torch.randn(1, H, N, 4, generator=g, device="cuda") * 0.4).contiguous()
    res = []
    for ring in (True, False):
        qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
        f1, f2 = fq.clone().requires_grad_(True), fk.clone().requires_grad_(True)
        o = (fb.ring_flashbias_attention(qq, kk, vv, f1, f2, mask="causal", comm=SoloRing()) if ring
             else fb.flashbias_attention(qq, kk, vv, f1, f2, mask="causal"))
        res.append([o.detach()] + list(torch.autograd.grad(o, (qq, kk, vv, f1, f2), do)))
    # same kernels; the ring plans its factor split from the rank alone (shard-invariant), so the two
    # paths may use different split levels: agreement at the bf16 level, not bitwise
    for name, a, b in zip(("o", "dq", "dk", "dv", "dfq", "dfk"), *res):
        err = float((a.double() - b.double()).abs().max() / b.double().abs().max())
        assert err < TOL, (name, err)
