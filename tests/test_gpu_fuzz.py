"""Seeded random sweep of the public API against a torch float64 reference:
shapes (ragged N/M, B/H, head dims 32/64/128 and non-power-of-two dims that
get zero-padded), factor ranks and broadcast patterns, masks, dtypes, static vs
learnable factors, dense bias — forward and backward.  Catches interactions the
hand-picked cases in test_gpu_kernels.py do not enumerate."""

import math
import random

import pytest
import torch

import paper_2505_12044_b200 as fb

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _ref(q, k, v, fq, fk, bias, causal):
    s = q.double() @ k.double().transpose(-1, -2) / math.sqrt(q.shape[-1])
    if fq is not None:
        s = s + fq.double() @ fk.double().transpose(-1, -2)
    if bias is not None:
        s = s + bias.double()
    if causal:
        m = torch.ones(s.shape[-2], s.shape[-1], dtype=torch.bool, device=s.device).triu(1)
        s = s.masked_fill(m, float("-inf"))
    return torch.softmax(s, -1) @ v.double()


def _relerr(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-12)).item()


def _case(seed):
    rnd = random.Random(seed)
    causal = rnd.random() < 0.4
    n = rnd.choice([64, 128, 200, 256, 320, 384, 512])
    m = n if causal else rnd.choice([96, 128, 250, 256, 333, 512])
    d = rnd.choice([32, 64, 128, 48, 80])
    B, H = rnd.choice([1, 2]), rnd.choice([1, 2, 3])
    kind = rnd.choice(["factored", "factored", "factored", "dense", "none"])
    r = rnd.choice([1, 2, 4, 9, 16])
    learn = kind == "factored" and rnd.random() < 0.4
    dtype = rnd.choice([torch.bfloat16, torch.bfloat16, torch.float16])
    fb_b = rnd.choice([1, B])
    fb_h = rnd.choice([1, H])
    return dict(causal=causal, n=n, m=m, d=d, B=B, H=H, kind=kind, r=r, learn=learn, dtype=dtype,
                fb_b=fb_b, fb_h=fb_h)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("FB_FUZZ_CASES", "60"))))
def test_random_case(seed):
    c = _case(seed)
    g = torch.Generator(device="cuda").manual_seed(1000 + seed)
    q = torch.randn(c["B"], c["H"], c["n"], c["d"], device="cuda", generator=g).to(c["dtype"])
    k = torch.randn(c["B"], c["H"], c["m"], c["d"], device="cuda", generator=g).to(c["dtype"])
    v = torch.randn(c["B"], c["H"], c["m"], c["d"], device="cuda", generator=g).to(c["dtype"])
    do = torch.randn(c["B"], c["H"], c["n"], c["d"], device="cuda", generator=g).to(c["dtype"])
    for t in (q, k, v):
        t.requires_grad_(True)
    fq = fk = bias = None
    mask = "causal" if c["causal"] else "none"
    if c["kind"] == "factored":
        fq = torch.randn(c["fb_b"], c["fb_h"], c["n"], c["r"], device="cuda", generator=g) * 0.5
        fk = torch.randn(c["fb_b"], c["fb_h"], c["m"], c["r"], device="cuda", generator=g) * 0.5
        if c["learn"]:
            fq.requires_grad_(True)
            fk.requires_grad_(True)
        out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    elif c["kind"] == "dense":
        bias = (torch.randn(1, c["H"], c["n"], c["m"], device="cuda", generator=g) * 2).to(c["dtype"])
        out = fb.tiled_attention(q, k, v, fb.DenseBias(bias), mask=mask)
    else:
        out = fb.tiled_attention(q, k, v, mask=mask)
    assert out.dtype == c["dtype"] and out.shape == q.shape, c
    leaves = [q, k, v] + ([fq, fk] if c["learn"] else [])
    grads = torch.autograd.grad(out, leaves, do)
    ref_leaves = [t.detach().double().requires_grad_(True) for t in leaves]
    rq, rk, rv = ref_leaves[:3]
    rfq = ref_leaves[3] if c["learn"] else (fq.double() if fq is not None else None)
    rfk = ref_leaves[4] if c["learn"] else (fk.double() if fk is not None else None)
    ref = _ref(rq, rk, rv, rfq, rfk, bias, c["causal"])
    assert _relerr(out, ref) < TOL, ("o", c)
    rgrads = torch.autograd.grad(ref, ref_leaves, do.double())
    for name, a, b in zip(["dq", "dk", "dv", "dfq", "dfk"], grads, rgrads):
        e = _relerr(a, b)
        assert e < TOL, (name, e, c)
