"""GPU numerics of the sm_100a kernels against a plain torch float64 reference
of the same op (materialised softmax).  Tolerances are the north-star ones:
bf16/fp16 2e-2 relative (max-abs / max|ref|), fp32 1e-5 relative."""

import math

import pytest
import torch

import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import attention as A

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
F32_TOL = 1e-5


def ref_attention(q, k, v, fq=None, fk=None, bias=None, causal=False, scale=None):
    qd, kd, vd = q.double(), k.double(), v.double()
    scale = scale if scale is not None else 1.0 / math.sqrt(q.shape[-1])
    s = qd @ kd.transpose(-1, -2) * scale
    if fq is not None:
        s = s + fq.double() @ fk.double().transpose(-1, -2)
    if bias is not None:
        s = s + bias.double()
    if causal:
        m = torch.ones(s.shape[-2], s.shape[-1], dtype=torch.bool, device=s.device).triu(1)
        s = s.masked_fill(m, float("-inf"))
    return torch.softmax(s, -1) @ vd


def relerr(a, b):
    a, b = a.detach().double(), b.detach().double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def _qkv(B, H, N, M, D, dtype, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn(B, H, N, D, device="cuda", generator=g).to(dtype)
    k = torch.randn(B, H, M, D, device="cuda", generator=g).to(dtype)
    v = torch.randn(B, H, M, D, device="cuda", generator=g).to(dtype)
    return q, k, v


@pytest.mark.parametrize("D", [32, 64, 128])
@pytest.mark.parametrize("N,M,causal", [(256, 256, False), (384, 384, True), (200, 333, False), (77, 77, True)])
def test_fwd_nobias(D, N, M, causal):
    q, k, v = _qkv(2, 3, N, M, D, torch.bfloat16)
    out = fb.tiled_attention(q, k, v, mask="causal" if causal else "none")
    ref = ref_attention(q, k, v, causal=causal)
    assert out.dtype == torch.bfloat16 and out.shape == q.shape
    assert relerr(out, ref) < BF16_TOL


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("R", [2, 9, 16, 64])
@pytest.mark.parametrize("causal", [False, True])
def test_fwd_factored(D, R, causal):
    N = 384
    q, k, v = _qkv(1, 2, N, N, D, torch.bfloat16, seed=R)
    g = torch.Generator(device="cuda").manual_seed(100 + R)
    fq = torch.randn(1, 2, N, R, device="cuda", generator=g) * 0.5
    fk = torch.randn(1, 2, N, R, device="cuda", generator=g) * 0.5
    if R == 64:  # rank 64 only fits unsplit panels: feed bf16-exact factors
        fq, fk = fq.bfloat16().float(), fk.bfloat16().float()
    out = fb.flashbias_attention(q, k, v, fq, fk, mask="causal" if causal else "none")
    ref = ref_attention(q, k, v, fq, fk, causal=causal)
    assert relerr(out, ref) < BF16_TOL


def test_fwd_alibi_long_split():
    N, H = 2048, 4
    q, k, v = _qkv(1, H, N, N, 128, torch.bfloat16, seed=5)
    slopes = [-(2.0 ** (-8.0 * (h + 1) / H)) for h in range(H)]
    fq, fk = fb.alibi_factors(slopes, N, N)
    out = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
    i = torch.arange(1, N + 1, device="cuda", dtype=torch.float64)
    dense = torch.tensor(slopes, device="cuda", dtype=torch.float64)[:, None, None] * (i[:, None] - i[None, :])
    ref = ref_attention(q, k, v, bias=dense[None], causal=True)
    assert relerr(out, ref) < BF16_TOL


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_fwd_dense_bias(D, causal):
    N = 320
    q, k, v = _qkv(2, 2, N, N, D, torch.bfloat16, seed=9)
    bias = (torch.randn(1, 2, N, N, device="cuda") * 2).bfloat16()
    out = fb.tiled_attention(q, k, v, fb.DenseBias(bias), mask="causal" if causal else "none")
    ref = ref_attention(q, k, v, bias=bias, causal=causal)
    assert relerr(out, ref) < BF16_TOL


def test_fwd_fp16():
    q, k, v = _qkv(1, 2, 256, 256, 64, torch.float16, seed=3)
    fq = torch.randn(1, 2, 256, 4, device="cuda")
    fk = torch.randn(1, 2, 256, 4, device="cuda")
    out = fb.flashbias_attention(q, k, v, fq, fk)
    assert relerr(out, ref_attention(q, k, v, fq, fk)) < BF16_TOL


@pytest.mark.parametrize("causal", [False, True])
def test_fwd_fp32_simt(causal):
    q, k, v = _qkv(1, 8, 1024, 1024, 64, torch.float32, seed=11)
    fq, fk = fb.alibi_factors([-(2.0 ** -(h + 1)) for h in range(8)], 1024, 1024)
    out = fb.flashbias_attention(q, k, v, fq, fk, mask="causal" if causal else "none")
    ref = ref_attention(q, k, v, fq, fk, causal=causal)
    assert out.dtype == torch.float32
    assert relerr(out, ref) < F32_TOL


@pytest.mark.parametrize("D", [32, 64, 128])
@pytest.mark.parametrize("N,M,causal", [(64, 64, False), (65, 130, False), (128, 128, True), (200, 200, False),
                                        (333, 333, True), (1000, 1000, False), (700, 2100, False)])
def test_fwd_fp32_simt_split_kv_shapes(D, N, M, causal):
    """The fp32 SIMT forward over the shapes that pick each split-KV cluster size (1/2/4/8 CTAs per row
    block) with one or several KV blocks per CTA, ragged tails, causal diagonals, factors and a dense
    bias; parity 1e-5 against torch float64."""
    H = 4
    q, k, v = _qkv(1, H, N, M, D, torch.float32, seed=N + M + D)
    fq = torch.randn(1, H, N, 2, device="cuda") * 0.5
    fk = torch.randn(1, H, M, 2, device="cuda") * 0.5
    mask = "causal" if causal else "none"
    out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    assert relerr(out, ref_attention(q, k, v, fq, fk, causal=causal)) < F32_TOL
    bias = torch.randn(1, H, N, M, device="cuda")
    out = fb.tiled_attention(q, k, v, fb.DenseBias(bias), mask=mask)
    assert relerr(out, ref_attention(q, k, v, bias=bias, causal=causal)) < F32_TOL


def test_many_heads_over_grid_y_limit():
    """B*H = 70000 planes (> the 65535 grid.y limit of the plane-indexed helper kernels: factor-panel
    split, backward preprocess): forward + backward with factors against torch float64 on sampled heads."""
    B, H, N, D = 2, 35000, 16, 64
    q, k, v = _qkv(B, H, N, N, D, torch.bfloat16, seed=5)
    for t in (q, k, v):
        t.requires_grad_(True)
    fq = torch.randn(B, H, N, 2, device="cuda") * 0.5
    fk = torch.randn(B, H, N, 2, device="cuda") * 0.5
    do = torch.randn(B, H, N, D, device="cuda").bfloat16()
    out = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
    out.backward(do)
    for b, h in ((0, 0), (1, 34999), (1, 30000)):
        qs, ks, vs = (t.detach()[b:b + 1, h:h + 1].double().requires_grad_(True) for t in (q, k, v))
        ref = ref_attention(qs, ks, vs, fq[b:b + 1, h:h + 1], fk[b:b + 1, h:h + 1], causal=True)
        assert relerr(out[b:b + 1, h:h + 1], ref) < BF16_TOL
        ref.backward(do[b:b + 1, h:h + 1].double())
        for got, t in ((q.grad, qs), (k.grad, ks), (v.grad, vs)):
            assert relerr(got[b:b + 1, h:h + 1], t.grad) < BF16_TOL


def _bwd_case(B, H, N, M, D, R, causal, dense=False, seed=0):
    q, k, v = _qkv(B, H, N, M, D, torch.bfloat16, seed=seed)
    q.requires_grad_(True)
    k.requires_grad_(True)
    v.requires_grad_(True)
    fq = fk = bias = None
    if R:
        g = torch.Generator(device="cuda").manual_seed(seed + 7)
        fq = (torch.randn(1, H, N, R, device="cuda", generator=g) * 0.5).requires_grad_(True)
        fk = (torch.randn(1, H, M, R, device="cuda", generator=g) * 0.5).requires_grad_(True)
    if dense:
        bias = (torch.randn(1, H, N, M, device="cuda") * 2).bfloat16()
    do = torch.randn(B, H, N, D, device="cuda").bfloat16()
    mask = "causal" if causal else "none"
    if R:
        out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    elif dense:
        out = fb.tiled_attention(q, k, v, fb.DenseBias(bias), mask=mask)
    else:
        out = fb.tiled_attention(q, k, v, mask=mask)
    out.backward(do)
    leaves = [q, k, v] + ([fq, fk] if R else [])
    got = [t.grad.clone() for t in leaves]
    ref_leaves = [t.detach().double().requires_grad_(True) for t in leaves]
    rq, rk, rv = ref_leaves[:3]
    rfq, rfk = (ref_leaves[3], ref_leaves[4]) if R else (None, None)
    ref = ref_attention(rq, rk, rv, rfq, rfk, bias=bias, causal=causal)
    ref.backward(do.double())
    for name, g_, r_ in zip(["dq", "dk", "dv", "dfq", "dfk"], got, ref_leaves):
        e = relerr(g_, r_.grad)
        assert e < BF16_TOL, f"{name}: rel err {e:.3e}"


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_bwd_nobias(D, causal):
    _bwd_case(2, 2, 256, 256, D, 0, causal)


@pytest.mark.parametrize("D,R", [(64, 9), (128, 2), (128, 16)])
@pytest.mark.parametrize("causal", [False, True])
def test_bwd_factored(D, R, causal):
    _bwd_case(2, 2, 384, 384, D, R, causal, seed=R)


def test_bwd_ragged():
    _bwd_case(1, 2, 200, 200, 64, 4, True, seed=1)
    _bwd_case(1, 2, 150, 333, 64, 4, False, seed=2)


@pytest.mark.parametrize("causal", [False, True])
def test_bwd_dense(causal):
    _bwd_case(1, 2, 256, 256, 128, 0, causal, dense=True)


def _bwd_static_case(B, H, N, M, D, R, causal, seed=0, factor_batch=1):
    """Static (non-learnable) factors: d=128 with Rpad <= 16 runs the 128x128-tile
    backward (fb_bwd_t128_sm100.cu); dq/dk/dv checked against torch fp64."""
    q, k, v = _qkv(B, H, N, M, D, torch.bfloat16, seed=seed)
    for t in (q, k, v):
        t.requires_grad_(True)
    g = torch.Generator(device="cuda").manual_seed(seed + 11)
    fq = torch.randn(factor_batch, H, N, R, device="cuda", generator=g) * 0.7
    fk = torch.randn(factor_batch, H, M, R, device="cuda", generator=g) * 0.7
    do = torch.randn(B, H, N, D, device="cuda", generator=g).bfloat16()
    mask = "causal" if causal else "none"
    out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    out.backward(do)
    ref_leaves = [t.detach().double().requires_grad_(True) for t in (q, k, v)]
    ref = ref_attention(*ref_leaves, fq.double(), fk.double(), causal=causal)
    ref.backward(do.double())
    for name, got, r_ in zip(["dq", "dk", "dv"], (q.grad, k.grad, v.grad), ref_leaves):
        e = relerr(got, r_.grad)
        assert e < BF16_TOL, f"{name}: rel err {e:.3e}"


@pytest.mark.parametrize("B,H,N,M,R,causal,fb_", [
    (2, 2, 384, 384, 2, True, 1),      # ALiBi-like rank 2 -> 3-way split, 1 panel; batch-broadcast factors
    (1, 2, 200, 200, 2, True, 1),      # ragged causal (N % 128 != 0)
    (1, 2, 150, 333, 4, False, 1),     # N != M, ragged both sides
    (2, 3, 257, 129, 2, False, 2),     # per-batch factors, 3 heads
    (1, 1, 640, 640, 0, True, 1),      # no factors (Rpad 0 instance)
])
def test_bwd_t128_static_factors(B, H, N, M, R, causal, fb_):
    if R == 0:
        _bwd_case(B, H, N, M, 128, 0, causal, seed=3)
    else:
        _bwd_static_case(B, H, N, M, 128, R, causal, seed=B * 10 + R, factor_batch=fb_)


@pytest.mark.parametrize("D,R,causal", [(128, 2, True), (128, 0, False), (64, 4, True)])
def test_bwd_fp16_static(D, R, causal):
    """fp16 inputs through the backward kernels (128x128-tile for d=128, fused 64-query for d=64)."""
    B, H, N = 1, 2, 320
    q, k, v = _qkv(B, H, N, N, D, torch.float16, seed=5)
    for t in (q, k, v):
        t.requires_grad_(True)
    g = torch.Generator(device="cuda").manual_seed(9)
    do = torch.randn(B, H, N, D, device="cuda", generator=g).half()
    mask = "causal" if causal else "none"
    if R:
        fq = torch.randn(1, H, N, R, device="cuda", generator=g) * 0.5
        fk = torch.randn(1, H, N, R, device="cuda", generator=g) * 0.5
        out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    else:
        fq = fk = None
        out = fb.tiled_attention(q, k, v, mask=mask)
    assert out.dtype == torch.float16
    out.backward(do)
    ref_leaves = [t.detach().double().requires_grad_(True) for t in (q, k, v)]
    ref = ref_attention(*ref_leaves, None if fq is None else fq.double(), None if fk is None else fk.double(),
                        causal=causal)
    ref.backward(do.double())
    for name, got, r_ in zip(["dq", "dk", "dv"], (q.grad, k.grad, v.grad), ref_leaves):
        e = relerr(got, r_.grad)
        assert e < BF16_TOL, f"{name}: rel err {e:.3e}"


def _bwd_learn_case(B, H, N, M, R, causal, seed=0, factor_batch=1, dtype=torch.bfloat16, alibi=False):
    """Learnable factors at d=128 with one 16-column panel: the 128x128-tile backward's LEARN variant
    (dUk / dUq as extra N=16 MMAs, fb_bwd_t128_sm100.cu); every gradient against torch fp64 autograd."""
    q, k, v = _qkv(B, H, N, M, 128, dtype, seed=seed)
    for t in (q, k, v):
        t.requires_grad_(True)
    g = torch.Generator(device="cuda").manual_seed(seed + 13)
    if alibi:  # ALiBi-shaped factors (3-way split of large-magnitude columns) with learnable slopes
        slopes = torch.tensor([-(2.0 ** (-8.0 * (i + 1) / H)) for i in range(H)], device="cuda")
        fq0, fk0 = fb.alibi_factors(slopes.tolist(), N, M)
        fq, fk = fq0.clone().float(), fk0.clone().float()
    else:
        fq = torch.randn(factor_batch, H, N, R, device="cuda", generator=g) * 0.6
        fk = torch.randn(factor_batch, H, M, R, device="cuda", generator=g) * 0.6
    fq.requires_grad_(True)
    fk.requires_grad_(True)
    do = torch.randn(B, H, N, 128, device="cuda", generator=g).to(dtype)
    mask = "causal" if causal else "none"
    out = fb.flashbias_attention(q, k, v, fq, fk, mask=mask)
    out.backward(do)
    leaves = [q, k, v, fq, fk]
    ref_leaves = [t.detach().double().requires_grad_(True) for t in leaves]
    ref = ref_attention(*ref_leaves, causal=causal)
    ref.backward(do.double())
    for name, t, r_ in zip(["dq", "dk", "dv", "dfq", "dfk"], leaves, ref_leaves):
        e = relerr(t.grad, r_.grad)
        assert e < BF16_TOL, f"{name}: rel err {e:.3e}"


@pytest.mark.parametrize("B,H,N,M,R,causal,fb_", [
    (2, 2, 384, 384, 2, True, 1),      # odd key-tile count: single-CTA variant; batch-broadcast factors
    (1, 2, 512, 512, 2, True, 1),      # even key-tile count: cluster-multicast variant, causal
    (2, 2, 512, 512, 4, False, 2),     # multicast, non-causal, per-batch factors
    (1, 2, 200, 200, 3, True, 1),      # ragged causal
    (1, 1, 150, 333, 5, False, 1),     # N != M, ragged both sides
])
def test_bwd_t128_learnable_factors(B, H, N, M, R, causal, fb_):
    plan = A.plan_factor_fold(torch.randn(1, 1, 8, R, device="cuda") * 0.6,
                              torch.randn(1, 1, 8, R, device="cuda") * 0.6, 1 / math.sqrt(128))
    assert R * plan.split * (plan.split + 1) // 2 <= 16  # one panel: the LEARN 128x128-tile kernel
    _bwd_learn_case(B, H, N, M, R, causal, seed=N + R, factor_batch=fb_)


def test_bwd_t128_learnable_alibi_slopes():
    """C3-shaped learnable ALiBi (rank 2, 3-way split into 12 columns) at N=2048, causal, 4 heads.

    dq/dk/dv at 2e-2 against fp64 autograd.  The factor gradient dfq = dS @ fk is a
    cancelling sum here (rows of dS sum to zero while fk grows linearly with the key
    index), so the kernel's bf16 dS operand bounds its accuracy, not the kernel:
    dfq/dfk are checked against the exact value at 2e-2 of the summand magnitude
    sum_j |dS_ij| |fk_j| (a bf16 dS element carries 2^-8 of its own size, so this
    is the scale its rounding error lives on)."""
    B, H, N = 1, 4, 2048
    q, k, v = _qkv(B, H, N, N, 128, torch.bfloat16, seed=7)
    for t in (q, k, v):
        t.requires_grad_(True)
    slopes = [-(2.0 ** (-8.0 * (i + 1) / H)) for i in range(H)]
    fq0, fk0 = fb.alibi_factors(slopes, N, N)
    fq, fk = fq0.clone().float().requires_grad_(True), fk0.clone().float().requires_grad_(True)
    do = torch.randn(B, H, N, 128, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)).bfloat16()
    out = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
    out.backward(do)
    leaves = [q, k, v, fq, fk]
    ref_leaves = [t.detach().double().requires_grad_(True) for t in leaves]
    ref = ref_attention(*ref_leaves, causal=True)
    ref.backward(do.double())
    for name, t, r_ in zip(["dq", "dk", "dv"], leaves[:3], ref_leaves[:3]):
        e = relerr(t.grad, r_.grad)
        assert e < BF16_TOL, f"{name}: rel err {e:.3e}"
    with torch.no_grad():  # dS in fp64 from the reference forward, then the kernel's bf16 rounding of it
        qd, kd, vd, fqd, fkd, dod = (x.double() for x in (q, k, v, fq, fk, do))
        s = qd @ kd.transpose(-1, -2) / math.sqrt(128) + fqd @ fkd.transpose(-1, -2)
        s = s.masked_fill(torch.ones(N, N, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
        p = torch.softmax(s, -1)
        dp = dod @ vd.transpose(-1, -2)
        ds = p * (dp - (dp * p).sum(-1, keepdim=True))
        scale_of = {"dfq": ds.abs() @ fkd.abs(), "dfk": ds.abs().transpose(-1, -2) @ fqd.abs()}
        exact = {"dfq": ref_leaves[3].grad, "dfk": ref_leaves[4].grad}
    for name, t in (("dfq", fq), ("dfk", fk)):
        got = t.grad.double()
        # rows whose dS is exactly 0 in fp64 (the first causal row) get the tensor's summand scale
        m = scale_of[name]
        e2 = float(((got - exact[name]).abs() / (m + 1e-3 * m.amax())).max())
        assert e2 < BF16_TOL, f"{name}: err {e2:.3e} relative to sum |dS| |f|"


def test_bwd_t128_learnable_fp16():
    _bwd_learn_case(1, 2, 256, 256, 2, True, seed=9, dtype=torch.float16)
