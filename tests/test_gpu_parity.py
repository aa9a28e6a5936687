"""GPU parity against the reference's own instances (tests/golden, produced by
running the reference package) and the CPU oracle on the same rounded inputs.

* fp32 path (SIMT kernel): vs the reference float64 outputs, 1e-5 relative.
* bf16 path (tcgen05 kernels): inputs rounded to bf16, vs the oracle on those
  rounded inputs, 2e-2 relative (max-abs / max|ref|).
Everything goes through the public drop-in API, hence through the C ABI."""

import json
import os

import numpy as np
import pytest

from oracle import flashbias_oracle as orc

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
CASES = json.load(open(os.path.join(HERE, "golden", "manifest.json")))["cases"]
F32_TOL, BF16_TOL = 1e-5, 2e-2


def fb():
    import paper_2505_12044_b200
    return paper_2505_12044_b200


def _inputs(case):
    return {k: G[f"{case['name']}/{k}"] for k in case["inputs"]}


def _run(case, a, precision=None):
    lib = fb()
    mask = case["mask"]
    if case["kind"] == "flashbias":
        return lib.flashbias_attention(a["q"], a["k"], a["v"], a["fq"], a["fk"], mask=mask, precision=precision)
    if case["kind"] == "tiled_factored":
        return lib.tiled_attention(a["q"], a["k"], a["v"], lib.FactoredBias(a["fq"], a["fk"]), mask=mask,
                                   precision=precision)
    if case["kind"] == "dense":
        return lib.tiled_attention(a["q"], a["k"], a["v"], lib.DenseBias(a["bias"]), mask=mask, precision=precision)
    return lib.tiled_attention(a["q"], a["k"], a["v"], mask=mask, precision=precision)


def _bf16(x):
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).bfloat16().double().numpy()


def _oracle(case, a):
    mask = case["mask"]
    c = a["q"].shape[1]
    if case["kind"] == "flashbias":
        return orc.flashbias_attention(a["q"], a["k"], a["v"], a["fq"], a["fk"], mask=mask)
    if case["kind"] == "tiled_factored":
        return orc.streaming_attention(a["q"], a["k"], a["v"], fq=a["fq"], fk=a["fk"], premul=np.sqrt(c),
                                       mask=mask)[0]
    if case["kind"] == "dense":
        return orc.streaming_attention(a["q"], a["k"], a["v"], bias=a["bias"], mask=mask)[0]
    return orc.materialized_attention(a["q"], a["k"], a["v"], mask=mask)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_fp32_path_matches_reference_golden(case):
    got = _run(case, _inputs(case))
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    assert orc.rel_max_err(got, G[f"{case['name']}/o"]) <= F32_TOL


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_bf16_path_matches_oracle_on_rounded_inputs(case):
    a = _inputs(case)
    # q/k/v (and a dense bias) are rounded to bf16 for both sides; logical
    # factors stay fp32 (the kernel splits them into bf16 panels itself)
    r = dict(a)
    for key in ("q", "k", "v", "bias"):
        if key in r:
            r[key] = _bf16(r[key])
    for key in ("fq", "fk"):
        if key in r:
            r[key] = np.asarray(r[key], dtype=np.float32).astype(np.float64)
    got = _run(case, r, precision="bf16")
    assert orc.rel_max_err(got, _oracle(case, r)) <= BF16_TOL


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reference_attention_matches_reference_golden(case):
    """reference_attention / attention_weights (ref attention.py:111-137: the materialised float64
    formula the reference's own tests use as ground truth) against the reference's golden outputs of
    every instance (dense, factored -- FactoredBias.dense() = fq fk^T, unscaled -- and no bias)."""
    lib = fb()
    a = _inputs(case)
    if "bias" in a:
        bias = lib.DenseBias(a["bias"])
    elif "fq" in a:
        bias = lib.FactoredBias(a["fq"], a["fk"])
    else:
        bias = lib.NO_BIAS
    got = lib.reference_attention(a["q"], a["k"], a["v"], bias, mask=case["mask"])
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    assert orc.rel_max_err(got, G[f"{case['name']}/o"]) <= 1e-10
    w = lib.attention_weights(a["q"], a["k"], bias, mask=case["mask"])
    assert np.allclose(w.sum(axis=-1), 1.0, atol=1e-12)
    assert orc.rel_max_err(w @ np.asarray(a["v"], dtype=np.float64), G[f"{case['name']}/o"]) <= 1e-10


def test_criterion1_all_200_instances_both_paths():
    """Acceptance criterion 1 (reference test_acceptance.py:27-48): 200 seeded
    instances, random shapes/masks/ranks.  fp32 path vs the reference's
    checksums; bf16 path vs the oracle on rounded inputs."""
    from paper_2505_12044_b200.rng import Rng
    lib = fb()
    rng = Rng(42)
    sums = G["crit1_checksums"]
    worst32 = worst16 = 0.0
    for idx in range(200):
        causal = bool(rng.uniform() < 0.4)
        n = int(rng.integers(1, 257)[0])
        m = n if causal else int(rng.integers(1, 257)[0])
        c = int(rng.integers(4, 65)[0])
        r = int(rng.integers(1, 33)[0])
        q, k, v = rng.normal(n, c), rng.normal(m, c), rng.normal(m, c)
        fq, fk = rng.normal(n, r), rng.normal(m, r)
        rng.integers(1, n + 1), rng.integers(1, m + 1)
        mask = "causal" if causal else "none"
        o = lib.flashbias_attention(q, k, v, fq, fk, mask=mask)
        got = np.array([o.sum(), (o * o).sum(), o[0, 0], o[-1, -1]])
        ref = sums[idx, 5:]
        worst32 = max(worst32, float(np.abs(got[2:] - ref[2:]).max()))
        assert abs(got[0] - ref[0]) <= 1e-5 * n * c and abs(got[1] - ref[1]) <= 1e-5 * n * c
        qb, kb, vb = _bf16(q), _bf16(k), _bf16(v)
        fq32, fk32 = fq.astype(np.float32).astype(np.float64), fk.astype(np.float32).astype(np.float64)
        o16 = lib.flashbias_attention(qb, kb, vb, fq32, fk32, mask=mask, precision="bf16")
        e = orc.rel_max_err(o16, orc.flashbias_attention(qb, kb, vb, fq32, fk32, mask=mask))
        worst16 = max(worst16, e)
    assert worst32 <= 1e-5
    assert worst16 <= BF16_TOL


def test_causal_rows_ignore_later_keys_bitwise():
    """Reference test_attention.py:97-107, on the tcgen05 path: perturbing keys
    after row i leaves rows <= i bit-identical."""
    import torch
    lib = fb()
    g = torch.Generator(device="cuda").manual_seed(5)
    n, i = 512, 200
    q, k, v = (torch.randn(1, 2, n, 64, device="cuda", generator=g).bfloat16() for _ in range(3))
    base = lib.tiled_attention(q, k, v, mask="causal")
    k2, v2 = k.clone(), v.clone()
    k2[..., i + 1:, :] += 10 * torch.randn_like(k2[..., i + 1:, :])
    v2[..., i + 1:, :] -= 3.0
    pert = lib.tiled_attention(q, k2, v2, mask="causal")
    assert torch.equal(pert[..., : i + 1, :], base[..., : i + 1, :])


def test_zero_factors_equal_no_bias_and_shift_invariance():
    import torch
    lib = fb()
    g = torch.Generator(device="cuda").manual_seed(6)
    q, k, v = (torch.randn(2, 2, 300, 128, device="cuda", generator=g).bfloat16() for _ in range(3))
    z = torch.zeros(1, 2, 300, 4, device="cuda")
    a = lib.flashbias_attention(q, k, v, z, z)
    b = lib.tiled_attention(q, k, v)
    assert torch.equal(a, b)
    fq = torch.randn(1, 2, 300, 3, device="cuda", generator=g)
    fk = torch.randn(1, 2, 300, 3, device="cuda", generator=g)
    base = lib.flashbias_attention(q, k, v, fq, fk)
    fq2 = torch.cat([fq, torch.full_like(fq[..., :1], 5.5)], -1)
    fk2 = torch.cat([fk, torch.ones_like(fk[..., :1])], -1)
    shifted = lib.flashbias_attention(q, k, v, fq2, fk2)
    assert orc.rel_max_err(shifted.double().cpu().numpy(), base.double().cpu().numpy()) <= BF16_TOL


@pytest.mark.parametrize("split_bwd", ["0", "1"])
def test_backward_vs_oracle_golden_instances(split_bwd):
    """Backward (no reference: SPEC.md:183) vs the oracle's analytic gradient on
    the golden crit-8 ALiBi instance and a d=128 instance, through both the
    fused (d=128) and the two-kernel backward (FB_FORCE_SPLIT_BWD=1)."""
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, sys
sys.path.insert(0, {os.path.dirname(HERE)!r})
import paper_2505_12044_b200 as fb
from oracle import flashbias_oracle as orc
G = np.load({os.path.join(HERE, 'golden', 'golden.npz')!r})
worst = 0.0
for name, d in (("crit8_alibi_causal_256", None), ("flashbias_causal_256", 128)):
    q, k, v = (G[name + "/" + x] for x in "qkv")
    fq, fk = G[name + "/fq"], G[name + "/fk"]
    if d is not None:  # widen to head dim 128 (zero channels change nothing but the 1/sqrt(C) scale)
        rng = np.random.default_rng(0)
        q, k, v = (np.concatenate([x, rng.standard_normal((x.shape[0], d - x.shape[1]))], 1) for x in (q, k, v))
    qt, kt, vt = (torch.tensor(x, device="cuda").bfloat16().requires_grad_(True) for x in (q, k, v))
    fqt = torch.tensor(fq, device="cuda", dtype=torch.float32).requires_grad_(True)
    fkt = torch.tensor(fk, device="cuda", dtype=torch.float32).requires_grad_(True)
    o = fb.flashbias_attention(qt, kt, vt, fqt, fkt, mask="causal")
    do = torch.randn_like(o)
    o.backward(do)
    g = orc.attention_bwd(*(t.detach().double().cpu().numpy() for t in (qt, kt, vt)), do.double().cpu().numpy(),
                          fq=fqt.detach().double().cpu().numpy(), fk=fkt.detach().double().cpu().numpy(),
                          premul=np.sqrt(qt.shape[-1]), mask="causal")
    for nm, t in (("dq", qt), ("dk", kt), ("dv", vt), ("dfq", fqt), ("dfk", fkt)):
        worst = max(worst, orc.rel_max_err(t.grad.double().cpu().numpy(), g[nm]))
print("WORST", worst)
"""
    env = dict(os.environ, FB_FORCE_SPLIT_BWD=split_bwd)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.strip().split("WORST")[-1])
    assert worst <= BF16_TOL


def test_decomposers_on_device_match_golden():
    lib = fb()
    for n, slope in ((33, 1.0), (64, 0.3), (512, 1.0)):
        f = lib.decompose_alibi(n, n, slope)
        assert np.array_equal(f.fq, G[f"alibi_{n}_{slope}/fq"]) and np.array_equal(f.fk, G[f"alibi_{n}_{slope}/fk"])
    f = lib.decompose_spatial(G["spatial_rng2/pq"], G["spatial_rng2/pk"], G["spatial_rng2/w"])
    assert np.abs(f.fq - G["spatial_rng2/fq"]).max() <= 1e-9 * np.abs(G["spatial_rng2/fq"]).max()
    dense = lib.generate_bias(lib.SpatialDistanceBias(G["spatial_rng2/pq"], G["spatial_rng2/pk"], G["spatial_rng2/w"]))
    assert np.abs(dense - G["spatial_rng2/dense"]).max() <= 1e-9 * np.abs(dense).max()
    # fp32 device factor kernels (K6) vs the closed forms
    import torch
    fq, fk = lib.alibi_factors([1.0, 0.5], 64, 64)
    ref_q, ref_k = orc.decompose_alibi(64, 64, 0.5)
    assert np.array_equal(fq[0, 1].double().cpu().numpy(), ref_q) and np.array_equal(fk[0, 1].double().cpu().numpy(), ref_k)
    pts = torch.rand(50, 3, device="cuda")
    w = torch.rand(50, device="cuda") + 0.5
    fq, fk = lib.spatial_factors(pts, pts, w)
    rq, rk = orc.decompose_spatial(pts.double().cpu().numpy(), pts.double().cpu().numpy(), w.double().cpu().numpy())
    assert np.abs(fq[0, 0].double().cpu().numpy() - rq).max() <= 1e-5
    assert np.abs(fk[0, 0].double().cpu().numpy() - rk).max() <= 1e-5


def test_svd_decompose_matches_reference_reports():
    lib = fb()
    fbias, rep = lib.svd_decompose(G["svd_rank8/b"], rank=8)
    ref = G["svd_rank8/report"]
    assert rep.rank_used == 8 and abs(rep.energy_retained - ref[1]) <= 1e-12
    assert np.abs(fbias.dense() - G["svd_rank8/recon"]).max() <= 1e-9
    _, rep = lib.svd_decompose(np.eye(4), energy=0.95)
    assert rep.rank_used == 4
    k0 = int(G["svd_crit3/reports"][0, 0])
    _, rep = lib.svd_decompose(G["svd_crit3/mat0"], rank=k0)
    assert abs(rep.energy_retained - G["svd_crit3/reports"][0, 1]) <= 1e-12
    assert abs(rep.rel_fro_err - G["svd_crit3/reports"][0, 3]) <= 1e-12
    # reconstruction_report on the same factors
    rr = lib.reconstruction_report(fbias, G["svd_rank8/b"])
    assert rr.rank_used == 8 and rr.max_abs_err <= 1e-9


def test_randomized_svd_close_to_exact():
    import torch
    lib = fb()
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 3000
    u = torch.linalg.qr(torch.randn(n, 32, device="cuda", generator=g, dtype=torch.float64))[0]
    vv = torch.linalg.qr(torch.randn(n, 32, device="cuda", generator=g, dtype=torch.float64))[0]
    s = 8 * 0.8 ** torch.arange(32, device="cuda", dtype=torch.float64)
    b = (u * s) @ vv.T + 1e-4 * torch.randn(n, n, device="cuda", generator=g, dtype=torch.float64)
    _, rep_r = lib.svd_decompose(b, rank=16, method="randomized")
    _, rep_e = lib.svd_decompose(b, rank=16, method="exact")
    assert abs(rep_r.rel_fro_err - rep_e.rel_fro_err) <= 1e-3 * max(rep_e.rel_fro_err, 1e-12) + 1e-9
