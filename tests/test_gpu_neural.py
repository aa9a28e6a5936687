"""GPU parity for the neural factor networks (ref: neural.py) and the
gravity / spherical generators (ref: bias.py:180-205) against golden vectors
produced by the reference (tests/golden/make_golden.py), plus the neural
factors feeding the FlashBias kernel (ref: test_integration.py:45-54)."""

import os

import numpy as np
import pytest
import torch

from oracle import flashbias_oracle as orc
import paper_2505_12044_b200 as fb

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def test_generators_match_reference():
    g = fb.generate_bias(fb.GravityBias(G["gravity/pos"], eps=0.05))
    assert np.abs(g - G["gravity/b"]).max() <= 1e-12 * np.abs(G["gravity/b"]).max()
    s = fb.generate_bias(fb.SphericalDistanceBias(G["neural_sph/ll"]))
    assert np.abs(s - G["neural_sph/target"]).max() <= 1e-12
    with pytest.raises(fb.ValidationError):
        fb.generate_bias(fb.SphericalDistanceBias(np.array([[2.0, 0.0]])))
    with pytest.raises(fb.ValidationError):
        fb.generate_bias(fb.GravityBias(np.zeros((3, 2))))


def test_factor_network_grads_match_reference():
    nets = fb.FactorNetworks.init(fb.Rng(22), 2, 5, 3)
    loss, grads = nets.loss_and_grads(G["neural_grad/xq"], G["neural_grad/xk"], G["neural_grad/target"])
    assert abs(loss - G["neural_grad/loss"][0]) <= 1e-12 * max(1.0, abs(loss))
    for i, g in enumerate(grads):
        assert g.is_cuda
        assert np.abs(g.cpu().numpy() - G[f"neural_grad/g{i}"]).max() <= 1e-12


def test_neural_fit_tracks_reference_trajectory():
    xq, target = G["neural_fit/xq"], G["neural_fit/target"]
    f, nets, losses = fb.neural_decompose(xq, xq, target, rank=4, hidden=16, iters=200, lr=1e-3,
                                          lr_decay=(0.5, 50), seed=1)
    ref = G["neural_fit/losses"]
    assert len(losses) == 200 and losses[-1] < losses[0]
    # float64 on both sides; only GEMM summation order differs
    assert np.abs(np.asarray(losses) - ref).max() <= 1e-9 * ref.max()
    want = G["neural_fit/fq"] @ G["neural_fit/fk"].T
    assert np.abs(f.fq @ f.fk.T - want).max() <= 1e-8 * np.abs(want).max()
    assert f.origin == "neural"


def test_neural_factors_feed_flashbias_within_bound():
    ll, target = G["neural_sph/ll"], G["neural_sph/target"]
    f, _, losses = fb.neural_decompose(ll, ll, target, rank=8, hidden=32, iters=400, seed=3)
    assert np.abs(np.asarray(losses) - G["neural_sph/losses"]).max() <= 1e-8 * G["neural_sph/losses"].max()
    rep = fb.reconstruction_report(f, target)
    assert abs(rep.max_abs_err - G["neural_sph/report"][0]) <= 1e-6
    rng = fb.Rng(57)
    q, k, v = rng.normal(48, 8), rng.normal(48, 8), rng.normal(48, 8)
    got = fb.flashbias_attention(q, k, v, f.fq, f.fk)  # fp32 path: exact in the factor term
    want = orc.materialized_attention(q, k, v, bias=target)
    assert np.abs(got - want).max() <= 2 * rep.max_abs_err  # ref: test_integration.py:45-54
    fq_t = torch.as_tensor(f.fq, device="cuda")
    fk_t = torch.as_tensor(f.fk, device="cuda")
    qb, kb, vb = (torch.as_tensor(x, device="cuda").bfloat16() for x in (q, k, v))
    ob = fb.flashbias_attention(qb, kb, vb, fq_t, fk_t)
    wantb = orc.flashbias_attention(*(t.double().cpu().numpy() for t in (qb, kb, vb)), f.fq, f.fk)
    assert orc.rel_max_err(ob.double().cpu().numpy(), wantb) <= 2e-2


def test_criterion_4_long_fit_on_device():
    ll = G["crit4/ll"]
    target = fb.generate_bias(fb.SphericalDistanceBias(ll))
    _, _, losses = fb.neural_decompose(ll, ll, target, rank=32, hidden=256, iters=10000, lr=1e-3, seed=7)
    assert losses[-1] <= losses[0] / 100
    windows = [float(np.mean(losses[i:i + 500])) for i in range(0, 10000, 500)]
    assert all(b <= a for a, b in zip(windows, windows[1:]))
    ref = G["crit4/losses"]
    assert abs(losses[0] - ref[0]) <= 1e-9 * ref[0]
    # chaotic amplification over 10k Adam steps is bounded; the end point stays close
    assert abs(losses[-1] - ref[-1]) <= 0.05 * ref[-1]


def test_reference_neural_error_cases():
    ok = np.ones((3, 2))
    with pytest.raises(fb.ShapeError):
        fb.neural_decompose(ok, np.ones((3, 3)), np.ones((3, 3)), rank=2, hidden=4, iters=1)
    with pytest.raises(fb.ShapeError):
        fb.neural_decompose(ok, ok, np.ones((4, 4)), rank=2, hidden=4, iters=1)
    with pytest.raises(fb.ValidationError):
        fb.neural_decompose(ok, ok, np.ones((3, 3)), rank=2, hidden=4, iters=0)
    with pytest.raises(fb.ValidationError):
        fb.neural_decompose(ok, ok, np.full((3, 3), np.nan), rank=2, hidden=4, iters=1)
    rng = fb.Rng(4)
    xq = rng.uniform(6, 2) * 1e150
    target = rng.normal(6, 6) * 1e160
    with pytest.raises(fb.TrainingError) as err:
        fb.neural_decompose(xq, xq, target, rank=2, hidden=4, iters=50, lr=1e100, seed=0)
    assert err.value.iteration >= 0
    a = fb.neural_decompose(G["neural_fit/xq"][:6], G["neural_fit/xq"][:5], G["neural_fit/target"][:6, :5],
                            rank=2, hidden=8, iters=40, seed=9)
    b = fb.neural_decompose(G["neural_fit/xq"][:6], G["neural_fit/xq"][:5], G["neural_fit/target"][:6, :5],
                            rank=2, hidden=8, iters=40, seed=9)
    assert np.array_equal(a[0].fq, b[0].fq) and a[2] == b[2]  # deterministic


@pytest.mark.parametrize("hidden,rank,split", [(32, 8, 2), (256, 32, 1), (64, 4, 3)])
def test_fused_mlp_prologue_matches_two_step_path(hidden, rank, split):
    """fb_mlp_factor_panels == evaluate the networks, then fb_prepare_factors."""
    from paper_2505_12044_b200 import attention as A
    rng = fb.Rng(91)
    xq, xk = rng.uniform(300, 2) * 2 - 1, rng.uniform(260, 2) * 2 - 1
    nets = fb.FactorNetworks.init(fb.Rng(5), 2, hidden, rank)
    uq, uk, f32q, f32k = nets.panels(xq, xk, premul=8.0, split=split, with_factors=True)
    fq, fk = nets.factors(xq, xk)  # float64 reference evaluation
    assert (f32q.double() - fq).abs().max().item() <= 1e-5 * max(1.0, fq.abs().max().item())
    assert (f32k.double() - fk).abs().max().item() <= 1e-5 * max(1.0, fk.abs().max().item())
    rq, rk = A.prepare_factor_panels(f32q, f32k, 8.0, split, torch.bfloat16)
    assert torch.equal(uq, rq) and torch.equal(uk, rk)


def test_neural_flashbias_attention_vs_oracle():
    ll, target = G["neural_sph/ll"], G["neural_sph/target"]
    f, nets, _ = fb.neural_decompose(ll, ll, target, rank=8, hidden=32, iters=100, seed=3)
    torch.manual_seed(4)
    q, k, v = (torch.randn(2, 3, 48, 64, device="cuda").bfloat16() for _ in range(3))
    for mask in ("none", "causal"):
        o = fb.neural_flashbias_attention(q, k, v, nets, ll, ll, mask=mask)
        want = orc.flashbias_attention(*(t.double().cpu().numpy() for t in (q, k, v)), f.fq, f.fk, mask=mask)
        assert orc.rel_max_err(o.double().cpu().numpy(), want) <= 2e-2
