"""Pin the CPU oracle (oracle/flashbias_oracle.py) and the host-side Rng
restatement to golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import flashbias_oracle as orc
from paper_2505_12044_b200.rng import Rng

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
MANIFEST = json.load(open(os.path.join(HERE, "golden", "manifest.json")))
CASES = MANIFEST["cases"]


def _run_oracle(case):
    name = case["name"]
    a = {key: G[f"{name}/{key}"] for key in case["inputs"]}
    mask = case["mask"]
    if case["kind"] == "flashbias":
        return orc.flashbias_attention(a["q"], a["k"], a["v"], a["fq"], a["fk"], mask=mask)
    if case["kind"] == "tiled_factored":
        o, _ = orc.streaming_attention(a["q"], a["k"], a["v"], fq=a["fq"], fk=a["fk"],
                                       premul=np.sqrt(a["q"].shape[1]), mask=mask)
        return o
    if case["kind"] == "dense":
        o, _ = orc.streaming_attention(a["q"], a["k"], a["v"], bias=a["bias"], mask=mask)
        return o
    return orc.materialized_attention(a["q"], a["k"], a["v"], mask=mask)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_golden(case):
    got = _run_oracle(case)
    want = G[f"{case['name']}/o"]
    assert np.abs(got - want).max() <= 1e-10


def test_oracle_materialized_equals_streaming_on_golden():
    for case in CASES:
        if case["kind"] != "flashbias":
            continue
        a = {key: G[f"{case['name']}/{key}"] for key in case["inputs"]}
        c = a["q"].shape[1]
        m = orc.materialized_attention(a["q"], a["k"], a["v"], fq=a["fq"], fk=a["fk"], premul=np.sqrt(c),
                                       mask=case["mask"])
        assert np.abs(m - G[f"{case['name']}/o"]).max() <= 1e-10


def test_single_token_passes_value():
    assert G["single_token/o"][0, 0] == 7.0


def test_shift_invariance_golden():
    assert np.abs(G["shift_invariance_12/o"] - G["shift_invariance_12/o_unshifted"]).max() <= 1e-12


def test_crit8_factored_equals_dense_golden():
    for n in (64, 256):
        assert np.abs(G[f"crit8_alibi_causal_{n}/o"] - G[f"crit8_alibi_causal_{n}/o_dense"]).max() <= 1e-10


def test_criterion1_checksums_all_200():
    """Replays all 200 criterion-1 instances through our Rng + the oracle and
    matches the reference's per-instance checksums (checksum of checksums)."""
    rng = Rng(42)
    sums = G["crit1_checksums"]
    for idx in range(200):
        causal = bool(rng.uniform() < 0.4)
        n = int(rng.integers(1, 257)[0])
        m = n if causal else int(rng.integers(1, 257)[0])
        c = int(rng.integers(4, 65)[0])
        r = int(rng.integers(1, 33)[0])
        q, k, v = rng.normal(n, c), rng.normal(m, c), rng.normal(m, c)
        fq, fk = rng.normal(n, r), rng.normal(m, r)
        rng.integers(1, n + 1), rng.integers(1, m + 1)  # tiles (advisory)
        o = orc.flashbias_attention(q, k, v, fq, fk, mask="causal" if causal else "none")
        row = sums[idx]
        assert (n, m, c, r, float(causal)) == tuple(row[:5])
        got = np.array([o.sum(), (o * o).sum(), o[0, 0], o[-1, -1]])
        assert np.abs(got - row[5:]).max() <= 1e-9 * max(1.0, np.abs(row[5:]).max())


def test_rng_streams_bit_exact():
    assert np.array_equal(Rng(0).uniform(9), G["rng/uniform_0"])
    assert np.array_equal(Rng(42).normal(7), G["rng/normal_42"])
    assert np.array_equal(Rng(123).integers(0, 100, 6).astype(np.float64), G["rng/integers_123"])
    assert np.array_equal(Rng(2 ** 40 + 3).normal(3, 2), G["rng/normal_big"])


def test_decomposers_golden():
    p = G["alibi4/pairs"]
    assert p[0] == 0.0 and p[1] == 2.0
    for n, slope in ((33, 1.0), (64, 0.3), (512, 1.0)):
        fq, fk = orc.decompose_alibi(n, n, slope)
        assert np.array_equal(fq, G[f"alibi_{n}_{slope}/fq"]) and np.array_equal(fk, G[f"alibi_{n}_{slope}/fk"])
        if n <= 64:
            assert np.abs(orc.alibi_dense(n, n, slope) - G[f"alibi_{n}_{slope}/dense"]).max() == 0.0
    fq, fk = orc.decompose_spatial(G["spatial_rng2/pq"], G["spatial_rng2/pk"], G["spatial_rng2/w"])
    assert np.array_equal(fq, G["spatial_rng2/fq"]) and np.array_equal(fk, G["spatial_rng2/fk"])
    dense = orc.spatial_dense(G["spatial_rng2/pq"], G["spatial_rng2/pk"], G["spatial_rng2/w"])
    assert np.abs(dense - G["spatial_rng2/dense"]).max() <= 1e-9 * np.abs(dense).max()
    fq, fk = orc.decompose_spatial(np.zeros((1, 3)), np.array([[1.0, 2.0, 2.0]]))
    assert (fq @ fk.T)[0, 0] == G["spatial_hand/value"][0, 0] == 9.0


def test_svd_golden():
    fq, fk, rep = orc.svd_decompose(G["svd_rank8/b"], rank=8)
    ref = G["svd_rank8/report"]
    assert rep["rank_used"] == ref[0] == 8
    assert abs(rep["energy_retained"] - ref[1]) <= 1e-12
    assert np.abs(fq @ fk.T - G["svd_rank8/recon"]).max() <= 1e-9
    _, _, rep = orc.svd_decompose(np.eye(4), energy=0.95)
    assert rep["rank_used"] == G["svd_identity/rank"][0] == 4
    k0 = int(G["svd_crit3/reports"][0, 0])
    _, _, rep = orc.svd_decompose(G["svd_crit3/mat0"], rank=k0)
    assert abs(rep["energy_retained"] - G["svd_crit3/reports"][0, 1]) <= 1e-12
    assert abs(rep["rel_fro_err"] - G["svd_crit3/reports"][0, 3]) <= 1e-12
    for row in G["svd_crit3/reports"]:
        assert abs(row[3] ** 2 + row[1] - 1.0) <= 1e-10  # Eckart-Young identity
    assert np.abs(orc.energy_profile(G["energy_profile/s"]) - G["energy_profile/out"]).max() == 0.0


def test_backward_oracle_finite_differences():
    rng = np.random.default_rng(0)
    q, k, v = rng.normal(size=(5, 3)), rng.normal(size=(6, 3)), rng.normal(size=(6, 3))
    fq, fk = rng.normal(size=(5, 2)), rng.normal(size=(6, 2))
    do = rng.normal(size=(5, 3))
    premul = np.sqrt(3.0)
    g = orc.attention_bwd(q, k, v, do, fq=fq, fk=fk, premul=premul)
    args = [q, k, v, fq, fk]

    def loss(*a):
        return (orc.streaming_attention(a[0], a[1], a[2], fq=a[3], fk=a[4], premul=premul)[0] * do).sum()

    for idx, name in enumerate(["dq", "dk", "dv", "dfq", "dfk"]):
        num = np.zeros_like(args[idx])
        for i in np.ndindex(args[idx].shape):
            up = [x.copy() for x in args]
            dn = [x.copy() for x in args]
            up[idx][i] += 1e-6
            dn[idx][i] -= 1e-6
            num[i] = (loss(*up) - loss(*dn)) / 2e-6
        assert np.abs(num - g[name]).max() <= 1e-7, name


def test_blocked_fwd_bwd_matches_materialised_backward():
    """The config-size GPU parity tests use the query-blocked restatement;
    it must equal attention_bwd (materialised) to rounding."""
    rng = np.random.default_rng(3)
    for mask in ("none", "causal"):
        n, d, r = 300, 16, 3
        q, k, v, do = (rng.standard_normal((n, d)) for _ in range(4))
        fq, fk = rng.standard_normal((n, r)), rng.standard_normal((n, r))
        a = orc.attention_bwd(q, k, v, do, fq=fq, fk=fk, premul=4.0, mask=mask)
        b = orc.blocked_attention_fwd_bwd(q, k, v, do, fq=fq, fk=fk, premul=4.0, mask=mask, block=64)
        for key in ("o", "dq", "dk", "dv", "dfq", "dfk"):
            assert orc.rel_max_err(b[key], a[key]) < 1e-12, (mask, key)
