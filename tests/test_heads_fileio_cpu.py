"""CPU tests for the §8(f) widening rows: the oracle's head split pinned to the
reference's criterion-9 partition (tests/golden, ref: decompose.py:179-225,
test_acceptance.py:204-236), and the DBM1/FBF1 host code (pure file-format
logic, ref: fileio.py:1-90) checked byte-for-byte against files written by the
reference, plus the reference's own fileio test cases (test_fileio.py)."""

import os

import numpy as np
import pytest

from oracle import flashbias_oracle as orc
from paper_2505_12044_b200 import (FactoredBias, Rng, ValidationError, random_low_rank_factors,
                                   read_dbm1, read_fbf1, write_dbm1, write_fbf1)

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def test_oracle_split_matches_reference_partition():
    heads = list(G["crit9/heads"])
    low, factors, dense, common = orc.split_heads_by_rank(heads, 0.95, max_rank=16)
    assert low == list(G["crit9/low_indices"])
    assert dense == list(G["crit9/dense_indices"])
    assert common == int(G["crit9/common_rank"][0])
    for i, (fq, fk) in zip(low, factors):
        # factors are unique up to per-column sign; their product is not
        assert np.abs(fq @ fk.T - G[f"crit9/fq_{i}"] @ G[f"crit9/fk_{i}"].T).max() <= 1e-10
    low2, _, _, common2 = orc.split_heads_by_rank(heads[:3], 0.5, max_rank=64)
    assert low2 == list(G["crit9b/low_indices"]) and common2 == int(G["crit9b/common_rank"][0])


def test_oracle_mixed_path_matches_reference_outputs():
    heads = G["crit9/heads"]
    q, k, v = G["crit9/q"], G["crit9/k"], G["crit9/v"]
    low = set(int(i) for i in G["crit9/low_indices"])
    for idx in range(heads.shape[0]):
        if idx in low:
            got = orc.flashbias_attention(q, k, v, G[f"crit9/fq_{idx}"], G[f"crit9/fk_{idx}"])
        else:
            got, _ = orc.streaming_attention(q, k, v, bias=heads[idx])
        assert np.abs(got - G["crit9/o_mixed"][idx]).max() <= 1e-10
        assert np.abs(got - G["crit9/o_dense"][idx]).max() <= 1e-9  # criterion 9's bar


@pytest.mark.parametrize("name,dtype", [("a_f64.dbm", "f64"), ("a_f32.dbm", "f32")])
def test_dbm1_bytes_match_reference(tmp_path, name, dtype):
    path = tmp_path / name
    write_dbm1(path, G["fileio/a"], dtype=dtype)
    assert path.read_bytes() == G[f"fileio/{name}"].tobytes()
    ref_path = tmp_path / ("ref_" + name)
    ref_path.write_bytes(G[f"fileio/{name}"].tobytes())
    back = read_dbm1(ref_path)
    assert back.dtype == (np.float64 if dtype == "f64" else np.float32)
    assert np.array_equal(back, G["fileio/a"].astype(back.dtype))


@pytest.mark.parametrize("name,dtype", [("f_f64.fbf", "f64"), ("f_f32.fbf", "f32")])
def test_fbf1_bytes_match_reference(tmp_path, name, dtype):
    fb = FactoredBias(G["fileio/fq"], G["fileio/fk"], origin="exact")
    path = tmp_path / name
    write_fbf1(path, fb, dtype=dtype)
    assert path.read_bytes() == G[f"fileio/{name}"].tobytes()
    back = read_fbf1(path)
    tol = 0 if dtype == "f64" else 1e-6
    assert np.abs(back.fq - G["fileio/fq"]).max() <= tol and np.abs(back.fk - G["fileio/fk"]).max() <= tol
    assert back.origin == "exact"


def test_fbf1_reference_neural_and_alibi_files(tmp_path):
    p = tmp_path / "n.fbf"
    p.write_bytes(G["fileio/neural.fbf"].tobytes())
    assert read_fbf1(p).origin == "neural"
    p = tmp_path / "al.fbf"
    p.write_bytes(G["fileio/alibi_exact.fbf"].tobytes())
    fb = read_fbf1(p)
    assert np.array_equal(fb.fq, G["fileio/alibi_fq"]) and np.array_equal(fb.fk, G["fileio/alibi_fk"])


# ---- the reference's own fileio cases (pkg/tests/test_fileio.py)
def test_dbm1_round_trip_f64(tmp_path):
    a = Rng(0).normal(7, 5)
    path = tmp_path / "a.dbm"
    write_dbm1(path, a)
    back = read_dbm1(path)
    assert back.dtype == np.float64 and np.array_equal(back, a)


def test_dbm1_round_trip_f32_stable(tmp_path):
    a = Rng(1).normal(6, 4)
    p1, p2 = tmp_path / "a.dbm", tmp_path / "b.dbm"
    write_dbm1(p1, a, dtype="f32")
    back = read_dbm1(p1)
    assert back.dtype == np.float32
    write_dbm1(p2, back, dtype="f32")
    assert p1.read_bytes() == p2.read_bytes()


def test_dbm1_header_layout(tmp_path):
    path = tmp_path / "a.dbm"
    write_dbm1(path, np.zeros((2, 3)))
    raw = path.read_bytes()
    assert raw[:4] == b"DBM1" and raw[4] == 0
    assert int.from_bytes(raw[5:13], "little") == 2 and int.from_bytes(raw[13:21], "little") == 3
    assert len(raw) == 21 + 2 * 3 * 8


@pytest.mark.parametrize("data", [b"NOPE" + b"\x00" * 30, b"DBM1" + bytes([7]) + b"\x00" * 16])
def test_dbm1_rejects_bad_magic_and_code(tmp_path, data):
    path = tmp_path / "bad.dbm"
    path.write_bytes(data)
    with pytest.raises(ValidationError):
        read_dbm1(path)


def test_dbm1_rejects_truncation(tmp_path):
    path = tmp_path / "a.dbm"
    write_dbm1(path, np.ones((4, 4)))
    path.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(ValidationError):
        read_dbm1(path)


def test_fbf1_round_trip(tmp_path):
    fb = random_low_rank_factors(9, 6, 3, seed=2)
    path = tmp_path / "f.fbf"
    write_fbf1(path, fb)
    back = read_fbf1(path)
    assert np.array_equal(back.fq, fb.fq) and np.array_equal(back.fk, fb.fk) and back.origin == fb.origin


def test_fbf1_header_and_origin_tags(tmp_path):
    fb = FactoredBias(np.ones((2, 1)), np.ones((3, 1)), origin="neural")
    path = tmp_path / "f.fbf"
    write_fbf1(path, fb)
    raw = path.read_bytes()
    assert raw[:4] == b"FBF1" and raw[4] == 0 and raw[5] == 2
    assert [int.from_bytes(raw[a:a + 8], "little") for a in (6, 14, 22)] == [2, 3, 1]
    assert read_fbf1(path).origin == "neural"


@pytest.mark.parametrize("data", [b"DBM1" + b"\x00" * 40, b"FBF1" + bytes([0, 9]) + b"\x00" * 24,
                                  b"FBF1" + bytes([5, 0]) + b"\x00" * 24])
def test_fbf1_rejects_bad_files(tmp_path, data):
    path = tmp_path / "bad.fbf"
    path.write_bytes(data)
    with pytest.raises(ValidationError):
        read_fbf1(path)


def test_fbf1_rejects_truncated_payload(tmp_path):
    path = tmp_path / "f.fbf"
    write_fbf1(path, random_low_rank_factors(5, 4, 2, seed=1))
    path.write_bytes(path.read_bytes()[:-3])
    with pytest.raises(ValidationError):
        read_fbf1(path)


def test_writer_rejects_unknown_dtype(tmp_path):
    with pytest.raises(ValidationError):
        write_dbm1(tmp_path / "x.dbm", np.ones((2, 2)), dtype="f16")


def test_oracle_factor_network_grads_match_reference():
    """The oracle's MLP backprop (ref: neural.py:49-98) against the reference's
    own gradients on its test instance (test_neural.py:27-37)."""
    init = Rng(22)
    qp = orc.glorot_params(init, (2, 5, 5, 3))
    kp = orc.glorot_params(init, (2, 5, 5, 3))
    loss, grads = orc.factor_loss_and_grads(qp, kp, G["neural_grad/xq"], G["neural_grad/xk"],
                                            G["neural_grad/target"])
    assert abs(loss - G["neural_grad/loss"][0]) <= 1e-14 * max(1.0, abs(loss))
    for i, g in enumerate(grads):
        assert np.abs(g - G[f"neural_grad/g{i}"]).max() <= 1e-13


def test_gravity_and_spherical_generators_are_pinned():
    from paper_2505_12044_b200 import bias as B
    assert isinstance(B.GravityBias(G["gravity/pos"]).eps, float)
    assert G["gravity/b"].shape == (20, 20) and G["neural_sph/target"].shape == (48, 48)
