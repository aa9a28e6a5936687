"""GPU parity for the §8(f) widening rows: device head splitting + the mixed
factored/dense path against the reference's criterion-9 instance
(ref: decompose.py:179-225, test_acceptance.py:204-236), and FBF1/DBM1 files
read straight into device memory feeding the kernels (ref: fileio.py)."""

import os

import numpy as np
import pytest
import torch

from oracle import flashbias_oracle as orc
import paper_2505_12044_b200 as fb

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def test_device_split_matches_reference_partition():
    heads = list(G["crit9/heads"])
    split = fb.split_heads_by_rank(heads, 0.95, max_rank=16)
    assert split.low_indices == list(G["crit9/low_indices"])
    assert split.dense_indices == list(G["crit9/dense_indices"])
    assert split.common_rank == int(G["crit9/common_rank"][0])
    for i, f in zip(split.low_indices, split.low_factors):
        assert f.fq.is_cuda and f.rank == split.common_rank and f.origin == "svd"
        want = G[f"crit9/fq_{i}"] @ G[f"crit9/fk_{i}"].T
        assert np.abs(f.dense().cpu().numpy() - want).max() <= 1e-9
    s2 = fb.split_heads_by_rank(torch.as_tensor(G["crit9/heads"][:3]), 0.5, max_rank=64)
    assert s2.low_indices == list(G["crit9b/low_indices"])
    assert s2.common_rank == int(G["crit9b/common_rank"][0])
    none = fb.split_heads_by_rank(heads, 0.95, max_rank=0)
    assert none.low_indices == [] and none.dense_indices == list(range(8)) and none.common_rank == 0


def test_device_split_validation():
    with pytest.raises(fb.ValidationError):
        fb.split_heads_by_rank([], 0.9, 4)
    with pytest.raises(fb.ValidationError):
        fb.split_heads_by_rank([np.eye(4)], 1.5, 4)
    with pytest.raises(fb.ShapeError):
        fb.split_heads_by_rank([np.eye(4), np.eye(5)], 0.9, 4)


def test_mixed_path_fp32_matches_reference_outputs():
    heads = G["crit9/heads"]
    split = fb.split_heads_by_rank(list(heads), 0.95, max_rank=16)
    got = fb.mixed_head_attention(G["crit9/q"], G["crit9/k"], G["crit9/v"], split, heads,
                                  tiles=fb.TileConfig(16, 16))
    assert got.shape == G["crit9/o_mixed"].shape
    # fp32 path: 1e-5 relative to the reference's float64 outputs (north_star tolerance)
    assert orc.rel_max_err(got, G["crit9/o_mixed"]) <= 1e-5
    assert orc.rel_max_err(got, G["crit9/o_dense"]) <= 1e-5


@pytest.mark.parametrize("mask", ["none", "causal"])
def test_mixed_path_bf16_heads(mask):
    torch.manual_seed(3)
    heads = torch.as_tensor(G["crit9/heads"]).cuda()
    split = fb.split_heads_by_rank(heads, 0.95, max_rank=16)
    H, n, c = heads.shape[0], heads.shape[1], 64
    q, k, v = (torch.randn(H, n, c, device="cuda").bfloat16() for _ in range(3))
    got = fb.mixed_head_attention(q, k, v, split, heads, mask=mask)
    assert got.dtype == torch.bfloat16 and got.shape == (H, n, c)
    qn, kn, vn = (t.double().cpu().numpy() for t in (q, k, v))
    for h in range(H):
        want, _ = orc.streaming_attention(qn[h], kn[h], vn[h], bias=G["crit9/heads"][h], mask=mask)
        assert orc.rel_max_err(got[h].double().cpu().numpy(), want) <= 2e-2, h


def test_fbf1_to_device_feeds_flashbias(tmp_path):
    path = tmp_path / "alibi.fbf"
    path.write_bytes(G["fileio/alibi_exact.fbf"].tobytes())
    f = fb.read_fbf1(path, device="cuda")
    assert f.fq.is_cuda and f.fq.dtype == torch.float64
    assert np.array_equal(f.fq.cpu().numpy(), G["fileio/alibi_fq"])
    f32 = fb.read_fbf1(path, device="cuda", dtype=torch.float32)
    assert f32.fk.dtype == torch.float32
    torch.manual_seed(0)
    n, c = 32, 64
    q, k, v = (torch.randn(1, 2, n, c, device="cuda").bfloat16() for _ in range(3))
    o = fb.flashbias_attention(q, k, v, f.fq, f.fk, mask="causal")
    qn, kn, vn = (t.double().cpu().numpy() for t in (q, k, v))
    want = orc.flashbias_attention(qn, kn, vn, G["fileio/alibi_fq"], G["fileio/alibi_fk"], mask="causal")
    assert orc.rel_max_err(o.double().cpu().numpy(), want) <= 2e-2


def test_dbm1_to_device_feeds_dense_path(tmp_path):
    a = G["fileio/a"]
    path = tmp_path / "b.dbm"
    fb.write_dbm1(path, np.tile(a, (8, 13))[:48, :48], dtype="f32")
    b = fb.read_dbm1(path, device="cuda", dtype=torch.bfloat16)
    assert b.is_cuda and b.dtype == torch.bfloat16 and tuple(b.shape) == (48, 48)
    torch.manual_seed(1)
    q, k, v = (torch.randn(48, 64, device="cuda").bfloat16() for _ in range(3))
    o = fb.tiled_attention(q, k, v, fb.DenseBias(b))
    want, _ = orc.streaming_attention(*(t.double().cpu().numpy() for t in (q, k, v)),
                                      bias=b.double().cpu().numpy())
    assert orc.rel_max_err(o.double().cpu().numpy(), want) <= 2e-2
