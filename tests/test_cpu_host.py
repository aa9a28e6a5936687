"""Host-side logic that needs no GPU: the C-ABI library loads and exports every
symbol include/flashbias_b200.h declares, the Python API validates exactly
like the reference (attention.py:77-108, 215-223; errors.py), and the
tile-size / split helpers behave as documented."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import _lib
from paper_2505_12044_b200.errors import ConfigError, MaskError, ShapeError, ValidationError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashbias_b200.h")


def _header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert _header_functions() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("native library not built (run __graft_entry__.build())")
    handle = ctypes.CDLL(_lib.LIB_PATH)
    for name in _header_functions():
        assert hasattr(handle, name), name
    lib = _lib.lib()
    assert lib.fb_abi_version() == 1
    # pure host helpers of the ABI can be called without a GPU
    assert lib.fb_factor_cols(2, 3) == 12 and lib.fb_factor_rpad(2, 3) == 16
    assert lib.fb_factor_cols(9, 2) == 27 and lib.fb_factor_rpad(9, 2) == 32
    assert lib.fb_factor_rpad(64, 1) == 64


def test_abi_validation_maps_to_reference_exceptions():
    """Shape/mask validation in the C ABI happens before any launch, so it is
    testable on a CPU-only host with fake device pointers."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("native library not built")
    lib = _lib.lib()

    def t(b, h, n, d, dtype=_lib.FB_BF16):
        x = _lib.FbTensor()
        x.data = 4096
        for i, s in enumerate((b, h, n, d)):
            x.shape[i] = s
        x.stride[3], x.stride[2], x.stride[1], x.stride[0] = 1, d, n * d, h * n * d
        x.dtype = dtype
        return x

    q, k, v, o = t(1, 2, 64, 64), t(1, 2, 80, 64), t(1, 2, 80, 64), t(1, 2, 64, 64)
    with pytest.raises(MaskError):
        _lib.check(lib.fb_attn_fwd(ctypes.byref(q), ctypes.byref(k), ctypes.byref(v), None, None, None, 1,
                                   0.125, ctypes.byref(o), None, None))
    kbad = t(1, 2, 80, 32)
    with pytest.raises(ShapeError):
        _lib.check(lib.fb_attn_fwd(ctypes.byref(q), ctypes.byref(kbad), ctypes.byref(v), None, None, None, 0,
                                   0.125, ctypes.byref(o), None, None))
    uq, uk = t(1, 2, 64, 16), t(1, 2, 80, 32)
    with pytest.raises(ShapeError):
        _lib.check(lib.fb_attn_fwd(ctypes.byref(q), ctypes.byref(k), ctypes.byref(v), ctypes.byref(uq),
                                   ctypes.byref(uk), None, 0, 0.125, ctypes.byref(o), None, None))
    with pytest.raises(ValidationError):
        _lib.check(lib.fb_attn_fwd(ctypes.byref(q), ctypes.byref(k), ctypes.byref(v), None, None, None, 7,
                                   0.125, ctypes.byref(o), None, None))
    q48, k48, v48, o48 = t(1, 2, 64, 48), t(1, 2, 64, 48), t(1, 2, 64, 48), t(1, 2, 64, 48)
    with pytest.raises(ConfigError):  # unpadded head dim is rejected, not silently handled
        _lib.check(lib.fb_attn_fwd(ctypes.byref(q48), ctypes.byref(k48), ctypes.byref(v48), None, None, None, 0,
                                   0.125, ctypes.byref(o48), None, None))


def test_python_validation_before_compute():
    q = np.ones((3, 2))
    with pytest.raises(MaskError):  # reference test_attention.py:65-68
        fb.reference_attention(q, np.ones((4, 2)), np.ones((4, 2)), mask="causal")
    with pytest.raises(MaskError):
        fb.flashbias_attention(q, np.ones((4, 2)), np.ones((4, 2)), np.ones((3, 1)), np.ones((4, 1)),
                               mask="causal")
    with pytest.raises(ShapeError):
        fb.flashbias_attention(q, np.ones((4, 3)), np.ones((4, 3)), np.ones((3, 1)), np.ones((4, 1)))
    with pytest.raises(ShapeError):
        fb.tiled_attention(q, np.ones((4, 2)), np.ones((5, 2)))
    with pytest.raises(ValidationError):
        fb.tiled_attention(q, np.ones((4, 2)), np.ones((4, 2)), mask="diagonal")
    with pytest.raises(ValidationError):
        fb.tiled_attention(q, np.ones((4, 2)), np.ones((4, 2)), tiles=(4, 4))


def test_errors_are_value_errors_like_reference():
    for cls in (ShapeError, MaskError, ConfigError, ValidationError):
        assert issubclass(cls, ValueError)
    e = fb.TrainingError("diverged", 17)
    assert isinstance(e, RuntimeError) and e.iteration == 17


def test_tile_config_and_choose_tile_sizes():
    tiles = fb.choose_tile_sizes(64, 64, 100 * 1024, 2)  # reference test_attention.py:214-216
    assert tiles.b_q == 96 and tiles.b_kv == 96
    with pytest.raises(ConfigError):
        fb.choose_tile_sizes(4096, 4096, 64, 8)
    with pytest.raises(ConfigError):
        fb.TileConfig(0, 4)
    for c, r, mult in ((1, 0, 1), (64, 16, 3), (128, 128, 20)):
        base = 4 * 8 * (c + r)
        assert fb.choose_tile_sizes(c, r, base * mult * 2, 8).b_q >= fb.choose_tile_sizes(c, r, base * mult, 8).b_q


def test_factored_bias_provider():
    fq, fk = np.ones((5, 3)), np.ones((7, 3))
    b = fb.FactoredBias(fq, fk)
    assert b.rank == 3 and b.storage_bytes() == (5 + 7) * 3 * 8
    assert b.dense().shape == (5, 7)
    with pytest.raises(ShapeError):
        fb.FactoredBias(np.ones((5, 3)), np.ones((7, 2)))
    with pytest.raises(ValidationError):
        fb.FactoredBias(fq, fk, origin="magic")
    assert fb.DenseBias(np.zeros((4, 6))).storage_bytes(2) == 48
    assert fb.NO_BIAS.storage_bytes() == 0


def test_choose_split_levels():
    torch = pytest.importorskip("torch")
    # exactly representable -> no split
    assert fb.choose_split(torch.ones(1, 1, 8, 2), torch.ones(1, 1, 8, 2)) == 1
    # ALiBi at N=16384 with a non power-of-two slope needs the 3-way split
    i = torch.arange(1, 16385, dtype=torch.float32)
    s = -(2.0 ** (-8 / 32 * 3))
    fq = torch.stack([torch.full_like(i, s), s * i], -1)[None, None]
    fk = torch.stack([-i, torch.ones_like(i)], -1)[None, None]
    assert fb.choose_split(fq, fk, premul=128 ** 0.5) == 3
    # spatial factors on a normalised grid settle for 2 (27 columns -> 2 panels)
    g = torch.rand(4096, 3)
    w = -(0.5 + 1.5 * torch.rand(4096))
    fq = torch.cat([w[:, None] * torch.stack([g[:, d] ** 2, torch.ones(4096), -2 * g[:, d]], -1) for d in range(3)], -1)
    fk = torch.cat([torch.stack([torch.ones(4096), g[:, d] ** 2, g[:, d]], -1) for d in range(3)], -1)
    assert fb.choose_split(fq[None, None], fk[None, None], premul=8.0) == 2


def test_flashbias_alias_package():
    import flashbias
    assert flashbias.flashbias_attention is fb.flashbias_attention
    assert set(["flashbias_attention", "tiled_attention", "svd_decompose", "decompose_alibi"]) <= set(flashbias.__all__)


def test_choose_split_raises_instead_of_dropping_below_its_bound():
    """R=64 factors premultiplied by sqrt(128) cannot meet
    1e-2 logits inside 64 panel columns -> ConfigError, never a silent k=1."""
    torch = pytest.importorskip("torch")
    g = torch.Generator().manual_seed(0)
    fq = (torch.randn(1, 1, 512, 64, generator=g) / 8).bfloat16().float()
    fk = torch.randn(1, 1, 512, 64, generator=g).bfloat16().float()
    with pytest.raises(ConfigError):
        fb.choose_split(fq, fk, premul=128 ** 0.5, max_cols=64)
    assert fb.choose_split(fq, fk, premul=1.0, max_cols=64) == 1


def test_factor_fold_plan():
    """north_star fold Q' = [scale*q, U] is chosen exactly when the reference
    order's sqrt(C) premultiplier would cost split columns."""
    torch = pytest.importorskip("torch")
    from paper_2505_12044_b200.attention import plan_factor_fold
    g = torch.Generator().manual_seed(1)
    fq = (torch.randn(1, 1, 256, 64, generator=g) / 8).bfloat16().float()
    fk = torch.randn(1, 1, 256, 64, generator=g).bfloat16().float()
    # d=128: 1/scale = sqrt(128) inexact -> Q' fold, no split
    p = plan_factor_fold(fq, fk, 128 ** -0.5, max_cols=64)
    assert p.q_fold and p.split == 1 and p.premul == 1.0 and p.kernel_scale == 1.0
    # d=64: sqrt(64) = 8 is a power of two -> reference order, exact, no split
    p = plan_factor_fold(fq, fk, 64 ** -0.5, max_cols=128)
    assert not p.q_fold and p.split == 1 and p.premul == 8.0
    # ALiBi at N=16384 needs the 3-way split either way -> reference order (no extra pass over q)
    i = torch.arange(1, 16385, dtype=torch.float32)
    s = -(2.0 ** (-8 / 32 * 3))
    fa = torch.stack([torch.full_like(i, s), s * i], -1)[None, None]
    fb_ = torch.stack([-i, torch.ones_like(i)], -1)[None, None]
    p = plan_factor_fold(fa, fb_, 128 ** -0.5, max_cols=64)
    assert not p.q_fold and p.split == 3
    # nothing fits -> ConfigError
    big = torch.randn(1, 1, 64, 64, generator=g) * 1e4
    with pytest.raises(ConfigError):
        plan_factor_fold(big, big, 128 ** -0.5, max_cols=64)


def test_split_cache_checks_object_identity():
    """a new factor tensor that reuses a freed allocation must not
    inherit the cached plan of the old one."""
    torch = pytest.importorskip("torch")
    from paper_2505_12044_b200 import attention as A
    A._SPLIT_CACHE.clear()
    fq = torch.ones(1, 1, 64, 2)
    fk = torch.ones(1, 1, 64, 2)
    p1 = A.plan_factor_fold_cached(fq, fk, fq, fk, 0.125, tol=1e-6)
    assert p1.split == 1
    fq2 = torch.full((1, 1, 64, 2), 1.0 + 2.0 ** -12)  # inexact in bf16: 2.4e-4 per rank at k=1
    fk2 = fk.clone()
    p2 = A.plan_factor_fold_cached(fq2, fk2, fq2, fk2, 0.125, tol=1e-6)
    assert p2.split > 1
    fq.mul_(1.0 + 2.0 ** -12)  # in-place write bumps the version -> re-planned
    assert A.plan_factor_fold_cached(fq, fk, fq, fk, 0.125, tol=1e-6).split > 1
    # views of the same factors (per-call head slices) hit the cache
    fq3, fk3 = torch.full((1, 3, 64, 2), 1.0 + 2.0 ** -12), torch.ones(1, 3, 64, 2)
    n0 = len(A._SPLIT_CACHE)
    for _ in range(3):
        A.plan_factor_fold_cached(fq3[:, 1:2], fk3[:, 1:2], fq3[:, 1:2], fk3[:, 1:2], 0.125, tol=1e-6)
    assert len(A._SPLIT_CACHE) == n0 + 1


def test_core_helpers_match_reference_semantics():
    a, b = np.arange(6.0).reshape(2, 3), np.ones((2, 2))
    assert fb.concat_cols(a, b).shape == (2, 5)
    with pytest.raises(ShapeError):
        fb.concat_cols(a, np.ones((3, 2)))
    with pytest.raises(ShapeError):
        fb.matmul(a, a)
    assert fb.matmul(a, a.T).shape == (2, 2)
    s = fb.softmax_rows(np.array([[1e300, 0.0], [0.0, 0.0]]))
    assert np.allclose(s, [[1.0, 0.0], [0.5, 0.5]])
    assert abs(fb.frobenius(np.array([[3.0, 4.0]])) - 5.0) < 1e-15
    with pytest.raises(ShapeError):
        fb.frobenius(np.ones(3))
