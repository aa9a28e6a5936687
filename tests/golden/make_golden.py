"""Generate golden vectors by running the REFERENCE package itself.

Run here (the reference exists only in the authoring container):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/flashbias under the alias ``flashbias_ref``
(so the name ``flashbias`` stays free for our drop-in), replays the instances
of the reference's own tests (pkg/tests/test_attention.py, test_acceptance.py,
test_decompose.py, test_integration.py) with the same ``Rng`` seeds, and
stores inputs and reference outputs in golden.npz + manifest.json.  The
committed fixtures pin both the CPU oracle (tests/test_oracle_golden.py) and
the GPU kernels (tests/test_gpu_parity.py); nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src/flashbias/__init__.py"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "flashbias_ref", REF_SRC, submodule_search_locations=[os.path.dirname(REF_SRC)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["flashbias_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def main() -> None:
    R = load_reference()
    arrays: dict = {}
    cases: list = []

    def put(name, kind, inputs: dict, outputs: dict, **meta):
        for key, val in {**inputs, **outputs}.items():
            arrays[f"{name}/{key}"] = np.asarray(val, dtype=np.float64)
        cases.append({"name": name, "kind": kind, "inputs": sorted(inputs), "outputs": sorted(outputs), **meta})

    # ---- attention instances (pkg/tests/test_attention.py)
    put("single_token", "reference", {"q": [[3.0]], "k": [[-2.0]], "v": [[7.0]]},
        {"o": R.reference_attention([[3.0]], [[-2.0]], [[7.0]])}, mask="none")

    rng = R.Rng(1)
    q, k, v = rng.normal(5, 3), rng.normal(6, 3), rng.normal(6, 3)
    put("zero_dense_bias", "dense", {"q": q, "k": k, "v": v, "bias": np.zeros((5, 6))},
        {"o": R.reference_attention(q, k, v, R.DenseBias(np.zeros((5, 6))))}, mask="none")

    rng = R.Rng(7)
    q, k, v = rng.normal(4, 2), rng.normal(4, 2), rng.normal(4, 2)
    b = rng.normal(4, 4)
    put("scalar_dense_rng7", "dense", {"q": q, "k": k, "v": v, "bias": b},
        {"o": R.reference_attention(q, k, v, R.DenseBias(b))}, mask="none")

    rng = R.Rng(17)
    q, k, v = rng.normal(6, 3), rng.normal(6, 3), rng.normal(6, 3)
    put("causal_rng17", "reference", {"q": q, "k": k, "v": v},
        {"o": R.reference_attention(q, k, v, mask="causal")}, mask="causal")

    rng = R.Rng(3)
    q, k, v = rng.normal(128, 16), rng.normal(128, 16), rng.normal(128, 16)
    b = rng.normal(128, 128)
    put("tiled_dense_128", "dense", {"q": q, "k": k, "v": v, "bias": b},
        {"o": R.tiled_attention(q, k, v, R.DenseBias(b), tiles=R.TileConfig(32, 32))}, mask="none")

    rng = R.Rng(4)
    q, k, v = rng.normal(40, 8), rng.normal(56, 8), rng.normal(56, 8)
    fq, fk = rng.normal(40, 5), rng.normal(56, 5)
    put("tiled_factored_40x56", "tiled_factored", {"q": q, "k": k, "v": v, "fq": fq, "fk": fk},
        {"o": R.tiled_attention(q, k, v, R.FactoredBias(fq, fk), tiles=R.TileConfig(16, 8))}, mask="none")

    rng = R.Rng(6)
    q, k, v = rng.normal(12, 4), rng.normal(12, 4), rng.normal(12, 4)
    z = np.zeros((12, 2))
    put("flashbias_zero_factors", "flashbias", {"q": q, "k": k, "v": v, "fq": z, "fk": z},
        {"o": R.flashbias_attention(q, k, v, z, z, tiles=R.TileConfig(5, 7))}, mask="none")

    rng = R.Rng(8)
    q, k, v = rng.normal(64, 8), rng.normal(64, 8), rng.normal(64, 8)
    fb = R.decompose_alibi(64, 64)
    put("flashbias_alibi_64", "flashbias", {"q": q, "k": k, "v": v, "fq": fb.fq, "fk": fb.fk},
        {"o": R.flashbias_attention(q, k, v, fb.fq, fb.fk, tiles=R.TileConfig(16, 24))}, mask="none")

    rng = R.Rng(9)
    q, k, v = rng.normal(256, 16), rng.normal(256, 16), rng.normal(256, 16)
    fq, fk = rng.normal(256, 16), rng.normal(256, 16)
    put("flashbias_causal_256", "flashbias", {"q": q, "k": k, "v": v, "fq": fq, "fk": fk},
        {"o": R.flashbias_attention(q, k, v, fq, fk, mask="causal", tiles=R.TileConfig(48, 32))}, mask="causal")

    rng = R.Rng(31)
    q, k, v = rng.normal(7, 3), rng.normal(7, 3), rng.normal(7, 3)
    fq, fk = rng.normal(7, 2), rng.normal(7, 2)
    for mask in ("none", "causal"):
        put(f"flashbias_scalar31_{mask}", "flashbias", {"q": q, "k": k, "v": v, "fq": fq, "fk": fk},
            {"o": R.flashbias_attention(q, k, v, fq, fk, mask=mask, tiles=R.TileConfig(3, 2))}, mask=mask)

    rng = R.Rng(14)
    q, k, v = rng.normal(24, 4) * 10, rng.normal(20, 4) * 10, rng.normal(20, 4)
    b = (rng.uniform(24, 20) * 2 - 1) * 1e3
    put("large_swings_14", "dense", {"q": q, "k": k, "v": v, "bias": b},
        {"o": R.tiled_attention(q, k, v, R.DenseBias(b), tiles=R.TileConfig(5, 7))}, mask="none")

    rng = R.Rng(12)
    q, k, v = rng.normal(10, 4), rng.normal(13, 4), rng.normal(13, 4)
    rng.normal(10, 13)
    fq, fk = rng.normal(10, 3), rng.normal(13, 3)
    fq2 = np.hstack([fq, np.full((10, 1), 5.5)])
    fk2 = np.hstack([fk, np.ones((13, 1))])
    put("shift_invariance_12", "flashbias", {"q": q, "k": k, "v": v, "fq": fq2, "fk": fk2},
        {"o": R.flashbias_attention(q, k, v, fq2, fk2, tiles=R.TileConfig(4, 5)),
         "o_unshifted": R.flashbias_attention(q, k, v, fq, fk, tiles=R.TileConfig(4, 5))}, mask="none")

    # ---- acceptance criterion 8 (causal + ALiBi factors)
    for n in (64, 256):
        rng = R.Rng(1000 + n)
        q, k, v = rng.normal(n, 16), rng.normal(n, 16), rng.normal(n, 16)
        fb = R.decompose_alibi(n, n)
        dense = R.generate_bias(R.AlibiBias(n, n))
        put(f"crit8_alibi_causal_{n}", "flashbias", {"q": q, "k": k, "v": v, "fq": fb.fq, "fk": fb.fk},
            {"o": R.flashbias_attention(q, k, v, fb.fq, fb.fk, mask="causal", tiles=R.TileConfig(48, 32)),
             "o_dense": R.reference_attention(q, k, v, R.DenseBias(dense), mask="causal")}, mask="causal")

    # ---- integration: exact spatial factors end to end (test_integration.py:22-28)
    rng = R.Rng(50)
    pts = rng.uniform(40, 3) * 10
    target = R.generate_bias(R.SpatialDistanceBias(pts, pts))
    fb = R.decompose_spatial(pts, pts)
    q, k = rng.normal(40, 8), rng.normal(40, 8)
    v = rng.uniform(40, 8) * 2.0 - 1.0
    put("integration_spatial_50", "flashbias", {"q": q, "k": k, "v": v, "fq": fb.fq, "fk": fb.fk, "pts": pts},
        {"o": R.flashbias_attention(q, k, v, fb.fq, fb.fk, tiles=R.TileConfig(16, 16)),
         "o_dense": R.reference_attention(q, k, v, R.DenseBias(target)), "target": target}, mask="none")

    # ---- acceptance criterion 1: 200 seeded instances (test_acceptance.py:27-48).
    # Full arrays for the first 12, per-instance checksums for all 200.
    rng = R.Rng(42)
    sums = []
    for idx in range(200):
        causal = bool(rng.uniform() < 0.4)
        n = int(rng.integers(1, 257)[0])
        m = n if causal else int(rng.integers(1, 257)[0])
        c = int(rng.integers(4, 65)[0])
        r = int(rng.integers(1, 33)[0])
        q, k, v = rng.normal(n, c), rng.normal(m, c), rng.normal(m, c)
        fq, fk = rng.normal(n, r), rng.normal(m, r)
        tiles = R.TileConfig(int(rng.integers(1, n + 1)[0]), int(rng.integers(1, m + 1)[0]))
        mask = "causal" if causal else "none"
        o = R.flashbias_attention(q, k, v, fq, fk, mask, tiles)
        sums.append([n, m, c, r, float(causal), o.sum(), (o * o).sum(), o[0, 0], o[-1, -1]])
        if idx < 12:
            put(f"crit1_{idx:03d}", "flashbias", {"q": q, "k": k, "v": v, "fq": fq, "fk": fk}, {"o": o},
                mask=mask)
    arrays["crit1_checksums"] = np.asarray(sums, dtype=np.float64)

    # ---- decomposers (test_decompose.py, test_acceptance.py:51-90)
    fb = R.decompose_alibi(4, 4)
    arrays["alibi4/pairs"] = np.array([fb.fq[0] @ fb.fk[0], fb.fq[2] @ fb.fk[0]])
    for n, slope in ((33, 1.0), (64, 0.3), (512, 1.0)):
        fb = R.decompose_alibi(n, n, slope=slope)
        arrays[f"alibi_{n}_{slope}/fq"] = fb.fq
        arrays[f"alibi_{n}_{slope}/fk"] = fb.fk
        if n <= 64:
            arrays[f"alibi_{n}_{slope}/dense"] = R.generate_bias(R.AlibiBias(n, n, slope=slope))
    rng = R.Rng(2)
    pq = rng.uniform(32, 3) * 2000 - 1000
    pk = rng.uniform(32, 3) * 2000 - 1000
    w = rng.uniform(32) * 1.5 + 0.5
    fb = R.decompose_spatial(pq, pk, w)
    for key, val in {"pq": pq, "pk": pk, "w": w, "fq": fb.fq, "fk": fb.fk,
                     "dense": R.generate_bias(R.SpatialDistanceBias(pq, pk, w))}.items():
        arrays[f"spatial_rng2/{key}"] = val
    fb = R.decompose_spatial(np.zeros((1, 3)), np.array([[1.0, 2.0, 2.0]]))
    arrays["spatial_hand/value"] = fb.dense()
    rng = R.Rng(3)
    b = rng.normal(64, 8) @ rng.normal(64, 8).T
    fb, rep = R.svd_decompose(b, rank=8)
    arrays["svd_rank8/b"] = b
    arrays["svd_rank8/recon"] = fb.dense()
    arrays["svd_rank8/report"] = np.array([rep.rank_used, rep.energy_retained, rep.max_abs_err, rep.rel_fro_err])
    fb, rep = R.svd_decompose(np.eye(4), energy=0.95)
    arrays["svd_identity/rank"] = np.array([rep.rank_used])
    rng = R.Rng(11)
    rng.normal(64, 8), rng.normal(64, 8)
    reps = []
    for _ in range(20):
        mat = rng.normal(48, 40)
        kk = int(rng.integers(1, 40)[0])
        _, rep = R.svd_decompose(mat, rank=kk)
        reps.append([kk, rep.energy_retained, rep.max_abs_err, rep.rel_fro_err])
        if len(reps) == 1:
            arrays["svd_crit3/mat0"] = mat
    arrays["svd_crit3/reports"] = np.asarray(reps)
    arrays["energy_profile/s"] = np.array([3.0, 2.0, 1.0, 0.5])
    arrays["energy_profile/out"] = R.energy_profile(np.array([3.0, 2.0, 1.0, 0.5]))

    # ---- Rng streams (rng.py) — pins our splitmix64 restatement
    arrays["rng/uniform_0"] = R.Rng(0).uniform(9)
    arrays["rng/normal_42"] = R.Rng(42).normal(7)
    arrays["rng/integers_123"] = R.Rng(123).integers(0, 100, 6).astype(np.float64)
    arrays["rng/normal_big"] = R.Rng(2 ** 40 + 3).normal(3, 2)

    # ---- acceptance criterion 9: head splitting / mixed path (test_acceptance.py:204-236)
    rng = R.Rng(77)
    n9 = 64
    heads = [rng.normal(n9, rank) @ rng.normal(n9, rank).T for rank in (1, 2, 4, 4, 8, 8)]
    for pos in (2, 5):
        heads.insert(pos, rng.normal(n9, n9))
    split = R.split_heads_by_rank(heads, 0.95, max_rank=16)
    q, k, v = rng.normal(n9, 16), rng.normal(n9, 16), rng.normal(n9, 16)
    arrays["crit9/heads"] = np.stack(heads)
    arrays["crit9/q"], arrays["crit9/k"], arrays["crit9/v"] = q, k, v
    arrays["crit9/low_indices"] = np.asarray(split.low_indices, dtype=np.int64)
    arrays["crit9/dense_indices"] = np.asarray(split.dense_indices, dtype=np.int64)
    arrays["crit9/common_rank"] = np.asarray([split.common_rank], dtype=np.int64)
    factored = dict(zip(split.low_indices, split.low_factors))
    outs, dense_ref = [], []
    for idx, head in enumerate(heads):
        dense_ref.append(R.reference_attention(q, k, v, R.DenseBias(head)))
        if idx in factored:
            fb = factored[idx]
            outs.append(R.flashbias_attention(q, k, v, fb.fq, fb.fk, tiles=R.TileConfig(16, 16)))
            arrays[f"crit9/fq_{idx}"], arrays[f"crit9/fk_{idx}"] = fb.fq, fb.fk
        else:
            outs.append(R.tiled_attention(q, k, v, R.DenseBias(head), tiles=R.TileConfig(16, 16)))
    arrays["crit9/o_mixed"] = np.stack(outs)
    arrays["crit9/o_dense"] = np.stack(dense_ref)
    # a second split instance: energy threshold low enough that every head is factored
    split2 = R.split_heads_by_rank(heads[:3], 0.5, max_rank=64)
    arrays["crit9b/low_indices"] = np.asarray(split2.low_indices, dtype=np.int64)
    arrays["crit9b/common_rank"] = np.asarray([split2.common_rank], dtype=np.int64)

    # ---- file formats (fileio.py; test_fileio.py): raw bytes written by the reference
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        def dump(name, writer, obj, **kw):
            path = os.path.join(td, name)
            writer(path, obj, **kw)
            with open(path, "rb") as f:
                arrays[f"fileio/{name}"] = np.frombuffer(f.read(), dtype=np.uint8).copy()
        a = R.Rng(0).normal(7, 5)
        arrays["fileio/a"] = a
        dump("a_f64.dbm", R.write_dbm1, a)
        dump("a_f32.dbm", R.write_dbm1, a, dtype="f32")
        fb = R.random_low_rank_factors(9, 6, 3, seed=2)
        arrays["fileio/fq"], arrays["fileio/fk"] = fb.fq, fb.fk
        dump("f_f64.fbf", R.write_fbf1, fb)
        dump("f_f32.fbf", R.write_fbf1, fb, dtype="f32")
        dump("neural.fbf", R.write_fbf1, R.FactoredBias(np.ones((2, 1)), np.ones((3, 1)), origin="neural"))
        fs = R.decompose_alibi(32, 32, slope=-0.25)
        arrays["fileio/alibi_fq"], arrays["fileio/alibi_fk"] = fs.fq, fs.fk
        dump("alibi_exact.fbf", R.write_fbf1, fs)

    # ---- neural decomposer (neural.py; test_neural.py, test_integration.py:45-54, criterion 4)
    rng = R.Rng(21)
    xq, xk = rng.uniform(4, 2), rng.uniform(4, 2)
    target = rng.normal(4, 4)
    nets = R.FactorNetworks.init(R.Rng(22), 2, 5, 3)
    loss, grads = nets.loss_and_grads(xq, xk, target)
    arrays["neural_grad/xq"], arrays["neural_grad/xk"], arrays["neural_grad/target"] = xq, xk, target
    arrays["neural_grad/loss"] = np.array([loss])
    for i, g in enumerate(grads):
        arrays[f"neural_grad/g{i}"] = g
    rng = R.Rng(5)
    xq = rng.uniform(10, 2)
    target = rng.normal(10, 10)
    fb, _, losses = R.neural_decompose(xq, xq, target, rank=4, hidden=16, iters=200, lr=1e-3,
                                       lr_decay=(0.5, 50), seed=1)
    arrays["neural_fit/xq"], arrays["neural_fit/target"] = xq, target
    arrays["neural_fit/losses"], arrays["neural_fit/fq"], arrays["neural_fit/fk"] = np.asarray(losses), fb.fq, fb.fk
    rng = R.Rng(56)
    ll = np.stack([rng.uniform(48) * np.pi - np.pi / 2, rng.uniform(48) * 2 * np.pi - np.pi], axis=1)
    target = R.generate_bias(R.SphericalDistanceBias(ll))
    fb, _, losses = R.neural_decompose(ll, ll, target, rank=8, hidden=32, iters=400, seed=3)
    rep = R.reconstruction_report(fb, target)
    arrays["neural_sph/ll"], arrays["neural_sph/target"] = ll, target
    arrays["neural_sph/losses"], arrays["neural_sph/fq"], arrays["neural_sph/fk"] = np.asarray(losses), fb.fq, fb.fk
    arrays["neural_sph/report"] = np.array([rep.max_abs_err, rep.rel_fro_err, rep.energy_retained])
    rng = R.Rng(2024)
    lat = rng.uniform(64) * np.pi - np.pi / 2
    lon = rng.uniform(64) * 2 * np.pi - np.pi
    ll = np.stack([lat, lon], axis=1)
    target = R.generate_bias(R.SphericalDistanceBias(ll))
    _, _, losses = R.neural_decompose(ll, ll, target, rank=32, hidden=256, iters=10000, lr=1e-3, seed=7)
    arrays["crit4/ll"], arrays["crit4/losses"] = ll, np.asarray(losses)
    pos = R.Rng(31).uniform(20, 2)
    arrays["gravity/pos"], arrays["gravity/b"] = pos, R.generate_bias(R.GravityBias(pos, eps=0.05))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"source": "reference flashbias 0.1.0 (pkg/src/flashbias), generated by make_golden.py",
                   "cases": cases}, f, indent=1)
    print(f"wrote {len(cases)} attention cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
