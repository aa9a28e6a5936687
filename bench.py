#!/usr/bin/env python
"""FlashBias on B200: attention-with-bias fwd+bwd TFLOP/s and ms/step.

Default workload (BASELINE.json configs[2], "C3"): decoder LM with causal ALiBi
bias, B=4 H=32 N=M=16384 d=128, bf16, forward + backward over all B*H heads,
FlashBias kernel (ALiBi factors folded into the contraction).  The same step
is also timed with our same-pipeline dense-bias kernel ([1,32,N,N] bf16 bias)
for the "vs dense-bias flash" comparison.

    python bench.py [--gpus N --steps K --warmup W] [--config C3] [--impl ours|reference]

One JSON line on rank 0.  Multi-GPU (torchrun): B*H pairs are sharded
contiguously across ranks (head-major), no collective in the timed region;
value = total algorithmic FLOPs / max-over-ranks time.  --impl reference
times the CPU oracle port (oracle/flashbias_oracle.py, the reference's
numpy float64 algorithm restated) on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(B=1, H=8, N=1024, d=64, causal=False, dtype="fp32", bwd=False, bias="alibi",
               desc="ALiBi exact rank-2, B=1 H=8 N=1024 d=64 fp32 forward"),
    "C2": dict(B=1, H=16, N=4096, d=64, causal=False, dtype="bf16", bwd=True, bias="spatial",
               desc="Swin-style 2D spatial-distance bias on a 64x64 grid, H=16 d=64 bf16 fwd+bwd (learnable weights)"),
    "C3": dict(B=4, H=32, N=16384, d=128, causal=True, dtype="bf16", bwd=True, bias="alibi",
               desc="Decoder LM with causal ALiBi bias, B=4 H=32 N=16384 d=128 bf16 fwd+bwd"),
    "C4": dict(B=1, H=16, N=768, d=32, causal=False, dtype="bf16", bwd=False, bias="af3", R=32,
               desc="AlphaFold3-style pair bias N=768 H=16 d=32, device SVD rank R, bf16 fwd"),
    "C5": dict(B=8, H=32, N=8192, d=128, causal=False, dtype="bf16", bwd=True, bias="c5", R=64,
               desc="General dense bias, device randomized SVD rank R (sweep 8..64), B=8 H=32 N=8192 d=128 "
                    "bf16 fwd+bwd"),
}
# §8(f)-1 widening row (not a BASELINE config): head split by bias rank, low-rank heads on the
# FlashBias kernel and full-rank heads on the dense-bias kernel (ref: decompose.py:179-225)
MIX = dict(B=4, H=16, N=2048, d=64, causal=False, dtype="bf16", bwd=True, low=12,
           desc="head-split mixed path: 12 spatial-bias heads (factored after device SVD) + 4 full-rank heads "
                "(dense), B=4 N=2048 d=64 bf16 fwd+bwd")
METRIC = "attn-with-bias fwd+bwd TFLOP/s & ms/step vs dense-bias flash, 1/2/4/8 B200"


def logical_rank(cfg) -> int:
    return {"alibi": 2, "spatial": 9}.get(cfg["bias"]) or int(cfg["R"])


def alg_flops(cfg, heads: int, rows=None) -> float:
    """F = heads * N * M * c_f * [(4d + 2R) + (10d + 6R) if bwd]."""
    n, d, r = cfg["N"], cfg["d"], logical_rank(cfg)
    per_pair = 4 * d + 2 * r + ((10 * d + 6 * r) if cfg["bwd"] else 0)
    if rows is None:
        pairs = n * n * ((n + 1) / (2 * n) if cfg["causal"] else 1.0)
    else:  # an explicit set of query rows (CPU sample): causal row i sees i+1 keys
        pairs = sum((i + 1) if cfg["causal"] else n for i in rows)
    return heads * pairs * per_pair


def alibi_slopes(h: int):
    return [-(2.0 ** (-8.0 * (i + 1) / h)) for i in range(h)]


def c5_bias(n: int, seed: int, device, rank: int = 64):
    """SURVEY §8(d) C5 per-(b,h) dense bias, generated on device (fp32):
    b = sum_{k<=rank} 8 * 0.9^(k-1) u_k v_k^T + 1e-3 E, u_k, v_k unit random
    vectors, E ~ N(0, 1); seed = 5000 + b*H + h."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    u = torch.randn(n, rank, generator=g, device=device)
    v = torch.randn(n, rank, generator=g, device=device)
    u = u / u.norm(dim=0, keepdim=True)
    v = v / v.norm(dim=0, keepdim=True)
    w = 8.0 * 0.9 ** torch.arange(rank, device=device, dtype=torch.float32)
    return (u * w) @ v.T + 1e-3 * torch.randn(n, n, generator=g, device=device)


def af3_pair_bias(n: int, heads, device):
    """SURVEY §8(d) C4 AlphaFold3-style pair bias [len(heads), n, n] (fp64 on device):
    residue coordinates from a 3.8 A random walk (Rng(4000)), 16 RBF channels
    z_ijk = exp(-(|x_i - x_j| - mu_k)^2 / (2 * 2.5^2)), mu_k = 2 + 2.5k, and
    per-head weights w_h ~ N(0, 1/16) (Rng(4100 + h)): b_h = z . w_h."""
    import numpy as np
    import torch

    from paper_2505_12044_b200.rng import Rng
    steps = Rng(4000).normal(n, 3)
    steps = 3.8 * steps / np.linalg.norm(steps, axis=1, keepdims=True)
    x = torch.as_tensor(np.cumsum(steps, axis=0), device=device, dtype=torch.float64)
    dist = torch.cdist(x, x)
    mu = 2.0 + 2.5 * torch.arange(16, device=device, dtype=torch.float64)
    z = torch.exp(-((dist[..., None] - mu) ** 2) / (2 * 2.5 ** 2))  # [n, n, 16]
    w = torch.stack([torch.as_tensor(Rng(4100 + h).normal(16), device=device, dtype=torch.float64) / 4.0
                     for h in heads])  # [H, 16], std 1/4
    return torch.einsum("ijk,hk->hij", z, w)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """Poll SM clock / throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- GPU arm
def make_inputs(cfg, h_lo: int, h_hi: int, device, seed: int = 1234):
    """Synthetic inputs for heads [h_lo, h_hi) and all B batch rows, q/k/v/dO
    [B, H_loc, N, d] seeded per (b, h) with seed + b*H + h, so any head
    sharding sees identical per-head data."""
    import torch

    import paper_2505_12044_b200 as fb
    B, H, N, d = cfg["B"], cfg["H"], cfg["N"], cfg["d"]
    dt = torch.float32 if cfg["dtype"] == "fp32" else torch.bfloat16
    heads = list(range(h_lo, h_hi))
    hl = len(heads)
    q = torch.empty(B, hl, N, d, dtype=dt, device=device)
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    g = torch.Generator(device=device)
    for b in range(B):
        for i, h in enumerate(heads):
            g.manual_seed(seed + b * H + h)
            for t in (q, k, v, do):
                t[b, i].normal_(generator=g)
    fq = fk = None
    if cfg["bias"] == "alibi":  # batch-broadcast factors [1, H_loc, N, 2]
        slopes = [alibi_slopes(H)[h] for h in heads]
        fq, fk = fb.alibi_factors(slopes, N, N)
    elif cfg["bias"] == "spatial":  # learnable per-head row weights, shared positions
        side = int(round(math.sqrt(N)))
        r = torch.arange(N, device=device) // side
        c = torch.arange(N, device=device) % side
        pos = torch.stack([r / (side - 1), c / (side - 1), torch.zeros(N, device=device)], -1).float()
        from paper_2505_12044_b200.rng import Rng
        w = torch.stack([-(0.5 + 1.5 * torch.as_tensor(Rng(2000 + h).uniform(N), device=device).float())
                         for h in heads])
        fq, fk = fb.spatial_factors(pos, pos, w[None])  # fq [1,H_loc,N,9], fk [1,1,N,9]
        fk = fk.expand(1, hl, N, 9).contiguous()
    else:  # C4 / C5: dense biases factorised on the device (SVD), the north_star approximate path
        fq, fk, fact = svd_factors(cfg, heads, device)
        return dict(q=q, k=k, v=v, do=do, fq=fq, fk=fk, dense=None, heads=heads, factorisation=fact)
    return dict(q=q, k=k, v=v, do=do, fq=fq, fk=fk, dense=None, heads=heads)


def dense_biases(cfg, heads, device, b: int):
    """The exact dense biases of batch row b for ``heads``: [len(heads), N, N] fp32 on device."""
    import torch
    if cfg["bias"] == "af3":
        return af3_pair_bias(cfg["N"], heads, device).float()
    return torch.stack([c5_bias(cfg["N"], 5000 + b * cfg["H"] + h, device) for h in heads])


def svd_factors(cfg, heads, device):
    """Device SVD of every (b, h) dense bias at rank R (C4: exact cuSOLVER SVD of the
    shared pair bias, B=1; C5: batched randomized SVD per batch row) -> fp32
    factors [B, H_loc, N, R] + the reconstruction report (ref decompose.py:98-165)."""
    import torch

    import paper_2505_12044_b200 as fb
    from paper_2505_12044_b200.decompose import randomized_svd
    B, N, R = cfg["B"], cfg["N"], int(cfg["R"])
    fq = torch.empty(B, len(heads), N, R, device=device)
    fk = torch.empty_like(fq)
    worst = {"max_abs_err": 0.0, "rel_fro_err": 0.0, "energy_retained": 1.0}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in range(B):
        bias = dense_biases(cfg, heads, device, b)
        if cfg["bias"] == "af3":  # exact SVD (cuSOLVER, fp64) per head, like the reference's dgesdd
            u, s, vh = torch.linalg.svd(bias.double(), full_matrices=False)
            u, s, vh = u[..., :R], s[..., :R], vh[..., :R, :]
        else:  # randomized range finder (K7), batched over the heads of this batch row
            u, s, vh = randomized_svd(bias, R)
        root = s.sqrt()
        # the approximate factorisation emits bf16 factors: bf16-exact inputs need no split under
        # the Q' = [scale*q, U] fold (their rounding is part of the reported reconstruction error)
        fq[b] = (u * root[..., None, :]).to(torch.bfloat16).float()
        fk[b] = (vh.transpose(-1, -2) * root[..., None, :]).to(torch.bfloat16).float()
        diff = fq[b].double() @ fk[b].double().transpose(-1, -2) - bias.double()
        nb = bias.double().pow(2).sum((-1, -2))
        rel = (diff.pow(2).sum((-1, -2)) / nb).sqrt()
        energy = (s.double().pow(2).sum(-1) / nb)
        worst["max_abs_err"] = max(worst["max_abs_err"], float(diff.abs().amax()))
        worst["rel_fro_err"] = max(worst["rel_fro_err"], float(rel.max()))
        worst["energy_retained"] = min(worst["energy_retained"], float(energy.min()))
        if b == 0:
            first = {"max_abs_err": round(float(diff[0].abs().amax()), 8), "rel_fro_err": round(float(rel[0]), 8),
                     "energy_retained": round(float(energy[0]), 8)}
        del bias, diff
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    method = "cuSOLVER SVD (fp64)" if cfg["bias"] == "af3" else "randomized SVD (fp32, cuBLAS GEMM + QR)"
    fact = {"rank": R, "method": method, "factor_dtype": "bf16", "heads": B * len(heads),
            "device_seconds": round(secs, 3),
            "ours_worst_head": {k_: round(v_, 8) for k_, v_ in worst.items()}, "ours_head0": first}
    del fb
    return fq, fk, fact


def reference_svd_report(cfg, n_heads: int = 1):
    """The reference's own error on sampled heads: oracle svd_decompose (numpy
    LAPACK dgesdd, float64; restating ref decompose.py:98-138) of the same exact
    dense bias (head h of batch row 0), shown next to our device factors' error
    on that head.  Returns a thread that fills ``.result`` (LAPACK releases the
    GIL, so it overlaps the GPU timing; the biases are copied to the host first)."""
    import threading

    from oracle import flashbias_oracle as orc
    mats = [dense_biases(cfg, [h], "cuda", 0)[0].double().cpu().numpy() for h in range(n_heads)]
    R = int(cfg["R"])

    class _T(threading.Thread):
        result = None

        def run(self):
            out = []
            for h, b64 in enumerate(mats):
                t0 = time.perf_counter()
                _, _, rep = orc.svd_decompose(b64, rank=R)
                out.append(dict(head=h, seconds=round(time.perf_counter() - t0, 2),
                                **{k_: round(float(v_), 8) for k_, v_ in rep.items() if k_ != "rank_used"}))
            self.result = out

    t = _T(daemon=True)
    t.start()
    return t


def learnable(cfg) -> bool:
    """Bias learnable on both arms: C2's spatial weights by default, --learnable elsewhere."""
    return cfg["bwd"] and not cfg.get("static") and (cfg["bias"] == "spatial" or cfg.get("learnable", False))


def step_fn(cfg, inp, mode: str):
    """One pass of the hot path: forward (+ backward) through the public API."""
    import paper_2505_12044_b200 as fb
    mask = "causal" if cfg["causal"] else "none"
    q, k, v = inp["q"], inp["k"], inp["v"]
    if cfg["bwd"]:
        q.requires_grad_(True)
        k.requires_grad_(True)
        v.requires_grad_(True)
        if learnable(cfg) and mode == "flashbias":  # learnable bias: factor gradients dfq / dfk
            inp["fq"].requires_grad_(True)
            inp["fk"].requires_grad_(True)
        if learnable(cfg) and mode == "dense":  # the same bias learnable on the dense arm: dB = dS
            inp["dense"].requires_grad_(True)

    def run():
        if mode == "flashbias":
            out = fb.flashbias_attention(q, k, v, inp["fq"], inp["fk"], mask=mask)
        else:
            out = fb.tiled_attention(q, k, v, fb.DenseBias(inp["dense"]), mask=mask)
        if cfg["bwd"]:
            cands = (q, k, v, inp["fq"], inp["fk"]) if mode == "flashbias" else (q, k, v, inp["dense"])
            grads = [t for t in cands if t is not None and t.requires_grad]
            import torch
            torch.autograd.grad(out, grads, inp["do"])
        return out

    return run


def time_steps(fn, steps: int, warmup: int, dist=None, graph: bool = False, flush: bool = False):
    """CUDA-event timing of `steps` calls after `warmup` untimed ones, barrier +
    synchronize on both sides.  graph=True captures one step in a CUDA graph
    (after warm-up) and times its replays — for the microsecond-scale configs
    whose step would otherwise be bound by Python launch overhead.
    flush=True writes a 256 MB buffer (> the 126 MB L2) before every step,
    outside the events that bracket that step, so small configs are not timed
    from a warm L2; the per-step event intervals are summed."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        fn = g.replay
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if flush else None
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if flush:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            scratch.fill_(1)
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        total = sum(a.elapsed_time(b) for a, b in evs)
    else:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(steps):
            fn()
        stop.record()
        torch.cuda.synchronize()
        total = start.elapsed_time(stop)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    return total / steps


def kernel_breakdown(cfg, inp, reps: int = 3):
    """Time the forward and backward C-ABI calls separately with CUDA events
    on the launching stream (the dominant-kernel roofline)."""
    import torch

    from paper_2505_12044_b200 import _lib, attention as A
    mask_code = 1 if cfg["causal"] else 0
    d = cfg["d"]
    q, k, v, do = (t.detach() for t in (inp["q"], inp["k"], inp["v"], inp["do"]))
    scale = 1.0 / math.sqrt(d)
    plan = A.plan_factor_fold_cached(inp["fq"], inp["fk"], inp["fq"], inp["fk"], scale,
                                     max_cols=64 if d == 128 else 128)  # as the step
    split = plan.split
    uq, uk = A.prepare_factor_panels(inp["fq"].detach(), inp["fk"].detach(), plan.premul, split, q.dtype)
    if plan.q_fold:
        q = (q * scale).contiguous()
    scale = plan.kernel_scale
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    o = lse = None
    fwd_ms, bwd_ms = [], []
    for _ in range(reps + 1):
        ev[0].record()
        o, lse = A._fwd_launch(q, k, v, uq, uk, None, mask_code, scale)
        ev[1].record()
        if cfg["bwd"]:
            A._bwd_launch(q, k, v, uq, uk, None, o, lse, do, mask_code, scale, learnable(cfg))
        ev[2].record()
        torch.cuda.synchronize()
        fwd_ms.append(ev[0].elapsed_time(ev[1]))
        bwd_ms.append(ev[1].elapsed_time(ev[2]))
    out["fwd_ms"] = statistics.median(fwd_ms[1:])
    out["bwd_ms"] = statistics.median(bwd_ms[1:]) if cfg["bwd"] else 0.0
    out["split"] = split
    out["q_fold"] = plan.q_fold
    out["rpad"] = int(uq.shape[-1])
    del _lib
    return out


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist_mod

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = int(os.environ.get("BENCH_FORCE_DEVICE", local))  # functional multi-rank test on one GPU
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: functional test of >1 ranks on one GPU
        if backend == "nccl":
            dist_mod.init_process_group("nccl", device_id=device)
        else:
            dist_mod.init_process_group(backend)
        dist = dist_mod
    from paper_2505_12044_b200 import _lib
    lib = _lib.lib()

    total_bh = cfg["B"] * cfg["H"]
    per = (cfg["H"] + world - 1) // world  # head-major shards: whole heads per rank
    lo, hi = min(rank * per, cfg["H"]), min((rank + 1) * per, cfg["H"])
    inp = make_inputs(cfg, lo, hi, device)
    n_loc = (hi - lo) * cfg["B"]

    ref_svd = None
    if "factorisation" in inp and rank == 0 and world == 1 and args.ref_svd_heads > 0:
        ref_svd = reference_svd_report(cfg, args.ref_svd_heads)
    fn = step_fn(cfg, inp, "flashbias")
    use_graph = alg_flops(cfg, total_bh) < 20e9 and not args.no_graph
    in_bytes = cfg["N"] * cfg["d"] * (2 if cfg["dtype"] == "bf16" else 4) * 4 * n_loc
    flush = in_bytes < 2 * 126e6  # inputs not much larger than L2: flush before every timed step
    fn()  # one eager step: count this library's kernel launches per step
    torch.cuda.synchronize()
    lib.fb_launch_count(1)
    fn()
    torch.cuda.synchronize()
    launches_per_step = int(lib.fb_launch_count(1))
    prof = os.environ.get("BENCH_PROFILE_RANGE") == "1"  # profiles/run_ncu.sh: ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        ms = time_steps(fn, args.steps, args.warmup, dist, graph=use_graph, flush=flush)
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
    launches_timed = launches_per_step * args.steps
    if dist is not None:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist_mod.ReduceOp.MAX)
        ms = float(t)
    flops = alg_flops(cfg, total_bh)
    tflops = flops / (ms * 1e-3) / 1e12
    gather_ms = None
    if dist is not None:  # NCCL all-gather of O and dQ/dK/dV after the kernels (outside the hot loop)
        from paper_2505_12044_b200.sharding import gather_heads
        outs = [inp["q"].detach()] * (4 if cfg["bwd"] else 1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        ev0.record()
        for t in outs:
            gather_heads(t, cfg["H"])
        ev1.record()
        torch.cuda.synchronize()
        t = torch.tensor([ev0.elapsed_time(ev1)], device=device)
        dist.all_reduce(t, op=dist_mod.ReduceOp.MAX)
        gather_ms = float(t)

    # dense-bias baseline on the same pipeline (same step, bias tensor [1,H_loc,N,N])
    dense_ms = sdpa = None
    if cfg["dtype"] == "bf16" and not args.skip_dense:
        import paper_2505_12044_b200 as fb
        with torch.no_grad():
            n = cfg["N"]
            fqd = inp["fq"].detach()
            if "factorisation" in inp:  # C4/C5: the EXACT dense biases the factors approximate
                dense = torch.empty(cfg["B"], hi - lo, n, n, dtype=torch.bfloat16, device=device)
                for b in range(cfg["B"]):
                    dense[b] = dense_biases(cfg, inp["heads"], device, b).bfloat16()
            else:  # closed-form biases: materialised from the exact factors (K8)
                dense = torch.empty(fqd.shape[0], hi - lo, n, n, dtype=torch.bfloat16, device=device)
                fkd = inp["fk"].detach()
                D = _lib.desc
                _lib.check(lib.fb_dense_from_factors(_lib.ref(D(fqd.float().contiguous())),
                                                     _lib.ref(D(fkd.float().contiguous())),
                                                     _lib.ref(D(dense)), _lib.stream_ptr(device)))
        inp["dense"] = dense
        dfn = step_fn(cfg, inp, "dense")
        dense_ms = time_steps(dfn, max(1, args.steps), max(1, min(args.warmup, 2)), dist, graph=use_graph,
                              flush=flush)
        if dist is not None:
            t = torch.tensor([dense_ms], device=device)
            dist.all_reduce(t, op=dist_mod.ReduceOp.MAX)
            dense_ms = float(t)
        if not args.skip_sdpa and world == 1:
            sdpa = sdpa_dense(cfg, inp, max(1, min(args.steps, 5)), flush)
        del dense, inp["dense"]
        del fb
        torch.cuda.empty_cache()

    kb = kernel_breakdown(cfg, inp) if cfg["dtype"] == "bf16" else None
    pk, pk_kind = peaks()
    roofline = None
    if kb is not None:
        fwd_cfg = dict(cfg, bwd=False)
        fwd_flops_loc = alg_flops(fwd_cfg, n_loc)
        bwd_flops_loc = alg_flops(cfg, n_loc) - fwd_flops_loc
        dom = "bwd" if kb["bwd_ms"] >= kb["fwd_ms"] else "fwd"
        dom_flops = bwd_flops_loc if dom == "bwd" else fwd_flops_loc
        dom_ms = kb["bwd_ms"] if dom == "bwd" else kb["fwd_ms"]
        achieved = dom_flops / (dom_ms * 1e-3) / 1e12
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(args.config, {}).get(dom)
            if traffic is not None and n_loc != total_bh:  # captured at N=1: this rank's share of the heads
                traffic = traffic * n_loc / total_bh
        e = 2  # bf16 operands: the bwd reads q, k, v, dO and writes dq, dk, dv; the fwd reads q, k, v, writes o
        alg_bytes = (7 if dom == "bwd" else 4) * n_loc * cfg["N"] * cfg["d"] * e
        roofline = {
            "traffic_algorithmic": alg_bytes,
            "traffic_note": ("ncu dram__bytes_read+write of one launch (profiles/ncu_traffic.json); the bwd excess over "
                             "the algorithmic bytes is the fp32 dQ accumulator's zero-fill read and write-back"
                             if dom == "bwd" else "ncu dram__bytes_read+write of one launch"),
            "bound": "tensor", "kernel": "fb_attn_bwd (dKV+dQ)" if dom == "bwd" else "fb_attn_fwd (K1)",
            "achieved": round(achieved, 1), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": round(achieved / pk["bf16_tflops"], 4), "peak_kind": pk_kind,
            "frac_of_sustained": round(achieved / pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), 4),
            "frac_of_spec_2250": round(achieved / 2250.0, 4), "traffic": traffic,
            "fwd_ms": round(kb["fwd_ms"], 3), "bwd_ms": round(kb["bwd_ms"], 3),
            "fwd_tflops": round(fwd_flops_loc / (kb["fwd_ms"] * 1e-3) / 1e12, 1),
            "bwd_tflops": round(bwd_flops_loc / (kb["bwd_ms"] * 1e-3) / 1e12, 1) if cfg["bwd"] else None,
            "factor_split": kb["split"], "factor_rpad": kb["rpad"], "q_fold": kb["q_fold"],
        }

    if kb is None:  # C1: the fp32 SIMT forward is the whole step (one launch per step)
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12  # FFMA lanes x 2 flops x max SM clock
        roofline = {"bound": "fp32 FMA (SIMT, accurate fp32 products for the 1e-5 contract)",
                    "kernel": "fwd_simt_tiled (split-KV thread-block cluster, DSMEM combine)",
                    "achieved": round(tflops, 2), "peak": round(fp32_peak, 1), "unit": "TFLOP/s",
                    "frac": round(tflops / fp32_peak, 4),
                    "peak_kind": "nominal fp32 FFMA peak (148 SMs x 128 lanes x 2 x 1965 MHz); no measured fp32 peak",
                    "traffic": None}
    e2e = run_e2e(cfg, inp, args, device, chunks=args.e2e_chunks, dist=dist, total_bh=total_bh) \
        if not args.skip_e2e else None
    result = {
        "metric": METRIC, "value": round(tflops, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if cfg["dtype"] == "bf16" else "f32",
        "data": "synthetic (per-(b,h) seeded N(0,1) q/k/v/dO; closed-form ALiBi/spatial or seeded low-rank factors)",
        "config": {"workload": args.config, "desc": cfg["desc"], "B": cfg["B"], "H": cfg["H"], "N": cfg["N"],
                   "M": cfg["N"], "d": cfg["d"], "R": logical_rank(cfg), "causal": cfg["causal"],
                   "bwd": cfg["bwd"], "parallelism": f"bh-shard{world}",
                   "l2": ("L2 flushed (256 MB write) before every timed step, outside its events" if flush
                          else "inputs larger than L2 (no flush needed)")},
        "collective": None if dist is None else {
            "backend": dist.get_backend(), "nranks": world,
            "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if dist.get_backend() == "nccl" else None,
            "where": "after the kernels only: all-gather of O / dQ / dK / dV head slices (no data-path collective)"},
        "gather_ms_per_step": None if gather_ms is None else round(gather_ms, 3),
        "ms_per_step_with_gather": None if gather_ms is None else round(ms + gather_ms, 3),
        "dense_bias_ms_per_step": None if dense_ms is None else round(dense_ms, 3),
        "speedup_vs_dense_bias": None if dense_ms is None else round(dense_ms / ms, 3),
        "dense_bias_note": dense_note(cfg),
        "dense_bias_sdpa": sdpa,
        "factorisation": inp.get("factorisation"),
        "roofline": roofline,
        "clocks": clk.summary(),
        "gpu_launches": launches_timed,
        "cuda_graph": use_graph,
        "e2e": e2e,
    }
    if ref_svd is not None:
        ref_svd.join()
        result["factorisation"]["reference_svd_decompose"] = ref_svd.result
    if rank == 0 and world == 1 and not args.skip_cpu:
        result["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_seconds)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


def dense_note(cfg) -> str:
    if cfg.get("dense_unavailable"):
        return cfg["dense_unavailable"]
    base = "our dense-bias arm (K3/K4, same pipeline) streams the bias as a bf16 [Bb,H,N,N] tensor"
    if cfg.get("bias") == "alibi" and cfg["N"] > 4096:
        return (base + f"; with ALiBi at N={cfg['N']} |b| reaches ~{int(cfg['N'] * 0.84)}, where bf16 spacing is "
                "up to 64: this arm is timing-only, its outputs are not parity-checked")
    return base + "; the bias magnitudes of this workload are representable in bf16 to ~3 significant digits"


def sdpa_dense(cfg, inp, steps: int, flush: bool):
    """Cross-check of the dense-bias arm (not a strawman): torch
    SDPA with the same bias as a float attn_mask (causal folded in as -inf),
    fwd (+bwd), on the cuDNN and memory-efficient backends."""
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel
    q, k, v, do = (inp[n].detach() for n in ("q", "k", "v", "do"))
    mask = inp["dense"]
    if cfg["causal"]:
        n = cfg["N"]
        mask.masked_fill_(torch.ones(n, n, dtype=torch.bool, device=mask.device).triu_(1), float("-inf"))
    res = {"note": "torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=bias[+causal -inf])"}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
        qq, kk, vv = (t.clone().requires_grad_(cfg["bwd"]) for t in (q, k, v))

        def run():
            with sdpa_kernel([be]):
                o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, attn_mask=mask)
                if cfg["bwd"]:
                    torch.autograd.grad(o, (qq, kk, vv), do)
        try:
            res[f"{name}_ms"] = round(time_steps(run, steps, 2, None, flush=flush), 3)
        except Exception as e:  # noqa: BLE001 - report why a backend cannot run this config
            res[f"{name}_ms"] = None
            res[f"{name}_error"] = f"{type(e).__name__}: {str(e).splitlines()[0][:160]}"
        del qq, kk, vv
        torch.cuda.empty_cache()
    return res


def run_mixed(args):
    """Head-split mixed path vs all heads on the dense-bias kernel (same step, same heads)."""
    import torch

    import paper_2505_12044_b200 as fb
    cfg = MIX
    torch.cuda.set_device(0)
    H, N, d, low = cfg["H"], cfg["N"], cfg["d"], cfg["low"]
    side = int(round(math.sqrt(N)))  # 2048 tokens: 32 x 64 grid
    r = torch.arange(N, device="cuda") // 64
    c = torch.arange(N, device="cuda") % 64
    pos = torch.stack([r / (side - 1), c / 63.0, torch.zeros(N, device="cuda")], -1).double()
    g = torch.Generator(device="cuda")
    heads = []
    for h in range(H):
        g.manual_seed(4000 + h)
        if h < low:
            w = -(0.5 + 1.5 * torch.rand(N, generator=g, device="cuda", dtype=torch.float64))
            heads.append(fb.generate_bias(fb.SpatialDistanceBias(pos, pos, w), device="cuda"))
        else:
            heads.append(torch.randn(N, N, generator=g, device="cuda", dtype=torch.float64))
    perm = torch.randperm(H, generator=torch.Generator().manual_seed(1)).tolist()  # interleave the two kinds
    stack = torch.stack([heads[i] for i in perm])
    t0 = time.perf_counter()
    split = fb.split_heads_by_rank(stack, 0.999, max_rank=32)
    split_s = time.perf_counter() - t0
    # offline head permutation: low-rank heads first, so both subsets are contiguous views
    order = split.permutation()
    split = split.permuted()
    stack = stack[order]
    B = cfg["B"]
    q, k, v, do = (torch.randn(B, H, N, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    dense16 = stack.bfloat16()
    for t in (q, k, v):
        t.requires_grad_(True)

    def mixed():
        o = fb.mixed_head_attention(q, k, v, split, dense16)
        torch.autograd.grad(o, (q, k, v), do)

    def all_dense():
        o = fb.tiled_attention(q, k, v, fb.DenseBias(dense16.unsqueeze(0)))
        torch.autograd.grad(o, (q, k, v), do)

    # both arms CUDA-graph captured (a ~0.3 ms step would otherwise time the Python launch path)
    with ClockSampler(0) as clk:
        ms = time_steps(mixed, args.steps, args.warmup, graph=not args.no_graph, flush=True)
    dense_ms = time_steps(all_dense, args.steps, max(3, args.warmup), graph=not args.no_graph, flush=True)
    rr = split.common_rank
    nl, nd = len(split.low_indices), len(split.dense_indices)
    flops = B * N * N * (nl * (14 * d + 8 * rr) + nd * 14 * d)
    print(json.dumps({
        "metric": METRIC, "value": round(flops / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "dtype": "bf16", "data": "synthetic (seeded spatial-distance heads + N(0,1) full-rank heads)",
        "config": {"workload": "MIX", "desc": cfg["desc"], "B": B, "H": H, "N": N, "d": d, "low_heads": nl,
                   "dense_heads": nd, "common_rank": rr, "split_seconds": round(split_s, 2)},
        "all_dense_ms_per_step": round(dense_ms, 3), "speedup_vs_all_dense": round(dense_ms / ms, 3),
        "cuda_graph": not args.no_graph, "l2": "L2 flushed (256 MB write) before every timed step, outside its events",
        "clocks": clk.summary(),
    }))


def run_e2e(cfg, inp, args, device, chunks: int = 8, dist=None, total_bh=None):
    """Same step through the public API with HOST (pinned) buffers: H2D of
    q/k/v/dO and D2H of O (+ dQ/dK/dV) inside the timed region.

    The heads are processed in `chunks` slices, software-pipelined over three
    streams: H2D of slice i+1 (copy-in stream) and D2H of slice i-1 (copy-out
    stream) run while slice i computes, so PCIe in, PCIe out (full duplex) and
    the kernels overlap.  Every byte of every step still crosses PCIe."""
    import torch

    import paper_2505_12044_b200 as fb
    mask = "causal" if cfg["causal"] else "none"
    host = {n: inp[n].detach().to("cpu").pin_memory() for n in ("q", "k", "v", "do")}
    outs = {n: torch.empty_like(host["q"]).pin_memory() for n in (["o", "dq", "dk", "dv"] if cfg["bwd"] else ["o"])}
    fq, fk = inp["fq"].detach(), inp["fk"].detach()
    h2d = sum(t.numel() * t.element_size() for n, t in host.items() if cfg["bwd"] or n != "do")
    d2h = sum(t.numel() * t.element_size() for t in outs.values())
    B, H = host["q"].shape[0], host["q"].shape[1]
    if h2d < (256 << 20):  # small steps: per-slice launch overhead outweighs the copy overlap
        chunks = 1
    per_b = max(1, min(H, chunks // B))  # chunks never cross a batch row: every slice is contiguous memory
    bounds = [(b, H * i // per_b, H * (i + 1) // per_b) for b in range(B) for i in range(per_b)]
    chunks = len(bounds)
    names_in = ["q", "k", "v", "do"] if cfg["bwd"] else ["q", "k", "v"]
    dev = {n: torch.empty(host[n].shape, dtype=host[n].dtype, device=device) for n in names_in}
    res = {n: torch.empty(host["q"].shape, dtype=host["q"].dtype, device=device) for n in outs}
    s_in, s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
    comp = torch.cuda.current_stream(device)

    def fslice(t, bb, a, b):
        t = t[min(bb, t.shape[0] - 1): min(bb, t.shape[0] - 1) + 1]
        return t if t.shape[1] == 1 else t[:, a:b]

    def step():
        ev_in = []
        for bb, a, b in bounds:  # all H2D slices queued on the copy-in stream, one event each
            with torch.cuda.stream(s_in):
                for n in names_in:
                    dev[n][bb:bb + 1, a:b].copy_(host[n][bb:bb + 1, a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
            ev_in.append(e)
        for (bb, a, b), e in zip(bounds, ev_in):
            comp.wait_event(e)
            q = dev["q"][bb:bb + 1, a:b].requires_grad_(cfg["bwd"])
            k = dev["k"][bb:bb + 1, a:b].requires_grad_(cfg["bwd"])
            v = dev["v"][bb:bb + 1, a:b].requires_grad_(cfg["bwd"])
            o = fb.flashbias_attention(q, k, v, fslice(fq, bb, a, b), fslice(fk, bb, a, b), mask=mask)
            res["o"][bb:bb + 1, a:b].copy_(o.detach())
            if cfg["bwd"]:
                gq, gk, gv = torch.autograd.grad(o, (q, k, v), dev["do"][bb:bb + 1, a:b])
                res["dq"][bb:bb + 1, a:b].copy_(gq)
                res["dk"][bb:bb + 1, a:b].copy_(gk)
                res["dv"][bb:bb + 1, a:b].copy_(gv)
            e2 = torch.cuda.Event()
            e2.record(comp)
            s_out.wait_event(e2)
            with torch.cuda.stream(s_out):
                for n in outs:
                    outs[n][bb:bb + 1, a:b].copy_(res[n][bb:bb + 1, a:b], non_blocking=True)
        comp.wait_stream(s_out)  # the step ends when the last D2H lands

    steps = max(1, min(args.steps, 5))
    ms = time_steps(step, steps, 1, dist)
    world = 1
    if dist is not None:  # whole job: every rank moves its own heads over its own PCIe link; max over ranks
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        world = dist.get_world_size()
        tb = torch.tensor([h2d, d2h], dtype=torch.float64, device=device)
        dist.all_reduce(tb)
        h2d, d2h = int(tb[0]), int(tb[1])
    flops = alg_flops(cfg, total_bh if total_bh is not None else inp["q"].shape[0] * inp["q"].shape[1])
    return {"value": round(flops / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s", "ms_per_step": round(ms, 2),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "head_chunks": chunks,
            "ranks": world,
            "path": "flashbias_attention (public API) on head slices of pinned host tensors, autograd backward; "
                    "H2D / compute / D2H software-pipelined over three streams"}


# ---------------------------------------------------------------------------- CPU arm
# The reference is pure numpy (no compiled code to build into oracle/_ref), so
# the CPU arm runs the oracle port of its streaming loop: streaming_attention
# (ref attention.py:140-202, the flashbias_attention path 205-230) for the
# forward and the query-blocked analytic backward (no reference backward:
# SPEC.md:183) on the SAME bf16-rounded inputs the GPU arm uses (seeded per
# (b, h) exactly like make_inputs), one head sample per single-threaded worker
# process (the reference CLI's default BLAS pinning, cli.py:28-37).

def _pin_blas():
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # noqa: BLE001
        pass


def _head_inputs(cfg, b: int, h: int, seed: int = 1234):
    """q, k, v, dO [N, d] of head (b, h) as float64 numpy arrays holding the GPU
    arm's bf16 values (same per-(b,h) seed and draw order as make_inputs; falls
    back to the CPU generator when no GPU is visible) + the factors."""
    import numpy as np
    import torch
    N, d, H = cfg["N"], cfg["d"], cfg["H"]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g = torch.Generator(device=dev).manual_seed(seed + b * H + h)
    qkvd = []
    for _ in range(4):
        t = torch.empty(N, d, device=dev).normal_(generator=g)
        qkvd.append((t if cfg["dtype"] == "fp32" else t.bfloat16()).double().cpu().numpy())
    from oracle import flashbias_oracle as orc
    if cfg["bias"] == "alibi":
        fq, fk = orc.decompose_alibi(N, N, alibi_slopes(H)[h])
    elif cfg["bias"] == "spatial":
        side = int(round(math.sqrt(N)))
        r, c = np.arange(N) // side, np.arange(N) % side
        pos = np.stack([r / (side - 1), c / (side - 1), np.zeros(N)], -1)
        from paper_2505_12044_b200.rng import Rng
        fq, fk = orc.decompose_spatial(pos, pos, -(0.5 + 1.5 * Rng(2000 + h).uniform(N)))
    else:  # SVD configs: rank-R factors of the same shape (values do not change the timed work)
        rng = np.random.default_rng(seed + b * H + h)
        fq, fk = rng.standard_normal((N, cfg["R"])) * 0.1, rng.standard_normal((N, cfg["R"])) * 0.1
    return qkvd, fq, fk


def _cpu_sample(payload):
    """One bounded sample in a worker: the last ``rows`` query rows of head
    (b, h) (causal: the rows that see the most keys) against all the keys they
    see, forward (streaming loop) + backward when the config has one."""
    path, cfg, rows = payload
    import numpy as np

    from oracle import flashbias_oracle as orc
    z = np.load(path)
    q, k, v, do, fq, fk = (z[n] for n in ("q", "k", "v", "do", "fq", "fk"))
    n, d = q.shape
    r0 = n - rows
    mask = "causal" if cfg["causal"] else "none"
    prem, scale = math.sqrt(d), 1.0 / math.sqrt(d)
    t0 = time.perf_counter()
    orc.streaming_attention(q[r0:], k, v, fq=fq[r0:], fk=fk, premul=prem, mask=mask, scale=scale, row0=r0)
    if cfg["bwd"]:
        orc.blocked_attention_fwd_bwd(q[r0:], k, v, do[r0:], fq=fq[r0:], fk=fk, premul=prem, mask=mask,
                                      scale=scale, block=256, row0=r0)
    return time.perf_counter() - t0, list(range(r0, n))


class CpuArm:
    """Spawn pool of single-threaded workers on all host cores; worker i runs
    head i (head-major (h, b) order) of the config on the GPU arm's inputs."""

    def __init__(self, cfg, workers: int = None):
        import multiprocessing as mp
        import tempfile

        import numpy as np
        self.cfg = cfg
        self.cores = workers or len(os.sched_getaffinity(0))
        self.dir = tempfile.mkdtemp(prefix="fb_cpu_arm_")
        self.paths = []
        B = cfg["B"]
        for i in range(self.cores):
            h, b = (i // B) % cfg["H"], i % B
            (q, k, v, do), fq, fk = _head_inputs(cfg, b, h)
            path = os.path.join(self.dir, f"head{i}.npz")
            np.savez(path, q=q, k=k, v=v, do=do, fq=fq, fk=fk)
            self.paths.append(path)
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_pin_blas)

    def step(self, rows: int):
        """Wall time and algorithmic FLOPs of one sample step (every worker one head sample)."""
        rows = min(rows, self.cfg["N"])
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_sample, [(p, self.cfg, rows) for p in self.paths])
        wall = time.perf_counter() - t0
        return wall, sum(alg_flops(self.cfg, 1, rows=r) for _, r in res)

    def close(self):
        import shutil
        self.pool.close()
        self.pool.join()
        shutil.rmtree(self.dir, ignore_errors=True)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, budget_s: float = 15.0, rows: int = 512):
    arm = CpuArm(cfg)
    try:
        arm.step(min(rows, 64))  # warm-up (imports, BLAS init)
        wall, flops = arm.step(rows)
    finally:
        arm.close()
    return {"value": flops / wall / 1e12, "unit": "TFLOP/s", "cores": arm.cores, "kind": "port",
            "cpu_model": _cpu_model(),
            "sample": f"{arm.cores} heads x last {rows} query rows of {cfg['desc']} (all keys they see), the GPU "
                      f"arm's bf16 inputs, fwd = oracle streaming loop (ref attention.py:140-230), bwd = "
                      f"query-blocked analytic restatement (no reference backward), one single-threaded process "
                      f"per core, measured wall {wall:.2f}s"}


def run_reference(args, cfg):
    """--impl reference: the reference algorithm's CPU rate on this host.  Each
    timed step is a bounded, measured sample (every core one head's last
    ``rows`` query rows, fwd + bwd); ms_per_step is that measured step, not an
    extrapolation.  The whole-config time is reported separately from one
    fully measured head per core (per-head medians)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows = {"C1": 1024, "C2": 512, "C3": 512, "C4": 768, "C5": 256}.get(args.config, 256)
    arm = CpuArm(cfg)
    try:
        for _ in range(args.warmup):
            arm.step(rows)
        walls, flops = [], 0.0
        for _ in range(args.steps):
            w, flops = arm.step(rows)
            walls.append(w)
        full = None
        if args.ref_full_heads:
            fw, ff = arm.step(cfg["N"])  # every core one WHOLE head, measured
            full = {"per_head_s": round(fw, 2), "heads_per_step": arm.cores,
                    "tflops": round(ff / fw / 1e12, 5),
                    "whole_config_s_at_this_rate": round(alg_flops(cfg, cfg["B"] * cfg["H"]) / (ff / fw), 1)}
    finally:
        arm.close()
    ms = statistics.median(walls) * 1e3
    value = flops / (ms * 1e-3) / 1e12
    sample = (f"per step: {arm.cores} heads x last {rows} query rows of {cfg['desc']}, the GPU arm's bf16 inputs, "
              f"oracle streaming loop fwd + blocked analytic bwd, float64 numpy, one single-threaded process per "
              f"core ({_cpu_model()})")
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": True,
        "impl": "reference", "dtype": "f64", "data": "synthetic (the GPU arm's seeded bf16 inputs)",
        "config": {"workload": args.config, "desc": cfg["desc"], "rows_per_head_sample": rows},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": arm.cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "full_heads": full,
        "note": "ms_per_step is the measured sample step (no extrapolation); full_heads times whole heads",
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS) + ["MIX"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-sdpa", action="store_true", help="skip the torch SDPA (cuDNN) dense-bias cross-check")
    ap.add_argument("--rank", type=int, default=None, help="C4/C5: SVD rank R (C5 sweep 8..64)")
    ap.add_argument("--ref-svd-heads", type=int, default=1,
                    help="C4/C5: heads whose reference (LAPACK) SVD error is reported next to ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-full-heads", type=int, default=1,
                    help="--impl reference: also time one whole head per core (per-head medians)")
    ap.add_argument("--no-graph", action="store_true", help="never CUDA-graph the step (small configs use graphs)")
    ap.add_argument("--learnable", action="store_true",
                    help="C4/C5: learnable bias on both arms (FlashBias dfq/dfk vs dense dB); C2 is learnable by default")
    ap.add_argument("--e2e-chunks", type=int, default=32,
                    help="head slices the e2e step is software-pipelined over (H2D / compute / D2H)")
    ap.add_argument("--static-factors", action="store_true",
                    help="C2: treat the spatial bias as fixed on both arms (no factor / bias gradients)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.config == "MIX":
        if args.impl == "ours":
            run_mixed(args)
        return
    cfg = dict(CONFIGS[args.config])
    if args.rank is not None:
        if "R" not in cfg:
            ap.error("--rank applies to the SVD configs C4/C5")
        cfg["R"] = args.rank
    if args.learnable:
        if args.config == "C3":  # FlashBias arm only: learnable ALiBi factors (the 128x128-tile LEARN kernel)
            args.skip_dense = True
            cfg["dense_unavailable"] = ("learnable dense arm not run: C3's dB = dS is a [4,32,16384,16384] bf16 "
                                        "buffer (68 GB) per step")
        cfg["learnable"] = True
        cfg["bwd"] = True
        cfg["desc"] += " [learnable bias: FlashBias dfq/dfk vs dense dB]"
    if args.static_factors:
        cfg["static"] = True
        cfg["desc"] += " [static factors: no factor gradients]"
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
