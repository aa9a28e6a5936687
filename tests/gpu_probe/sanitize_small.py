"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck):
one forward + backward through every kernel family (d = 32/64/128, factored,
dense, no bias, causal, factor gradients, the 128x128-tile and fused
backwards, the deterministic two-kernel backward, the fp32 SIMT forward).
    compute-sanitizer --tool memcheck python tests/gpu_probe/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2505_12044_b200 as fb

torch.manual_seed(0)
cases = []
for D in (32, 64, 128):
    for causal in (False, True):
        for kind in ("factored", "dense", "none", "learn", "det"):
            cases.append((D, causal, kind))
for D, causal, kind in cases:
    N = 256 if D == 128 else 192
    q, k, v, do = (torch.randn(1, 2, N, D, device="cuda").bfloat16() for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)
    mask = "causal" if causal else "none"
    fq = (torch.randn(1, 2, N, 2, device="cuda") * 0.3)
    fk = (torch.randn(1, 2, N, 2, device="cuda") * 0.3)
    wrt = [q, k, v]
    if kind == "dense":
        o = fb.tiled_attention(q, k, v, fb.DenseBias(torch.randn(1, 2, N, N, device="cuda")), mask=mask)
    elif kind == "none":
        o = fb.tiled_attention(q, k, v, mask=mask)
    else:
        if kind == "learn":
            fq.requires_grad_(True)
            fk.requires_grad_(True)
            wrt += [fq, fk]
        o = fb.flashbias_attention(q, k, v, fq, fk, mask=mask, deterministic=(kind == "det"))
    torch.autograd.grad(o, wrt, do)
    torch.cuda.synchronize()
    print("ok", D, mask, kind, flush=True)
# fp32 SIMT forward: split-KV clusters of 2 (N=200) and 4 (N=1024, the C1 shape), causal and ragged
for n, causal in ((200, False), (1024, False), (333, True)):
    qf, kf, vf = (torch.randn(1, 2, n, 64, device="cuda") for _ in range(3))
    fb.flashbias_attention(qf, kf, vf, torch.randn(1, 2, n, 2, device="cuda"), torch.randn(1, 2, n, 2, device="cuda"),
                           mask="causal" if causal else "none")
    torch.cuda.synchronize()
    print("ok fp32", n, causal, flush=True)
print("SANITIZE_WORKLOAD_DONE")
