"""Timeline of one CTA of the fwd and fused bwd kernels (FB_TRACE build).
FLASHBIAS_B200_TRACE=1 python tests/gpu_probe/trace_run.py [cta]"""
import ctypes, os, sys, collections
os.environ["FLASHBIAS_B200_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import _lib
lib = _lib.lib()
lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
B, H, N, D = 1, 4, 16384, 128
q, k, v, do = (torch.randn(B, H, N, D, device="cuda").bfloat16() for _ in range(4))
slopes = [-(2.0 ** (-8.0 * (i + 1) / 32)) for i in range(H)]
fq, fk = fb.alibi_factors(slopes, N, N)
buf = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 40

def run(which):
    buf.zero_()
    q.requires_grad_(True); k.requires_grad_(True); v.requires_grad_(True)
    o = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")  # warm
    torch.autograd.grad(o, (q, k, v), do)
    torch.cuda.synchronize()
    lib.fb_debug_set_trace(buf.data_ptr(), cta)
    o = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
    if which == "bwd":
        lib.fb_debug_set_trace(None, -1)
        torch.cuda.synchronize(); buf.zero_()
        lib.fb_debug_set_trace(buf.data_ptr(), cta)
        torch.autograd.grad(o, (q, k, v), do)
    torch.cuda.synchronize()
    lib.fb_debug_set_trace(None, -1)
    n = int(buf[0]); recs = buf[1:n + 1].cpu().tolist()
    ev = [((r >> 56) & 0xff, (r >> 40) & 0xffff, r & 0xffffffffff) for r in recs]
    t0 = min(e[2] for e in ev)
    return sorted([(e[2] - t0, e[0], e[1]) for e in ev])

names = {2: "MMA S", 3: "MMA PV", 10: "sm start", 11: "sm end", 20: "load", 30: "mma dV", 31: "mma ST", 32: "mma dK",
         33: "mma dQT", 34: "mma dPT", 40: "A start", 41: "A end", 42: "B start", 43: "B end", 50: "drain start",
         51: "drain end", 60: "load"}
for which in ("fwd", "bwd"):
    tl = run(which)
    print(f"===== {which}: {len(tl)} events, span {tl[-1][0]} cycles")
    for t, e, a in tl[:70]:
        print(f"{t:9d} {names.get(e, e):12s} {a}")
    # interval stats
    starts = collections.defaultdict(dict)
    if which == "fwd":
        for t, e, a in tl:
            if e in (10, 11): starts[(a >> 12, a & 4095)][e] = t
        d = [v[11] - v[10] for v in starts.values() if 10 in v and 11 in v]
        print("softmax per block: mean", sum(d) / len(d), "min", min(d), "max", max(d))
        sm = sorted(t for t, e, a in tl if e == 10)
        print("mean period between softmax starts (both tiles):", (sm[-1] - sm[0]) / (len(sm) - 1))
    else:
        for t, e, a in tl:
            if e in (40, 41, 42, 43): starts[a][e] = t
        A = [v[41] - v[40] for v in starts.values() if 40 in v and 41 in v]
        Bd = [v[43] - v[42] for v in starts.values() if 42 in v and 43 in v]
        wait = [v[42] - v[41] for v in starts.values() if 41 in v and 42 in v]
        print("phase A mean", sum(A) / len(A), "phase B mean", sum(Bd) / len(Bd), "wait A->B", sum(wait) / len(wait))
        a0 = sorted(t for t, e, a in tl if e == 40)
        print("block period", (a0[-1] - a0[0]) / (len(a0) - 1), "blocks", len(a0))
