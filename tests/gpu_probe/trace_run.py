"""Timeline of one CTA of the fwd and fused bwd kernels (FB_TRACE build).
python tests/gpu_probe/trace_run.py [cta] [H]"""
import ctypes, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), "libflashbias_b200_trace.so")  # debug build
lib = _lib.lib()
lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 40
H = int(sys.argv[2]) if len(sys.argv) > 2 else 4
head0 = int(sys.argv[3]) if len(sys.argv) > 3 else 16
B, N, D = 1, 16384, 128
q, k, v, do = (torch.randn(B, H, N, D, device="cuda").bfloat16() for _ in range(4))
slopes = [-(2.0 ** (-8.0 * (head0 + i + 1) / 32)) for i in range(H)]
fq, fk = fb.alibi_factors(slopes, N, N)
buf = torch.zeros(32 * 2048, dtype=torch.int64, device="cuda")

def grab():
    torch.cuda.synchronize()
    lib.fb_debug_set_trace(None, -1)
    a = buf.view(32, 2048).cpu()
    ev = [(int(a[e, i]), e, i) for e in range(32) for i in range(2048) if a[e, i] != 0]
    t0 = min(x[0] for x in ev)
    return sorted((t - t0, e, i) for t, e, i in ev)

q.requires_grad_(True); k.requires_grad_(True); v.requires_grad_(True)
o = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
torch.autograd.grad(o, (q, k, v), do)
torch.cuda.synchronize()
buf.zero_(); lib.fb_debug_set_trace(buf.data_ptr(), cta)
o = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
fwd = grab()
buf.zero_(); lib.fb_debug_set_trace(buf.data_ptr(), cta)
torch.autograd.grad(o, (q, k, v), do)
bwd = grab()

names = {2: "MMA S", 3: "MMA PV", 4: "load", 5: "sm start", 6: "sm end(w0)", 10: "mma dV", 11: "mma ST(c+1)",
         12: "mma dK", 13: "mma dQT", 14: "mma dPT(c+1)", 15: "A start", 16: "A end(w0)", 17: "B start",
         18: "B end(w0)", 19: "drain start", 20: "drain end", 21: "load"}
import json as _json
_json.dump({"fwd": fwd, "bwd": bwd}, open(os.environ.get("TRACE_DUMP", "gpurun_out/trace_events.json"), "w"))
for nm, tl in (("fwd", fwd), ("bwd", bwd)):
    print(f"===== {nm}: {len(tl)} events, span {tl[-1][0]} cycles")
    for t, e, a in tl[: 90 if nm == "fwd" else 120]:
        if 22 <= e <= 29:
            continue
        print(f"{t:9d} {str(names.get(e, e)):13s} {a}")
d = collections.defaultdict(dict)
for t, e, a in fwd:
    d[a][e] = t
sm = [v[6] - v[5] for v in d.values() if 5 in v and 6 in v]
slow = [max(v.get(22 + w, 0) for w in range(4)) - v[5] for v in d.values() if 5 in v and 22 in v]
print("fwd softmax per block (warp0):", sum(sm) / len(sm), " slowest warp:", sum(slow) / max(1, len(slow)))
st = sorted(t for t, e, a in fwd if e == 5)
print("fwd mean gap between softmax starts (alternating tiles):", (st[-1] - st[0]) / (len(st) - 1))
mma = sorted(t for t, e, a in fwd if e in (2, 3))
print("fwd MMA issue events:", len(mma))
d = collections.defaultdict(dict)
for t, e, a in bwd:
    d[a][e] = t
A = [v[16] - v[15] for v in d.values() if 15 in v and 16 in v]
Bp = [v[18] - v[17] for v in d.values() if 17 in v and 18 in v]
print("bwd phase A (w0)", sum(A) / len(A), "| phase B (w0)", sum(Bp) / len(Bp))
a0 = sorted(t for t, e, a in bwd if e == 15)
print("bwd block period", (a0[-1] - a0[0]) / (len(a0) - 1), "blocks", len(a0))
