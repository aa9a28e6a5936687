"""Timeline of one CTA of the backward kernel (FB_TRACE build):
python tests/gpu_probe/trace_bwd.py [cta] [H] [first_block] [nblocks]"""
import ctypes, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), os.environ.get("TRACE_LIB", "libflashbias_b200_trace.so"))  # debug build
lib = _lib.lib()
lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 40
H = int(sys.argv[2]) if len(sys.argv) > 2 else 4
j0 = int(sys.argv[3]) if len(sys.argv) > 3 else 10
nb = int(sys.argv[4]) if len(sys.argv) > 4 else 3
B, N, D = 1, 16384, 128
q, k, v, do = (torch.randn(B, H, N, D, device="cuda").bfloat16() for _ in range(4))
slopes = [-(2.0 ** (-8.0 * (i + 1) / 32)) for i in range(H)]
fq, fk = fb.alibi_factors(slopes, N, N)
buf = torch.zeros(32 * 2048, dtype=torch.int64, device="cuda")
q.requires_grad_(True); k.requires_grad_(True); v.requires_grad_(True)
o = fb.flashbias_attention(q, k, v, fq, fk, mask="causal")
torch.autograd.grad(o, (q, k, v), do, retain_graph=True)
torch.cuda.synchronize()
buf.zero_(); lib.fb_debug_set_trace(buf.data_ptr(), cta)
torch.autograd.grad(o, (q, k, v), do)
torch.cuda.synchronize()
lib.fb_debug_set_trace(None, -1)
a = buf.view(32, 2048).cpu()
ev = [(int(a[e, i]), e, i) for e in range(32) for i in range(2048) if a[e, i] != 0]
t0 = min(x[0] for x in ev)
tl = sorted((t - t0, e, i) for t, e, i in ev)
names = {10: "mma dV", 11: "mma S", 12: "mma dK", 13: "mma dQ", 14: "mma dP", 15: "A0 start", 16: "A0 end",
         17: "B0 start", 18: "B0 end", 22: "A1 start", 23: "A1 end", 24: "B1 start", 25: "B1 end",
         19: "drain start", 20: "drain end", 21: "load dO"}
print(f"span {tl[-1][0]} cycles, {len(tl)} events")
prev = None
for t, e, i in tl:
    if j0 <= i < j0 + nb and e < 26:
        print(f"{t:9d} {'+%d' % (t - prev) if prev is not None else '':>7s} {str(names.get(e, e)):12s} {i}")
        prev = t
per = collections.defaultdict(dict)
for t, e, i in tl:
    per[e][i] = t
def avg(e0, e1):
    xs = [per[e1][i] - per[e0][i] for i in per[e0] if i in per[e1]]
    return sum(xs) / max(1, len(xs))
print("A0 %.0f  A1 %.0f  B0 %.0f  B1 %.0f  drain %.0f" % (avg(15, 16), avg(22, 23), avg(17, 18), avg(24, 25), avg(19, 20)))
s = sorted(per[11].values())
print("period (S issue) %.1f cycles over %d blocks" % ((s[-1] - s[0]) / max(1, len(s) - 1), len(s)))

# per-chunk drain breakdown (events 26..30 of the leader drain thread, index j*8+c)
import statistics as _st
def seg(e0, e1):
    xs = [per[e1][i] - per[e0][i] for i in per.get(e0, {}) if i in per.get(e1, {})]
    return _st.median(xs) if xs else float("nan")
print("drain chunk medians: wait_read %.0f  bar1+sts %.0f  fence %.0f  bar2 %.0f  issue->next %.0f" % (
    seg(26, 27), seg(27, 28), seg(28, 29), seg(29, 30),
    _st.median([per[26][i + 1] - per[30][i] for i in per.get(30, {}) if i + 1 in per.get(26, {})] or [float("nan")])))
