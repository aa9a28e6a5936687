"""Run one small backward case on a library variant and report errors / mbarrier
reports: FLASHBIAS_B200_VARIANT=<name> python tests/gpu_probe/variant_case.py B H N D causal"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2505_12044_b200 import _lib
if os.environ.get("FLASHBIAS_B200_VARIANT"):
    _lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), "libflashbias_b200_%s.so" % os.environ["FLASHBIAS_B200_VARIANT"])
import paper_2505_12044_b200 as fb
B, H, N, D, causal = (int(x) for x in sys.argv[1:6])
torch.manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, D, device="cuda").bfloat16() for _ in range(4))
for t in (q, k, v):
    t.requires_grad_(True)
o = fb.tiled_attention(q, k, v, mask="causal" if causal else "none")
o.backward(do)
torch.cuda.synchronize()
r = [t.detach().double().requires_grad_(True) for t in (q, k, v)]
s = r[0] @ r[1].transpose(-1, -2) / D ** 0.5
if causal:
    s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
(s.softmax(-1) @ r[2]).backward(do.double())
for name, a, b in zip("qkv", (q, k, v), r):
    print(name, float((a.grad.double() - b.grad).abs().max() / b.grad.abs().max()))
