import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2505_12044_b200 as fb
for (n, m, c) in ((5, 6, 3), (4, 4, 2), (24, 20, 4), (128, 128, 16), (130, 136, 16), (130, 130, 16)):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(n, c, device="cuda", generator=g).bfloat16()
    k = torch.randn(m, c, device="cuda", generator=g).bfloat16()
    v = torch.randn(m, c, device="cuda", generator=g).bfloat16()
    b = torch.randn(n, m, device="cuda", generator=g).bfloat16()
    o = fb.tiled_attention(q, k, v, fb.DenseBias(b))
    o0 = fb.tiled_attention(q, k, v, fb.DenseBias(torch.zeros_like(b)))
    onb = fb.tiled_attention(q, k, v)
    s = q.double() @ k.double().T / c ** 0.5
    ref = torch.softmax(s + b.double(), -1) @ v.double()
    ref0 = torch.softmax(s, -1) @ v.double()
    print(n, m, c, "bias err", float((o.double() - ref).abs().max()), "zero-bias err", float((o0.double() - ref0).abs().max()),
          "nobias err", float((onb.double() - ref0).abs().max()))
