import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, math
import paper_2505_12044_b200 as fb
H, N, d = 16, 2048, 64
g = torch.Generator(device="cuda")
heads = []
for h in range(H):
    g.manual_seed(4000 + h)
    heads.append(torch.randn(N, 8, device="cuda", generator=g, dtype=torch.float64) @ torch.randn(8, N, device="cuda", generator=g, dtype=torch.float64) if h < 12 else torch.randn(N, N, generator=g, device="cuda", dtype=torch.float64))
stack = torch.stack(heads)
split = fb.split_heads_by_rank(stack, 0.999, max_rank=32)
print("split", split.low_indices, split.common_rank)
q, k, v, do = (torch.randn(H, N, d, device="cuda", generator=g).bfloat16() for _ in range(4))
dense16 = stack.bfloat16()
for t in (q, k, v): t.requires_grad_(True)
def mixed():
    o = fb.mixed_head_attention(q, k, v, split, dense16)
    torch.autograd.grad(o, (q, k, v), do)
for _ in range(3): mixed()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3): mixed()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15))
