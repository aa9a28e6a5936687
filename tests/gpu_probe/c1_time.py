"""C1 (fp32 SIMT forward) time and parity for a library variant:
FLASHBIAS_B200_VARIANT=<name> python tests/gpu_probe/c1_time.py [N] [D]
Prints the median per-call device time (L2 flushed before each call, outside the
events) and the max relative error against a float64 torch evaluation."""
import json, math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2505_12044_b200 import _lib
if os.environ.get("FLASHBIAS_B200_VARIANT"):
    _lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), "libflashbias_b200_%s.so" % os.environ["FLASHBIAS_B200_VARIANT"])
import paper_2505_12044_b200 as fb
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
D = int(sys.argv[2]) if len(sys.argv) > 2 else 64
H = 8
torch.manual_seed(0)
q, k, v = (torch.randn(1, H, N, D, device="cuda") for _ in range(3))
slopes = [2.0 ** (-8.0 * (h + 1) / H) for h in range(H)]
fq, fk = fb.alibi_factors(slopes, N, N)
fq, fk = fq.float(), fk.float()
out = fb.flashbias_attention(q, k, v, fq, fk)
qd, kd, vd = q.double(), k.double(), v.double()
logits = qd @ kd.transpose(-1, -2) / math.sqrt(D) + fq.double() @ fk.double().transpose(-1, -2)
ref = logits.softmax(-1) @ vd
err = float((out.double() - ref).abs().max() / ref.abs().max())
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(40):
    scratch.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fb.flashbias_attention(q, k, v, fq, fk)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
print(json.dumps({"variant": os.environ.get("FLASHBIAS_B200_VARIANT", ""), "N": N, "D": D,
                  "ms": round(statistics.median(ts), 4), "rel_err": err}))
