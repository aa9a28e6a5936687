"""In-situ kernel timeline of the C3 (or given) bench step via torch.profiler
(CUPTI activity records, steady state after warm-up): per-kernel device time
per step and the idle gap between kernels.  python tests/gpu_probe/step_profile.py [C3]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import bench

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"])
inp = bench.make_inputs(cfg, 0, cfg["H"], torch.device("cuda"))
step = bench.step_fn(cfg, inp, "flashbias")
for _ in range(5):
    step()
torch.cuda.synchronize()
steps = 6
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in evs:
    tot[e.name[:60]] += e.time_range.elapsed_us()
    cnt[e.name[:60]] += 1
span = (evs[-1].time_range.end - evs[0].time_range.start) / steps
busy = sum(tot.values()) / steps
gaps = []
for a, b in zip(evs, evs[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 5:
        gaps.append((round(g, 1), a.name[:40], b.name[:40]))
print(json.dumps({"step_us": round(span, 1), "busy_us": round(busy, 1),
                  "kernels_us_per_step": {k: round(v / steps, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1])},
                  "counts": dict(cnt), "largest_gaps_us": sorted(gaps, reverse=True)[:12]}, indent=1))
