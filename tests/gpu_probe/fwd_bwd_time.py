"""Time the C3 forward and forward+backward separately (CUDA events, median
of reps) for quick A/B runs of library variants (FLASHBIAS_B200_VARIANT)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2505_12044_b200 as fb
from paper_2505_12044_b200 import _lib
# probe only: load _lib/libflashbias_b200_<name>.so -- before ANY library call (make_inputs builds the
# ALiBi factors on the device through the library; the path is read once, at the first load)
if os.environ.get("FLASHBIAS_B200_VARIANT"):
    _lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), "libflashbias_b200_%s.so" % os.environ["FLASHBIAS_B200_VARIANT"])
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
inp = bench.make_inputs(cfg, 0, cfg["H"], torch.device("cuda"))
mask = "causal" if cfg["causal"] else "none"
q, k, v = inp["q"], inp["k"], inp["v"]
def fwd():
    with torch.no_grad():
        fb.flashbias_attention(q, k, v, inp["fq"], inp["fk"], mask=mask)
step = bench.step_fn(cfg, inp, "flashbias")
def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)
f = timeit(fwd)
s = timeit(step)
fl_f = bench.alg_flops(dict(cfg, bwd=False), cfg["B"] * cfg["H"])
fl_s = bench.alg_flops(cfg, cfg["B"] * cfg["H"])
assert _lib.lib()._name == _lib.LIB_PATH, "variant library not loaded"
print(json.dumps({"variant": os.environ.get("FLASHBIAS_B200_VARIANT", ""), "fwd_ms": round(f, 3),
                  "fwd_tflops": round(fl_f / f / 1e9, 1), "step_ms": round(s, 3), "step_tflops": round(fl_s / s / 1e9, 1),
                  "bwd_ms_est": round(s - f, 3)}))
