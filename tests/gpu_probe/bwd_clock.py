"""Effective SM clock and cycles per 128x128 block inside the C3 backward (t128
kernel built with -DT128_EXP_CLOCKS: each CTA records clock64 / globaltimer at
start and end).  Cold = after 3 s idle; hot = after 4 s of back-to-back steps.
python tests/gpu_probe/bwd_clock.py   (needs _lib/libflashbias_b200_clk.so)"""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
from paper_2505_12044_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(_lib.LIB_PATH), "libflashbias_b200_clk.so")
lib = _lib.lib()
lib.fb_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = bench.CONFIGS["C3"]
inp = bench.make_inputs(cfg, 0, cfg["H"], torch.device("cuda"))
step = bench.step_fn(cfg, inp, "flashbias")
nkt = cfg["N"] // 128
buf = torch.zeros(4 * cfg["B"] * cfg["H"] * nkt, dtype=torch.int64, device="cuda")


def measure(tag):
    buf.zero_()
    lib.fb_debug_set_trace(buf.data_ptr(), -1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    step()
    b.record()
    torch.cuda.synchronize()
    lib.fb_debug_set_trace(None, -1)
    t = buf.view(-1, 4).cpu().double()
    ok = t[:, 0] > 0
    t = t[ok]
    cyc = t[:, 2] - t[:, 0]
    ns = t[:, 3] - t[:, 1]
    kt = torch.arange(len(ok))[ok] % nkt
    nblk = (nkt - (kt & ~1)).double()  # MC pairs start at the even tile's diagonal block
    span_ns = float(t[:, 3].max() - t[:, 1].min())
    long = ns > 50e3
    return {"tag": tag, "step_ms": round(a.elapsed_time(b), 3), "bwd_span_ms": round(span_ns / 1e6, 3),
            "eff_mhz_long_ctas": round(float((cyc[long] / ns[long]).median()) * 1e3, 1),
            "cycles_per_block_median": round(float((cyc / nblk)[long].median()), 1),
            "sum_cycles_per_sm_per_block": round(float(cyc.sum() / 148 / (nblk.sum() / 148)), 1)}


for _ in range(3):
    step()
torch.cuda.synchronize()
time.sleep(3)
print(json.dumps(measure("cold")))
t0 = time.time()
while time.time() - t0 < 4:
    step()
print(json.dumps(measure("hot")))
