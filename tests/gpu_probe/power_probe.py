"""SM clock and board power while the C3 forward / backward / whole step run back to back
(is the kernel clock- or power-bound?).  Each phase loops for ~4 s under an nvidia-smi sampler
(20 ms period); prints per-phase ms per call, median SM clock, median power and the cycles per
128x128 backward block implied by ms x clock.

    python tests/gpu_probe/power_probe.py [C3]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_12044_b200 as fb  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
inp = bench.make_inputs(cfg, 0, cfg["H"], torch.device("cuda"))
mask = "causal" if cfg["causal"] else "none"
q, k, v = (inp[x].detach().requires_grad_(True) for x in ("q", "k", "v"))
do = torch.randn_like(q)


def fwd():
    with torch.no_grad():
        fb.flashbias_attention(q, k, v, inp["fq"], inp["fk"], mask=mask)


out = fb.flashbias_attention(q, k, v, inp["fq"], inp["fk"], mask=mask)


def bwd():
    torch.autograd.grad(out, (q, k, v), do, retain_graph=True)


def step():
    o = fb.flashbias_attention(q, k, v, inp["fq"], inp["fk"], mask=mask)
    torch.autograd.grad(o, (q, k, v), do)


def phase(fn, seconds=4.0):
    import threading

    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    clk, pw, reasons, stop = [], [], set(), threading.Event()

    def sample():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            reasons.add(int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            time.sleep(0.02)

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    a.record()
    th = threading.Thread(target=sample, daemon=True)
    th.start()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    clk, pw = clk[len(clk) // 5:], pw[len(pw) // 5:]  # drop the ramp
    return {"ms": round(a.elapsed_time(b) / n, 3), "calls": n, "sm_mhz_median": statistics.median(clk),
            "sm_mhz_min": min(clk), "power_w_median": statistics.median(pw), "reason_masks": sorted(reasons)}


res = {"fwd": phase(fwd), "bwd": phase(bwd), "step": phase(step)}
if cfg["causal"]:
    nt = (cfg["N"] + 127) // 128
    blocks = cfg["B"] * cfg["H"] * nt * (nt + 1) // 2
    per_sm = blocks / 148
    r = res["bwd"]
    if r["sm_mhz_median"]:
        r["cycles_per_block_at_median_clock"] = round(r["ms"] * 1e-3 * r["sm_mhz_median"] * 1e6 / per_sm)
print(json.dumps(res))
