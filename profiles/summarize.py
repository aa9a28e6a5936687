#!/usr/bin/env python
"""Summarise ncu captures (gpurun_out/prof_<tag>_*.ncu-rep + launches_<tag>.csv)
into profiles/ncu_<tag>.md and profiles/ncu_traffic.json (per-launch DRAM bytes
consumed by bench.py's roofline.traffic).

    python profiles/summarize.py r02 C3
"""

import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (elapsed cycles / s)"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tensor (UTCHMMA bf16) % of peak"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU ex2) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__m_l1tex2xbar_write_bytes.sum", "SM->L2 write bytes (dQ reduce-adds)"),
    ("l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed", "SM->L2 write % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM read bytes (TMA loads)"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "L2 read hits (sectors)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput % (active)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("lts__t_sectors_op_red.sum", "L2 reduction sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1}


def raw(rep):
    if rep.endswith(".csv"):  # exported on the GPU box by run_ncu.sh
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_num(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNITS.get(u, 1)


def main(tag, cfg):
    lines = [f"# ncu summary — {tag}, {cfg}", "",
             f"Captured with `profiles/run_ncu.sh {tag} {cfg}` on one B200 (`--set full --clock-control none`), "
             f"bench.py workload {cfg}, one launch per kernel after warm-up. "
             "ncu replays each kernel ~40x with cold caches: compare shares/ratios, not absolute times.", ""]
    traffic = {}
    reps = {}
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_{cfg}_*.ncu-rep")) +
                      glob.glob(os.path.join(OUT, f"prof_{tag}_{cfg}_*.raw.csv"))):
        name = os.path.basename(rep)[len(f"prof_{tag}_{cfg}_"):].split(".")[0]
        reps.setdefault(name, rep)
    for name, rep in sorted(reps.items()):
        m = raw(rep)
        lines += [f"## {name}", "", "| metric | value |", "|---|---|"]
        got = {}
        for key, label in METRICS:
            if key in m:
                v, u = m[key]
                got[key] = to_num(v, u)
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        rd, wr = got.get("dram__bytes_read.sum"), got.get("dram__bytes_write.sum")
        if isinstance(rd, float) and isinstance(wr, float):
            kind = "fwd" if "fwd" in name else "bwd"
            traffic[kind] = rd + wr
            lines.append(f"| DRAM read+write per launch | {(rd + wr) / 1e9:.2f} GB |")
        lines.append("")
    lf = os.path.join(OUT, f"launches_{tag}_{cfg}.csv")
    if os.path.exists(lf):
        rows = list(csv.reader(open(lf)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        tot = {}
        for r in rows[hdr + 1:]:
            if len(r) > vi:
                k = r[ki].split("(")[0].replace("void ", "")
                tot[k] = tot.get(k, 0.0) + to_num(r[vi], r[ui])
        s = sum(tot.values())
        lines += [f"## launch list (every kernel of one {cfg} bench step: bench.py --steps 1 --warmup 1, cold-cache "
                  "serialised replays)", "", "| kernel | total time | share |",
                  "|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| `{k}` | {v * 1e3:.2f} ms | {v / s:.1%} |")
        lines.append("")
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}_{cfg}.md"), "w").write("\n".join(lines))
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    data[cfg] = {**data.get(cfg, {}), **traffic, "tag": tag}
    json.dump(data, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02", sys.argv[2] if len(sys.argv) > 2 else "C3")
