#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) and an ncu --set full
report into profiles/<tag>_*.{json,md}.

    python scripts/ncu_summary.py --tag r1 --launches gpurun_out/launches.csv \
        --report gpurun_out/prof_full.ncu-rep
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    # tcgen05 utilisation: cycles the tensor pipe is busy over elapsed SM cycles -- agrees with
    # the kernel's flop rate / (148 SMs x 8192 bf16 flop/clk x the SM clock under ncu)
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "utchmma_bf16_ops": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "tensor_mem_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_bf16_ops_pct": "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l2_pct_peak": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct_peak": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_cycles_active": "sm__cycles_active.avg",
}


def to_us(v: float, unit: str) -> float:
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3,
            "ms": v * 1e3, "second": v * 1e6, "s": v * 1e6}.get(unit, v)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(to_us(float(r[vi].replace(",", "")), r[ui]))
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot}
            for k, v in agg.items()}


def full_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = collections.OrderedDict()
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        name = r[ki].split("(")[0]
        d = {}
        for key, m in METRICS.items():
            idx = [j for j, h in enumerate(hdr) if h == m] + \
                  [j for j, h in enumerate(hdr) if h.endswith("." + m)]
            vals = []
            for j in idx:
                try:
                    vals.append((j, float(r[j].replace(",", ""))))
                except ValueError:
                    pass
            if vals:
                i, v = vals[0]
                u = units[i]
                if key == "duration_us":
                    v = to_us(v, u)
                elif key.endswith("_bytes"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[key] = v
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
        res.setdefault(name, []).append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", default="profiles")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    summary = {}
    md = [f"# ncu summary ({a.tag})", ""]
    if a.launches:
        L = launches(a.launches)
        summary["launch_list"] = L
        md += ["## Launch list (cold, serialised; compare shares)", "",
               "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, v in sorted(L.items(), key=lambda kv: -kv[1]["share"]):
            md.append(f"| {k} | {v['launches']} | {v['mean_us']:.1f} | {v['share']:.3f} |")
        md.append("")
    if a.report:
        R = full_report(a.report)
        summary["full"] = R
        md += ["## ncu --set full", "",
               "| kernel | us | DRAM bytes | DRAM % | L2 % | tensor pipe active % (sm__pipe_tensor_cycles_active) | sm__mem_tensor_cycles_active % | SM % | regs | grid |",
               "|---|---|---|---|---|---|---|---|---|---|"]
        for k, lst in R.items():
            for d in lst:
                md.append(f"| {k} | {d.get('duration_us', 0):.1f} | {d.get('dram_bytes', 0) / 1e6:.1f} MB"
                          f" | {d.get('dram_pct_peak', 0):.1f} | {d.get('l2_pct_peak', 0):.1f}"
                          f" | {d.get('tensor_pipe_pct', 0):.1f} | {d.get('tensor_mem_pct', 0):.1f}"
                          f" | {d.get('sm_pct_peak', 0):.1f}"
                          f" | {d.get('registers', 0):.0f} | {d.get('grid', 0):.0f} |")
        rec = [(k, d) for k, lst in R.items() for d in lst if d.get("utchmma_bf16_ops")]
        if rec:
            md += ["", "Tensor-pipe reconciliation: bf16 UTCHMMA ops (flops, incl. tile padding) / duration"
                   " vs 148 SMs x 8192 flop/clk x the SM clock ncu ran at:", "",
                   "| kernel | bf16 flops | us | TFLOP/s | SM GHz | peak at that clock | ratio | tensor pipe active % |",
                   "|---|---|---|---|---|---|---|---|"]
            for k, d in rec:
                ghz = d.get("sm_clock_ghz", 0) / (1e9 if d.get("sm_clock_ghz", 0) > 1e3 else 1)
                tf = d["utchmma_bf16_ops"] / (d["duration_us"] * 1e-6) / 1e12
                pk = 148 * 8192 * ghz * 1e9 / 1e12
                md.append(f"| {k} | {d['utchmma_bf16_ops']:.3e} | {d['duration_us']:.1f} | {tf:.0f} | {ghz:.3f}"
                          f" | {pk:.0f} | {tf / pk:.3f} | {d.get('tensor_pipe_pct', 0):.1f} |")
    json.dump(summary, open(os.path.join(a.out, f"ncu_{a.tag}.json"), "w"), indent=1)
    open(os.path.join(a.out, f"ncu_{a.tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
