#!/usr/bin/env python
"""Summarise scripts/ncu_mem_r2.sh (memory kernels of the bench step under ncu,
uniform-word and Zipf streams) into a markdown table: per kernel the mean
duration, DRAM bytes and GB/s against the measured HBM copy bandwidth
(MEASURED_PEAKS.json) and the measured random-32-B-sector roofline
(profiles/sector_roofline_r1.md, ~1.6 TB/s), L2 bytes and hit rate.

    python scripts/mem_summary.py gpurun_out/ncu_uniform_r2.csv gpurun_out/ncu_zipf_r2.csv > profiles/ncu_mem_r2.md
"""
import collections
import csv
import json
import os
import sys

SECTOR_GBS = 1600.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    out = collections.OrderedDict()
    for r in rows:
        if r[0] == "ID" or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
        out.setdefault(k, collections.defaultdict(list))[d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    return out


def main():
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    print("# Memory kernels of the bench step under ncu (bf16 step, 64 x 2,048 queries)\n")
    print(f"`scripts/ncu_mem_r2.sh` (`ncu --metrics ... --clock-control none`, 5 launches per kernel, cold and "
          f"serialised by the profiler), `scripts/mem_summary.py`.  GB/s = DRAM bytes / duration; "
          f"HBM peak {hbm:.0f} GB/s (MEASURED_PEAKS.json copy bandwidth), random 32-B sector roofline "
          f"~{SECTOR_GBS:.0f} GB/s (`profiles/sector_roofline_r1.md`).\n")
    for path in sys.argv[1:]:
        name = "uniform-word stream (no Zipf reuse)" if "uniform" in path else "Zipf stream (the bench's)"
        print(f"## {name}\n")
        print("| kernel | us | DRAM MB | DRAM GB/s | of HBM | of sector roofline | L2 MB | L2 hit % |")
        print("|---|---|---|---|---|---|---|---|")
        for k, mm in load(path).items():
            n = len(mm["gpu__time_duration.sum"])
            avg = lambda m: sum(mm[m]) / max(1, len(mm[m]))
            t = avg("gpu__time_duration.sum")                      # ns
            b = avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")
            gbs = b / t
            print(f"| {k} | {t / 1e3:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / hbm:.2f} | {gbs / SECTOR_GBS:.2f} | "
                  f"{avg('lts__t_bytes.sum') / 1e6:.1f} | {avg('lts__t_sector_hit_rate.pct'):.1f} |")
        print()


if __name__ == "__main__":
    main()
