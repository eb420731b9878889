#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun).

  python tools/ncu_summary.py --launches gpurun_out/launches.csv \
      --rep gpurun_out/prof.ncu-rep --title "..." > profiles/rNN_xxx.md

--launches: the `--metrics gpu__time_duration.sum` launch list (per-kernel share).
--rep:      a `--set full` capture; prints the key SOL / memory / occupancy rows
            and DRAM bytes per launch of every captured kernel.
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict


def _csv_rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path):
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total µs | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k[:70]}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    out.append(f"| **total** | {sum(cnt.values())} | {T:.1f} | 100% |")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def rep(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = _csv_rows(txt)
    h = rows[0]
    idx = {k: h.index(k) for k in KEYS if k in h}
    name_i = h.index("Kernel Name")
    out = []
    for r in rows[2:]:
        out.append(f"- `{r[name_i].split('(')[0]}` grid {r[idx['launch__grid_size']]}")
        for k, i in idx.items():
            out.append(f"  - {k} = {r[i]} {rows[1][i]}")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--cmd", default="")
    a = ap.parse_args()
    print(f"# {a.title}\n")
    if a.cmd:
        print(f"Command: `{a.cmd}`\n")
    if a.launches:
        print("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n")
        print(launches(a.launches) + "\n")
    if a.rep:
        print("## ncu --set full (per captured launch)\n")
        print(rep(a.rep) + "\n")


if __name__ == "__main__":
    main()
