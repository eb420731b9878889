#!/usr/bin/env python
"""Collect per-launch DRAM traffic and duration of captured kernels from ncu reports
into profiles/ncu_traffic.json (read by bench.py's roofline.traffic).

  python tools/ncu_traffic.py gpurun_out/full_*.ncu-rep > profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def rows(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
    r = list(csv.reader(io.StringIO("\n".join(lines))))
    return r[0], r[1], r[2:]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def main():
    out = {"how": "ncu --set full --clock-control none, first launch of each kernel in a cfg2 256^3 V-cycle "
                  "(tools/prof_vcycle.py); dram bytes = dram__bytes_read.sum + dram__bytes_write.sum",
           "kernels": {}}
    for path in sys.argv[1:]:
        h, u, data = rows(path)
        i = {k: h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                     "gpu__time_duration.sum", "launch__grid_size")}
        for r in data:
            name = r[i["Kernel Name"]].split("(")[0].replace("void ", "")
            rd = float(r[i["dram__bytes_read.sum"]]) * SCALE[u[i["dram__bytes_read.sum"]]]
            wr = float(r[i["dram__bytes_write.sum"]]) * SCALE[u[i["dram__bytes_write.sum"]]]
            t = float(r[i["gpu__time_duration.sum"]]) * SCALE[u[i["gpu__time_duration.sum"]]]
            out["kernels"].setdefault(name, {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                             "duration_us_under_ncu": t, "grid": int(r[i["launch__grid_size"]]),
                                             "report": path.split("/")[-1]})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
