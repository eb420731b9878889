#!/usr/bin/env python
"""CUDA-event timing of the detail-coefficient kernel (mg_detail) on a
large leaf field, against the HBM roofline (8 B read per node, the kernel's only HBM
traffic besides 8 B per block written).

  python tools/time_detail.py [--blocks 30000] [--W 4] [--reps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=30000)
    ap.add_argument("--W", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2512_08555_b200 import detail
    f = torch.randn((a.blocks, 16, 16, 16), dtype=torch.float64, device="cuda")
    for _ in range(3):
        detail(f, 16, a.W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        detail(f, 16, a.W)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.5)
    gbs = f.numel() * 8 / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": "k_detail", "W": a.W, "blocks": a.blocks, "nodes": f.numel(), "ms": ms,
                      "gbs": gbs, "frac_of_hbm_peak": gbs / peak}), flush=True)


if __name__ == "__main__":
    main()
