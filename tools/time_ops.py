#!/usr/bin/env python
"""Quick CUDA-event timing of single operators and the V-cycle (tuning aid).

  python tools/time_ops.py [--cfg cfg2] [--n 256] [--reps 50]

Prints ms per launch of: smooth (finest level), residual (finest), and one V-cycle
(graph-launched), plus the smoother's algorithmic GB/s (24 B / unknown).
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
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--tag", default="")
    ap.add_argument("--coarse", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2512_08555_b200 import Solver
    from paper_2512_08555_b200.mg import OPS
    from workloads import configs as C
    if a.cfg == "cfg2":
        cfg = C.cfg2(a.n, coarse_n=a.coarse or None)
    else:
        cfg = getattr(C, a.cfg)(a.n) if a.cfg == "cfg3" else getattr(C, a.cfg)()
    dom, leaves, f = C.build(cfg)
    S = Solver(cfg, leaves)
    S.set_rhs(torch.from_numpy(f).cuda())
    S.vcycle(2)
    top = S.num_levels() - 1
    info = S.level_info(top)
    n = info["nreal"] * info["B"] ** 3
    out = {"tag": a.tag, "cfg": cfg["name"], "unknowns_finest": n}
    for name in ("smooth", "residual"):
        S.time_op(OPS[name], top, 3)
        ms = S.time_op(OPS[name], top, a.reps)
        out[name + "_us"] = round(ms * 1e3, 2)
        out[name + "_gbs"] = round(24 * n / (ms * 1e-3) / 1e9, 1)
    S.use_graph(True)
    S.vcycle(3)
    ms = S.time_op(100, 0, a.reps)
    out["vcycle_ms"] = round(ms, 4)
    out["vcycle_unknowns_per_s"] = f.size / (ms * 1e-3)
    S.use_graph(True)
    S.set_rhs(torch.from_numpy(f).cuda())
    cyc, rel, ok = S.solve(cfg["tol"], 30)
    out["cycles_to_tol"] = cyc
    out["levels"] = S.num_levels()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
