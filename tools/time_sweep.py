#!/usr/bin/env python
"""Finest-level RB sweep kernel time per tile-staging variant (mg_desc.staging: 0 cp.async,
1 TMA tensor copies) on cfg2 and cfg5, from the per-stage CUDA
events of non-graph V-cycles; the solutions of all variants must agree bitwise (the
staging moves the same values).

  python tools/time_sweep.py [--configs cfg2,cfg5] [--stagings 0,1] [--cycles 6]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg2,cfg5")
    ap.add_argument("--stagings", default="0,1")
    ap.add_argument("--cycles", type=int, default=6)
    ap.add_argument("--extra", default="{}", help="extra cfg keys (json), e.g. pencil_blocks")
    ap.add_argument("--lib", default="", help="libmg.so to load instead of the in-tree one (A/B builds)")
    args = ap.parse_args()
    import torch

    if args.lib:
        from paper_2512_08555_b200.mg import load_library
        load_library(args.lib)

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    for name in args.configs.split(","):
        cfg = C.cfg5() if name == "cfg5" else C.cfg2(256)
        cfg.update(json.loads(args.extra))
        _, lv, f = C.build(cfg)
        fd = torch.from_numpy(f).cuda()
        ref = None
        for st in [int(x) for x in args.stagings.split(",")]:
            c = dict(cfg)
            c["staging"] = st
            S = Solver(c, lv)
            S.set_rhs(fd)
            S.vcycle(2)
            u = S.get_solution().cpu().numpy()
            same = None if ref is None else bool(np.array_equal(u, ref))
            if ref is None:
                ref = u
            S.set_rhs(fd)
            S.vcycle(1)
            S.profile(True)
            S.vcycle(args.cycles)
            p = S.profile_read()
            S.profile(False)
            nl = S.num_levels()
            rows = {}
            for m in range(1, nl):
                tot, cnt = p["smooth"][0][m], p["smooth"][1][m]
                info = S.level_info(m)
                n = info["nreal"] * info["B"] ** 3
                if cnt:
                    ms = tot / cnt
                    rows[m] = {"us": round(ms * 1e3, 2), "TBps": round(24 * n / (ms * 1e-3) / 1e12, 3)}
            S.use_graph(True)
            S.vcycle(2)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.vcycle(10)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"config": name, "lib": args.lib, "staging": st, "bitwise_same_as_first": same, "sweep": rows,
                              "vcycle_ms": e0.elapsed_time(e1) / 10}), flush=True)
            del S
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
