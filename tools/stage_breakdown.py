#!/usr/bin/env python
"""Per-level, per-stage CUDA-event breakdown of a V-cycle (non-graph launches).

  python tools/stage_breakdown.py [--cfg cfg2|cfg2_m6|…] [--cycles 5]
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
    ap.add_argument("--cycles", type=int, default=5)
    ap.add_argument("--extra", default="{}", help="extra cfg keys (json), e.g. fuse, pencil_blocks")
    ap.add_argument("--lib", default="", help="libmg.so to load instead of the in-tree one (A/B builds)")
    a = ap.parse_args()
    import torch

    if a.lib:
        from paper_2512_08555_b200.mg import load_library
        load_library(a.lib)

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    name = a.cfg[:-3] if a.cfg.endswith("_m6") else a.cfg
    cfg = getattr(C, name)()
    if a.cfg.endswith("_m6"):  # the 6th-order variant
        cfg = dict(cfg, order=6, name=a.cfg)
    dom, leaves, f = C.build(cfg)
    cfg = dict(cfg, **json.loads(a.extra))
    S = Solver(cfg, leaves)
    S.set_rhs(torch.from_numpy(f).cuda())
    S.vcycle(2)
    S.use_graph(False)
    S.profile(True)
    S.vcycle(a.cycles)
    prof = S.profile_read()
    S.profile(False)
    nlev = S.num_levels()
    rows = {}
    for st, (ms, cnt) in prof.items():
        for m in range(nlev):
            if cnt[m]:
                rows.setdefault(st, {})[m] = (round(ms[m] / a.cycles * 1e3, 1), round(cnt[m] / a.cycles, 2))
    info = [S.level_info(m) for m in range(nlev)]
    print(json.dumps({"cfg": a.cfg, "extra": a.extra, "blocks": [i["nreal"] for i in info], "ghosts": [i["nghost"] for i in info],
                      "us_per_cycle[stage][level]=(us, launches)": rows}), flush=True)
    S.use_graph(True)
    runs = sorted(S.time_op("vcycle", 0, 20) for _ in range(5))
    print(json.dumps({"cfg": a.cfg, "lib": a.lib, "extra": a.extra, "graph_ms_per_vcycle": runs[2], "runs": runs}),
          flush=True)


if __name__ == "__main__":
    main()
