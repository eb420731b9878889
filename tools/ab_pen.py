#!/usr/bin/env python
"""A/B timing of host-side scheduling choices and kernel builds on one config (tuning aid).

  python tools/ab_pen.py --cfg cfg5 --cfgset pencil_order=2 pencil_blocks=4   # mg_desc variant controls
  python tools/ab_pen.py --lib _ab/x/libmg.so                                 # a tools/ab_build.py build
  python tools/ab_pen.py --env MG_EXP_X --settings "" "1"                     # a temporary getenv switch
                                                                              # compiled into an experiment

Per setting (twice, interleaved): per-level stage times of non-graph V-cycles (CUDA events per
stage, us per launch, index = level) and the graph-launched V-cycle time.  The library itself
reads no environment variables; --env only serves experiments that add one temporarily.
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
    ap.add_argument("--cfg", default="cfg5")
    ap.add_argument("--settings", nargs="*", default=[""])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--env", default="MG_EXP_PEN")
    ap.add_argument("--cfgset", nargs="*", default=[], help="cfg overrides key=int (mg_desc variant controls)")
    ap.add_argument("--lib", default="", help="libmg.so to load instead of the in-tree one (A/B builds)")
    a = ap.parse_args()
    import torch

    if a.lib:
        from paper_2512_08555_b200.mg import load_library
        load_library(a.lib)

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    cfg = getattr(C, a.cfg)()
    dom, leaves, f = C.build(cfg)
    for kv in a.cfgset:
        k, v = kv.split("=")
        cfg[k] = int(v)
    fd = torch.from_numpy(f).cuda()
    for rnd in range(2):
        for st in a.settings:
            if st:
                os.environ[a.env] = st
            else:
                os.environ.pop(a.env, None)
            S = Solver(cfg, leaves)
            S.set_rhs(fd)
            S.vcycle(2)
            S.profile(True)
            S.vcycle(a.reps)
            torch.cuda.synchronize()
            pr = S.profile_read()
            S.profile(False)
            out = {"setting": st, "lib": a.lib, "cfgset": a.cfgset, "round": rnd}
            for stage in ("smooth", "restrict", "fas", "ghost", "prolong"):
                ms, n = pr[stage]
                out[stage + "_us"] = [round(1e3 * m / max(c, 1), 1) for m, c in zip(ms, n)]
            S.use_graph(True)
            S.vcycle(3)
            out["vcycle_graph_ms"] = round(S.time_op(100, 0, a.reps), 4)
            out["residual"] = S.residual_norm()[1]
            print(json.dumps(out), flush=True)
            del S
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
