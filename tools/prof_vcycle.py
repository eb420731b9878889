#!/usr/bin/env python
"""Short driver for ncu captures: build a config, set the RHS, run a few V-cycles.

  python tools/prof_vcycle.py [--cfg cfg2|cfg3|cfg4|cfg5] [--n 256] [--cycles 3] [--graph]

Launches only this library's kernels (+ cuFFT for the coarse solve); no oracle.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--cycles", type=int, default=3)
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    if a.cfg in ("cfg2", "cfg3"):
        cfg = getattr(C, a.cfg)(a.n)
    else:
        cfg = getattr(C, a.cfg)()
    t = time.time()
    dom, leaves, f = C.build(cfg)
    print(f"built {a.cfg}: {len(leaves)} leaves in {time.time() - t:.1f}s", flush=True)
    S = Solver(cfg, leaves)
    S.use_graph(a.graph)
    S.set_rhs(torch.from_numpy(f).cuda())
    S.vcycle(a.cycles)
    torch.cuda.synchronize()
    print("residual", S.residual_norm(), flush=True)


if __name__ == "__main__":
    main()
