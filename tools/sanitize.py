#!/usr/bin/env python
"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / initcheck /
synccheck): cfg1 (periodic, B=16 z-split sweeps, sub-base B<16 levels, 4^3 coarse
FFT) and a 2-level x-periodic / y,z-unbounded layout with resolution jumps (ghost
boxes, exterior band, 1- and 2-block pencils, fused residual+restriction), M = 4 and
6, graph and non-graph V-cycles, the composite norm and the device Cauchy criterion.

  compute-sanitizer --tool memcheck python tools/sanitize.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2512_08555_b200 import Solver
    from tests.test_gpu_parity import _cfg
    for name, extra in (("cfg1", {}), ("puu1", {}), ("puu1", {"pencil_blocks": 2}), ("puu1_m6", {}),
                        ("cfg3_64", {"pencil_blocks": 2})):
        cfg, lv, f = _cfg(name)
        cfg = dict(cfg)
        cfg.update(extra)
        s = Solver(cfg, lv)
        s.set_rhs(torch.from_numpy(f).cuda())
        s.vcycle(1)
        s.use_graph(True)
        s.vcycle(1)
        a, r = s.residual_norm()
        c, v, ok = s.solve(1e-30, 2, 1)
        torch.cuda.synchronize()
        print(f"{name} {extra}: rel residual {r:.3e}, cauchy {v:.3e}", flush=True)
        del s


if __name__ == "__main__":
    main()
