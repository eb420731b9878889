#!/usr/bin/env python
"""Run the five BASELINE configs at full size through the C-ABI on the GPU.

  python tools/run_configs.py [--only cfg3,cfg5,tube,tube_m6] [--json out.jsonl]

Per config: layout size, levels, V-cycles to the config's tolerance (or its fixed
cycle count), the composite relative residual history, CUDA-event time per V-cycle
(graph-launched), and the error against the closed form where one exists
(cfg1: f/σ2 (A6); cfg2: per-mode exact discrete solution; cfg3: -erf(r/(√2σ))/(4πr)).
No oracle is run here (tests/ compare against the oracle).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def analytic(name, cfg, dom, leaves, f):
    from workloads import sources as S
    from workloads.layouts import block_node_coords
    name = name[:-3] if name.endswith("_m6") else name
    if name == "cfg1":
        s2 = -12 * math.sin(math.pi / 32) ** 2 * 32 ** 2
        return f / s2, "exact discrete f/sigma2"
    if name == "cfg2":
        N = cfg["base_blocks"][0] * cfg["B"]
        k, a, phi = S.fourier_modes(cfg.get("seed", 2))
        h = 1.0 / N
        J = np.arange(N) / N
        uh = np.zeros((N, N, N))
        X = J[:, None, None]
        Y = J[None, :, None]
        Z = J[None, None, :]
        for kk, aa, pp in zip(k, a, phi):
            sh = [2 * np.cos(2 * np.pi * kd / N) - 2 for kd in kk]
            s4 = (sum(sh) + (sh[0] * sh[1] + sh[1] * sh[2] + sh[2] * sh[0]) / 6) / h ** 2
            rho = 1 + sum(sh) / 12
            if cfg["order"] == 6:   # E13: symbol and right-hand-side factor of M = 6 (Z24)
                s4 += sh[0] * sh[1] * sh[2] / 30 / h ** 2
                rho += (sh[0] * sh[1] + sh[1] * sh[2] + sh[2] * sh[0]) / 90 - (sh[0] ** 2 + sh[1] ** 2 + sh[2] ** 2) / 240
            uh += aa * rho / s4 * np.cos(2 * np.pi * (kk[0] * X + kk[1] * Y + kk[2] * Z) + pp)
        return S.dense_to_blocks(dom, leaves, uh), "exact discrete (per mode rho4/sigma4), mod mean"
    if name == "cfg3":
        return S.sample_on_leaves(dom, leaves, S.gaussian_potential), "continuum -erf(r/(sqrt2 sigma))/(4 pi r)"
    return None, None


def run(name, args):
    import torch

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    if name.endswith("_m6"):  # the 6th-order variant of a config
        cfg = getattr(C, name[:-3])()
        cfg["order"] = 6
        cfg["name"] = name
    else:
        cfg = getattr(C, name)()
    t0 = time.time()
    dom, leaves, f = C.build(cfg)
    t_build = time.time() - t0
    S = Solver(cfg, leaves)
    nlev = S.num_levels()
    info = [S.level_info(m) for m in range(nlev)]
    S.use_graph(True)
    fd = torch.from_numpy(f).cuda()
    S.set_rhs(fd)
    hist = []
    cycles = cfg.get("cycles", 0) or 0
    maxc = cycles if cycles else 40
    for c in range(maxc):
        S.vcycle(1)
        hist.append(S.residual_norm()[1])
        if not cycles and hist[-1] <= cfg["tol"]:
            break
    ncyc = len(hist)
    # timing: graph-launched V-cycles from the converged state
    ms = S.time_op("vcycle", 0, 10)
    out = {"config": name, "leaves": int(len(leaves)), "leaf_unknowns": int(f.size), "levels": nlev,
           "blocks_per_level": [int(i["nreal"]) for i in info], "ghost_blocks": [int(i["nghost"]) for i in info],
           "cycles": ncyc, "rel_residual": hist, "ms_per_vcycle": ms,
           "unknowns_per_s": f.size / (ms * 1e-3), "layout_build_s": round(t_build, 1)}
    ua, what = analytic(name, cfg, dom, leaves, f)
    if ua is not None:
        u = S.get_solution().cpu().numpy()
        if name == "cfg2":
            u = u - u.mean()
            ua = ua - ua.mean()
        out["err_vs_analytic"] = float(np.abs(u - ua).max() / np.abs(ua).max())
        out["analytic"] = what
        if name == "cfg3":
            # the origin is level-0 node J = N/2 = 128: block (8, 8, 8), local (0, 0, 0)
            n = int(np.nonzero((leaves == np.array([0, 8, 8, 8])).all(axis=1))[0][0])
            out["u_origin"] = float(u[n, 0, 0, 0])
            out["u_origin_analytic"] = -math.sqrt(2 / math.pi) / (4 * math.pi * 0.08)
    S.close()
    return out


def run_tube(name, a):
    """Vortex-tube vector solve: the three components of ∇²u = -∇×ω
    on one handle, each to the config's tolerance; E∞ against the closed-form velocity."""
    import torch

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C
    cfg = dict(C.tube(order=6 if "_m6" in name else 4))
    batched = "batched" in name
    if batched:                 # one 3-component V-cycle (mg_desc.ncomp = 3)
        cfg["ncomp"] = 3
    t0 = time.time()
    dom, leaves, f3, u3 = C.build_vector(cfg)
    t_build = time.time() - t0
    S = Solver(cfg, leaves)
    S.use_graph(True)
    fd = [torch.from_numpy(f).cuda() for f in f3]
    S.solve_vector(fd, cfg["tol"], 40)          # warm-up (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    us, stats = S.solve_vector(fd, cfg["tol"], 40)
    e1.record()
    torch.cuda.synchronize()
    ms_solve = e0.elapsed_time(e1)
    ms_cycle = S.time_op("vcycle", 0, 10)
    info = [S.level_info(m) for m in range(S.num_levels())]
    err = [float(np.abs(us[c].cpu().numpy() - u3[c]).max()) for c in range(3)]
    S.close()
    return {"config": name, "leaves": int(len(leaves)), "leaf_unknowns_per_component": int(f3[0].size),
            "levels": len(info), "blocks_per_level": [int(i["nreal"]) for i in info],
            "ghost_blocks": [int(i["nghost"]) for i in info],
            "cycles_per_component": [c for c, _, _ in stats], "rel_residual": [r for _, r, _ in stats],
            "ms_per_vcycle": ms_cycle, "ms_vector_solve": ms_solve,
            "einf_vs_analytic": err, "u_max": float(np.abs(u3[0]).max()), "layout_build_s": round(t_build, 1),
            "note": ("one batched 3-component solve (ncomp = 3): every launch covers all components"
                     if batched else
                     "three scalar solves on one handle; the z component has f_z = 0 (u_z = 0, no cycles)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    for name in a.only.split(","):
        try:
            r = run_tube(name, a) if name.startswith("tube") else run(name, a)
        except Exception as e:  # report and continue with the next config
            r = {"config": name, "error": repr(e)}
        line = json.dumps(r)
        print(line, flush=True)
        if a.json:
            with open(a.json, "a") as fh:
                fh.write(line + "\n")


if __name__ == "__main__":
    main()
