#!/usr/bin/env python
"""Benchmark: V-cycle throughput of the B200 adaptive multigrid solver.

Workload (BASELINE.json configs[1], the metric's config): uniform periodic 256^3
(4096 blocks of 16^3), 4th-order Mehrstellen, red-black V(2,2), 3 MG levels down
to a 64^3 cuFFT coarse solve; source = 64 seeded Fourier modes (workloads.configs.cfg2).
A step = one full V-cycle (all hot-path kernels of every level + coarse solve).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]

Under torchrun (N > 1) every rank solves its own replica (the north star is one
GPU, no sharding), scaling = weak, timing = max over ranks.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V-cycle unknowns/s and smoother+residual HBM GB/s (% of B200 peak), fp64"
UNIT = "unknowns/s"
NORTH_STAR_PEAK_GBS = 8000.0


def peak_hbm():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.p = None
        self.index = index

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def max_over_ranks(x, dist, device):
    """Max of a per-rank float over all ranks (device timing rule: the slowest rank)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(kernel_prefix):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return None
    for k, v in d.get("kernels", {}).items():
        if k.startswith(kernel_prefix):
            return v.get("dram_bytes_per_launch")
    return None


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if ws > 1:
        import torch.distributed as dist_
        dist = dist_
        backend = "nccl" if args.impl == "mine" else "gloo"
        dist.init_process_group(backend=backend)
    return ws, rank, local, dist


def build_workload(N=256):
    from workloads import configs as C
    cfg = C.cfg2(N)
    dom, leaves, f = C.build(cfg)
    return cfg, leaves, f


def cpu_baseline(cfg, leaves, f):
    """The oracle as it stands, one V-cycle of the full workload on the host."""
    from oracle.mg_oracle import Oracle
    o = Oracle(cfg, leaves)
    o.set_rhs(f)
    t = time.perf_counter()
    o.vcycle(1)
    dt = time.perf_counter() - t
    n = f.size
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 V-cycle of the full cfg2 256^3 workload ({n} leaf unknowns), numpy oracle, "
                      f"single thread, {dt:.1f} s"}


def run_reference(args, ws, rank, dist):
    """--impl reference: the CPU oracle (this tier's reference arm) on a bounded sample."""
    if rank != 0:
        return
    from oracle.mg_oracle import Oracle
    # per-step sample sized so that the whole --steps K --warmup W run stays within a few
    # minutes (measured oracle V-cycle on one core: 128^3 ~1.8 s, 64^3 ~0.25 s, 32^3 ~0.04 s)
    if args.ref_n <= 0:
        est = {128: 1.8, 64: 0.25, 32: 0.04}
        nsteps = args.steps + args.warmup
        args.ref_n = next((n for n in (128, 64) if est[n] * nsteps <= 150.0), 32)
    cfg, leaves, f = build_workload(args.ref_n)
    o = Oracle(cfg, leaves)
    o.set_rhs(f)
    for _ in range(args.warmup):
        o.vcycle(1)
    t = time.perf_counter()
    for _ in range(args.steps):
        o.vcycle(1)
    dt = (time.perf_counter() - t) / args.steps
    n = f.size
    val = n / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 recipe (periodic, M=4 Mehrstellen, RB V(2,2), 64 seeded Fourier modes) "
                                   f"at {args.ref_n}^3 as a bounded CPU sample of the 256^3 workload", "leaf_unknowns": n},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"1 oracle V-cycle of the cfg2 recipe at {args.ref_n}^3 per step"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_mine(args, ws, rank, local, dist):
    import torch

    from paper_2512_08555_b200 import Solver

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg, leaves, f = build_workload(256)
    nleaf_unknowns = f.size
    S = Solver(cfg, leaves)
    f_dev = torch.from_numpy(f).to(dev)
    S.set_rhs(f_dev)
    nlev = S.num_levels()
    levels = [S.level_info(m) for m in range(nlev)]

    # launches per V-cycle (our kernels only; cuFFT's own kernels excluded)
    S.use_graph(False)
    c0 = S.kernel_launches()
    S.vcycle(1)
    torch.cuda.synchronize()
    launches_per_cycle = S.kernel_launches() - c0

    # ---- timed region: K V-cycles, each one CUDA-graph launch
    S.use_graph(True)
    S.set_rhs(f_dev)
    for _ in range(args.warmup):
        S.vcycle(1)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            S.vcycle(1)
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, dev)
    clocks = clk.summary()
    value = nleaf_unknowns * ws / (ms * 1e-3)

    # ---- same K cycles without graph, CUDA events around every stage (live kernel durations)
    S.use_graph(False)
    S.profile(True)
    kp = min(args.steps, 50)
    for _ in range(kp):
        S.vcycle(1)
    prof = S.profile_read()
    S.profile(False)
    top = nlev - 1
    Nf = levels[top]["nreal"] * levels[top]["B"] ** 3
    # dominant kernel = stage x level with the largest total time
    best = max(((s, m) for s in prof for m in range(nlev)), key=lambda sm: prof[sm[0]][0][sm[1]])
    bytes_per_unknown = {"smooth": 24, "smooth_res": 32, "residual": 24, "prolong": 8 * (2 + 2 / 8),
                         "restrict": 8 * (1 + 1 / 8 * 3)}
    st, lv = best
    Nl = levels[lv]["nreal"] * levels[lv]["B"] ** 3
    avg_ms = prof[st][0][lv] / max(1, prof[st][1][lv])
    alg_bytes = bytes_per_unknown.get(st, 24) * Nl
    achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    # per-kernel algorithmic GB/s on the finest level (SURVEY §8(d) byte counts)
    kernels = {}
    # the V-cycle computes the finest residual inside the fused residual+restriction
    # kernel; the standalone residual kernel is timed on its own (same level, 50 launches)
    res_ms = S.time_op("residual", top, 50)
    kernels["residual_standalone"] = {"avg_ms": res_ms, "alg_bytes_per_unknown": 24,
                                      "gbs": 24 * Nf / (res_ms * 1e-3) / 1e9,
                                      "frac": 24 * Nf / (res_ms * 1e-3) / 1e9 / peak_hbm()[0],
                                      "what": "k_res_pencil alone (mg_time_op RESIDUAL on the finest level)"}
    for st_name, bpu in (("smooth", 24), ("smooth_res", 32), ("residual", 24), ("prolong", 18), ("restrict", 18)):
        tot, cnt = prof[st_name][0][top], prof[st_name][1][top]
        if cnt:
            kms = tot / cnt
            kernels[st_name] = {"avg_ms": kms, "alg_bytes_per_unknown": bpu, "gbs": bpu * Nf / (kms * 1e-3) / 1e9,
                                "frac": bpu * Nf / (kms * 1e-3) / 1e9 / peak_hbm()[0], "launches_per_cycle": cnt / kp}
    # the smoother+residual pair of the last pre-smoothing step on the finest level: two
    # kernels (sweep, then residual), 24 B/unknown each; also against the 32 B/unknown a
    # single fused sweep+residual pass would need (the pair's lower bound)
    pair_ms = kernels["smooth"]["avg_ms"] + kernels["residual_standalone"]["avg_ms"]
    fused_gbs = 48 * Nf / (pair_ms * 1e-3) / 1e9
    coarse_ms = prof["coarse"][0][0] / max(1, prof["coarse"][1][0])
    stage_ms = {s: round(sum(prof[s][0]) / kp, 5) for s in prof}

    # V-cycle roofline: stage accounting b = 24(eta1+eta2)+52 B per smoothed unknown
    smoothed = sum(l["nreal"] * l["B"] ** 3 for l in levels[1:])
    eta = cfg["eta1"] + cfg["eta2"]
    rl_stage_ms = smoothed * (24 * eta + 52) / (peak * 1e9) * 1e3
    rl_fused_ms = smoothed * (24 * eta + 4) / (peak * 1e9) * 1e3

    # ---- e2e: the public API on host buffers (pinned), H2D + solve to 1e-10 + D2H per step
    S.use_graph(True)
    S.set_rhs(f_dev)
    ncyc, rel, ok = S.solve(1e-10, 30)
    fh = torch.from_numpy(f).pin_memory().numpy()
    uh = torch.empty(f.shape, dtype=torch.float64).pin_memory().numpy()
    S.run_host(fh, uh, ncyc)
    ke = max(1, min(args.steps, 5))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # CUDA events on the stream the library enqueues on (the legacy default stream):
    # mg_run_host enqueues H2D, set_rhs, the cycles and D2H there and synchronises
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(ke):
        rel_e2e = S.run_host(fh, uh, ncyc)
    h1.record(stream)
    torch.cuda.synchronize()
    te = max_over_ranks(h0.elapsed_time(h1) / ke * 1e-3, dist, dev)
    e2e = {"value": nleaf_unknowns * ncyc * ws / te, "unit": UNIT, "h2d_bytes_per_step": int(f.nbytes),
           "time_to_solution_ms": te * 1e3,
           "d2h_bytes_per_step": int(f.nbytes + 8), "cycles_per_step": ncyc, "rel_residual": rel_e2e,
           "ms_per_step": te * 1e3, "what": "mg_run_host: pinned f -> device, set_rhs (f*), V-cycles to rel. "
                                            "residual 1e-10, u -> pinned host"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: uniform periodic 256^3 (4096 blocks 16^3), M=4 Mehrstellen, RB V(2,2), "
                                   "3 MG levels (256^3, 128^3, 64^3 cuFFT coarse solve), 64 seeded Fourier modes",
                       "leaf_unknowns": nleaf_unknowns, "levels": nlev, "graph": True,
                       "l2": "inputs larger than L2 (u,u',f,r at 256^3 = 537 MB working set)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic("k_rb_pencil") if st == "smooth" else None,
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write "
                                           "per launch of the finest-level sweep)",
                         "peak_source": peak_src,
                         "kernel": f"{st} (level {lv}, {Nl} unknowns/launch)",
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms,
                         "frac_of_8TBps": achieved / NORTH_STAR_PEAK_GBS},
            "smoother_residual": {"gbs": fused_gbs, "ms": pair_ms, "frac": fused_gbs / peak,
                                  "unknowns_per_s": Nf / (pair_ms * 1e-3), "alg_bytes_per_unknown": 48,
                                  "frac_vs_fused_32B": 32 * Nf / (pair_ms * 1e-3) / 1e9 / peak,
                                  "what": "finest level: RB sweep kernel + standalone residual kernel (two "
                                          "launches, 24 B per unknown each); frac_vs_fused_32B rates the pair "
                                          "against one fused pass (32 B per unknown). In the V-cycle the "
                                          "residual is fused with the restriction ('restrict' stage: 16 B read "
                                          "+ 2 B coarse writes per fine unknown)"},
            "finest_level_kernels": kernels,
            "vcycle_roofline": {"stage_accounting_ms": rl_stage_ms, "fused_min_ms": rl_fused_ms,
                                "frac_stage": rl_stage_ms / ms, "frac_fused_min": rl_fused_ms / ms,
                                "excl_coarse_value": nleaf_unknowns / ((ms - coarse_ms) * 1e-3)},
            "coarse_solve_ms": coarse_ms, "stage_ms_per_cycle": stage_ms,
            "gpu_launches": launches_per_cycle * args.steps, "launches_per_cycle": launches_per_cycle,
            "clocks": clocks, "e2e": e2e}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, leaves, f)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["mine", "reference"], default="mine")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-n", type=int, default=0,
                    help="grid of the oracle's bounded sample (--impl reference); 0 = the largest of "
                         "128/64/32 that keeps the run within ~2.5 minutes")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank, dist)
    else:
        run_mine(args, ws, rank, local, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
