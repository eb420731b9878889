#!/usr/bin/env python
"""Benchmark: V-cycle throughput of the B200 adaptive multigrid solver.

Headline workload (BASELINE.json configs[4], the largest single-GPU configuration):
cfg5 — adaptive 5-level grid, 30,003 leaf blocks of 16^3 (122.9M leaf unknowns,
34,216 real blocks on 5 levels), refined around a perturbed torus, x periodic / y, z
unbounded, 4th-order Mehrstellen, red-black V(2,2), cuFFT + LGF coarse solve on the
128 x 270 x 270 padded level 0 (workloads.configs.cfg5).  Secondary key "cfg2": the
uniform periodic 256^3 workload (configs[1]).  A step = one full V-cycle (every
hot-path kernel of every level + the coarse solve), one CUDA-graph launch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                  [--workload cfg5|cfg2] [--no-secondary] [--no-cpu-baseline]

Under torchrun (N > 1) every rank solves its own replica (the north star is one GPU,
no sharding), scaling = weak, timing = max over ranks.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
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
# algorithmic bytes per unknown of the level the stage is booked on (DESIGN.md
# §6): sweep (read u, f; write
# u'), residual (read u, f; write r), prolongation (read u, coarse ε; write u), fused
# residual + restriction (read u, f; write coarse u, coarse r: 16 + 2), FAS right-hand side
# on the coarse level (read u, r; write û; f on covered nodes only, not counted)
BYTES_PER_UNKNOWN = {"smooth": 24, "smooth_res": 32, "residual": 24, "prolong": 18, "restrict": 18, "fas": 24}


def peak_hbm():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM copy on this pool)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region:
    an NVML thread polling every 2 ms between __enter__ and __exit__ (the main thread
    waits in cudaEventSynchronize, which releases the GIL); nvidia-smi -lms 50 when NVML
    is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.p = None
        self.thread = None
        self.sm, self.mx, self.reasons, self.source = [], None, set(), None
        self.out = ""

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            return pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(self.index).uuid))
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        import threading
        try:
            import pynvml
            h = self._nvml_handle()
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons.update(n for n, bit in bits.items() if r & bit)
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.source = "nvml, 2 ms polling during the timed region"
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi -lms 50"
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=1)
            return
        if self.p is not None:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                self.sm.append(float(parts[0]))
                self.mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:]):
                if v.lower() in ("active", "1"):
                    self.reasons.add(n)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "sm_mhz_min": min(self.sm) if self.sm else None, "source": self.source}


def max_over_ranks(x, dist, device):
    """Max of a per-rank float over all ranks (device timing rule: the slowest rank)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(workload, kernel_prefix, level):
    """DRAM bytes (read + write) per launch of a kernel from the committed `ncu --set
    full` capture summary (profiles/ncu_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return None, None
    for k, v in d.get("by_workload", {}).get(workload, {}).items():
        if k.startswith(kernel_prefix) and v.get("level") == level:
            return v.get("dram_bytes_per_launch"), v.get("report")
    return None, None


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


# ------------------------------------------------------------------ workloads
def workload_cfg(name):
    from workloads import configs as C
    if name == "cfg5":
        return C.cfg5()
    if name == "cfg2":
        return C.cfg2(256)
    raise KeyError(name)


def oracle_sample_cfg(name, sample="full"):
    """The bounded CPU sample of a workload (same recipe, reduced size): cfg5 -> the
    cfg5 recipe (5 levels, perturbed torus, PUU, M=4, RB V(2,2)) on a 4^3 base with a
    smaller torus (R = 0.12, sigma = 0.02): 568 leaves, 2.33M leaf unknowns, ~7 s per
    oracle V-cycle on one core ('tiny': 2 levels, 99 leaves, ~3 s, for tests); cfg2 ->
    the cfg2 recipe at 128^3 ('tiny': 32^3)."""
    from workloads import configs as C
    if name == "cfg5":
        return C.cfg5(base=4, max_level=4 if sample == "full" else 1, target=1000 if sample == "full" else 100,
                      R=0.12, sigma=0.02)
    return C.cfg2(128 if sample == "full" else 32)


WORKLOAD_TEXT = {
    "cfg5": "cfg5: adaptive 5-level grid around a perturbed torus (R=0.5, sigma=0.03, 5% random modes), "
            "30003 leaf blocks 16^3, x periodic / y,z unbounded, M=4 Mehrstellen, RB V(2,2), cuFFT+LGF "
            "coarse solve of the 128x270x270 padded level 0",
    "cfg2": "cfg2: uniform periodic 256^3 (4096 blocks 16^3), M=4 Mehrstellen, RB V(2,2), 3 MG levels "
            "(256^3, 128^3, 64^3 cuFFT coarse solve), 64 seeded Fourier modes",
}


# ------------------------------------------------------------------ oracle timing
def _oracle_proc(name, sample, conn, barrier):
    """Worker process: builds the oracle on the sample once, then per request runs one
    V-cycle (started together with the other workers at a barrier) and reports
    (leaf unknowns, seconds)."""
    sys.path.insert(0, ROOT)
    from oracle.mg_oracle import Oracle
    from workloads import configs as C
    cfg = oracle_sample_cfg(name, sample)
    dom, leaves, f = C.build(cfg)
    o = Oracle(cfg, leaves)
    o.set_rhs(f)
    conn.send("ready")
    while conn.recv() == "cycle":
        barrier.wait()
        t = time.perf_counter()
        o.vcycle(1)
        conn.send((f.size, time.perf_counter() - t))


class OraclePool:
    """P oracle processes (one per host core; spawned, numpy single-threaded each)."""

    def __init__(self, name, sample, P):
        ctx = mp.get_context("spawn")
        env = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env:
            os.environ[k] = "1"
        b = ctx.Barrier(P)
        self.conns, self.procs = [], []
        for _ in range(P):
            a, c = ctx.Pipe()
            pr = ctx.Process(target=_oracle_proc, args=(name, sample, c, b), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for a in self.conns:
            assert a.recv() == "ready"
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v

    def cycle(self):
        """One concurrent V-cycle in every worker: (total unknowns, slowest seconds)."""
        for a in self.conns:
            a.send("cycle")
        res = [a.recv() for a in self.conns]
        return sum(r[0] for r in res), max(r[1] for r in res)

    def close(self):
        for a in self.conns:
            a.send("stop")
        for pr in self.procs:
            pr.join(timeout=30)


def host_cores():
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


MAX_ORACLE_PROCS = 32


def cpu_baseline(name):
    """The oracle as it stands (numpy, single-threaded per process) on a bounded sample of
    the workload: one V-cycle alone on 1 core, and one V-cycle per process on all host
    cores (independent processes, up to 32, started together)."""
    cores, model = host_cores()
    cfg = oracle_sample_cfg(name, "full")
    from workloads import configs as C
    C.leaves_for(cfg)                       # layout cache filled before the workers start
    one = OraclePool(name, "full", 1)
    n1, t1 = one.cycle()
    one.close()
    P = min(cores, MAX_ORACLE_PROCS)
    pool = OraclePool(name, "full", P)
    nall, tall = pool.cycle()
    pool.close()
    return {"value": nall / tall, "unit": UNIT, "cores": P, "kind": "oracle",
            "single_core": {"value": n1 / t1, "unit": UNIT, "cores": 1, "seconds": t1},
            "host": {"cores_available": cores, "cpu_model": model},
            "sample": f"1 oracle V-cycle of {cfg['name']} ({n1} leaf unknowns; the {name} recipe at reduced "
                      f"size) per process: {P} concurrent processes ({tall:.1f} s), and alone on 1 core "
                      f"({t1:.1f} s); reference CPU baseline, not the target"}


def run_reference(args, ws, rank, dist):
    """--impl reference: the CPU oracle (this tier's reference arm) on a bounded sample of
    the same workload; each step = one oracle V-cycle of the sample in each of P worker
    processes (one per host core, P <= 32), started together; value = all workers'
    leaf unknowns / the slowest worker's V-cycle time."""
    if rank != 0:
        return
    name = args.workload
    cores, model = host_cores()
    P = min(cores, MAX_ORACLE_PROCS)
    if args.ref_sample == "auto":
        args.ref_sample = "full" if (args.steps + args.warmup) * 13.0 <= 180.0 else "tiny"
    cfg = oracle_sample_cfg(name, args.ref_sample)
    from workloads import configs as C
    C.leaves_for(cfg)
    pool = OraclePool(name, args.ref_sample, P)
    times, n = [], 0
    for it in range(args.warmup + args.steps):
        n, dt = pool.cycle()
        if it >= args.warmup:
            times.append(dt)
    pool.close()
    dt = sum(times) / len(times)
    val = n / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[name] + f" -- bounded CPU sample: {cfg['name']} (the same recipe "
                                   "at reduced size), one V-cycle per worker process per step",
                       "leaf_unknowns_per_process": n // P, "processes": P},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": P, "kind": "oracle",
                             "host": {"cores_available": cores, "cpu_model": model},
                             "sample": f"1 oracle V-cycle of {cfg['name']} per process per step, {P} processes"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def measure(S, cfg, args, dist, dev, ws, local, with_clocks=True):
    """V-cycle timing (graph, CUDA events), per-stage live kernel times (non-graph,
    CUDA events per stage), roofline of the dominant kernel."""
    import torch
    nlev = S.num_levels()
    levels = [S.level_info(m) for m in range(nlev)]
    # launches per V-cycle (our kernels only; cuFFT's own kernels excluded)
    S.use_graph(False)
    c0 = S.kernel_launches()
    S.vcycle(1)
    torch.cuda.synchronize()
    launches_per_cycle = S.kernel_launches() - c0

    S.use_graph(True)
    for _ in range(args.warmup):
        S.vcycle(1)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def timed_region():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(local) if with_clocks else None
        if clk:
            clk.__enter__()
        e0.record(stream)
        for _ in range(args.steps):
            S.vcycle(1)
        e1.record(stream)
        torch.cuda.synchronize()
        if clk:
            clk.__exit__()
        if dist:
            dist.barrier()
        return max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, dev), clk

    ms, clk = timed_region()
    # timing rule: a region that saw a hardware / thermal slowdown, or SM clocks well
    # below max with no reason, is rejected and measured once more
    remeasured, flag = None, 0.0
    if clk:
        c = clk.summary()
        bad = [r for r in c["reasons"] if r != "sw_power_cap"]
        low = c["sm_mhz"] is not None and c["sm_max_mhz"] and not c["reasons"] and c["sm_mhz"] < 0.85 * c["sm_max_mhz"]
        flag = 1.0 if (bad or low) else 0.0
    if max_over_ranks(flag, dist, dev) > 0:  # every rank re-runs the region (barriers inside)
        remeasured = {"first_ms_per_step": ms, "first_clocks": clk.summary() if clk else None}
        ms, clk = timed_region()

    # per-stage live timing (CUDA events on the library's stream around every stage)
    S.use_graph(False)
    S.profile(True)
    kp = max(3, min(args.steps, 10))
    for _ in range(kp):
        S.vcycle(1)
    prof = S.profile_read()
    S.profile(False)
    peak, peak_src = peak_hbm()
    kernels = {}
    for st in BYTES_PER_UNKNOWN:
        for m in range(nlev):
            tot, cnt = prof[st][0][m], prof[st][1][m]
            if not cnt:
                continue
            Nl = levels[m]["nreal"] * levels[m]["B"] ** 3
            kms = tot / cnt
            gbs = BYTES_PER_UNKNOWN[st] * Nl / (kms * 1e-3) / 1e9
            kernels[f"{st}@{m}"] = {"avg_ms": kms, "launches_per_cycle": cnt / kp, "unknowns": Nl,
                                    "alg_bytes_per_unknown": BYTES_PER_UNKNOWN[st], "gbs": gbs, "frac": gbs / peak,
                                    "share_of_cycle": tot / kp / ms}
    dom = max(kernels, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches_per_cycle"])
    st, lv = dom.split("@")
    lv = int(lv)
    K = kernels[dom]
    stage_ms = {s: round(sum(prof[s][0]) / kp, 5) for s in prof}
    coarse_ms = prof["coarse"][0][0] / max(1, prof["coarse"][1][0])
    smoothed = sum(l["nreal"] * l["B"] ** 3 for l in levels[1:])
    eta = cfg["eta1"] + cfg["eta2"]
    rl_stage_ms = smoothed * (24 * eta + 52) / (peak * 1e9) * 1e3
    rl_fused_ms = smoothed * (24 * eta + 4) / (peak * 1e9) * 1e3
    return dict(ms=ms, clocks=dict(clk.summary(), remeasured=remeasured) if clk else None, levels=levels, kernels=kernels, dom=(st, lv, K),
                stage_ms=stage_ms, coarse_ms=coarse_ms, launches_per_cycle=launches_per_cycle,
                rl_stage_ms=rl_stage_ms, rl_fused_ms=rl_fused_ms, peak=peak, peak_src=peak_src)


def smoother_residual(S, levels):
    """The smoother + residual of the last pre-smoothing step on the
    finest level, kernels only (no ghost refresh), 20 launches each: the production pair
    (RB pencil sweep 24 B + residual pencil kernel 24 B per unknown; in the V-cycle the
    residual is fused with the restriction instead) and the single-pass fused tile kernel
    (32 B per unknown); fractions of the measured HBM peak on each one's bytes, and of
    the pair against the 32 B a single pass needs."""
    top = len(levels) - 1
    Nf = levels[top]["nreal"] * levels[top]["B"] ** 3
    peak = peak_hbm()[0]
    out = {}
    for name, op, bpu in (("pair", "smooth_residual_pair", 48), ("fused_tile", "smooth_residual_fused_tile", 32)):
        S.time_op(op, top, 3)
        ms = S.time_op(op, top, 20)
        gbs = bpu * Nf / (ms * 1e-3) / 1e9
        out[name] = {"avg_ms": ms, "alg_bytes_per_unknown": bpu, "gbs": gbs, "frac": gbs / peak,
                     "frac_vs_single_pass_32B": 32 * Nf / (ms * 1e-3) / 1e9 / peak,
                     "unknowns_per_s": Nf / (ms * 1e-3)}
    out["what"] = ("finest level, kernels only: 'pair' = k_rb_pencil then k_res_pencil (production; in the "
                   "V-cycle the residual is fused with the restriction, k_rr2_pencil); 'fused_tile' = one "
                   "k_smooth2 pass (halo-3 tile: red, black and r = f - Lu)")
    out["unknowns"] = Nf
    return out


def run_mine(args, ws, rank, local, dist):
    import torch

    from paper_2512_08555_b200 import Solver
    from workloads import configs as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    name = args.workload
    cfg = workload_cfg(name)
    dom, leaves, f = C.build(cfg)
    nleaf_unknowns = f.size
    t_setup = time.perf_counter()
    S = Solver(cfg, leaves)
    setup = {"ms": (time.perf_counter() - t_setup) * 1e3, "phases_ms": S.setup_times(),
             "what": "mg_create of the workload layout (host tables, device allocation, coarse-solve setup)"}
    f_dev = torch.from_numpy(f).to(dev)
    S.set_rhs(f_dev)
    R = measure(S, cfg, args, dist, dev, ws, local)
    ms = R["ms"]
    value = nleaf_unknowns * ws / (ms * 1e-3)
    st, lv, K = R["dom"]
    peak = R["peak"]
    traffic, report = ncu_traffic(name, {"smooth": "k_rb_pencil", "restrict": "k_rr2_pencil",
                                         "prolong": "k_prolong2"}.get(st, st), lv)
    sr = smoother_residual(S, R["levels"])

    # ---- e2e: the public API on host buffers (pinned), H2D + solve to 1e-10 + D2H per step
    S.use_graph(True)
    S.set_rhs(f_dev)
    ncyc, rel, ok = S.solve(1e-10, 40)
    fh = torch.from_numpy(f).pin_memory().numpy()
    uh = torch.empty(f.shape, dtype=torch.float64).pin_memory().numpy()
    S.run_host(fh, uh, ncyc)
    ke = max(1, min(args.steps, 3))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(ke):
        rel_e2e = S.run_host(fh, uh, ncyc)
    h1.record(stream)
    torch.cuda.synchronize()
    te = max_over_ranks(h0.elapsed_time(h1) / ke * 1e-3, dist, dev)
    e2e = {"value": nleaf_unknowns * ncyc * ws / te, "unit": UNIT, "h2d_bytes_per_step": int(f.nbytes),
           "d2h_bytes_per_step": int(f.nbytes + 8), "cycles_per_step": ncyc, "rel_residual": rel_e2e,
           "time_to_solution_ms": te * 1e3,
           "what": "mg_run_host: pinned f -> device, set_rhs (f*), V-cycles to rel. residual 1e-10, u -> pinned host"}
    levels = R["levels"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[name], "leaf_unknowns": nleaf_unknowns, "leaves": len(leaves),
                       "levels": len(levels), "blocks_per_level": [l["nreal"] for l in levels],
                       "ghost_blocks_per_level": [l["nghost"] for l in levels], "graph": True,
                       "l2": "inputs larger than L2 (working set of u, u', f, r, u_hat on all levels >> 126 MB)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": K["gbs"], "peak": peak, "unit": "GB/s", "frac": K["gbs"] / peak,
                         "traffic": traffic,
                         "traffic_source": f"profiles/ncu_traffic.json ({report})" if report else None,
                         "peak_source": R["peak_src"],
                         "kernel": f"{st} on level {lv} ({K['unknowns']} unknowns per launch, "
                                   f"{K['alg_bytes_per_unknown']} B algorithmic per unknown)",
                         "alg_bytes_per_launch": K["alg_bytes_per_unknown"] * K["unknowns"],
                         "avg_launch_ms": K["avg_ms"], "share_of_cycle": K["share_of_cycle"],
                         "frac_of_8TBps": K["gbs"] / NORTH_STAR_PEAK_GBS},
            "smoother_residual": sr,
            "kernels": R["kernels"],
            "vcycle_roofline": {"stage_accounting_ms": R["rl_stage_ms"], "fused_min_ms": R["rl_fused_ms"],
                                "frac_stage": R["rl_stage_ms"] / ms, "frac_fused_min": R["rl_fused_ms"] / ms,
                                "excl_coarse_value": nleaf_unknowns / ((ms - R["coarse_ms"]) * 1e-3)},
            "coarse_solve_ms": R["coarse_ms"], "stage_ms_per_cycle": R["stage_ms"],
            "gpu_launches": R["launches_per_cycle"] * args.steps, "launches_per_cycle": R["launches_per_cycle"],
            "clocks": R["clocks"], "e2e": e2e, "setup": setup}
    del S
    torch.cuda.empty_cache()

    # ---- secondary workload: cfg2 (uniform periodic 256^3)
    if not args.no_secondary and name == "cfg5":
        c2 = workload_cfg("cfg2")
        _, lv2, f2 = C.build(c2)
        S2 = Solver(c2, lv2)
        S2.set_rhs(torch.from_numpy(f2).to(dev))
        R2 = measure(S2, c2, args, dist, dev, ws, local, with_clocks=False)
        st2, l2, K2 = R2["dom"]
        line["cfg2"] = {"workload": WORKLOAD_TEXT["cfg2"], "value": f2.size * ws / (R2["ms"] * 1e-3),
                        "ms_per_step": R2["ms"], "unit": UNIT,
                        "roofline": {"kernel": f"{st2} on level {l2}", "achieved": K2["gbs"], "frac": K2["gbs"] / peak,
                                     "avg_launch_ms": K2["avg_ms"]},
                        "smoother_residual": smoother_residual(S2, R2["levels"]), "kernels": R2["kernels"],
                        "vcycle_roofline": {"frac_stage": R2["rl_stage_ms"] / R2["ms"],
                                            "frac_fused_min": R2["rl_fused_ms"] / R2["ms"]},
                        "coarse_solve_ms": R2["coarse_ms"], "launches_per_cycle": R2["launches_per_cycle"]}
        line["gpu_launches"] += R2["launches_per_cycle"] * args.steps
        del S2
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["mine", "reference"], default="mine")
    ap.add_argument("--workload", choices=["cfg5", "cfg2"], default="cfg5")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", choices=["auto", "full", "tiny"], default="auto",
                    help="--impl reference: the oracle sample per step; auto = full (5 levels, ~13 s per step "
                         "with all cores busy) when the whole run stays under ~3 minutes, else tiny (2 levels)")
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
