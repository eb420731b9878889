"""Thin ctypes binding of libmg.so (include/mg.h): argument marshalling only.

Every step of the solve runs in the library's CUDA kernels (plus cuFFT for the
coarse level).  There is no CPU fallback: if libmg.so or a CUDA device is
missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmg.so")

MG_BC_PERIODIC, MG_BC_UNBOUNDED, MG_BC_EVEN, MG_BC_ODD = 0, 1, 2, 3
MG_SMOOTHER_JACOBI, MG_SMOOTHER_RBGS = 0, 1
MG_CRIT_RESIDUAL, MG_CRIT_CAUCHY = 0, 1
MG_FIELD_U, MG_FIELD_F, MG_FIELD_R, MG_FIELD_UHAT = 0, 1, 2, 3
OPS = dict(refresh=0, smooth=1, residual=2, restrict=3, prolong=4, inject_up=5, coarse_solve=6,
           smooth_residual=7)
MG_OK, MG_WARN_NOT_CONVERGED = 0, 1
MG_ALL_BLOCKS = 0x10000

EXPORTS = ["mg_create", "mg_destroy", "mg_last_error", "mg_set_rhs", "mg_set_solution", "mg_get_solution",
           "mg_vcycle", "mg_residual_norm", "mg_solve", "mg_run_host", "mg_use_graph", "mg_level_info",
           "mg_level_blocks", "mg_num_levels", "mg_debug_field", "mg_debug_apply", "mg_time_op", "mg_profile",
           "mg_profile_read", "mg_kernel_launches", "mg_detail", "mg_adapt", "mg_debug_poison", "mg_transfer",
           "mg_setup_times"]
STAGES = ["smooth", "smooth_res", "residual", "ghost", "restrict", "prolong", "coarse", "inject_up", "norm", "fas"]


class MgDesc(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("h0", C.c_double), ("base_blocks", C.c_int32 * 3),
                ("block_size", C.c_int32), ("bc", C.c_int32 * 6), ("order", C.c_int32),
                ("coarse_n", C.c_int32), ("smoother", C.c_int32), ("omega", C.c_double),
                ("eta1", C.c_int32), ("eta2", C.c_int32), ("allow_unbounded_refined", C.c_int32),
                ("n_leaf", C.c_int64), ("leaves", C.POINTER(C.c_int32)), ("pencil_blocks", C.c_int32),
                ("zsplit", C.c_int32), ("fuse", C.c_int32), ("ncomp", C.c_int32), ("coarse_pruning", C.c_int32),
                ("staging", C.c_int32), ("ghost_kernel", C.c_int32), ("pencil_order", C.c_int32)]


class MgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libmg error {code}: {msg}")
        self.code = code


_lib = None


def load_library(path: str = _LIB_PATH):
    """Load libmg.so (fails loudly when the CUDA extension has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_2512_08555_b200.build` (nvcc, sm_100a)")
    lib = C.CDLL(path)
    P, I, D = C.c_void_p, C.c_int, C.c_double
    lib.mg_create.argtypes = [C.POINTER(MgDesc), P, C.POINTER(P)]
    lib.mg_destroy.argtypes = [P]
    lib.mg_destroy.restype = None
    lib.mg_last_error.argtypes = [P]
    lib.mg_last_error.restype = C.c_char_p
    for name in ("mg_set_rhs", "mg_set_solution", "mg_get_solution"):
        getattr(lib, name).argtypes = [P, P]
    lib.mg_vcycle.argtypes = [P, I]
    lib.mg_residual_norm.argtypes = [P, C.POINTER(D), C.POINTER(D)]
    lib.mg_solve.argtypes = [P, D, I, I, C.POINTER(I), C.POINTER(D)]
    lib.mg_run_host.argtypes = [P, P, P, I, C.POINTER(D)]
    lib.mg_use_graph.argtypes = [P, I]
    lib.mg_level_info.argtypes = [P, I, C.POINTER(C.c_int64)]
    lib.mg_level_blocks.argtypes = [P, I, C.POINTER(C.c_int32)]
    lib.mg_num_levels.argtypes = [P]
    lib.mg_debug_field.argtypes = [P, I, I, I, P]
    lib.mg_debug_apply.argtypes = [P, I, I]
    lib.mg_debug_poison.argtypes = [P]
    lib.mg_transfer.argtypes = [P, P]
    lib.mg_time_op.argtypes = [P, I, I, I, C.POINTER(D)]
    lib.mg_profile.argtypes = [P, I]
    lib.mg_profile_read.argtypes = [P, C.POINTER(D), C.POINTER(C.c_int64)]
    lib.mg_setup_times.argtypes = [P, C.POINTER(D)]
    lib.mg_kernel_launches.argtypes = []
    lib.mg_kernel_launches.restype = C.c_int64
    I32P = C.POINTER(C.c_int32)
    lib.mg_detail.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, P, P]
    lib.mg_adapt.argtypes = [I32P, I32P, C.c_int32, I32P, C.c_int32, C.POINTER(D), D, D, C.c_int32, I32P,
                             C.c_int32, I32P, I32P]
    lib.mg_detail.restype = C.c_int
    lib.mg_adapt.restype = C.c_int
    for name in EXPORTS:
        if name not in ("mg_destroy", "mg_last_error", "mg_kernel_launches"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _ptr(t):
    """Device pointer of a CUDA tensor (contiguous fp64)."""
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return C.c_void_p(t.data_ptr())


def detail(field, B, W, stream=None):
    """mg_detail: detail coefficient γ per leaf block of a leaf-ordered device field
    [n, B, B, B] (fp64 CUDA tensor); returns a [n] fp64 CUDA tensor."""
    import torch
    lib = load_library()
    n = int(field.shape[0])
    g = torch.empty(n, dtype=torch.float64, device=field.device)
    if stream is None:
        stream = torch.cuda.current_stream()
    rc = lib.mg_detail(_ptr(field) if n else None, n, int(B), int(W), _ptr(g) if n else None,
                       C.c_void_p(stream.cuda_stream))
    if rc < 0:
        raise MgError(rc, "mg_detail")
    return g


def adapt(cfg, leaves, gamma, eps_r, eps_c, max_level):
    """mg_adapt: new leaf list (int32 [m, 4], sorted) and the number of suppressed
    refinements, from per-leaf γ (host array) — host code in libmg.so."""
    lib = load_library()
    lv = np.ascontiguousarray(np.asarray(leaves, dtype=np.int32).reshape(-1, 4))
    g = np.ascontiguousarray(np.asarray(gamma, dtype=np.float64).reshape(-1))
    bb = (C.c_int32 * 3)(*[int(v) for v in cfg["base_blocks"]])
    bc3 = [int(v) for v in cfg["bc"]]
    bc = (C.c_int32 * 6)(bc3[0], bc3[0], bc3[1], bc3[1], bc3[2], bc3[2])
    n_out, n_sup = C.c_int32(), C.c_int32()
    cap = max(8 * len(lv), 64)
    while True:
        out = np.zeros((cap, 4), dtype=np.int32)
        rc = lib.mg_adapt(bb, bc, int(cfg.get("allow_unbounded_refined", 0)),
                          lv.ctypes.data_as(C.POINTER(C.c_int32)), len(lv),
                          g.ctypes.data_as(C.POINTER(C.c_double)), float(eps_r), float(eps_c), int(max_level),
                          out.ctypes.data_as(C.POINTER(C.c_int32)), cap, C.byref(n_out), C.byref(n_sup))
        if rc == MG_OK:
            return out[:n_out.value].copy(), n_sup.value
        if n_out.value > cap:
            cap = n_out.value
            continue
        raise MgError(rc, "mg_adapt")


class Solver:
    """Handle of one solver instance (mg_create ... mg_destroy)."""

    def __init__(self, cfg: dict, leaves: np.ndarray, stream=None):
        import torch
        self.lib = load_library()
        self.torch = torch
        lv = np.ascontiguousarray(np.asarray(leaves, dtype=np.int32).reshape(-1, 4))
        self._leaves = lv
        d = MgDesc()
        d.origin[:] = [float(v) for v in cfg["origin"]]
        d.h0 = float(cfg["h0"])
        d.base_blocks[:] = [int(v) for v in cfg["base_blocks"]]
        d.block_size = int(cfg["B"])
        # per axis: an int (both faces) or a (low, high) pair, e.g. (MG_BC_ODD, MG_BC_UNBOUNDED)
        faces = [(int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v)) for v in cfg["bc"]]
        d.bc[:] = [faces[0][0], faces[0][1], faces[1][0], faces[1][1], faces[2][0], faces[2][1]]
        d.order = int(cfg["order"])
        d.coarse_n = int(cfg.get("coarse_n", 0) or 0)
        d.smoother = int(cfg["smoother"])
        d.omega = float(cfg["omega"])
        d.eta1 = int(cfg["eta1"])
        d.eta2 = int(cfg["eta2"])
        d.allow_unbounded_refined = int(cfg.get("allow_unbounded_refined", 0))
        # kernel-variant controls (tests only; 0 = automatic)
        d.pencil_blocks = int(cfg.get("pencil_blocks", 0))
        d.zsplit = int(cfg.get("zsplit", 0))
        d.fuse = int(cfg.get("fuse", 0))
        d.staging = int(cfg.get("staging", 0))
        d.ncomp = int(cfg.get("ncomp", 1))
        d.coarse_pruning = int(cfg.get("coarse_pruning", 0))
        d.ghost_kernel = int(cfg.get("ghost_kernel", 0))
        d.pencil_order = int(cfg.get("pencil_order", 0))
        self.nc = max(1, d.ncomp)
        d.n_leaf = len(lv)
        d.leaves = lv.ctypes.data_as(C.POINTER(C.c_int32))
        self.B = int(cfg["B"])
        self.n_leaf = len(lv)
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        h = C.c_void_p()
        self._check(self.lib.mg_create(C.byref(d), C.c_void_p(stream.cuda_stream), C.byref(h)), None)
        self.h = h

    # ---------------------------------------------------------------- helpers
    def _check(self, rc, h="self"):
        if rc < 0:
            hh = self.h if h == "self" else None
            raise MgError(rc, self.lib.mg_last_error(hh).decode())
        return rc

    def close(self):
        if getattr(self, "h", None):
            self.lib.mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def leaf_shape(self):
        """[n_leaf, B, B, B], or [ncomp, n_leaf, B, B, B] for a batched handle."""
        s = (self.n_leaf, self.B, self.B, self.B)
        return (self.nc,) + s if self.nc > 1 else s

    # ---------------------------------------------------------------- API
    def set_rhs(self, f):
        self._check(self.lib.mg_set_rhs(self.h, _ptr(f)))

    def set_solution(self, u):
        self._check(self.lib.mg_set_solution(self.h, _ptr(u)))

    def get_solution(self, out=None):
        t = self.torch
        if out is None:
            out = t.empty(self.leaf_shape(), dtype=t.float64, device="cuda")
        self._check(self.lib.mg_get_solution(self.h, _ptr(out)))
        return out

    def vcycle(self, n=1):
        self._check(self.lib.mg_vcycle(self.h, int(n)))

    def residual_norm(self):
        a, r = C.c_double(), C.c_double()
        self._check(self.lib.mg_residual_norm(self.h, C.byref(a), C.byref(r)))
        return a.value, r.value

    def solve(self, tol, max_cycles=50, criterion=MG_CRIT_RESIDUAL):
        c, v = C.c_int(), C.c_double()
        rc = self._check(self.lib.mg_solve(self.h, float(tol), int(max_cycles), int(criterion), C.byref(c),
                                           C.byref(v)))
        return c.value, v.value, rc == MG_OK

    def solve_vector(self, f_components, tol, max_cycles=50, criterion=MG_CRIT_RESIDUAL):
        """Vector Poisson problem (the Biot–Savart law ∇²u = -∇×ω of P:627-631).
        On a handle created with ncomp = len(f_components) all components go through ONE
        batched solve: every V-cycle kernel launch covers all components, the tables,
        ghost boxes and the coarse-solve FFT plan are shared, the stopping test is the
        max over components (returns one stats tuple per component, all equal).
        Otherwise one scalar solve per component on this handle (a zero component is
        solved exactly by u = 0 without cycling).  f_components: sequence of leaf-ordered
        device tensors; returns ([u_c], [(cycles, rel, converged)])."""
        import torch
        if self.nc > 1:
            if len(f_components) != self.nc:
                raise ValueError(f"handle has ncomp={self.nc}, got {len(f_components)} components")
            f = torch.stack([t.contiguous() for t in f_components]).contiguous()
            self.set_rhs(f)
            self.set_solution(torch.zeros_like(f))
            st = self.solve(tol, max_cycles, criterion)
            u = self.get_solution()
            return [u[c] for c in range(self.nc)], [st] * self.nc
        us, stats = [], []
        for f in f_components:
            if not bool(torch.any(f != 0)):
                us.append(torch.zeros_like(f))
                stats.append((0, 0.0, True))
                continue
            self.set_rhs(f)
            self.set_solution(torch.zeros_like(f))
            stats.append(self.solve(tol, max_cycles, criterion))
            us.append(self.get_solution())
        return us, stats

    def run_host(self, f_host: np.ndarray, u_host: np.ndarray, ncycles: int) -> float:
        r = C.c_double()
        self._check(self.lib.mg_run_host(self.h, C.c_void_p(f_host.ctypes.data), C.c_void_p(u_host.ctypes.data),
                                         int(ncycles), C.byref(r)))
        return r.value

    def use_graph(self, on=True):
        self._check(self.lib.mg_use_graph(self.h, 1 if on else 0))

    def num_levels(self):
        return self._check(self.lib.mg_num_levels(self.h))

    def level_info(self, m):
        info = (C.c_int64 * 10)()
        self._check(self.lib.mg_level_info(self.h, int(m), info))
        keys = ["B", "nreal", "nghost", "Nx", "Ny", "Nz", "amr", "n_c2f", "n_inject", "n_leaf_blocks"]
        return dict(zip(keys, list(info)))

    def level_blocks(self, m, ghosts=False):
        info = self.level_info(m)
        n = info["nreal"] + (info["nghost"] if ghosts else 0)
        out = np.zeros((n, 3), dtype=np.int32)
        code = int(m) | (MG_ALL_BLOCKS if ghosts else 0)
        self._check(self.lib.mg_level_blocks(self.h, code, out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    def debug_field(self, field, m, tensor=None, ghosts=False):
        """Export (tensor None) or import a level field [nreal, B, B, B]; with
        ghosts=True export real then ghost blocks [nreal + nghost, B, B, B]."""
        t = self.torch
        info = self.level_info(m)
        if tensor is None:
            n = info["nreal"] + (info["nghost"] if ghosts else 0)
            out = t.empty((n, info["B"], info["B"], info["B"]), dtype=t.float64, device="cuda")
            self._check(self.lib.mg_debug_field(self.h, int(field), int(m), 2 if ghosts else 0, _ptr(out)))
            return out
        self._check(self.lib.mg_debug_field(self.h, int(field), int(m), 3 if ghosts else 1, _ptr(tensor)))

    def transfer_from(self, other):
        """mg_transfer: u on this (adapted) grid from the solution of `other` (call after
        set_rhs)."""
        self._check(self.lib.mg_transfer(self.h, other.h))

    def debug_poison(self):
        """NaN into every ghost-block node outside the needed halo (mg_debug_poison)."""
        self._check(self.lib.mg_debug_poison(self.h))

    def debug_apply(self, op, m):
        self._check(self.lib.mg_debug_apply(self.h, OPS[op] if isinstance(op, str) else int(op), int(m)))

    def profile(self, on=True):
        """Start (clears) / stop per-stage CUDA-event timing of non-graph launches."""
        self._check(self.lib.mg_profile(self.h, 1 if on else 0))

    def profile_read(self):
        """{stage: (ms[level], count[level])} accumulated since profile(True)."""
        nl = self.num_levels()
        ms = (C.c_double * (len(STAGES) * nl))()
        n = (C.c_int64 * (len(STAGES) * nl))()
        self._check(self.lib.mg_profile_read(self.h, ms, n))
        return {s: (list(ms[i * nl:(i + 1) * nl]), list(n[i * nl:(i + 1) * nl])) for i, s in enumerate(STAGES)}

    def kernel_launches(self):
        return int(self.lib.mg_kernel_launches())

    def setup_times(self):
        """Host wall time (ms) of mg_create's phases (include/mg.h mg_setup_times)."""
        ms = (C.c_double * 6)()
        self._check(self.lib.mg_setup_times(self.h, ms))
        return dict(zip(["hierarchy", "ghosts", "ghost_boxes", "pencils", "device_alloc", "coarse_setup"], list(ms)))

    def time_op(self, op, m, reps):
        ms = C.c_double()
        code = {"smooth_residual_fused_tile": -1, "smooth_residual_pair": -2, "vcycle": 100}.get(
            op, OPS.get(op, op)) if isinstance(op, str) else op
        self._check(self.lib.mg_time_op(self.h, int(code), int(m), int(reps), C.byref(ms)))
        return ms.value
