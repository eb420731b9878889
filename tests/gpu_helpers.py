"""Helpers shared by the -m gpu parity tests: map between the GPU's per-level block
storage (exported through mg_debug_field) and the oracle's dense level lattices, and a
per-process memo of oracle states (the oracle does not depend on the kernel-variant
controls, so the variant tests reuse one oracle trajectory per layout)."""
import copy
import hashlib
from collections import OrderedDict

import numpy as np

# mg_desc kernel-variant controls: they select GPU kernels only, never the oracle
VARIANT_KNOBS = ("pencil_blocks", "zsplit", "fuse", "staging", "ghost_kernel", "coarse_pruning", "pencil_order")
_OCACHE = OrderedDict()
_OCACHE_MAX = 24


def oracle_key(cfg, leaves, f):
    items = tuple(sorted((k, repr(v)) for k, v in cfg.items() if k not in VARIANT_KNOBS))
    h = hashlib.sha1(np.ascontiguousarray(np.asarray(leaves)).tobytes())
    h.update(np.ascontiguousarray(np.asarray(f)).tobytes())
    return items, h.hexdigest()


def memo_get(key):
    if key in _OCACHE:
        _OCACHE.move_to_end(key)
        return copy.deepcopy(_OCACHE[key])
    return None


def memo_put(key, oracle):
    _OCACHE[key] = copy.deepcopy(oracle)
    while len(_OCACHE) > _OCACHE_MAX:
        _OCACHE.popitem(last=False)


def blocks_to_dense(blocks, coords, B, n, lo=(0, 0, 0), fill=np.nan):
    """blocks [nb, B, B, B] ([b, z, y, x]) at block coords -> the oracle's level array
    [nx, ny, nz] over the window [lo, lo + n) of level-global node indices."""
    out = np.full(tuple(n), fill)
    for b, c in enumerate(coords.tolist()):
        i, j, k = (c[a] * B - lo[a] for a in range(3))
        out[i:i + B, j:j + B, k:k + B] = blocks[b].transpose(2, 1, 0)
    return out


def dense_to_blocks(dense, coords, B, lo=(0, 0, 0)):
    out = np.empty((len(coords), B, B, B))
    for b, c in enumerate(coords.tolist()):
        i, j, k = (c[a] * B - lo[a] for a in range(3))
        out[b] = dense[i:i + B, j:j + B, k:k + B].transpose(2, 1, 0)
    return out


def rel_err(a, b, denom=None):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.abs(a - b).max()
    s = np.abs(b).max() if denom is None else denom
    return d / s if s > 0 else d


class Pair:
    """An oracle and a GPU solver built from the same config, leaves and f."""

    def __init__(self, cfg, leaves, f):
        import torch

        from oracle.mg_oracle import Oracle
        from paper_2512_08555_b200 import Solver

        self.torch = torch
        self.key = oracle_key(cfg, leaves, f)
        self.ncyc = 0
        self.o = memo_get((self.key, 0))
        if self.o is None:
            self.o = Oracle(cfg, leaves)
            self.o.set_rhs(f)
            memo_put((self.key, 0), self.o)
        self.g = Solver(cfg, leaves)
        self.f = f
        self.g.set_rhs(torch.from_numpy(np.ascontiguousarray(f)).cuda())
        assert self.g.num_levels() == len(self.o.levels)
        self.coords = [self.g.level_blocks(m) for m in range(self.g.num_levels())]
        self.B = [self.g.level_info(m)["B"] for m in range(self.g.num_levels())]

    def ocycle(self):
        """One oracle V-cycle, memoised per (layout, cycle count): only for tests whose
        oracle is cycled and read, never modified in between."""
        self.ncyc += 1
        o = memo_get((self.key, self.ncyc))
        if o is None:
            self.o.vcycle(1)
            memo_put((self.key, self.ncyc), self.o)
        else:
            self.o = o

    def gpu_field(self, field, m):
        from paper_2512_08555_b200 import MG_FIELD_F, MG_FIELD_R, MG_FIELD_U, MG_FIELD_UHAT
        code = dict(u=MG_FIELD_U, f=MG_FIELD_F, r=MG_FIELD_R, uhat=MG_FIELD_UHAT)[field]
        t = self.g.debug_field(code, m).cpu().numpy()
        L = self.o.levels[m]
        return blocks_to_dense(t, self.coords[m], self.B[m], L.n, L.lo)

    def push(self, field, m, dense):
        from paper_2512_08555_b200 import MG_FIELD_F, MG_FIELD_R, MG_FIELD_U, MG_FIELD_UHAT
        code = dict(u=MG_FIELD_U, f=MG_FIELD_F, r=MG_FIELD_R, uhat=MG_FIELD_UHAT)[field]
        t = self.torch.from_numpy(dense_to_blocks(dense, self.coords[m], self.B[m], self.o.levels[m].lo)).cuda()
        self.g.debug_field(code, m, t)

    def push_state(self):
        """Copy the oracle's u, f, uhat on every level into the GPU level storage."""
        for m, L in enumerate(self.o.levels):
            self.push("u", m, L.u)
            self.push("f", m, L.f)
            self.push("uhat", m, L.uhat)

    def solution(self):
        return self.g.get_solution().cpu().numpy()

    def push_exterior(self, field, m, ext_arr):
        """Write the oracle's extended-array values (pad E) at the exterior ghost-block
        nodes of GPU level m (U1 band snapshots), keeping everything else."""
        from oracle.mg_oracle import E
        from paper_2512_08555_b200 import MG_FIELD_F, MG_FIELD_R, MG_FIELD_U, MG_FIELD_UHAT
        code = dict(u=MG_FIELD_U, f=MG_FIELD_F, r=MG_FIELD_R, uhat=MG_FIELD_UHAT)[field]
        allb = self.g.debug_field(code, m, ghosts=True).cpu().numpy()
        coords = self.g.level_blocks(m, ghosts=True)
        nreal = self.g.level_info(m)["nreal"]
        B = self.B[m]
        N = self.o.levels[m].N
        lo = self.o.levels[m].lo
        per = self.o.per
        for g in range(nreal, len(coords)):
            c = coords[g]
            if all(per[a] or 0 <= c[a] * B < N[a] for a in range(3)):
                continue                      # a jump ghost block, not exterior
            for lz in range(B):
                for ly in range(B):
                    for lx in range(B):
                        X = (c[0] * B + lx + E - lo[0], c[1] * B + ly + E - lo[1], c[2] * B + lz + E - lo[2])
                        if all(0 <= X[a] < ext_arr.shape[a] for a in range(3)) and np.isfinite(ext_arr[X]):
                            allb[g, lz, ly, lx] = ext_arr[X]
        self.g.debug_field(code, m, self.torch.from_numpy(allb).cuda(), ghosts=True)
