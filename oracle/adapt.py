"""ORACLE (test infrastructure only) — grid adaptation of the multiresolution grid
(§2.1, SPEC.md ops detail_coefficient / adapt /
enforce_two_to_one), plain numpy and Python sets.

Only tests/, __graft_entry__.smoke() and bench.py may import this module; the CUDA
path never does (its detail kernel is mg_adapt.cu, its tree logic mg_adapt.cpp).

detail(u_block, W) — the detail coefficient γ of one block ("a so-called detail
  coefficient γ"; SPEC: "the maximum absolute difference between a block's node values
  and the order-W polynomial interpolation of the coarsened (every-other-node)
  samples"; reading A1 in DESIGN.md): the coarse samples are the block's nodes with
  all-even local indices; along every axis an odd index j takes the W-point Lagrange
  interpolant of the even positions j-(W-1), j-(W-3), …, j+(W-1), shifted by steps of
  2 to stay inside the block (one-sided near its last node — SPEC "offset stencils
  drawn from interior nodes"); tensor product applied x, then y, then z; γ = max over
  the block's nodes of |u - P u|.

adapt(...) — P:65: "A grid block is refined into 8 finer blocks whenever its wavelet
  transform yields a so-called detail coefficient γ above ε_r. Alternatively, when all
  8 blocks involve detail coefficients below the coarsening threshold ε_c, they revert
  back to a single grid block"; "two adjacent blocks cannot have a resolution jump
  larger than one level" (26-neighbour 2:1 balance, refinement only); blocks touching
  an unbounded face stay at level 0 unless U1 is allowed.  Steps (reading A2):
  (1) refine the leaves with γ > ε_r below max_level; (2) coarsen complete octets of
  leaves, none refined in (1), all γ < ε_c, whose parent keeps the 2:1 constraint with
  the grid of (1); (3) balance by refinement until every leaf's parent has its 26
  neighbours present as blocks.
"""
from __future__ import annotations

import numpy as np

# 26 neighbour offsets (dx, dy, dz), dz slowest (the order of the tie-breaking scan)
OFFS26 = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dx, dy, dz) != (0, 0, 0)]


def taps_1d(j, B, W):
    """Even source positions and Lagrange weights of the order-W rule at odd j."""
    lo = j - (W - 1)
    lo = max(lo, 0)
    lo = min(lo, B - 2 - 2 * (W - 1))
    e = [lo + 2 * t for t in range(W)]
    w = []
    for t in range(W):
        num, den = 1.0, 1.0
        for s in range(W):
            if s != t:
                num *= (j - e[s])
                den *= (e[t] - e[s])
        w.append(num / den)
    return e, w


def interp_block(u, W):
    """P u on every node of one block u[z, y, x] (B^3) from its all-even nodes."""
    B = u.shape[0]
    rules = {}
    for j in range(B):
        rules[j] = ([j], [1.0]) if j % 2 == 0 else taps_1d(j, B, W)
    # pass x on even (z, y) rows, pass y on even z planes, pass z everywhere
    P1 = np.zeros((B, B, B))
    for z in range(0, B, 2):
        for y in range(0, B, 2):
            for x in range(B):
                e, w = rules[x]
                P1[z, y, x] = sum(wt * u[z, y, xe] for xe, wt in zip(e, w))
    P2 = np.zeros((B, B, B))
    for z in range(0, B, 2):
        for y in range(B):
            e, w = rules[y]
            P2[z, y, :] = sum(wt * P1[z, ye, :] for ye, wt in zip(e, w))
    P3 = np.zeros((B, B, B))
    for z in range(B):
        e, w = rules[z]
        P3[z] = sum(wt * P2[ze] for ze, wt in zip(e, w))
    return P3


def detail(u, W):
    """γ of one block (see the module header)."""
    return float(np.abs(u - interp_block(u, W)).max())


def details(field, W):
    """γ per leaf of a leaf-ordered field [n, B, B, B]."""
    return np.array([detail(field[n], W) for n in range(field.shape[0])])


class _Grid:
    def __init__(self, base_blocks, bc, allow_unbounded):
        self.nb0 = [int(v) for v in base_blocks]
        self.per = [int(b) == 0 for b in bc]
        self.allow = bool(allow_unbounded)

    def nb(self, lev, a):
        return self.nb0[a] << lev

    def wrap(self, lev, c):
        out = []
        for a in range(3):
            v = c[a]
            n = self.nb(lev, a)
            if self.per[a]:
                v %= n
            elif not 0 <= v < n:
                return None
            out.append(v)
        return tuple(out)

    def touches_unbounded(self, lev, c):
        return any((not self.per[a]) and (c[a] == 0 or c[a] == self.nb(lev, a) - 1) for a in range(3))


def _blocks_of(leaves):
    blocks = set()
    for (lev, x, y, z) in leaves:
        c = (x, y, z)
        for m in range(lev, -1, -1):
            blocks.add((m,) + c)
            c = (c[0] >> 1, c[1] >> 1, c[2] >> 1)
    return blocks


def _children(lev, c):
    return [(lev + 1, 2 * c[0] + i, 2 * c[1] + j, 2 * c[2] + k) for k in (0, 1) for j in (0, 1) for i in (0, 1)]


def _adapt_once(G, L, gam, eps_r, eps_c, max_level, forbidden):
    """One pass of steps (1)-(3); ('ok', leaves, suppressed) or ('bad', block) when the
    balance would have to refine a block that may not be refined (unbounded face, or
    forbidden by an earlier pass)."""
    def frozen(k):
        return (G.touches_unbounded(k[0], k[1:]) and not G.allow) or k in forbidden

    suppressed = 0
    refine = set()
    for lf in L:
        if gam[lf] > eps_r and lf[0] < max_level:
            if frozen(lf):
                suppressed += 1
                continue
            refine.add(lf)
    L1 = (L - refine) | {ch for lf in refine for ch in _children(lf[0], lf[1:])}
    blocks1 = _blocks_of(L1)
    parents = {}
    for lf in L:
        if lf[0] > 0 and lf not in refine:
            p = (lf[0] - 1, lf[1] >> 1, lf[2] >> 1, lf[3] >> 1)
            parents.setdefault(p, []).append(lf)
    coarsen = []
    for p, kids in parents.items():
        if len(kids) != 8 or not all(gam[k] < eps_c for k in kids):
            continue
        ok = True
        for o in OFFS26:
            q = G.wrap(p[0], (p[1] + o[0], p[2] + o[1], p[3] + o[2]))
            if q is None:
                continue
            for ch in _children(p[0], q):   # blocks two levels finer than p next to p
                if (ch[0] + 1, 2 * ch[1], 2 * ch[2], 2 * ch[3]) in blocks1:
                    ok = False
        if ok:
            coarsen.append(p)
    L2 = set(L1)
    for p in coarsen:
        for ch in _children(p[0], p[1:]):
            L2.discard(ch)
        L2.add(p)
    blocks = _blocks_of(L2)
    changed = True
    while changed:
        changed = False
        for lf in sorted(L2):
            if lf not in L2 or lf[0] < 2:
                continue
            m = lf[0] - 1
            for o in OFFS26:
                n = G.wrap(lf[0], (lf[1] + o[0], lf[2] + o[1], lf[3] + o[2]))
                if n is None:
                    continue
                q = (n[0] >> 1, n[1] >> 1, n[2] >> 1)   # the region of neighbour n needs level >= m
                if (m,) + q in blocks:
                    continue
                a, c = m, q
                while a > 0 and (a,) + c not in L2:
                    a, c = a - 1, (c[0] >> 1, c[1] >> 1, c[2] >> 1)
                if (a,) + c not in L2:
                    raise ValueError("leaves do not cover the domain")
                if frozen((a,) + c):
                    return "bad", (lf[0] - 1, lf[1] >> 1, lf[2] >> 1, lf[3] >> 1)
                L2.discard((a,) + c)
                for ch in _children(a, c):
                    L2.add(ch)
                    blocks.add(ch)
                changed = True
    return "ok", L2, suppressed


def adapt(base_blocks, bc, leaves, gamma, eps_r, eps_c, max_level, allow_unbounded=False):
    """New leaf set (sorted int32 rows (level, x, y, z)) and the number of leaves with
    γ > ε_r left unrefined by the constraints (diagnostic).  When the 2:1 balance would
    have to refine a block touching an unbounded face, the parent of the leaf
    that needs it is barred from refinement and the pass restarts from the input
    (reading A2), so the output always satisfies nesting, 2:1 and P:367."""
    G = _Grid(base_blocks, bc, allow_unbounded)
    L = {tuple(int(v) for v in r) for r in leaves}
    gam = {tuple(int(v) for v in r): float(g) for r, g in zip(leaves, gamma)}
    _validate(G, L, len(leaves))
    forbidden = set()
    while True:
        res = _adapt_once(G, L, gam, eps_r, eps_c, max_level, forbidden)
        if res[0] == "ok":
            out = np.array(sorted(res[1]), dtype=np.int32).reshape(-1, 4)
            return out, res[2]
        if res[1] in forbidden:          # no progress (cannot happen on a valid input)
            raise LayoutError("2:1", "adaptation made no progress")
        forbidden.add(res[1])


class LayoutError(ValueError):
    """Invalid input leaf set; `kind` in {"nesting", "2:1", "unbounded"} (the rules of
    P:65 and P:367 that mg_create also enforces)."""

    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def _validate(G, L, n_in):
    """No duplicates, no leaf with a descendant, complete octets, level 0 covered, no
    refined leaf on an unbounded face unless allowed.  (An input that is not 2:1
    balanced is accepted: step (3) balances it, or reports "2:1" when that would need
    a frozen block refined and barring parents makes no progress.)"""
    if len(L) != n_in:
        raise LayoutError("nesting", "duplicate leaf")
    blocks = _blocks_of(L)
    for lf in L:
        if any(ch in blocks for ch in _children(lf[0], lf[1:])):
            raise LayoutError("nesting", "leaf is also refined")
    for b in blocks:
        if b not in L and not all(ch in blocks for ch in _children(b[0], b[1:])):
            raise LayoutError("nesting", "partially refined block")
    if sum(1 for b in blocks if b[0] == 0) != G.nb0[0] * G.nb0[1] * G.nb0[2]:
        raise LayoutError("nesting", "level 0 not covered")
    for lf in L:
        if lf[0] > 0 and not G.allow and G.touches_unbounded(lf[0], lf[1:]):
            raise LayoutError("unbounded", "refined leaf on an unbounded face")

