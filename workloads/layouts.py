"""Block-layout (leaf list) generators for the block-structured multiresolution grid.

The grid follows PAPER.md §2.1: a forest of octrees of fixed-size
blocks, each refined into 8 finer blocks, with the 2:1 constraint ("two adjacent
blocks cannot have a resolution jump larger than one level") and, per
§3.3, "every block containing an unbounded boundary must be at the
coarsest level".  A layout is a leaf list: int32 rows ``(level, bi, bj, bk)``
(the SPEC.md grid-dump order ``level i j k``).  Level-k block (bi,bj,bk) owns the
level-global node indices ``B*(bi,bj,bk) + [0,B)^3``.

This module is harness code (no method arithmetic); the refinement *criterion*
used for configs 4/5 is a workload recipe, not the paper's
wavelet detail coefficient (that adaptation is out of this round's scope).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

PERIODIC = 0
UNBOUNDED = 1

OFFS26 = [o for o in itertools.product((-1, 0, 1), repeat=3) if o != (0, 0, 0)]


@dataclass
class Domain:
    """Geometry of the composite grid.

    origin: physical coordinates of level-global node 0.
    h0:     spacing of AMR level 0.
    base_blocks: number of level-0 blocks per axis.
    B:      nodes per block edge.
    bc:     per axis, PERIODIC or UNBOUNDED.
    """

    origin: tuple
    h0: float
    base_blocks: tuple
    B: int
    bc: tuple

    def nblocks(self, level: int) -> np.ndarray:
        return np.asarray(self.base_blocks, dtype=np.int64) << level

    def nnodes(self, level: int) -> np.ndarray:
        return self.nblocks(level) * self.B

    def h(self, level: int) -> float:
        return self.h0 / (1 << level)


def uniform_leaves(dom: Domain, level: int = 0) -> np.ndarray:
    nb = dom.nblocks(level)
    rows = [(level, i, j, k) for k in range(nb[2]) for j in range(nb[1]) for i in range(nb[0])]
    return np.asarray(rows, dtype=np.int32).reshape(-1, 4)


class Tree:
    """Set of existing blocks per level (leaves + internal nodes)."""

    def __init__(self, dom: Domain):
        self.dom = dom
        nb = dom.nblocks(0)
        self._nb0 = tuple(int(v) for v in nb)
        # an axis entry is PERIODIC, UNBOUNDED, or a (low, high) face pair (semi-unbounded:
        # an even/odd low face with an unbounded high face); only PERIODIC wraps
        self._per = tuple(dom.bc[d] == PERIODIC for d in range(3))
        self.nodes: dict[int, set] = {0: {(i, j, k) for i in range(nb[0]) for j in range(nb[1]) for k in range(nb[2])}}

    def has(self, lev, b):
        return b in self.nodes.get(lev, ())

    def refined(self, lev, b):
        return (2 * b[0], 2 * b[1], 2 * b[2]) in self.nodes.get(lev + 1, ())

    def refine(self, lev, b):
        s = self.nodes.setdefault(lev + 1, set())
        for o in itertools.product((0, 1), repeat=3):
            s.add((2 * b[0] + o[0], 2 * b[1] + o[1], 2 * b[2] + o[2]))

    def unrefine(self, lev, b):
        """Remove all descendants of (lev, b)."""
        stack = [(lev, b)]
        while stack:
            l, c = stack.pop()
            for o in itertools.product((0, 1), repeat=3):
                ch = (2 * c[0] + o[0], 2 * c[1] + o[1], 2 * c[2] + o[2])
                if ch in self.nodes.get(l + 1, ()):
                    self.nodes[l + 1].discard(ch)
                    stack.append((l + 1, ch))

    def leaves(self):
        out = []
        for lev in sorted(self.nodes):
            for b in sorted(self.nodes[lev], key=lambda t: (t[2], t[1], t[0])):
                if not self.refined(lev, b):
                    out.append((lev, *b))
        return np.asarray(out, dtype=np.int32).reshape(-1, 4)

    def wrap(self, lev, b):
        """Periodic wrap of block coords; None if outside an unbounded axis."""
        c = list(b)
        for d in range(3):
            n = self._nb0[d] << lev
            if self._per[d]:
                c[d] %= n
            elif not (0 <= c[d] < n):
                return None
        return tuple(c)

    def touches_unbounded_face(self, lev, b):
        nb = self.dom.nblocks(lev)
        return any(self.dom.bc[d] != PERIODIC and (b[d] == 0 or b[d] == nb[d] - 1) for d in range(3))

    def ensure(self, lev, b, forbid):
        """Make block (lev, b) exist by refining ancestors. Returns the forbidden
        ancestor that would have to be refined, or None on success."""
        if lev == 0 or self.has(lev, b):
            return None
        p = (b[0] // 2, b[1] // 2, b[2] // 2)
        r = self.ensure(lev - 1, p, forbid)
        if r is not None:
            return r
        if forbid(lev - 1, p):
            return (lev - 1, p)
        self.refine(lev - 1, p)
        return None

    def balance(self, forbid):
        """26-neighbour 2:1 balance. Returns [] or the list of (leaf_level, leaf)
        whose refinement cannot be balanced without refining a forbidden block.

        One pass from the finest level down suffices: making the level-(lev-1)
        neighbourhood of a level-lev leaf exist only refines blocks of levels
        <= lev-2, i.e. creates blocks of levels < lev, which are visited later."""
        bad = []
        for lev in sorted(self.nodes, reverse=True):
            if lev < 2:
                continue
            for b in sorted(self.nodes[lev]):
                if self.refined(lev, b):
                    continue
                for o in OFFS26:
                    n = self.wrap(lev, (b[0] + o[0], b[1] + o[1], b[2] + o[2]))
                    if n is None:
                        continue
                    p = (n[0] // 2, n[1] // 2, n[2] // 2)
                    if self.has(lev - 1, p):
                        continue
                    r = self.ensure(lev - 1, p, forbid)
                    if r is not None:
                        bad.append((lev, b))
                        break
            if bad:
                break
        return bad


def check_layout(dom: Domain, leaves: np.ndarray) -> None:
    """Validate nesting/coverage, 26-neighbour 2:1 balance and the unbounded-face
    rule. Raises ValueError."""
    t = Tree(dom)
    t.nodes = {}
    leafset = set()
    for lev, i, j, k in leaves.tolist():
        leafset.add((lev, (i, j, k)))
        t.nodes.setdefault(lev, set()).add((i, j, k))
        c = (i, j, k)
        for l in range(lev - 1, -1, -1):
            c = (c[0] // 2, c[1] // 2, c[2] // 2)
            t.nodes.setdefault(l, set()).add(c)
    nb0 = dom.nblocks(0)
    if len(t.nodes.get(0, ())) != int(np.prod(nb0)):
        raise ValueError("level 0 not fully covered")
    # every internal node must have all 8 children
    for lev in t.nodes:
        for b in t.nodes[lev]:
            kids = [(2 * b[0] + o[0], 2 * b[1] + o[1], 2 * b[2] + o[2]) for o in itertools.product((0, 1), repeat=3)]
            present = [c in t.nodes.get(lev + 1, ()) for c in kids]
            if any(present) and not all(present):
                raise ValueError(f"block {lev},{b} partially refined")
            if any(present) and (lev, b) in leafset:
                raise ValueError(f"leaf {lev},{b} also refined")
    for lev, b in leafset:
        if lev > 0 and t.touches_unbounded_face(lev, b):
            raise ValueError(f"refined block {lev},{b} touches an unbounded face")
        for o in OFFS26:
            n = t.wrap(lev, (b[0] + o[0], b[1] + o[1], b[2] + o[2]))
            if n is None:
                continue
            # the region of neighbour n must be covered by leaves of level >= lev-1
            if lev >= 2:
                p = (n[0] // 2, n[1] // 2, n[2] // 2)
                if not t.has(lev - 1, p):
                    raise ValueError(f"2:1 violated near {lev},{b}")


def adaptive_leaves(dom: Domain, max_level: int, score, tau: float) -> np.ndarray:
    """Refine every block whose score(level, blocks)*... exceeds tau, top-down,
    then 2:1-balance; blocks touching unbounded faces are never refined.
    `score(level, coords[n,3]) -> array[n]` (max |f| h_level^2 over block nodes).
    """
    dom_forbid = set()

    def forbid(lev, b):
        return (lev, b) in dom_forbid or Tree.touches_unbounded_face(t, lev, b) or lev >= max_level

    while True:
        t = Tree(dom)
        for lev in range(max_level):
            cand = sorted(b for b in t.nodes.get(lev, ()) if not forbid(lev, b))
            if not cand:
                break
            s = score(lev, np.asarray(cand, dtype=np.int64))
            for b, v in zip(cand, s):
                if v > tau:
                    t.refine(lev, b)
        bad = t.balance(forbid)
        if not bad:
            return t.leaves()
        for lev, b in bad:
            dom_forbid.add((lev - 1, (b[0] // 2, b[1] // 2, b[2] // 2)))


def bisect_tau(dom: Domain, max_level: int, score, target: int, iters: int = 40):
    """Deterministic log-bisection of tau so the leaf count is closest to target."""
    cache = {}

    def cached(lev, coords):
        out = np.empty(len(coords))
        miss = [i for i, c in enumerate(map(tuple, coords.tolist())) if (lev, c) not in cache]
        if miss:
            v = score(lev, coords[miss])
            for i, x in zip(miss, v):
                cache[(lev, tuple(coords[i].tolist()))] = float(x)
        for i, c in enumerate(map(tuple, coords.tolist())):
            out[i] = cache[(lev, c)]
        return out

    lo, hi = -12.0, 6.0  # log10 tau
    best = None
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        leaves = adaptive_leaves(dom, max_level, cached, 10.0 ** mid)
        n = len(leaves)
        if best is None or abs(n - target) < abs(best[1] - target):
            best = (10.0 ** mid, n, leaves)
        if n > target:
            lo = mid
        else:
            hi = mid
        if n == target:
            break
    return best


def block_node_coords(dom: Domain, lev: int, coords: np.ndarray):
    """Physical coordinates (x[n,B], y[n,B], z[n,B]) of the nodes of blocks."""
    h = dom.h(lev)
    loc = np.arange(dom.B)
    out = []
    for d in range(3):
        J = coords[:, d:d + 1].astype(np.int64) * dom.B + loc[None, :]
        out.append(dom.origin[d] + J * h)
    return out


def corner_nested_leaves(dom: Domain, depth: int, corner=(0, 0, 0)) -> np.ndarray:
    """Fig.-1 style layout: refine the block at `corner` repeatedly,
    then 2:1-balance.  Used by the parity tests."""
    t = Tree(dom)
    b = tuple(corner)
    for lev in range(depth):
        t.refine(lev, b)
        b = (2 * b[0], 2 * b[1], 2 * b[2])
    bad = t.balance(lambda l, c: t.touches_unbounded_face(l, c))
    if bad:
        raise ValueError("corner layout cannot be balanced")
    return t.leaves()


def random_leaves(dom: Domain, max_level: int, seed: int, p: float = 0.3) -> np.ndarray:
    """Seeded random 2:1-balanced layout (refine each refinable leaf with prob p)."""
    rng = np.random.default_rng(seed)
    t = Tree(dom)
    for lev in range(max_level):
        for b in sorted(t.nodes.get(lev, ())):
            if t.touches_unbounded_face(lev, b):
                continue
            if rng.random() < p:
                t.refine(lev, b)
    bad = t.balance(lambda l, c: t.touches_unbounded_face(l, c) or l >= max_level)
    if bad:
        raise ValueError("random layout cannot be balanced")
    return t.leaves()
