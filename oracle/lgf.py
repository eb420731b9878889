"""ORACLE (test infrastructure only) — lattice Green's functions and coarse kernels.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The CUDA path never does.

PAPER.md §2.2 (E5): the coarse direct solve convolves with the lattice
Green's function G[n] of the *same* difference operator, ℒG[n] = δ[n]; §3.3
 requires that compatibility.  Construction (reading R-LGF):
solve ℒG = δ exactly in the box |n|_inf <= R with the continuum free-space
Green's function imposed on the box shell (3D: -1/(4π|n|); 2D: (1/2π) ln|n|,
then shifted so G[0,0] = 0, the 2D convention), using the sine transform
(DST-I), which diagonalises every operator that is a polynomial in the 1D
second differences δ² with zero Dirichlet data.

2-unbounded kernel: E14 (Spietz): zero periodic wavenumber -> 2D LGF,
elsewhere 1/σ_ℒ(k) of the 3D operator.  Here the periodic axis is x (reading Z22).
"""
from __future__ import annotations

import functools
import math

import numpy as np
from scipy.fft import dstn


def smooth7(n: int) -> int:
    """Smallest integer >= n whose prime factors are all <= 7."""
    m = max(n, 1)
    while True:
        r = m
        for p in (2, 3, 5, 7):
            while r % p == 0:
                r //= p
        if r == 1:
            return m
        m += 1


def pad_size(N: int, ge: int) -> int:
    """Padded transform length along an unbounded axis: smallest 7-smooth integer
    >= 2N + 2*ge - 1, so that outputs on [-ge, N+ge) see no aliasing (reading Z21)."""
    return smooth7(2 * N + 2 * ge - 1)


def box_radius(P: int) -> int:
    """Half-width of the box in which the LGF is solved (reading R-LGF)."""
    return P // 2 + 8


def lattice_symbol_poly(lams, order):
    """Symbol of Δ^M (times h^2) as a polynomial of the δ² eigenvalues, E8/E12/E13:
    M=2: Σλ; M=4: Σλ + (1/6)Σ_{d<e} λ_d λ_e; M=6: M=4 + (1/30) λ_x λ_y λ_z."""
    s = sum(lams)
    if order == 2:
        return s
    pair = 0.0
    n = len(lams)
    for a in range(n):
        for b in range(a + 1, n):
            pair = pair + lams[a] * lams[b]
    s = s + pair / 6.0
    if order == 6 and n == 3:
        s = s + lams[0] * lams[1] * lams[2] / 30.0
    return s


def _apply_op(G, order):
    """ℒG at the interior of an array (dimension 2 or 3), literal E8/E12 form."""
    def d2(A, ax):
        out = np.full_like(A, np.nan)
        sl = [slice(None)] * A.ndim
        c = [slice(None)] * A.ndim
        m = [slice(None)] * A.ndim
        p = [slice(None)] * A.ndim
        c[ax] = slice(1, -1)
        m[ax] = slice(0, -2)
        p[ax] = slice(2, None)
        out[tuple(c)] = A[tuple(m)] - 2 * A[tuple(c)] + A[tuple(p)]
        return out
    nd = G.ndim
    D = [d2(G, a) for a in range(nd)]
    res = sum(D)
    if order >= 4:
        for a in range(nd):
            for b in range(a + 1, nd):
                res = res + d2(D[a], b) / 6.0
    if order == 6 and nd == 3:
        res = res + d2(d2(D[0], 1), 2) / 30.0
    return res


def box_lgf(dim: int, order: int, R: int) -> np.ndarray:
    """G on the box [-R, R]^dim (index n+R), solving ℒG = δ exactly inside.  (A read-only
    table, memoised per (dim, order, R): the tests build many oracles on one domain.)"""
    return _box_lgf(dim, order, R)


@functools.lru_cache(maxsize=8)
def _box_lgf(dim: int, order: int, R: int) -> np.ndarray:
    n = 2 * R + 1
    idx = np.arange(-R, R + 1, dtype=np.float64)
    grids = np.meshgrid(*([idx] * dim), indexing="ij")
    r = np.sqrt(sum(g * g for g in grids))
    shell = np.zeros((n,) * dim, dtype=bool)
    for a in range(dim):
        sl = [slice(None)] * dim
        sl[a] = 0
        shell[tuple(sl)] = True
        sl[a] = -1
        shell[tuple(sl)] = True
    rr = np.where(r > 0, r, 1.0)
    if dim == 3:
        cont = -1.0 / (4 * np.pi * rr)
    else:
        cont = np.log(rr) / (2 * np.pi)
    Gb = np.where(shell, cont, 0.0)
    rhs = -_apply_op(Gb, order)          # move the shell values to the right side
    inner = (slice(1, -1),) * dim
    b = rhs[inner]
    b[(R - 1,) * dim] += 1.0             # δ at the origin
    m = n - 2
    j = np.arange(1, m + 1)
    lam1 = 2 * np.cos(np.pi * j / (m + 1)) - 2
    lams = np.meshgrid(*([lam1] * dim), indexing="ij")
    Lam = lattice_symbol_poly(lams, order)
    bh = dstn(b, type=1, norm="ortho")
    Gi = dstn(bh / Lam, type=1, norm="ortho")
    G = Gb.copy()
    G[inner] = Gi
    if dim == 2:
        G = G - G[R, R]
    G.setflags(write=False)
    return G


def wrapped_table(G: np.ndarray, R: int, shape) -> np.ndarray:
    """Sample G (box, index n+R) on a periodic torus of `shape`: T[i] = G[n(i)],
    n(i) = i for i <= P/2 else i - P (per axis)."""
    idxs = []
    for P in shape:
        i = np.arange(P)
        n = np.where(i <= P // 2, i, i - P)
        if np.any(np.abs(n) > R):
            raise ValueError("LGF box too small for the padded torus")
        idxs.append(n + R)
    return G[np.ix_(*idxs)]
