"""ORACLE (test infrastructure only) — the same operators as oracle/mg_oracle.py,
evaluated at ONE node from a value accessor, for sampled checks at full size.

Only tests/, __graft_entry__.smoke() and bench.py may import this module; the CUDA
path never does.  `get(J)` returns the value of a level field at the level-global
node J = (Jx, Jy, Jz) (the caller resolves blocks, periodic wrap and availability).

* Δ_h^M (E8 for M=2; Mehrstellen E12 for M=4, E13 for M=6, fig:stencils P:272-328):
  M=2: (Σ_faces u - 6u)/h²;  M=4: (2 Σ_faces u + Σ_edges u - 24 u)/(6h²);
  M=6: (14 Σ_faces u + 3 Σ_edges u + Σ_corners u - 128 u)/(30h²).
* R_h^M f (right side of E12/E13): M=2: f;  M=4: f + (1/12) Σ_d δ²_d f;
  M=6: f + (1/12) Σ_d δ²_d f + (1/90) Σ_{d<e} δ²_d δ²_e f - (1/240) Σ_d δ⁴_d f
  (reading Z24 of the garbled P:359).
* damped Jacobi / red-black node update (readings Z9/Z10):
  u_new = u + ω (f* - Δ_h^M u)/d, d = centre coefficient of Δ_h^M (-6/h², -4/h²,
  -128/(30h²)); red = even level-global parity, updated from old values; black from
  red-new face (and, M=6, corner) neighbours and old edge/centre values.
"""
from __future__ import annotations

FACES = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
EDGES = [(a, b, 0) for a in (-1, 1) for b in (-1, 1)] + [(a, 0, c) for a in (-1, 1) for c in (-1, 1)] + \
        [(0, b, c) for b in (-1, 1) for c in (-1, 1)]
CORNERS = [(a, b, c) for a in (-1, 1) for b in (-1, 1) for c in (-1, 1)]


def _add(J, o):
    return (J[0] + o[0], J[1] + o[1], J[2] + o[2])


def stencil_nodes(order):
    """Offsets Δ_h^M reads (centre first)."""
    return [(0, 0, 0)] + FACES + (EDGES if order >= 4 else []) + (CORNERS if order == 6 else [])


def lap_at(get, J, h, order):
    """Δ_h^M u at node J (fig:stencils integer tables × 1/h², 1/(6h²), 1/(30h²))."""
    c = get(J)
    F = sum(get(_add(J, o)) for o in FACES)
    if order == 2:
        return (F - 6.0 * c) / (h * h)
    E = sum(get(_add(J, o)) for o in EDGES)
    if order == 4:
        return (2.0 * F + E - 24.0 * c) / (6.0 * h * h)
    K = sum(get(_add(J, o)) for o in CORNERS)
    return (14.0 * F + 3.0 * E + K - 128.0 * c) / (30.0 * h * h)


def diag(h, order):
    return {2: -6.0, 4: -4.0, 6: -128.0 / 30.0}[order] / (h * h)


def rhs_at(getf, J, order):
    """R_h^M f at node J (f* of P:346)."""
    f = getf(J)
    if order == 2:
        return f

    def unit(d, k):
        o = [0, 0, 0]
        o[d] = k
        return tuple(o)

    def d2(d, K):  # δ²_d f at node K
        return getf(_add(K, unit(d, -1))) - 2.0 * getf(K) + getf(_add(K, unit(d, 1)))

    s = sum(d2(d, J) for d in range(3))
    if order == 4:
        return f + s / 12.0
    # M = 6 (E13, Z24): mixed δ²_d δ²_e and fourth differences δ⁴_d
    mixed = 0.0
    for d in range(3):
        for e in range(d + 1, 3):
            mixed += d2(d, _add(J, unit(e, -1))) - 2.0 * d2(d, J) + d2(d, _add(J, unit(e, 1)))
    quart = 0.0
    for d in range(3):
        quart += (getf(_add(J, unit(d, -2))) - 4.0 * getf(_add(J, unit(d, -1))) + 6.0 * f
                  - 4.0 * getf(_add(J, unit(d, 1))) + getf(_add(J, unit(d, 2))))
    return f + s / 12.0 + mixed / 90.0 - quart / 240.0


def is_red(J):
    return (J[0] + J[1] + J[2]) % 2 == 0


def rb_red_new(get_old, fstar, J, h, order, omega):
    """New value of a red node after the red half-sweep (all operands old)."""
    return get_old(J) + omega * (fstar(J) - lap_at(get_old, J, h, order)) / diag(h, order)


def rb_sweep_at(get_old, fstar, J, h, order, omega):
    """Value of node J after one full red-black sweep (no frozen ghosts involved:
    the caller only samples nodes whose 2-node neighbourhood is inside the level)."""
    if is_red(J):
        return rb_red_new(get_old, fstar, J, h, order, omega)

    def get_mid(K):
        return rb_red_new(get_old, fstar, K, h, order, omega) if is_red(K) else get_old(K)

    return get_old(J) + omega * (fstar(J) - lap_at(get_mid, J, h, order)) / diag(h, order)


def residual_at(get_u, fstar, J, h, order):
    """r = f* - Δ_h^M u at node J (Alg. 1)."""
    return fstar(J) - lap_at(get_u, J, h, order)
