"""Pins of Oracle.smooth and of the composite residual norm against closed forms.

These call the oracle's own entry points (Oracle.smooth, Oracle.residual_norm) on
impulse inputs whose one-sweep results follow by hand from the paper's stencil
tables (fig:stencils) and the smoother definitions (damped Jacobi and
red-black Gauss-Seidel; readings Z9/Z10: red = even (Jx+Jy+Jz) first, each
colour from a snapshot).  Every expected value below is typed from the paper's
integer stencil weights, never computed by the oracle:

  centre d:     M=2  -6/h^2      M=4  -24/(6h^2)     M=6  -128/(30h^2)
  face c_f:     M=2   1/h^2      M=4    2/(6h^2)     M=6    14/(30h^2)
  edge c_e:     M=2   0          M=4    1/(6h^2)     M=6     3/(30h^2)
  corner c_k:   M=2   0          M=4    0            M=6     1/(30h^2)

A mistake such as black-before-red, a black half-sweep that reads the old red
values, a dropped ω or a wrong diagonal fails one of these.
"""
import numpy as np
import pytest

from oracle import mg_oracle as MO
from workloads import layouts as Lay

H = 1.0 / 32
COEF = {  # (centre, face, edge, corner) x h^2, from fig:stencils
    2: (-6.0, 1.0, 0.0, 0.0),
    4: (-24.0 / 6.0, 2.0 / 6.0, 1.0 / 6.0, 0.0),
    6: (-128.0 / 30.0, 14.0 / 30.0, 3.0 / 30.0, 1.0 / 30.0),
}


def _uniform_oracle(order, smoother, omega):
    d = dict(origin=(0.0, 0.0, 0.0), h0=H, base_blocks=(2, 2, 2), B=16, bc=(0, 0, 0), order=order,
             smoother=smoother, omega=omega, eta1=1, eta2=1, coarse_n=0)
    dom = Lay.Domain((0.0, 0.0, 0.0), H, (2, 2, 2), 16, (0, 0, 0))
    o = MO.Oracle(d, Lay.uniform_leaves(dom, 0))
    L = o.levels[0]
    L.u = np.zeros(tuple(L.N))
    L.f = np.zeros(tuple(L.N))
    return o, L


def _offsets():
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                yield (dx, dy, dz), abs(dx) + abs(dy) + abs(dz)


@pytest.mark.parametrize("order", [2, 4, 6])
@pytest.mark.parametrize("omega", [1.0, 0.8])
def test_rb_sweep_red_impulse(order, omega):
    """f* = δ at a red node R, u = 0: after one RB sweep (red first, snapshot per colour)
    u(R) = ω f/d; every black neighbour b gets -ω c_{b} u(R)/d (it reads the NEW red
    value); every other node — every other red node included — stays 0."""
    o, L = _uniform_oracle(order, MO.RBGS, omega)
    R = (5, 7, 8)                        # 5+7+8 even: red
    fval = 3.0
    L.f[R] = fval
    o.smooth(0)
    cd, cf, ce, ck = COEF[order]
    d = cd / H ** 2
    uR = omega * fval / d
    expect = np.zeros(tuple(L.N))
    expect[R] = uR
    for off, n in _offsets():
        if n in (1, 3):                  # odd offsets are black
            c = (cf if n == 1 else ck) / H ** 2
            expect[tuple(R[a] + off[a] for a in range(3))] = -omega * c * uR / d
    assert np.allclose(L.u, expect, rtol=1e-14, atol=1e-14 * abs(uR))
    assert L.u[R] == pytest.approx(uR, rel=1e-15)
    # the edge neighbours (even offsets) are red: untouched by the sweep
    assert L.u[R[0] + 1, R[1] + 1, R[2]] == 0.0
    red = (np.indices(tuple(L.N)).sum(axis=0) % 2) == 0
    red[R] = False
    assert not np.any(L.u[red])


@pytest.mark.parametrize("order", [2, 4, 6])
def test_rb_sweep_black_impulse(order):
    """f* = δ at a black node: the red half-sweep sees only zeros, the black half-sweep
    updates every black node from the snapshot, so only that node changes, to ω f/d.
    (Black-first ordering would also move its red face neighbours.)"""
    omega = 0.9
    o, L = _uniform_oracle(order, MO.RBGS, omega)
    Bn = (4, 7, 8)                       # odd: black
    L.f[Bn] = -2.0
    o.smooth(0)
    d = COEF[order][0] / H ** 2
    expect = np.zeros(tuple(L.N))
    expect[Bn] = omega * (-2.0) / d
    assert np.array_equal(L.u != 0, expect != 0)
    assert L.u[Bn] == pytest.approx(expect[Bn], rel=1e-15)


@pytest.mark.parametrize("order", [2, 4, 6])
def test_jacobi_impulse_two_sweeps(order):
    """Damped Jacobi (north-star ω = 2/3): every node from the old values.  One
    sweep with f = δ: only the impulse node moves, to ω f/d.  A second sweep: that node
    becomes u1 + ω(f - d u1)/d, each neighbour at offset class k gets -ω c_k u1/d."""
    omega = 2.0 / 3.0
    o, L = _uniform_oracle(order, MO.JACOBI, omega)
    P = (9, 3, 12)
    fval = 1.5
    L.f[P] = fval
    o.smooth(0)
    d = COEF[order][0] / H ** 2
    u1 = omega * fval / d
    assert L.u[P] == pytest.approx(u1, rel=1e-15)
    assert np.count_nonzero(L.u) == 1
    o.smooth(0)
    expect = np.zeros(tuple(L.N))
    expect[P] = u1 + omega * (fval - d * u1) / d
    for off, n in _offsets():
        if n:
            c = COEF[order][n] / H ** 2
            expect[tuple(P[a] + off[a] for a in range(3))] = -omega * c * u1 / d
    assert np.allclose(L.u, expect, rtol=1e-14, atol=1e-14 * abs(u1))


def test_rb_periodic_wrap():
    """The colour is the parity of the level-global index; on a periodic axis of even
    length the wrap keeps it, so an impulse on the face J = 0 reaches J = N-1."""
    o, L = _uniform_oracle(4, MO.RBGS, 1.0)
    R = (0, 4, 6)
    L.f[R] = 1.0
    o.smooth(0)
    d = COEF[4][0] / H ** 2
    uR = 1.0 / d
    assert L.u[31, 4, 6] == pytest.approx(-COEF[4][1] / H ** 2 * uR / d, rel=1e-14)


# ------------------------------------------------------------- composite residual (P12)
def _two_level_periodic():
    dom = Lay.Domain((0.0, 0.0, 0.0), 1 / 32, (2, 2, 2), 16, (0, 0, 0))
    lv = Lay.corner_nested_leaves(dom, 1)
    d = dict(origin=(0, 0, 0), h0=1 / 32, base_blocks=(2, 2, 2), B=16, bc=(0, 0, 0), order=4, smoother=1,
             omega=1.0, eta1=2, eta2=2, coarse_n=0)
    o = MO.Oracle(d, lv)
    o.set_rhs(np.zeros((len(lv), 16, 16, 16)))
    return o


def test_composite_residual_leaf_only():
    """a9 / P:170: the composite residual is max |f* - Δu| over LEAF nodes of all levels.
    With f = 0 and u = 0 it is 0.  A perturbation δ of one fine leaf node gives
    |d_1| δ (the largest stencil weight, at that node; d_1 = 4/h_1^2); of a coarse leaf
    node far from the jump |d_0| δ; of a covered coarse node (stored value never read:
    lookups take the injected fine value) nothing."""
    o = _two_level_periodic()
    assert o.fstar_norm == 0.0
    assert o.residual_norm() == (0.0, 0.0)
    C, F = o.levels
    h0, h1 = C.h, F.h
    # covered coarse node deep inside the refined octant: no effect
    assert C.cov[4, 4, 4] and not C.leaf[4, 4, 4]
    C.u[4, 4, 4] = 7.0
    assert o.residual_norm()[0] == 0.0
    C.u[4, 4, 4] = 0.0
    # a fine leaf node
    delta = 1e-3
    assert F.leaf[10, 11, 12]
    F.u[10, 11, 12] = delta
    assert o.residual_norm()[0] == pytest.approx(4.0 / h1 ** 2 * delta, rel=1e-14)
    F.u[10, 11, 12] = 0.0
    # a coarse leaf node 8 nodes from the refined region
    assert C.leaf[24, 24, 24]
    C.u[24, 24, 24] = delta
    assert o.residual_norm()[0] == pytest.approx(4.0 / h0 ** 2 * delta, rel=1e-14)
