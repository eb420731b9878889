"""Pins of the oracle's discrete operators against what the paper and mathematics fix.

P1: fig:stencils integer tables, row sums, closed-form
polynomial images, truncation order under refinement; smoother single-node closed
form (P5).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import mg_oracle as MO

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _impulse_response(order, h=1.0):
    X = np.zeros((5, 5, 5))
    X[2, 2, 2] = 1.0
    # L is symmetric, so L applied to a unit impulse gives the stencil weights
    return MO.apply_L(X, h, order)[1:4, 1:4, 1:4]


@pytest.mark.parametrize("order", [2, 4, 6])
def test_lhs_matches_fig_stencils(order):
    g = json.load(open(os.path.join(GOLD, "stencils.json")))[str(order)]
    scale = {2: 1.0, 4: 6.0, 6: 30.0}[order]
    W = _impulse_response(order) * scale
    for off in np.ndindex(3, 3, 3):
        nz = sum(1 for o in off if o != 1)
        cls = ["centre", "face", "edge", "corner"][nz]
        assert W[off] == pytest.approx(g[cls], abs=1e-12), (off, W[off])
    assert abs(W.sum()) < 1e-12          # consistency: row sum zero


def test_rhs4_weights_and_row_sum():
    g = json.load(open(os.path.join(GOLD, "stencils.json")))["rhs4"]
    X = np.zeros((5, 5, 5))
    X[2, 2, 2] = 1.0
    R = MO.apply_R(X, 4)[1:4, 1:4, 1:4]
    assert R[1, 1, 1] == pytest.approx(g["centre"], abs=1e-15)
    for off in [(0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)]:
        assert R[off] == pytest.approx(g["face"], abs=1e-15)
    assert R.sum() == pytest.approx(1.0, abs=1e-15)
    assert np.array_equal(MO.apply_R(X, 2), X)         # M=2: f* = f bitwise


def test_polynomial_closed_forms():
    # Δ_h^4 x^4 = 12 x^2 + 2 h^2 and R_h^4 (12 x^2) = 12 x^2 + 2 h^2,
    # i.e. the 4th-order scheme is exact for u = x^4.
    h = 0.1
    J = np.arange(-3, 4) * h
    x = J[:, None, None] + 0 * J[None, :, None] + 0 * J[None, None, :]
    L = MO.apply_L(x ** 4, h, 4)[3, 3, 3]
    assert L == pytest.approx(12 * 0 ** 2 + 2 * h * h, rel=1e-12)
    xs = x + 0.37
    L = MO.apply_L(xs ** 4, h, 4)[3, 3, 3]
    assert L == pytest.approx(12 * 0.37 ** 2 + 2 * h * h, rel=1e-12)
    R = MO.apply_R(12 * xs ** 2, 4)[3, 3, 3]
    assert R == pytest.approx(12 * 0.37 ** 2 + 2 * h * h, rel=1e-12)
    # M=2 is exact on quadratics
    L2 = MO.apply_L(xs ** 2 + 3 * xs, h, 2)[3, 3, 3]
    assert L2 == pytest.approx(2.0, rel=1e-12)


@pytest.mark.parametrize("order,expected", [(2, 2.0), (4, 4.0), (6, 6.0)])
def test_truncation_order(order, expected):
    # defect Δ_h^M u - R_h^M(∇²u) for a smooth periodic u decays as h^M
    errs = []
    for n in (32, 64):
        h = 1.0 / n
        J = (np.arange(-MO.E, n + MO.E)) * h
        X, Y, Z = np.meshgrid(J, J, J, indexing="ij")
        u = np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y + 0.3) * np.sin(2 * np.pi * Z + 1.0)
        lap = -12 * np.pi ** 2 * u
        d = MO.apply_L(u, h, order) - MO.apply_R(lap, order)
        sl = (slice(MO.E, MO.E + n),) * 3
        errs.append(np.abs(d[sl]).max())
    rate = math.log2(errs[0] / errs[1])
    assert abs(rate - expected) < 0.15, (errs, rate)


def test_jacobi_single_node_closed_form():
    # u = 0, f = δ: one damped-Jacobi sweep of Oracle.smooth leaves ω f / d at the node
    # and nothing elsewhere; d typed from fig:stencils.
    # (Two-sweep and red-black impulse pins: tests/test_oracle_smoother_pins.py.)
    from workloads import layouts as Lay
    for order, centre in ((2, -6.0), (4, -24.0 / 6.0), (6, -128.0 / 30.0)):
        h = 1 / 32
        d = dict(origin=(0.0, 0.0, 0.0), h0=h, base_blocks=(2, 2, 2), B=16, bc=(0, 0, 0), order=order,
                 smoother=MO.JACOBI, omega=2 / 3, eta1=1, eta2=1, coarse_n=0)
        o = MO.Oracle(d, Lay.uniform_leaves(Lay.Domain((0.0, 0.0, 0.0), h, (2, 2, 2), 16, (0, 0, 0)), 0))
        L = o.levels[0]
        L.u = np.zeros(tuple(L.N))
        L.f = np.zeros(tuple(L.N))
        L.f[3, 4, 5] = 3.0
        o.smooth(0)
        assert L.u[3, 4, 5] == pytest.approx((2 / 3) * 3.0 * h * h / centre, rel=1e-15)
        assert np.count_nonzero(L.u) == 1
