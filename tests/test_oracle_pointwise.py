"""Pins of oracle/pointwise.py (single-node operators used by the full-size sampled
GPU checks) against closed forms, polynomial exactness of the
compact schemes (E12/E13) and the dense oracle."""
import numpy as np
import pytest

from oracle import mg_oracle as MO
from oracle import pointwise as PW


def _poly_get(fn, h):
    return lambda J: fn(J[0] * h, J[1] * h, J[2] * h)


@pytest.mark.parametrize("h", [0.1, 0.03])
def test_lap4_x4_closed_form(h):
    # Δ_h^4 x^4 = 12 x^2 + 2 h^2 (A1; the 1D second difference of x^4)
    for J in [(3, -2, 5), (0, 0, 0), (-7, 1, 2)]:
        x = J[0] * h
        v = PW.lap_at(_poly_get(lambda x, y, z: x ** 4, h), J, h, 4)
        assert v == pytest.approx(12 * x * x + 2 * h * h, rel=1e-12, abs=1e-12)


def test_mehrstellen_exact_on_x2y2():
    # Δ_h^4 (x²y²) = R_h^4 (2x² + 2y²) = 2x² + 2y² + (2/3)h²: the compact scheme is exact here
    h = 0.05
    u = _poly_get(lambda x, y, z: x * x * y * y, h)
    f = _poly_get(lambda x, y, z: 2 * x * x + 2 * y * y, h)
    for J in [(1, 2, 3), (-4, 5, 0)]:
        x, y = J[0] * h, J[1] * h
        lhs = PW.lap_at(u, J, h, 4)
        rhs = PW.rhs_at(f, J, 4)
        assert lhs == pytest.approx(rhs, rel=1e-12)
        assert lhs == pytest.approx(2 * x * x + 2 * y * y + 2 * h * h / 3, rel=1e-12)


def test_lap2_is_seven_point():
    h = 0.1
    u = _poly_get(lambda x, y, z: x ** 2 + 3 * y ** 2 - z ** 2, h)
    assert PW.lap_at(u, (2, -1, 4), h, 2) == pytest.approx(2 + 6 - 2, rel=1e-12)


def test_jacobi_single_node_closed_form():
    # u = 0 everywhere except f*: one update gives ω f*/d (P5)
    h, w = 0.125, 2 / 3
    v = PW.rb_red_new(lambda J: 0.0, lambda J: 3.0, (0, 0, 0), h, 4, w)
    assert v == pytest.approx(w * 3.0 / (-4.0 / h ** 2), rel=1e-15)


@pytest.mark.parametrize("h", [0.1, 0.03])
def test_lap6_reduces_to_second_difference(h):
    # a function of x alone: the 27-point M=6 stencil collapses to δ²_x/h² (weights
    # 14+12+4 = 30 on x±h, -128+56+12 = -60 on x): Δ_h^6 x^4 = 12 x^2 + 2 h^2
    for J in [(3, -2, 5), (0, 0, 0), (-7, 1, 2)]:
        x = J[0] * h
        v = PW.lap_at(_poly_get(lambda x, y, z: x ** 4, h), J, h, 6)
        assert v == pytest.approx(12 * x * x + 2 * h * h, rel=1e-11, abs=1e-11)


@pytest.mark.parametrize("u,f", [
    (lambda x, y, z: x ** 4 * y ** 2, lambda x, y, z: 12 * x * x * y * y + 2 * x ** 4),
    (lambda x, y, z: (x * y * z) ** 2, lambda x, y, z: 2 * (y * y * z * z + x * x * z * z + x * x * y * y)),
    (lambda x, y, z: x ** 6 - 3 * y ** 3 * z, lambda x, y, z: 30 * x ** 4 - 18 * y * z),
])
def test_mehrstellen6_exact_on_degree6(u, f):
    # the sixth-order compact scheme (E13) reproduces polynomial solutions up to degree
    # 6: Δ_h^6 u = R_h^6 Δu exactly (a dropped or mis-weighted term of either side, or a
    # wrong sign of the δ⁴ term, breaks this)
    h = 0.07
    for J in [(1, 2, 3), (-4, 5, 0), (2, -3, -1)]:
        lhs = PW.lap_at(_poly_get(u, h), J, h, 6)
        rhs = PW.rhs_at(_poly_get(f, h), J, 6)
        assert lhs == pytest.approx(rhs, rel=1e-11, abs=1e-11)


@pytest.mark.parametrize("order", [4, 6])
def test_rb_sweep_matches_dense_oracle(order):
    """One RB sweep on a periodic 32^3 level: pointwise (node by node) == dense."""
    d = dict(origin=(0, 0, 0), h0=1 / 32, base_blocks=(2, 2, 2), B=16, bc=(0, 0, 0), order=order, smoother=1,
             omega=1.0, eta1=2, eta2=2, coarse_n=0)
    leaves = np.array([(0, i, j, k) for k in range(2) for j in range(2) for i in range(2)])
    o = MO.Oracle(d, leaves)
    rng = np.random.default_rng(7)
    L = o.levels[0]
    L.u = rng.standard_normal(L.u.shape)
    L.f = rng.standard_normal(L.f.shape)
    u0, f0 = L.u.copy(), L.f.copy()
    o.smooth(0)
    N = 32
    get = lambda J: u0[J[0] % N, J[1] % N, J[2] % N]  # noqa: E731
    fs = lambda J: f0[J[0] % N, J[1] % N, J[2] % N]  # noqa: E731
    for J in [(0, 0, 0), (5, 7, 9), (31, 0, 16), (15, 16, 17), (1, 2, 4)]:
        v = PW.rb_sweep_at(get, fs, J, L.h, order, 1.0)
        assert v == pytest.approx(L.u[J], rel=1e-12, abs=1e-12 * np.abs(L.u).max())
