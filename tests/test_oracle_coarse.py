"""Pins of the oracle's coarse direct solve and lattice Green's functions (P6)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import gamma

from oracle import lgf as LGF
from oracle import mg_oracle as MO
from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_watson_constant_closed_form():
    g = json.load(open(os.path.join(GOLD, "lgf.json")))
    # simple-cubic Watson integral (1/π³)∫∫∫ dθ/(3 - Σcosθ) in Gamma closed form
    W = math.sqrt(6) / (96 * math.pi ** 3) * gamma(1 / 24) * gamma(5 / 24) * gamma(7 / 24) * gamma(11 / 24)
    assert -W / 2 == pytest.approx(g["watson_7pt_G0"]["value"], abs=1e-13)
    G = LGF.box_lgf(3, 2, 48)
    # box construction converges to the infinite-lattice value as R^-3 (shell error)
    assert G[48, 48, 48] == pytest.approx(-W / 2, abs=2e-7)


def test_square_lattice_lgf():
    g = json.load(open(os.path.join(GOLD, "lgf.json")))
    G = LGF.box_lgf(2, 2, 96)
    assert G[97, 96] == pytest.approx(g["square_5pt_G10"]["value"], abs=1e-13)
    assert G[97, 97] == pytest.approx(g["square_5pt_G11"]["value"], abs=1e-9)


@pytest.mark.parametrize("dim,order", [(2, 2), (2, 4), (3, 2), (3, 4)])
def test_box_lgf_is_exact_inverse(dim, order):
    R = 20
    G = LGF.box_lgf(dim, order, R)
    LG = LGF._apply_op(G, order)
    inner = (slice(1, -1),) * dim
    d = np.zeros_like(G)
    d[(R,) * dim] = 1.0
    assert np.abs(LG[inner] - d[inner]).max() < 1e-13
    # symmetry under reflections and axis permutations
    assert np.abs(G - G[::-1]).max() < 1e-14
    assert np.abs(G - np.swapaxes(G, 0, 1)).max() < 1e-14


def _single_level(bc, n=32, order=4):
    d = dict(origin=(0.0, 0.0, 0.0), h0=1 / n, base_blocks=(n // 16,) * 3, B=16, bc=bc, order=order,
             smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
    return MO.Oracle(d, Lay.uniform_leaves(C.domain(d)))


ALL_BC = [(0, 0, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0), (1, 1, 1)]


@pytest.mark.parametrize("bc", ALL_BC)
@pytest.mark.parametrize("order", [2, 4, 6])
def test_direct_solve_discrete_exactness(bc, order):
    """Δ_h^M (S_0 f) = f on every domain node and on the exterior band (GE layers), for
    every mix of periodic / unbounded axes: the coarse kernel is the exact inverse of
    the multigrid operator on the zero-padded lattice."""
    o = _single_level(bc, order=order)
    c = o.levels[0]
    rng = np.random.default_rng(7)
    f = rng.normal(size=tuple(c.N))
    if bc == (0, 0, 0):
        f -= f.mean()
    c.f = f
    o.coarse_solve()
    X = o.lookup(0, o.uvals())
    Lu = MO.apply_L(X, c.h, order)
    Fe = o._pad(f, fill=0.0)          # periodic images / zero beyond unbounded faces
    lo, hi = MO.E - (MO.GE - 1), MO.E + 32 + (MO.GE - 1)
    sl = tuple(slice(MO.E, MO.E + 32) if bc[a] == 0 else slice(lo, hi) for a in range(3))
    err = np.abs(Lu[sl] - Fe[sl]).max() / np.abs(f).max()
    assert err < 1e-12, err
    if bc == (0, 0, 0):
        assert abs(c.u.mean()) < 1e-14 * np.abs(c.u).max()     # zero average


def test_one_dimensional_lgf_closed_form():
    """The 1D lattice Green's function used for one unbounded axis: δ²(|n|/2) = δ[n]."""
    n = np.arange(-20, 21)
    G = np.abs(n) / 2.0
    d2 = G[:-2] - 2 * G[1:-1] + G[2:]
    assert np.array_equal(d2, (n[1:-1] == 0).astype(float))


@pytest.mark.parametrize("bc", [(0, 0, 1), (1, 0, 1)])
def test_product_manufactured_mixed_fourth_order(bc):
    """Manufactured products in the spirit of E25-E28 for other periodic /
    unbounded mixes: u = Π_d g_d(x_d) with g = u_per on periodic axes and u_unb (compact,
    so the free-space solution) on unbounded ones; 4th-order convergence of S_0."""
    errs = []
    for n in (32, 64):
        d = dict(origin=(0.0, 0.0, 0.0), h0=1 / n, base_blocks=(n // 16,) * 3, B=16, bc=bc,
                 order=4, smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
        dom = C.domain(d)
        lv = Lay.uniform_leaves(dom)
        g = [S.u_per if b == 0 else S.u_unb for b in bc]
        d2g = [S.d2u_per if b == 0 else S.d2u_unb for b in bc]

        def fn(x, y, z):
            X = (x, y, z)
            tot = 0.0
            for k in range(3):
                term = 1.0
                for a in range(3):
                    term = term * (d2g[a](X[a]) if a == k else g[a](X[a]))
                tot = tot + term
            return tot

        f = S.sample_on_leaves(dom, lv, fn)
        ue = S.sample_on_leaves(dom, lv, lambda x, y, z: g[0](x) * g[1](y) * g[2](z))
        o = MO.Oracle(d, lv)
        o.set_rhs(f)
        o.vcycle(1)
        errs.append(np.abs(o.get_solution() - ue).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 3.6, (errs, rate)


def test_free_space_gaussian_fourth_order():
    """UUU direct solve of a Gaussian charge vs -Q erf(r/(sqrt2 σ))/(4πr): E∞ ∝ h^4."""
    errs = []
    for n in (32, 64):
        d = dict(origin=(-1.0, -1.0, -1.0), h0=2 / n, base_blocks=(n // 16,) * 3, B=16, bc=(1, 1, 1),
                 order=4, smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
        dom = C.domain(d)
        lv = Lay.uniform_leaves(dom)
        o = MO.Oracle(d, lv)
        sig = 0.2
        f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=sig))
        ue = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_potential(x, y, z, sigma=sig))
        o.set_rhs(f)
        o.vcycle(1)          # single level: the V-cycle is the direct solve
        errs.append(np.abs(o.get_solution() - ue).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 3.6, (errs, rate)


def test_product_manufactured_puu_fourth_order():
    """E25-E28: u = u_per(x) u_unb(y) u_unb(z) on the unit cube, x periodic."""
    errs = []
    for n in (32, 64):
        d = dict(origin=(0.0, 0.0, 0.0), h0=1 / n, base_blocks=(n // 16,) * 3, B=16, bc=(0, 1, 1),
                 order=4, smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
        dom = C.domain(d)
        lv = Lay.uniform_leaves(dom)

        def fn(x, y, z):
            return (S.d2u_per(x) * S.u_unb(y) * S.u_unb(z) + S.u_per(x) * S.d2u_unb(y) * S.u_unb(z)
                    + S.u_per(x) * S.u_unb(y) * S.d2u_unb(z))

        f = S.sample_on_leaves(dom, lv, fn)
        ue = S.sample_on_leaves(dom, lv, lambda x, y, z: S.u_per(x) * S.u_unb(y) * S.u_unb(z))
        o = MO.Oracle(d, lv)
        o.set_rhs(f)
        o.vcycle(1)
        errs.append(np.abs(o.get_solution() - ue).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 3.6, (errs, rate)


def test_manufactured_second_derivatives():
    # the harness' analytic f is the Laplacian of u_ref (finite-difference check)
    x = np.linspace(0.05, 0.95, 37)
    e = 1e-4
    for u, d2u in ((S.u_per, S.d2u_per), (S.u_unb, S.d2u_unb)):
        fd = (u(x + e) - 2 * u(x) + u(x - e)) / e ** 2
        assert np.abs(fd - d2u(x)).max() < 1e-5 * max(1.0, np.abs(d2u(x)).max())


def test_pad_size_rule():
    assert LGF.pad_size(128, 5) == 270
    assert LGF.pad_size(32, 5) == 75
    assert LGF.smooth7(73) == 75


def test_sixth_order_periodic_product_convergence():
    """M = 6 (E13 with the δ²_yδ²_z reading Z24): the compact scheme with
    its radius-2 right-hand side converges at 6th order on a smooth periodic product."""
    errs = []
    for n in (16, 32):
        d = dict(origin=(0.0, 0.0, 0.0), h0=1 / n, base_blocks=(n // 16,) * 3, B=16, bc=(0, 0, 0),
                 order=6, smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
        dom = C.domain(d)
        lv = Lay.uniform_leaves(dom)

        def fn(x, y, z):
            return (S.d2u_per(x) * S.u_per(y) * S.u_per(z) + S.u_per(x) * S.d2u_per(y) * S.u_per(z)
                    + S.u_per(x) * S.u_per(y) * S.d2u_per(z))

        f = S.sample_on_leaves(dom, lv, fn)
        f = f - f.mean()
        ue = S.sample_on_leaves(dom, lv, lambda x, y, z: S.u_per(x) * S.u_per(y) * S.u_per(z))
        o = MO.Oracle(d, lv)
        o.set_rhs(f)
        o.vcycle(1)
        u = o.get_solution()
        errs.append(np.abs((u - u.mean()) - (ue - ue.mean())).max())
    rate = math.log2(errs[0] / errs[1])
    assert rate > 5.4, (errs, rate)
