"""Pins of the oracle's V-cycle (Alg. 1) against closed forms and invariants
(P7-P9, P11 of SURVEY §8(c))."""
import math

import numpy as np
import pytest

from oracle import mg_oracle as MO
from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S


def test_cfg1_closed_form():
    """Config 1: f = sin sin sin on the periodic 32^3 lattice is a lattice eigenmode:
    u_h = f / σ2, σ2 = -12 sin²(π/32)·32² (A6)."""
    cfg = C.cfg1()
    dom, lv, f = C.build(cfg)
    s2 = -12 * math.sin(math.pi / 32) ** 2 * 32 ** 2
    assert s2 == pytest.approx(-118.0552372026, abs=1e-9)
    uh = f / s2
    assert np.abs(uh).max() == pytest.approx(8.470611077459e-3, abs=1e-14)
    assert abs(np.abs(uh).max() / (1 / (12 * math.pi ** 2)) - 1 - 3.219e-3) < 1e-5
    o = MO.Oracle(cfg, lv)
    o.set_rhs(f)
    hist = []
    for _ in range(cfg["cycles"]):
        o.vcycle(1)
        hist.append(o.residual_norm()[1])
    err = np.abs(o.get_solution() - uh).max()
    assert err < 1e-7 * np.abs(uh).max() * 1e2          # ≪ discretisation error 3e-3
    rates = np.array(hist[1:]) / np.array(hist[:-1])
    assert np.all(rates < 0.3)


def test_cfg2_reduced_closed_form_and_fixed_point():
    """Config 2 recipe at 64^3: the exact discrete solution is per mode
    a (ρ4/σ4) cos(2πk·x+φ), ρ4 = 1 + Σŝ/12 (A6)."""
    cfg = C.cfg2(64)
    dom, lv, f = C.build(cfg)
    k, a, phi = S.fourier_modes(2)
    N = 64
    J = np.arange(N) / N
    X, Y, Z = np.meshgrid(J, J, J, indexing="ij")
    uh = np.zeros_like(X)
    h = 1 / N
    for kk, aa, pp in zip(k, a, phi):
        sh = [2 * np.cos(2 * np.pi * kd / N) - 2 for kd in kk]
        s4 = (sum(sh) + (sh[0] * sh[1] + sh[1] * sh[2] + sh[2] * sh[0]) / 6) / h ** 2
        rho = 1 + sum(sh) / 12
        uh += aa * rho / s4 * np.cos(2 * np.pi * (kk[0] * X + kk[1] * Y + kk[2] * Z) + pp)
    uh_b = S.dense_to_blocks(dom, lv, uh)
    o = MO.Oracle(cfg, lv)
    o.set_rhs(f)
    cyc, hist = o.solve(1e-10, max_cycles=20)
    assert hist[-1] <= 1e-10 and cyc <= 12
    u = o.get_solution()
    u = u - u.mean()
    assert np.abs(u - uh_b).max() / np.abs(uh_b).max() < 1e-8
    # fixed point: the exact discrete solution is invariant
    o2 = MO.Oracle(cfg, lv)
    o2.set_rhs(f)
    o2.set_solution(uh_b)
    before = o2.get_solution()
    o2.vcycle(1)
    after = o2.get_solution()
    d = after - before
    assert np.abs(d - d.mean()).max() < 1e-10 * np.abs(before).max()


def _puu_adaptive():
    d = dict(origin=(0.0, 0.0, 0.0), h0=1 / 32, base_blocks=(2, 4, 4), B=16, bc=(0, 1, 1), order=4,
             smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(d)
    t = Lay.Tree(dom)
    for b in sorted(t.nodes[0]):
        if 1 <= b[1] <= 2 and 1 <= b[2] <= 2 and b[0] == 0:
            t.refine(0, b)
    lv = t.leaves()
    Lay.check_layout(dom, lv)
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.06, c=(0.3, 0.5, 0.5)))
    return d, lv, f


def test_adaptive_puu_converges_and_is_deterministic():
    d, lv, f = _puu_adaptive()
    o = MO.Oracle(d, lv)
    o.set_rhs(f)
    cyc, hist = o.solve(1e-10, max_cycles=20)
    assert hist[-1] <= 1e-10, hist
    rates = np.array(hist[2:]) / np.array(hist[1:-1])
    assert np.all(rates < 0.35), rates
    # bitwise determinism
    o2 = MO.Oracle(d, lv)
    o2.set_rhs(f)
    o2.vcycle(3)
    o3 = MO.Oracle(d, lv)
    o3.set_rhs(f)
    o3.vcycle(3)
    assert np.array_equal(o2.get_solution(), o3.get_solution())
    # the converged composite solution is a fixed point of the cycle
    u = o.get_solution()
    o.vcycle(1)
    assert np.abs(o.get_solution() - u).max() < 1e-9 * np.abs(u).max()


def test_adaptive_periodic_singular_stall_and_cauchy():
    """Periodic + jumps: the residual stalls above zero (E15-E19) while
    the Cauchy increment (E20) keeps decreasing."""
    dom = Lay.Domain((0.0, 0.0, 0.0), 1 / 32, (2, 2, 2), 16, (0, 0, 0))
    lv = Lay.corner_nested_leaves(dom, 1)
    d = dict(origin=(0, 0, 0), h0=1 / 32, base_blocks=(2, 2, 2), B=16, bc=(0, 0, 0), order=4, smoother=1,
             omega=1.0, eta1=2, eta2=2, coarse_n=0)
    sig = 0.08

    def fn(x, y, z):
        r2 = (x - 0.25) ** 2 + (y - 0.25) ** 2 + (z - 0.25) ** 2
        return (4 * r2 / sig ** 4 - 6 / sig ** 2) * np.exp(-r2 / sig ** 2)   # E24 with reading Z25

    f = S.sample_on_leaves(dom, lv, fn)
    o = MO.Oracle(d, lv)
    o.set_rhs(f)
    res, inc = [], []
    prev = o.get_solution()
    for _ in range(16):
        o.vcycle(1)
        u = o.get_solution()
        res.append(o.residual_norm()[1])
        inc.append(np.abs(u - prev).max() / np.abs(u).max())
        prev = u
    # the residual stalls: it stops decreasing at a level far above round-off ...
    assert res[7] > 1e-8
    assert abs(res[-1] - res[7]) < 1e-3 * res[7], res
    # ... while the Cauchy increment (E20) keeps contracting to round-off
    assert inc[-1] < 1e-13 and inc[-1] < 1e-5 * inc[7], inc
    # and mg_solve's Cauchy criterion stops, the residual criterion would not
    o2 = MO.Oracle(d, lv)
    o2.set_rhs(f)
    cyc, hist = o2.solve(1e-9, max_cycles=25, criterion="cauchy")
    assert cyc < 25 and hist[-1] < 1e-9
    o3 = MO.Oracle(d, lv)
    o3.set_rhs(f)
    cyc3, hist3 = o3.solve(1e-9, max_cycles=12, criterion="residual")
    assert cyc3 == 12 and hist3[-1] > 1e-8


def test_cfg3_reduced_free_space_fourth_order():
    """Config 3 recipe (UUU, Gaussian σ=0.08, reading U1) at 32^3 and 64^3: the
    V-cycle converges and the origin value approaches the free-space closed form
    -Q erf(r/(√2σ))/(4πr) -> -√(2/π)/(4πσ) at 4th order (P10, E12 design order)."""
    errs = []
    for N, cn in ((32, 8), (64, 16)):
        cfg = C.cfg3(N, coarse_n=cn)
        dom, lv, f = C.build(cfg)
        o = MO.Oracle(cfg, lv)
        o.set_rhs(f)
        hist = []
        for _ in range(14):
            o.vcycle(1)
            hist.append(o.residual_norm()[1])
        assert hist[-1] < 1e-8 * (N / 32) and hist[-1] < hist[0] * 1e-6
        u = o.get_solution()
        c = N // 32
        n = int(np.nonzero((lv == np.array([0, c, c, c])).all(axis=1))[0][0])
        errs.append(abs(u[n, 0, 0, 0] + math.sqrt(2 / math.pi) / (4 * math.pi * 0.08)))
    order = math.log2(errs[0] / errs[1])
    assert 3.4 < order < 4.8, (errs, order)
