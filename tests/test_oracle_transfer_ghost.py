"""Pins of the oracle's inter-grid transfers and ghost interpolation (P2, P3, P4)."""
import numpy as np
import pytest

from oracle import mg_oracle as MO
from workloads import layouts as Lay


def test_lagrange_weights_textbook():
    # 4-point and 6-point midpoint Lagrange weights (standard tables)
    assert np.allclose(MO.lagrange_midpoint_weights(4), np.array([-1, 9, 9, -1]) / 16, atol=1e-16)
    assert np.allclose(MO.lagrange_midpoint_weights(6), np.array([3, -25, 150, 150, -25, 3]) / 256, atol=1e-16)
    assert np.allclose(MO.lagrange_midpoint_weights(8),
                       np.array([-5, 49, -245, 1225, 1225, -245, 49, -5]) / 2048, atol=1e-16)


def _mid_layout(order=4, bc=(0, 0, 0), depth=1):
    dom = Lay.Domain((0.0, 0.0, 0.0), 1 / 64, (4, 4, 4), 16, bc)
    t = Lay.Tree(dom)
    for b in sorted(t.nodes[0]):
        if all(1 <= c <= 2 for c in b):
            t.refine(0, b)
    if depth == 2:
        for b in sorted(t.nodes[1]):
            if all(3 <= c <= 4 for c in b):
                t.refine(1, b)
    leaves = t.leaves()
    Lay.check_layout(dom, leaves)
    desc = dict(origin=dom.origin, h0=dom.h0, base_blocks=dom.base_blocks, B=16, bc=bc, order=order,
                smoother=1, omega=1.0, eta1=1, eta2=1, coarse_n=0)
    return dom, leaves, desc


@pytest.mark.parametrize("order", [2, 4])
def test_ghost_fill_polynomial_exactness(order):
    """c2f reproduces every polynomial of degree < I = M+2 at all jump ghosts incl.
    edges and corners, through the f2c-injected source W."""
    dom, leaves, desc = _mid_layout(order, depth=2)
    o = MO.Oracle(desc, leaves)
    I = order + 2
    rng = np.random.default_rng(1)
    coef = rng.normal(size=(I, I, I))

    def poly(Lv):
        # level-global J of the extended (window + pad) positions
        idx = [(np.arange(-MO.E, n + MO.E) + lo) * Lv.h for n, lo in zip(Lv.n, Lv.lo)]
        X, Y, Z = np.meshgrid(*idx, indexing="ij")
        out = np.zeros_like(X)
        for a in range(I):
            for b in range(I - a):
                for c in range(I - a - b):
                    out += coef[a, b, c] * X ** a * Y ** b * Z ** c
        return out

    for Lv in o.levels:
        Lv.u = o._interior(poly(Lv), Lv).copy()
    vals = o.uvals()
    for m in range(1, len(o.levels)):
        Lv = o.levels[m]
        X = o.lookup(m, vals)
        P = poly(Lv)
        ghost = ~Lv.mask_ext
        # ghosts inside the periodic domain, within 3 nodes of the level-m region
        near = np.zeros_like(ghost)
        mk = Lv.mask_ext
        for s in [(a, b, c) for a in range(-3, 4) for b in range(-3, 4) for c in range(-3, 4)]:
            near |= np.roll(mk, s, axis=(0, 1, 2))
        sel = ghost & near
        # (np.roll wraps: drop the 3 outermost layers of the extended array)
        sel[:3] = sel[-3:] = False
        sel[:, :3] = sel[:, -3:] = False
        sel[:, :, :3] = sel[:, :, -3:] = False
        assert sel.sum() > 1000
        err = np.abs(X[sel] - P[sel]).max() / np.abs(P[sel]).max()
        assert err < 1e-12, (m, err)


def test_fw_restriction_preserves_linears_and_prolong_trilinear():
    dom, leaves, desc = _mid_layout(4)
    o = MO.Oracle(desc, leaves)
    L1, L0 = o.levels[1], o.levels[0]
    # residual r = f - Δu with u = 0: put a linear function in f on level 1
    J = [np.arange(n) * L1.h for n in L1.N]
    X, Y, Z = np.meshgrid(*J, indexing="ij")
    L1.f = 1.5 + 2 * X - Y + 0.5 * Z
    L1.u[:] = 0
    L0.u[:] = 0
    o.restrict(1)
    Jc = [np.arange(n) * L0.h for n in L0.N]
    Xc, Yc, Zc = np.meshgrid(*Jc, indexing="ij")
    lin = 1.5 + 2 * Xc - Yc + 0.5 * Zc
    # interior covered nodes (FW stencil inside level 1): exact
    inner = np.zeros_like(L0.cov)
    inner[17:47, 17:47, 17:47] = True
    assert np.abs(L0.r[inner] - lin[inner]).max() < 1e-13
    # prolongation: ε trilinear -> fine nodes receive the trilinear function exactly
    L0.uhat = np.zeros_like(L0.u)
    L0.u = np.where(L0.mask, (1 + Xc) * (2 - Yc) * (0.5 + Zc), 0.0)
    L1.u[:] = 0
    o.prolong(1)
    want = (1 + X) * (2 - Y) * (0.5 + Z)
    assert np.abs(L1.u[L1.mask] - want[L1.mask]).max() < 1e-14


def test_injection_bitwise():
    dom, leaves, desc = _mid_layout(4)
    o = MO.Oracle(desc, leaves)
    rng = np.random.default_rng(3)
    o.levels[1].u = rng.normal(size=tuple(o.levels[1].N))
    o.inject_up()
    C = o.levels[0]
    assert np.array_equal(C.u[C.cov], o.levels[1].u[::2, ::2, ::2][C.cov])
