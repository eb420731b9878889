"""Semi-unbounded directions ("an odd or even condition is enforced in a first
direction ... while an unbounded one is imposed in the opposite"; reading S1): the
oracle's mirror-image coarse solve pinned by the image-charge closed form of a Gaussian
next to the symmetric face, the odd plane, and the discrete equation at the wall."""
import numpy as np
import pytest

from oracle import mg_oracle as MO
from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S

EVEN, ODD, U, P = 2, 3, 1, 0
SIG, CX = 0.08, 0.3


def _case(n, sym, others=(U, U), order=4):
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / (16 * n), base_blocks=(n, n, n), B=16,
               bc=((sym, U), others[0], others[1]), order=order, smoother=1, omega=1.0, eta1=2, eta2=2,
               coarse_n=0)
    dom = C.domain(cfg)
    lv = Lay.uniform_leaves(dom)
    s = 1.0 if sym == EVEN else -1.0
    c, ci = (CX, 0.5, 0.5), (-CX, 0.5, 0.5)          # the charge and its mirror image
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=SIG, c=c)
                           + s * S.gaussian_charge(x, y, z, sigma=SIG, c=ci))
    ua = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_potential(x, y, z, sigma=SIG, c=c)
                            + s * S.gaussian_potential(x, y, z, sigma=SIG, c=ci))
    return cfg, lv, f, ua


def _solve(cfg, lv, f):
    o = MO.Oracle(cfg, lv)
    o.set_rhs(f)
    o.vcycle(1)                    # single level: the direct solve is exact
    return o


@pytest.mark.parametrize("sym", [EVEN, ODD])
def test_image_charge_closed_form_4th_order(sym):
    errs = []
    for n in (2, 4):
        cfg, lv, f, ua = _case(n, sym)
        o = _solve(cfg, lv, f)
        assert o.residual_norm()[1] < 1e-11          # discrete equation incl. the wall nodes
        errs.append(np.abs(o.get_solution() - ua).max())
    assert errs[0] / errs[1] > 12, errs             # 4th order (Mehrstellen + LGF)
    assert errs[1] < 2e-5 * np.abs(ua).max()


def test_odd_face_plane_is_zero_and_even_face_symmetric():
    cfg, lv, f, ua = _case(2, ODD)
    o = _solve(cfg, lv, f)
    u0 = o.levels[0].u
    assert np.abs(u0[0]).max() <= 1e-13 * np.abs(u0).max()       # u(0, y, z) = 0
    # even face: the band below x = 0 mirrors the interior
    cfg, lv, f, ua = _case(2, EVEN)
    o = _solve(cfg, lv, f)
    L0, E = o.levels[0], MO.E
    for k in (1, 2):
        assert np.allclose(L0.band[E - k, E:E + 32, E:E + 32], L0.u[k], rtol=0, atol=1e-13 * np.abs(L0.u).max())


@pytest.mark.parametrize("others", [(P, U), (U, P)])
def test_semi_unbounded_mixed_with_periodic(others):
    """x semi-unbounded with one periodic and one unbounded axis: the discrete solution
    satisfies the discrete equation everywhere (incl. wall nodes) and is odd/even."""
    cfg, lv, f, ua = _case(2, ODD, others)
    o = _solve(cfg, lv, f)
    assert o.residual_norm()[1] < 1e-11
    assert np.abs(o.levels[0].u[0]).max() <= 1e-13 * np.abs(o.levels[0].u).max()


# ------------------------------------------------------------- both faces symmetric (S2)
def _ss_case(pair, k, others=(P, P), n=2, order=4):
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / (16 * n), base_blocks=(n, n, n), B=16,
               bc=(pair, others[0], others[1]), order=order, smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    lv = Lay.uniform_leaves(dom)
    N = 16 * n
    if pair == (ODD, ODD):
        th = np.pi * k / N                           # DST-I mode sin(π k J / N)
        fn = lambda x, y, z: np.sin(th * x * N) + 0 * y + 0 * z   # noqa: E731
    else:
        th = np.pi * (2 * k + 1) / (2 * N)           # DCT-III mode cos(π (2k+1) J / (2N))
        fn = lambda x, y, z: np.cos(th * x * N) + 0 * y + 0 * z   # noqa: E731
    f = S.sample_on_leaves(dom, lv, fn)
    return cfg, lv, f, th, N


@pytest.mark.parametrize("pair,k", [((ODD, ODD), 1), ((ODD, ODD), 5), ((EVEN, ODD), 0), ((EVEN, ODD), 3)])
def test_symmetric_both_faces_eigenmode_exact(pair, k):
    """Homogeneous Dirichlet (ODD/ODD) and Neumann-Dirichlet (EVEN/ODD) along x:
    a sine / shifted-cosine mode is a lattice eigenfunction, so the discrete solution is
    f (1 + ŝ/12) / (ŝ/h²), ŝ = 2cos θ - 2 (M = 4; A6), including the wall nodes."""
    cfg, lv, f, th, N = _ss_case(pair, k)
    o = _solve(cfg, lv, f)
    h = 1.0 / N
    sh = 2 * np.cos(th) - 2
    uexp = f * (1 + sh / 12) / (sh / h ** 2)
    assert np.abs(o.get_solution() - uexp).max() <= 1e-11 * np.abs(uexp).max()
    assert o.residual_norm()[1] < 1e-11


def test_symmetric_both_faces_with_unbounded_axes():
    """ODD/ODD x with unbounded y, z: the discrete equation holds everywhere (walls and
    band) and the solution is odd about x = 0."""
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / 32, base_blocks=(2, 2, 2), B=16,
               bc=((ODD, ODD), U, U), order=4, smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    lv = Lay.uniform_leaves(dom)
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.08, c=(0.4, 0.5, 0.5)))
    o = _solve(cfg, lv, f)
    assert o.residual_norm()[1] < 1e-11
    u0 = o.levels[0].u
    assert np.abs(u0[0]).max() <= 1e-13 * np.abs(u0).max()


# ------------------------------------------------------------- EVEN / EVEN (reading S3)
def _ee_case(others, n=2, order=4):
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / (16 * n), base_blocks=(n, n, n), B=16,
               bc=((EVEN, EVEN), others[0], others[1]), order=order, smoother=1, omega=1.0, eta1=2, eta2=2,
               coarse_n=0)
    dom = C.domain(cfg)
    return cfg, dom, Lay.uniform_leaves(dom)


@pytest.mark.parametrize("order", [2, 4, 6])
@pytest.mark.parametrize("k", [1, 4, 9])
def test_even_even_eigenmode_exact(order, k):
    """Homogeneous Neumann on both x faces, walls at nodes 0 and N-1 (reading S3):
    cos(θ J), θ = πk/(N-1), is a lattice eigenfunction of every Mehrstellen operator with
    the mirrored ghosts, eigenvalue σ_M(θ, θ_y, 0) from the stencil symbol (A1); f* =
    R_h^M f scales it by ρ_M, so u = f ρ_M / σ_M exactly, walls included."""
    cfg, dom, lv = _ee_case((P, P), order=order)
    N = 32
    h = 1.0 / N
    th, ky = np.pi * k / (N - 1), 2 * np.pi * 3 / N
    fn = lambda x, y, z: np.cos(th * x * N) * np.cos(ky * y * N) + 0 * z   # noqa: E731
    f = S.sample_on_leaves(dom, lv, fn)
    o = _solve(cfg, lv, f)
    sx, sy = 2 * np.cos(th) - 2, 2 * np.cos(ky) - 2
    # symbols typed from fig:stencils (M = 2, 4, 6) and the right-hand sides E10-E13
    sig = {2: sx + sy, 4: sx + sy + sx * sy / 6, 6: sx + sy + sx * sy / 6}[order] / h ** 2
    rho = {2: 1.0, 4: 1 + (sx + sy) / 12, 6: 1 + (sx + sy) / 12 + sx * sy / 90 - (sx * sx + sy * sy) / 240}[order]
    uexp = f * rho / sig
    assert np.abs(o.get_solution() - uexp).max() <= 1e-11 * np.abs(uexp).max()


def test_even_even_singular_zero_mean_and_neumann_convergence():
    """Pure Neumann box (EVEN/EVEN on all axes): the constant is in the null space, the
    coarse solve returns the zero-(weighted-)mean solution; with the compatible
    manufactured u = cos(πx/Lx) cos(πy/Ly) + cos(2πz/Lz), L = (N-1)h (walls at 0 and L),
    the discrete solution converges to u at 4th order (M = 4) mod the constant."""
    errs = []
    for n in (2, 4):
        cfg, dom, lv = _ee_case(((EVEN, EVEN), (EVEN, EVEN)), n=n)
        N = 16 * n
        L = (N - 1) / N
        ue = lambda x, y, z: np.cos(np.pi * x / L) * np.cos(np.pi * y / L) + np.cos(2 * np.pi * z / L)  # noqa: E731
        fe = lambda x, y, z: (-2 * (np.pi / L) ** 2 * np.cos(np.pi * x / L) * np.cos(np.pi * y / L)  # noqa: E731
                              - (2 * np.pi / L) ** 2 * np.cos(2 * np.pi * z / L))
        f = S.sample_on_leaves(dom, lv, fe)
        o = _solve(cfg, lv, f)
        assert o.residual_norm()[1] < 1e-10        # the discrete equation, walls included
        u = o.get_solution()
        ua = S.sample_on_leaves(dom, lv, ue)
        d = u - ua
        errs.append(np.abs(d - d.mean()).max())
    rate = np.log2(errs[0] / errs[1])
    assert 3.6 < rate < 4.6, (errs, rate)


def test_even_even_rejects_unbounded_axes():
    cfg, dom, lv = _ee_case((U, P))
    with pytest.raises(ValueError):
        MO.Oracle(cfg, lv)
