"""Semi-unbounded directions on the GPU (reading S1): a Gaussian charge next to
an even / odd face, on a 2-level grid, solved to 1e-10 and compared with the
image-charge closed form."""
import numpy as np
import pytest

from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S

EVEN, ODD, U, P = 2, 3, 1, 0


def _run(n, sym, others):
    import torch

    from paper_2512_08555_b200 import Solver
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / (16 * n), base_blocks=(n, n, n), B=16,
               bc=((sym, U), others[0], others[1]), order=4, smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    t = Lay.Tree(dom)
    for b in sorted(t.nodes[0]):               # refine the interior around the charge
        if all(n // 4 <= b[a] < n - n // 4 for a in range(3)):
            t.refine(0, b)
    lv = t.leaves()
    Lay.check_layout(dom, lv)
    s = 1.0 if sym == EVEN else -1.0
    c, ci = (0.3, 0.5, 0.5), (-0.3, 0.5, 0.5)
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.08, c=c)
                           + s * S.gaussian_charge(x, y, z, sigma=0.08, c=ci))
    ua = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_potential(x, y, z, sigma=0.08, c=c)
                            + s * S.gaussian_potential(x, y, z, sigma=0.08, c=ci))
    S_ = Solver(cfg, lv)
    S_.use_graph(True)
    S_.set_rhs(torch.from_numpy(f).cuda())
    cyc, rel, ok = S_.solve(1e-10, 30)
    assert ok, (cyc, rel)
    return np.abs(S_.get_solution().cpu().numpy() - ua).max(), np.abs(ua).max()


@pytest.mark.gpu
@pytest.mark.parametrize("sym", [EVEN, ODD])
def test_semi_unbounded_image_charge(sym):
    """64^3 level 0 with the interior refined once: E∞ against the image-charge closed
    form below the uniform 64^3 oracle error (tests/test_oracle_semi.py pins the 4th-order
    convergence of the same discretisation on the CPU)."""
    e, umax = _run(4, sym, (U, U))
    assert e < 2e-5 * umax, (e, umax)


@pytest.mark.gpu
@pytest.mark.parametrize("pair,k", [((ODD, ODD), 3), ((EVEN, ODD), 2)])
def test_symmetric_both_faces_eigenmode_gpu(pair, k):
    """Homogeneous Dirichlet / Neumann-Dirichlet along x (reading S2) on a uniform
    64^3 grid (y, z periodic): a sine / shifted-cosine lattice eigenmode is solved
    exactly, f (1 + ŝ/12) / (ŝ/h²) (A6), walls included."""
    import torch

    from paper_2512_08555_b200 import Solver
    n = 4
    N = 16 * n
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / N, base_blocks=(n, n, n), B=16, bc=(pair, P, P), order=4,
               smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    lv = Lay.uniform_leaves(dom)
    th = np.pi * k / N if pair == (ODD, ODD) else np.pi * (2 * k + 1) / (2 * N)
    trig = np.sin if pair == (ODD, ODD) else np.cos
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: trig(th * x * N) + 0 * y + 0 * z)
    s = Solver(cfg, lv)
    s.set_rhs(torch.from_numpy(f).cuda())
    s.vcycle(1)                     # one level: the coarse solve is the solution
    sh = 2 * np.cos(th) - 2
    uexp = f * (1 + sh / 12) / (sh * N * N)
    u = s.get_solution().cpu().numpy()
    assert np.abs(u - uexp).max() <= 1e-11 * np.abs(uexp).max()
    assert s.residual_norm()[1] < 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("k,order", [(3, 4), (7, 6)])
def test_even_even_eigenmode_gpu(k, order):
    """Homogeneous Neumann on both x faces (walls at nodes 0 and N-1; reading S3) with y, z
    periodic, uniform 64^3: cos(θ J), θ = πk/(N-1), is solved exactly through the C-ABI,
    u = f ρ_M / σ_M (tests/test_oracle_semi.py pins the same closed form for the oracle)."""
    import torch

    from paper_2512_08555_b200 import Solver
    n = 4
    N = 16 * n
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1.0 / N, base_blocks=(n, n, n), B=16, bc=((EVEN, EVEN), P, P),
               order=order, smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    lv = Lay.uniform_leaves(dom)
    th = np.pi * k / (N - 1)
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: np.cos(th * x * N) + 0 * y + 0 * z)
    s = Solver(cfg, lv)
    s.set_rhs(torch.from_numpy(f).cuda())
    s.vcycle(1)
    sx = 2 * np.cos(th) - 2
    rho = 1 + sx / 12 - (sx * sx / 240 if order == 6 else 0.0)
    uexp = f * rho / (sx * N * N)
    u = s.get_solution().cpu().numpy()
    assert np.abs(u - uexp).max() <= 1e-11 * np.abs(uexp).max()
    assert s.residual_norm()[1] < 1e-11
