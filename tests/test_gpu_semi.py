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
