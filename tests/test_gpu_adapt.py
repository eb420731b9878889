"""Grid adaptation on the GPU: the detail-coefficient kernel
(mg_detail) against oracle/adapt.py on random and smooth fields, and the adaptation
pipeline (GPU details -> mg_adapt -> resample -> ...) against the oracle pipeline fed
the same γ, ending in a solver built on the adapted grid."""
import numpy as np
import pytest

from oracle import adapt as OA
from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S


def _gpu_detail(f, B, W):
    import torch

    from paper_2512_08555_b200 import detail
    return detail(torch.from_numpy(np.ascontiguousarray(f)).cuda(), B, W).cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("B,W", [(16, 2), (16, 4), (16, 6), (8, 2), (8, 4)])
def test_detail_kernel_parity(B, W):
    rng = np.random.default_rng(B * 10 + W)
    n = 37
    f = rng.standard_normal((n, B, B, B))
    z, y, x = np.meshgrid(np.arange(B), np.arange(B), np.arange(B), indexing="ij")
    f[:5] = np.sin(0.3 * x + 0.2 * y - 0.1 * z)[None] * np.arange(1, 6)[:, None, None, None]
    f[5] = (x / B) ** (W - 1)                           # γ = 0 up to rounding
    g = _gpu_detail(f, B, W)
    ref = OA.details(f, W)
    scale = np.abs(f).reshape(n, -1).max(axis=1)
    assert np.all(np.abs(g - ref) <= 1e-12 * scale), np.abs(g - ref).max()
    assert g[5] <= 1e-13


@pytest.mark.gpu
def test_detail_edge_cases():
    import torch

    from paper_2512_08555_b200 import MgError, detail
    assert detail(torch.zeros((0, 16, 16, 16), dtype=torch.float64, device="cuda"), 16, 4).numel() == 0
    with pytest.raises(MgError):
        detail(torch.zeros((2, 8, 8, 8), dtype=torch.float64, device="cuda"), 8, 6)   # 8 taps span > block
    with pytest.raises(MgError):
        detail(torch.zeros((2, 16, 16, 16), dtype=torch.float64, device="cuda"), 16, 3)


@pytest.mark.gpu
def test_adaptation_pipeline_matches_oracle_and_solves():
    import torch

    from paper_2512_08555_b200 import Solver, adapt
    cfg = dict(origin=(0.0, 0.0, 0.0), h0=1 / 64, base_blocks=(4, 4, 4), B=16, bc=(0, 1, 1), order=4,
               smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(cfg)
    blob = lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.06, c=(0.45, 0.5, 0.55))  # noqa: E731
    lv = Lay.uniform_leaves(dom)
    steps = 0
    while True:
        f = S.sample_on_leaves(dom, lv, blob)
        g = _gpu_detail(f, 16, 4)
        new_g, _ = adapt(cfg, lv, g, 1e-3 * np.abs(f).max(), 1e-5 * np.abs(f).max(), 2)
        new_o, _ = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, g, 1e-3 * np.abs(f).max(),
                            1e-5 * np.abs(f).max(), 2)
        assert np.array_equal(new_g, new_o)
        steps += 1
        if np.array_equal(new_g, np.array(sorted(map(tuple, lv)), dtype=np.int32)) or steps > 6:
            break
        lv = new_g
    Lay.check_layout(dom, lv)
    assert lv[:, 0].max() == 2
    s = Solver(cfg, lv)
    s.set_rhs(torch.from_numpy(S.sample_on_leaves(dom, lv, blob)).cuda())
    cyc, rel, ok = s.solve(1e-9, 30)
    assert ok, (cyc, rel)


@pytest.mark.gpu
def test_transfer_onto_adapted_grid_matches_oracle():
    """mg_transfer (reading A3): after 3 V-cycles on the old grid, u moves onto an adapted
    grid (one x-block coarsened, one refined; x periodic, y, z unbounded) exactly as the
    oracle's transfer_from (copies bit for bit, trilinear within round-off), and the
    adapted grid solves from that warm start."""
    import torch

    from paper_2512_08555_b200 import Solver
    from tests.test_oracle_adapt import _transfer_pair
    from workloads import sources as S
    MO, d, old_lv, new_lv = _transfer_pair()
    dom = C.domain(d)
    src = lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.06, c=(0.35, 0.5, 0.5))  # noqa: E731
    f_old = S.sample_on_leaves(dom, old_lv, src)
    f_new = S.sample_on_leaves(dom, new_lv, src)
    o_old = MO.Oracle(d, old_lv)
    o_old.set_rhs(f_old)
    o_old.vcycle(3)
    g_old = Solver(d, old_lv)
    g_old.set_rhs(torch.from_numpy(f_old).cuda())
    g_old.vcycle(3)
    o_new = MO.Oracle(d, new_lv)
    o_new.set_rhs(f_new)
    o_new.transfer_from(o_old)
    g_new = Solver(d, new_lv)
    g_new.set_rhs(torch.from_numpy(f_new).cuda())
    g_new.transfer_from(g_old)
    ug, uo = g_new.get_solution().cpu().numpy(), o_new.get_solution()
    assert np.abs(ug - uo).max() <= 1e-9 * np.abs(uo).max()
    cyc, rel, ok = g_new.solve(1e-10, 40)
    cold = Solver(d, new_lv)
    cold.set_rhs(torch.from_numpy(f_new).cuda())
    cyc0, rel0, ok0 = cold.solve(1e-10, 40)
    # the warm start (3 cycles' worth of the old grid) needs no more cycles than u = 0
    assert ok and ok0 and cyc <= cyc0, (cyc, cyc0)
