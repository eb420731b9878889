"""Edge cases and error behaviour of the C-ABI (include/mg.h conventions): invalid
layouts and arguments return the documented negative codes, calls out of order are
rejected, degenerate right-hand sides and non-convergence are reported, and small
block sizes / single-block levels still match the oracle."""
import numpy as np
import pytest

from tests.gpu_helpers import Pair, rel_err
from workloads import configs as C
from workloads import layouts as Lay
from workloads import sources as S

MG_WARN_NOT_CONVERGED, MG_ERR_ARG, MG_ERR_LAYOUT_NESTING, MG_ERR_LAYOUT_2TO1 = 1, -1, -2, -3
MG_ERR_UNBOUNDED_REFINED, MG_ERR_BC, MG_ERR_ORDER, MG_ERR_STATE, MG_ERR_NONFINITE = -4, -5, -6, -7, -10


def _base(**kw):
    d = dict(origin=(0.0, 0.0, 0.0), h0=1 / 64, base_blocks=(4, 4, 4), B=16, bc=(0, 0, 0), order=4,
             smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    d.update(kw)
    return d


def _err_code(d, leaves):
    from paper_2512_08555_b200 import MgError, Solver
    with pytest.raises(MgError) as e:
        Solver(d, leaves)
    return e.value.code


@pytest.mark.gpu
def test_invalid_descriptions_return_codes():
    d = _base()
    lv = Lay.uniform_leaves(C.domain(d))
    assert _err_code(_base(order=8), lv) == MG_ERR_ORDER               # M in {2, 4, 6}
    assert _err_code(_base(bc=(1, 2, 1)), lv) == MG_ERR_BC            # EVEN/EVEN with unbounded axes
    assert _err_code(_base(bc=(0, (3, 2), 0)), lv) == MG_ERR_BC       # ODD/EVEN is not a supported pair
    assert _err_code(_base(B=12), lv) == MG_ERR_ARG
    assert _err_code(d, lv[:-1]) == MG_ERR_LAYOUT_NESTING           # a hole in level 0
    # 2:1 violation: one level-0 block refined twice in a corner
    t = Lay.Tree(C.domain(d))
    t.refine(0, (0, 0, 0))
    t.refine(1, (0, 0, 0))
    assert _err_code(d, t.leaves()) == MG_ERR_LAYOUT_2TO1
    # refinement touching an unbounded face without the U1 opt-in
    du = _base(bc=(0, 1, 1))
    t = Lay.Tree(C.domain(du))
    t.refine(0, (1, 0, 1))
    t.balance(lambda lev, c: False)
    assert _err_code(du, t.leaves()) == MG_ERR_UNBOUNDED_REFINED


@pytest.mark.gpu
def test_call_order_zero_rhs_nonfinite_and_not_converged():
    import torch

    from paper_2512_08555_b200 import MgError, Solver
    d = _base()
    lv = Lay.uniform_leaves(C.domain(d))
    s = Solver(d, lv)
    with pytest.raises(MgError) as e:
        s.vcycle(1)                      # before mg_set_rhs
    assert e.value.code == MG_ERR_STATE
    # zero right-hand side: the zero solution is exact, the norms are 0 (no division by 0)
    s.set_rhs(torch.zeros(s.leaf_shape(), dtype=torch.float64, device="cuda"))
    s.vcycle(2)
    a, r = s.residual_norm()
    assert a == 0.0 and r == 0.0
    assert float(s.get_solution().abs().max()) == 0.0
    # non-finite data are reported by the norm (MG_ERR_NONFINITE)
    f = torch.zeros(s.leaf_shape(), dtype=torch.float64, device="cuda")
    f[3, 4, 5, 6] = float("nan")
    with pytest.raises(MgError) as e:
        s.set_rhs(f)
    assert e.value.code == MG_ERR_NONFINITE
    # not converged within max_cycles: a positive warning, the partial solution is kept
    # (three levels: with coarse_n = 0 the single level is solved exactly in one cycle)
    d3 = _base(coarse_n=16)
    s = Solver(d3, lv)
    fs = S.dense_to_blocks(C.domain(d3), lv, S.fourier_dense(64, S.fourier_modes(2)))
    s.set_rhs(torch.from_numpy(fs).cuda())
    cyc, rel, ok = s.solve(1e-14, 1)
    assert cyc == 1 and not ok and rel > 1e-14
    assert float(s.get_solution().abs().max()) > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("B", [8])
def test_block_size_8_parity(B):
    """B = 8 blocks (generic kernels, no pencils) on a 2-level periodic-unbounded layout."""
    d = dict(origin=(0.0, 0.0, 0.0), h0=1 / 32, base_blocks=(4, 4, 4), B=B, bc=(0, 1, 1), order=4,
             smoother=1, omega=1.0, eta1=2, eta2=2, coarse_n=0)
    dom = C.domain(d)
    t = Lay.Tree(dom)
    for b in sorted(t.nodes[0]):
        if 1 <= b[1] <= 2 and 1 <= b[2] <= 2:
            t.refine(0, b)
    lv = t.leaves()
    f = S.sample_on_leaves(dom, lv, lambda x, y, z: S.gaussian_charge(x, y, z, sigma=0.1, c=(0.4, 0.5, 0.5)))
    p = Pair(d, lv, f)
    for _ in range(2):
        p.ocycle()
        p.g.vcycle(1)
    assert rel_err(p.solution(), p.o.get_solution()) < 1e-9


@pytest.mark.gpu
def test_variant_controls_rejected():
    d = _base()
    lv = Lay.uniform_leaves(C.domain(d))
    assert _err_code(_base(pencil_blocks=5), lv) == MG_ERR_ARG
    assert _err_code(_base(zsplit=3), lv) == MG_ERR_ARG
    assert _err_code(_base(pencil_order=3), lv) == MG_ERR_ARG
    assert _err_code(_base(fuse=2), lv) == MG_ERR_ARG


@pytest.mark.gpu
def test_cauchy_criterion_on_device_matches_oracle():
    """E20 on the singular periodic adaptive problem, where the residual
    stalls: the device-side Cauchy criterion stops after the same number of cycles as
    the oracle's, with the same increment; an unknown criterion is MG_ERR_ARG."""
    import torch

    from paper_2512_08555_b200 import MgError
    from tests.test_gpu_parity import _cfg
    cfg, lv, f = _cfg("per_adapt")
    p = Pair(cfg, lv, f)
    cyc_o, hist = p.o.solve(1e-9, max_cycles=25, criterion="cauchy")
    cyc_g, val_g, ok = p.g.solve(1e-9, 25, 1)
    assert ok and cyc_g == cyc_o, (cyc_g, cyc_o)
    assert abs(val_g - hist[-1]) <= 1e-6 * hist[-1] + 1e-15, (val_g, hist[-1])
    assert rel_err(p.solution(), p.o.get_solution()) < 1e-9
    with pytest.raises(MgError) as e:
        p.g.solve(1e-9, 3, 7)
    assert e.value.code == MG_ERR_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("name,variant", [("puu2", {}), ("puu2", {"pencil_blocks": 2}), ("cfg3_64", {}),
                                          ("cfg3_64", {"pencil_blocks": 4}), ("ou_uu", {}), ("oo_pp", {}),
                                          ("per_adapt", {}), ("cfg5_small", {}), ("puu1_m6", {}),
                                          ("cfg3_64_m6", {"pencil_blocks": 2}), ("cfg5_small", {"ghost_kernel": 2}),
                                          ("cfg3_64", {"ghost_kernel": 2}), ("puu1_m6", {"ghost_kernel": 2}),
                                          ("cfg5_small", {"pencil_blocks": 4, "pencil_order": 2})])
def test_poisoned_unneeded_ghosts_are_never_read(name, variant):
    """initcheck substitute (compute-sanitizer is closed on this pool): every ghost-block
    node outside the needed halo holds NaN (mg_debug_poison); V-cycles, the composite
    norm and the Cauchy increment stay finite and match the oracle, so no kernel reads
    outside the designed footprint."""
    import torch

    from tests.test_gpu_parity import _cfg
    cfg, lv, f = _cfg(name)
    cfg = dict(cfg)
    cfg.update(variant)
    p = Pair(cfg, lv, f)
    p.g.debug_poison()
    for _ in range(2):
        p.ocycle()
        p.g.vcycle(1)
    u = p.solution()
    assert np.isfinite(u).all()
    assert rel_err(u, p.o.get_solution()) < 1e-9
    a, r = p.g.residual_norm()
    assert np.isfinite(a)
    c, v, ok = p.g.solve(1e-30, 1, 1)
    assert np.isfinite(v)
