"""Parity of every kernel variant the automatic choice takes at full size, on small
layouts (the production variants — 2- and 4-block pencils, sweeps without
the z-split, the fused residual+restriction and fused last-pre-sweep kernels next to
jump and exterior ghost blocks — must match the oracle element-wise).

mg_desc.pencil_blocks / zsplit / fuse force the variant (include/mg.h); the oracle is
the same for all of them.  Tolerances as in test_gpu_parity: ≤1e-12 per operator,
≤1e-9 on u after V-cycles.
"""
import numpy as np
import pytest

from tests.gpu_helpers import Pair, rel_err
from tests.test_gpu_parity import CYCLE_TOL, OP_TOL, _cfg, _prepared

# jumps and exterior (U1) ghost blocks: puu2, cfg3_64, per_adapt; ghost-free: cfg2_64.  (The
# semi-unbounded ou_uu, whose oracle costs ~25 s per test, stays in test_gpu_parity: its
# symmetric face changes only the coarse solve, not the pencil kernels varied here.)
LAYOUTS = ["puu2", "cfg3_64", "per_adapt", "cfg2_64"]
VARIANTS = [dict(pencil_blocks=1, zsplit=1), dict(pencil_blocks=1, zsplit=2), dict(pencil_blocks=2),
            dict(pencil_blocks=3), dict(pencil_blocks=4), dict(pencil_blocks=2, fuse=1), dict(pencil_blocks=2, staging=1),
            dict(ghost_kernel=1), dict(ghost_kernel=2),
            # z-aligned chunks in z-major launch order (the automatic choice on levels of >= 24 waves)
            dict(pencil_blocks=4, pencil_order=2), dict(pencil_blocks=3, pencil_order=2)]


def _vid(v):
    return "-".join(f"{'o' if k == 'pencil_order' else k[0]}{v[k]}" for k in sorted(v))


def _with(name, variant, order=None):
    cfg, lv, f = _cfg(name)
    cfg = dict(cfg)
    cfg.update(variant)
    if order:
        cfg["order"] = order
    return cfg, lv, f


# M = 4 on every layout x variant; M = 6 (k_rb6_pencil, the radius-2 RHS) on the
# multi-block-pencil variants of two layouts with ghost blocks
CASES = [(n, v, 4) for n in LAYOUTS for v in VARIANTS] + \
        [(n, v, 6) for n in ("puu2", "cfg3_64") for v in VARIANTS[1:5] + VARIANTS[9:10]]


@pytest.mark.gpu
@pytest.mark.parametrize("name,variant,order", CASES, ids=lambda x: _vid(x) if isinstance(x, dict) else str(x))
def test_vcycle_parity_variants(name, variant, order):
    cfg, lv, f = _with(name, variant, order)
    p = Pair(cfg, lv, f)
    for c in range(2):
        p.ocycle()
        p.g.vcycle(1)
        e = rel_err(p.solution(), p.o.get_solution())
        assert e < CYCLE_TOL, (name, variant, c, e)
    ro, rg = p.o.residual_norm(), p.g.residual_norm()
    assert abs(rg[1] - ro[1]) <= 1e-6 * ro[1] + 1e-12, (rg, ro)


def _prep(name, variant, order):
    import tests.test_gpu_parity as T
    orig = T._cfg
    T._cfg = lambda n: _with(n, variant, order)
    try:
        return _prepared(name)
    finally:
        T._cfg = orig


OP_CASES = [(n, v, 4) for n in ("puu2", "cfg3_64", "per_adapt") for v in VARIANTS] + \
           [("cfg3_64", v, 6) for v in VARIANTS[1:4]]


@pytest.mark.gpu
@pytest.mark.parametrize("name,variant,order", OP_CASES, ids=lambda x: _vid(x) if isinstance(x, dict) else str(x))
def test_ops_parity_variants(name, variant, order):
    """smooth, residual (and the composite norm), restrict (+ FAS RHS + û), prolong."""
    p = _prep(name, variant, order)
    top = len(p.o.levels) - 1
    # residual first: the per-operator order matters on the oracle side, whose ghost
    # refresh never writes the coarse covered nodes (the GPU's f2c injection does; in
    # Alg. 1 the restriction overwrites them before any coarse residual reads them)
    for m in range(0, top + 1):
        L = p.o.levels[m]
        r = p.o.residual(m)
        p.g.debug_apply("residual", m)
        Lu = p.o.Lu(m)
        den = max(np.abs(L.f[L.mask]).max(), np.abs(Lu[L.mask]).max())
        e = rel_err(p.gpu_field("r", m)[L.mask], r[L.mask], den)
        assert e < OP_TOL, ("residual", m, e)
    assert abs(p.g.residual_norm()[0] - p.o.residual_norm()[0]) <= OP_TOL * max(1.0, p.o.fstar_norm) * 1e2
    # the GPU ghost refreshes above injected level-m values into the covered nodes of
    # level m-1 (f2c lists); the oracle keeps them in a copy (W_{m-1}): restart both
    # sides from the oracle's state before the next operator
    p.push_state()
    for m in range(1, top + 1):
        p.o.smooth(m)
        p.g.debug_apply("smooth", m)
        L = p.o.levels[m]
        e = rel_err(p.gpu_field("u", m)[L.mask], L.u[L.mask])
        assert e < OP_TOL, ("smooth", m, e)
    for m in range(top, 0, -1):
        p.o.restrict(m)
        p.g.debug_apply("restrict", m)
        C_ = p.o.levels[m - 1]
        # f = r + Δu is residual-type: denominator max(|f|, |Δu|)
        den_f = max(np.abs(C_.f[C_.cov]).max(), np.abs(p.o.Lu(m - 1)[C_.cov]).max())
        for fld, ref in (("u", C_.u), ("f", C_.f), ("uhat", C_.uhat)):
            e = rel_err(p.gpu_field(fld, m - 1)[C_.cov], ref[C_.cov], den_f if fld == "f" else None)
            assert e < OP_TOL, ("restrict", m, fld, e)
    for m in range(1, top + 1):
        p.o.prolong(m)
        p.g.debug_apply("prolong", m)
        L = p.o.levels[m]
        e = rel_err(p.gpu_field("u", m)[L.mask], L.u[L.mask])
        assert e < OP_TOL, ("prolong", m, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [dict(), dict(pencil_blocks=4), dict(fuse=1)], ids=_vid)
@pytest.mark.parametrize("name", ["cfg2_128", "cfg3_128"])
def test_large_level_parity(name, variant):
    """Levels of >= 148 blocks (512 at 128^3): the automatic choice there is 1-block
    pencils without z-split; forced 4-block pencils and unfused kernels too."""
    cfg, lv, f = _with(name, variant)
    p = Pair(cfg, lv, f)
    assert p.g.level_info(len(p.o.levels) - 1)["nreal"] >= 148
    for c in range(2):
        p.ocycle()
        p.g.vcycle(1)
        e = rel_err(p.solution(), p.o.get_solution())
        assert e < CYCLE_TOL, (name, c, e)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [dict(pencil_blocks=2), dict(pencil_blocks=3), dict(pencil_blocks=4),
                                     dict(pencil_blocks=1, zsplit=1), dict(pencil_blocks=4, pencil_order=2),
                                     dict(pencil_blocks=2, pencil_order=2)],
                         ids=_vid)
def test_cfg5_shaped_variants(variant):
    """The 5-level PUU torus layout (cfg5 recipe, reduced) with forced pencil lengths."""
    cfg, lv, f = _with("cfg5_small", variant)
    p = Pair(cfg, lv, f)
    for c in range(3):
        p.ocycle()
        p.g.vcycle(1)
        e = rel_err(p.solution(), p.o.get_solution())
        assert e < CYCLE_TOL, (variant, c, e)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["puu2", "cfg3_64", "cfg2_64", "cfg5_small"])
def test_tma_and_cpasync_staging_bitwise(name):
    """The RB sweep's plane tiles staged by cp.async (default) or by TMA tensor copies
    (mg_desc.staging = 1) move the same values: V-cycle results are bitwise identical."""
    import torch

    from paper_2512_08555_b200 import Solver
    cfg, lv, f = _cfg(name)
    outs = []
    for st in (0, 1):
        c = dict(cfg)
        c["staging"] = st
        s = Solver(c, lv)
        s.set_rhs(torch.from_numpy(f).cuda())
        s.vcycle(2)
        outs.append(s.get_solution().cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["puu1", "puu2", "cfg4_small", "cfg5_small"])
def test_pruned_coarse_solve_matches_3d_and_oracle(name):
    """The x-periodic, y/z-unbounded coarse solve through 1-D cuFFT transforms (default)
    equals the oracle at the per-operator tolerance on the level-0 nodes, and its exterior
    band (read by the level-0 leaf residual) gives the oracle's composite residual; the
    plain padded 3-D transform (mg_desc.coarse_pruning = 1) and the fused shared-memory FFT
    kernels of mg_fft.cu (2) give the same level-0 values and band."""
    import torch

    from paper_2512_08555_b200 import Solver
    p = _prepared(name)
    c = p.o.levels[0]
    rng = np.random.default_rng(3)
    c.f = rng.standard_normal(c.f.shape)
    p.push("f", 0, c.f)
    p.o.coarse_solve()
    p.g.debug_apply("coarse_solve", 0)
    assert rel_err(p.gpu_field("u", 0), c.u) < OP_TOL
    ro, rg = p.o.residual_norm()[0], p.g.residual_norm()[0]
    assert abs(rg - ro) <= 1e-10 * max(1.0, np.abs(c.f).max())
    cfg, lv, f = _cfg(name)
    for mode in (1, 2):   # the padded 3-D transform; the fused FFT kernels
        c2 = dict(cfg)
        c2["coarse_pruning"] = mode
        q = Solver(c2, lv)
        q.set_rhs(torch.from_numpy(f).cuda())
        for m in range(len(p.o.levels)):          # the same state as p's GPU side
            for fld in (0, 1, 3):
                q.debug_field(fld, m, p.g.debug_field(fld, m))
        q.debug_apply("coarse_solve", 0)
        assert abs(q.residual_norm()[0] - rg) <= 1e-12 * max(1.0, rg), mode
        assert rel_err(q.debug_field(0, 0).cpu().numpy(), p.g.debug_field(0, 0).cpu().numpy()) < 1e-13, mode
