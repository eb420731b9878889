"""Pins of oracle/adapt.py (grid adaptation, SPEC.md
detail_coefficient / adapt / enforce_two_to_one) and parity of the host C-ABI
mg_adapt with it (pure host code: runs without a GPU)."""
import numpy as np
import pytest

from oracle import adapt as OA
from workloads import sources as S
from workloads import configs as C
from workloads import layouts as Lay

B = 16
Z, Y, X = np.meshgrid(np.arange(B), np.arange(B), np.arange(B), indexing="ij")


@pytest.mark.parametrize("W", [2, 4, 6])
def test_detail_vanishes_below_degree_W(W):
    h = 1 / 16
    assert OA.detail(np.full((B, B, B), 3.7), W) <= 1e-14 * 3.7     # constants (weights sum to 1)
    # tensor products of degree W-1 per axis are reproduced by the order-W interpolant
    u = (X * h) ** (W - 1) * (1 + Y * h) ** (W - 1) * (Z * h - 0.3) ** (W - 1)
    assert OA.detail(u, W) <= 1e-12 * np.abs(u).max()


@pytest.mark.parametrize("W", [2, 4, 6])
def test_detail_scales_as_h_to_the_W(W):
    # SPEC: γ(h/2)/γ(h) -> 2^-W for monomials of degree >= W (x^W: exactly, by the
    # W-th derivative being constant)
    g1 = OA.detail((X / 16) ** W, W)
    g2 = OA.detail((X / 32) ** W, W)
    assert g1 > 0 and g1 / g2 == pytest.approx(2.0 ** W, rel=1e-9)


def test_centred_weights_are_textbook():
    e, w = OA.taps_1d(7, 16, 4)
    assert e == [4, 6, 8, 10] and np.allclose(w, [-1 / 16, 9 / 16, 9 / 16, -1 / 16], rtol=0, atol=1e-15)
    e, w = OA.taps_1d(15, 16, 4)                      # one-sided at the block's last node
    assert e == [8, 10, 12, 14] and abs(sum(w) - 1) < 1e-14
    assert np.allclose(w, [-5 / 16, 21 / 16, -35 / 16, 35 / 16], rtol=0, atol=1e-14)


def _cfg(bc):
    return dict(base_blocks=(4, 4, 4), bc=bc, B=16, h0=1 / 64, origin=(0.0, 0.0, 0.0))


def test_adapt_zero_field_and_idempotent():
    cfg = _cfg((0, 0, 0))
    lv = Lay.uniform_leaves(C.domain(cfg))
    out, sup = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, np.zeros(len(lv)), 1e-3, 1e-4, 3)
    assert np.array_equal(out, np.array(sorted(map(tuple, lv)), dtype=np.int32)) and sup == 0


def test_adapt_gaussian_cluster_invariants_and_fixed_point():
    """Adapt on the details of a sampled Gaussian until the grid stops changing: nested
    cluster around the centre, 2:1 and P:367 hold (checked by the independent layout
    checker), fewer blocks than uniform refinement, and one more pass is a no-op."""
    cfg = _cfg((0, 1, 1))
    dom = C.domain(cfg)
    fn = lambda x, y, z: np.exp(-((x - .5) ** 2 + (y - .5) ** 2 + (z - .5) ** 2) / .01)  # noqa: E731
    lv = Lay.uniform_leaves(dom)
    for _ in range(6):
        f = Lay_sample(dom, lv, fn)
        g = OA.details(f, 4)
        new, _ = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, g, 1e-4, 1e-6, 3)
        if np.array_equal(new, np.array(sorted(map(tuple, lv)), dtype=np.int32)):
            break
        lv = new
    else:
        pytest.fail("no fixed point")
    Lay.check_layout(dom, lv)
    assert lv[:, 0].max() >= 2 and len(lv) < 64 * 8 ** 3
    fine = lv[lv[:, 0] == lv[:, 0].max()]
    c = (fine[:, 1:] + 0.5) / (4 << int(lv[:, 0].max()))
    assert np.abs(c - 0.5).max() < 0.3                    # the finest blocks sit at the centre


def Lay_sample(dom, lv, fn):
    from workloads import sources as S
    return S.sample_on_leaves(dom, lv, fn)


def test_balance_adds_ring_around_deep_block():
    """An input with a level-2 block family inside a level-0 sea (unbalanced): with no
    refinement or coarsening requested, the balance adds the level-1 ring."""
    cfg = _cfg((0, 0, 0))
    t = Lay.Tree(C.domain(cfg))
    t.refine(0, (1, 1, 1))
    t.refine(1, (2, 2, 2))
    lv = t.leaves()
    out, _ = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, np.zeros(len(lv)), 1.0, 0.0, 3)
    Lay.check_layout(C.domain(cfg), out)
    assert (out[:, 0] == 1).sum() > (lv[:, 0] == 1).sum()


def test_unbounded_face_blocks_stay_level0():
    cfg = _cfg((1, 1, 1))
    lv = Lay.uniform_leaves(C.domain(cfg))
    out, sup = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, np.ones(len(lv)), 0.5, 0.0, 2)
    Lay.check_layout(C.domain(cfg), out)
    assert sup == 56                                      # the 4^3 - 2^3 face blocks
    assert set(map(tuple, out[out[:, 0] > 0][:, 1:] >> out[out[:, 0] > 0][:, :1])) <= {
        (i, j, k) for i in (1, 2) for j in (1, 2) for k in (1, 2)}


@pytest.mark.parametrize("bc", [(0, 0, 0), (0, 1, 1), (1, 1, 0), (1, 1, 1)])
def test_host_abi_adapt_matches_oracle(bc):
    """libmg.so's mg_adapt (C++) == the oracle, bit for bit, over repeated random
    adaptations (identical γ on both sides)."""
    from paper_2512_08555_b200.mg import _LIB_PATH, adapt
    import os
    if not os.path.exists(_LIB_PATH):
        pytest.skip("libmg.so not built")
    cfg = _cfg(bc)
    dom = C.domain(cfg)
    rng = np.random.default_rng(sum(bc))
    lv = Lay.uniform_leaves(dom)
    for _ in range(4):
        g = rng.random(len(lv))
        a, sa = adapt(cfg, lv, g, 0.6, 0.3, 3)
        b, sb = OA.adapt(cfg["base_blocks"], cfg["bc"], lv, g, 0.6, 0.3, 3)
        assert np.array_equal(a, b) and sa == sb
        Lay.check_layout(dom, a)
        lv = a


def _unbalanced_nest():
    """ADVICE r1 regression: 3^3 unbounded base, levels 0/1/2 nested around block
    (1,1,1) without the 2:1 ring (used to loop forever)."""
    lv = [(0, i, j, k) for k in range(3) for j in range(3) for i in range(3) if (i, j, k) != (1, 1, 1)]
    kids = [(1, 2 + i, 2 + j, 2 + k) for k in range(2) for j in range(2) for i in range(2)]
    lv += [c for c in kids if c != (1, 2, 2, 2)]
    lv += [(2, 4 + i, 4 + j, 4 + k) for k in range(2) for j in range(2) for i in range(2)]
    return np.array(lv, dtype=np.int32)


def test_adapt_rejects_invalid_input():
    lv = _unbalanced_nest()
    g = np.full(len(lv), 0.5)
    with pytest.raises(OA.LayoutError) as e:
        OA.adapt((3, 3, 3), (1, 1, 1), lv, g, 1.0, 0.1, 3)
    assert e.value.kind == "2:1"
    dup = np.concatenate([lv[:1], lv])
    with pytest.raises(OA.LayoutError):
        OA.adapt((3, 3, 3), (1, 1, 1), dup, np.full(len(dup), 0.5), 1.0, 0.1, 3)
    hole = lv[1:]                                      # level 0 not covered
    with pytest.raises(OA.LayoutError):
        OA.adapt((3, 3, 3), (1, 1, 1), hole, np.full(len(hole), 0.5), 1.0, 0.1, 3)


def test_host_abi_adapt_rejects_invalid_input():
    import ctypes as Cc
    import os
    from paper_2512_08555_b200.mg import _LIB_PATH, load_library
    if not os.path.exists(_LIB_PATH):
        pytest.skip("libmg.so not built")
    lib = load_library()
    I32 = Cc.c_int32
    bb = (I32 * 3)(3, 3, 3)
    bc = (I32 * 6)(1, 1, 1, 1, 1, 1)
    for lv, code in ((_unbalanced_nest(), -3), (np.concatenate([_unbalanced_nest()[:1], _unbalanced_nest()]), -2),
                     (_unbalanced_nest()[1:], -2)):
        lv = np.ascontiguousarray(lv, dtype=np.int32)
        g = np.full(len(lv), 0.5)
        out = np.zeros((4096, 4), dtype=np.int32)
        n_out = I32()
        rc = lib.mg_adapt(bb, bc, 0, lv.ctypes.data_as(Cc.POINTER(I32)), len(lv),
                          g.ctypes.data_as(Cc.POINTER(Cc.c_double)), 1.0, 0.1, 3,
                          out.ctypes.data_as(Cc.POINTER(I32)), 4096, Cc.byref(n_out), None)
        assert rc == code, (rc, code)


# ------------------------------------------------------------- field transfer (A3)
def _transfer_pair(poly=None):
    from oracle import mg_oracle as MO
    dom = Lay.Domain((0.0, 0.0, 0.0), 1 / 64, (4, 4, 4), 16, (0, 1, 1))
    d = dict(origin=(0.0, 0.0, 0.0), h0=1 / 64, base_blocks=(4, 4, 4), B=16, bc=(0, 1, 1), order=4, smoother=1,
             omega=1.0, eta1=2, eta2=2, coarse_n=0)
    t = Lay.Tree(dom)
    for b in sorted(t.nodes[0]):
        if all(1 <= b[a] <= 2 for a in (1, 2)) and b[0] in (0, 1):
            t.refine(0, b)
    old_lv = t.leaves()
    t2 = Lay.Tree(dom)                      # adapted: x-block 0 coarsened, x-block 2 refined
    for b in sorted(t2.nodes[0]):
        if all(1 <= b[a] <= 2 for a in (1, 2)) and b[0] in (1, 2):
            t2.refine(0, b)
    new_lv = t2.leaves()
    return MO, d, old_lv, new_lv


def test_transfer_trilinear_exact_and_identity():
    """The transfer reproduces a trilinear field exactly on refined, kept and coarsened
    blocks (prolongation exactness + injection), and is the identity when the layout is
    unchanged.  (x is periodic: the refined region stays clear of the wrap, where a
    polynomial is not periodic.)"""
    MO, d, old_lv, new_lv = _transfer_pair()
    o_old = MO.Oracle(d, old_lv)
    fn = lambda x, y, z: 1.0 + 2.0 * x - y + 0.5 * z + 0.3 * x * y - 0.7 * y * z + 0.2 * x * y * z  # noqa: E731
    dom = Lay.Domain((0.0, 0.0, 0.0), 1 / 64, (4, 4, 4), 16, (0, 1, 1))
    o_old.set_solution(S.sample_on_leaves(dom, old_lv, fn))
    o_new = MO.Oracle(d, new_lv)
    o_new.transfer_from(o_old)
    want = S.sample_on_leaves(dom, new_lv, fn)
    assert np.abs(o_new.get_solution() - want).max() < 1e-13
    o_same = MO.Oracle(d, old_lv)
    o_same.transfer_from(o_old)
    assert np.array_equal(o_same.get_solution(), o_old.get_solution())
