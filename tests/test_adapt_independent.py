"""Grid adaptation pinned by an independent formulation.

oracle/adapt.py and the host pass in libmg.so (mg_adapt) both walk leaf sets in the
same step order (reading A2).  This test restates the three rules of P:65 on dense
per-level block arrays — a different algorithm, written from the rules, not from
either implementation:

  refine:  every leaf with γ > ε_r below max_level is split into its 8 children
           ("refined into 8 finer blocks whenever ... γ above ε_r"), except blocks
           touching an unbounded face;
  coarsen: 8 sibling leaves, none refined, all γ < ε_c, revert to their parent
           when no block two levels finer than the parent lies in its 26-neighbourhood
           (the parent must keep 2:1 with the refined grid);
  balance: "two adjacent blocks cannot have a resolution jump larger than one level"
           (P:65): for every block at level m >= 2 the parents of its 26 neighbours
           must exist; processed from the finest level down (a block added at level
           m-1 can only impose requirements on level m-2), adding whole octets.

On layouts where the balance never has to refine a frozen block (periodic domains, or
refinement away from the unbounded faces) the result is unique — the minimal balanced
refinement — so all three implementations must return the same leaf set.
"""
import numpy as np
import pytest

from oracle import adapt as OA

OFF = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def _up(a):
    """level-l array -> level-(l+1) array (every child of a marked block)."""
    return a.repeat(2, 0).repeat(2, 1).repeat(2, 2)


def _down_any(a, f=2):
    """level-(l+k) array -> level-l array (some descendant marked), f = 2^k."""
    n = [s // f for s in a.shape]
    return a.reshape(n[0], f, n[1], f, n[2], f).any(axis=(1, 3, 5))


def _dilate26(a, per):
    """mark every block whose 26-neighbourhood (itself included) holds a marked block;
    periodic axes wrap, the others clip."""
    out = np.zeros_like(a)
    for o in OFF:
        s = a
        for ax in range(3):
            if o[ax] == 0:
                continue
            if per[ax]:
                s = np.roll(s, o[ax], axis=ax)
            else:
                t = np.zeros_like(s)
                if o[ax] > 0:
                    sl_dst = [slice(None)] * 3
                    sl_src = [slice(None)] * 3
                    sl_dst[ax] = slice(1, None)
                    sl_src[ax] = slice(0, -1)
                else:
                    sl_dst = [slice(None)] * 3
                    sl_src = [slice(None)] * 3
                    sl_dst[ax] = slice(0, -1)
                    sl_src[ax] = slice(1, None)
                t[tuple(sl_dst)] = s[tuple(sl_src)]
                s = t
        out |= s
    return out


def dense_adapt(base, bc, leaves, gamma, eps_r, eps_c, max_level):
    per = [int(b) == 0 for b in bc]
    L = max(max_level, int(max(lv[0] for lv in leaves))) + 1
    dims = [tuple(int(b) << l for b in base) for l in range(L + 2)]  # (x, y, z) per level
    leaf = [np.zeros(d, bool) for d in dims]
    gam = [np.full(d, np.nan) for d in dims]
    for (l, x, y, z), g in zip(leaves, gamma):
        leaf[l][x, y, z] = True
        gam[l][x, y, z] = g

    def frozen(l):
        f = np.zeros(dims[l], bool)
        for ax in range(3):
            if not per[ax]:
                sl = [slice(None)] * 3
                sl[ax] = 0
                f[tuple(sl)] = True
                sl[ax] = -1
                f[tuple(sl)] = True
        return f

    def exist_of(lf):
        ex = [a.copy() for a in lf]
        for l in range(len(ex) - 1, 0, -1):
            ex[l - 1] |= _down_any(ex[l])
        return ex

    # refine
    ref = [leaf[l] & (np.nan_to_num(gam[l], nan=-np.inf) > eps_r) & (l < max_level) & ~frozen(l)
           for l in range(L + 2)]
    leaf1 = [leaf[l] & ~ref[l] for l in range(L + 2)]
    for l in range(L + 1):
        leaf1[l + 1] |= _up(ref[l])
    ex1 = exist_of(leaf1)
    # coarsen
    leaf2 = [a.copy() for a in leaf1]
    for l in range(L + 1):
        kids = leaf[l + 1] & ~ref[l + 1] & (np.nan_to_num(gam[l + 1], nan=np.inf) < eps_c)
        n = dims[l]
        octet = kids.reshape(n[0], 2, n[1], 2, n[2], 2).all(axis=(1, 3, 5))
        deep = _down_any(ex1[l + 2], 4) if l + 2 < len(ex1) else np.zeros(n, bool)
        ok = octet & ~_dilate26(deep, per)
        leaf2[l] |= ok
        leaf2[l + 1] &= ~_up(ok)
    # balance, finest level first
    ex = exist_of(leaf2)
    for m in range(L + 1, 1, -1):
        need = _down_any(_dilate26(ex[m], per))  # level m-1: parents of the neighbours
        add = need & ~ex[m - 1]
        j = m - 1
        while add.any():
            par = _down_any(add)  # level j-1 blocks that must be refined
            if j - 1 == 0:
                assert not (par & frozen(0)).any(), "balance would refine a frozen block"
            ex[j] |= _up(par)  # whole octets
            add = par & ~ex[j - 1]
            j -= 1
    out = []
    for l in range(len(ex)):
        kids = _down_any(ex[l + 1]) if l + 1 < len(ex) else np.zeros(dims[l], bool)
        lf = ex[l] & ~kids
        for x, y, z in zip(*np.nonzero(lf)):
            out.append((l, int(x), int(y), int(z)))
    return np.array(sorted(out), dtype=np.int32).reshape(-1, 4)


def _layouts():
    """valid inputs: start from the base grid and refine random blocks (with γ = ∞)
    through the dense rules themselves, then draw fresh γ for the cases."""
    rng = np.random.default_rng(11)
    cases = []
    for base, bc, mx in [((2, 2, 2), (0, 0, 0), 3), ((4, 2, 2), (0, 0, 0), 3), ((3, 3, 2), (0, 0, 0), 2),
                         ((6, 6, 6), (0, 1, 1), 2), ((6, 5, 6), (1, 1, 1), 2)]:
        lv = [(0, x, y, z) for z in range(base[2]) for y in range(base[1]) for x in range(base[0])]
        per = [b == 0 for b in bc]
        for _ in range(2):
            g = []
            for (l, x, y, z) in lv:
                c = (x, y, z)
                near_face = any(not per[a] and (c[a] <= 1 or c[a] >= (base[a] << l) - 2) for a in range(3))
                g.append(np.inf if (not near_face and rng.random() < 0.3) else 0.0)
            lv = [tuple(r) for r in dense_adapt(base, bc, lv, g, 1.0, -1.0, mx)]
        for seed in range(3):
            gamma = rng.random(len(lv))
            # keep the refinement two blocks away from unbounded faces (no frozen block in
            # the balance: the conflict-free case, where the result is unique)
            for n, (l, x, y, z) in enumerate(lv):
                c = (x, y, z)
                if any(not per[a] and (c[a] <= 2 or c[a] >= (base[a] << l) - 3) for a in range(3)):
                    gamma[n] = min(gamma[n], 0.5)
            cases.append((base, bc, lv, gamma, 0.8, 0.3, mx))
    return cases


CASES = _layouts()


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_adapt_equals_dense_rules(i):
    base, bc, lv, gamma, er, ec, mx = CASES[i]
    try:
        want = dense_adapt(base, bc, lv, gamma, er, ec, mx)
    except AssertionError:
        pytest.skip("balance meets a frozen block: outcome rule-dependent (reading A2)")
    got, _ = OA.adapt(base, bc, np.array(lv, dtype=np.int32), gamma, er, ec, mx)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_host_mg_adapt_equals_dense_rules(i):
    from paper_2512_08555_b200 import adapt
    base, bc, lv, gamma, er, ec, mx = CASES[i]
    try:
        want = dense_adapt(base, bc, lv, gamma, er, ec, mx)
    except AssertionError:
        pytest.skip("balance meets a frozen block: outcome rule-dependent (reading A2)")
    cfg = {"base_blocks": base, "bc": bc}
    got, _ = adapt(cfg, np.array(lv, dtype=np.int32), gamma, er, ec, mx)
    assert np.array_equal(got, want)


def test_dense_rules_balance_ring():
    """the dense rules on a closed form: a periodic 2^3 base grid refined three times at
    the origin block.  The 8 level-3 leaves need the level-2 blocks {7, 0, 1}^3 (parents of
    their 26 neighbours, wrapped); those need the level-1 blocks {3, 0, 1}^3, so every
    level-0 block is refined (64 level-1 blocks), the level-1 blocks {3, 0}^3 are refined
    (level-2 blocks {6, 7, 0, 1}^3) and level-2 block (0, 0, 0) holds the level-3 leaves:
    8 + 63 + 56 = 127 leaves."""
    base, bc = (2, 2, 2), (0, 0, 0)
    lv = [(0, x, y, z) for z in range(2) for y in range(2) for x in range(2)]
    for _ in range(3):
        g = [np.inf if r[1:] == (0, 0, 0) else 0.0 for r in lv]
        lv = [tuple(int(v) for v in r) for r in dense_adapt(base, bc, lv, g, 1.0, -1.0, 3)]
    by = {l: {r[1:] for r in lv if r[0] == l} for l in range(4)}
    assert len(by[3]) == 8 and len(by[2]) == 63 and len(by[1]) == 56 and len(by[0]) == 0
    ring = {(x, y, z) for x in (6, 7, 0, 1) for y in (6, 7, 0, 1) for z in (6, 7, 0, 1)}
    assert by[2] == ring - {(0, 0, 0)}
    # the same through the oracle and the host pass (γ refines only the origin chain)
    lv0 = [(0, x, y, z) for z in range(2) for y in range(2) for x in range(2)]
    from paper_2512_08555_b200 import adapt
    a, b = lv0, lv0
    for _ in range(3):
        ga = [np.inf if r[1:] == (0, 0, 0) else 0.0 for r in a]
        gb = [np.inf if r[1:] == (0, 0, 0) else 0.0 for r in b]
        a = [tuple(r) for r in OA.adapt(base, bc, np.array(a, dtype=np.int32), np.array(ga), 1.0, -1.0, 3)[0]]
        b = [tuple(r) for r in adapt({"base_blocks": base, "bc": bc}, np.array(b, dtype=np.int32), np.array(gb),
                                     1.0, -1.0, 3)[0]]
    assert sorted(a) == sorted(lv) == sorted(b)
