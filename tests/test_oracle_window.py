"""The oracle's window storage (levels on their block bounding box, oracle/mg_oracle.py
header) changes array indices only: with every level windowed the results equal the
whole-lattice oracle bit for bit, and a deep (5-level) cfg5-shaped layout contracts."""
import numpy as np
import pytest

from oracle import mg_oracle as MO
from tests.test_gpu_parity import _cfg


def _run(name, window_nodes, cycles=2, monkeypatch=None):
    monkeypatch.setattr(MO, "WINDOW_NODES", window_nodes)
    cfg, lv, f = _cfg(name)
    o = MO.Oracle(cfg, lv)
    o.set_rhs(f)
    o.vcycle(cycles)
    return o, o.get_solution(), o.residual_norm()


@pytest.mark.parametrize("name", ["puu2", "per_adapt", "ou_uu"])
def test_window_equals_whole_lattice(name, monkeypatch):
    o_full, u_full, r_full = _run(name, 1 << 40, monkeypatch=monkeypatch)
    o_win, u_win, r_win = _run(name, 0, monkeypatch=monkeypatch)
    assert any(not all(L.full) for L in o_win.levels[1:])       # something was windowed
    assert all(all(L.full) for L in o_full.levels)
    assert np.array_equal(u_full, u_win)
    assert r_full == r_win


def test_cfg5_shaped_layout_contracts():
    """5 AMR levels (cfg5 recipe, reduced torus): per-cycle contraction of the composite
    residual (P7: < 1, stable) on windowed levels."""
    cfg, lv, f = _cfg("cfg5_small")
    o = MO.Oracle(cfg, lv)
    assert len(o.levels) == 5 and any(not all(L.full) for L in o.levels)
    o.set_rhs(f)
    hist = []
    for _ in range(3):
        o.vcycle(1)
        hist.append(o.residual_norm()[1])
    assert hist[1] < 0.25 * hist[0] and hist[2] < 0.25 * hist[1], hist
