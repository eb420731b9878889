"""C-ABI argument checking that needs no GPU (include/mg.h error conventions): calls
rejected before any CUDA work return the documented codes."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2512_08555_b200.mg import _LIB_PATH, MG_OK

MG_ERR_ARG = -1


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_LIB_PATH):
        pytest.skip("libmg.so not built")
    from paper_2512_08555_b200.mg import load_library
    return load_library()


def test_detail_rejects_bad_arguments(lib):
    p = C.c_void_p(1)   # never dereferenced: the checks come first
    assert lib.mg_detail(None, 0, 16, 4, None, None) == MG_OK               # nothing to do
    assert lib.mg_detail(None, 3, 16, 4, None, None) == MG_ERR_ARG          # null buffers
    assert lib.mg_detail(p, 3, 12, 4, p, None) == MG_ERR_ARG                # B not in {8, 16}
    assert lib.mg_detail(p, 3, 16, 3, p, None) == MG_ERR_ARG                # W odd
    assert lib.mg_detail(p, 3, 8, 6, p, None) == MG_ERR_ARG                 # 2(W-1) > B-2
    assert lib.mg_detail(p, -1, 16, 4, p, None) == MG_ERR_ARG


def test_adapt_reports_capacity_and_bad_input(lib):
    I32 = C.c_int32
    bb = (I32 * 3)(2, 2, 2)
    bc = (I32 * 6)(0, 0, 0, 0, 0, 0)
    lv = np.array([(0, i, j, k) for k in range(2) for j in range(2) for i in range(2)], dtype=np.int32)
    g = np.ones(8)
    n_out, n_sup = I32(), I32()
    out = np.zeros((4, 4), dtype=np.int32)                                   # too small for 64 leaves
    rc = lib.mg_adapt(bb, bc, 0, lv.ctypes.data_as(C.POINTER(I32)), 8, g.ctypes.data_as(C.POINTER(C.c_double)),
                      0.5, 0.0, 1, out.ctypes.data_as(C.POINTER(I32)), 4, C.byref(n_out), C.byref(n_sup))
    assert rc == MG_ERR_ARG and n_out.value == 64                          # every block refined once
    bad = (I32 * 3)(0, 2, 2)
    rc = lib.mg_adapt(bad, bc, 0, lv.ctypes.data_as(C.POINTER(I32)), 8, g.ctypes.data_as(C.POINTER(C.c_double)),
                      0.5, 0.0, 1, out.ctypes.data_as(C.POINTER(I32)), 4, C.byref(n_out), None)
    assert rc == MG_ERR_ARG
