"""The C-ABI library loads and exports every symbol include/cbm_b200.h
declares; host-side argument validation works without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2409_02208_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "cbm_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cbm_b200_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(P.library_path)
    syms = declared_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(P.EXPORTED_SYMBOLS)


def test_library_is_sm100a_only():
    blob = open(P.library_path, "rb").read()
    assert b"sm_100a" in blob


def test_upload_rejects_malformed_views_before_touching_the_device():
    c = P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[0, 1], [0, 1], [2]]), 0)
    bad = P.CbmMatrix(c.n_rows, c.n_cols, c.alpha, False, c.parent.copy(), c.row_ptr, c.col_idx,
                      c.values * 2)
    with pytest.raises(ValueError, match="must be \\+1 or -1"):
        P.DeviceCbm(bad)
    cyc = P.CbmMatrix(c.n_rows, c.n_cols, c.alpha, False, np.array([1, 0, 0xFFFFFFFF]),
                      c.row_ptr, c.col_idx, c.values)
    with pytest.raises(ValueError, match="cycle"):
        P.DeviceCbm(cyc)
    selfp = P.CbmMatrix(c.n_rows, c.n_cols, c.alpha, False, np.array([0, 0, 0xFFFFFFFF]),
                        c.row_ptr, c.col_idx, c.values)
    with pytest.raises(ValueError, match="bad parent link at row 0"):
        P.DeviceCbm(selfp)


def test_generators_are_seeded_and_reproducible():
    a = P.generate_graph("community", [512, 64, 0.5, 0.01], 3)
    b = P.generate_graph("community", [512, 64, 0.5, 0.01], 3)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    d = a.dense()
    assert np.array_equal(d, d.T) and np.all(np.diag(d) == 0)   # symmetric, no self-loops
    x = P.generate_dense("int", 100, 7, 1, -8, 8)
    assert x.min() >= -8 and x.max() <= 8 and np.all(x == np.round(x))
    g = P.generate_dense("normal", 1000, 100, 2)
    assert abs(g.mean()) < 0.02 and abs(g.std() - 1) < 0.02


def test_uniform_dense_matches_reference_random_dense():
    import oracle as O
    got = P.generate_dense("uniform", 13, 7, 42, -1.0, 1.0)
    want = O.oracle_random_dense(13, 7, -1.0, 1.0, 42)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_random_binary_generator_matches_reference_stream():
    import oracle as O
    a = P.generate_graph("random_binary", [20, 30, 0.3], 77)
    rp, ci = O.oracle_random_binary(20, 30, 0.3, 77)
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)


def test_upload_rejects_unknown_kernel_option():
    c = P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[0, 1], [0, 1], [2]]), 0)
    with pytest.raises(ValueError, match="kernel must be"):
        P.DeviceCbm(c, kernel="register")
    opt = P._Options()
    P._lib.cbm_b200_default_options(ctypes.byref(opt))
    opt.kernel = 2
    h = ctypes.c_void_p()
    view = c._view()
    rc = P._lib.cbm_b200_upload(ctypes.byref(view), ctypes.byref(opt), ctypes.byref(h))
    assert rc == 1 and b"options.kernel" in P._lib.cbm_b200_last_error()
    assert not h.value
