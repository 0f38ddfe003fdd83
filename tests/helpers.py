"""Shared test helpers (fixture loading, comparisons)."""
from __future__ import annotations

import glob
import os

import numpy as np

import oracle as O
import paper_2409_02208_b200 as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def golden_csr(g) -> P.CsrBinaryMatrix:
    return P.CsrBinaryMatrix(int(g["a_n_rows"]), int(g["a_n_cols"]), g["a_row_ptr"],
                             g["a_col_idx"])


def golden_cbm(g) -> P.CbmMatrix:
    norm = bool(int(g["normalized"]))
    return P.CbmMatrix(int(g["n_rows"]), int(g["n_cols"]), int(g["alpha"]), norm, g["parent"],
                       g["row_ptr"], g["col_idx"], g["values"],
                       g["row_scale"] if norm else None, g["topo_order"], g["branch_ptr"])


def oracle_arrays(c: P.CbmMatrix) -> O.RefCbmArrays:
    return O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized, c.parent, c.row_ptr,
                          c.col_idx, c.values, c.row_scale, c.topo_order, c.branch_ptr)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(got, want, what=""):
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    diff = np.nonzero(bits(got) != bits(want))
    n = diff[0].size
    assert n == 0, f"{what}: {n} of {got.size} elements differ in bits; first at {tuple(d[0] for d in diff)}: {got[tuple(d[0] for d in diff)]} vs {want[tuple(d[0] for d in diff)]}"


def normwise_err(got, want):
    """max|G-R| / max|R| (SURVEY §8d Gate 2)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.abs(want).max() if want.size else 0.0
    num = np.abs(got - want).max() if want.size else 0.0
    return num / den if den > 0 else num


def same_cbm(a: P.CbmMatrix, b) -> bool:
    ok = (np.array_equal(a.parent, b.parent) and np.array_equal(a.row_ptr, b.row_ptr)
          and np.array_equal(a.col_idx, b.col_idx)
          and np.array_equal(bits(a.values), bits(b.values)))
    if a.topo_order is not None and b.topo_order is not None:
        ok = ok and np.array_equal(a.topo_order, b.topo_order)
    if a.is_normalized:
        ok = ok and np.array_equal(bits(a.row_scale), bits(b.row_scale))
    return bool(ok)
