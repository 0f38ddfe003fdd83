"""The restated generators (oracle/gen_oracle.c), which bench.py's reference arm
uses so it never loads the product library, draw exactly the product's
graphs and operands (csrc/graphs.cpp, cbm_b200_gen_dense) on every config's
generator kind."""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import bits

CASES = [
    ("community", [4096, 64, 0.5, 0.001], 0xC0F60000),
    ("community", [3001, 500, 0.8, 1e-3], 0xC0F60003),
    ("pa_triangle", [19717, 2, 0.3], 0xC0F60001),
    ("pa_triangle", [500, 3, 0.9], 11),
    ("clique_overlay", [23586, 120000, 2, 10, 1.1], 0xC0F60002),
    ("clique_overlay", [5000, 8000, 2, 16, 1.1], 0xC0F60004),
    ("random_binary", [40, 70, 0.2], 5),
]


@pytest.mark.parametrize("kind,params,seed", CASES)
def test_restated_graph_generators_match_the_product(kind, params, seed):
    a = P.generate_graph(kind, params, seed)
    n, ncols, rp, ci = O.oracle_gen_graph(kind, params, seed)
    assert (n, ncols) == (a.n_rows, a.n_cols)
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(ci, a.col_idx)


@pytest.mark.parametrize("kind,lo,hi", [("int", -8, 8), ("normal", 0, 0), ("glorot", 0, 0)])
def test_restated_dense_generators_match_the_product(kind, lo, hi):
    for rows, cols in ((1, 1), (37, 13), (1000, 64)):
        if kind == "glorot":
            got = O.oracle_gen_dense("glorot", rows, cols, 0xC0F62003)
            want = P.generate_dense("glorot", rows, cols, 0xC0F62003)
        else:
            got = O.oracle_gen_dense(kind, rows, cols, 0xC0F61004, lo, hi)
            want = P.generate_dense(kind, rows, cols, 0xC0F61004, lo, hi)
        assert np.array_equal(bits(got), bits(want)), (kind, rows, cols)
