"""Host builder parity: our build_cbm / build_cbm_normalized reproduce the
reference builder (proj/src/builder.cpp) field for field."""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import golden_cbm, golden_csr, golden_names, load_golden, same_cbm

NAMES = golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_builder_matches_golden(name):
    g = load_golden(name)
    a = golden_csr(g)
    want = golden_cbm(g)
    build = P.build_cbm_normalized if want.is_normalized else P.build_cbm
    got = build(a, want.alpha, threads=2)
    assert same_cbm(got, want), name
    assert np.array_equal(got.branch_ptr, want.branch_ptr)
    assert list(P.count_scalar_ops(got)) == g["ops"].tolist()


def _ref_vs_ours(a_ref, alpha, normalized, threads=3):
    m, n, rp, ci = a_ref.arrays()
    want = O.RefCbm.build(a_ref, alpha, 1, normalized).arrays()
    build = P.build_cbm_normalized if normalized else P.build_cbm
    got = build(P.CsrBinaryMatrix(m, n, rp, ci), alpha, threads)
    return same_cbm(got, want) and np.array_equal(got.branch_ptr, want.branch_ptr)


@pytest.mark.parametrize("normalized", [False, True])
def test_builder_matches_reference_acceptance_suite(normalized):
    """acceptance.cpp:57-70 instances (first 120) x alpha {0,1,2,4,8}."""
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    rng = np.random.default_rng(7)
    for k in range(120):
        n = int(rng.integers(1, 65))
        m = n if normalized else int(rng.integers(1, 65))
        dens = float(rng.uniform(0.05, 0.5))
        a = O.RefCsr.random_binary(m, n, dens, 0xA0000 + k)
        for alpha in (0, 1, 2, 4, 8):
            assert _ref_vs_ours(a, alpha, normalized), (k, alpha)


def test_builder_matches_reference_structured_graphs():
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    for a in (O.RefCsr.community_graph(50, 40, 40, 1, 0xC0FFEE),
              O.RefCsr.citation_graph(2708, 10556, 0xC04A)):
        for alpha in (0, 4):
            assert _ref_vs_ours(a, alpha, False)
            assert _ref_vs_ours(a, alpha, True)


def test_builder_cfg0_full_size_matches_reference():
    """cfg[0] (n = 4096) at full size: our builder == reference builder."""
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    a = P.generate_graph("community", [4096, 64, 0.5, 0.001], 0xC0F60000)
    ra = O.RefCsr.from_arrays(a.n_rows, a.n_cols, a.row_ptr, a.col_idx)
    assert _ref_vs_ours(ra, 0, False, threads=8)


def test_builder_thread_count_independent():
    a = P.generate_graph("pa_triangle", [3000, 2, 0.3], 5)
    c1 = P.build_cbm_normalized(a, 0, threads=1)
    for t in (2, 8):
        assert same_cbm(P.build_cbm_normalized(a, 0, threads=t), c1)


def test_known_answers():
    # test_kernels.cpp:146-176: worked example, star chain, zero matrix
    a = P.CsrBinaryMatrix.from_rows(3, [[0, 1], [0, 1]])
    c = P.build_cbm(a, 0)
    assert P.count_scalar_ops(c) == (2, 1)
    assert c.row_ptr[2] - c.row_ptr[1] == 0
    eye = P.CsrBinaryMatrix.from_rows(4, [[0], [1], [2], [3]])
    assert P.count_scalar_ops(P.build_cbm(eye, 0)) == (4, 0)
    zero = P.CsrBinaryMatrix.from_rows(3, [[], []])
    assert P.count_scalar_ops(P.build_cbm(zero, 0)) == (0, 0)


def test_scalar_op_bound():
    """test_kernels.cpp:165-176: multiply_adds + update_adds <= nnz(A)."""
    rng = np.random.default_rng(200)
    for seed in range(200, 240):
        m, n = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        rp, ci = O.oracle_random_binary(m, n, float(rng.uniform(0.05, 0.5)), seed)
        a = P.CsrBinaryMatrix(m, n, rp, ci)
        for alpha in (0, 1, 2, 4, 8):
            assert sum(P.count_scalar_ops(P.build_cbm(a, alpha))) <= a.nnz


def test_builder_errors_mirror_reference():
    rect = P.CsrBinaryMatrix.from_rows(3, [[0], [1]])
    with pytest.raises(ValueError, match="must be square"):
        P.build_cbm_normalized(rect, 0)
    iso = P.CsrBinaryMatrix.from_rows(2, [[1], []])
    with pytest.raises(ValueError, match="zero degree at row 1"):
        P.build_cbm_normalized(iso, 0, degree_mode="original")
    bad = P.CsrBinaryMatrix(2, 2, np.array([0, 2, 3], np.uint64), np.array([1, 0, 1], np.uint32))
    with pytest.raises(ValueError, match="not strictly increasing"):
        P.build_cbm(bad, 0)
    oob = P.CsrBinaryMatrix(1, 2, np.array([0, 1], np.uint64), np.array([5], np.uint32))
    with pytest.raises(ValueError, match="out of range"):
        P.build_cbm(oob, 0)


@pytest.mark.parametrize("kind,params,normalized", [
    ("community", [3000, 500, 0.8, 1e-3], True),        # cascading contractions (cfg[3] shape)
    ("community", [4096, 64, 0.5, 0.001], False),       # cfg[0] shape
    ("pa_triangle", [5000, 2, 0.3], True),              # cfg[1] shape
    ("clique_overlay", [4000, 15000, 2, 10, 1.1], False),  # cfg[2] shape, scaled
])
def test_heap_edmonds_equals_round_synchronous(kind, params, normalized):
    """The mergeable-heap Edmonds (default) selects exactly the reference's
    round-synchronous contraction result (restated in min_arborescence)."""
    a = P.generate_graph(kind, params, 11)
    build = P.build_cbm_normalized if normalized else P.build_cbm
    for alpha in (0, 4):
        h = build(a, alpha, threads=8, arborescence="heap")
        r = build(a, alpha, threads=8, arborescence="rounds")
        assert same_cbm(h, r)
        assert h.build_stats["rounds"] == r.build_stats["rounds"]


def test_heap_edmonds_matches_reference_on_community_cascade():
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    a = P.generate_graph("community", [1500, 500, 0.8, 1e-3], 3)
    ra = O.RefCsr.from_arrays(a.n_rows, a.n_cols, a.row_ptr, a.col_idx)
    assert _ref_vs_ours(ra, 0, True, threads=8)
