"""Dense-block path (tcgen05 tensor cores for the columns a 128-row tile shares,
the streaming kernel for the cold entries on top) against the oracle.

Bars as for every default-mode path: bit-exact on integer X for binary
matrices (the tf32 hi/lo split of an integer is the integer itself, sums of
small integers are exact in any order); max|G-R|/max|R| <= 1e-5 otherwise.
"""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import assert_bitwise, normwise_err, oracle_arrays

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-5


def run(c, x, **opt):
    op = P.DeviceCbm(c, device=0, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    y = op.spmm(xt).cpu().numpy()
    info = op.info()
    op.close()
    return y, info


def community(n, size, p_in, p_out, seed):
    return P.generate_graph("community", [n, size, p_in, p_out], seed)


@pytest.mark.parametrize("d", [32, 33, 50, 64, 96, 128, 200, 256, 260])
def test_binary_integer_x_bitwise(d):
    a = community(1000, 100, 0.5, 0.01, 21)
    c = P.build_cbm(a, 0, 4)
    x = P.generate_dense("int", a.n_cols, d, 5 + d, -8, 8)
    got, info = run(c, x, dense=1)
    assert info["dense_active"] and info["dense_chunks"] > 0 and info["cold_entries"] > 0
    assert info["dense_entries"] + info["cold_entries"] == a.nnz
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), f"dense d={d}")


@pytest.mark.parametrize("d", [32, 128, 256])
def test_normalized_gaussian_normwise(d):
    a = community(1500, 120, 0.6, 0.005, 22)
    c = P.build_cbm_normalized(a, 0, 4)
    x = P.generate_dense("normal", a.n_cols, d, 7)
    got, info = run(c, x, dense=1)
    assert info["dense_active"]
    want = O.oracle_spmm(oracle_arrays(c), x)
    assert normwise_err(got, want) <= TOL
    # and against the exact product, as tight as the reference itself
    e = O.oracle_exact_spmm(a.row_ptr, a.col_idx, x, c.row_scale, add_identity=True)
    assert np.abs(got - e).max() / np.abs(e).max() <= 2e-6


def test_ragged_edges_leading_dimension_and_relu():
    # m not a multiple of 128, X and Y column slabs of wider buffers
    a = community(777, 60, 0.7, 0.02, 23)
    c = P.build_cbm_normalized(a, 0, 4)
    d = 72
    xw = P.generate_dense("normal", a.n_cols, 100, 8)
    want = O.oracle_spmm(oracle_arrays(c), np.ascontiguousarray(xw[:, 10:10 + d]))
    op = P.DeviceCbm(c, device=0, dense=1)
    xt = torch.from_numpy(xw).cuda()
    yw = torch.full((a.n_rows, 90), 7.0, device="cuda")
    op.spmm_into(xt[:, 10:10 + d], yw[:, 5:5 + d])
    got = yw.cpu().numpy()
    assert normwise_err(got[:, 5:5 + d], want) <= TOL
    assert np.all(got[:, :5] == 7.0) and np.all(got[:, 5 + d:] == 7.0)
    r = op.spmm(xt[:, 10:10 + d].contiguous(), relu=True).cpu().numpy()
    assert normwise_err(r, np.where(want < 0, np.float32(0), want)) <= TOL


def test_tiles_without_shared_columns_and_empty_rows():
    # a random sparse matrix: most tiles have no column shared by 3 rows
    rp, ci = O.oracle_random_binary(600, 5000, 0.001, 31)
    a = P.CsrBinaryMatrix(600, 5000, rp, ci)
    c = P.build_cbm(a, 0, 4)
    x = P.generate_dense("int", 5000, 64, 9, -8, 8)
    got, info = run(c, x, dense=1)
    assert info["dense_active"]
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), "sparse tiles")


def test_dense_min_threshold_moves_entries():
    a = community(1000, 100, 0.5, 0.01, 24)
    c = P.build_cbm(a, 0, 4)
    x = P.generate_dense("int", a.n_cols, 64, 10, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    seen = []
    for mc in (1, 3, 40, 200):
        got, info = run(c, x, dense=1, dense_min=mc)
        assert_bitwise(got, want, f"dense_min={mc}")
        seen.append(info["dense_entries"])
    assert seen[0] == a.nnz and seen[-1] == 0 and seen[0] >= seen[1] >= seen[2]


def test_auto_picks_dense_on_community_blocks_and_falls_back_narrow():
    # enough 128-row tiles with shared columns to fill the SMs (auto rule)
    a = community(24000, 400, 0.5, 1e-4, 25)
    c = P.build_cbm_normalized(a, 0, 4)
    op = P.DeviceCbm(c, device=0)
    assert op.info()["dense_active"]
    assert op.info()["dense_chunks"] >= 8 * 148
    x = P.generate_dense("normal", a.n_cols, 16, 11)     # d < 32: streaming kernel
    got = op.spmm(torch.from_numpy(x).cuda()).cpu().numpy()
    assert normwise_err(got, O.oracle_spmm(oracle_arrays(c), x)) <= TOL
    assert op.info()["launches_per_call"] == 1


def test_auto_keeps_small_matrices_off_the_dense_path():
    a = community(4096, 256, 0.6, 0.001, 27)
    c = P.build_cbm_normalized(a, 0, 4)
    assert not P.DeviceCbm(c, device=0).info()["dense_active"]


def test_order_faithful_never_takes_the_dense_path():
    a = community(1000, 100, 0.5, 0.01, 26)
    c = P.build_cbm_normalized(a, 0, 4)
    op = P.DeviceCbm(c, device=0, order_faithful=True)
    assert not op.info()["dense_active"]


def test_cfg0_full_size_dense_bitwise():
    from paper_2409_02208_b200.workloads import WORKLOADS
    wl = WORKLOADS["cfg0"]
    a = wl.graph()
    c = wl.build(a, 4)
    x = wl.operand(a.n_cols)
    got, info = run(c, x, dense=1)
    assert info["dense_active"]
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), "cfg0 dense")
