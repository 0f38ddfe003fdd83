"""Hub-row panel (the longest rows of a power-law matrix multiplied as one
tile on the tensor cores, everything else on the streaming kernel) against
the oracle.

Bars as for every default-mode path: bit-exact on integer X for binary
matrices; max|G-R|/max|R| <= 1e-5 otherwise.
"""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import assert_bitwise, normwise_err, oracle_arrays

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-5


def overlay(n, groups, hi, seed):
    # Zipf clique overlay (cfg[2] / cfg[4]'s generator): a few hub rows hold a
    # large share of the entries
    return P.generate_graph("clique_overlay", [n, groups, 2, hi, 1.1], seed)


def run(c, x, relu=False, **opt):
    op = P.DeviceCbm(c, device=0, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    y = op.spmm(xt, relu=relu).cpu().numpy()
    info = op.info()
    op.close()
    return y, info


@pytest.mark.parametrize("d", [32, 33, 50, 64, 100, 128, 256, 260])
def test_binary_integer_x_bitwise(d):
    a = overlay(6000, 20000, 8, 41)
    c = P.build_cbm(a, 8, 4)
    x = P.generate_dense("int", a.n_cols, d, 3 + d, -8, 8)
    got, info = run(c, x, hub=1)
    assert info["hub_active"] and info["hub_rows"] == 128 and info["hub_entries"] > 0
    assert info["nnz_delta"] == c.nnz
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), f"hub d={d}")


@pytest.mark.parametrize("d", [1, 4, 8, 16, 24])
def test_narrow_x_takes_the_hub_rows_own_operator(d):
    a = overlay(5000, 15000, 8, 42)
    c = P.build_cbm(a, 8, 4)
    x = P.generate_dense("int", a.n_cols, d, 5 + d, -8, 8)
    got, info = run(c, x, hub=1)
    assert info["hub_active"]
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), f"hub narrow d={d}")


@pytest.mark.parametrize("d", [16, 64, 256])
def test_normalized_gaussian_normwise(d):
    a = overlay(6000, 20000, 10, 43)
    c = P.build_cbm_normalized(a, 8, 4)
    x = P.generate_dense("normal", a.n_cols, d, 9)
    got, info = run(c, x, hub=1)
    assert info["hub_active"]
    want = O.oracle_spmm(oracle_arrays(c), x)
    assert normwise_err(got, want) <= TOL
    e = O.oracle_exact_spmm(a.row_ptr, a.col_idx, x, c.row_scale, add_identity=True)
    assert np.abs(got - e).max() / np.abs(e).max() <= 2e-6


def test_children_of_hub_rows_and_relu_and_leading_dimensions():
    # alpha = 0: deep chains, some of them hanging off the hub rows
    a = overlay(3000, 9000, 6, 44)
    c = P.build_cbm(a, 0, 4)
    d = 72
    xw = P.generate_dense("int", a.n_cols, 100, 8, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), np.ascontiguousarray(xw[:, 10:10 + d]))
    op = P.DeviceCbm(c, device=0, hub=1)
    assert op.info()["hub_active"]
    xt = torch.from_numpy(xw).cuda()
    yw = torch.full((a.n_rows, 90), 7.0, device="cuda")
    op.spmm_into(xt[:, 10:10 + d], yw[:, 5:5 + d])
    got = yw.cpu().numpy()
    assert_bitwise(np.ascontiguousarray(got[:, 5:5 + d]), want, "hub slab")
    assert np.all(got[:, :5] == 7.0) and np.all(got[:, 5 + d:] == 7.0)
    r = op.spmm(xt[:, 10:10 + d].contiguous(), relu=True).cpu().numpy()
    assert_bitwise(r, np.where(want < 0, np.float32(0), want), "hub relu")
    v = op.spmv(xt[:, 3].contiguous()).cpu().numpy()
    assert_bitwise(v.reshape(-1, 1), O.oracle_spmm(oracle_arrays(c),
                                                  np.ascontiguousarray(xw[:, 3:4])), "hub spmv")


def test_host_entry_and_repeated_calls():
    a = overlay(4000, 12000, 8, 45)
    c = P.build_cbm(a, 8, 4)
    x = P.generate_dense("int", a.n_cols, 256, 12, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    op = P.DeviceCbm(c, device=0, hub=1)
    for _ in range(3):
        assert_bitwise(op.spmm_host(x), want, "hub host entry")


def test_auto_rule_and_order_faithful():
    small = overlay(3000, 9000, 6, 46)
    c = P.build_cbm(small, 8, 4)
    assert not P.DeviceCbm(c, device=0).info()["hub_active"]          # too small for auto
    assert not P.DeviceCbm(c, device=0, hub=1, order_faithful=True).info()["hub_active"]
    big = overlay(120000, 600000, 10, 47)
    cb = P.csr_operator(big)
    plan = P.plan_hub(cb)
    op = P.DeviceCbm(cb, device=0)
    assert bool(op.info()["hub_active"]) == bool(plan["active"])
    x = P.generate_dense("int", big.n_cols, 64, 13, -8, 8)
    got = op.spmm(torch.from_numpy(x).cuda()).cpu().numpy()
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(cb), x), "hub auto")
