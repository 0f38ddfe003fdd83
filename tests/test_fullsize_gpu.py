"""Full-size parity at the BASELINE.json configs the bench measures, checked
directly against the reference compiled from its sources (oracle/_ref,
kernels.cpp:105-123 spmm_into, gcn.cpp:22-33 gcn_forward) and against the C
restatement (oracle/liboracle.so).

The reference pins its own kernel the same way: staged == dense within
tolerance on random suites, sequential == staged bitwise
(test_kernels.cpp:75-144), and acceptance criterion 8 (acceptance.cpp:247-262).
Bars (north_star): the default mode (the mode every bench number uses: split
rows, flattening, lane groups, the tiled path, fused FMAs) is bit-exact on
integer X for binary matrices and within max|G-R|/max|R| <= 1e-5 otherwise;
the order-faithful mode is bit-identical for any X.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import assert_bitwise, normwise_err, oracle_arrays
from paper_2409_02208_b200.workloads import WORKLOADS

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(),
                                                  reason="oracle/_ref not built")]
torch = pytest.importorskip("torch")

TOL = 1e-5
THREADS = os.cpu_count() or 1


def ref_cbm(c):
    return O.RefCbm.from_arrays(oracle_arrays(c))


def run(c, x, **opt):
    op = P.DeviceCbm(c, device=0, **opt)
    y = op.spmm(torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()
    info = op.info()
    op.close()
    return y, info


@pytest.fixture(scope="module")
def cfg2():
    wl = WORKLOADS["cfg2"]
    a = wl.graph()
    return wl, a, wl.build(a, THREADS)


@pytest.fixture(scope="module")
def cfg3():
    wl = WORKLOADS["cfg3"]
    a = wl.graph()
    return wl, a, wl.build(a, THREADS)


@pytest.fixture(scope="module")
def cfg4():
    wl = WORKLOADS["cfg4_b256"]
    a = wl.graph()
    return wl, a, wl.build(a, THREADS)


def test_cfg2_full_size_default_and_faithful(cfg2):
    wl, a, c = cfg2
    assert a.n_rows == 235868
    x = wl.operand(a.n_cols)                       # N(0,1), d = 128
    want = ref_cbm(c).spmm(x, THREADS)
    got, info = run(c, x)                          # auto: hub-row panel + streaming kernel
    assert info["hub_active"] and info["hub_rows"] == 128
    assert normwise_err(got, want) <= TOL
    got_s, info_s = run(c, x, hub=0)               # streaming kernel alone
    assert not info_s["hub_active"]
    assert normwise_err(got_s, want) <= TOL
    got_f, _ = run(c, x, order_faithful=True)
    assert_bitwise(got_f, want, "cfg2 order-faithful vs reference spmm_into")
    # the restatement agrees with the compiled reference at full size too
    assert_bitwise(O.oracle_spmm(oracle_arrays(c), x), want, "cfg2 oracle vs reference")


def test_cfg2_full_size_integer_x_bitwise(cfg2):
    wl, a, c = cfg2
    x = P.generate_dense("int", a.n_cols, 64, 0xC0F61102, -8, 8)
    want = ref_cbm(c).spmm(x, THREADS)
    got, info = run(c, x)                           # default mode: hub panel on the tensor cores
    assert info["hub_active"]
    assert_bitwise(got, want, "cfg2 default mode, integer X")
    got, _ = run(c, x, hub=0)                       # lane groups at d=64
    assert_bitwise(got, want, "cfg2 default mode without the hub panel, integer X")


def test_cfg3_full_size_default_and_faithful(cfg3):
    wl, a, c = cfg3
    assert a.n_rows == 132534 and c.is_normalized
    x = wl.operand(a.n_cols)                       # N(0,1), d = 256
    want = ref_cbm(c).spmm(x, THREADS)
    got, info = run(c, x)                          # auto: the dense-block path on cfg3
    assert info["dense_active"]
    assert normwise_err(got, want) <= TOL
    got_t, info_t = run(c, x, dense=0)             # the tiled path
    assert info_t["tile_active"]
    assert normwise_err(got_t, want) <= TOL
    got_s, _ = run(c, x, dense=0, tile=0)          # streaming kernel, default mode
    assert normwise_err(got_s, want) <= TOL
    got_f, _ = run(c, x, order_faithful=True)
    assert_bitwise(got_f, want, "cfg3 order-faithful vs reference spmm_into")


def test_cfg3_binary_integer_x_bitwise(cfg3):
    # the same graph as a binary CBM: integer X sums are exact in any order
    wl, a, _ = cfg3
    c = P.build_cbm(a, 0, THREADS)
    x = P.generate_dense("int", a.n_cols, 256, 0xC0F61103, -8, 8)
    want = ref_cbm(c).spmm(x, THREADS)
    got, info = run(c, x)
    assert_bitwise(got, want, "cfg3 binary, default mode, integer X")


def test_cfg3_gcn_forward_full_size(cfg3):
    """configs[3]: 2-layer GCN, W0 128x256 and W1 256x112 (Glorot, seeded)."""
    wl, a, c = cfg3
    x = P.generate_dense("normal", a.n_cols, 128, 0xC0F61003)
    w0 = P.generate_dense("glorot", 128, 256, 0xC0F62003)
    w1 = P.generate_dense("glorot", 256, 112, 0xC0F62103)
    want = ref_cbm(c).gcn_forward(x, w0, w1, THREADS)
    for faithful in (True, False):
        op = P.DeviceCbm(c, device=0, order_faithful=faithful)
        got = op.gcn_forward(torch.from_numpy(x).cuda(), torch.from_numpy(w0).cuda(),
                             torch.from_numpy(w1).cuda()).cpu().numpy()
        op.close()
        if faithful:
            assert_bitwise(got, want, "cfg3 GCN order-faithful vs reference gcn_forward")
        else:
            assert normwise_err(got, want) <= TOL


def test_cfg4_full_size_binary(cfg4):
    """configs[4] (the metric's scaling sweep), binary, at the bench's d=256
    (N(0,1), normwise) and at d=32 on integer X (bitwise)."""
    wl, a, c = cfg4
    assert a.n_rows == 2449029
    rc = ref_cbm(c)
    x = wl.operand(a.n_cols)
    want = rc.spmm(x, THREADS)
    got, info = run(c, x)
    assert info["hub_active"] and info["hub_entries"] > 20_000_000
    # the hub row has ~1.4M entries: the reference's sequential f32 sum is
    # itself ~3e-5 (normwise) from the exact product, so the device result is
    # judged against the f64 product on a column sample when it differs from
    # the reference by more than the tolerance (oracle.judge_parity)
    j = O.judge_parity(got, want, TOL, lambda cols: O.oracle_exact_spmm(
        a.row_ptr, a.col_idx, x[:, cols]))
    assert j["ok"], j
    if "exact_err" in j:
        assert j["exact_err"] <= j["reference_exact_err"], j
    del got, want, x
    xi = P.generate_dense("int", a.n_cols, 32, 0xC0F61104, -8, 8)
    got, _ = run(c, xi)
    assert_bitwise(got, rc.spmm(xi, THREADS), "cfg4 binary, integer X, d=32")


# ---- the oracle's pins, re-run on the GPU box (the driver's -m gpu set) ----
def test_oracle_pins_rerun_on_gpu_box():
    import test_oracle as T
    T.test_golden_fixture_set_present()
    T.test_known_answers_in_golden()
    for name in T.NAMES:
        T.test_oracle_matches_golden(name)
    T.test_restated_generators_match_reference_streams()
    for normalized in (False, True):
        T.test_oracle_matches_reference_random_suite(normalized)
    T.test_oracle_csr_baseline_matches_reference()


def test_builder_pins_rerun_on_gpu_box():
    """The builder against the compiled reference (test_builder.py), re-run
    where the driver runs the -m gpu set."""
    import test_builder as B
    for name in B.NAMES:
        B.test_builder_matches_golden(name)
    for normalized in (False, True):
        B.test_builder_matches_reference_acceptance_suite(normalized)
    for name in dir(B):
        fn = getattr(B, name)
        if name.startswith("test_") and callable(fn) and fn.__code__.co_argcount == 0:
            fn()
