"""GCN end to end on the GPU (gcn.cpp:22-33): bit-exact against the
reference's gcn_forward (f32 build) — ordered GEMM kernel, ReLU fused into the
first CBM product, both A_hat products through the CBM kernel."""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import assert_bitwise, golden_cbm, load_golden, oracle_arrays

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def test_dense_matmul_matches_reference_arithmetic():
    rng = np.random.default_rng(3)
    for m, k, n in ((1, 1, 1), (37, 53, 130), (300, 128, 256), (64, 256, 112)):
        a = rng.standard_normal((m, k)).astype(np.float32)
        a[rng.random((m, k)) < 0.2] = 0.0          # zero lhs entries are skipped
        b = rng.standard_normal((k, n)).astype(np.float32)
        assert_bitwise(P.dense_matmul(_t(a), _t(b)).cpu().numpy(), O.oracle_dense_matmul(a, b),
                       f"gemm {m}x{k}x{n}")


def test_gcn_golden_fixture_bitwise():
    g = load_golden("gcn_small")             # reference gcn_forward output
    c = golden_cbm(g)
    op = P.DeviceCbm(c, order_faithful=True)
    out = op.gcn_forward(_t(g["x"]), _t(g["w0"]), _t(g["w1"])).cpu().numpy()
    assert_bitwise(out, g["y"], "gcn_small")


@pytest.mark.parametrize("faithful", [True, False])
def test_gcn_cfg3_shape_scaled(faithful):
    """cfg[3] shape (communities of 500, 0.8 / 1e-4), scaled to 6000 nodes,
    f=128, hidden=256, classes=112, Glorot weights."""
    a = P.generate_graph("community", [6000, 500, 0.8, 1e-4], 0xC0F60003)
    c = P.build_cbm_normalized(a, 0, threads=8)
    x = P.generate_dense("normal", 6000, 128, 0xC0F61003)
    w0 = P.generate_dense("glorot", 128, 256, 0xC0F62003)
    w1 = P.generate_dense("glorot", 256, 112, 0xC0F62004)
    want = O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1)
    got = P.DeviceCbm(c, order_faithful=faithful).gcn_forward(_t(x), _t(w0), _t(w1)).cpu().numpy()
    if faithful:
        assert_bitwise(got, want, "gcn cfg3-shape")
    else:
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= 1e-5


def test_gcn_errors_mirror_reference():
    a = P.CsrBinaryMatrix.from_rows(3, [[1], [0, 2], [1]])
    plain = P.DeviceCbm(P.build_cbm(a, 0))
    x = torch.zeros((3, 4), device="cuda")
    w0 = torch.zeros((4, 2), device="cuda")
    w1 = torch.zeros((2, 2), device="cuda")
    with pytest.raises(ValueError, match="adjacency must be normalized"):
        plain.gcn_forward(x, w0, w1)
    norm = P.DeviceCbm(P.build_cbm_normalized(a, 0))
    with pytest.raises(ValueError, match="feature rows must match nodes"):
        norm.gcn_forward(torch.zeros((4, 4), device="cuda"), w0, w1)


def test_gcn_sharded_nccl_world1_bitwise():
    """gcn_forward_sharded through NCCL (one rank here; the same code path
    all-gathers the hidden slabs at N>1) equals gcn_forward bit for bit."""
    import os
    import torch.distributed as dist
    from paper_2409_02208_b200.sharding import gcn_forward_sharded
    a = P.generate_graph("community", [3000, 500, 0.8, 1e-4], 91)
    c = P.build_cbm_normalized(a, 0, threads=8)
    x = P.generate_dense("normal", 3000, 64, 92)
    w0 = P.generate_dense("glorot", 64, 96, 93)
    w1 = P.generate_dense("glorot", 96, 40, 94)
    op = P.DeviceCbm(c, order_faithful=True)
    want = op.gcn_forward(_t(x), _t(w0), _t(w1)).cpu().numpy()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        got = gcn_forward_sharded(op, _t(x), _t(w0), _t(w1)).cpu().numpy()
    finally:
        dist.destroy_process_group()
    assert_bitwise(got, want, "sharded gcn")
    assert_bitwise(got, O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1), "vs oracle")


@pytest.mark.parametrize("hid", [24, 48])
def test_gcn_narrow_hidden_default_mode(hid):
    """Default mode with a narrow hidden layer: the ReLU-fused Â product runs
    with lane groups (several deltas per warp instruction); 1e-5 normwise."""
    a = P.generate_graph("community", [3000, 300, 0.7, 2e-4], 151)
    c = P.build_cbm_normalized(a, 0, threads=8)
    x = P.generate_dense("normal", 3000, 40, 152)
    w0 = P.generate_dense("glorot", 40, hid, 153)
    w1 = P.generate_dense("glorot", hid, 7, 154)
    want = O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1)
    got = P.DeviceCbm(c).gcn_forward(_t(x), _t(w0), _t(w1)).cpu().numpy()
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= 1e-5
