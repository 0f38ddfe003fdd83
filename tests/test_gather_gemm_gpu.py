"""Fused all-gather + GEMM of the multi-GPU GCN (cbm_b200_gemm_parts, CUDA IPC;
DESIGN.md §7).

* The part-wise GEMM on one device equals dense_matmul of the concatenated
  operand bit for bit (ordered) or within 1e-5 (FFMA), with several outputs.
* gcn_forward_sharded(fused=True) over NCCL at world 1 equals gcn_forward.
* Two processes on the one GPU of this box, each its own rank (gloo for the
  handle exchange and barriers), map each other's Z slab and output buffer
  through CUDA IPC and run the fused kernel: both hold the reference's
  gcn_forward bits. The kernels never wait on each other (host barriers only),
  so sharing the GPU does not change what is tested: the IPC mapping, the
  peer-pointer reads and the fan-out stores.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import assert_bitwise, normwise_err, oracle_arrays

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.mark.parametrize("widths", [[40], [12, 12, 16], [8, 4, 4, 8, 16, 8, 4, 12]])
@pytest.mark.parametrize("n", [7, 112, 300])
def test_gemm_parts_equals_concatenated_gemm(widths, n):
    m = 1000
    rng = np.random.default_rng(sum(widths) + n)
    zs = [rng.standard_normal((m, w)).astype(np.float32) for w in widths]
    zs[0][rng.random((m, widths[0])) < 0.3] = 0.0  # zero lhs entries are skipped
    b = rng.standard_normal((sum(widths), n)).astype(np.float32)
    full = np.ascontiguousarray(np.concatenate(zs, axis=1))
    want = P.dense_matmul(_t(full), _t(b)).cpu().numpy()
    assert_bitwise(want, O.oracle_dense_matmul(full, b), "dense_matmul vs oracle")
    parts = [_t(z) for z in zs]
    ld = n + 5
    outs = [torch.full((m, ld), -1.0, device="cuda") for _ in range(3)]
    P.gemm_parts(parts, widths, m, _t(b), outs, ld, ordered=True)
    torch.cuda.synchronize()
    for o in outs:
        assert_bitwise(o[:, :n].cpu().numpy(), want, "ordered parts")
        assert (o[:, n:] == -1.0).all()
    fast = [torch.empty((m, n), device="cuda")]
    P.gemm_parts(parts, widths, m, _t(b), fast, n, ordered=False)
    torch.cuda.synchronize()
    assert normwise_err(fast[0].cpu().numpy(), want) <= 1e-5


def test_dense_matmul_nonfinite_rhs_and_zero_lhs():
    """dense.cpp:42 skips zero lhs entries: 0 * inf must not turn into NaN,
    while a nonzero lhs times inf must (k-steps with a non-finite B row take the
    per-entry skip)."""
    rng = np.random.default_rng(5)
    m, k, n = 300, 37, 70
    a = rng.standard_normal((m, k)).astype(np.float32)
    a[rng.random((m, k)) < 0.4] = 0.0
    a[:, 3] = 0.0
    b = rng.standard_normal((k, n)).astype(np.float32)
    b[3, 5] = np.inf
    b[3, 6] = np.nan
    b[20, 7] = -np.inf
    want = O.oracle_dense_matmul(a, b)
    got = P.dense_matmul(_t(a), _t(b)).cpu().numpy()
    assert_bitwise(got, want, "nonfinite rhs")
    assert np.isfinite(got[:, 5]).all() or not np.isfinite(want[:, 5]).all()


def _gcn_inputs():
    a = P.generate_graph("community", [3000, 500, 0.8, 1e-4], 91)
    c = P.build_cbm_normalized(a, 0, threads=8)
    x = P.generate_dense("normal", 3000, 64, 92)
    w0 = P.generate_dense("glorot", 64, 96, 93)
    w1 = P.generate_dense("glorot", 96, 40, 94)
    return c, x, w0, w1


def test_fused_gcn_nccl_world1_bitwise():
    import torch.distributed as dist
    from paper_2409_02208_b200.sharding import gcn_forward_sharded
    c, x, w0, w1 = _gcn_inputs()
    op = P.DeviceCbm(c, order_faithful=True)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        got = gcn_forward_sharded(op, _t(x), _t(w0), _t(w1), fused=True).cpu().numpy()
    finally:
        dist.destroy_process_group()
    assert_bitwise(got, O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1), "fused world 1")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, q, faithful):
    import torch.distributed as dist
    from paper_2409_02208_b200.sharding import gcn_forward_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, x, w0, w1 = _gcn_inputs()
        op = P.DeviceCbm(c, order_faithful=faithful)
        got = gcn_forward_sharded(op, _t(x), _t(w0), _t(w1), fused=True).cpu().numpy()
        q.put((rank, got))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("faithful", [True, False])
def test_fused_gcn_two_processes_ipc(faithful):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, faithful)) for r in range(2)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=300) for _ in range(2))
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    c, x, w0, w1 = _gcn_inputs()
    want = O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1)
    for r in range(2):
        if faithful:
            assert_bitwise(results[r], want, f"rank {r}")
        else:
            assert normwise_err(results[r], want) <= 1e-5
    assert np.array_equal(results[0].view(np.uint32), results[1].view(np.uint32))
