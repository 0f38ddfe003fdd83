"""Column sharding of Y = A X across GPUs.

Every operation of the reference multiply (proj/src/kernels.cpp:27-62) acts
on one feature column j independently, so rank r of N holds a full replica of
the uploaded CBM and multiplies its own contiguous column slab of X; the
slabs of Y are bit-identical to the corresponding columns of the 1-GPU
result and no collective is needed for A.X itself. Slabs are multiples of 4
columns (16-byte rows for the LDG.128 lanes) where the width allows.
"""
from __future__ import annotations

from . import column_slab as _native_slab


def column_slab(d: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) columns of `rank`: contiguous, balanced in units of 4 columns
    (the library's cbm_b200_column_slab, so every rank and the single-process
    cbm_b200_spmm_sharded agree on the partition)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_slab: bad rank/world")
    return _native_slab(d, world, rank)


def all_slabs(d: int, world: int) -> list[tuple[int, int]]:
    return [column_slab(d, world, r) for r in range(world)]


class _DeviceCompute:
    """The product's compute for one rank: the reference-exact GEMM and the
    CBM multiply (ReLU fused into the epilogue) on this rank's GPU."""

    def __init__(self, op):
        self.op = op

    def matmul(self, a, b):
        from . import dense_matmul
        return dense_matmul(a, b)

    def spmm(self, x, relu=False):
        return self.op.spmm(x.contiguous(), relu=relu)


def _gather_columns(local, slabs, rank, group):
    """All-gather column slabs (n x w_r each) into one row-major n x d tensor."""
    import torch
    import torch.distributed as dist
    n = local.shape[0]
    wmax = max(hi - lo for lo, hi in slabs)
    send = torch.zeros((n, wmax), dtype=local.dtype, device=local.device)
    send[:, :local.shape[1]] = local
    recv = [torch.empty_like(send) for _ in slabs]
    dist.all_gather(recv, send, group=group)
    full = torch.empty((n, slabs[-1][1]), dtype=local.dtype, device=local.device)
    for (lo, hi), blk in zip(slabs, recv):
        full[:, lo:hi] = blk[:, :hi - lo]
    return full


def gcn_forward_sharded(op, x, w0, w1, group=None, compute=None):
    """gcn_forward (gcn.cpp:22-33) over the ranks of `group`, bit-identical to
    one GPU.

    Rank r owns the hidden columns column_slab(hid, world, r):
      T_r = X . W0[:, slab]       (reference-exact GEMM: each column exact)
      H_r = relu(A_hat . T_r)     (CBM multiply, ReLU in the epilogue)
      Z_r = A_hat . H_r
    The one real exchange is the all-gather of the Z slabs (NCCL over
    NVLink; ~n*hid*4 bytes), after which rank r forms its class columns
    Z . W1[:, cslab] in the reference's ascending order and a small second
    all-gather assembles the n x classes output on every rank. `x`, `w0`,
    `w1` are replicated on every rank (torch tensors on the rank's device).
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cm = compute if compute is not None else _DeviceCompute(op)
    hid, classes = w0.shape[1], w1.shape[1]
    if w0.shape[0] != x.shape[1] or w1.shape[0] != hid:
        raise ValueError("dense_matmul: inner dimensions differ")
    hslabs = all_slabs(hid, world)
    lo, hi = hslabs[rank]
    t = cm.matmul(x, w0[:, lo:hi].contiguous())
    h = cm.spmm(t, relu=True)
    z = cm.spmm(h)
    z_full = _gather_columns(z, hslabs, rank, group)
    cslabs = all_slabs(classes, world)
    clo, chi = cslabs[rank]
    o = cm.matmul(z_full, w1[:, clo:chi].contiguous())
    return _gather_columns(o, cslabs, rank, group)
