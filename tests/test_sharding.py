"""Column sharding host logic, including a world-size-2 gloo run on CPU: each
rank computes its column slab (with the oracle standing in for its GPU), the
slabs are all-gathered, and the result equals the single-device product bit
for bit (columns are independent in kernels.cpp:27-62)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2409_02208_b200 as P
from paper_2409_02208_b200.sharding import all_slabs, column_slab
from helpers import oracle_arrays


@pytest.mark.parametrize("d,world", [(512, 8), (64, 8), (130, 4), (7, 2), (1, 2), (3, 8)])
def test_slabs_partition_columns(d, world):
    slabs = all_slabs(d, world)
    covered = []
    for lo, hi in slabs:
        assert 0 <= lo <= hi <= d
        covered.extend(range(lo, hi))
    assert covered == list(range(d))
    for lo, hi in slabs[:-1]:
        assert lo % 4 == 0


@pytest.mark.parametrize("d,world", [(512, 8), (64, 8), (130, 4), (7, 2), (1, 2), (0, 3)])
def test_native_slabs_match_the_balanced_unit_partition(d, world):
    units = (d + 3) // 4
    for r in range(world):
        lo = min(d, units * r // world * 4)
        hi = max(lo, min(d, units * (r + 1) // world * 4))
        assert column_slab(d, world, r) == (lo, hi)
    with pytest.raises(ValueError):
        column_slab(d, world, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = P.generate_graph("pa_triangle", [1500, 2, 0.3], 5)
    c = P.build_cbm_normalized(a, 0)
    x = P.generate_dense("normal", a.n_cols, 96, 6)
    lo, hi = column_slab(96, world, rank)
    y_local = O.oracle_spmm(oracle_arrays(c), np.ascontiguousarray(x[:, lo:hi]))
    pieces = [None] * world
    dist.all_gather_object(pieces, (lo, hi, y_local))
    if rank == 0:
        y = np.empty((c.n_rows, 96), np.float32)
        for lo_, hi_, blk in pieces:
            y[:, lo_:hi_] = blk
        out.put(y)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_column_shards_reassemble_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    y = q.get(timeout=240)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    a = P.generate_graph("pa_triangle", [1500, 2, 0.3], 5)
    c = P.build_cbm_normalized(a, 0)
    x = P.generate_dense("normal", a.n_cols, 96, 6)
    want = O.oracle_spmm(oracle_arrays(c), x)
    assert np.array_equal(y.view(np.uint32), want.view(np.uint32))


class _OracleCompute:
    """Test stand-in for a rank's GPU: the oracle restatement on CPU tensors
    (the product's compute is _DeviceCompute; this exercises the partition,
    the all-gathers and the repacking)."""

    def __init__(self, arrays):
        self.arrays = arrays

    def matmul(self, a, b):
        return torch.from_numpy(O.oracle_dense_matmul(a.numpy(), b.contiguous().numpy()))

    def gather_gemm(self, z, hslabs, w1, rank, group, ordered):
        """CPU stand-in for the fused peer-memory gather-GEMM: the peers' Z
        slabs are fetched with a gloo all-gather (the device reads them in
        place over NVLink), rank r computes its row block, the blocks are
        gathered back (the device stores them into every rank's output)."""
        from paper_2409_02208_b200.sharding import row_block
        world = len(hslabs)
        slabs = [None] * world
        dist.all_gather_object(slabs, z.numpy(), group=group)
        r0, r1 = row_block(z.shape[0], world, rank)
        zr = np.ascontiguousarray(np.concatenate([sl[r0:r1] for sl in slabs], axis=1))
        mine = O.oracle_dense_matmul(zr, w1.contiguous().numpy())
        blocks = [None] * world
        dist.all_gather_object(blocks, mine, group=group)
        return torch.from_numpy(np.ascontiguousarray(np.concatenate(blocks, axis=0)))

    def spmm(self, x, relu=False):
        y = O.oracle_spmm(self.arrays, np.ascontiguousarray(x.numpy()))
        if relu:
            y = np.where(y < 0, np.float32(0), y)
        return torch.from_numpy(np.ascontiguousarray(y, np.float32))


def _gcn_inputs():
    a = P.generate_graph("community", [600, 50, 0.5, 0.01], 81)
    c = P.build_cbm_normalized(a, 0)
    x = P.generate_dense("normal", 600, 24, 82)
    w0 = P.generate_dense("glorot", 24, 40, 83)
    w1 = P.generate_dense("glorot", 40, 10, 84)
    return c, x, w0, w1


def _gcn_worker(rank, world, port, out, fused=False):
    from paper_2409_02208_b200.sharding import gcn_forward_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, x, w0, w1 = _gcn_inputs()
    got = gcn_forward_sharded(None, torch.from_numpy(x), torch.from_numpy(w0),
                              torch.from_numpy(w1), compute=_OracleCompute(oracle_arrays(c)),
                              fused=fused)
    out.put((rank, got.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_gloo_world2_sharded_gcn_bitwise(fused):
    """Hidden-column shards + all-gather (gcn_forward_sharded) on 2 gloo ranks:
    both ranks hold the single-device gcn_forward output bit for bit. fused:
    the row-block gather-GEMM partition (rank r's rows over the concatenated
    slabs, ascending k) instead of two all-gathers."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gcn_worker, args=(r, 2, port, q, fused)) for r in range(2)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=240) for _ in range(2))
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    c, x, w0, w1 = _gcn_inputs()
    want = O.oracle_gcn_forward(oracle_arrays(c), x, w0, w1)
    for r in range(2):
        assert np.array_equal(results[r].view(np.uint32), want.view(np.uint32)), r


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 7])
def test_row_partition_reassembles_exactly(parts):
    """2-D partition row groups (sharding.row_partition): every group's
    sub-CBM is a valid container, groups cover the rows once, flattened rows
    keep their exact integer sums, and Y[rows_g] = sub_g . X reassembles the
    full multiply (oracle on each group, integer X: exact in any order)."""
    from paper_2409_02208_b200.sharding import row_partition
    a = P.generate_graph("clique_overlay", [1500, 6000, 2, 8, 1.1], 0xC0F60000 + 91)
    c = P.build_cbm(a, 4)
    x = P.generate_dense("int", a.n_cols, 20, 0xC0F61000 + 91, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    groups = row_partition(a, c, parts)
    assert len(groups) == parts
    seen = np.concatenate([rows for rows, _ in groups])
    assert np.array_equal(seen, np.arange(c.n_rows))
    got = np.empty_like(want)
    for rows, sub in groups:
        assert sub.n_rows == len(rows) and sub.n_cols == c.n_cols
        par = sub.parent[sub.parent != P.VIRTUAL_PARENT]
        assert np.all(par < sub.n_rows)  # parents inside the group
        got[rows] = O.oracle_spmm(oracle_arrays(sub), x)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # the heaviest group is no heavier than under the plain delta-count cut
    # (the refinement only keeps a cut that lowers it)
    from paper_2409_02208_b200.sharding import _balanced_cuts, _group_cost, _max_group
    clen = np.diff(c.row_ptr.astype(np.int64))
    alen = np.diff(a.row_ptr.astype(np.int64))
    par = c.parent.astype(np.int64)
    plain = _balanced_cuts(clen, parts)
    heavy = max(int(sub.row_ptr[-1]) for _, sub in groups)
    assert heavy <= _max_group(_group_cost(plain, par, clen, alen), plain)


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_row_partition_normalized_row_blocks(parts):
    """Normalized CBMs cut into row blocks: each block keeps the whole matrix's
    column scale (col_scale) and its own rows' scale (row_scale); flattened
    rows become rows of A + I with values s[col]. Reassembled through the
    oracle, the blocks give the full multiply within the default-mode bar."""
    from paper_2409_02208_b200.sharding import row_partition
    from helpers import normwise_err
    a = P.generate_graph("community", [1200, 80, 0.4, 0.01], 0xC0F60000 + 93)
    c = P.build_cbm_normalized(a, 0, 4)
    x = P.generate_dense("normal", a.n_cols, 24, 0xC0F61000 + 93)
    want = O.oracle_spmm(oracle_arrays(c), x)
    got = np.empty_like(want)
    for rows, sub in row_partition(a, c, parts):
        assert sub.is_normalized and sub.n_cols == c.n_cols
        assert np.array_equal(sub.row_scale, c.row_scale[rows])
        assert np.array_equal(sub.col_scale, c.row_scale)
        # every delta value is +-col_scale[col] (load_cbm's rule, per column)
        assert np.array_equal(np.abs(sub.values), sub.col_scale[sub.col_idx])
        got[rows] = O.oracle_spmm(oracle_arrays(sub), x)
    assert normwise_err(got, want) <= 1e-6


@pytest.mark.parametrize("world,row_groups", [(4, 1), (4, 2), (4, 4), (6, 3)])
def test_grid_position_covers_every_block_once(world, row_groups):
    from paper_2409_02208_b200.sharding import grid_position
    pos = [grid_position(world, r, row_groups) for r in range(world)]
    assert sorted((g, s) for g, s, _ in pos) == [(g, s) for g in range(row_groups)
                                                for s in range(world // row_groups)]
    assert all(n == world // row_groups for _, _, n in pos)
    with pytest.raises(ValueError):
        grid_position(4, 0, 3)


def _grid_worker(rank, world, row_groups, port, out):
    from paper_2409_02208_b200.sharding import grid_position, row_partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = P.generate_graph("clique_overlay", [1500, 6000, 2, 8, 1.1], 0xC0F60000 + 92)
    c = P.build_cbm(a, 2)
    x = P.generate_dense("int", a.n_cols, 40, 0xC0F61000 + 92, -8, 8)
    g, s, n_slabs = grid_position(world, rank, row_groups)
    rows, sub = row_partition(a, c, row_groups)[g]
    lo, hi = column_slab(40, n_slabs, s)
    blk = O.oracle_spmm(oracle_arrays(sub), np.ascontiguousarray(x[:, lo:hi]))
    pieces = [None] * world
    dist.all_gather_object(pieces, (rows, lo, hi, blk))
    if rank == 0:
        y = np.full((c.n_rows, 40), np.nan, np.float32)
        for rows_, lo_, hi_, blk_ in pieces:
            y[rows_, lo_:hi_] = blk_
        out.put(y)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world4_2d_partition_reassembles_bitwise():
    """bench.py --row-groups 2 at N = 4 (2 row groups x 2 column slabs), each
    rank's block from the oracle on its sub-CBM and slab, gathered over gloo:
    the blocks tile Y exactly once and equal the full multiply bit for bit
    (integer X)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, 4, 2, port, q)) for r in range(4)]
    for p_ in procs:
        p_.start()
    y = q.get(timeout=240)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    a = P.generate_graph("clique_overlay", [1500, 6000, 2, 8, 1.1], 0xC0F60000 + 92)
    c = P.build_cbm(a, 2)
    x = P.generate_dense("int", a.n_cols, 40, 0xC0F61000 + 92, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    assert np.array_equal(y.view(np.uint32), want.view(np.uint32))


def test_auto_row_groups_matches_the_projection_choice():
    """The (R, C) per N that profiles/r01e_project_2d.jsonl measured best."""
    from paper_2409_02208_b200.sharding import auto_row_groups
    assert [auto_row_groups(128, n) for n in (1, 2, 4, 8)] == [1, 2, 4, 8]
    assert [auto_row_groups(64, n) for n in (1, 2, 4, 8)] == [1, 2, 4, 8]
    assert [auto_row_groups(256, n) for n in (1, 2, 4, 8)] == [1, 1, 2, 4]
    assert auto_row_groups(512, 6) == 2


@pytest.mark.gpu
def test_device_multiplies_normalized_row_blocks():
    """Each normalized row block uploads through the view's col_scale (a
    rectangular normalized CBM) and multiplies like the oracle on the block."""
    import torch
    from paper_2409_02208_b200.sharding import row_partition
    from helpers import normwise_err
    a = P.generate_graph("community", [3000, 150, 0.4, 0.005], 0xC0F60000 + 94)
    c = P.build_cbm_normalized(a, 0, 4)
    x = P.generate_dense("normal", a.n_cols, 64, 0xC0F61000 + 94)
    for rows, sub in row_partition(a, c, 3):
        want = O.oracle_spmm(oracle_arrays(sub), x)
        for faithful in (True, False):
            got = P.DeviceCbm(sub, device=0, order_faithful=faithful).spmm(
                torch.from_numpy(x).cuda()).cpu().numpy()
            if faithful:
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
            else:
                assert normwise_err(got, want) <= 1e-5
