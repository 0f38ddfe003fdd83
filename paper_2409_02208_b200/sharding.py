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


def row_block(n: int, world: int, rank: int) -> tuple[int, int]:
    """[r0, r1) rows of `rank` for the fused gather-GEMM (balanced, contiguous)."""
    return n * rank // world, n * (rank + 1) // world


def _gather_rows(ptr, data, rows):
    """Concatenated data[ptr[r]:ptr[r+1]] for r in rows (vectorised)."""
    import numpy as np
    ptr = np.asarray(ptr, np.int64)
    starts = ptr[rows]
    lens = ptr[rows + 1] - starts
    total = int(lens.sum())
    if total == 0:
        return data[:0]
    base = np.repeat(starts - (np.cumsum(lens) - lens), lens)
    return data[base + np.arange(total)]


def _balanced_cuts(cost, parts):
    import numpy as np
    m = len(cost)
    cum = np.cumsum(cost)
    total = int(cum[-1]) if m else 0
    cuts = [0] + [int(np.searchsorted(cum, total * k / parts, side="left")) + 1
                  for k in range(1, parts)] + [m]
    return np.maximum.accumulate(np.minimum(np.asarray(cuts), m))


def _group_cost(cuts, par, clen, alen):
    """Per-row stored length under `cuts`: the deltas, or the A row when the
    parent lies in another group (flattened)."""
    import numpy as np
    from . import VIRTUAL_PARENT
    group = np.searchsorted(cuts, np.arange(len(par)), side="right") - 1
    virt = par == VIRTUAL_PARENT
    pg = np.searchsorted(cuts, np.where(virt, 0, par), side="right") - 1
    return np.where(~virt & (pg != group), alen, clen)


def _max_group(cost, cuts):
    import numpy as np
    cum = np.concatenate([[0], np.cumsum(cost)])
    return int(np.max(cum[cuts[1:]] - cum[cuts[:-1]]))


def _with_identity(a):
    """Row pointers and columns of A + I (the pattern a normalized CBM
    represents, normalized_adjacency_csr, gcn.cpp:48-89)."""
    import numpy as np
    n = a.n_rows
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_ptr.astype(np.int64)))
    r = np.concatenate([rows, np.arange(n, dtype=np.int64)])
    cc = np.concatenate([a.col_idx.astype(np.int64), np.arange(n, dtype=np.int64)])
    order = np.lexsort((cc, r))
    r, cc = r[order], cc[order]
    keep = np.ones(r.size, bool)
    keep[1:] = (r[1:] != r[:-1]) | (cc[1:] != cc[:-1])
    r, cc = r[keep], cc[keep]
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.uint64)
    return ptr, cc.astype(np.uint32)


def row_partition(a, c, parts: int):
    """Row groups of a 2-D (row group x column slab) partition of a CBM
    (DESIGN.md §7): contiguous row ranges balanced by stored length (delta
    count, refined to count flattened rows at their full length). A row whose
    parent lies in another range is flattened (its deltas become its full row
    with a virtual parent, as the tiled path does for cut trees), so a group
    never waits on another and no collective is needed. Returns
    [(global row ids, sub-CBM of those rows x all columns)], one per group;
    Y[rows_g] = sub_g . X. Integer-valued X gives the exact sums of the full
    multiply; otherwise the flattened rows sum in a different order (within
    the default mode's tolerance).

    Normalized CBMs: the full rows are those of A + I, the delta values stay
    +-s[col] (the column scale), and each block carries the column scale of
    the whole matrix (col_scale) beside its own rows' scale (row_scale): a
    rectangular row block the reference's square container cannot hold
    (io.cpp:369-380), uploaded through the view's col_scale."""
    import numpy as np
    from . import VIRTUAL_PARENT, CbmMatrix
    if parts < 1:
        raise ValueError("row_partition: parts must be >= 1")
    if a.n_rows != c.n_rows or a.n_cols != c.n_cols:
        raise ValueError("row_partition: A and its CBM differ in shape")
    norm = bool(c.is_normalized)
    if norm:
        a_ptr, a_col = _with_identity(a)
    else:
        a_ptr, a_col = a.row_ptr, a.col_idx
    m = c.n_rows
    clen = np.diff(c.row_ptr.astype(np.int64))
    alen_all = np.diff(a_ptr.astype(np.int64))
    par_all = c.parent.astype(np.int64)
    cuts = _balanced_cuts(clen, parts)
    # refine: balance the lengths AFTER flattening (a flattened row costs its
    # full row, not its deltas); keep whichever cut has the lightest heaviest group
    best = (_max_group(_group_cost(cuts, par_all, clen, alen_all), cuts), cuts)
    for _ in range(4):
        cuts = _balanced_cuts(_group_cost(cuts, par_all, clen, alen_all), parts)
        heavy = _max_group(_group_cost(cuts, par_all, clen, alen_all), cuts)
        if heavy < best[0]:
            best = (heavy, cuts)
    cuts = best[1]
    out = []
    for g in range(parts):
        lo, hi = int(cuts[g]), int(cuts[g + 1])
        rows = np.arange(lo, hi, dtype=np.int64)
        par = par_all[lo:hi]
        virt = par == VIRTUAL_PARENT
        inside = ~virt & (par >= lo) & (par < hi)
        flat = ~virt & ~inside
        parent = np.where(inside, par - lo, VIRTUAL_PARENT).astype(np.uint32)
        alen = alen_all[lo:hi]
        lens = np.where(flat, alen, clen[lo:hi])
        row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        row_of = np.repeat(np.arange(hi - lo), lens)
        fpos = flat[row_of]
        col_idx = np.empty(int(row_ptr[-1]), np.uint32)
        values = np.empty(int(row_ptr[-1]), np.float32)
        col_idx[fpos] = _gather_rows(a_ptr, a_col, rows[flat])
        values[fpos] = c.row_scale[col_idx[fpos]] if norm else 1.0
        col_idx[~fpos] = _gather_rows(c.row_ptr, c.col_idx, rows[~flat])
        values[~fpos] = _gather_rows(c.row_ptr, c.values, rows[~flat])
        out.append((rows, CbmMatrix(hi - lo, c.n_cols, c.alpha, norm, parent, row_ptr, col_idx,
                                    values,
                                    row_scale=c.row_scale[lo:hi] if norm else None,
                                    col_scale=c.row_scale if norm else None)))
    return out


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

    def gather_gemm(self, z, hslabs, w1, rank, group, ordered):
        """out = [Z_0 | ... | Z_{N-1}] . W1 on every rank, fused: rank r's GEMM
        reads the rows [r0, r1) of every peer's Z slab over NVLink (CUDA IPC)
        and writes its output rows into every rank's output buffer
        (cbm_b200_gemm_parts). No staging copy of the gathered Z exists."""
        import torch
        import torch.distributed as dist
        from . import gemm_parts, ipc_close, ipc_handle, ipc_open
        world = len(hslabs)
        n, classes = z.shape[0], w1.shape[1]
        z = z.contiguous()
        out = torch.empty((n, classes), dtype=torch.float32, device=z.device)
        widths = [hi - lo for lo, hi in hslabs]
        if world == 1:
            gemm_parts([z], widths, n, w1, [out], classes, ordered)
            return out
        torch.cuda.synchronize(z.device)  # Z complete before peers read it
        mine = (ipc_handle(z), ipc_handle(out))
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        dev = z.device.index
        maps = []  # (peer base pointer to unmap)
        zp, op = [], []
        for s_, (hz, ho) in enumerate(handles):
            if s_ == rank:
                zp.append(z.data_ptr())
                op.append(out.data_ptr())
                continue
            pz, po = ipc_open(hz, dev), ipc_open(ho, dev)
            maps += [pz - hz[1], po - ho[1]]
            zp.append(pz)
            op.append(po)
        r0, r1 = row_block(n, world, rank)
        parts = [p + r0 * w * 4 for p, w in zip(zp, widths)]
        outs = [p + r0 * classes * 4 for p in op]
        dist.barrier(group=group)  # every rank has mapped every buffer
        gemm_parts(parts, widths, r1 - r0, w1, outs, classes, ordered)
        torch.cuda.synchronize(z.device)
        dist.barrier(group=group)  # every rank's rows have landed in `out`
        for p in maps:
            ipc_close(p)
        return out


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


def gcn_forward_sharded(op, x, w0, w1, group=None, compute=None, fused=False):
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

    fused=True replaces both all-gathers and the last GEMM with one kernel per
    rank (compute.gather_gemm): rank r computes the output rows
    row_block(n, world, r) reading every peer's Z slab in place over NVLink and
    storing its rows into every rank's output; the ascending-k order over the
    concatenated slabs is the reference's, so the result is the same bits.
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
    if fused:
        ordered = bool(op.info()["order_faithful"]) if op is not None else True
        return cm.gather_gemm(z, hslabs, w1, rank, group, ordered)
    z_full = _gather_columns(z, hslabs, rank, group)
    cslabs = all_slabs(classes, world)
    clo, chi = cslabs[rank]
    o = cm.matmul(z_full, w1[:, clo:chi].contiguous())
    return _gather_columns(o, cslabs, rank, group)


def grid_position(world: int, rank: int, row_groups: int) -> tuple[int, int, int]:
    """Rank -> (row group, column-slab rank, column slabs) of the 2-D
    partition N = row_groups x (N / row_groups), row-group major: ranks
    g*C .. g*C+C-1 share row group g (sharding.row_partition) and split its
    columns with column_slab(d, C, .). row_groups = 1 is the column-only
    split. Like the column split it needs no collective: each rank owns the
    block Y[rows_g, slab]."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("grid_position: bad rank/world")
    if row_groups < 1 or world % row_groups:
        raise ValueError("grid_position: row_groups must divide world")
    slabs = world // row_groups
    return rank // slabs, rank % slabs, slabs


def auto_row_groups(d: int, world: int) -> int:
    """Row groups for N ranks of a binary CBM: keep column slabs >= 128
    wide (C = the largest divisor of N not above d / 128) and give the rest
    of N to row groups. Chosen from the per-rank projection
    (profiles/r01e_project_2d.jsonl): every rank walks its
    group's whole structure whatever its width, so narrow slabs stop
    scaling while row groups shrink the structure itself."""
    if world < 1:
        raise ValueError("auto_row_groups: world must be >= 1")
    slabs = max(c for c in range(1, world + 1) if world % c == 0 and c <= max(1, d // 128))
    return world // slabs
