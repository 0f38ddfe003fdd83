"""Dev tool: is the streaming kernel on hub-heavy graphs limited by L2 slice
hot-spotting on the most-referenced X rows?

Times the uncompressed matrix (csr_operator: every parent virtual) of a
workload, then the same matrix with every column referenced more than T times
redirected round-robin to ceil(deg/T) replica rows appended to X (same sums,
the hot rows spread over more L2 slices). A large drop means hot-spotting.

Usage: python tools/probe_hubs.py cfg2 [T1,T2,...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def timeit(op, x, y, flush, reps=20):
    s = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        flush.fill_(float(i))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        op.spmm_into(x, y, s)
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def remap(a, thresh):
    """Columns with > thresh references -> round-robin over replicas."""
    ci = a.col_idx.astype(np.int64)
    deg = np.bincount(ci, minlength=a.n_cols)
    hot = np.nonzero(deg > thresh)[0]
    reps = -(-deg[hot] // thresh)  # replicas per hot column (incl. the original)
    extra = int((reps - 1).sum())
    base = np.zeros(a.n_cols, np.int64)
    base[hot] = a.n_cols + np.concatenate([[0], np.cumsum(reps - 1)[:-1]])
    nrep = np.ones(a.n_cols, np.int64)
    nrep[hot] = reps
    # occurrence number of each reference within its column
    order = np.argsort(ci, kind="stable")
    occ = np.empty_like(ci)
    starts = np.concatenate([[0], np.cumsum(deg)[:-1]])
    occ[order] = np.arange(ci.size) - starts[ci[order]]
    k = occ % nrep[ci]
    new = np.where(k == 0, ci, base[ci] + k - 1)
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.astype(np.int64)))
    o = np.lexsort((new, rows))
    src = np.arange(a.n_cols, dtype=np.int64)
    src_extra = np.repeat(hot, reps - 1)
    b = P.CsrBinaryMatrix(a.n_rows, a.n_cols + extra, a.row_ptr.copy(),
                          new[o].astype(np.uint32))
    return b, np.concatenate([src, src_extra]), len(hot), extra, int(deg.max())


def main():
    name = sys.argv[1]
    ths = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8192, 2048, 512]
    wl = WORKLOADS[name]
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    a = wl.graph()
    x0 = torch.from_numpy(wl.operand(a.n_cols)).to(dev)
    y = torch.empty((a.n_rows, wl.d), device=dev)
    op = P.DeviceCbm(P.csr_operator(a))
    t0 = timeit(op, x0, y, flush)
    ref = y.clone()
    print(f"{name} d={wl.d} nnz={a.nnz} csr: {t0:.1f} us", flush=True)
    for th in ths:
        b, src, nhot, extra, dmax = remap(a, th)
        x = x0[torch.from_numpy(src).to(dev)]
        opb = P.DeviceCbm(P.csr_operator(b))
        t = timeit(opb, x, y, flush)
        err = float((y - ref).abs().max() / ref.abs().max())
        print(f"  T={th:6d}: {nhot} hot columns (max degree {dmax}), {extra} replica rows: "
              f"{t:.1f} us ({t0 / t:.2f}x)  normwise diff {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
