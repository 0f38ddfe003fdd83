"""Column-shard scaling measured per rank on one B200 (dev tool).

A rank of an N-GPU column-sharded multiply holds a replica of
the CBM and multiplies its own contiguous column slab of X; there is no
collective on the A.X path, so the N-GPU step is the slowest rank's step.
This tool times, on one GPU, exactly the work each rank does (its slab as a
contiguous n x d_r operand, L2 flushed before every call, CUDA events) and
reports the N-GPU whole-job throughput that follows: 2*nnz*d / max_r t_r.
It is a per-rank measurement, not an N-GPU run: it assumes the ranks do not
slow each other down, which holds when nothing crosses NVLink.

Binary workloads also get the 2-D partition (sharding.row_partition): N =
R row groups x C column slabs, each rank timed on its group's sub-CBM at its
slab width; the best (R, C) per N is reported beside the column-only split.

Usage: python tools/project_shards.py cfg1            (the bench workload)
       python tools/project_shards.py cfg4            (2.45M rows, d = 64/128/256,
                                                       binary and normalized; slow build)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.sharding import all_slabs  # noqa: E402
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
            ts.append(a.elapsed_time(b))
    return float(np.mean(ts))


def sweep(name, a, c, normalized, ds, flush, dev):
    nnz = a.nnz + (a.n_rows if normalized else 0)  # generators draw no self-loops
    op = P.DeviceCbm(c)
    for d in ds:
        x_full = P.generate_dense("normal", a.n_cols, d, 0xC0F61000 + 4)
        base = None
        for world in (1, 2, 4, 8):
            widths = sorted({hi - lo for lo, hi in all_slabs(d, world)}, reverse=True)
            t_max = 0.0
            for w in widths:  # every distinct slab width (ranks of equal width do equal work)
                x = torch.from_numpy(np.ascontiguousarray(x_full[:, :w])).to(dev)
                y = torch.empty((a.n_rows, w), device=dev)
                t_max = max(t_max, timeit(op, x, y, flush))
                del x, y
            value = 2.0 * nnz * d / (t_max * 1e-3) / 1e9
            base = base or value
            print(json.dumps({"workload": name, "normalized": normalized, "d": d, "n_gpus": world,
                              "slab_widths": widths, "ms_max_rank": t_max,
                              "projected_gflops": value, "speedup_vs_1": value / base,
                              "note": "per-rank slab timed on one B200; N-GPU step = max over ranks"}),
                  flush=True)


def sweep2d(name, a, c, ds, flush, dev):
    """N = R x C ranks: row group g of R (sharding.row_partition) x column slab
    of C; every rank's (sub-CBM, slab width) timed; N-GPU step = max."""
    from paper_2409_02208_b200.sharding import row_partition
    nnz = a.nnz
    groups = {R: [(rows, P.DeviceCbm(sub)) for rows, sub in row_partition(a, c, R)]
              for R in (2, 4, 8)}
    groups[1] = [(None, P.DeviceCbm(c))]
    for d in ds:
        x_full = P.generate_dense("normal", a.n_cols, d, 0xC0F61000 + 4)
        base = None
        cache = {}
        for world in (1, 2, 4, 8):
            best = None
            for R in (1, 2, 4, 8):
                if world % R:
                    continue
                C = world // R
                widths = sorted({hi - lo for lo, hi in all_slabs(d, C)}, reverse=True)
                t_max = 0.0
                for w in widths:
                    x = torch.from_numpy(np.ascontiguousarray(x_full[:, :w])).to(dev)
                    ops = groups[R]
                    for gi, (rows, op) in enumerate(ops):
                        key = (R, gi, w)
                        if key not in cache:
                            n_out = c.n_rows if rows is None else len(rows)
                            y = torch.empty((n_out, w), device=dev)
                            cache[key] = timeit(op, x, y, flush)
                            del y
                        t_max = max(t_max, cache[key])
                    del x
                if best is None or t_max < best[0]:
                    group_ms = [round(cache[(R, gi, widths[0])], 4) for gi in range(R)]
                    best = (t_max, R, C, widths, group_ms)
            t_max, R, C, widths, group_ms = best
            value = 2.0 * nnz * d / (t_max * 1e-3) / 1e9
            base = base or value
            print(json.dumps({"workload": name, "normalized": False, "d": d, "n_gpus": world,
                              "partition": f"{R} row groups x {C} column slabs",
                              "slab_widths": widths, "ms_max_rank": t_max,
                              "group_ms_widest_slab": group_ms,
                              "projected_gflops": value, "speedup_vs_1": value / base,
                              "note": "2-D partition; per-rank work timed on one B200; "
                                      "N-GPU step = max over ranks"}), flush=True)


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    threads = os.cpu_count() or 8
    if which == "cfg4":
        wl = WORKLOADS["cfg4_64"]
        a = wl.graph()
        for normalized in (False, True):
            c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, wl.alpha, threads)
            if "--2d" in sys.argv:
                if not normalized:
                    sweep2d("cfg4", a, c, (64, 128, 256), flush, dev)
            else:
                sweep("cfg4", a, c, normalized, (64, 128, 256), flush, dev)
            del c
            if "--2d" in sys.argv:
                break
    else:
        wl = WORKLOADS[which]
        a = wl.graph()
        c = wl.build(a, threads)
        if "--2d" in sys.argv:
            sweep2d(which, a, c, (wl.d,), flush, dev)
        else:
            sweep(which, a, c, wl.normalized, (wl.d,), flush, dev)


if __name__ == "__main__":
    main()
