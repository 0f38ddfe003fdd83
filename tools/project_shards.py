"""Column-shard scaling measured per rank on one B200 (dev tool).

A rank of an N-GPU column-sharded multiply holds a replica of
the CBM and multiplies its own contiguous column slab of X; there is no
collective on the A.X path, so the N-GPU step is the slowest rank's step.
This tool times, on one GPU, exactly the work each rank does (its slab as a
contiguous n x d_r operand, L2 flushed before every call, CUDA events) and
reports the N-GPU whole-job throughput that follows: 2*nnz*d / max_r t_r.
It is a per-rank measurement, not an N-GPU run: it assumes the ranks do not
slow each other down, which holds when nothing crosses NVLink.

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
            sweep("cfg4", a, c, normalized, (64, 128, 256), flush, dev)
            del c
    else:
        wl = WORKLOADS[which]
        a = wl.graph()
        c = wl.build(a, threads)
        sweep(which, a, c, wl.normalized, (wl.d,), flush, dev)


if __name__ == "__main__":
    main()
