"""cfg[4] scaling-sweep shapes on one GPU (dev tool; bench.py times one d per run).

Builds the 2.45M-row clique overlay once (binary, then normalized), then times
A.X at d = 64, 128, 256 with the L2 flushed before every call, the streaming
and (when selected) tiled kernels, the uncompressed comparator and the
host-buffer entry point. One JSON line per (build, d) to stdout.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def timeit(fn, flush, reps=20):
    s = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        flush.fill_(float(i))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    wl = WORKLOADS["cfg4_64"]
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    t0 = time.time()
    a = wl.graph()
    t_graph = time.time() - t0
    for normalized in (False, True):
        t0 = time.time()
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, wl.alpha, os.cpu_count())
        t_build = time.time() - t0
        nnz = a.nnz if not normalized else a.nnz + a.n_rows  # no self-loops in the generator
        ops = {"auto": P.DeviceCbm(c)}
        info = ops["auto"].info()
        csr = P.DeviceCbm(P.csr_operator(a, normalized))
        for d in (64, 128, 256):
            x_host = torch.from_numpy(P.generate_dense("normal", a.n_cols, d, 0xC0F61004)).pin_memory()
            x = x_host.to(dev)
            y = torch.empty((a.n_rows, d), device=dev)
            out = {"workload": f"cfg4 {'normalized' if normalized else 'binary'} d={d}",
                   "n": a.n_rows, "nnz": int(nnz), "nnz_delta": int(c.nnz), "alpha": wl.alpha,
                   "build_s": t_build, "graph_s": t_graph,
                   "tile_active": info["tile_active"],
                   "tile_staged_fraction": info["tile_staged_deltas"] / max(1, info["tile_deltas"])}
            ms = timeit(lambda: ops["auto"].spmm_into(x, y), flush)
            out["ms"] = ms
            out["gflops"] = 2.0 * nnz * d / (ms * 1e-3) / 1e9
            b_alg = 4 * info["nnz_delta"] + 12 * a.n_rows + (4 * a.n_rows if normalized else 0) + 4 * d * (a.n_cols + a.n_rows)
            out["hbm_frac"] = b_alg / (ms * 1e-3) / 1e9 / 6548.5
            ms_csr = timeit(lambda: csr.spmm_into(x, y), flush, reps=10)
            out["csr_ms"] = ms_csr
            y_host = torch.empty((a.n_rows, d), dtype=torch.float32).pin_memory()
            s = torch.cuda.current_stream()
            ops["auto"].spmm_host_ptr(x_host.data_ptr(), a.n_cols, d, y_host.data_ptr(), a.n_rows, d, s)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                ops["auto"].spmm_host_ptr(x_host.data_ptr(), a.n_cols, d, y_host.data_ptr(), a.n_rows, d, s)
            e1.record(s)
            torch.cuda.synchronize()
            out["e2e_gflops"] = 2.0 * nnz * d / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e9
            print(json.dumps(out), flush=True)
            del x, y, x_host, y_host
        del ops, csr, c


if __name__ == "__main__":
    main()
