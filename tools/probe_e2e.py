"""Dev tool: host-buffer entry point (cbm_b200_spmm_host) vs column-chunk count.

Usage: python tools/probe_e2e.py cfg1 1,2,4,8
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(name, chunks):
    import time
    import torch
    import paper_2409_02208_b200 as P
    from paper_2409_02208_b200.workloads import WORKLOADS
    wl = WORKLOADS[name]
    a = wl.graph()
    c = wl.build(a, os.cpu_count() or 8)
    x = torch.from_numpy(wl.operand(a.n_cols)).pin_memory()
    y = torch.empty((a.n_rows, wl.d), dtype=torch.float32).pin_memory()
    op = P.DeviceCbm(c)
    s = torch.cuda.current_stream()
    for _ in range(3):
        op.spmm_host_ptr(x.data_ptr(), a.n_cols, wl.d, y.data_ptr(), a.n_rows, wl.d, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    reps = 30
    t0 = time.perf_counter()
    for _ in range(reps):
        op.spmm_host_ptr(x.data_ptr(), a.n_cols, wl.d, y.data_ptr(), a.n_rows, wl.d, s)
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e6
    ev = e0.elapsed_time(e1) / reps * 1e3
    # copies alone
    xd = torch.empty((a.n_cols, wl.d), device="cuda")
    yd = torch.empty((a.n_rows, wl.d), device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            xd.copy_(x, non_blocking=True)
        with torch.cuda.stream(s2):
            y.copy_(yd, non_blocking=True)
        torch.cuda.synchronize()
    both = (time.perf_counter() - t0) / reps * 1e6
    print(f"{name} chunks={chunks}: spmm_host events {ev:8.1f} us  wall {wall:8.1f} us | "
          f"concurrent H2D+D2H of X,Y alone (wall) {both:8.1f} us", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 3:
        one(sys.argv[1], sys.argv[3])
    else:
        for ch in sys.argv[2].split(","):
            env = dict(os.environ, CBM_B200_HOST_CHUNKS=ch)
            if ch == "0":  # the library's default chunking
                env.pop("CBM_B200_HOST_CHUNKS")
            if "/" in ch:  # explicit widths, e.g. 32/96/128/128/96/32
                env.pop("CBM_B200_HOST_CHUNKS")
                env["CBM_B200_HOST_WIDTHS"] = ch.replace("/", ",")
            subprocess.run([sys.executable, __file__, sys.argv[1], "", ch], env=env, check=True)
