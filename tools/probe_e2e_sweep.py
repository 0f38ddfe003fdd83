"""Dev tool: the host-buffer entry point (cbm_b200_spmm_host) under several
column-chunk plans, one build (the plan is read per call from
CBM_B200_HOST_CHUNKS / CBM_B200_HOST_WIDTHS).

Usage: python tools/probe_e2e_sweep.py cfg4_b256 default 2 4 8 128/128 64/64/64/64 ...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def main():
    name, plans = sys.argv[1], sys.argv[2:]
    wl = WORKLOADS[name]
    a = wl.graph()
    c = wl.build(a, os.cpu_count() or 8)
    x = torch.from_numpy(wl.operand(a.n_cols)).pin_memory()
    y = torch.empty((a.n_rows, wl.d), dtype=torch.float32).pin_memory()
    op = P.DeviceCbm(c)
    s = torch.cuda.current_stream()
    reps = int(os.environ.get("REPS", "8"))
    for plan in plans:
        os.environ.pop("CBM_B200_HOST_CHUNKS", None)
        os.environ.pop("CBM_B200_HOST_WIDTHS", None)
        if "/" in plan:
            os.environ["CBM_B200_HOST_WIDTHS"] = plan.replace("/", ",")
        elif plan != "default":
            os.environ["CBM_B200_HOST_CHUNKS"] = plan
        for _ in range(2):
            op.spmm_host_ptr(x.data_ptr(), a.n_cols, wl.d, y.data_ptr(), a.n_rows, wl.d, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            op.spmm_host_ptr(x.data_ptr(), a.n_cols, wl.d, y.data_ptr(), a.n_rows, wl.d, s)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"{name} plan={plan}: {e0.elapsed_time(e1) / reps:8.2f} ms per call", flush=True)
    xd = torch.empty((a.n_cols, wl.d), device="cuda")
    yd = torch.empty((a.n_rows, wl.d), device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for label, both in (("H2D X alone", 0), ("D2H Y alone", 1), ("H2D X + D2H Y concurrent", 2)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            if both in (0, 2):
                with torch.cuda.stream(s1):
                    xd.copy_(x, non_blocking=True)
            if both in (1, 2):
                with torch.cuda.stream(s2):
                    y.copy_(yd, non_blocking=True)
            torch.cuda.synchronize()
        print(f"{name} {label} (contiguous, wall): {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms",
              flush=True)


if __name__ == "__main__":
    main()
