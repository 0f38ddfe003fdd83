"""Dev tool: spmv (d = 1) timings, default and order-faithful modes.

Usage: python tools/probe_spmv.py cfg1,cfg3
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    for name in sys.argv[1].split(","):
        wl = WORKLOADS[name]
        a = wl.graph()
        c = wl.build(a, os.cpu_count() or 8)
        v = torch.from_numpy(wl.operand(a.n_cols, 1)).to(dev)
        u = torch.empty((a.n_rows, 1), device=dev)
        for faithful in (False, True):
            op = P.DeviceCbm(c, order_faithful=faithful)
            s = torch.cuda.current_stream()
            ts = []
            for i in range(23):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                op.spmv_into(v, u, s)
                e1.record(s)
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            nnz = a.nnz + (a.n_rows if wl.normalized else 0)
            t = float(np.median(ts))
            print(f"{name} spmv faithful={faithful}: {t:9.1f} us  {2 * nnz / t / 1e3:8.2f} GFLOP/s "
                  f"launches={op.info()['launches_per_call']}", flush=True)
            op.close()


if __name__ == "__main__":
    main()
