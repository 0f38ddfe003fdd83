"""Dev tool: GCN forward (gcn.cpp:22-33) timing breakdown on cfg[3]'s shape.

Usage: python tools/probe_gcn.py [cfg3]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def ev_time(fn, reps=10):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    wl = WORKLOADS[name]
    a = wl.graph()
    c = wl.build(a, os.cpu_count() or 8)
    n, f, hid, classes = a.n_rows, 128, 256, 112
    x = torch.from_numpy(P.generate_dense("normal", n, f, 0xC0F61003)).cuda()
    w0 = torch.from_numpy(P.generate_dense("glorot", f, hid, 0xC0F62003)).cuda()
    w1 = torch.from_numpy(P.generate_dense("glorot", hid, classes, 0xC0F62004)).cuda()
    for faithful in (False, True):
        op = P.DeviceCbm(c, order_faithful=faithful)
        h0 = P.dense_matmul(x, w0)
        t_g0 = ev_time(lambda: P.dense_matmul(x, w0))
        t_s1 = ev_time(lambda: op.spmm(h0, relu=True))
        h1 = op.spmm(h0, relu=True)
        t_s2 = ev_time(lambda: op.spmm(h1))
        h2 = op.spmm(h1)
        t_g1 = ev_time(lambda: P.dense_matmul(h2, w1))
        t_all = ev_time(lambda: op.gcn_forward(x, w0, w1))
        gf0 = 2 * n * f * hid / t_g0 / 1e3
        gf1 = 2 * n * hid * classes / t_g1 / 1e3
        print(f"{name} faithful={faithful}: X.W0 {t_g0:8.1f} us ({gf0 / 1e3:.1f} TFLOP/s)  "
              f"relu(A.) {t_s1:8.1f} us  A. {t_s2:8.1f} us  .W1 {t_g1:8.1f} us ({gf1 / 1e3:.1f} TFLOP/s)  "
              f"gcn_forward {t_all:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
