"""Kernel timing experiments (development tool, not part of the product)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_02208_b200 as P
from paper_2409_02208_b200.workloads import WORKLOADS

def timeit(op, x, y, flush, reps=30):
    s = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        if flush is not None: flush.fill_(float(i))
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); op.spmm_into(x, y, s); b.record(s)
        torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), float(np.min(ts))

dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
for name in sys.argv[1].split(","):
    wl = WORKLOADS[name]
    a = wl.graph(); c = wl.build(a, 8)
    for d in [int(v) for v in sys.argv[2].split(",")]:
        x = torch.from_numpy(wl.operand(a.n_cols, d)).to(dev)
        y = torch.empty((a.n_rows, d), device=dev)
        variants = {"default": c}
        nodep = P.CbmMatrix(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                            np.full(c.n_rows, 0xFFFFFFFF, np.uint32), c.row_ptr, c.col_idx,
                            c.values, c.row_scale)
        variants["nodep"] = nodep
        empty = P.CbmMatrix(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                            np.full(c.n_rows, 0xFFFFFFFF, np.uint32), np.zeros(c.n_rows + 1, np.uint64),
                            np.zeros(0, np.uint32), np.zeros(0, np.float32), c.row_scale)
        variants["empty"] = empty
        only = sys.argv[3] if len(sys.argv) > 3 else None
        for vn, cc in variants.items():
            if only and vn != only:
                continue
            for faithful, kern, segs in ((False, "auto", 0), (False, "auto", 1)):
                if vn != "default" and (faithful or segs):
                    continue
                op = P.DeviceCbm(cc, order_faithful=faithful, kernel=kern, prefetch=bool(segs))
                med_f, min_f = timeit(op, x, y, flush)
                med, mn = timeit(op, x, y, None)
                print(f"{name} d={d} {vn:8s} prefetch={segs} flush med {med_f:8.1f}us  noflush med {med:8.1f}us min {mn:8.1f}us  info={ {k: op.info()[k] for k in ('n_levels','n_items','launches_per_call')} }", flush=True)
