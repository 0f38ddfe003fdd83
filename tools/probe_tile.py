"""Tiled path vs streaming kernel timings (development tool, not the product).

  python tools/probe_tile.py cfg0,cfg3 [d,...] [opt=v,...;opt=v,...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def timeit(op, x, y, flush, reps=30):
    s = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        if flush is not None:
            flush.fill_(float(i))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        op.spmm_into(x, y, s)
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, device=dev)
names = sys.argv[1].split(",")
ds = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 and sys.argv[2] else None
variants = [{"tile": 0}, {"tile": 1}]
if len(sys.argv) > 3:
    variants = [{"tile": 0}] + [dict((kv.split("=")[0], int(kv.split("=")[1]))
                                     for kv in grp.split(",")) for grp in sys.argv[3].split(";")]
for name in names:
    wl = WORKLOADS[name]
    t0 = time.time()
    a = wl.graph()
    c = wl.build(a, os.cpu_count())
    print(f"{name}: build {time.time() - t0:.1f}s nnz(delta) {c.nnz}", flush=True)
    for d in ds or [wl.d]:
        x = torch.from_numpy(wl.operand(a.n_cols, d)).to(dev)
        y = torch.empty((a.n_rows, d), device=dev)
        ref = None
        for v in variants:
            t1 = time.time()
            op = P.DeviceCbm(c, **v)
            up = time.time() - t1
            med_f, min_f = timeit(op, x, y, flush)
            med, mn = timeit(op, x, y, None)
            got = y.clone()
            if ref is None:
                ref = got
                err = 0.0
            else:
                err = ((got - ref).abs().max() / ref.abs().max()).item()
            i = op.info()
            extra = ""
            if i["tile_blocks"]:
                extra = (f" blocks {i['tile_blocks']} maxrows {i['tile_max_rows']} maxstaged "
                         f"{i['tile_max_staged']} staged {i['tile_staged_deltas'] / max(1, i['tile_deltas']):.3f}"
                         f" reuse {i['tile_staged_deltas'] / max(1, i['tile_staged_rows']):.1f} cut {i['tile_cut_rows']}")
            print(f"  d={d} {v}: flush med {med_f:8.1f}us min {min_f:8.1f} | noflush med {med:8.1f}us"
                  f" | active {i['tile_active']} upload {up:.2f}s err {err:.2e}{extra}", flush=True)
