"""Dev tool: kernel time vs DeviceCbm upload options.

Usage: python tools/probe_split.py cfg3,cfg2 "32:32,128:32,256:64,1024:128"
       python tools/probe_split.py cfg1 '[{"max_segments": 2}, {}]'   (JSON option dicts)
"""
import json
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


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, device=dev)
    if sys.argv[2].lstrip().startswith("["):
        grid = json.loads(sys.argv[2])
    else:
        grid = [dict(zip(("split_threshold", "chunk"), (int(v) for v in g.split(":"))))
                for g in sys.argv[2].split(",")]
    for name in sys.argv[1].split(","):
        wl = WORKLOADS[name]
        a = wl.graph()
        c = wl.build(a, os.cpu_count() or 8)
        x = torch.from_numpy(wl.operand(a.n_cols)).to(dev)
        y = torch.empty((a.n_rows, wl.d), device=dev)
        ref = None
        for opts in grid:
            op = P.DeviceCbm(c, **opts)
            t = timeit(op, x, y, flush)
            got = y.clone()
            if ref is None:
                ref = got
            err = float((got - ref).abs().max() / ref.abs().max())
            info = op.info()
            print(f"{name} {json.dumps(opts):45s}: {t:9.1f} us  items={info['n_items']} "
                  f"chunks={info['n_chunk_items']} launches={info['launches_per_call']} "
                  f"err_vs_first={err:.2e}", flush=True)
            op.close()


if __name__ == "__main__":
    main()
