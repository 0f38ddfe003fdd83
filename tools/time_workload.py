"""Dev A/B timer: one BASELINE workload, several upload option sets, CUDA-event
timed multiplies with the L2 flushed before each, parity against the
reference's spmm_into (oracle/_ref). One JSON line per option set.

  python tools/time_workload.py cfg3 '{"dense":0}' '{"dense":1}' ...
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402


def main():
    name = sys.argv[1]
    sets = [json.loads(s) for s in sys.argv[2:]] or [{}]
    reps = int(os.environ.get("REPS", "10"))
    wl = WORKLOADS[name]
    t0 = time.time()
    a = wl.graph()
    c = wl.build(a, os.cpu_count())
    t_build = time.time() - t0
    nnz = a.nnz + (a.n_rows if wl.normalized else 0)
    x_np = wl.operand(a.n_cols)
    x = torch.from_numpy(x_np).cuda()
    y = torch.empty((a.n_rows, wl.d), device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    want = None
    if O.ref_available() and os.environ.get("NOCHECK") != "1":
        want = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                                                   c.parent, c.row_ptr, c.col_idx, c.values,
                                                   c.row_scale)).spmm(x_np, os.cpu_count())
    s = torch.cuda.current_stream()
    for opts in sets:
        opts = dict(opts)
        slab = int(opts.pop("_slab", 0))   # > 0: one launch per column slab of this width
        for k, v in opts.pop("_env", {}).items():   # dev env switches read per launch
            os.environ[k] = str(v)
        t0 = time.time()
        op = P.DeviceCbm(c, device=0, **opts)

        def mult():
            if slab <= 0:
                op.spmm_into(x, y, s)
            else:
                for lo in range(0, wl.d, slab):
                    op.spmm_into(x[:, lo:lo + slab], y[:, lo:lo + slab], s)
        t_up = time.time() - t0
        mult()
        torch.cuda.synchronize()
        out = {"workload": name, "opts": opts, "slab": slab, "build_s": t_build, "upload_s": t_up}
        if want is not None:
            out["parity"] = O.judge_parity(
                y.cpu().numpy(), want, 1e-5,
                lambda cols: O.oracle_exact_spmm(a.row_ptr, a.col_idx, x_np[:, cols],
                                                 c.row_scale if wl.normalized else None,
                                                 add_identity=wl.normalized))
        ts = []
        for i in range(reps + 2):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            mult()
            e1.record(s)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        info = op.info()
        ms = float(np.median(ts))
        out.update({"ms": ms, "ms_min": float(np.min(ts)),
                    "gflops": 2.0 * nnz * wl.d / (ms * 1e-3) / 1e9,
                    "info": {k: info[k] for k in ("dense_active", "dense_tiles", "dense_chunks",
                                                  "dense_entries", "cold_entries", "tile_active",
                                                  "nnz_effective", "launches_per_call")}})
        print(json.dumps(out), flush=True)
        op.close()


if __name__ == "__main__":
    main()
