"""Dev tool: per-warp timeline of one cbm_kernel call (CBM_B200_TRACE).

Usage: CBM_B200_TRACE=/tmp/t.txt python tools/trace_warps.py cfg1 [kernel-opts]
Runs a few multiplies of a workload, then summarises the last traced call:
start skew, time to first data, finish-time spread per warp and per SM.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2409_02208_b200 as P
    from paper_2409_02208_b200 import workloads as WL
    path = os.environ.get("CBM_B200_TRACE")
    assert path, "set CBM_B200_TRACE"
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    w = WL.WORKLOADS[name]
    a = w.graph()
    c = w.build(a, os.cpu_count() or 1)
    x = torch.from_numpy(w.operand(a.n_rows)).cuda()
    d = P.DeviceCbm(c)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    if os.path.exists(path):
        os.remove(path)
    for _ in range(4):
        flush.zero_()
        d.spmm(x)
    torch.cuda.synchronize()
    calls = open(path).read().split("call ")[1:]
    rows = np.array([[int(v) for v in l.split()] for l in calls[-1].splitlines()[1:]], np.int64)
    rows = rows[rows[:, 1] > 0]
    t0 = rows[:, 1].min()
    st, first, end = (rows[:, 1] - t0) / 1e3, (rows[:, 2] - t0) / 1e3, (rows[:, 3] - t0) / 1e3
    sm = rows[:, 4] & 0xFFFF
    nw = (rows[:, 4] >> 16) & 0xFFFF
    deltas = rows[:, 4] >> 32
    q = lambda a: " ".join(f"{v:7.2f}" for v in np.percentile(a, [0, 10, 50, 90, 99, 100]))
    info = d.info()
    span = end.max()
    gb = info["nnz_effective"] * w.d * 4 / 1e9
    print(f"{name}: warps {len(rows)}  span {span:.1f} us  gathers {gb:.2f} GB -> "
          f"{gb / span * 1e3:.1f} TB/s over the span  info {info}")
    print("  pctl 0/10/50/90/99/100 (us from first warp start)")
    print("  start      ", q(st))
    print("  first data ", q(first))
    print("  end        ", q(end))
    print("  busy       ", q(end - st))
    print("  tickets/w  ", q(nw), "   deltas/w", q(deltas))
    sm_end = np.array([end[sm == k].max() for k in np.unique(sm)])
    print("  SM finish  ", q(sm_end))
    # correlation of finish time with work
    print("  corr(end, deltas) = %.2f  corr(end, tickets) = %.2f" %
          (np.corrcoef(end, deltas)[0, 1], np.corrcoef(end, nw)[0, 1]))


if __name__ == "__main__":
    main()
