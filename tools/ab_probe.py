"""Dev tool: A/B two in-tree builds of the library on the same box.

    python tools/ab_probe.py <alt.so> <rounds> cfg1,cfg3 [d]

Builds each workload's CBM once (cached as .npz under /tmp), then times the
multiply (CUDA events, L2 flushed before each call, median of 50) in fresh
subprocesses that load the default build (A) and the alternative (B),
interleaved round by round.
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cache_path(name):
    return f"/tmp/ab_{name}.npz"


def build(name):
    import paper_2409_02208_b200 as P
    from paper_2409_02208_b200.workloads import WORKLOADS
    wl = WORKLOADS[name]
    if os.path.exists(cache_path(name)):
        return
    a = wl.graph()
    c = wl.build(a, os.cpu_count() or 8)
    np.savez(cache_path(name), parent=c.parent, row_ptr=c.row_ptr, col_idx=c.col_idx,
             values=c.values, row_scale=c.row_scale if c.row_scale is not None else np.zeros(0),
             meta=np.array([c.n_rows, c.n_cols, c.alpha, int(c.is_normalized)]))


def time_one(name, d):
    import torch
    import paper_2409_02208_b200 as P
    from paper_2409_02208_b200.workloads import WORKLOADS
    wl = WORKLOADS[name]
    z = np.load(cache_path(name))
    m, n, alpha, norm = (int(v) for v in z["meta"])
    c = P.CbmMatrix(m, n, alpha, bool(norm), z["parent"], z["row_ptr"], z["col_idx"], z["values"],
                    z["row_scale"] if norm else None)
    d = d or wl.d
    x = torch.from_numpy(wl.operand(n, d)).cuda()
    y = torch.empty((m, d), device="cuda")
    op = P.DeviceCbm(c)
    flush = torch.empty(64 << 20, device="cuda")
    s = torch.cuda.current_stream()
    ts = []
    for i in range(55):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        op.spmm_into(x, y, s)
        e1.record(s)
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    # event times are quantized (~0.5 us): the mean keeps sub-quantum differences
    print(f"{np.mean(ts):.3f}" if os.environ.get("AB_MEAN") else f"{np.median(ts):.2f}")


def main():
    if sys.argv[1] == "--one":
        time_one(sys.argv[2], int(sys.argv[3]))
        return
    alt, rounds, names = sys.argv[1], int(sys.argv[2]), sys.argv[3].split(",")
    d = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    for name in names:
        build(name)
    res = {}
    for r in range(rounds):
        for name in names:
            for lib in ("libcbm_b200.so", alt):
                env = dict(os.environ, CBM_B200_LIB=lib.split(":")[0])
                if lib != "libcbm_b200.so" and os.environ.get("AB_ALT_ENV"):  # K=V for the B arm
                    k, v = os.environ["AB_ALT_ENV"].split("=", 1)
                    env[k] = v
                out = subprocess.run([sys.executable, __file__, "--one", name, str(d)], env=env,
                                     capture_output=True, text=True, check=True).stdout.strip()
                res.setdefault((name, lib), []).append(float(out))
                print(f"round {r} {name} {lib}: {out} us", flush=True)
    for (name, lib), v in sorted(res.items()):
        print(f"SUMMARY {name:6s} {lib:28s} median {np.median(v):9.2f} us  all {v}")


if __name__ == "__main__":
    main()
