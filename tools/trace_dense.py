"""Dev tool: summarise CTA 0's dense_kernel timeline (CBM_B200_DENSE_TRACE).

    CBM_B200_DENSE_TRACE=/tmp/t.txt python tools/time_workload.py cfg3 '{}'
    python tools/trace_dense.py /tmp/t.txt

Per role: the period between consecutive chunks it handles and the mean
cycles between its stamps (waits and work phases), over the last traced call.
"""
import sys

import numpy as np

ROLES = {0: ("MMA issuer", ["wait xfull", "wait bfull", "issue+commit"]),
         1: ("metadata loader", ["wait mempty", "copy+signal"]),
         2: ("B expander 0", ["wait mfull", "wait bempty", "fill+signal"]),
         3: ("X gatherer 0", ["wait mfull", "wait sempty", "issue+signal"]),
         4: ("converter set 0 / quarter 0", ["wait mfull", "wait sfull", "wait xempty",
                                             "LDS+split+tcgen05.st", "wait::st+signal"]),
         5: ("epilogue quarter 0 (per unit)", ["wait accfull", "drain+store"])}


def main():
    calls, cur = [], None
    for line in open(sys.argv[1]):
        if line.startswith("call"):
            cur = []
            calls.append(cur)
        elif cur is not None:
            cur.append([int(v) for v in line.split()])
    a = np.array(calls[-1], dtype=np.int64)
    t_min = a[:, 2][a[:, 2] > 0].min()
    for role, (name, phases) in ROLES.items():
        r = a[a[:, 0] == role]
        if len(r) < 3:
            continue
        r = r[np.argsort(r[:, 1])]
        period = np.diff(r[:, 2]) / np.maximum(1, np.diff(r[:, 1]))
        print(f"{name}: {len(r)} stamped, first at +{r[0, 2] - t_min} cyc, "
              f"median cycles per chunk index {np.median(period):.0f} (mean {period.mean():.0f})")
        for k, ph in enumerate(phases):
            d = r[:, 3 + k] - r[:, 2 + k]
            d = d[(r[:, 3 + k] > 0)]
            print(f"    {ph:24s} mean {d.mean():8.0f}  median {np.median(d):8.0f}  p95 {np.percentile(d, 95):8.0f}")


if __name__ == "__main__":
    main()
