"""Dev tool: per-unit timeline of the tiled kernel (CBM_B200_TILE_TRACE).
  CBM_B200_TILE_TRACE=/tmp/t.txt python tools/trace_tile.py [n] [d] [opt=v,...]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_02208_b200 as P
from paper_2409_02208_b200.workloads import WORKLOADS
path = os.environ["CBM_B200_TILE_TRACE"]
arg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 else {}
opts.setdefault("tile", 1)
if arg in WORKLOADS:
    wl = WORKLOADS[arg]; a = wl.graph(); c = wl.build(a, os.cpu_count())
else:
    n = int(arg); a = P.generate_graph("community", [n, 500, 0.8, 13.0 / n], 0xC0F60003)
    c = P.build_cbm_normalized(a, 0, threads=os.cpu_count())
h = P.DeviceCbm(c, **opts)
x = torch.from_numpy(P.generate_dense("normal", a.n_cols, d, 1)).cuda()
y = torch.empty((a.n_rows, d), device="cuda")
flush = torch.empty(64 << 20, device="cuda")
if os.path.exists(path): os.remove(path)
for _ in range(3):
    flush.fill_(1.0); h.spmm_into(x, y); torch.cuda.synchronize()
lines = open(path).read().strip().split("\n")
last = max(i for i, l in enumerate(lines) if l.startswith("call"))
t = np.array([[int(v) for v in l.split()] for l in lines[last + 1:]], dtype=np.int64)
sm, t0, t1, t2 = t[:, 1], t[:, 2], t[:, 3], t[:, 4]
base = t0.min()
print(lines[last], "kernel span us", (t2.max() - base) / 1e3)
print("stage us: mean %.1f p50 %.1f max %.1f" % ((t1 - t0).mean() / 1e3, np.median(t1 - t0) / 1e3, (t1 - t0).max() / 1e3))
print("rows  us: mean %.1f p50 %.1f max %.1f min %.1f" % ((t2 - t1).mean() / 1e3, np.median(t2 - t1) / 1e3, (t2 - t1).max() / 1e3, (t2 - t1).min() / 1e3))
busy = np.zeros(sm.max() + 1); last_end = np.zeros(sm.max() + 1); first = np.full(sm.max() + 1, 1e30)
for s_, a_, c_ in zip(sm, t0, t2):
    busy[s_] += c_ - a_; last_end[s_] = max(last_end[s_], c_); first[s_] = min(first[s_], a_)
print("per-SM busy us: mean %.1f min %.1f max %.1f; SM end spread us: %.1f..%.1f" % (busy.mean() / 1e3, busy.min() / 1e3, busy.max() / 1e3, (last_end.min() - base) / 1e3, (last_end.max() - base) / 1e3))
print("units per SM: min %d max %d" % (np.bincount(sm).min(), np.bincount(sm).max()))
