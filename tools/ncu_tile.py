"""Minimal driver for ncu captures of the tiled kernel (dev tool).
  python tools/ncu_tile.py [n] [d] [opt=v,...]   (community graph, blocks of 500)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_02208_b200 as P
from paper_2409_02208_b200.workloads import WORKLOADS
arg = sys.argv[1] if len(sys.argv) > 1 else "26500"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 else {"tile": 1}
if arg in WORKLOADS:
    wl = WORKLOADS[arg]
    a = wl.graph()
    c = wl.build(a, os.cpu_count())
else:
    a = P.generate_graph("community", [int(arg), 500, 0.8, 13.0 / int(arg)], 0xC0F60003)
    c = P.build_cbm_normalized(a, 0, threads=os.cpu_count())
n = a.n_rows
h = P.DeviceCbm(c, **opts)
x = torch.from_numpy(P.generate_dense("normal", n, d, 1)).cuda()
y = torch.empty((n, d), device="cuda")
for _ in range(3):
    h.spmm_into(x, y)
torch.cuda.synchronize()
print("ok", h.info()["tile_active"])
