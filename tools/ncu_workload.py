"""Dev tool: build a BASELINE workload and run a few multiplies, for ncu
captures (`ncu --set full -k regex:<kernel> -s 2 -c 1 python tools/ncu_workload.py cfg4_b256`).
Prints the event time of each call (not a bench number: under ncu the times
are replay times)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_02208_b200 as P  # noqa: E402
from paper_2409_02208_b200.workloads import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_b256"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
extra = dict(kv.split("=") for kv in sys.argv[3:])
wl = WORKLOADS[name]
t0 = time.time()
a = wl.graph()
c = P.csr_operator(a, wl.normalized) if extra.get("csr") == "1" else wl.build(a, os.cpu_count())
opts = {k: int(v) for k, v in extra.items() if k != "csr"}
op = P.DeviceCbm(c, device=0, **opts)
x = torch.from_numpy(wl.operand(a.n_cols)).cuda()
y = torch.empty((a.n_rows, wl.d), device="cuda")
print(f"prep {time.time() - t0:.1f}s info {op.info()}", flush=True)
s = torch.cuda.current_stream()
for i in range(calls):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    op.spmm_into(x, y, s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"call {i}: {e0.elapsed_time(e1):.3f} ms", flush=True)
