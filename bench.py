#!/usr/bin/env python
"""Benchmark of the CBM multiply Y = A.X on B200 (BASELINE.json metric).

Prints ONE JSON line on rank 0. A "step" is one multiply over the whole
workload (all d columns; rows x columns partitioned across ranks when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4_b256]
  python bench.py --impl reference ...   # the reference's own CPU path

Default workload: cfg4_b256 = BASELINE.json configs[4] (the "1/2/4/8 B200"
scaling sweep the metric is quoted on), binary A.X at d=256 — the largest
single-GPU configuration. The north_star's "config 3" (configs[3]: normalized
A_hat.X at d=256, the GCN's products) is measured in the same run and carried
as the `north_star_cfg3` key.

value    : effective GFLOP/s = 2 * nnz(represented A) * d / t, device-resident
           operands, CUDA events on the launching stream, L2 flushed (256 MiB
           write) before every timed step; whole job, max time over ranks.
parity   : before any timing, Y is compared with the reference's own
           spmm_into (oracle/_ref, the reference compiled from its sources) on
           the same CBM and X: bitwise for integer X on a binary matrix,
           max|G-R|/max|R| <= 1e-5 otherwise (north_star tolerance). A failed
           check withholds `value` (cbm_main.cpp:254-269 does the same).
e2e      : the same metric through the C-ABI host-buffer entry point
           (cbm_b200_spmm_host: pinned H2D of X, multiply, D2H of Y, sync).
roofline : B_alg per launch / kernel time against MEASURED_PEAKS.json
           hbm_gbs (DESIGN.md §6 Roofline).
cpu_baseline : the reference's spmm_into AND csr_spmm_into (oracle/_ref) on
           this host, pinned like pin_to_cores (cbm_main.cpp:92-104), at
           T = all host threads and T = 1; runtime_reduction_pct as
           cbm_main.cpp:276-283.
comparators : gpu_csr_comparator (the uncompressed matrix through the same
           kernels: the paper's runtime reduction on this GPU) and
           cusparse_comparator (cuSPARSE CSR SpMM fp32, the vendor bar);
           reported only, never on the product path.
north_star_cfg3 : configs[3] in the same run: A_hat.X at d=256 (value, roofline,
           parity) and its 2-layer GCN forward (gcn.cpp:22-33) timed and
           checked against the reference's gcn_forward.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CBM A·X effective GFLOP/s (2·nnz·d/t)"
UNIT = "GFLOP/s"
L2_FLUSH_BYTES = 256 << 20
TOL = 1e-5           # north_star: <= 1e-5 relative (normwise)
DEFAULT_CONFIG = "cfg4_b256"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=6.0,
                    help="seconds of reference work per CPU-baseline leg (bounded sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the pre-timing check (dev only: the line then has no value)")
    ap.add_argument("--no-north-star", action="store_true",
                    help="do not measure configs[3] beside the workload")
    ap.add_argument("--order-faithful", action="store_true")
    ap.add_argument("--kernel", default="auto", choices=["auto", "scalar"])
    ap.add_argument("--tile", type=int, default=-1, choices=[-1, 0, 1],
                    help="tiled path: -1 auto (community-structured matrices), 0 off, 1 force")
    ap.add_argument("--no-csr-comparator", action="store_true",
                    help="skip timing the uncompressed (CSR) matrix with the same kernel")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--row-groups", type=int, default=-1,
                    help="2-D partition (binary workloads): N = row groups x column slabs, "
                         "rank r owns Y[rows of group r // C, slab r % C] (DESIGN.md §7); "
                         "-1 = auto (sharding.auto_row_groups), 1 = column slabs only")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# launcher: --gpus N re-executes itself under torch.distributed.run
# ---------------------------------------------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args):
    """`python bench.py --gpus N` (N > 1, no torchrun env) -> one rank per GPU.
    Returns an exit code when it relaunched, None when this process is a rank."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # dev-only plumbing check of the N-rank code path on a one-GPU box:
    # BENCH_DEV_SHARE_GPU=1 puts every rank on cuda:0 with gloo collectives
    # (no data-path collective exists, so ranks never wait on each other's
    # kernels; numbers from such a run are not bench values)
    if os.environ.get("BENCH_DEV_SHARE_GPU") == "1":
        local = 0
    return rank, world, local


# ---------------------------------------------------------------------------
# shared helpers
# ---------------------------------------------------------------------------
def load_workloads():
    """The workload table, loaded by file path so the reference arm never
    imports (and so never loads) the product package."""
    path = os.path.join(ROOT, "paper_2409_02208_b200", "workloads.py")
    spec = importlib.util.spec_from_file_location("cbm_bench_workloads", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod.WORKLOADS


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(workload)
    return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/cbm_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def b_alg_bytes(nnz_delta, n_rows, n_cols, d, normalized):
    """4 nnz(Delta) + 12 n (+4 n normalized) + 4 d (n_cols + n_rows)."""
    s = 4 * nnz_delta + 12 * n_rows + (4 * n_rows if normalized else 0)
    return s + 4 * d * (n_cols + n_rows)


def represented_nnz(n_rows, row_ptr, col_idx, normalized):
    """nnz(A), or nnz(A + I) for the normalized operator (builder.cpp:452)."""
    nnz = int(row_ptr[-1])
    if not normalized:
        return nnz
    rp = np.asarray(row_ptr, np.int64)
    rows = np.repeat(np.arange(n_rows), np.diff(rp))
    has_diag = np.zeros(n_rows, bool)
    has_diag[rows[np.asarray(col_idx) == rows]] = True
    return nnz + int((~has_diag).sum())


def parity(got, want, exact):
    """SURVEY §8d gates: bitwise (integer X, binary) or normwise <= 1e-5."""
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    if got.shape != want.shape:
        return {"ok": False, "why": f"shape {got.shape} vs {want.shape}"}
    if exact:
        nd = int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
        return {"ok": nd == 0, "mode": "bitwise", "differing": nd}
    den = float(np.abs(want).max()) if want.size else 0.0
    num = float(np.abs(got.astype(np.float64) - want).max()) if want.size else 0.0
    err = num / den if den > 0 else num
    return {"ok": err <= TOL, "mode": f"normwise max|G-R|/max|R| <= {TOL:g}",
            "normwise_err": err}


class Pinned:
    """pin_to_cores (cbm_main.cpp:92-104): cores 0..T-1 for the CPU legs."""

    def __init__(self, threads):
        self.threads = threads

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        hw = os.cpu_count() or 1
        take = min(max(self.threads, 1), hw)
        try:
            os.sched_setaffinity(0, set(range(take)))
            self.ok = True
        except OSError:
            self.ok = False
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def time_reference(op, x, threads, seconds, n_rows):
    """Mean seconds per call of a reference operator (RefCbm: spmm_into,
    RefCsrReal: csr_spmm_into), one untimed warm-up first (time_runs,
    cbm_main.cpp:116-122), at least 2 calls, about `seconds` of work."""
    with Pinned(threads) as pin:
        t, runs = op.time_spmm(x, threads, 2, seconds)
    return t, runs, pin.ok


def cpu_legs(O, rc, rcsr, x, nnz, d, threads, seconds, flops_note):
    """The reference's CBM and CSR CPU paths at T = all and T = 1. The T = 1
    legs run on a column slab of X (columns are independent, kernels.cpp:27-62,
    so GFLOP/s is per-column work) sized to a bounded sample."""
    out = {"cores": threads, "cpu_model": cpu_model(), "pinned": True}
    legs = {}
    slab1 = d
    per_col = 2.0 * nnz
    # ~2 GFLOP per T=1 call at most (a few seconds of one core)
    while slab1 > 4 and per_col * slab1 > 2e9:
        slab1 //= 2
    x1 = np.ascontiguousarray(x[:, :slab1])
    for name, op in (("cbm", rc), ("csr", rcsr)):
        if op is None:
            continue
        for t, xx, w in ((threads, x, d), (1, x1, slab1)):
            s, runs, pinned = time_reference(op, xx, t, seconds, None)
            legs[f"{name}_t{'all' if t == threads else 1}"] = {
                "gflops": per_col * w / s / 1e9, "ms_per_call": s * 1e3, "threads": t,
                "columns": w, "calls": runs, "pinned": pinned}
    out["legs"] = legs
    if "cbm_tall" in legs and "csr_tall" in legs:
        tc, tr = legs["cbm_tall"]["ms_per_call"], legs["csr_tall"]["ms_per_call"]
        out["runtime_reduction_pct"] = (tr - tc) / tr * 100.0   # cbm_main.cpp:276-283
    if "cbm_t1" in legs and "csr_t1" in legs:
        tc, tr = legs["cbm_t1"]["ms_per_call"], legs["csr_t1"]["ms_per_call"]
        out["runtime_reduction_pct_t1"] = (tr - tc) / tr * 100.0
    out["note"] = flops_note
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU path (oracle/_ref), no product code
# ---------------------------------------------------------------------------
def ref_operands(O, wl):
    """Graph and X through the restated generators (oracle/gen_oracle.c)."""
    n, ncols, rp, ci = O.oracle_gen_graph(wl.graph_kind, list(wl.graph_params), wl.graph_seed)
    lo, hi = wl.x_range
    x = O.oracle_gen_dense(wl.x_kind, ncols, wl.d, wl.x_seed, lo, hi)
    return n, ncols, rp, ci, x


def run_reference(args, wl):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    t0 = time.perf_counter()
    n, ncols, rp, ci, x = ref_operands(O, wl)
    t_gen = time.perf_counter() - t0
    nnz = represented_nnz(n, rp, ci, wl.normalized)
    csr = O.RefCsr.from_arrays(n, ncols, rp, ci)
    # The reference's own builder is O(m^2) (builder.cpp:80-109):
    # it finishes in seconds only on the small configs. Where it does, the
    # timed path is its CBM spmm_into; otherwise its CSR csr_spmm_into on
    # to_real(A) / normalized_adjacency_csr(A) (kernels.cpp:152-168), the
    # stock path the reference's CLI times beside the CBM.
    t0 = time.perf_counter()
    if n <= 50000:
        op = O.RefCbm.build(csr, wl.alpha, args.threads, wl.normalized)
        path = "reference build_cbm + spmm_into (CBM)"
    else:
        op = O.RefCsrReal(csr, wl.normalized)
        path = ("reference csr_spmm_into on "
                + ("normalized_adjacency_csr(A)" if wl.normalized else "to_real(A)")
                + " (its build_cbm is O(m^2) here)")
    t_prep = time.perf_counter() - t0
    # bounded sample per step: a column slab of X sized to ~2-3 s of
    # all-thread work (columns are independent; GFLOP/s counts its own columns)
    w = wl.d
    while w > 4 and 2.0 * nnz * w > 50e9:
        w //= 2
    xs = np.ascontiguousarray(x[:, :w])
    with Pinned(args.threads):
        op.time_spmm(xs, args.threads, 1, 0.0)            # warm-up
        ts = []
        for _ in range(max(1, args.steps)):
            s, _r = op.time_spmm(xs, args.threads, 1, 0.0)
            ts.append(s)
    t = float(statistics.mean(ts))
    v = 2.0 * nnz * w / t / 1e9
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": len(ts),
           "warmup": 1, "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded generators restated in oracle/gen_oracle.c)",
           "impl": "reference",
           "config": {"workload": wl.name, "n": n, "nnz": nnz, "d": wl.d,
                      "alpha": wl.alpha, "normalized": wl.normalized, "path": path,
                      "columns_per_step": w, "gen_s": t_gen, "prep_s": t_prep},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": args.threads,
                            "cpu_model": cpu_model(), "kind": "reference",
                            "sample": f"{path}: X[:, :{w}] of the {wl.name} operand per step, "
                                      f"{len(ts)} steps after 1 warm-up, pinned to cores "
                                      f"0..{args.threads - 1}"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def time_steps(fn, steps, stream, flush):
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))             # L2 flush, outside the event pair
        starts[i].record(stream)
        fn()
        ends[i].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def roofline_for(info, ms, n_out, n_cols, d_local, normalized, workload):
    peak, peak_src = peaks()
    b_alg = b_alg_bytes(info["nnz_delta"], n_out, n_cols, d_local, normalized)
    achieved = b_alg / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    dense = bool(info["dense_active"]) and d_local >= 32
    tiled = not dense and bool(info["tile_active"]) and d_local >= 32
    if dense:
        # the tensor-core part loads one X row slice per chunk column, the cold
        # part gathers one per entry
        l2_bytes = (int(info["dense_chunks"]) * 32 + int(info["cold_entries"])) * d_local * 4
    elif tiled:
        l2_bytes = (int(info["tile_staged_rows"]) + int(info["tile_deltas"])
                    - int(info["tile_staged_deltas"])) * d_local * 4
    else:
        l2_bytes = int(info["nnz_effective"]) * d_local * 4
    hub = bool(info.get("hub_active")) and d_local >= 32
    if hub:
        # the hub-row panel loads one X row slice per chunk column for all of
        # its rows; nnz_effective above already excludes those rows
        l2_bytes += int(info["hub_chunks"]) * 32 * d_local * 4
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
         "frac": achieved / peak, "traffic": traffic_for(workload), "b_alg_bytes": b_alg,
         "kernel": (("dense_kernel (tcgen05) + cbm_kernel (cold entries)" if dense else
                     "tile_kernel" if tiled else "cbm_kernel")
                    + (" + dense_kernel (tcgen05, hub-row panel) + hub_reduce_kernel" if hub else "")),
         "peak_source": peak_src,
         # what bounds the gather: X rows moved L2 -> SM per step (one row per
         # summed delta)
         "l2_gather": {"bytes": l2_bytes,
                       "achieved_tbps": l2_bytes / (ms * 1e-3) / 1e12 if ms > 0 else 0.0}}
    if tiled:
        r["smem_gather_bytes"] = int(info["tile_staged_deltas"]) * d_local * 4
    if hub:
        r["hub_panel"] = {"rows": int(info["hub_rows"]), "entries": int(info["hub_entries"]),
                          "chunks": int(info["hub_chunks"])}
    return r


def cusparse_comparator(a, x, normalized, flops, ms, steps, stream, flush, dev):
    """The vendor bar: cuSPARSE CSR SpMM (fp32, through
    torch.sparse's CSR @ dense) on the same represented matrix and X. A reported
    comparator only: the product path never calls it."""
    import torch
    try:
        rp = np.asarray(a.row_ptr, np.int64)
        ci = np.asarray(a.col_idx, np.int64)
        if normalized:
            n = a.n_rows
            rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
            has_diag = np.zeros(n, bool)
            has_diag[rows[rows == ci]] = True
            add = np.nonzero(~has_diag)[0]
            rows = np.concatenate([rows, add])
            ci = np.concatenate([ci, add])
            o = np.lexsort((ci, rows))
            rows, ci = rows[o], ci[o]
            rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int64)
            s = (np.float32(1.0) / np.sqrt(np.diff(rp).astype(np.float64)).astype(np.float32))
            vals = (s[rows] * s[ci]).astype(np.float32)
        else:
            vals = np.ones(ci.size, np.float32)
        A = torch.sparse_csr_tensor(torch.from_numpy(rp).to(dev).to(torch.int32),
                                    torch.from_numpy(ci).to(dev).to(torch.int32),
                                    torch.from_numpy(vals).to(dev),
                                    size=(a.n_rows, a.n_cols))
        for _ in range(3):
            yy = torch.sparse.mm(A, x)
        torch.cuda.synchronize()
        holder = [yy]

        def fn():
            holder[0] = torch.sparse.mm(A, x)
        cs_ms = float(statistics.mean(time_steps(fn, steps, stream, flush)))
        return {"ms_per_step": cs_ms, "value": flops / (cs_ms * 1e-3) / 1e9,
                "ours_over_cusparse": cs_ms / ms if ms > 0 else None,
                "note": "cuSPARSE CSR SpMM fp32 via torch.sparse.mm (allocates its output "
                        "inside the timed call); reported comparator, not on the product path"}
    except Exception as e:  # the comparator must never take the bench line down
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


def run_north_star(args, P, O, WL, dev, stream, flush):
    """configs[3] (north_star "config 3"): normalized A_hat.X at d=256 on one
    GPU, parity-gated like the headline, same timing rules."""
    import torch
    wl = WL["cfg3"]
    a = wl.graph()
    nnz = represented_nnz(a.n_rows, a.row_ptr, a.col_idx, True)
    t0 = time.perf_counter()
    c = wl.build(a, args.threads)
    t_build = time.perf_counter() - t0
    op = P.DeviceCbm(c, device=dev.index)
    info = op.info()
    x_np = wl.operand(a.n_cols)
    x = torch.from_numpy(x_np).to(dev)
    y = torch.empty((a.n_rows, wl.d), dtype=torch.float32, device=dev)
    op.reserve(wl.d)
    op.spmm_into(x, y, stream)
    torch.cuda.synchronize()
    out = {"workload": "cfg3", "n": a.n_rows, "nnz": nnz, "nnz_delta": int(c.nnz), "d": wl.d,
           "alpha": wl.alpha, "build_s": t_build}
    if O is not None and O.ref_available():
        rc = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                                                 c.parent, c.row_ptr, c.col_idx, c.values,
                                                 c.row_scale))
        out["parity"] = O.judge_parity(
            y.cpu().numpy(), rc.spmm(x_np, args.threads), TOL,
            lambda cols: O.oracle_exact_spmm(a.row_ptr, a.col_idx, x_np[:, cols], c.row_scale,
                                             add_identity=True))
        out["parity"]["against"] = "reference spmm_into (oracle/_ref)"
    for _ in range(max(3, args.warmup)):
        op.spmm_into(x, y, stream)
    torch.cuda.synchronize()
    ms = float(statistics.mean(time_steps(lambda: op.spmm_into(x, y, stream),
                                          args.steps, stream, flush)))
    gated = out.get("parity", {}).get("ok", False)
    out["ms_per_step"] = ms
    out["value"] = 2.0 * nnz * wl.d / (ms * 1e-3) / 1e9 if gated else None
    out["unit"] = UNIT
    out["roofline"] = roofline_for(info, ms, a.n_rows, a.n_cols, wl.d, True, "cfg3")
    out["gpu_launches_per_step"] = int(op.info()["launches_per_call"])
    # configs[3] as BASELINE.json states it: 2-layer GCN inference
    # A_hat relu(A_hat X W0) W1 (gcn.cpp:22-33), X n x 128, W0 128 x 256, W1 256 x 112
    # (Glorot, seeded), the dense products by our GEMM kernel, A_hat. by the CBM path
    try:
        xg = P.generate_dense("normal", a.n_cols, 128, 0xC0F61003)
        w0 = P.generate_dense("glorot", 128, 256, 0xC0F62003)
        w1 = P.generate_dense("glorot", 256, 112, 0xC0F62103)
        tx, t0, t1 = (torch.from_numpy(t).to(dev) for t in (xg, w0, w1))
        got = op.gcn_forward(tx, t0, t1, stream)
        torch.cuda.synchronize()
        gcn = {"shape": "X n x 128, W0 128 x 256, W1 256 x 112"}
        if O is not None and O.ref_available():
            want = rc.gcn_forward(xg, w0, w1, args.threads)
            den = float(np.abs(want).max()) or 1.0
            err = float(np.abs(got.cpu().numpy().astype(np.float64) - want).max()) / den
            gcn["parity"] = {"ok": err <= TOL, "normwise_err": err,
                             "against": "reference gcn_forward (oracle/_ref)"}
        for _ in range(3):
            op.gcn_forward(tx, t0, t1, stream)
        torch.cuda.synchronize()
        gcn["ms_per_forward"] = float(statistics.mean(time_steps(
            lambda: op.gcn_forward(tx, t0, t1, stream), min(args.steps, 20), stream, flush)))
        gcn["gpu_launches_per_forward"] = int(op.info()["launches_per_call"])
        out["gcn_forward"] = gcn
    except Exception as e:  # an extra key must never take the bench line down
        out["gcn_forward"] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    op.close()
    return out


def run_ours(args, wl, WL):
    import torch
    rank, world, local = dist_env()
    share = os.environ.get("BENCH_DEV_SHARE_GPU") == "1"
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")         # init log: nranks per comm
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2409_02208_b200 as P
    O = None
    try:
        import oracle as O   # the checker and the CPU baseline only
    except OSError:
        O = None

    a = wl.graph()
    nnz = represented_nnz(a.n_rows, a.row_ptr, a.col_idx, wl.normalized)
    t0 = time.perf_counter()
    c = wl.build(a, args.threads)
    t_build = time.perf_counter() - t0
    from paper_2409_02208_b200.sharding import (auto_row_groups, column_slab, grid_position,
                                                row_partition)
    if args.row_groups < 0:
        args.row_groups = auto_row_groups(wl.d, world)
    group, slab_rank, n_slabs = grid_position(world, rank, args.row_groups)
    c_local, n_out, rows_g = c, a.n_rows, None
    if args.row_groups > 1:
        # this rank's row group (cross-group parents flattened); host-side
        # construction, outside every timed region like the build itself
        t0 = time.perf_counter()
        rows_g, c_local = row_partition(a, c, args.row_groups)[group]
        n_out = len(rows_g)
        t_build += time.perf_counter() - t0
    t0 = time.perf_counter()
    op = P.DeviceCbm(c_local, device=local, order_faithful=args.order_faithful,
                     kernel=args.kernel, tile=args.tile)
    torch.cuda.synchronize()
    t_upload = time.perf_counter() - t0
    info = op.info()

    lo, hi = column_slab(wl.d, n_slabs, slab_rank)
    d_local = hi - lo
    x_full = wl.operand(a.n_cols)
    x_host = torch.from_numpy(np.ascontiguousarray(x_full[:, lo:hi])).pin_memory()
    x = x_host.to(dev)
    y = torch.empty((n_out, d_local), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    op.reserve(max(1, d_local))
    stream = torch.cuda.current_stream()

    def step():
        if d_local:
            op.spmm_into(x, y, stream)

    # ---- parity gate (before any timing): this rank's block of Y against the
    # reference's spmm_into on the same CBM (cbm_main.cpp:254-269)
    step()
    torch.cuda.synchronize()
    gate = {"ok": False, "why": "not checked"}
    ref_cbm = None
    if args.no_parity:
        gate = {"ok": False, "why": "--no-parity"}
    elif O is not None and O.ref_available():
        # the reference multiplies the WHOLE matrix (a row block of a normalized
        # CBM is not a container it accepts); this rank's rows are taken from it
        ref_cbm = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha,
                                                      c.is_normalized, c.parent, c.row_ptr,
                                                      c.col_idx, c.values, c.row_scale))
        threads = max(1, args.threads // max(1, world))
        want = ref_cbm.spmm(x_host.numpy(), threads) if d_local else np.zeros((n_out, 0))
        if rows_g is not None:
            want = want[rows_g]
        if wl.x_kind == "int" and not wl.normalized:
            gate = parity(y.cpu().numpy(), want, exact=True)
        else:
            def exact(cols):
                e = O.oracle_exact_spmm(a.row_ptr, a.col_idx, x_host.numpy()[:, cols],
                                        c.row_scale if wl.normalized else None,
                                        add_identity=wl.normalized)
                return e if rows_g is None else e[rows_g]
            gate = O.judge_parity(y.cpu().numpy(), want, TOL, exact)
        gate["against"] = "reference spmm_into (oracle/_ref) on the same CBM and X"
        del want
    else:
        gate = {"ok": False, "why": "oracle/_ref not available"}

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    with sampler:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        dev_ms = time_steps(step, args.steps, stream, flush)
        if dist:
            dist.barrier()
        total_ms = float(sum(dev_ms))
        launches = op.info()["launches_per_call"] * args.steps if d_local else 0

        # e2e: C-ABI host-buffer entry point, pinned host memory
        y_host = torch.empty((n_out, d_local), dtype=torch.float32).pin_memory()
        e2e_steps = max(3, min(args.steps, 20))
        for _ in range(2):
            if d_local:
                op.spmm_host_ptr(x_host.data_ptr(), a.n_cols, d_local, y_host.data_ptr(),
                                 n_out, d_local, stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        es = torch.cuda.Event(enable_timing=True)
        ee = torch.cuda.Event(enable_timing=True)
        es.record(stream)
        for _ in range(e2e_steps):
            if d_local:
                op.spmm_host_ptr(x_host.data_ptr(), a.n_cols, d_local, y_host.data_ptr(),
                                 n_out, d_local, stream)
        ee.record(stream)
        torch.cuda.synchronize()
        e2e_ms = es.elapsed_time(ee) / e2e_steps
        if dist:
            dist.barrier()

    ok_local = 1.0 if gate.get("ok") else 0.0
    t = torch.tensor([total_ms, e2e_ms, -ok_local], dtype=torch.float64,
                     device="cpu" if share else dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, all_ok = float(t[0]), float(t[1]), float(t[2]) < 0
    ms = total_ms / args.steps

    flops = 2.0 * nnz * wl.d
    value = flops / (ms * 1e-3) / 1e9
    e2e_value = flops / (e2e_ms * 1e-3) / 1e9
    roofline = roofline_for(info, ms, n_out, a.n_cols, d_local, wl.normalized, wl.name)

    gpu_csr = None
    if not args.no_csr_comparator and args.row_groups == 1 and world == 1:
        # same kernel on the uncompressed matrix: the paper's runtime reduction
        # (t_csr - t_cbm) / t_csr, both on this B200
        csr_op = P.DeviceCbm(P.csr_operator(a, wl.normalized), device=local, tile=args.tile)
        csr_op.reserve(max(1, d_local))
        for _ in range(3):
            csr_op.spmm_into(x, y, stream)
        torch.cuda.synchronize()
        csr_ms = float(statistics.mean(time_steps(lambda: csr_op.spmm_into(x, y, stream),
                                                  min(args.steps, 20), stream, flush)))
        gpu_csr = {"ms_per_step": csr_ms, "value": flops / (csr_ms * 1e-3) / 1e9,
                   "runtime_reduction_pct": (csr_ms - ms) / csr_ms * 100.0,
                   "note": "uncompressed matrix through the same kernels (every parent virtual)"}
        csr_op.close()

    cusparse = None
    if not args.no_csr_comparator and args.row_groups == 1 and world == 1 and d_local:
        cusparse = cusparse_comparator(a, x, wl.normalized, flops, ms, min(args.steps, 20),
                                       stream, flush, dev)

    spmv = None
    if rank == 0 and world == 1:
        # spmv (d = 1, the lane-per-delta kernel) on the same whole matrix
        v = torch.from_numpy(wl.operand(a.n_cols, 1)).to(dev)
        u = torch.empty((n_out, 1), dtype=torch.float32, device=dev)
        op.reserve(1)
        for _ in range(3):
            op.spmv_into(v, u, stream)
        torch.cuda.synchronize()
        spmv_ms = float(statistics.mean(time_steps(lambda: op.spmv_into(v, u, stream),
                                                   min(args.steps, 20), stream, flush)))
        spmv = {"ms_per_call": spmv_ms, "value": 2.0 * nnz / (spmv_ms * 1e-3) / 1e9,
                "unit": UNIT, "kernel": "cbm_spmv_kernel", "l2": "flushed before every call"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and O is not None \
            and O.ref_available():
        if ref_cbm is None:
            ref_cbm = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha,
                                                          c.is_normalized, c.parent, c.row_ptr,
                                                          c.col_idx, c.values, c.row_scale))
        ref_csr = O.RefCsrReal(O.RefCsr.from_arrays(a.n_rows, a.n_cols, a.row_ptr, a.col_idx),
                               wl.normalized)
        legs = cpu_legs(O, ref_cbm, ref_csr, x_host.numpy(), nnz, wl.d, args.threads,
                        args.cpu_seconds, "reference spmm_into (CBM built by our builder, "
                        "field-identical to build_cbm, wrapped in the reference's validating "
                        "CbmMatrix) and csr_spmm_into on "
                        + ("normalized_adjacency_csr(A)" if wl.normalized else "to_real(A)"))
        cbm_all = legs["legs"]["cbm_tall"]
        cpu = {"value": cbm_all["gflops"], "unit": UNIT, "cores": args.threads,
               "kind": "reference",
               "sample": f"full {wl.name} multiply (reference spmm_into, f32 build) x "
                         f"{cbm_all['calls']} calls after 1 warm-up at T={args.threads}; T=1 "
                         f"legs on X[:, :{legs['legs']['cbm_t1']['columns']}]",
               **legs}
        del ref_csr
    del ref_cbm

    north = None
    if rank == 0 and world == 1 and not args.no_north_star and wl.name != "cfg3":
        op.close()   # free the headline matrix before the second workload
        north = run_north_star(args, P, O, WL, dev, stream, flush)

    out = {"metric": METRIC, "value": value if all_ok else None, "unit": UNIT,
           "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded generators, DESIGN.md §8)",
           "config": {"workload": wl.name, "note": wl.note, "n": a.n_rows, "nnz": nnz,
                      "nnz_delta": int(c.nnz), "nnz_delta_local": info["nnz_delta"],
                      "d": wl.d, "d_per_rank": d_local,
                      "alpha": wl.alpha, "normalized": wl.normalized,
                      "parallelism": (f"column-shard x{world}" if args.row_groups == 1 else
                                      f"{args.row_groups} row groups x {n_slabs} column slabs"),
                      "order_faithful": bool(args.order_faithful), "kernel": args.kernel,
                      "tile": args.tile,
                      "l2": "flushed (256 MiB write) before every timed step",
                      "levels": info["n_levels"], "chunk_items": info["n_chunk_items"],
                      "actual_ops_per_step": int(sum(P.count_scalar_ops(c_local)) * d_local),
                      "build_s": t_build, "upload_s": t_upload,
                      "seeds": {"graph": hex(wl.graph_seed), "x": hex(wl.x_seed)}},
           "parity": dict(gate, all_ranks_ok=all_ok),
           "roofline": roofline,
           "cpu_baseline": cpu,
           "gpu_csr_comparator": gpu_csr,
           "cusparse_comparator": cusparse,
           "spmv": spmv,
           "e2e": {"value": e2e_value, "unit": UNIT,
                   "h2d_bytes_per_step": int(a.n_cols * d_local * 4),
                   "d2h_bytes_per_step": int(n_out * d_local * 4),
                   "entry": "cbm_b200_spmm_host (C ABI, pinned host buffers)"},
           "gpu_launches": int(launches),
           "clocks": sampler.summary()}
    if north is not None:
        out["north_star_cfg3"] = north
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if all_ok else 1


def main():
    args = parse()
    rc = maybe_relaunch(args)
    if rc is not None:
        return rc
    WL = load_workloads()
    wl = WL[args.config]
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl, WL)


if __name__ == "__main__":
    sys.exit(main())
