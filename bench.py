#!/usr/bin/env python
"""Benchmark of the CBM multiply Y = A.X on B200 (BASELINE.json metric).

Prints ONE JSON line on rank 0. A "step" is one multiply over the whole
workload (all d columns, column-sharded across ranks when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1]
  python bench.py --impl reference ...   # reference CPU path (oracle/_ref)

value    : effective GFLOP/s = 2 * nnz(represented A) * d / t, device-resident
           operands, CUDA events on the launching stream, L2 flushed (256 MiB
           write) before every timed step; whole job, max time over ranks.
e2e      : the same metric through the C-ABI host-buffer entry point
           (cbm_b200_spmm_host: pinned H2D of X, multiply, D2H of Y, sync).
roofline : B_alg / kernel time against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline : the reference's own spmm_into (compiled from its sources into
           oracle/_ref) on this host's cores, same CBM, same operand.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="bounded CPU-baseline sample (seconds of reference work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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


def represented_nnz(a, normalized):
    if not normalized:
        return a.nnz
    # nnz(A + I): add the diagonal entries that are missing
    rp, ci = a.row_ptr.astype(np.int64), a.col_idx
    rows = np.repeat(np.arange(a.n_rows), np.diff(rp))
    has_diag = np.zeros(a.n_rows, bool)
    has_diag[rows[ci == rows]] = True
    return a.nnz + int((~has_diag).sum())


# ---------------------------------------------------------------------------
def run_reference(args, wl):
    """--impl reference: the reference's own CPU spmm_into (oracle/_ref)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    a = wl.graph()
    nnz = represented_nnz(a, wl.normalized)
    t0 = time.perf_counter()
    if a.n_rows <= 50000:
        # the reference's own builder (builder.cpp:394-429)
        ra = O.RefCsr.from_arrays(a.n_rows, a.n_cols, a.row_ptr, a.col_idx)
        rc = O.RefCbm.build(ra, wl.alpha, args.threads, wl.normalized)
        built_by = "reference build_cbm"
    else:
        # O(m^2) reference builder is infeasible here: our builder's
        # output (field-identical on every size both can build) wrapped by the
        # reference's own validating constructors
        c = wl.build(a, args.threads)
        rc = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                                                 c.parent, c.row_ptr, c.col_idx, c.values,
                                                 c.row_scale))
        built_by = "ours (identical chain), wrapped in reference CbmMatrix"
    t_build = time.perf_counter() - t0
    x = wl.operand(a.n_cols)
    t, runs = rc.time_spmm(x, args.threads, max(1, args.steps), 0.0)
    flops = 2.0 * nnz * wl.d
    v = flops / t / 1e9
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": runs,
           "warmup": 1, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, DESIGN.md §Workloads)",
           "impl": "reference",
           "config": {"workload": wl.name, "n": a.n_rows, "nnz": nnz, "d": wl.d,
                      "alpha": wl.alpha, "normalized": wl.normalized,
                      "build_s": t_build, "built_by": built_by},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": args.threads,
                            "kind": "reference",
                            "sample": f"full {wl.name} multiply x {runs} calls after 1 warm-up "
                                      "(time_runs protocol, cbm_main.cpp:116-122)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_ours(args, wl):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if os.environ.get("BENCH_DEV_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2409_02208_b200 as P

    a = wl.graph()
    nnz = represented_nnz(a, wl.normalized)
    t0 = time.perf_counter()
    c = wl.build(a, args.threads)
    t_build = time.perf_counter() - t0
    from paper_2409_02208_b200.sharding import (auto_row_groups, column_slab, grid_position,
                                                row_partition)
    if args.row_groups < 0:
        args.row_groups = 1 if wl.normalized else auto_row_groups(wl.d, world)
    group, slab_rank, n_slabs = grid_position(world, rank, args.row_groups)
    c_local, n_out = c, a.n_rows
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
    del x_full
    x = x_host.to(dev)
    y = torch.empty((n_out, d_local), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    op.reserve(max(1, d_local))
    stream = torch.cuda.current_stream()

    def step():
        if d_local:
            op.spmm_into(x, y, stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    with sampler:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))             # L2 flush, outside the event pair
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        dev_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total_ms = float(sum(dev_ms))
        launches = op.info()["launches_per_call"] * args.steps if d_local else 0

        # e2e: C-ABI host-buffer entry point, pinned host memory
        y_host = torch.empty((n_out, d_local), dtype=torch.float32).pin_memory()
        e2e_steps = max(3, min(args.steps, 50))
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

    t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64,
                     device="cpu" if os.environ.get("BENCH_DEV_SHARE_GPU") == "1" else dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms = float(t[0]), float(t[1])
    ms = total_ms / args.steps

    flops = 2.0 * nnz * wl.d
    value = flops / (ms * 1e-3) / 1e9
    e2e_value = flops / (e2e_ms * 1e-3) / 1e9

    # roofline of the dominant (only) kernel: B_alg per launch / its duration.
    # With pre-scaling (normalized, dense rows) two kernels run; the step is
    # then attributed to the pair (documented in DESIGN.md).
    peak, peak_src = peaks()
    b_alg_local = b_alg_bytes(info["nnz_delta"], n_out, a.n_cols, d_local, wl.normalized)
    achieved = b_alg_local / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    tiled = bool(info["tile_active"]) and d_local >= 32
    if tiled:
        # tiled path: staged X rows come through L2 once per (block, slab) unit,
        # cold deltas gather their rows from L2, staged deltas read shared memory
        l2_bytes = (int(info["tile_staged_rows"]) + int(info["tile_deltas"])
                    - int(info["tile_staged_deltas"])) * d_local * 4
        smem_bytes = int(info["tile_staged_deltas"]) * d_local * 4
    else:
        l2_bytes = int(info["nnz_effective"]) * d_local * 4
        smem_bytes = 0
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_for(wl.name),
                "b_alg_bytes": b_alg_local, "kernel": "tile_kernel" if tiled else "cbm_kernel",
                "peak_source": peak_src,
                # what actually bounds the gather: X rows moved L2 -> SM per step
                # (one row per summed delta) against the measured gather rate of
                # profiles/r01_ubench_gather.txt
                "l2_gather": {"bytes": l2_bytes,
                              "achieved_tbps": l2_bytes / (ms * 1e-3) / 1e12 if ms > 0 else 0.0,
                              "measured_peak_tbps": 15.7}}
    if tiled:
        roofline["smem_gather"] = {
            "bytes": smem_bytes,
            "achieved_tbps": smem_bytes / (ms * 1e-3) / 1e12 if ms > 0 else 0.0,
            "staged_fraction": int(info["tile_staged_deltas"]) / max(1, int(info["tile_deltas"])),
            "blocks": int(info["tile_blocks"]),
            "note": "staged deltas read the shared-memory X tile (128 B/clk/SM LSU limit)"}

    gpu_csr = None
    if not args.no_csr_comparator and args.row_groups == 1:
        # same kernel on the uncompressed matrix: the paper's runtime reduction
        # (t_csr - t_cbm) / t_csr, both on this B200
        csr_op = P.DeviceCbm(P.csr_operator(a, wl.normalized), device=local)
        csr_op.reserve(max(1, d_local))
        if d_local:
            for _ in range(3):
                csr_op.spmm_into(x, y, stream)
        torch.cuda.synchronize()
        t_csr = []
        for i in range(min(args.steps, 50)):
            flush.fill_(float(i))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if d_local:
                csr_op.spmm_into(x, y, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            t_csr.append(e0.elapsed_time(e1))
        csr_ms = float(statistics.mean(t_csr))
        gpu_csr = {"ms_per_step": csr_ms, "value": flops / (csr_ms * 1e-3) / 1e9,
                   "runtime_reduction_pct": (csr_ms - ms) / csr_ms * 100.0,
                   "note": "uncompressed matrix through the same kernel (every parent virtual)"}
        del csr_op

    # spmv (d = 1, the lane-per-delta kernel) on the same matrix: reported
    # beside the headline, with the reference's spmv_into on the host cores
    spmv = None
    if rank == 0:
        v = torch.from_numpy(wl.operand(a.n_cols, 1)).to(dev)
        u = torch.empty((n_out, 1), dtype=torch.float32, device=dev)
        op.reserve(1)
        for _ in range(3):
            op.spmv_into(v, u, stream)
        torch.cuda.synchronize()
        t_v = []
        for i in range(min(args.steps, 50)):
            flush.fill_(float(i))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            op.spmv_into(v, u, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            t_v.append(e0.elapsed_time(e1))
        spmv_ms = float(statistics.mean(t_v))
        spmv = {"ms_per_call": spmv_ms, "value": 2.0 * nnz / (spmv_ms * 1e-3) / 1e9,
                "unit": UNIT, "kernel": "cbm_spmv_kernel", "l2": "flushed before every call"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, wl, c, nnz)
        if spmv is not None and cpu is not None:
            spmv["cpu_reference"] = cpu_spmv(args, wl, c, nnz)

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded generators, DESIGN.md §Workloads)",
           "config": {"workload": wl.name, "note": wl.note, "n": a.n_rows, "nnz": nnz,
                      "nnz_delta": info["nnz_delta"], "d": wl.d, "d_per_rank": d_local,
                      "alpha": wl.alpha, "normalized": wl.normalized,
                      "parallelism": (f"column-shard x{world}" if args.row_groups == 1 else
                                      f"{args.row_groups} row groups x {n_slabs} column slabs"),
                      "order_faithful": bool(args.order_faithful), "kernel": args.kernel,
                      "tile": args.tile,
                      "l2": "flushed (256 MiB write) before every timed step",
                      "levels": info["n_levels"], "chunk_items": info["n_chunk_items"],
                      "actual_ops_per_step": int(sum(P.count_scalar_ops(c_local)) * d_local),
                      "build_s": t_build, "upload_s": t_upload},
           "roofline": roofline,
           "cpu_baseline": cpu,
           "gpu_csr_comparator": gpu_csr,
           "spmv": spmv,
           "e2e": {"value": e2e_value, "unit": UNIT,
                   "h2d_bytes_per_step": int(a.n_cols * d_local * 4),
                   "d2h_bytes_per_step": int(n_out * d_local * 4),
                   "entry": "cbm_b200_spmm_host (C ABI, pinned host buffers)"},
           "gpu_launches": int(launches),
           "clocks": sampler.summary()}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(args, wl, c, nnz):
    """The reference's spmm_into on this host (oracle/_ref), same CBM and X."""
    import oracle as O
    if not O.ref_available():
        return None
    rc = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                                             c.parent, c.row_ptr, c.col_idx, c.values,
                                             c.row_scale))
    x = wl.operand(c.n_cols)
    t, runs = rc.time_spmm(x, args.threads, 3, args.cpu_seconds)
    return {"value": 2.0 * nnz * wl.d / t / 1e9, "unit": UNIT, "cores": args.threads,
            "kind": "reference",
            "sample": f"full {wl.name} multiply (reference spmm_into, f32 build) x {runs} calls "
                      f"after 1 warm-up, {t * 1e3:.2f} ms/call"}


def cpu_spmv(args, wl, c, nnz):
    """The reference's spmv_into on this host (oracle/_ref), same CBM, d = 1."""
    import oracle as O
    rc = O.RefCbm.from_arrays(O.RefCbmArrays(c.n_rows, c.n_cols, c.alpha, c.is_normalized,
                                             c.parent, c.row_ptr, c.col_idx, c.values,
                                             c.row_scale))
    v = wl.operand(c.n_cols, 1)
    t, runs = rc.time_spmv(v, args.threads, 3, min(2.0, args.cpu_seconds))
    return {"value": 2.0 * nnz / t / 1e9, "unit": UNIT, "cores": args.threads,
            "kind": "reference", "sample": f"spmv_into x {runs} calls, {t * 1e3:.3f} ms/call"}


def main():
    args = parse()
    from paper_2409_02208_b200.workloads import WORKLOADS
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())
