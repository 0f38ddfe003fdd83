"""Summarise an .ncu-rep (dev tool): key metrics + stall reasons + hot SASS."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed_op_global_ld.sum"]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")][:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w); print(f"  {w:60s} {r[i]:>16s} {units[i]}")
    items = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try: items.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError: pass
    tot = sum(v for v, _ in items) or 1
    print("  stalls:", ", ".join(f"{h} {v/tot*100:.0f}%" for v, h in sorted(items, reverse=True)[:8]))
