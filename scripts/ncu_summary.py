"""Compact summary of one ncu --set full capture (raw page CSV) for profiles/:
duration, DRAM traffic, pipe utilisations, issue activity and the top warp-stall reasons.

  python scripts/ncu_summary.py <raw.csv> [label]"""
import csv
import sys

path = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else path
rows = [r for r in csv.reader(ln for ln in open(path) if not ln.startswith("=="))]
hdr, units = rows[0], rows[1]
data_rows = rows[2:]  # one row per captured kernel

keys = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
for data in data_rows:
    get = {h: (data[i], units[i]) for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: {label}")
    for k in keys:
        if k in get:
            v, u = get[k]
            print(f"{k:70s} {v} {u}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((int(data[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1
    print("top warp-stall reasons (pc samples):")
    for v, h in sorted(stalls, reverse=True)[:6]:
        print(f"  {h:30s} {v:8d}  {100.0 * v / tot:5.1f}%")
