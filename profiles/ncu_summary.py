"""Print the key ncu metrics of a .ncu-rep (first profiled launch).

usage: python profiles/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum")
STALL = "smsp__pcsamp_warps_issue_stalled_"

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
name_i = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
if name_i is not None:
    print("kernel:", vals[name_i][:100])
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        print(f"  {k} = {vals[i]} {units[i]}")
stalls = []
for i, k in enumerate(hdr):
    if k.startswith(STALL) and not k.endswith("_not_issued"):
        try:
            stalls.append((float(vals[i].replace(",", "")), k[len(STALL):]))
        except ValueError:
            pass
tot = sum(v for v, _ in stalls) or 1.0
print("  top stall reasons (pc sampling):")
for v, k in sorted(stalls, reverse=True)[:8]:
    print(f"    {k:40s} {100 * v / tot:5.1f}%")
