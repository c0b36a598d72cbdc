"""Key ncu metrics for the kernels of a report: python tools_ncu_summary.py rep [regex]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "details", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", f"regex:{sys.argv[2]}"]
rows = list(csv.reader(subprocess.run(args, capture_output=True, text=True).stdout.splitlines()))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "L1/TEX Cache Throughput",
        "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "Theoretical Occupancy")
for r in rows[1:]:
    if r[mi] in want:
        print(f"{r[ki][:40]:40s} | {r[mi]:38s} {r[vi]} {r[ui]}")
