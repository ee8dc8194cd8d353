"""Key metrics of each kernel in an ncu report (details page, csv)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate",
        "L1/TEX Hit Rate", "No Eligible", "Mem Busy", "Max Bandwidth", "Dynamic Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
cur = None
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (d.get("ID"), d.get("Kernel Name", "")[:80])
    if k != cur:
        cur = k
        print("==", k[0], k[1])
    if d.get("Metric Name") in KEYS:
        print(f"   {d['Metric Name']:40s} {d['Metric Value']:>20s} {d['Metric Unit']}")
