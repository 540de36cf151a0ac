"""Key ncu 'details' metrics per kernel launch in a report."""
import csv, sys, subprocess
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Issued Warp Per Scheduler",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "SM Frequency", "L1/TEX Hit Rate", "Mem Busy", "Max Bandwidth",
        "Compute (SM) Throughput"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d["Metric Name"] in want:
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"], d["Metric Unit"])
