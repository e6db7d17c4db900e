"""Key metrics + top stall reasons of an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
ni = h.index("Kernel Name")
keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Grid Size", "Block Size", "Waves Per SM", "Theoretical Occupancy", "Dynamic Shared Memory Per Block",
        "Compute (SM) Throughput", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Ipc Active"]
print(rows[1][ni][:120])
for r in rows[1:]:
    if r[mi] in keep:
        print(f"  {r[mi]:40s} {r[vi]:>12s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh, vals = rr[0], rr[2]
stalls = [(hh[i], float(vals[i])) for i in range(len(hh))
          if hh[i].startswith("smsp__average_warp_latency_issue_stalled_") and hh[i].endswith(".ratio")
          and vals[i].replace(".", "", 1).isdigit()]
stalls.sort(key=lambda x: -x[1])
print("  top stalls (cycles per issued instr):", ", ".join(f"{n.split('stalled_')[1].split('.')[0]}={v:.1f}" for n, v in stalls[:6]))
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]:
    if k in hh:
        print(f"  {k} = {vals[hh.index(k)]} {rr[1][hh.index(k)]}")
