"""Hottest SASS instructions (warp stall samples) of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((int(r[wi]), i, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{d[0]:6d} {100*d[0]/tot:5.1f}%  [{d[1]:4d}] {d[2][:90]}")
