"""Per-source-line warp-instruction and stall-sample counts of an ncu report (needs -lineinfo)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, res = None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] in ("Function Name", "Line No"):
        continue
    if len(r) > 7 and r[2] == "-":
        try:
            res.append((int(r[7]), int(r[4]), cur, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "stall" else 0
tot = sum(x[key] for x in res)
print("total", "stall samples" if key else "warp instructions", tot)
for x in sorted(res, key=lambda x: -x[key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{x[0]:9d} {x[1]:6d}  {x[2]}:{x[3]}  {x[4]}")
