"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the last K rounds."""
import collections
import csv
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
per_round = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
# a round ends with rollback_commit_kernel
ends = [i for i, (n, _) in enumerate(ks) if "rollback_commit" in n]
a, b = ends[-3] + 1, ends[-1] + 1
tail = ks[a:b]
nr = 2
def short(n):
    n = re.sub(r"\(.*", "", n).replace("seed::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return n[:50]
agg = collections.OrderedDict()
for n, v in tail:
    s = short(n)
    x = agg.setdefault(s, [0, 0.0])
    x[0] += 1
    x[1] += v
tot = sum(v for _, v in tail)
print(f"{len(tail)//nr} launches/round, kernel-time sum per round {tot/nr/1e6:.3f} ms")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} n/round={c/nr:6.1f} us/round={v/nr/1e3:9.1f} avg_us={v/c/1e3:8.2f} share={v/tot:.3f}")
