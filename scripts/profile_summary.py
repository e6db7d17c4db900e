"""Summarise the ncu evidence of scripts/profile_round.sh into profiles/<round>/ and
profiles/ncu_traffic.json (read by bench.py for roofline.traffic, keyed by config).

    CFG=sweep python scripts/profile_summary.py gpurun_out/prof profiles/r02
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
lines = []


def short(n):
    n = re.sub(r"\(.*", "", n).replace("seed::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return n[:48]


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    return h, rows[hi + 1:]


# ---- plain bench line
plain = [l for l in open(os.path.join(src, "plain.log")) if l.startswith("{")]
bench = json.loads(plain[-1]) if plain else {}
lines.append("# ncu evidence (" + os.path.basename(dst) + ")\n")
if bench:
    rf = bench.get("roofline", {})
    lines.append(f"Plain run (no profiler): {bench['ms_per_step']:.3f} ms/round, {bench['value']:.1f} tokens/s; "
                 f"K2 achieved {rf.get('achieved', 0):.0f} GB/s = {rf.get('frac', 0):.3f} of {rf.get('peak')} GB/s; "
                 f"algorithmic bytes per GEMM launch {rf.get('bytes_per_launch', 0)/1e6:.2f} MB.\n")

# ---- launch list (gpu__time_duration per launch), last two rounds
h, rs = read_ncu_csv(os.path.join(src, "launches.csv"))
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rs if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
ends = [i for i, (n, _) in enumerate(ks) if "rollback_commit" in n]
a, b = ends[-3] + 1, ends[-1] + 1
tail = ks[a:b]
agg = collections.OrderedDict()
for n, v in tail:
    x = agg.setdefault(short(n), [0, 0.0])
    x[0] += 1
    x[1] += v
tot = sum(v for _, v in tail)
unit = 1e3 if max(v for _, v in tail) > 1e3 else 1.0   # ns -> us when ncu printed ns
lines.append("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 2 --warmup 3 --no-cpu-baseline)\n")
lines.append("Cold-cache, serialised per-launch times (no PDL overlap), last two rounds, per round:\n")
lines.append("| kernel | launches | us / round | avg us | share |\n|---|---|---|---|---|")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {k} | {c/2:.0f} | {v/2/unit:.1f} | {v/c/unit:.2f} | {v/tot:.3f} |")
lines.append(f"\nSum of serialised kernel times per round: {tot/2/unit/1e3:.3f} ms.\n")

# ---- per-launch DRAM traffic of one round
h, rs = read_ncu_csv(os.path.join(src, "round_dram.csv"))
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
per = collections.OrderedDict()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rs:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[idi], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
gem = [d for d in per.values() if "gemm_splitk" in d["name"]]
tr = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in gem]
avg_tr = sum(tr) / max(len(tr), 1)
lines.append("## DRAM traffic per launch (one round, `dram__bytes_read.sum + dram__bytes_write.sum`)\n")
kinds = collections.OrderedDict()
for d in per.values():
    x = kinds.setdefault(short(d["name"]), [0, 0.0, 0.0])
    x[0] += 1
    x[1] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    x[2] += d.get("gpu__time_duration.sum", 0)
lines.append("| kernel | launches | MB / launch | us / launch (serialised) |\n|---|---|---|---|")
for k, (c, by, t) in kinds.items():
    lines.append(f"| {k} | {c} | {by/c/1e6:.2f} | {t/c:.2f} |")
if bench:
    alg = bench["roofline"]["bytes_per_launch"]
    lines.append(f"\nK2 (gemm_splitk) over the round's {len(gem)} launches: DRAM {avg_tr/1e6:.2f} MB per launch vs "
                 f"{alg/1e6:.2f} MB algorithmic (ratio {avg_tr/alg:.3f}).\n")
tpath = os.path.join(os.path.dirname(dst.rstrip('/')), "ncu_traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
traffic = {k: v for k, v in traffic.items() if isinstance(v, dict)}
cfgname = os.environ.get("CFG", "sweep")
traffic[cfgname] = {"k2_gemm": avg_tr, "source": f"{dst}/summary.md: ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                    f"mean over the {len(gem)} GEMM launches of one {cfgname} round"}
json.dump(traffic, open(tpath, "w"), indent=1)

# ---- full captures
for rep, what in (("gemm_gu_l1", "verify gate/up GEMM, layer 1"), ("gemm_qkv_l1", "verify QKV GEMM, layer 1"),
                  ("gemm_o_l1", "verify O GEMM, layer 1"), ("attn_l1", "verify attention, layer 1"),
                  ("k4", "K4 vocab_verify_kernel"), ("k1", "K1 draft_sample_kernel (draft step 2)")):
    p = os.path.join(src, rep + ".ncu-rep")
    if not os.path.exists(p):
        continue
    out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hh, uu, vv = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
            "launch__cluster_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
    lines.append(f"## Full capture: {what} (`--set full --clock-control none`)\n")
    lines.append("| metric | value |\n|---|---|")
    for w in want:
        if w in hh:
            i = hh.index(w)
            lines.append(f"| {w} | {vv[i]} {uu[i]} |")
    lines.append("")
    shutil.copy(p, os.path.join(dst, rep + ".ncu-rep"))

for f in ("launches.csv", "round_dram.csv"):
    shutil.copy(os.path.join(src, f), os.path.join(dst, f))
open(os.path.join(dst, "summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
