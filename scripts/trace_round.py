"""Device-timed breakdown of one round (profile mode): where the round's time goes.

    CFG=sweep STREAMS=24 python scripts/trace_round.py

Every libseed kernel of a round carries a %globaltimer record (first CTA start, first CTA past the
PDL wait, last CTA end, kind).  Each launch is charged its critical-path interval
[max(release, previous end), end]; the intervals partition the round's timeline.
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import seedgen
import paper_2406_18200_b200 as pkg

cfg_name = os.environ.get("CFG", "gsm8k")
cfg = seedgen.CONFIGS[cfg_name]
ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
n = int(os.environ.get("STREAMS", cfg["n_streams"]))
g = cfg["gamma"]
prompts = seedgen.prompts(cfg_name, n_streams=n)
dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=g, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=400,
                     max_streams=n, max_batch=n, max_ctx=max(len(p) for p in prompts) + 420, profile=True)
del dW, tW
for i, p in enumerate(prompts):
    eng.add_stream(i, p)
times, traces = [], []
for r in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = eng.schedule()
    t1 = time.perf_counter()
    eng.draft(b)
    t2 = time.perf_counter()
    eng.verify(b)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    times.append((t1 - t0, t2 - t1, t3 - t2, t4 - t0))
    if r >= 4:
        eng.schedule(0)
        traces.append(eng.launch_trace())
tm = np.array(times[4:]) * 1e3
print(f"{cfg_name} N={n}: host ms: schedule {tm[:,0].mean():.3f} draft-enqueue {tm[:,1].mean():.3f} "
      f"verify-enqueue {tm[:,2].mean():.3f} | wall per round (synced) {tm[:,3].mean():.3f}")

KIND = {1: "gemm", 2: "attn", 3: "K4", 4: "K1", 5: "embed", 6: "K5"}
L_d, L_t = ds["n_layers"], ts["n_layers"]
names = []
for j in range(g):
    if j == 0:   # later steps' embeddings are written by the previous step's K1 (EmbedNext)
        names.append(f"d{j}.embed")
    for l in range(L_d):
        names += [f"d{j}.L{l}.qkv", f"d{j}.L{l}.attn", f"d{j}.L{l}.o", f"d{j}.L{l}.gu", f"d{j}.L{l}.down"]
    names += [f"d{j}.lm", f"d{j}.K1"]
names.append("t.embed")
for l in range(L_t):
    names += [f"t.L{l}.qkv", f"t.L{l}.attn", f"t.L{l}.o", f"t.L{l}.gu", f"t.L{l}.down"]
names += ["t.lm", "t.K4", "t.K5"]


def exposed(tr):
    out, prev = [], None
    for s, r, e, k in tr:
        beg = max(r, prev) if prev is not None else r
        out.append((max(0, e - beg) / 1e3, (e - s) / 1e3, (r - prev) / 1e3 if prev is not None else 0.0))
        prev = e if prev is None else max(prev, e)
    return np.array(out)


assert len(traces[0]) == len(names), (len(traces[0]), len(names))
ex = np.stack([exposed(t) for t in traces])           # [rounds][launch][exposed, span, gap]
spans = np.array([(t[:, 2].max() - t[:, 0].min()) / 1e3 for t in traces])
print(f"traced launches {len(names)}; round span (first start -> last end) {np.median(spans):.1f} us "
      f"(min {spans.min():.1f}); sum of exposed {np.median(ex[:, :, 0].sum(1)):.1f} us")
kinds = traces[0][:, 3]
for k in sorted(set(kinds.tolist())):
    sel = kinds == k
    print(f"  {KIND.get(int(k), k):6s} n={sel.sum():4d} exposed/round {np.median(ex[:, sel, 0].sum(1)):8.1f} us")
nd = 1 + g * (5 * L_d + 2)
print(f"draft phase exposed {np.median(ex[:, :nd, 0].sum(1)):.1f} us; verify phase {np.median(ex[:, nd:, 0].sum(1)):.1f} us")


def per_kind(prefix, lo, hi):
    groups = {}
    for i in range(lo, hi):
        key = names[i].split(".")[-1]
        groups.setdefault(key, []).append(i)
    for key, idx in groups.items():
        v = np.median(ex[:, idx, :], axis=0)
        print(f"  {prefix} {key:6s} n={len(idx):3d} exposed {v[:,0].mean():7.2f} span {v[:,1].mean():7.2f} "
              f"gap-before {v[:,2].mean():6.2f} us")


print("draft phase per kind (median over rounds, mean over launches):")
per_kind("d", 0, nd)
print("verify phase per kind:")
per_kind("t", nd, len(names))
print("first verify layers (exposed, span, gap us):")
med = np.median(ex, axis=0)
for i in range(nd, nd + 12):
    print(f"    {names[i]:12s} {med[i,0]:8.2f} {med[i,1]:8.2f} {med[i,2]:8.2f}")
if os.environ.get("SEED_CTA_TRACE") == "1":
    tr = traces[-1]
    ph = ["release", "prod_done", "first_full", "mma_done", "acc0_ready", "epi_done", "end", "part_stored",
          "ticket", "reduced", "chunk0", "chunk1", "first_refill"]
    for want in ["t.L1.qkv", "t.L1.o", "t.L1.gu", "t.L1.down", "t.lm", "d1.L0.gu", "d1.L0.down", "d1.L0.o"]:
        i = names.index(want)
        ct = eng.gemm_cta_trace(i)[:512 * 16].reshape(512, 16)
        rel = tr[i, 1]
        used = ct[:, 7] >= tr[i, 0]
        ct = ct[used]
        print(f"{want}: {used.sum()} CTAs; release->end {(tr[i,2]-rel)/1e3:.2f} us; phase - release (us): min / med / max")
        for k, name in enumerate(ph):
            v = (ct[:, k + 1] - rel) / 1e3
            v = v[ct[:, k + 1] >= tr[i, 0]]
            if len(v) == 0:
                continue
            print(f"    {name:11s} {v.min():8.2f} {np.median(v):8.2f} {v.max():8.2f}")
        last = np.argmax(ct[:, 7])
        print("    last CTA:", " ".join(f"{(ct[last, k + 1] - rel)/1e3:.2f}" for k in range(len(ph))))
    for want in ["t.L1.attn", "d1.L0.attn", "d1.L1.attn"]:
        i = names.index(want)
        raw = eng.gemm_cta_trace(i).reshape(-1, 8)
        rel = tr[i, 1]
        used = raw[:, 5] >= tr[i, 0]
        ct = raw[used]
        print(f"{want}: {used.sum()} CTAs; release->end {(tr[i,2]-rel)/1e3:.2f} us; phase - release (us): min / med / max")
        for k, name in enumerate(["start", "release", "tiles", "stored", "merge", "end", "q_ready", "tile1_done"]):
            v = (ct[:, k] - rel) / 1e3
            v = v[ct[:, k] >= tr[i, 0]]
            if len(v):
                print(f"    {name:11s} {v.min():8.2f} {np.median(v):8.2f} {v.max():8.2f}")
eng.close()
