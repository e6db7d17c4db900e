"""Real-execution GEMM trace of one GSM8K-shape round (profile mode): where the round's time goes."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import seedgen
import paper_2406_18200_b200 as pkg

cfg = seedgen.CONFIGS[os.environ.get("CFG", "gsm8k")]
ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
n = int(os.environ.get("STREAMS", cfg["n_streams"]))
g = cfg["gamma"]
prompts = seedgen.prompts(os.environ.get("CFG", "gsm8k"), n_streams=n)
dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=g, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=400,
                     max_streams=n, max_batch=n, max_ctx=max(len(p) for p in prompts) + 420, profile=True)
del dW, tW
for i, p in enumerate(prompts):
    eng.add_stream(i, p)
times = []
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
tr = eng.gemm_trace()
tm = np.array(times[4:]) * 1e3
print(f"host ms: schedule {tm[:,0].mean():.3f} draft-enqueue {tm[:,1].mean():.3f} verify-enqueue {tm[:,2].mean():.3f}"
      f" | wall per round (synced) {tm[:,3].mean():.3f}")
L_d, L_t = ds["n_layers"], ts["n_layers"]
nd = g * (5 * L_d + 1)
names = []
for j in range(g):
    for l in range(L_d):
        names += [f"d{j}.L{l}.qkv", f"d{j}.L{l}.attn", f"d{j}.L{l}.o", f"d{j}.L{l}.gu", f"d{j}.L{l}.down"]
    names.append(f"d{j}.lm")
for l in range(L_t):
    names += [f"t.L{l}.qkv", f"t.L{l}.attn", f"t.L{l}.o", f"t.L{l}.gu", f"t.L{l}.down"]
names.append("t.lm")
t0 = tr[0, 0]
prev_end = None
rows = []
for i, (s, rel, e) in enumerate(tr):
    gap = (rel - prev_end) / 1e3 if prev_end is not None else 0.0
    rows.append((names[i] if i < len(names) else str(i), (s - t0) / 1e3, (rel - t0) / 1e3, (e - t0) / 1e3,
                 (e - s) / 1e3, (e - max(rel, prev_end or rel)) / 1e3, gap))
    prev_end = e
span = (tr[-1, 2] - tr[0, 0]) / 1e3
print(f"traced launches {len(tr)}; first start -> last end {span:.1f} us")
draft_end = tr[nd - 1, 2]
print(f"draft phase (first GEMM start -> last draft GEMM end): {(draft_end - t0)/1e3:.1f} us")
vt = tr[nd:]
print(f"verify GEMMs: first start -> last end {(vt[-1,2]-vt[0,0])/1e3:.1f} us")
gaps = np.array([r[6] for r in rows[nd:]])
expo = np.array([r[5] for r in rows[nd:]])
print(f"verify: sum exposed GEMM time {expo.sum():.1f} us, sum gaps (prev end -> release) {gaps.sum():.1f} us")
kinds = {}
for r in rows[nd:]:
    k = r[0].split(".")[-1]
    kinds.setdefault(k, []).append((r[4], r[5], r[6]))
for k, v in kinds.items():
    v = np.array(v)
    print(f"  {k:5s} n={len(v):3d} span {v[:,0].mean():7.2f} exposed {v[:,1].mean():7.2f} gap-before {v[:,2].mean():7.2f} us")
dk = {}
for r in rows[:nd]:
    k = r[0].split(".")[-1]
    dk.setdefault(k, []).append((r[4], r[5], r[6]))
print("draft phase per kind:")
for k, v in dk.items():
    v = np.array(v)
    print(f"  {k:5s} n={len(v):3d} span {v[:,0].mean():7.2f} exposed {v[:,1].mean():7.2f} gap-before {v[:,2].mean():7.2f} us")
for r in rows[nd:nd + 15]:
    print("   ", " ".join(f"{x:9.2f}" if isinstance(x, float) else f"{x:12s}" for x in r))
if os.environ.get("SEED_CTA_TRACE") == "1":
    # per-CTA phases of the layer-1 verify GEMMs and the LM head, relative to the launch release
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
    # attention CTA phases (layer 1): start, release, tiles ready, chunk stored, ticket, end
    i = names.index("t.L1.attn")
    raw = eng.gemm_cta_trace(i).reshape(-1, 8)
    rel = tr[i, 1]
    used = raw[:, 5] >= tr[i, 0]
    ct = raw[used]
    print(f"t.L1.attn: {used.sum()} CTAs; release->end {(tr[i,2]-rel)/1e3:.2f} us; phase - release (us): min / med / max")
    for k, name in enumerate(["start", "release", "tiles", "stored", "ticket", "end"]):
        v = (ct[:, k] - rel) / 1e3
        v = v[ct[:, k] >= tr[i, 0]]
        if len(v):
            print(f"    {name:11s} {v.min():8.2f} {np.median(v):8.2f} {v.max():8.2f}")
