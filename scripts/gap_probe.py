"""Where the host sits between rounds (CFG, default sweep): device-idle gap between round r's end
and round r+1's first enqueue, the device time from enqueue to the round's end, and host-side
phase times of seed_schedule_round / seed_draft_round / seed_verify."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import seedgen
import paper_2406_18200_b200 as pkg

CFG = os.environ.get("CFG", "sweep")
cfg = seedgen.CONFIGS[CFG]
ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
n, g = int(os.environ.get("STREAMS", cfg["n_streams"])), cfg["gamma"]
R = int(os.environ.get("ROUNDS", "20"))
prompts = seedgen.prompts(CFG, n_streams=n)
dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=g, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=(R + 20) * (g + 1),
                     max_streams=n, max_batch=n, max_ctx=max(len(p) for p in prompts) + (R + 20) * (g + 1) + 16, profile=True)
eng.set_profile(False)
del dW, tW
for i, p in enumerate(prompts):
    eng.add_stream(i, p)
for _ in range(5):
    b = eng.schedule()
    eng.draft(b)
    eng.verify(b)
eng.schedule(0)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
host = np.zeros((R, 3))
for r in range(R):
    t0 = time.perf_counter()
    b = eng.schedule()
    t1 = time.perf_counter()
    ev_s[r].record(st)
    eng.draft(b)
    t2 = time.perf_counter()
    eng.verify(b)
    t3 = time.perf_counter()
    ev_e[r].record(st)
    host[r] = (t1 - t0, t2 - t1, t3 - t2)
torch.cuda.synchronize()
gap = [ev_e[r].elapsed_time(ev_s[r + 1]) * 1e3 for r in range(R - 1)]
dev = [ev_s[r].elapsed_time(ev_e[r]) * 1e3 for r in range(R)]
tot = ev_s[0].elapsed_time(ev_e[R - 1]) / R * 1e3
print(f"{CFG} N={n}: per round {tot:.1f} us; device enqueue->end median {np.median(dev):.1f} us; "
      f"idle gap end->next enqueue median {np.median(gap):.1f} us (min {min(gap):.1f}, max {max(gap):.1f})")
print("host us median: schedule %.1f  draft %.1f  verify %.1f" % tuple(np.median(host, axis=0) * 1e6))

# profiled rounds: device event time enqueue->end vs the traced kernel span of the same round
eng.set_profile(True)
b = eng.schedule()
eng.draft(b)
eng.verify(b)
eng.schedule(0)
rows = []
for r in range(8):
    b = eng.schedule()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.draft(b)
    eng.verify(b)
    e1.record(st)
    eng.schedule(0)
    tr = eng.launch_trace()
    span = (tr[:, 2].max() - tr[:, 0].min()) / 1e3
    order = np.argsort(tr[:, 0])
    t = tr[order]
    gaps = np.maximum(0, t[1:, 0] - np.maximum.accumulate(t[:-1, 2])) / 1e3
    top = np.argsort(-gaps)[:5]
    rows.append((e0.elapsed_time(e1) * 1e3, span, gaps.sum(), [(int(i), int(t[i, 3]), int(t[i + 1, 3]), round(float(gaps[i]), 1)) for i in top]))
for ev, span, gs, top in rows:
    print(f"profiled: event {ev:.1f} us, traced span {span:.1f} us, outside span {ev - span:.1f} us, "
          f"idle inside span {gs:.1f} us; largest gaps (idx, kind, next kind, us) {top}")
