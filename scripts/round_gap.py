"""GPU idle time between consecutive rounds (host scheduling + graph launch), with CUDA events."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import seedgen
import paper_2406_18200_b200 as pkg

CFG = os.environ.get("CFG", "gsm8k")
cfg = seedgen.CONFIGS[CFG]
ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
n, g = int(os.environ.get("STREAMS", cfg["n_streams"])), cfg["gamma"]
prompts = seedgen.prompts(CFG, n_streams=n)
dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=g, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=400,
                     max_streams=n, max_batch=n, max_ctx=max(len(p) for p in prompts) + 420)
del dW, tW
for i, p in enumerate(prompts):
    eng.add_stream(i, p)
st = torch.cuda.current_stream()
for _ in range(3):
    b = eng.schedule()
    eng.draft(b)
    eng.verify(b)
torch.cuda.synchronize()
gaps, rounds = [], []
prev_end = None
for _ in range(12):
    b = eng.schedule()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.draft(b)
    eng.verify(b)
    e1.record(st)
    if prev_end is not None:
        gaps.append((prev_end, e0))
    rounds.append((e0, e1))
    prev_end = e1
torch.cuda.synchronize()
g_ms = [a.elapsed_time(b) for a, b in gaps]
r_ms = [a.elapsed_time(b) for a, b in rounds]
print(f"round (events around draft+verify) mean {np.mean(r_ms):.3f} ms; idle gap between rounds mean {np.mean(g_ms)*1e3:.1f} us "
      f"(min {np.min(g_ms)*1e3:.1f}, max {np.max(g_ms)*1e3:.1f})")
