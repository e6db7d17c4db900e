"""One round (CFG, default the sweep shape) bracketed by cudaProfilerStart/Stop, for `ncu --profile-from-start off`."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import seedgen
import paper_2406_18200_b200 as pkg

CFG = os.environ.get("CFG", "sweep")
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
for _ in range(4):
    b = eng.schedule()
    eng.draft(b)
    eng.verify(b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
b = eng.schedule()
eng.draft(b)
eng.verify(b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
