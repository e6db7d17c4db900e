#!/usr/bin/env python
"""Wall time of seed_add_stream (prefill of both models) vs prompt length; next-round evidence."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_2406_18200_b200 as pkg  # noqa: E402

for dname, tname in (("llama_68m", "llama2_7b"), ("llama_160m", "llama2_13b")):
    ds, ts = seedgen.SHAPES[dname], seedgen.SHAPES[tname]
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=1, max_new=8, max_streams=2, max_batch=2,
                         max_ctx=2100)
    rng = np.random.default_rng(0)
    gid = 0
    for n in (64, 256, 512, 1024, 2048):
        p = rng.integers(3, ts["vocab"], size=n).tolist()
        ts_ = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.add_stream(gid, p)
            torch.cuda.synchronize()
            ts_.append(time.perf_counter() - t0)
            eng.remove_stream(gid)
            gid += 1
        t = min(ts_)
        flops = 2 * 6.6e9 * n if tname == "llama2_7b" else 2 * 12.85e9 * n
        print(json.dumps({"target": tname, "prompt": n, "ms": round(1e3 * t, 2),
                          "target_tflops_per_s": round(flops / t / 1e12, 1)}))
    eng.close()
    del dW, tW
    torch.cuda.empty_cache()
