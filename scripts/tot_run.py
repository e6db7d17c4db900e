#!/usr/bin/env python
"""One ToT-BFS tree (Alg. 2) at a paper workload shape on the GPU, through the C ABI.

    python scripts/tot_run.py [--config gsm8k] [--depth 4] [--n 3] [--b 1] [--l 64]

Defaults follow App. D: GSM8K depth 4, CW 2, BW 7, n = 3 thoughts; b = 1 ("We select the
one with the highest values").  Random-init weights and seedgen prompts, so the thoughts are
noise; what is measured is the tree's wall time, rounds and emitted tokens per second with
every token produced by libseed (paper_2406_18200_b200.tot.EngineGenerator).
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import seedgen  # noqa: E402
import paper_2406_18200_b200 as pkg  # noqa: E402
from paper_2406_18200_b200 import tot  # noqa: E402

DEPTH = {"gsm8k": 4, "cw": 2, "bw": 7, "sweep": 4, "toy": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gsm8k")
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--l", type=int, default=64)
    ap.add_argument("--no-share", action="store_true", help="prefill every sibling (no seed_fork_stream)")
    ap.add_argument("--tree", default="", help="k_config tree rounds, e.g. 2,2,1 (default: the chain)")
    a = ap.parse_args()
    cfg = seedgen.CONFIGS[a.config]
    depth = a.depth or DEPTH[a.config]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    prompt = seedgen.prompts(a.config)[0]
    width = a.n * a.b
    max_ctx = len(prompt) + 8 + (depth + 1) * a.l + 128
    tree = [int(c) for c in a.tree.split(",")] if a.tree else None
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=cfg["gamma"], temperature=1.0, seed=seedgen.PHILOX_SEED,
                         max_new=a.l, max_streams=width, max_batch=width, max_ctx=max_ctx, tree=tree)
    V = ts["vocab"]
    tcfg = tot.ToTConfig(depth=depth, n=a.n, b=a.b, eval_prefix=(1, 29871), eval_suffix=(29901,),
                         digit_base=29896 if V > 29906 else 3)
    gen = tot.EngineGenerator(eng, share_prefix=not a.no_share)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tot.ToTBFS(gen, tcfg).build(prompt)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    streams = sum(c[1] for c in res.calls)
    print(json.dumps({"workload": a.config, "k_config": tree, "depth": depth, "n": a.n, "b": a.b, "l": a.l,
                      "scheduler_calls": len(res.calls), "streams": streams, "rounds": gen.rounds,
                      "prefills": gen.prefills, "t_admit_s": gen.t_add, "t_rounds_s": gen.t_rounds, "share_prefix": gen.share_prefix,
                      "tokens": streams * a.l, "wall_s": dt, "tokens_per_s_wall": streams * a.l / dt,
                      "ms_per_round_wall": 1e3 * dt / max(gen.rounds, 1),
                      "scores": [lv["scores"] for lv in res.levels], "answer_len": len(res.answer)}))
    eng.close()


if __name__ == "__main__":
    main()
