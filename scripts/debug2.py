import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import seedgen
import paper_2406_18200_b200 as pkg
def cuda(W):
    return {"embed": W["embed"].cuda(), "final_norm": W["final_norm"].cuda(), "lm_head": W["lm_head"].cuda(),
            "layers": [{k: v.cuda() for k, v in L.items()} for L in W["layers"]]}
ds, ts = seedgen.SHAPES["toy_draft"], seedgen.SHAPES["toy_target"]
dW, tW = cuda(seedgen.model_weights(ds, 2)), cuda(seedgen.model_weights(ts, 1))
prompts = seedgen.prompts("toy") + [[5, 6, 7, 8, 9]]
def run(cap, log):
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=14,
                         max_streams=4, max_batch=cap, max_ctx=256)
    for i, p in enumerate(prompts):
        eng.add_stream(i, p)
    while True:
        b = eng.schedule(cap)
        if not b: break
        eng.draft(b)
        zt0 = None
        eng.verify(b)
        torch.cuda.synchronize()
        zt, zd, xs = eng.last_round(len(b))
        for k, s in enumerate(b):
            log.append((s, eng.stream_info(s)["r"], xs[k].cpu().numpy().tolist(), zd[k].cpu().numpy(), zt[k].cpu().numpy()))
    out = [eng.tokens(i) for i in range(len(prompts))]
    eng.close()
    return out
la, lb, lc = [], [], []
oa = run(1, la); ob = run(2, lb); oc = run(1, lc)
print("C=1 twice equal:", oa == oc)
print("C=1 vs C=2 equal:", oa == ob)
for s in range(4): print(s, oa[s], ob[s])
# compare per (stream, round)
da = {(s, r): (x, zd, zt) for s, r, x, zd, zt in la}
db = {(s, r): (x, zd, zt) for s, r, x, zd, zt in lb}
for key in sorted(da):
    if key not in db: continue
    xa, zda, zta = da[key]; xb, zdb, ztb = db[key]
    dd = np.abs(zda - zdb).max(); dt = np.abs(zta - ztb).max()
    if xa != xb or dd > 0 or dt > 0:
        print("stream", key[0], "round(after)", key[1], "xs", xa, xb, "max|dzd|", dd, "max|dzt|", dt,
              "dzd rows", np.abs(zda - zdb).max(axis=1), "dzt rows", np.abs(zta - ztb).max(axis=1))
