import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import seedgen
from oracle import sampling as sp
from paper_2406_18200_b200 import ops
SEED = seedgen.PHILOX_SEED
B, g, V = 96, 4, 32000
zt, zd = seedgen.synthetic_logits(B, g, V, 1.0, 0.3, seed=1000*0 + V + g)
sids = np.arange(B, dtype=np.int64) * 7919
rs = (np.arange(B) % 5).astype(np.int32)
xs = np.random.default_rng(0).integers(0, V, size=(B, g)).astype(np.int32)
out = ops.verify(torch.from_numpy(zt).cuda(), torch.from_numpy(zd).cuda(), torch.from_numpy(xs).cuda(), 1.0, SEED, sids, rs)
st = out["stats"].cpu().numpy()
bad = 0
for b in range(B):
    rows = [zt[b, j] for j in range(g + 1)] + [zd[b, j] for j in range(g)]
    for r, z in enumerate(rows):
        a = sp.scaled_logits(z, 1.0).astype(np.float64)
        i = int(np.argmax(a)); m = a[i]; e = np.exp(a - m); e[i] = 0; l1 = np.log1p(e.sum())
        if abs(st[b, r, 0] - m) > 0 or abs(st[b, r, 1] - l1) > 1e-12:
            bad += 1
            if bad < 10:
                # which slice is missing?
                print("b", b, "row", r, "gpu m", st[b, r, 0], "ref m", m, "gpu l1p", st[b, r, 1], "ref", l1)
print("bad rows", bad, "of", B * (2 * g + 1))
