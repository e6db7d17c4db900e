import os, sys
sys.path.insert(0, os.getcwd())
import torch, seedgen
from paper_2406_18200_b200 import ops
for (N, K) in [(4096, 4096), (4096, 11008), (12288, 4096), (22016, 4096)]:
    W = seedgen.bf16_matrix(N, K, seed=1).cuda()
    X = seedgen.bf16_matrix(120, 4096 if K == 4096 else K, seed=2).cuda()
    Y120 = ops.gemm(W, X); Y120b = ops.gemm(W, X)
    Y15 = ops.gemm(W, X[:15].contiguous()); Y16 = ops.gemm(W, X[:16].contiguous()); Y64 = ops.gemm(W, X[:64].contiguous())
    Y1 = ops.gemm(W, X[7:8].contiguous())
    def cmp(a, b, name):
        d = (a != b)
        nz = d.nonzero()
        print(f"N={N} K={K} {name}: mismatches {int(d.sum())} max {float((a-b).abs().max()):.3e}",
              "first", nz[:4].tolist(), "cols mod 128", sorted(set((nz[:, 1] % 128).tolist()))[:10] if len(nz) else "")
    cmp(Y120, Y120b, "120 vs 120 again")
    cmp(Y120[:15], Y15, "120 vs 15")
    cmp(Y120[:16], Y16, "120 vs 16")
    cmp(Y120[:64], Y64, "120 vs 64")
    cmp(Y120[7:8], Y1, "120 vs 1")
