"""Isolated time of the vocabulary kernels (K1 draft sampler, K4 verification) at round shapes:
20 back-to-back launches captured in one CUDA graph, replayed, CUDA events (L2-warm logits, as
in the round where the LM head just wrote them).

    python scripts/vocab_bench.py [B] [gamma]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2406_18200_b200 import _lib

B = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = int(sys.argv[2]) if len(sys.argv) > 2 else 4
V, SEED = 32000, 0x5EED2406
torch.manual_seed(0)
zt = (torch.randn(B, g + 1, V, device="cuda") * 2).contiguous()
zd = (zt[:, :g] + torch.randn(B, g, V, device="cuda") * 0.5).contiguous()
xs = torch.randint(3, V, (B, g), dtype=torch.int32, device="cuda")
sids = torch.as_tensor((np.arange(B) * 7919 + 1).astype(np.int32), device="cuda")
rs = torch.as_tensor((np.arange(B) % 5).astype(np.int32), device="cuda")
zrow = zd[:, 0].contiguous()
out = torch.empty(B, dtype=torch.int32, device="cuda")
out_tok = torch.empty((B, g + 1), dtype=torch.int32, device="cuda")
out_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
out_acc = torch.empty(B, dtype=torch.int32, device="cuda")
L = _lib.load()
P = lambda t: t.data_ptr()
S = lambda: torch.cuda.current_stream().cuda_stream


def k1_call():
    assert L.seed_op_draft_sample(P(zrow), V, B, V, 1.0, SEED, P(sids), P(rs), 1, P(out), S()) == 0


def k4_call():
    assert L.seed_op_verify(P(zt), P(zd), P(xs), B, g, V, 1.0, SEED, P(sids), P(rs), 1, P(out_tok), P(out_cnt),
                            P(out_acc), None, None, S()) == 0


def timed(fn, reps=20, iters=10):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * iters)


k1 = timed(k1_call)
k4 = timed(k4_call)
print(f"B={B} gamma={g}: K1 {k1:.2f} us per launch, K4 {k4:.2f} us per launch")
