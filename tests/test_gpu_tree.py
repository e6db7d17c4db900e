"""GPU parity of the k_config tree kernels (tree.cu: K1T draft_topk, K4T verify_tree) against
oracle/tree.py on the same seeded logits, through the C ABI (seed_ops.h).  Decisions bit-exact
except oracle-flagged near-ties (R16); the all-ones k_config also equals the chain kernel (K4).
"""
import numpy as np
import pytest
import torch

import seedgen
from oracle import philox as ph
from oracle import sampling as sp
from oracle import tree as tr

pytestmark = pytest.mark.gpu
SEED = seedgen.PHILOX_SEED


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_18200_b200 import ops as o
    return o


@pytest.mark.parametrize("V,B,m,T", [(32, 400, 2, 1.0), (32, 400, 4, 0.2), (32000, 48, 2, 1.0), (32000, 48, 3, 0.2),
                                     (32000, 24, 1, 1.0)])
def test_draft_topk_vs_oracle(ops, V, B, m, T):
    rng = np.random.default_rng(V + m)
    z = (rng.standard_normal((B, V)) * 2).astype(np.float32)
    sids = rng.integers(0, 2**31, size=B)
    rs = rng.integers(0, 30, size=B).astype(np.int32)
    node = 5
    got = ops.draft_topk(torch.from_numpy(z).cuda(), T, SEED, sids, rs, node, m).cpu().numpy()
    flagged = 0
    for b in range(B):
        a = sp.scaled_logits(z[b], T).astype(np.float64)
        u = ph.race_uniforms(SEED, int(sids[b]), int(rs[b]), ph.TAG_DRAFT, node + 1, V)
        top, gap = tr.race_top(a, u, m)
        if gap < 1e-6:
            flagged += 1
            continue
        assert got[b].tolist() == top, (b, got[b], top)
    assert flagged <= 1


def _tree_inputs(counts, B, V, sigma, noise, T, seed):
    """Per-stream node rows and the oracle's drafted tokens (drawn from the draft rows)."""
    parent, _ = tr.tree_shape(counts)
    nn = len(parent)
    rng = np.random.default_rng(seed)
    zt = (rng.standard_normal((B, nn, V)) * sigma).astype(np.float32)
    zd = (zt + rng.standard_normal((B, nn, V)) * noise).astype(np.float32)
    sids = np.arange(B, dtype=np.int64) * 104729 + seed
    rs = (np.arange(B) % 7).astype(np.int32)
    tok = np.zeros((B, nn), dtype=np.int32)
    trees = []
    for b in range(B):
        t = tr.draft_tree(lambda n, path, b=b: zd[b, n], counts, T, SEED, int(sids[b]), int(rs[b]))
        tok[b, 1:] = t.tokens[1:]
        trees.append(t)
    return zt, zd, tok, sids, rs, trees


@pytest.mark.parametrize("counts,V,B,sigma,noise,T", [((2, 2, 1), 32, 600, 1.0, 0.5, 1.0), ((3, 1), 32, 600, 1.0, 0.8, 1.0),
                                                      ((2, 2, 1), 32000, 48, 1.0, 0.3, 1.0),
                                                      ((4, 2, 1), 32000, 24, 3.0, 1.0, 0.2),
                                                      ((1, 1, 1, 1), 32000, 24, 1.0, 0.3, 1.0)])
def test_verify_tree_vs_oracle(ops, counts, V, B, sigma, noise, T):
    zt, zd, tok, sids, rs, trees = _tree_inputs(counts, B, V, sigma, noise, T, seed=len(counts) * 31 + V % 97)
    for bonus in (True, False):
        out = ops.verify_tree(torch.from_numpy(zt).cuda(), torch.from_numpy(zd).cuda(), torch.from_numpy(tok).cuda(),
                              counts, T, SEED, sids, rs, bonus=bonus)
        ot, oc, on = (out[k].cpu().numpy() for k in ("out_tok", "out_cnt", "out_node"))
        flagged = mism = 0
        for b in range(B):
            r = tr.verify_tree(lambda n, b=b: zt[b, n], lambda n, b=b: zd[b, n], trees[b], T, SEED, int(sids[b]),
                               int(rs[b]), bonus=bonus)
            if r.flags:
                flagged += 1
                continue
            same = ot[b, :oc[b]].tolist() == r.emitted and on[b, :len(r.accepted_nodes)].tolist() == r.accepted_nodes
            mism += not same
        assert mism == 0, f"{mism} unflagged mismatches"
        assert flagged <= max(1, B // 100)


def test_all_ones_tree_equals_chain_kernel(ops):
    """The all-ones k_config through K4T gives K4's (the chain kernel's) emitted tokens."""
    g, V, B, T = 4, 32000, 48, 1.0
    counts = (1,) * g
    zt, zd, tok, sids, rs, _ = _tree_inputs(counts, B, V, 1.0, 0.3, T, seed=99)
    tree = ops.verify_tree(torch.from_numpy(zt).cuda(), torch.from_numpy(zd).cuda(), torch.from_numpy(tok).cuda(),
                           counts, T, SEED, sids, rs)
    # chain layout: target rows 0..g, draft rows 0..g-1, drafted x_1..x_g = the tree's node tokens
    chain = ops.verify(torch.from_numpy(zt).cuda(), torch.from_numpy(zd[:, :g].copy()).cuda(),
                       torch.from_numpy(tok[:, 1:].copy()).cuda(), T, SEED, sids, rs, want_dbg=False)
    assert torch.equal(tree["out_cnt"], chain["out_cnt"])
    assert torch.equal(tree["out_tok"], chain["out_tok"])


def _rel_rows(a, b):
    return (np.abs(a - b).max(axis=-1) / np.maximum(np.abs(b).max(axis=-1), 1e-30))


@pytest.mark.parametrize("name,counts,ctx", [("toy_target", (2, 2, 1), 37), ("llama_68m", (3, 1), 300),
                                             ("llama2_7b", (2, 2, 1), 290), ("llama2_7b", (4, 2, 1), 129),
                                             ("llama2_7b", (1, 1, 1, 1), 200)])
def test_tree_layer_vs_oracle(ops, name, counts, ctx):
    """Tree attention (Figure 7): the GPU layer over a k_config tree (root + BFS nodes, RoPE at
    ctx + depth, ancestor mask) against the oracle's per-path causal layers; 2e-2 relative per row
    (bf16 GEMMs, like the decoder-layer test)."""
    from oracle import llama as ll
    parent, _ = tr.tree_shape(counts)
    M = len(parent)
    shape = seedgen.SHAPES[name]
    sh = ll.LlamaShape(**shape)
    L = seedgen.layer_weights(shape, 77, 0)
    x = seedgen.hidden_states(M, sh.d_model, seed=M + ctx)
    hk, dh = sh.kv_heads, sh.head_dim
    kp = seedgen.bf16_matrix(ctx, hk * dh, seed=ctx + 1, std=1.0).reshape(ctx, hk, dh)
    vp = seedgen.bf16_matrix(ctx, hk * dh, seed=ctx + 2, std=1.0).reshape(ctx, hk, dh)
    x_out, k_new, v_new = ops.decoder_layer_tree(shape, {k: v.cuda() for k, v in L.items()},
                                                 torch.from_numpy(x).cuda(), ctx, parent, kp.cuda().contiguous(),
                                                 vp.cuda().contiguous())
    ref_x, ref_k, ref_v = tr.tree_layer_forward(sh, L, x, parent, ctx, kp.double().numpy(), vp.double().numpy(),
                                                mode="bf16")
    assert _rel_rows(x_out.double().cpu().numpy() - x, ref_x - x).max() < 2e-2
    assert _rel_rows(k_new.double().cpu().numpy().reshape(M, -1), ref_k.reshape(M, -1)).max() < 2e-2
    assert _rel_rows(v_new.double().cpu().numpy().reshape(M, -1), ref_v.reshape(M, -1)).max() < 2e-2
    if all(c == 1 for c in counts):   # the chain tree is the causal layer bit for bit
        xo, kn, vn = ops.decoder_layer(shape, {k: v.cuda() for k, v in L.items()}, torch.from_numpy(x).cuda(), ctx,
                                       kp.cuda().contiguous(), vp.cuda().contiguous())
        assert torch.equal(xo, x_out) and torch.equal(kn, k_new) and torch.equal(vn, v_new)
