"""GPU parity of the forward path and the whole round, through the C ABI.

Forward (P4): per-layer parity on seeded hidden states / caches vs the bf16-faithful oracle,
per-row ||d delta||_inf / ||delta||_inf <= 2e-2 on the layer update; whole-model logits of
the toy and 2-layer 68M shapes within 2e-2 relative.
Round (P6): free-running toy rounds vs the oracle's own rounds; a decision may differ only
where the oracle's margin is inside the logits tolerance band (then the stream is no longer
compared).  P5/P8: cached == recomputed logits and capacity invariance (GPU only).
"""
import numpy as np
import pytest
import torch

import seedgen
from oracle import llama as ll
from oracle.scheduler import RoundScheduler
from oracle.seed_round import SeedOracle

pytestmark = pytest.mark.gpu
SEED = seedgen.PHILOX_SEED


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2406_18200_b200 as p
    return p


def _cuda(W):
    return {"embed": W["embed"].cuda(), "final_norm": W["final_norm"].cuda(), "lm_head": W["lm_head"].cuda(),
            "layers": [{k: v.cuda() for k, v in L.items()} if L is not None else None for L in W["layers"]]}


def _rel_rows(a, b):
    return (np.abs(a - b).max(axis=-1) / np.maximum(np.abs(b).max(axis=-1), 1e-30))


@pytest.mark.parametrize("name,M,ctx", [("toy_target", 5, 0), ("toy_target", 9, 37), ("toy_draft", 2, 130),
                                        ("llama_68m", 3, 0), ("llama_68m", 5, 300), ("llama2_7b", 15, 0),
                                        ("llama2_7b", 5, 290), ("llama2_7b", 1, 129), ("llama2_13b", 12, 300)])
def test_decoder_layer_vs_oracle(pkg, name, M, ctx):
    shape = seedgen.SHAPES[name]
    sh = ll.LlamaShape(**shape)
    L = seedgen.layer_weights(shape, 77, 0)
    x = seedgen.hidden_states(M, sh.d_model, seed=M + ctx)
    hk, dh = sh.kv_heads, sh.head_dim
    kp = seedgen.bf16_matrix(max(ctx, 1), hk * dh, seed=ctx + 1, std=1.0)[:ctx].reshape(ctx, hk, dh)
    vp = seedgen.bf16_matrix(max(ctx, 1), hk * dh, seed=ctx + 2, std=1.0)[:ctx].reshape(ctx, hk, dh)
    x_out, k_new, v_new = pkg.ops.decoder_layer(shape, {k: v.cuda() for k, v in L.items()}, torch.from_numpy(x).cuda(),
                                                ctx, kp.cuda().contiguous() if ctx else None,
                                                vp.cuda().contiguous() if ctx else None)
    ref_x, ref_k, ref_v = ll.layer_forward(sh, L, x, np.arange(ctx, ctx + M), kp.double().numpy(),
                                           vp.double().numpy(), mode="bf16")
    delta_gpu = x_out.double().cpu().numpy() - x
    delta_ref = ref_x - x
    assert _rel_rows(delta_gpu, delta_ref).max() < 2e-2
    kg = k_new.double().cpu().numpy().reshape(M, -1)
    assert _rel_rows(kg, ref_k.reshape(M, -1)).max() < 2e-2
    vg = v_new.double().cpu().numpy().reshape(M, -1)
    assert _rel_rows(vg, ref_v.reshape(M, -1)).max() < 2e-2


def _engine(pkg, dname, tname, gamma=4, T=1.0, max_new=16, streams=4, batch=4, max_ctx=256, bonus=True,
            dseed=seedgen.DRAFT_SEED, tseed=seedgen.TARGET_SEED):
    ds, ts = seedgen.SHAPES[dname], seedgen.SHAPES[tname]
    dW, tW = seedgen.model_weights(ds, dseed), seedgen.model_weights(ts, tseed)
    eng = pkg.SeedEngine(ds, _cuda(dW), ts, _cuda(tW), gamma=gamma, temperature=T, seed=SEED, bonus=bonus,
                         max_new=max_new, max_streams=streams, max_batch=batch, max_ctx=max_ctx)
    return eng, (ds, dW, ts, tW)


@pytest.mark.parametrize("dname,tname,n", [("toy_draft", "toy_target", 40), ("llama_68m", "llama_68m", 24)])
def test_forward_logits_vs_oracle(pkg, dname, tname, n):
    eng, (ds, dW, ts, tW) = _engine(pkg, dname, tname)
    toks = np.random.default_rng(1).integers(3, ts["vocab"], size=n).tolist()
    for which, shape, W in ((0, ds, dW), (1, ts, tW)):
        got = eng.forward_logits(which, toks).double().cpu().numpy()
        ref = ll.forward(ll.LlamaShape(**shape), W, toks, mode="bf16")
        assert _rel_rows(got, ref).max() < 2e-2
    eng.close()


@pytest.mark.parametrize("tname", ["llama2_7b", "llama2_13b"])
def test_forward_slice_full_width_vs_oracle(pkg, tname):
    """P4(ii): a 2-layer slice of the full-width target (d = 4096 / 5120, V = 32000) end to end,
    prefilled in several chunks, logits within 2e-2 of the bf16-faithful oracle."""
    ts = dict(seedgen.SHAPES[tname], n_layers=2)
    ds = seedgen.SHAPES["llama_68m"]
    dW, tW = seedgen.model_weights(ds, seedgen.DRAFT_SEED), seedgen.model_weights(ts, seedgen.TARGET_SEED)
    eng = pkg.SeedEngine(ds, _cuda(dW), ts, _cuda(tW), gamma=4, temperature=1.0, seed=SEED, max_new=8,
                         max_streams=1, max_batch=1, max_ctx=600)
    toks = np.random.default_rng(7).integers(3, ts["vocab"], size=300).tolist()   # > one 256-row chunk
    got = eng.forward_logits(1, toks).double().cpu().numpy()
    rows = [0, 1, 100, 255, 256, 299]                                             # sampled rows
    sh = ll.LlamaShape(**ts)
    ref = ll.forward_batch(sh, tW, [(toks, ll.KVCache(sh))], mode="bf16", logits_rows=[rows])[0]
    assert _rel_rows(got[rows], ref).max() < 2e-2
    eng.close()


def test_cached_round_logits_equal_recompute(pkg):
    """P5: the verify row for T[-1] (cached decode after rounds) equals a from-scratch forward over T."""
    eng, _ = _engine(pkg, "toy_draft", "toy_target", max_new=40)
    prompt = seedgen.prompts("toy")[0]
    eng.add_stream(0, prompt)
    for _ in range(5):
        b = eng.schedule()
        eng.draft(b)
        eng.verify(b)
        torch.cuda.synchronize()
    T = prompt + eng.tokens(0)
    b = eng.schedule()
    eng.draft(b)
    eng.verify(b)
    zt, zd, xs = eng.last_round(1)
    full = eng.forward_logits(1, T + xs[0].cpu().tolist())
    got = zt[0].cpu().numpy()
    ref = full[len(T) - 1:].cpu().numpy()
    assert _rel_rows(got, ref).max() < 1e-5
    eng.close()


def test_capacity_invariance_gpu(pkg):
    """P8 / S:218: tokens per stream identical for C in {1, 2, 4}."""
    outs = []
    prompts = seedgen.prompts("toy") + [[5, 6, 7, 8, 9]]
    for cap in (1, 2, 4):
        eng, _ = _engine(pkg, "toy_draft", "toy_target", max_new=14, streams=4, batch=cap)
        for i, p in enumerate(prompts):
            eng.add_stream(i, p)
        while True:
            b = eng.schedule(cap)
            if not b:
                break
            eng.draft(b)
            eng.verify(b)
        outs.append([eng.tokens(i) for i in range(len(prompts))])
        eng.close()
    assert outs[0] == outs[1] == outs[2]
    assert all(len(t) == 14 for t in outs[0])


@pytest.mark.parametrize("T,bonus", [(1.0, True), (0.2, True), (1.0, False)])
def test_toy_rounds_vs_oracle(pkg, T, bonus):
    """P6 (free-running): the GPU and the oracle run the toy workload independently."""
    cfg = seedgen.CONFIGS["toy"]
    eng, (ds, dW, ts, tW) = _engine(pkg, cfg["draft"], cfg["target"], gamma=cfg["gamma"], T=T,
                                    max_new=cfg["max_new"], streams=3, batch=3, bonus=bonus)
    orc = SeedOracle(ll.LlamaShape(**ts), tW, ll.LlamaShape(**ds), dW, gamma=cfg["gamma"], temperature=T, seed=SEED,
                     bonus=bonus, max_new=cfg["max_new"], keep_logits=True)
    prompts = seedgen.prompts("toy")
    for i, p in enumerate(prompts):
        eng.add_stream(i, p)
        orc.add_stream(i, p)
    while True:
        b = eng.schedule(3)
        if not b:
            break
        eng.draft(b)
        eng.verify(b)
    ref_out, rounds, _ = orc.run(3)
    band = 2e-2
    exact = 0
    for s in range(3):
        got, ref = eng.tokens(s), ref_out[s]
        assert len(got) == len(ref) == cfg["max_new"]
        if got == ref:
            exact += 1
            continue
        first = next(i for i in range(len(ref)) if got[i] != ref[i])
        pos = 0
        for recs in rounds:                       # find the oracle round that emitted position `first`
            rec = next((r for r in recs if r.sid == s), None)
            if rec is None:
                continue
            if pos + len(rec.emitted) > first:
                near = min(rec.draft_gaps + rec.accept_margins + [rec.race_gap])
                assert near < band, f"stream {s} diverges at {first} with oracle margin {near}"
                break
            pos += len(rec.emitted)
    assert exact >= 1
    eng.close()


@pytest.mark.parametrize("n_tok", [700, 1030])
def test_long_prefill_splits_vs_oracle(pkg, n_tok):
    """K3 split-KV path: a 1-layer full-width 7B prefill of 700 / 1030 tokens (chunks of 256 rows,
    rows attending to 3-5 splits of 256 keys merged by the last split to finish) against the
    bf16-faithful oracle on sampled rows."""
    ts = dict(seedgen.SHAPES["llama2_7b"], n_layers=1)
    ds = seedgen.SHAPES["llama_68m"]
    dW, tW = seedgen.model_weights(ds, seedgen.DRAFT_SEED), seedgen.model_weights(ts, seedgen.TARGET_SEED)
    eng = pkg.SeedEngine(ds, _cuda(dW), ts, _cuda(tW), gamma=4, temperature=1.0, seed=SEED, max_new=8,
                         max_streams=1, max_batch=1, max_ctx=1100)
    toks = np.random.default_rng(n_tok).integers(3, ts["vocab"], size=n_tok).tolist()
    got = eng.forward_logits(1, toks).double().cpu().numpy()
    rows = [0, 255, 256, 511, 512, 699, n_tok - 1]
    sh = ll.LlamaShape(**ts)
    ref = ll.forward_batch(sh, tW, [(toks, ll.KVCache(sh))], mode="bf16", logits_rows=[rows])[0]
    assert _rel_rows(got[rows], ref).max() < 2e-2
    eng.close()


_ROUNDS_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import seedgen, paper_2406_18200_b200 as pkg
ds = seedgen.SHAPES['llama_68m']
ts = dict(seedgen.SHAPES['llama2_7b'], n_layers=1)
dW, tW = seedgen.model_weights(ds, seedgen.DRAFT_SEED), seedgen.model_weights(ts, seedgen.TARGET_SEED)
cu = lambda W: {'embed': W['embed'].cuda(), 'final_norm': W['final_norm'].cuda(), 'lm_head': W['lm_head'].cuda(),
                'layers': [{k: v.cuda() for k, v in L.items()} for L in W['layers']]}
dWc, tWc = cu(dW), cu(tW)
rng = np.random.default_rng(5)
prompts = [rng.integers(3, ts['vocab'], size=int(rng.integers(60, 700))).tolist() for _ in range(32)]
def run(ids):
    eng = pkg.SeedEngine(ds, dWc, ts, tWc, gamma=4, temperature=1.0, seed=seedgen.PHILOX_SEED, max_new=64,
                         max_streams=32, max_batch=32, max_ctx=1024)
    for i in ids:
        eng.add_stream(i, prompts[i])
    for _ in range(3):
        b = eng.schedule()
        eng.round_host(b)
    zt, zd, xs = eng.last_round(len(ids))
    pos = {g: k for k, g in enumerate(b)}
    out = {g: (eng.tokens(g), zt[pos[g]].cpu().numpy(), zd[pos[g]].cpu().numpy()) for g in ids}
    eng.close()
    return out
big = run(list(range(32)))
for g in (0, 7, 31):
    small = run([g])[g]
    assert small[0] == big[g][0], (g, small[0], big[g][0])
    assert np.array_equal(small[1], big[g][1]), g
    assert np.array_equal(small[2], big[g][2]), g
print("ok")
"""


def test_batch_invariance_rounds(pkg, tmp_path):
    """R19: a stream's rounds -- tokens, target and draft logits -- are bit-identical whether it runs
    alone or in a batch of 32 streams with 60..700-token prompts (every GEMM reduction order is a
    function of the shape, every attention split / merge order a function of the key positions).
    Run in a subprocess so the 7B-width weights are freed afterwards."""
    import os
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", _ROUNDS_SCRIPT], capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
