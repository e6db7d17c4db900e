"""ToT-BFS (Alg. 2) on the GPU round, through the C ABI.

1. The product driver builds a toy tree with every token from libseed (EngineGenerator).
2. Each generation call is re-run by the oracle (SeedOracle, same global ids and prefixes):
   tokens must match per stream, except a stream whose first differing token comes from an
   oracle decision inside the logits tolerance band (the rule of test_toy_rounds_vs_oracle).
3. The oracle's literal Alg. 2 (brute-force subset arg-max) replayed on the GPU's generations
   must choose the identical tree and answer.
"""
import numpy as np
import pytest
import torch

import seedgen
from oracle import llama as ll
from oracle import tot as otot
from oracle.seed_round import SeedOracle

pytestmark = pytest.mark.gpu
SEED = seedgen.PHILOX_SEED
BAND = 2e-2


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2406_18200_b200 as p
    return p


def _cuda(W):
    return {"embed": W["embed"].cuda(), "final_norm": W["final_norm"].cuda(), "lm_head": W["lm_head"].cuda(),
            "layers": [{k: v.cuda() for k, v in L.items()} for L in W["layers"]]}


def _check_call(models, gamma, max_new, prefixes, gids, got):
    """Returns the number of streams that match the oracle exactly; asserts the rest diverge
    only inside the tolerance band."""
    ds, dW, ts, tW = models
    orc = SeedOracle(ll.LlamaShape(**ts), tW, ll.LlamaShape(**ds), dW, gamma=gamma, temperature=1.0, seed=SEED,
                     max_new=max_new)
    for g, p in zip(gids, prefixes):
        orc.add_stream(g, p)
    ref_out, rounds, _ = orc.run(len(gids))
    exact = 0
    for g, out in zip(gids, got):
        ref = ref_out[g]
        assert len(out) == len(ref) == max_new
        if out == ref:
            exact += 1
            continue
        first = next(i for i in range(len(ref)) if out[i] != ref[i])
        pos = 0
        for recs in rounds:
            rec = next((r for r in recs if r.sid == g), None)
            if rec is None:
                continue
            if pos + len(rec.emitted) > first:
                near = min(rec.draft_gaps + rec.accept_margins + [rec.race_gap])
                assert near < BAND, f"stream {g} diverges at {first} with oracle margin {near}"
                break
            pos += len(rec.emitted)
    return exact


@pytest.mark.parametrize("depth,n,b", [(2, 3, 1), (3, 3, 2)])
def test_tot_bfs_vs_oracle(pkg, depth, n, b):
    from paper_2406_18200_b200 import tot as ptot
    cfg = seedgen.CONFIGS["toy"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    dW, tW = seedgen.model_weights(ds, seedgen.DRAFT_SEED), seedgen.model_weights(ts, seedgen.TARGET_SEED)
    max_new = 8
    eng = pkg.SeedEngine(ds, _cuda(dW), ts, _cuda(tW), gamma=cfg["gamma"], temperature=1.0, seed=SEED,
                         max_new=max_new, max_streams=n * b, max_batch=n * b, max_ctx=256)
    log = []
    gen = ptot.EngineGenerator(eng)

    def logged(prefixes, gids):
        outs = gen(prefixes, gids)
        log.append((prefixes, gids, outs))
        return outs

    tcfg = ptot.ToTConfig(depth=depth, n=n, b=b, eval_prefix=(1, 2), eval_suffix=(31,), digit_base=3)
    res = ptot.ToTBFS(logged, tcfg).build(seedgen.prompts("toy")[0])
    eng.close()
    assert len(log) == 2 * depth + 1 and gen.rounds > 0

    streams = exact = 0
    for prefixes, gids, outs in log:
        exact += _check_call((ds, dW, ts, tW), cfg["gamma"], max_new, prefixes, gids, outs)
        streams += len(gids)
    assert exact >= streams // 2

    replay = iter(log)

    def replayed(prefixes, gids):
        p, g, o = next(replay)
        assert p == prefixes and g == gids
        return o
    ans, levels, calls = otot.seed_bfs(seedgen.prompts("toy")[0], replayed, depth, n, b, (1, 2), (31,),
                                       digit_base=3)
    assert res.calls == calls and res.answer == ans
    for a, o in zip(res.levels, levels):
        assert a["states"] == o["states"] and a["scores"] == o["scores"] and a["keep"] == o["keep"]


@pytest.mark.parametrize("dname,tname,plen", [("toy_draft", "toy_target", 8), ("toy_draft", "toy_target", 77),
                                              ("toy_draft", "toy_target", 17), ("toy_draft", "toy_target", 18),
                                              ("llama_68m", "llama_68m", 150), ("llama_68m", "llama_68m", 145),
                                              ("llama_68m", "llama_68m", 146)])
def test_fork_stream_equals_add_stream(pkg, dname, tname, plen):
    """seed_fork_stream (shared full prefix pages + a copied partial page) == seed_add_stream."""
    ds, ts = seedgen.SHAPES[dname], seedgen.SHAPES[tname]
    dW = _cuda(seedgen.model_weights(ds, seedgen.DRAFT_SEED))
    tW = _cuda(seedgen.model_weights(ts, seedgen.TARGET_SEED))
    prompt = np.random.default_rng(plen).integers(3, ts["vocab"], size=plen).tolist()
    outs = []
    for fork in (False, True):
        eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=SEED, max_new=24, max_streams=4,
                             max_batch=4, max_ctx=512)
        eng.add_stream(10, prompt)
        for g in (11, 12, 13):
            eng.fork_stream(10, g) if fork else eng.add_stream(g, prompt)
        if fork:
            assert eng.stream_info(11)["pages"] == eng.stream_info(10)["pages"]
            with pytest.raises(pkg.SeedError):
                eng.fork_stream(99, 14)                      # unknown source
        eng.remove_stream(10)                                # shared prefix pages must outlive the source
        eng.add_stream(20, prompt[::-1])                     # reuses freed pages; must not clobber shared ones
        while True:
            b = eng.schedule()
            if not b:
                break
            eng.draft(b)
            eng.verify(b)
        outs.append([eng.tokens(g) for g in (11, 12, 13, 20)])
        if fork:
            with pytest.raises(pkg.SeedError):
                eng.fork_stream(12, 15)                      # source already ran rounds
        eng.close()
    assert outs[0] == outs[1]
    assert all(len(t) == 24 for t in outs[1])
    assert len({tuple(t) for t in outs[1]}) > 1              # distinct Philox streams per id


def test_tot_shared_prefix_same_tree(pkg):
    from paper_2406_18200_b200 import tot as ptot
    cfg = seedgen.CONFIGS["toy"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    dW = _cuda(seedgen.model_weights(ds, seedgen.DRAFT_SEED))
    tW = _cuda(seedgen.model_weights(ts, seedgen.TARGET_SEED))
    trees = []
    for share in (False, True):
        eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=cfg["gamma"], temperature=1.0, seed=SEED, max_new=8,
                             max_streams=6, max_batch=6, max_ctx=256)
        gen = ptot.EngineGenerator(eng, share_prefix=share)
        tcfg = ptot.ToTConfig(depth=3, n=3, b=2, eval_prefix=(1, 2), eval_suffix=(31,), digit_base=3)
        res = ptot.ToTBFS(gen, tcfg).build(seedgen.prompts("toy")[0])
        trees.append((res.answer, [(lv["states"], lv["scores"], lv["keep"]) for lv in res.levels], gen.prefills))
        eng.close()
    assert trees[0][:2] == trees[1][:2]
    assert trees[1][2] < trees[0][2]
