"""Whole-round parity at the production shapes, through the C ABI.

Teacher-forced protocol: every round the oracle re-derives, from the GPU round's OWN logits,
  * each drafted token x_j (the DRAFT race on the GPU's draft row j, tag DRAFT slot j), and
  * the accept decisions, the accepted length a and the emitted tokens (accept / residual / bonus
    races on the GPU's target and draft rows; oracle.sampling.verify_stream),
and they must equal the GPU's bit for bit, except decisions the oracle flags as near-ties
(|u - rho| < 1e-6, race top-2 gap < 1e-6: R16), which must stay below 1e-5 of all decisions.
Forward fidelity is checked separately: per round, the GPU's verify logits of a 2-layer slice of
the full-width 7B target at 24 streams (multi-sequence paged attention with splits) against the
bf16-faithful oracle fed the same drafted tokens (P4, 2e-2 relative).
Shapes: GSM8K (N=3, 7B, gamma 4, T 1.0 and 0.2), Creative Writing (N=5, gamma 6), Blocksworld
(N=12, 13B + 160M, gamma 5), scaling sweep (N=24).  Inputs from seedgen only.
"""
import numpy as np
import pytest
import torch

import seedgen
from oracle import llama as ll
from oracle import sampling as sp
from oracle.seed_round import SeedOracle

pytestmark = pytest.mark.gpu
SEED = seedgen.PHILOX_SEED


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2406_18200_b200 as p
    return p


def _engine(pkg, cfg_name, T=1.0, n=None, max_new=None, target=None, bonus=True):
    cfg = seedgen.CONFIGS[cfg_name]
    ds = seedgen.SHAPES[cfg["draft"]]
    ts = target or seedgen.SHAPES[cfg["target"]]
    n = n or cfg["n_streams"]
    prompts = seedgen.prompts(cfg_name, n_streams=n)
    max_new = max_new or 40 * (cfg["gamma"] + 1)
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=cfg["gamma"], temperature=T, seed=SEED, bonus=bonus, max_new=max_new,
                         max_streams=n, max_batch=n, max_ctx=max(len(p) for p in prompts) + max_new + 8)
    del dW, tW
    torch.cuda.empty_cache()
    for i, p in enumerate(prompts):
        eng.add_stream(i, p)
    return eng, cfg, prompts


def _teacher_forced_rounds(eng, gamma, T, rounds, bonus=True):
    """Run `rounds` rounds; after each, re-derive every decision from the GPU's logits."""
    decisions = flagged = compared = 0
    for _ in range(rounds):
        b = eng.schedule()
        if not b:
            break
        r_of = {gid: eng.stream_info(gid)["r"] for gid in b}
        tok, cnt = eng.round_host(b)
        zt, zd, xs = (t.cpu().numpy() for t in eng.last_round(len(b)))
        for k, gid in enumerate(b):
            r = r_of[gid]
            for j in range(gamma):
                x, gap = sp.draft_token(zd[k, j], T, SEED, gid, r, j + 1)
                decisions += 1
                if gap < 1e-6:
                    flagged += 1
                else:
                    assert x == xs[k, j], (gid, r, j, x, xs[k, j])
            res = sp.verify_stream(zt[k], zd[k], xs[k].tolist(), T, SEED, gid, r, bonus=bonus)
            decisions += min(res.a + 1, gamma) + (1 if res.y is not None else 0)
            if res.flags:
                flagged += res.flags
                continue
            assert tok[k, :cnt[k]].tolist() == res.emitted, (gid, r, tok[k], res.emitted)
            compared += 1
    return decisions, flagged, compared


@pytest.mark.parametrize("cfg_name,T,rounds,n", [("gsm8k", 1.0, 20, None), ("gsm8k", 0.2, 20, None),
                                                 ("cw", 1.0, 20, None), ("sweep", 1.0, 20, 24)])
def test_teacher_forced_rounds_7b(pkg, cfg_name, T, rounds, n):
    eng, cfg, _ = _engine(pkg, cfg_name, T=T, n=n)
    decisions, flagged, compared = _teacher_forced_rounds(eng, cfg["gamma"], T, rounds)
    eng.close()
    print(f"{cfg_name} T={T}: {decisions} decisions, {flagged} flagged, {compared} stream-rounds compared")
    assert compared > 0.9 * rounds * (n or cfg["n_streams"])
    assert flagged <= max(1, 1e-5 * decisions)


def test_teacher_forced_rounds_13b(pkg):
    eng, cfg, _ = _engine(pkg, "bw", n=12)
    decisions, flagged, compared = _teacher_forced_rounds(eng, cfg["gamma"], 1.0, 12)
    eng.close()
    assert compared > 0.9 * 12 * 12
    assert flagged <= max(1, 1e-5 * decisions)


def test_teacher_forced_bonus_off(pkg):
    """bonus = 0 (Alg. 1 literal, R1): a = gamma emits x_1..x_gamma only."""
    eng, cfg, _ = _engine(pkg, "gsm8k", bonus=False)
    decisions, flagged, compared = _teacher_forced_rounds(eng, cfg["gamma"], 1.0, 10, bonus=False)
    eng.close()
    assert compared >= 27 and flagged <= 1


def test_round_logits_2layer_slice_vs_oracle(pkg):
    """P4 per round at the sweep batch: 24 streams with 40..300-token prompts (rows attending across
    split boundaries), a 2-layer slice of the full-width 7B target.  Each round the oracle runs the
    same verify inputs ([T[-1], x_1..x_gamma] with the GPU's drafted x) through its own cache and
    the GPU's emitted tokens are committed to both (teacher forcing)."""
    ts = dict(seedgen.SHAPES["llama2_7b"], n_layers=2)
    ds = seedgen.SHAPES["llama_68m"]
    g, n, T, max_new = 4, 24, 1.0, 30
    rng = np.random.default_rng(77)
    prompts = [rng.integers(3, ts["vocab"], size=int(rng.integers(40, 300))).tolist() for _ in range(n)]
    dW, tW = seedgen.model_weights(ds, seedgen.DRAFT_SEED), seedgen.model_weights(ts, seedgen.TARGET_SEED)
    cu = lambda W: {"embed": W["embed"].cuda(), "final_norm": W["final_norm"].cuda(),
                    "lm_head": W["lm_head"].cuda(), "layers": [{k: v.cuda() for k, v in L.items()} for L in W["layers"]]}
    eng = pkg.SeedEngine(ds, cu(dW), ts, cu(tW), gamma=g, temperature=T, seed=SEED, max_new=max_new, max_streams=n,
                         max_batch=n, max_ctx=400)
    orc = SeedOracle(ll.LlamaShape(**ts), tW, ll.LlamaShape(**ds), dW, gamma=g, temperature=T, seed=SEED,
                     max_new=max_new)
    for i, p in enumerate(prompts):
        eng.add_stream(i, p)
        orc.add_stream(i, p)
    worst = 0.0
    for _ in range(3):
        b = eng.schedule()
        tok, cnt = eng.round_host(b)
        zt, _, xs = eng.last_round(len(b))
        zt, xs = zt.double().cpu().numpy(), xs.cpu().numpy()
        ref = orc.verify(b, {gid: xs[k].tolist() for k, gid in enumerate(b)})
        for k, gid in enumerate(b):
            rel = np.abs(zt[k] - ref[gid]).max(axis=-1) / np.abs(ref[gid]).max(axis=-1)
            worst = max(worst, rel.max())
            orc.commit(orc.streams[gid], tok[k, :cnt[k]].tolist())
    eng.close()
    print(f"2-layer slice, 24 streams, 3 rounds: worst row rel err {worst:.3e}")
    assert worst < 2e-2


def test_device_error_word(pkg):
    """SEED_EDEVICE: non-finite draft logits (a NaN LM head) leave the draft race without a finite
    key (bit 2) and the next step's embedding gather sees id -1 (bit 1, read as id 0): reported by
    the next seed_schedule_round, cumulative in seed_device_status, context not poisoned."""
    cfg = seedgen.CONFIGS["toy"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    dW["lm_head"] = torch.full_like(dW["lm_head"], float("nan"))
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=SEED, max_new=8, max_streams=2,
                         max_batch=2, max_ctx=64)
    eng.add_stream(0, [3, 4, 5, 6])
    b = eng.schedule()
    eng.draft(b)
    eng.verify(b)
    with pytest.raises(pkg.SeedError) as e:
        eng.schedule()
    assert e.value.status == 7
    bits, _ = eng.device_status()
    assert bits & 2 and bits & 1
    eng.close()


def test_round_api_state_rules(pkg):
    """Calls that change streams are refused between seed_draft_round and seed_verify (ESTATE,
    not poisoning); an empty batch is a valid round; page sizes must hold whole 16-key tiles."""
    cfg = seedgen.CONFIGS["toy"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    dW = seedgen.model_weights(ds, seedgen.DRAFT_SEED, device="cuda")
    tW = seedgen.model_weights(ts, seedgen.TARGET_SEED, device="cuda")
    for bad in (8, 24, 48, 512):
        with pytest.raises(pkg.SeedError):
            pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=SEED, max_new=8, max_streams=2,
                           max_batch=2, max_ctx=64, page_tokens=bad)
    eng = pkg.SeedEngine(ds, dW, ts, tW, gamma=4, temperature=1.0, seed=SEED, max_new=8, max_streams=3,
                         max_batch=3, max_ctx=64, page_tokens=32)
    eng.add_stream(0, [3, 4, 5, 6])
    eng.add_stream(1, [7, 8, 9])
    b = eng.schedule()
    eng.draft(b)
    for call in (lambda: eng.add_stream(2, [3, 4]), lambda: eng.remove_stream(0), lambda: eng.fork_stream(0, 5),
                 lambda: eng.forward_logits(1, [3, 4])):
        with pytest.raises(pkg.SeedError) as e:
            call()
        assert e.value.status == 5
    eng.verify(b)
    assert eng.global_pending() == 2
    eng.draft([])
    eng.verify([])                       # an empty round (a rank whose streams are done, world > 1)
    while eng.global_pending() > 0:
        b = eng.schedule()
        eng.draft(b)
        eng.verify(b)
    assert len(eng.tokens(0)) == 8 and len(eng.tokens(1)) == 8
    eng.remove_stream(0)
    eng.add_stream(0, [3, 4, 5, 6])      # a removed id may be added again, from scratch
    assert eng.tokens(0) == []
    eng.close()


@pytest.mark.parametrize("n", [48, 192])
def test_teacher_forced_rounds_large_n(pkg, n):
    """Scaling-sweep shape beyond one 256-row token tile (BASELINE configs[4], N up to 192 on one GPU):
    the verify forward runs M = 5n rows in token tiles of 256 (weights streamed once per token tile,
    L2-shared), draft step 1 runs 2n rows; decisions re-derived from the GPU's logits as above."""
    eng, cfg, _ = _engine(pkg, "sweep", n=n, max_new=40)
    decisions, flagged, compared = _teacher_forced_rounds(eng, cfg["gamma"], 1.0, 3)
    eng.close()
    assert compared > 0.9 * 3 * n
    assert flagged <= max(1, 1e-5 * decisions)
