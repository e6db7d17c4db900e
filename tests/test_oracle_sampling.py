"""Oracle pins for speculative sampling -- all CPU, no GPU.

Pins: SPEC worked example, q == p accepts all (north_star),
exact enumeration losslessness, chi-square goodness of fit for
the race sampler and for the whole round (north_star: alpha = 0.01, 1e6
samples), alpha = sum min(p, q), closed-form E[emitted]
(Leviathan et al. eq. 1), log-softmax against scipy / mpmath.
"""
import itertools
import math
import os

import mpmath
import numpy as np
import pytest
from scipy import special, stats

from oracle import philox as ph
from oracle import sampling as sp

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_example.txt")
SEED = 0x5EED2406


def _gold():
    d = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        d[k] = [float(x) for x in v]
    return d


def test_spec_worked_example():
    g = _gold()
    zt, zd = np.log(g["p_t"]), np.log(g["p_d"])
    lp = sp.logsoftmax_tail(sp.scaled_logits(zt, 1.0))
    lq = sp.logsoftmax_tail(sp.scaled_logits(zd, 1.0))
    x = int(g["drafted"][0])
    assert abs(sp.accept_prob(lp[x], lq[x]) - g["accept"][0]) < 1e-6
    w = sp.residual_logweights(lp, lq)
    res = np.exp(w - np.max(w))
    res /= res.sum()
    np.testing.assert_allclose(res, g["residual"], atol=1e-12)


def test_logsoftmax_matches_scipy_and_mpmath():
    rng = np.random.default_rng(0)
    for T in (1.0, 0.2):
        z = (rng.standard_normal(1000) * 3).astype(np.float32)
        a = sp.scaled_logits(z, T)
        np.testing.assert_allclose(sp.logsoftmax_tail(a), special.log_softmax(a.astype(np.float64)), atol=1e-12)
    # low temperature: the top probability is 1 - O(1e-8); the tail form keeps log p exact
    a = np.array([0.0, -18.0, -19.5, -25.0], dtype=np.float32)
    lp = sp.logsoftmax_tail(a)
    mp = [float(mpmath.mpf(float(x)) - mpmath.log(sum(mpmath.e ** mpmath.mpf(float(y)) for y in a))) for x in a]
    np.testing.assert_allclose(lp, mp, rtol=1e-14, atol=1e-15)


def test_q_equals_p_accepts_everything():
    rng = np.random.default_rng(1)
    for T in (1.0, 0.2):
        for gamma in (1, 4, 6):
            zt = (rng.standard_normal((gamma + 1, 64)) * 2).astype(np.float32)
            zd = zt[:gamma].copy()
            xs = [int(rng.integers(0, 64)) for _ in range(gamma)]
            for sid in range(20):
                r = sp.verify_stream(zt, zd, xs, T, SEED, sid, 0, bonus=True)
                assert r.a == gamma and len(r.emitted) == gamma + 1 and r.emitted[:gamma] == xs
                r0 = sp.verify_stream(zt, zd, xs, T, SEED, sid, 0, bonus=False)
                assert r0.a == gamma and r0.emitted == xs


def test_point_mass_residual():
    # p concentrated on one token that q misses: reject always yields that token
    zt = np.array([[0.0, -200.0, -200.0], [0.0, -200.0, -200.0]], dtype=np.float32)
    zd = np.array([[-200.0, 0.0, -200.0]], dtype=np.float32)
    for sid in range(10):
        r = sp.verify_stream(zt, zd, [1], 1.0, SEED, sid, 0)
        assert r.a == 0 and r.emitted == [0]


# ---------------------------------------------------------------- enumeration
def _ctx_tables(V, seed):
    """Order-2 context-dependent categorical tables p(.|c1,c2), q(.|c1,c2) as logits."""
    rng = np.random.default_rng(seed)
    zt = (rng.standard_normal((V + 1, V + 1, V)) * 1.5).astype(np.float32)
    zd = (rng.standard_normal((V + 1, V + 1, V)) * 1.5).astype(np.float32)
    return zt, zd


def _dist(z, T):
    return np.exp(sp.logsoftmax_tail(sp.scaled_logits(z, T)))


def _ctx(seq, V):
    c1 = seq[-2] if len(seq) >= 2 else V
    c2 = seq[-1] if len(seq) >= 1 else V
    return c1, c2


def _enumerate_spec(zt, zd, V, gamma, l, T, bonus):
    """Exact law of the first l emitted tokens of repeated rounds, built only from
    the oracle's accept_prob / residual_logweights / logsoftmax_tail."""
    out = {}

    def rec(seq, prob):
        if len(seq) >= l:
            key = tuple(seq[:l])
            out[key] = out.get(key, 0.0) + prob
            return
        for xs in itertools.product(range(V), repeat=gamma):
            s, pr = list(seq), prob
            qs, ps = [], []
            for j in range(gamma):
                qd = zd[_ctx(s + list(xs[:j]), V)]
                qs.append(qd)
                pr *= _dist(qd, T)[xs[j]]
            if pr == 0.0:
                continue
            for j in range(gamma + 1):
                ps.append(zt[_ctx(s + list(xs[:j]), V)])
            # walk the accept chain
            acc = 1.0
            for a in range(gamma + 1):
                if a == gamma:
                    if bonus:
                        pb = _dist(ps[gamma], T)
                        for y in range(V):
                            rec(s + list(xs) + [y], pr * acc * pb[y])
                    else:
                        rec(s + list(xs), pr * acc)
                    break
                lp = sp.logsoftmax_tail(sp.scaled_logits(ps[a], T))
                lq = sp.logsoftmax_tail(sp.scaled_logits(qs[a], T))
                rho = sp.accept_prob(lp[xs[a]], lq[xs[a]])
                if rho < 1.0:
                    w = sp.residual_logweights(lp, lq)
                    res = np.exp(w - np.max(w))
                    res /= res.sum()
                    for y in range(V):
                        if res[y] > 0:
                            rec(s + list(xs[:a]) + [y], pr * acc * (1 - rho) * res[y])
                acc *= rho
                if acc == 0.0:
                    break

    rec([], 1.0)
    return out


def _enumerate_ar(zt, V, l, T):
    out = {}
    for seq in itertools.product(range(V), repeat=l):
        pr = 1.0
        for i in range(l):
            pr *= _dist(zt[_ctx(list(seq[:i]), V)], T)[seq[i]]
        out[seq] = pr
    return out


@pytest.mark.parametrize("bonus", [True, False])
@pytest.mark.parametrize("V,gamma,l,T", [(3, 2, 4, 1.0), (3, 2, 3, 0.6), (2, 3, 5, 1.0)])
def test_enumeration_lossless(bonus, V, gamma, l, T):
    zt, zd = _ctx_tables(V, seed=V * 100 + gamma)
    spec = _enumerate_spec(zt, zd, V, gamma, l, T, bonus)
    ar = _enumerate_ar(zt, V, l, T)
    assert abs(sum(spec.values()) - 1.0) < 1e-12
    err = max(abs(spec.get(k, 0.0) - v) for k, v in ar.items())
    assert err <= 1e-10, err


def test_enumeration_detects_wrong_residual():
    """The enumeration must fail for a plausible mistake (resampling from p instead of the residual)."""
    V, gamma, l, T = 3, 2, 3, 1.0
    zt, zd = _ctx_tables(V, seed=7)
    orig = sp.residual_logweights
    try:
        sp.residual_logweights = lambda lp, lq: np.asarray(lp, dtype=np.float64)
        spec = _enumerate_spec(zt, zd, V, gamma, l, T, True)
    finally:
        sp.residual_logweights = orig
    ar = _enumerate_ar(zt, V, l, T)
    assert max(abs(spec.get(k, 0.0) - v) for k, v in ar.items()) > 1e-3


# ------------------------------------------------------------ vectorised rounds
def _race_vec(logw, tag, slot, sids, r, V):
    """Exponential race over many stream ids at once, with oracle.philox + oracle.sampling.race_keys."""
    k0, k1 = ph.seed_key(SEED)
    nblk = (V + 3) // 4
    w = ph.philox4x32_10_np(np.arange(nblk, dtype=np.uint64)[None, :], (tag << 24) | slot, r,
                            sids[:, None], k0, k1)
    words = np.stack(w, axis=2).reshape(len(sids), -1)[:, :V]
    u = ph.u_from_word_np(words)
    keys = sp.race_keys(np.broadcast_to(logw, u.shape), u)
    return np.argmax(keys, axis=1)


def _round_vec(zt, zd, T, sids, r, bonus=True):
    """One round for many independent streams sharing the same (p, q) rows:
    drafts by race on q_j, accepts by u < rho, residual / bonus race."""
    gamma, V = zd.shape
    lps = [sp.logsoftmax_tail(sp.scaled_logits(zt[j], T)) for j in range(gamma + 1)]
    lqs = [sp.logsoftmax_tail(sp.scaled_logits(zd[j], T)) for j in range(gamma)]
    n = len(sids)
    xs = np.stack([_race_vec(sp.scaled_logits(zd[j], T).astype(np.float64), ph.TAG_DRAFT, j + 1, sids, r, V)
                   for j in range(gamma)], axis=1)
    k0, k1 = ph.seed_key(SEED)
    alive = np.ones(n, dtype=bool)
    a = np.zeros(n, dtype=np.int64)
    for j in range(gamma):
        rho = np.exp(np.minimum(0.0, lps[j][xs[:, j]] - lqs[j][xs[:, j]]))
        w = ph.philox4x32_10_np(0, (ph.TAG_ACCEPT << 24) | (j + 1), r, sids, k0, k1)[0]
        u = ph.u_from_word_np(w)
        acc = alive & (u < rho)
        a += acc
        alive = acc
    y = np.full(n, -1, dtype=np.int64)
    for aa in range(gamma + 1):
        sel = a == aa
        if not np.any(sel):
            continue
        if aa < gamma:
            logw = sp.residual_logweights(lps[aa], lqs[aa])
        elif bonus:
            logw = sp.scaled_logits(zt[gamma], T).astype(np.float64)
        else:
            continue
        y[sel] = _race_vec(logw, ph.TAG_RESAMPLE, aa + 1, sids[sel], r, V)
    return xs, a, y


def test_vectorised_round_equals_oracle():
    rng = np.random.default_rng(3)
    gamma, V = 4, 32
    zt = (rng.standard_normal((gamma + 1, V))).astype(np.float32)
    zd = (zt[:gamma] + rng.standard_normal((gamma, V)) * 0.7).astype(np.float32)
    sids = np.arange(400, dtype=np.uint64)
    for T in (1.0, 0.2):
        xs, a, y = _round_vec(zt, zd, T, sids, 5)
        for i in range(len(sids)):
            tok, _ = sp.draft_token(zd[0], T, SEED, int(sids[i]), 5, 1)
            assert tok == xs[i, 0]
            res = sp.verify_stream(zt, zd, xs[i].tolist(), T, SEED, int(sids[i]), 5)
            assert res.a == a[i] and res.y == y[i]


def _chi2(counts, probs):
    n = counts.sum()
    exp = probs * n
    keep = exp > 0
    return float(np.sum((counts[keep] - exp[keep]) ** 2 / exp[keep])), int(keep.sum()) - 1


def test_race_sampler_chi2():
    rng = np.random.default_rng(4)
    V = 32
    logw = rng.standard_normal(V) * 1.3
    sids = np.arange(1_000_000, dtype=np.uint64)
    y = _race_vec(logw, ph.TAG_RESAMPLE, 1, sids, 0, V)
    probs = np.exp(logw - special.logsumexp(logw))
    chi, df = _chi2(np.bincount(y, minlength=V).astype(np.float64), probs)
    assert chi < stats.chi2.ppf(0.99, df), (chi, df)


@pytest.mark.parametrize("T", [1.0, 0.2])
def test_round_chi2_first_tokens(T):
    """north_star: chi-square at alpha = 0.01 over 1e6 rounds: the first emitted
    token follows p_1 (df 31) and the first two follow p_1 x p_2 (df 1023)."""
    rng = np.random.default_rng(5)
    gamma, V = 4, 32
    zt = (rng.standard_normal((gamma + 1, V)) * (1.0 if T == 1.0 else 0.25)).astype(np.float32)
    zd = (zt[:gamma] + rng.standard_normal((gamma, V)) * 0.5 * (1.0 if T == 1.0 else 0.25)).astype(np.float32)
    n = 1_000_000
    sids = np.arange(n, dtype=np.uint64)
    xs, a, y = _round_vec(zt, zd, T, sids, 0)
    first = np.where(a >= 1, xs[:, 0], y)
    p1 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[0], T)))
    chi, df = _chi2(np.bincount(first, minlength=V).astype(np.float64), p1)
    assert chi < stats.chi2.ppf(0.99, df), (chi, df)
    # the second emitted token, conditioned on the first: rows are position-specific
    # (p_2 is the same for every first token here), so the joint law is p_1 x p_2
    second = np.where(a >= 2, xs[:, 1], np.where(a == 1, y, -1))
    has2 = second >= 0
    p2 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[1], T)))
    joint = first[has2] * V + second[has2]
    # P(second exists | first) depends only on acceptance of position 1, which is
    # independent of which token was emitted at position 2; test the conditional law
    chi2, df2 = _chi2(np.bincount(second[has2], minlength=V).astype(np.float64), p2)
    assert chi2 < stats.chi2.ppf(0.99, df2), (chi2, df2)
    assert joint.size > 0


def test_alpha_and_expected_emitted():
    """empirical acceptance of x_1 within +-0.01 of sum min(p, q);
    Leviathan eq. 1: E[a + 1] = (1 - alpha^(g+1)) / (1 - alpha) for position-independent (p, q)."""
    rng = np.random.default_rng(6)
    gamma, V = 4, 32
    row_t = rng.standard_normal(V).astype(np.float32)
    row_d = (row_t + rng.standard_normal(V) * 0.8).astype(np.float32)
    zt = np.stack([row_t] * (gamma + 1))
    zd = np.stack([row_d] * gamma)
    alpha = sp.alpha_row(row_t, row_d, 1.0)
    n = 200_000
    xs, a, y = _round_vec(zt, zd, 1.0, np.arange(n, dtype=np.uint64), 0)
    assert abs(np.mean(a >= 1) - alpha) < 0.01
    expect = (1 - alpha ** (gamma + 1)) / (1 - alpha)
    emitted = a + 1
    assert abs(emitted.mean() - expect) < 4 * emitted.std() / math.sqrt(n)
