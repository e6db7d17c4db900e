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


def _rows(rng, n_pos, V, T):
    """Position-specific target / draft logits rows (context-free, so AR sampling is a product law)."""
    sc = 1.0 if T == 1.0 else 0.25
    zt = (rng.standard_normal((n_pos, V)) * sc).astype(np.float32)
    zd = (zt + rng.standard_normal((n_pos, V)) * 0.5 * sc).astype(np.float32)
    return zt, zd


def _emitted(xs, a, y, gamma):
    """Emitted token lists per stream from a vectorised round (x_1..x_a, then y when y >= 0)."""
    return [list(xs[i, :a[i]]) + ([int(y[i])] if y[i] >= 0 else []) for i in range(len(a))]


@pytest.mark.parametrize("T", [1.0, 0.2])
def test_round_chi2_first_tokens(T):
    """north_star: chi-square at alpha = 0.01 over 1e6 streams: the first emitted token follows
    p_1 (df 31) and the first two follow p_1 x p_2 (df 1023).  Rows are position-specific and
    context-free, so target-only sampling is the product law; a stream whose first round emitted one
    token runs a second round (stream-local round 1, positions 2 ..) for its second token."""
    rng = np.random.default_rng(5)
    gamma, V = 4, 32
    zt, zd = _rows(rng, 2 * gamma + 2, V, T)
    n = 1_000_000
    sids = np.arange(n, dtype=np.uint64)
    xs, a, y = _round_vec(zt[:gamma + 1], zd[:gamma], T, sids, 0)
    first = np.where(a >= 1, xs[:, 0], y)
    second = np.where(a >= 2, xs[:, 1], np.where(a == 1, y, -1))
    one = second < 0                       # the first round emitted one token: round 2 from position 2
    xs2, a2, y2 = _round_vec(zt[1:gamma + 2], zd[1:gamma + 1], T, sids[one], 1)
    second[one] = np.where(a2 >= 1, xs2[:, 0], y2)
    p1 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[0], T)))
    p2 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[1], T)))
    chi, df = _chi2(np.bincount(first, minlength=V).astype(np.float64), p1)
    assert chi < stats.chi2.ppf(0.99, df), (chi, df)
    # joint law of the first two tokens: p_1 x p_2 (df 1023; cells with expectation < 5 pooled)
    pj = np.outer(p1, p2).reshape(-1)
    cnt = np.bincount(first * V + second, minlength=V * V).astype(np.float64)
    keep = n * pj >= 5
    cj = np.append(cnt[keep], cnt[~keep].sum())
    pk = np.append(pj[keep], pj[~keep].sum())
    chi2j, dfj = _chi2(cj, pk)
    assert dfj >= 500, dfj
    assert chi2j < stats.chi2.ppf(0.99, dfj), (chi2j, dfj)


def test_round_chi2_detects_wrong_bonus():
    """The joint test must catch a plausible mistake: the bonus token drawn from p_gamma (the row
    of the last draft position) instead of p_{gamma+1}."""
    rng = np.random.default_rng(8)
    gamma, V, T = 1, 32, 1.0
    zt, zd = _rows(rng, 2 * gamma + 2, V, T)
    zd[:] = zt                             # q == p: every draft accepted, the bonus is always token 2
    n = 200_000
    bad = zt.copy()
    bad[gamma] = zt[gamma - 1]
    xs, a, y = _round_vec(bad[:gamma + 1], zd[:gamma], T, np.arange(n, dtype=np.uint64), 0)
    p2 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[1], T)))
    chi, df = _chi2(np.bincount(y, minlength=V).astype(np.float64), p2)
    assert chi > stats.chi2.ppf(0.99, df)


@pytest.mark.parametrize("T", [1.0, 0.2])
def test_bonus_token_chi2(T):
    """R1 (Leviathan et al., cited P:93): on full acceptance the bonus token follows p_{gamma+1}.
    Over 1e6 rounds on the toy V = 32, the bonus tokens of all-accepted rounds pass chi-square at
    alpha = 0.01 against p_{gamma+1} (df 31)."""
    rng = np.random.default_rng(9)
    gamma, V = 4, 32
    zt, zd = _rows(rng, gamma + 1, V, T)
    zd = (zt[:gamma] + (zd[:gamma] - zt[:gamma]) * 0.3).astype(np.float32)   # q close to p: frequent a = gamma
    n = 1_000_000
    xs, a, y = _round_vec(zt, zd, T, np.arange(n, dtype=np.uint64), 0)
    full = a == gamma
    assert full.sum() > 50_000
    pb = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[gamma], T)))
    chi, df = _chi2(np.bincount(y[full], minlength=V).astype(np.float64), pb)
    assert chi < stats.chi2.ppf(0.99, df), (chi, df)
    # the same rounds against the WRONG row (p_gamma) must fail: the test has power
    pw = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt[gamma - 1], T)))
    chi_w, _ = _chi2(np.bincount(y[full], minlength=V).astype(np.float64), pw)
    assert chi_w > stats.chi2.ppf(0.99, df)


def test_empty_residual_fallback():
    """R3 edge case (only through rounding): the drafted token x has p(x) < q(x) but every other
    token's p and q agree to fp64 precision, so max(0, p - q) is empty after rounding.  The oracle
    then draws from the bonus rule on the same row with the same uniforms and flags the decision."""
    V, gamma, T = 64, 1, 1.0
    rng = np.random.default_rng(12)
    zd = (rng.standard_normal((gamma, V))).astype(np.float32)
    x = int(np.argmin(zd[0]))
    zd[0, x] = np.float32(zd[0].max() - 60.0)     # q(x) ~ e^-60: its change is invisible in S'
    zt = np.zeros((gamma + 1, V), dtype=np.float32)
    zt[:gamma] = zd
    zt[0, x] = zd[0, x] - np.float32(5.0)         # p(x) = e^-5 q(x): rho ~ 0.0067
    zt[gamma] = rng.standard_normal(V).astype(np.float32)
    lp = sp.logsoftmax_tail(sp.scaled_logits(zt[0], T))
    lq = sp.logsoftmax_tail(sp.scaled_logits(zd[0], T))
    assert np.all(sp.residual_logweights(lp, lq) == -np.inf)
    hits = 0
    for sid in range(200):
        r = sp.verify_stream(zt, zd, [x], T, SEED, sid, 0)
        if r.a == 0:
            hits += 1
            assert r.fallback and r.flags >= 1
            u = ph.race_uniforms(SEED, sid, 0, ph.TAG_RESAMPLE, 1, V)
            assert r.y == sp.race(sp.scaled_logits(zt[0], T).astype(np.float64), u)[0]
    assert hits > 150


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
