"""Oracle pins for multi-candidate (tree) drafting and verification (oracle/tree.py; §3.2
P:107-113, App. B) -- CPU only.

Pins: the k_config tree shape and Figure 7's ancestor mask against a recursive walk;
the all-ones k_config reproduces the chain (`sampling.draft_token` / `verify_stream`) bit for bit
(S:131); exhaustive enumeration of every candidate tree and every verification outcome gives exactly
the target's autoregressive law (losslessness, V <= 4, k <= 3, counts <= 3, <= 1e-10), and
fails for a plausible mistake (candidates drawn WITH replacement but verified as if without);
chi-square of the race's top-2 draw against the exact without-replacement law; more candidates
accept more (App. B claim).
"""
import itertools
import math

import numpy as np
import pytest
from scipy import stats

from oracle import philox as ph
from oracle import sampling as sp
from oracle import tree as tr

SEED = 0x5EED2406


def test_tree_shape_and_mask():
    parent, depth = tr.tree_shape((2, 2, 1))
    assert len(parent) - 1 == 2 + 4 + 4                          # S:114 example
    assert depth[1:] == [1, 1, 2, 2, 2, 2, 3, 3, 3, 3]
    ch = tr.children(parent)
    assert ch[0] == [1, 2] and ch[1] == [3, 4] and ch[2] == [5, 6] and ch[3] == [7]
    mask = tr.ancestor_mask(parent)

    def anc(r):                                                    # recursive walk
        return set() if r == 0 else {r} | anc(parent[r])
    for r in range(1, len(parent)):
        for c in range(1, len(parent)):
            assert mask[r - 1, c - 1] == (c in anc(r))
    p1, _ = tr.tree_shape((1, 1, 1))
    assert (tr.ancestor_mask(p1) == np.tril(np.ones((3, 3), dtype=bool))).all()   # S:113 chain example


def test_all_ones_is_the_chain():
    rng = np.random.default_rng(2)
    V, g = 64, 4
    for T in (1.0, 0.2):
        for sid in range(40):
            zd = (rng.standard_normal((g, V)) * 2).astype(np.float32)
            zt = (zd[[0, 1, 2, 3, 3]] + rng.standard_normal((g + 1, V)) * 0.5).astype(np.float32)
            tree = tr.draft_tree(lambda n, path: zd[n], (1,) * g, T, SEED, sid, 3)
            xs = [sp.draft_token(zd[j], T, SEED, sid, 3, j + 1)[0] for j in range(g)]
            assert tree.tokens[1:] == xs
            rt = tr.verify_tree(lambda n: zt[n], lambda n: zd[n], tree, T, SEED, sid, 3)
            rc = sp.verify_stream(zt, zd, xs, T, SEED, sid, 3)
            assert rt.emitted == rc.emitted and len(rt.path) == rc.a


# ---------------------------------------------------------------- exhaustive enumeration
def _tables(V, seed):
    rng = np.random.default_rng(seed)
    zt = (rng.standard_normal((V + 1, V + 1, V)) * 1.5).astype(np.float32)
    zd = (rng.standard_normal((V + 1, V + 1, V)) * 1.5).astype(np.float32)
    return zt, zd


def _ctx(seq, V):
    return (seq[-2] if len(seq) >= 2 else V, seq[-1] if len(seq) >= 1 else V)


def _dist(z, T):
    return np.exp(sp.logsoftmax_tail(sp.scaled_logits(z, T)))


def _ordered_draws(q, m, replace):
    """Every ordered m-tuple and its probability: without replacement q(c1) q(c2)/(1 - q(c1)) ..."""
    V = len(q)
    for tup in itertools.product(range(V), repeat=m):
        if not replace and len(set(tup)) < m:
            continue
        pr, rest = 1.0, 1.0
        for c in tup:
            pr *= q[c] / (rest if not replace else 1.0)
            if not replace:
                rest -= q[c]
        if pr > 0:
            yield tup, pr


def _round_law(zt, zd, V, counts, T, bonus, seq, replace=False):
    """Law of one round's emitted tokens from context seq: {tuple: prob}, built from the oracle's
    rejection_chain (acceptance probabilities and residuals) and exact sampling probabilities."""
    K = len(counts)
    out = {}

    def walk(path, depth, pr):
        ctx = seq + path
        lp = sp.logsoftmax_tail(sp.scaled_logits(zt[_ctx(ctx, V)], T))
        lq = sp.logsoftmax_tail(sp.scaled_logits(zd[_ctx(ctx, V)], T))
        for cands, ps in _ordered_draws(np.exp(lq), counts[depth], replace):
            rhos, w, _ = tr.rejection_chain(lp, lq, list(cands))
            rest = pr * ps
            for c, rho in zip(cands, rhos):
                if rho > 0:
                    if depth + 1 == K:
                        if bonus:
                            pb = _dist(zt[_ctx(ctx + [c], V)], T)
                            for y in range(V):
                                key = tuple(path + [c, y])
                                out[key] = out.get(key, 0.0) + rest * rho * pb[y]
                        else:
                            key = tuple(path + [c])
                            out[key] = out.get(key, 0.0) + rest * rho
                    else:
                        walk(path + [c], depth + 1, rest * rho)
                rest *= 1.0 - rho
                if rest == 0.0:
                    break
            if rest > 0.0:
                res = np.exp(w - np.max(w))
                res /= res.sum()
                for y in range(V):
                    if res[y] > 0:
                        key = tuple(path + [y])
                        out[key] = out.get(key, 0.0) + rest * res[y]

    walk([], 0, 1.0)
    return out


def _sequence_law(zt, zd, V, counts, T, bonus, l, replace=False):
    law = {}

    def rec(seq, pr):
        if len(seq) >= l:
            key = tuple(seq[:l])
            law[key] = law.get(key, 0.0) + pr
            return
        for emitted, p in _round_law(zt, zd, V, counts, T, bonus, seq, replace).items():
            rec(seq + list(emitted), pr * p)

    rec([], 1.0)
    return law


def _ar_law(zt, V, l, T):
    law = {}
    for seq in itertools.product(range(V), repeat=l):
        pr = 1.0
        for i in range(l):
            pr *= _dist(zt[_ctx(list(seq[:i]), V)], T)[seq[i]]
        law[seq] = pr
    return law


@pytest.mark.parametrize("V,counts,l,T,bonus", [(3, (2, 1), 3, 1.0, True), (3, (2, 2), 3, 1.0, True),
                                               (3, (1, 2), 3, 0.6, False), (4, (3,), 2, 1.0, True),
                                               (3, (3, 1), 3, 1.0, False), (4, (2, 1, 1), 3, 0.8, True)])
def test_tree_enumeration_lossless(V, counts, l, T, bonus):
    """the emitted sequence's law equals autoregressive sampling from the target."""
    zt, zd = _tables(V, seed=V * 10 + sum(counts))
    spec = _sequence_law(zt, zd, V, counts, T, bonus, l)
    ar = _ar_law(zt, V, l, T)
    assert abs(sum(spec.values()) - 1.0) < 1e-12
    err = max(abs(spec.get(k, 0.0) - v) for k, v in ar.items())
    assert err <= 1e-10, err


def test_tree_enumeration_detects_with_replacement():
    """Power: candidates drawn WITH replacement but verified with the without-replacement update
    is not lossless -- the enumeration must see it."""
    V, counts, l, T = 3, (2, 1), 3, 1.0
    zt, zd = _tables(V, seed=5)
    spec = _sequence_law(zt, zd, V, counts, T, True, l, replace=True)
    ar = _ar_law(zt, V, l, T)
    tot = sum(spec.values())
    assert max(abs(spec.get(k, 0.0) / tot - v) for k, v in ar.items()) > 1e-3


# ---------------------------------------------------------------- sampling checks
def test_race_top2_is_without_replacement():
    """The race's top-2 over 2e5 stream ids follows q(c1) q(c2) / (1 - q(c1)) (chi-square, alpha 0.01)."""
    rng = np.random.default_rng(4)
    V, n = 8, 200_000
    logw = rng.standard_normal(V)
    q = np.exp(logw - np.logaddexp.reduce(logw))
    k0, k1 = ph.seed_key(SEED)
    sids = np.arange(n, dtype=np.uint64)
    w = ph.philox4x32_10_np(np.arange(2, dtype=np.uint64)[None, :], (ph.TAG_DRAFT << 24) | 1, 0, sids[:, None], k0, k1)
    u = ph.u_from_word_np(np.stack(w, axis=2).reshape(n, -1)[:, :V])
    keys = sp.race_keys(np.broadcast_to(logw, u.shape), u)
    order = np.argsort(-keys, axis=1, kind="stable")
    pairs = order[:, 0] * V + order[:, 1]
    cnt = np.bincount(pairs, minlength=V * V).astype(float)
    exp = np.array([q[a] * q[b] / (1 - q[a]) if a != b else 0.0 for a in range(V) for b in range(V)]) * n
    keep = exp > 0
    chi = np.sum((cnt[keep] - exp[keep]) ** 2 / exp[keep])
    assert chi < stats.chi2.ppf(0.99, keep.sum() - 1), chi
    assert cnt[~keep].sum() == 0
    # the oracle's race_top agrees with the vectorised draw on the first ids
    for i in range(50):
        top, _ = tr.race_top(logw, u[i], 2)
        assert top == [int(order[i, 0]), int(order[i, 1])]


def test_more_candidates_accept_more():
    """App. B / S:143: mean accepted length with counts (2,1,1) >= (1,1,1) (3 sigma slack)."""
    rng = np.random.default_rng(9)
    V, T = 32, 1.0
    zt_rows = (rng.standard_normal((64, V))).astype(np.float32)
    zd_rows = (zt_rows + rng.standard_normal((64, V)) * 1.0).astype(np.float32)

    def zd_of(n, path):
        return zd_rows[(len(path) * 7 + sum(path)) % 64]

    def mean_acc(counts, n=3000):
        acc = []
        for sid in range(n):
            tree = tr.draft_tree(zd_of, counts, T, SEED, sid, 0)
            zt_of = lambda node: zt_rows[(len(tr.path_tokens(tree.parent, tree.tokens, node)) * 7 +
                                         sum(tr.path_tokens(tree.parent, tree.tokens, node))) % 64]
            zd_node = lambda node: zd_of(node, tr.path_tokens(tree.parent, tree.tokens, node))
            acc.append(len(tr.verify_tree(zt_of, zd_node, tree, T, SEED, sid, 0).path))
        return np.mean(acc), np.std(acc) / math.sqrt(n)

    m1, s1 = mean_acc((1, 1, 1))
    m2, s2 = mean_acc((2, 1, 1))
    assert m2 >= m1 - 3 * math.hypot(s1, s2), (m1, m2)
    assert m2 > m1


def test_tree_layer_chain_is_causal_layer():
    """A chain-shaped tree (parent[i] = i - 1) is the causal layer over the same rows, and a row's
    output does not depend on rows outside its path (siblings swapped -> same outputs)."""
    import seedgen
    from oracle import llama as ll
    shape = seedgen.SHAPES["toy_target"]
    sh = ll.LlamaShape(**shape)
    L = seedgen.layer_weights(shape, 77, 0)
    M, ctx = 5, 7
    x = seedgen.hidden_states(M, sh.d_model, seed=3)
    kc = np.random.default_rng(1).standard_normal((ctx, sh.kv_heads, sh.head_dim))
    vc = np.random.default_rng(2).standard_normal((ctx, sh.kv_heads, sh.head_dim))
    got = tr.tree_layer_forward(sh, L, x, [-1, 0, 1, 2, 3], ctx, kc, vc, mode="fp64")
    ref = ll.layer_forward(sh, L, x, np.arange(ctx, ctx + M), kc, vc, mode="fp64")
    for a, b in zip(got, ref):
        assert np.allclose(a, b, rtol=0, atol=1e-12)
    # star tree: rows 1..4 children of the root; reordering the children permutes their outputs only
    star = tr.tree_layer_forward(sh, L, x, [-1, 0, 0, 0, 0], ctx, kc, vc, mode="fp64")[0]
    perm = [0, 3, 1, 4, 2]
    star_p = tr.tree_layer_forward(sh, L, x[perm], [-1, 0, 0, 0, 0], ctx, kc, vc, mode="fp64")[0]
    assert np.allclose(star_p, star[perm], rtol=0, atol=1e-12)
    # and a child of the root equals the two-row causal layer [root, child]
    two = ll.layer_forward(sh, L, x[[0, 2]], np.arange(ctx, ctx + 2), kc, vc, mode="fp64")[0]
    assert np.allclose(star[2], two[1], rtol=0, atol=1e-12)
