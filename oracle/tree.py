"""Multi-candidate (tree) drafting and verification -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §3.2 (several candidates per draft position, the target verifies the
whole candidate tree in one pass with a tree attention mask, "share the caches of generated
tokens"), Appendix B (k_config = (2,2,1) -> "the first two positions each sampling 2
candidates", Figure 7's mask) and SPEC.md spec-sampling: CandidateTree, draft,
verify_tree by recursive rejection over candidates sampled without replacement.  The paper names
MCSD but never specifies its rule; this follows SPEC's reading, which is the
multi-candidate rule without replacement:

  at node n with target distribution p and draft distribution q (the one n's children were
  drawn from), children c_1, c_2, ... in their sampled order:
    accept c_i with probability min(1, p(c_i) / q(c_i));
    on rejection:  p <- norm(max(0, p - q)),  q <- q with c_i removed, renormalised;
  the first accepted child becomes the path; if every child is rejected the correction is drawn
  from the final p; if the walk reaches depth K the bonus token is drawn from the leaf's p (R1).

Readings (R36): node numbering is breadth-first with the root (the context T) = 0, so
the all-ones k_config reproduces the chain numbering exactly (node j = depth j); the Philox
slots are the chain's: DRAFT race of node n's children = slot n + 1, ACCEPT of child c = slot c,
RESAMPLE / bonus race at node n = slot n + 1.  Children are drawn without replacement by the
top-m of the same exponential race the chain uses (its first key is the chain's draft token).
The draft distribution softmax(a / T) is positive everywhere for finite logits, so the fan-out
never shrinks (SPEC's degenerate-support rule never triggers).  Everything is fp64 in log space
after the exact fp32 front end, with the chain's tail-excluded log-softmax (R13); with k_config
all ones every decision is the chain's (`verify_stream`) bit for bit.
"""
import math
from dataclasses import dataclass, field

import numpy as np

from . import llama as _ll
from . import philox as _ph
from . import sampling as _sp

NEG_INF = -math.inf


def tree_shape(counts):
    """Breadth-first tree of k_config `counts`: parent[i], depth[i] for nodes 1..n (root 0)."""
    parent, depth = [-1], [0]
    level = [0]
    for d, m in enumerate(counts, start=1):
        nxt = []
        for p in level:
            for _ in range(m):
                parent.append(p)
                depth.append(d)
                nxt.append(len(parent) - 1)
        level = nxt
    return parent, depth


def children(parent):
    ch = [[] for _ in parent]
    for i, p in enumerate(parent):
        if p >= 0:
            ch[p].append(i)
    return ch


def ancestor_mask(parent):
    """mask[r][c] = c is r or an ancestor of r (Figure 7), over nodes 1..n."""
    n = len(parent) - 1
    mask = np.zeros((n, n), dtype=bool)
    for r in range(1, n + 1):
        c = r
        while c > 0:
            mask[r - 1, c - 1] = True
            c = parent[c]
    return mask


def race_top(logw, u, m):
    """The m largest race keys w_v - log(-log1p(-u_v)), decreasing (ties -> smaller id first):
    a draw of m distinct ids without replacement from softmax(logw) (the Gumbel-top-m property of
    the exponential race).  Returns (ids, gap between the m-th and (m+1)-th keys)."""
    keys = _sp.race_keys(logw, u)
    order = sorted(range(len(keys)), key=lambda v: (-keys[v], v))
    top = [v for v in order[:m] if np.isfinite(keys[v])]
    gaps = [keys[order[i]] - keys[order[i + 1]] for i in range(min(m, len(order) - 1))]
    return top, (min(gaps) if gaps else math.inf)


@dataclass
class Tree:
    counts: tuple
    parent: list
    depth: list
    tokens: list = field(default_factory=list)     # tokens[i] for nodes 1..n (tokens[0] unused)
    gaps: list = field(default_factory=list)        # race gaps of each expansion (near-tie flags)


def draft_tree(zd_of, counts, T, seed, sid, r):
    """S:108-116 draft: breadth-first, node n's children are the top-counts[d] of the race over the
    draft row conditioned on n's path (zd_of(n, path_tokens) -> logits), slot n + 1."""
    parent, depth = tree_shape(counts)
    ch = children(parent)
    tokens = [None] * len(parent)
    gaps = []
    for n in range(len(parent)):
        if not ch[n]:
            continue
        path = path_tokens(parent, tokens, n)
        a = _sp.scaled_logits(zd_of(n, path), T).astype(np.float64)
        u = _ph.race_uniforms(seed, sid, r, _ph.TAG_DRAFT, n + 1, a.shape[-1])
        top, gap = race_top(a, u, len(ch[n]))
        gaps.append(gap)
        for c, v in zip(ch[n], top):
            tokens[c] = int(v)
    return Tree(tuple(counts), parent, depth, tokens, gaps)


def path_tokens(parent, tokens, n):
    out = []
    while n > 0:
        out.append(tokens[n])
        n = parent[n]
    return out[::-1]


def rejection_chain(lp, lq, cands):
    """Recursive rejection at one node (module docstring): for candidates c_1, c_2, ... the
    acceptance probability rho_i = min(1, p_i(c_i) / q_i(c_i)) under the distributions left after
    rejecting c_1..c_{i-1}; and the unnormalised log-weights of the correction distribution after
    rejecting all of them.  p_{i+1} = norm(max(0, p_i - q_i)), q_{i+1} = q_i without c_i.
    Returns (rhos, final_logw, fallback).  The first candidate's rho and the single-candidate
    residual are exactly the chain's (sampling.accept_prob / residual_logweights)."""
    lp = np.asarray(lp, dtype=np.float64)
    lq = np.asarray(lq, dtype=np.float64)
    rhos, w, fallback = [], None, False
    for i, x in enumerate(cands):
        rhos.append(_sp.accept_prob(lp[x], lq[x]))
        w = _sp.residual_logweights(lp, lq)
        if not np.any(np.isfinite(w)):             # empty residual (rounding only): keep p
            fallback = True
            w = lp.copy()
        lp = w - np.logaddexp.reduce(w[np.isfinite(w)])
        rest = -math.expm1(lq[x])                  # 1 - q(x): the mass left after removing x
        lq = lq - math.log(rest) if rest > 0.0 else np.full_like(lq, NEG_INF)
        lq[x] = NEG_INF
    return rhos, w, fallback


class TreeResult:
    __slots__ = ("path", "emitted", "y", "flags", "fallback", "accepted_nodes")

    def __init__(self):
        self.path, self.emitted, self.y, self.flags, self.fallback, self.accepted_nodes = [], [], None, 0, False, []


def verify_tree(zt_of, zd_of, tree, T, seed, sid, r, bonus=True, flag_eps=1e-6):
    """S:126-133 verify_tree by recursive rejection (module docstring).  zt_of(n) / zd_of(n): the
    target / draft logits rows at node n (the distributions of n's children)."""
    ch = children(tree.parent)
    res = TreeResult()
    node = 0
    while ch[node]:
        a_t = _sp.scaled_logits(zt_of(node), T)
        lp = _sp.logsoftmax_tail(a_t)
        lq = _sp.logsoftmax_tail(_sp.scaled_logits(zd_of(node), T))
        cands = [tree.tokens[c] for c in ch[node]]
        rhos, _, _ = rejection_chain(lp, lq, cands)
        accepted, n_rej = None, 0
        for c, rho in zip(ch[node], rhos):
            u = _ph.philox_u(seed, sid, r, _ph.TAG_ACCEPT, c, 0, 0)
            if abs(u - rho) < flag_eps:
                res.flags += 1
            if u < rho:
                accepted = c
                break
            n_rej += 1
        if accepted is None:                       # every child rejected: correction from the residual
            _, w, fb = rejection_chain(lp, lq, cands)
            if fb:
                res.fallback = True
                res.flags += 1
                if len(cands) == 1:                # the chain's fallback: the bonus rule on this row
                    w = a_t.astype(np.float64)
            u = _ph.race_uniforms(seed, sid, r, _ph.TAG_RESAMPLE, node + 1, lp.shape[-1])
            y, gap = _sp.race(w, u)
            if gap < flag_eps:
                res.flags += 1
            res.y = y
            break
        node = accepted
        res.accepted_nodes.append(node)
        res.path.append(tree.tokens[node])
    else:
        if bonus:                                  # the leaf was accepted: bonus token (R1)
            a = _sp.scaled_logits(zt_of(node), T).astype(np.float64)
            u = _ph.race_uniforms(seed, sid, r, _ph.TAG_RESAMPLE, node + 1, a.shape[-1])
            y, gap = _sp.race(a, u)
            if gap < flag_eps:
                res.flags += 1
            res.y = y
    res.emitted = list(res.path) + ([int(res.y)] if res.y is not None else [])
    return res


def tree_layer_forward(shape, L, x, parent, ctx, k_cache, v_cache, mode="bf16"):
    """One decoder layer over a tree of rows (Figure 7): row 0 is the root at
    position ctx, row i (parent[i] < i) sits at position ctx + depth(i) and sees the cached keys and
    the rows on its root-to-row path.  By definition each row's output is the last row of the causal
    layer (`llama.layer_forward`) over its path; returns (x_out, k_new, v_new) like layer_forward."""
    x = np.asarray(x, dtype=np.float64)
    M = len(parent)
    outs, ks, vs = [None] * M, [None] * M, [None] * M
    for i in range(M):
        path = []
        n = i
        while n >= 0:
            path.append(n)
            n = parent[n]
        path = path[::-1]
        xo, kn, vn = _ll.layer_forward(shape, L, x[path], np.arange(ctx, ctx + len(path)), k_cache, v_cache, mode=mode)
        outs[i], ks[i], vs[i] = xo[-1], kn[-1], vn[-1]
    return np.stack(outs), np.stack(ks), np.stack(vs)
