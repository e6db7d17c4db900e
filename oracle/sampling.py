"""Speculative sampling, step by step in the paper's order -- TEST INFRASTRUCTURE ONLY.

Paper passages followed:
  P:98   draft x_i ~ p_d(x | x_<i, c), i = 1..k (autoregressive drafting)
  P:99   the target scores all drafted positions in parallel
  P:100  x_i is accepted with probability min(1, p_t / p_d)
  P:101  "Once a token is rejected, the verifying terminates and a resampling
         phase follows to return a new token by M_t"
  P:103  "equivalent to sampling directly from the target LLM" (losslessness)
Readings ("Readings of the paper"):
  R1  bonus token from p_{gamma+1} on full acceptance (Leviathan et al., cited P:93)
  R2  accept iff u < rho (strict), u on the odd 2^-24 grid
  R3  the resampled token comes from norm(max(0, p - q))
  R4  temperature: a = fl32(z / T) for draft and target alike
  R13 log space: rho = exp(min(0, lp - lq))
  R14 ties -> smallest token id
Everything after the exact fp32 front end a = fl32(z / T) is fp64.

Sampling of a categorical with log-weights w uses the exponential race:
  y = argmax_v (w_v - log E_v),  E_v = -log1p(-u_v)  iid Exp(1)
(the Gumbel-max trick written with exponentials), which draws v with
probability exp(w_v) / sum exp(w).
"""
import math

import numpy as np

from . import philox as _ph

NEG_INF = -math.inf


def scaled_logits(z, T):
    """R4: a_v = fl32(z_v / T), an IEEE fp32 division."""
    z32 = np.asarray(z, dtype=np.float32)
    return (z32 / np.float32(T)).astype(np.float32)


def logsoftmax_tail(a):
    """log softmax(a) with the argmax term kept out of the sum (DESIGN R13).

    i* = first argmax, m = a_{i*}, S' = sum_{v != i*} exp(a_v - m),
    lp_v = a_v - m - log1p(S').  Mathematically log(exp(a_v) / sum exp(a)).
    """
    a64 = np.asarray(a, dtype=np.float64)
    i = int(np.argmax(a64))          # numpy argmax returns the first maximum
    m = a64[i]
    e = np.exp(a64 - m)
    e[i] = 0.0
    s = float(np.sum(e))
    return a64 - m - math.log1p(s)


def accept_prob(lp_x, lq_x):
    """P:100 min(1, p_t / p_d), written in log space (R13)."""
    return math.exp(min(0.0, float(lp_x) - float(lq_x)))


def residual_logweights(lp, lq):
    """R3: log of max(0, p - q) (unnormalised): lp + log(1 - exp(lq - lp)) where q < p."""
    lp = np.asarray(lp, dtype=np.float64)
    lq = np.asarray(lq, dtype=np.float64)
    out = np.full(lp.shape, NEG_INF)
    pos = lq < lp
    out[pos] = lp[pos] + np.log(-np.expm1(lq[pos] - lp[pos]))
    return out


def race_keys(logw, u):
    """Race keys k_v = w_v - log(E_v), E_v = -log1p(-u_v); -inf where w_v = -inf."""
    logw = np.asarray(logw, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    E = -np.log1p(-u)
    keys = np.full(logw.shape, NEG_INF)
    fin = np.isfinite(logw)
    keys[fin] = logw[fin] - np.log(E[fin])
    return keys


def race(logw, u):
    """Exponential race: (argmax_v k_v with ties to the smallest v, top-2 key gap).

    Returns (-1, inf) when every weight is -inf.
    """
    keys = race_keys(logw, u)
    if not np.any(np.isfinite(keys)):
        return -1, math.inf
    arg = int(np.argmax(keys))       # first maximum = smallest id on ties (R14)
    best = keys[arg]
    rest = np.delete(keys, arg)
    gap = best - float(np.max(rest)) if rest.size and np.isfinite(np.max(rest)) else math.inf
    return arg, gap


def draft_token(zd_row, T, seed, sid, r, j):
    """P:98 x_j ~ q_j = softmax(a^d_j), sampled by race on a^d_j (tag DRAFT, slot j)."""
    ad = scaled_logits(zd_row, T)
    u = _ph.race_uniforms(seed, sid, r, _ph.TAG_DRAFT, j, ad.shape[-1])
    tok, gap = race(ad.astype(np.float64), u)
    return tok, gap


class VerifyResult:
    __slots__ = ("a", "emitted", "y", "flags", "accept_margins", "race_gap", "fallback")

    def __init__(self):
        self.a = 0
        self.emitted = []
        self.y = None
        self.flags = 0
        self.accept_margins = []
        self.race_gap = math.inf
        self.fallback = False


def verify_stream(zt, zd, xs, T, seed, sid, r, bonus=True, flag_eps=1e-6):
    """One stream's verification (Alg. 1).

    zt: target logits [gamma+1][V] for inputs [T_s[-1], x_1..x_gamma]
    zd: draft logits  [gamma][V]   (row j-1 conditions on x_<j)
    xs: drafted tokens x_1..x_gamma
    Returns a VerifyResult: a = #leading accepts, emitted = x_1..x_a (+ y).
    """
    gamma = len(xs)
    V = np.asarray(zt).shape[-1]
    res = VerifyResult()
    lps = [logsoftmax_tail(scaled_logits(zt[j], T)) for j in range(gamma + 1)]
    lqs = [logsoftmax_tail(scaled_logits(zd[j], T)) for j in range(gamma)]
    a = 0
    for j in range(1, gamma + 1):                     # P:267 for j = 1..k
        x = int(xs[j - 1])
        rho = accept_prob(lps[j - 1][x], lqs[j - 1][x])
        u = _ph.philox_u(seed, sid, r, _ph.TAG_ACCEPT, j, 0, 0)
        res.accept_margins.append(abs(u - rho))
        if abs(u - rho) < flag_eps:
            res.flags += 1
        if u < rho:                                   # P:268-271 accepted
            a += 1
        else:                                         # P:272-274 reject -> resample, break
            break
    res.a = a
    if a < gamma:
        w = residual_logweights(lps[a], lqs[a])
        u = _ph.race_uniforms(seed, sid, r, _ph.TAG_RESAMPLE, a + 1, V)
        y, gap = race(w, u)
        if y < 0:                                     # empty residual (rounding only): bonus rule
            res.fallback = True
            res.flags += 1
            y, gap = race(scaled_logits(zt[a], T).astype(np.float64), u)
        res.y, res.race_gap = y, gap
    elif bonus:                                       # R1: bonus token from p_{gamma+1}
        u = _ph.race_uniforms(seed, sid, r, _ph.TAG_RESAMPLE, gamma + 1, V)
        y, gap = race(scaled_logits(zt[gamma], T).astype(np.float64), u)
        res.y, res.race_gap = y, gap
    if res.race_gap < flag_eps:
        res.flags += 1
    res.emitted = [int(x) for x in xs[:a]] + ([int(res.y)] if res.y is not None else [])
    return res


def alpha_row(zt_row, zd_row, T):
    """S:135-143 expected acceptance alpha = sum_v min(p_v, q_v)."""
    p = np.exp(logsoftmax_tail(scaled_logits(zt_row, T)))
    q = np.exp(logsoftmax_tail(scaled_logits(zd_row, T)))
    return float(np.sum(np.minimum(p, q)))
