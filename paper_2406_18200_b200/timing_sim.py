"""Discrete-event timing model of the four execution strategies of Fig. 1.

PAPER.md Fig. 1: (a) serial AR, (b) serial SD, (c) scheduled SD -- "several parallel
draft models and one target model" -- and (d) parallel (one target instance per sequence).
The paper gives no numeric timings ("a unit length of execution time"), so every time here is a
parameter in integer ticks; nothing is cited as a paper value.  Host-only; no token computation.

Service model (DESIGN R29): a round of stream s drafts k tokens (k * t_draft), then the target
verifies it (t_verify, plus t_resample when a draft token is rejected, Fig. 2 caption P:193);
each draft token is accepted with probability alpha, the round stops at the first rejection and
emits accepted + 1 tokens (the resampled or bonus token).  A sequence is done after l tokens.
Accepted counts are drawn per (stream, round) from one seeded generator before simulating, so
every strategy sees the same draws (common random numbers).

  serial       n * l target AR steps back to back (t_target_ar each)
  serial-sd    the n SD sequences back to back
  scheduled-sd Alg. 1: drafters run in parallel; the ONE target serves finished drafts FCFS
               (ties -> lowest stream id, R10), one verification at a time
  batched-sd   this build's lock-step form (R9): all undone streams draft together, then ONE
               batched verification whose time is t_verify_batch(m) for m streams
  pipelined-sd §8(f) rank 2 / Fig. 1(c) overlap: the streams split into two lock-step groups
               (even / odd ids); group A's batched verification runs while group B drafts and
               vice versa, each phase lasting max(verify, draft)
  parallel     n independent target AR sequences fully overlapped (n target instances)
"""
import heapq
from dataclasses import dataclass

import numpy as np


@dataclass
class TimingParams:
    t_draft: int = 1          # ticks per draft token
    t_verify: int = 1         # ticks per (single-stream) verification
    t_resample: int = 1       # extra ticks when a draft token is rejected
    t_target_ar: int = 3      # ticks per target AR token
    n: int = 3
    k: int = 4
    l: int = 16
    alpha: float = 0.7
    seed: int = 0

    def validate(self):
        if min(self.t_draft, self.t_verify, self.t_target_ar) <= 0 or self.t_resample < 0:
            raise ValueError("times must be > 0 (t_resample >= 0)")
        if not 0.0 <= self.alpha <= 1.0 or self.n < 1 or self.k < 1 or self.l < 1:
            raise ValueError("alpha in [0, 1], n, k, l >= 1")


@dataclass
class StrategyResult:
    strategy: str
    makespan: int
    target_busy: int
    tokens: int
    peak_target_instances: int

    @property
    def busy_fraction(self):
        return self.target_busy / self.makespan

    @property
    def tokens_per_tick(self):
        return self.tokens / self.makespan


def accept_draws(p):
    """[n][max_rounds] accepted draft tokens per round: truncated geometric (stop at first reject)."""
    rng = np.random.default_rng(p.seed)
    u = rng.random((p.n, p.l, p.k))
    acc = (u < p.alpha).astype(np.int64)
    return np.cumprod(acc, axis=2).sum(axis=2)          # leading accepts per (stream, round)


def _rounds(p, draws, s):
    """Per-round (accepted, rejected?) of stream s until l tokens."""
    out, L, r = [], 0, 0
    while L < p.l:
        a = int(draws[s, r])
        out.append((a, a < p.k))
        L += a + 1
        r += 1
    return out


def simulate(strategy, p, t_verify_batch=None):
    p.validate()
    draws = accept_draws(p)
    toks = p.n * p.l
    if strategy == "serial":
        T = p.n * p.l * p.t_target_ar
        return StrategyResult(strategy, T, T, toks, 1)
    if strategy == "parallel":
        T = p.l * p.t_target_ar
        return StrategyResult(strategy, T, T, toks, p.n)
    rounds = [_rounds(p, draws, s) for s in range(p.n)]
    vt = lambda rej: p.t_verify + (p.t_resample if rej else 0)     # noqa: E731
    if strategy == "serial-sd":
        T = busy = 0
        for s in range(p.n):
            for a, rej in rounds[s]:
                T += p.k * p.t_draft + vt(rej)
                busy += vt(rej)
        return StrategyResult(strategy, T, busy, toks, 1)
    if strategy == "scheduled-sd":
        # events: (time a draft becomes ready, stream id); the target serves FCFS, one at a time
        ready = [(p.k * p.t_draft, s) for s in range(p.n)]
        heapq.heapify(ready)
        nxt = [0] * p.n
        t_free = busy = end = 0
        while ready:
            t_ready, s = heapq.heappop(ready)
            a, rej = rounds[s][nxt[s]]
            start = max(t_free, t_ready)
            t_free = start + vt(rej)
            busy += vt(rej)
            nxt[s] += 1
            end = max(end, t_free)
            if nxt[s] < len(rounds[s]):
                heapq.heappush(ready, (t_free + p.k * p.t_draft, s))
        return StrategyResult(strategy, end, busy, toks, 1)
    if strategy == "batched-sd":
        tvb = t_verify_batch or (lambda m: p.t_verify)
        nxt = [0] * p.n
        T = busy = 0
        while True:
            live = [s for s in range(p.n) if nxt[s] < len(rounds[s])]
            if not live:
                break
            rej = any(rounds[s][nxt[s]][1] for s in live)
            v = tvb(len(live)) + (p.t_resample if rej else 0)
            T += p.k * p.t_draft + v
            busy += v
            for s in live:
                nxt[s] += 1
        return StrategyResult(strategy, T, busy, toks, 1)
    if strategy == "pipelined-sd":
        tvb = t_verify_batch or (lambda m: p.t_verify)
        nxt = [0] * p.n
        groups = [list(range(0, p.n, 2)), list(range(1, p.n, 2))]
        live = lambda g: [s for s in groups[g] if nxt[s] < len(rounds[s])]     # noqa: E731
        T = p.k * p.t_draft if live(0) else 0            # group A drafts alone first
        busy, g = 0, 0
        while live(0) or live(1):
            lv = live(g)
            v = 0
            if lv:
                rej = any(rounds[s][nxt[s]][1] for s in lv)
                v = tvb(len(lv)) + (p.t_resample if rej else 0)
                for s in lv:
                    nxt[s] += 1
            d = p.k * p.t_draft if live(1 - g) else 0    # the other group drafts meanwhile
            T += max(v, d)
            busy += v
            g = 1 - g
        return StrategyResult(strategy, T, busy, toks, 1)
    raise ValueError(f"unknown strategy {strategy}")


STRATEGIES = ("serial", "serial-sd", "scheduled-sd", "batched-sd", "pipelined-sd", "parallel")


def sweep(params_list, strategies=STRATEGIES, t_verify_batch=None):
    """CSV rows: strategy, n, k, l, alpha, makespan, busy_fraction, tokens_per_tick, speedup_vs_serial."""
    rows = ["strategy,n,k,l,alpha,makespan,busy_fraction,tokens_per_tick,speedup_vs_serial"]
    for p in params_list:
        base = simulate("serial", p).makespan
        for st in strategies:
            r = simulate(st, p, t_verify_batch)
            rows.append(f"{st},{p.n},{p.k},{p.l},{p.alpha},{r.makespan},{r.busy_fraction:.4f},"
                        f"{r.tokens_per_tick:.4f},{base / r.makespan:.4f}")
    return rows
