"""One draft-then-verify round per stream and the run loop -- TEST INFRASTRUCTURE ONLY.

Follows Alg. 1 in the lock-step batched reading (DESIGN R9):
  a1  scheduler pops <= C ready streams FCFS
  a2  each stream drafts gamma tokens autoregressively
  a3  the target scores [T_s[-1], x_1..x_gamma]
  a4  accept / resample / bonus                             (R1-R4)
  a5  commit, truncate to l, roll the caches back           (R6, R7)
  a6  re-enqueue undone streams
KV convention (R6): before a round the target cache holds |T_s| - 1 tokens;
the draft cache holds min(|T_s| - 1, entries written) and the tokens
T_s[len(draft cache):] (1 or 2) are still pending for the draft.
"""
from dataclasses import dataclass, field

import numpy as np

from . import llama as _ll
from . import sampling as _sp
from .scheduler import RoundScheduler


@dataclass
class StreamState:
    sid: int
    T: list                     # validated tokens (prompt + emitted)
    prompt_len: int
    tcache: object
    dcache: object
    L: int = 0                  # new validated tokens (R7: starts at 0)
    r: int = 0                  # stream-local round counter (R5)
    done: bool = False
    history: list = field(default_factory=list)

    @property
    def pending(self):
        return self.T[len(self.dcache):]


@dataclass
class RoundRecord:
    sid: int
    r: int
    xs: list
    a: int
    emitted: list
    flags: int
    accept_margins: list
    race_gap: float
    draft_gaps: list
    zt: np.ndarray = None
    zd: np.ndarray = None


class SeedOracle:
    """Plain CPU model of the whole round, one stream after another."""

    def __init__(self, tshape, tW, dshape, dW, gamma, temperature, seed, bonus=True,
                 max_new=64, mode="bf16", keep_logits=False):
        assert tshape.vocab == dshape.vocab, "shared vocabulary (S:38)"
        self.ts, self.tW, self.ds, self.dW = tshape, tW, dshape, dW
        self.gamma, self.T, self.seed = int(gamma), float(temperature), int(seed)
        self.bonus, self.max_new, self.mode = bool(bonus), int(max_new), mode
        self.keep_logits = keep_logits
        self.streams = {}

    def add_stream(self, sid, prompt):
        """Alg. 1 Initialize: prefill both models with the prefix."""
        prompt = [int(t) for t in prompt]
        assert len(prompt) >= 1
        st = StreamState(sid=int(sid), T=list(prompt), prompt_len=len(prompt),
                         tcache=_ll.KVCache(self.ts), dcache=_ll.KVCache(self.ds))
        if len(prompt) > 1:
            _ll.forward_batch(self.ts, self.tW, [(prompt[:-1], st.tcache)], mode=self.mode, logits_rows=[[]])
            _ll.forward_batch(self.ds, self.dW, [(prompt[:-1], st.dcache)], mode=self.mode, logits_rows=[[]])
        self.streams[st.sid] = st
        return st

    def draft(self, batch):
        """a2: gamma autoregressive draft steps for every stream in the batch."""
        g = self.gamma
        xs = {s: [] for s in batch}
        zds = {s: [] for s in batch}
        gaps = {s: [] for s in batch}
        for j in range(1, g + 1):
            seqs, rows = [], []
            for s in batch:
                st = self.streams[s]
                toks = st.pending if j == 1 else [xs[s][-1]]
                seqs.append((toks, st.dcache))
                rows.append([len(toks) - 1])
            outs = _ll.forward_batch(self.ds, self.dW, seqs, mode=self.mode, logits_rows=rows)
            for s, z in zip(batch, outs):
                st = self.streams[s]
                tok, gap = _sp.draft_token(z[0], self.T, self.seed, st.sid, st.r, j)
                xs[s].append(tok)
                zds[s].append(z[0])
                gaps[s].append(gap)
        return xs, zds, gaps

    def verify(self, batch, xs):
        """a3: one target forward over [T_s[-1], x_1..x_gamma] per stream."""
        seqs = [([self.streams[s].T[-1]] + xs[s], self.streams[s].tcache) for s in batch]
        outs = _ll.forward_batch(self.ts, self.tW, seqs, mode=self.mode)
        return {s: z for s, z in zip(batch, outs)}

    def round(self, batch):
        xs, zds, gaps = self.draft(batch)
        zts = self.verify(batch, xs)
        recs = []
        for s in batch:
            st = self.streams[s]
            zt, zd = zts[s], np.stack(zds[s])
            res = _sp.verify_stream(zt, zd, xs[s], self.T, self.seed, st.sid, st.r, bonus=self.bonus)
            recs.append(RoundRecord(st.sid, st.r, list(xs[s]), res.a, list(res.emitted), res.flags,
                                    res.accept_margins, res.race_gap, gaps[s],
                                    zt if self.keep_logits else None, zd if self.keep_logits else None))
            self.commit(st, res.emitted)
        return recs

    def commit(self, st, emitted):
        """a5: append, truncate to l, roll both caches back (R6)."""
        room = self.max_new - st.L
        emitted = emitted[:room]
        st.T.extend(emitted)
        st.L += len(emitted)
        st.history.append(list(emitted))
        st.r += 1
        st.tcache.truncate(len(st.T) - 1)
        st.dcache.truncate(min(len(st.T) - 1, len(st.dcache)))
        if st.L >= self.max_new:
            st.done = True

    def run(self, capacity, max_rounds=100000):
        """Alg. 1 main loop in lock-step batches; returns {sid: new tokens}."""
        sched = RoundScheduler(self.streams.keys())
        rounds = []
        for _ in range(max_rounds):
            if sched.all_done():
                break
            batch = sched.schedule(capacity)
            recs = self.round(batch)
            rounds.append(recs)
            sched.complete(batch, [self.streams[s].done for s in batch])
        out = {s: st.T[st.prompt_len:] for s, st in self.streams.items()}
        return out, rounds, sched


def verify_batch(zt, zd, xs, temperature, seed, sids, rs, bonus=True):
    """a4 alone, on given logits (K4 parity): zt [B][g+1][V], zd [B][g][V], xs [B][g]."""
    return [_sp.verify_stream(zt[b], zd[b], xs[b], temperature, seed, int(sids[b]), int(rs[b]), bonus=bonus)
            for b in range(len(sids))]
