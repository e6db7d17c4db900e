"""Rounds-scheduled FCFS scheduler (Alg. 1) -- TEST INFRASTRUCTURE ONLY.

Paper passages followed:
  P:201     finished drafts are "placed into a queue"
  P:204     "a sequence of draft tokens is dequeued in the FCFS manner"
  P:206     "Upon completion of the verification ... the draft model proceeds to
            the drafting process in the next iteration" (rounds)
  P:250     verify queue Q, draft label map (ready flag) initialised to 1
  P:259     ready[i] <- 0 after drafting;  P:277 ready[i] <- 1 after verification
  P:255/263 loops run while some L_i < l; DESIGN R7: done when L_i >= l
Readings: R8 (ready-flag semantics follow Alg. 1), R9 (one batched verify per
round), R10 (ties -> lowest global id), R11 (capacity C per round).

Lock-step batched form: a round pops up to C streams that are ready and not
done, FCFS; after verification the undone ones re-enter at the tail in batch
order with ready = 1.  With C >= #active this is lock-step; with C < #active it
is round-robin, i.e. the paper's "rounds".
"""
from collections import deque


class DeadlockError(RuntimeError):
    """S:213 liveness: every ready flag is 0 with an empty queue while work remains."""


class RoundScheduler:
    def __init__(self, stream_ids):
        ids = sorted(int(s) for s in stream_ids)           # R10 ties -> lowest id
        self.queue = deque(ids)
        self.ready = {s: 1 for s in ids}                   # P:250 all ones
        self.done = {s: False for s in ids}
        self.dropped = []                                  # S:211 done streams met in the queue
        self.trace = []                                    # (event, sid)

    def add(self, sid):
        sid = int(sid)
        self.ready[sid] = 1
        self.done[sid] = False
        self.queue.append(sid)
        self.trace.append(("enqueue", sid))

    def all_done(self):
        return all(self.done.values())

    def schedule(self, capacity):
        """Pop up to `capacity` ready, undone streams in FCFS order."""
        batch = []
        while self.queue and len(batch) < capacity:
            sid = self.queue.popleft()
            if self.done[sid]:
                self.dropped.append(sid)
                continue
            assert self.ready[sid] == 1, "ready-flag safety (S:223)"
            self.ready[sid] = 0
            batch.append(sid)
            self.trace.append(("dequeue", sid))
        if not batch and not self.all_done():
            raise DeadlockError("no ready stream while some L_i < l")
        return batch

    def complete(self, batch, done_flags):
        """After verification: ready <- 1; undone streams re-enqueue at the tail."""
        for sid, dn in zip(batch, done_flags):
            self.ready[sid] = 1
            self.done[sid] = bool(dn)
            self.trace.append(("verified", sid))
            if not dn:
                self.queue.append(sid)
                self.trace.append(("enqueue", sid))
