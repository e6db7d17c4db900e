"""ToT-BFS driver (Alg. 2, App. C) over the C ABI -- SURVEY §8(f) rank 1.

Host logic only: every token is produced by libseed's round (seed_schedule_round ->
seed_draft_round -> seed_verify) through `EngineGenerator`.  Per tree level:

  * Thought Generator ("Generate thoughts in Parallel"): every surviving state c gets n
    streams with the identical prefix c (§4.1: "the input instructions are the same"); all
    |S_{i-1}| * n streams of the level are admitted to ONE scheduler run (DESIGN R28: pooled,
    so the target verifies them together; tokens do not depend on the pooling because the
    Philox counters are keyed by global stream id and stream-local round, and the kernels are
    batch-invariant -- R19).
  * State Evaluator: one stream per candidate with the prompt
    eval_prefix + state + eval_suffix (distinct prefixes), value parsed from the response (R26).
  * Selection: argmax over size-b subsets of the score sum == the b highest scores,
    ties to the earlier-created candidate (R25); kept states stay in creation order.
  * Return: one more generation (n = 1) from the best kept state.

Global stream ids come from one counter in call order (R27); finished streams are removed
(seed_remove_stream frees their KV pages) so max_streams bounds one call, not the tree.
"""
import time
from dataclasses import dataclass, field


@dataclass
class ToTConfig:
    depth: int                      # step limit T (App. D: GSM8K 4, CW 2, BW 7)
    n: int = 3                      # thoughts per expanded state
    b: int = 1                      # breadth limit
    eval_prefix: tuple = ()         # evaluator template tokens before the state
    eval_suffix: tuple = ()         # ... and after it (the "value:" slot)
    digit_base: int = None          # scalar mode: tokens digit_base..digit_base+9 mean 0..9
    table: dict = None              # classifier mode: token -> value (e.g. good -> 1, bad -> 0)
    default: float = 0.0            # unparseable response


@dataclass
class ToTResult:
    answer: list
    levels: list = field(default_factory=list)   # per level: states, scores, keep, parent
    calls: list = field(default_factory=list)    # ("G" | "E", number of streams)
    rounds: int = 0


def value_of(response, cfg):
    """R26: first token that the classifier table knows, or that lies in the digit range."""
    for t in response:
        if cfg.table is not None and t in cfg.table:
            return float(cfg.table[t])
        if cfg.digit_base is not None and cfg.digit_base <= t < cfg.digit_base + 10:
            return float(t - cfg.digit_base)
    return float(cfg.default)


def top_b(scores, b):
    """Indices of the b largest scores, stable (earlier index wins a tie), returned ascending."""
    order = sorted(range(len(scores)), key=lambda j: (-scores[j], j))
    return sorted(order[:min(b, len(scores))])


class EngineGenerator:
    """G(p_theta, prefixes): run SeedEngine rounds until every stream of the call is done.

    share_prefix: a prefix repeated inside one call (the n thoughts of a state) is prefilled once;
    its siblings get a device copy of those K/V pages (seed_fork_stream) -- same tokens.
    """

    def __init__(self, engine, share_prefix=True):
        self.eng = engine
        self.share_prefix = share_prefix
        self.rounds = 0
        self.prefills = 0
        self.t_add = self.t_rounds = 0.0      # host wall seconds (admission incl. prefill / round loop)

    def __call__(self, prefixes, gids):
        eng = self.eng
        t0 = time.perf_counter()
        first = {}
        for g, p in zip(gids, prefixes):
            key = tuple(p)
            if self.share_prefix and key in first:
                eng.fork_stream(first[key], g)
                continue
            eng.add_stream(g, p)
            first[key] = g
            self.prefills += 1
        t1 = time.perf_counter()
        while True:
            batch = eng.schedule()
            if not batch:
                break
            eng.draft(batch)
            eng.verify(batch)
            self.rounds += 1
        self.t_add += t1 - t0
        self.t_rounds += time.perf_counter() - t1
        outs = []
        for g in gids:
            outs.append(eng.tokens(g))          # seed_get_tokens: the new tokens only
            eng.remove_stream(g)
        return outs


class ToTBFS:
    """Alg. 2 driver; `generate(prefixes, gids) -> [new tokens]` is EngineGenerator on a GPU."""

    def __init__(self, generate, cfg, first_gid=0):
        if cfg.depth < 1 or cfg.n < 1 or cfg.b < 1:
            raise ValueError("ToT-BFS needs depth >= 1, n >= 1, b >= 1")
        self.generate, self.cfg, self.next_gid = generate, cfg, int(first_gid)

    def _run(self, prefixes, tag, res):
        gids = list(range(self.next_gid, self.next_gid + len(prefixes)))
        self.next_gid += len(prefixes)
        res.calls.append((tag, len(prefixes)))
        return self.generate(prefixes, gids)

    def build(self, prompt):
        cfg = self.cfg
        res = ToTResult(answer=[])
        S = [list(prompt)]
        for _ in range(cfg.depth):
            parent = [i for i in range(len(S)) for _ in range(cfg.n)]
            thoughts = self._run([S[i] for i in parent], "G", res)
            cand = [S[i] + z for i, z in zip(parent, thoughts)]
            resp = self._run([list(cfg.eval_prefix) + c + list(cfg.eval_suffix) for c in cand], "E", res)
            scores = [value_of(r, cfg) for r in resp]
            keep = top_b(scores, cfg.b)
            res.levels.append({"states": cand, "scores": scores, "keep": keep, "parent": parent})
            S = [cand[j] for j in keep]
        last = res.levels[-1]
        best = keep[top_b([last["scores"][j] for j in keep], 1)[0]]
        res.answer = self._run([last["states"][best]], "G", res)[0]
        res.rounds = getattr(self.generate, "rounds", 0)
        return res
