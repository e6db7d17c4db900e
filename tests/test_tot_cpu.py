"""ToT-BFS (Alg. 2): oracle pins and the product driver's host logic, on CPU.

The generator is an injected deterministic function of (global id, prefix) -- the token path
is covered by test_gpu_tot.py.  Pins of oracle/tot.py that do not use its own code:
  * b >= n^T keeps every node, so the answer must come from the best of ALL n^T leaves found
    by recursive exhaustive enumeration (brute force over the full candidate tree);
  * call accounting 2T + 1 with n * |S_{i-1}| streams per generation batch;
  * App. D value strategies on hand-written responses; the stable tie rule on (5, 5, 3).
The product driver (paper_2406_18200_b200.tot) must then reproduce the oracle's tree exactly.
"""
import itertools

import numpy as np
import pytest

from oracle import tot as otot
from paper_2406_18200_b200 import tot as ptot

V, LEN = 16, 3
DIGIT = 3                      # tokens 3..12 mean 0..9


def fake_generate(prefixes, gids):
    """Deterministic stand-in for G: tokens depend on the stream id and the prefix."""
    outs = []
    for g, p in zip(gids, prefixes):
        rng = np.random.default_rng([int(g), len(p), int(sum(p)) % 100003, int(p[-1])])
        outs.append(rng.integers(0, V, size=LEN).tolist())
    return outs


def _cfgs(T, n, b):
    return ptot.ToTConfig(depth=T, n=n, b=b, eval_prefix=(1, 2), eval_suffix=(15,), digit_base=DIGIT)


def _oracle(prompt, T, n, b, gen=fake_generate):
    return otot.seed_bfs(prompt, gen, T, n, b, (1, 2), (15,), digit_base=DIGIT)


def test_parse_value_app_d():
    assert otot.parse_value([0, 1, DIGIT + 7, DIGIT + 2], digit_base=DIGIT) == 7.0       # scalar "7 ..."
    assert otot.parse_value([9, 4], table={9: 1, 4: 0}) == 1.0                          # "good" first
    assert otot.parse_value([0, 1, 2], digit_base=DIGIT, default=0.0) == 0.0             # no value
    assert otot.parse_value([], digit_base=DIGIT, default=-1.0) == -1.0
    cfg = ptot.ToTConfig(depth=1, digit_base=DIGIT)
    for r in ([0, 1, DIGIT + 7], [2, 2], [DIGIT + 9, DIGIT]):
        assert ptot.value_of(r, cfg) == otot.parse_value(r, digit_base=DIGIT)


def test_tie_rule_5_5_3():
    assert ptot.top_b([5.0, 5.0, 3.0], 1) == [0]
    gen_scores = iter([[DIGIT + 5], [DIGIT + 5], [DIGIT + 3]])

    def gen(prefixes, gids):
        if prefixes[0][:2] == [1, 2]:                      # evaluator prompts
            return [next(gen_scores) for _ in prefixes]
        return [[0] for _ in prefixes]
    _, levels, _ = _oracle([7, 7], 1, 3, 1, gen)
    assert levels[0]["keep"] == [0]


def _leaves(prompt, T, n, gen_first_gid):
    """Exhaustive enumeration of the full tree when b keeps everything: gids follow the same
    counter as BFS (level by level), so rebuild level by level and return all leaves."""
    gid = gen_first_gid
    level = [list(prompt)]
    for _ in range(T):
        parents = [c for c in level for _ in range(n)]
        outs = fake_generate(parents, list(range(gid, gid + len(parents))))
        gid += len(parents)
        cand = [c + z for c, z in zip(parents, outs)]
        outs_e = fake_generate([[1, 2] + c + [15] for c in cand], list(range(gid, gid + len(cand))))
        gid += len(cand)
        scores = [otot.parse_value(o, digit_base=DIGIT) for o in outs_e]
        level = cand
    return level, scores


@pytest.mark.parametrize("T,n", [(1, 3), (2, 3), (3, 2)])
def test_full_breadth_equals_exhaustive(T, n):
    prompt = [5, 9, 4]
    leaves, scores = _leaves(prompt, T, n, 0)
    best = max(range(len(leaves)), key=lambda j: (scores[j], -j))
    ans, levels, _ = _oracle(prompt, T, n, n ** T)
    assert levels[-1]["states"] == leaves and levels[-1]["scores"] == scores
    gid_final = sum(2 * n ** i for i in range(1, T + 1))
    assert ans == fake_generate([leaves[best]], [gid_final])[0]


@pytest.mark.parametrize("T,n,b", [(1, 1, 1), (2, 3, 1), (3, 3, 2), (4, 3, 3), (2, 2, 5), (7, 3, 1)])
def test_oracle_invariants_and_product_parity(T, n, b):
    prompt = [5, 9, 4, 11]
    ans, levels, calls = _oracle(prompt, T, n, b)
    # call accounting: T x (G + E) + final G; n * |S_{i-1}| streams per expansion
    assert [c[0] for c in calls] == ["G", "E"] * T + ["G"]
    width = 1
    for i, lv in enumerate(levels):
        assert calls[2 * i][1] == n * width == len(lv["states"])
        k = min(b, len(lv["states"]))
        assert len(lv["keep"]) == k
        best = max(sum(c) for c in itertools.combinations(lv["scores"], k))   # selection optimality
        assert sum(lv["scores"][j] for j in lv["keep"]) == best
        prev = [prompt] if i == 0 else [levels[i - 1]["states"][j] for j in levels[i - 1]["keep"]]
        for s, p in zip(lv["states"], lv["parent"]):                         # ancestry
            assert s[:len(prev[p])] == prev[p] and len(s) == len(prev[p]) + LEN
        width = k
    # the product driver reproduces the oracle's tree
    res = ptot.ToTBFS(fake_generate, _cfgs(T, n, b)).build(prompt)
    assert res.calls == calls
    assert res.answer == ans
    for a, o in zip(res.levels, levels):
        assert a["states"] == o["states"] and a["scores"] == o["scores"]
        assert a["keep"] == o["keep"] and a["parent"] == o["parent"]


def test_driver_rejects_bad_config():
    with pytest.raises(ValueError):
        ptot.ToTBFS(fake_generate, ptot.ToTConfig(depth=0))


class _FakeEngine:
    """Records the C-ABI calls EngineGenerator makes (host logic only)."""

    def __init__(self):
        self.calls, self.live, self.prefix = [], set(), {}

    def add_stream(self, g, p):
        self.calls.append(("add", g))
        self.live.add(g)
        self.prefix[g] = list(p)

    def fork_stream(self, src, g):
        assert src in self.live
        self.calls.append(("fork", src, g))
        self.live.add(g)
        self.prefix[g] = list(self.prefix[src])

    def schedule(self):
        b = sorted(g for g in self.live if ("done", g) not in self.calls)
        return b

    def draft(self, b):
        self.calls.append(("draft", tuple(b)))

    def verify(self, b):
        self.calls += [("done", g) for g in b]

    def tokens(self, g):
        return fake_generate([self.prefix[g]], [g])[0]

    def remove_stream(self, g):
        self.live.remove(g)
        self.calls.append(("remove", g))


@pytest.mark.parametrize("share", [True, False])
def test_engine_generator_forks_repeated_prefixes(share):
    eng = _FakeEngine()
    gen = ptot.EngineGenerator(eng, share_prefix=share)
    prefixes = [[5, 6], [5, 6], [7, 8], [5, 6], [7, 8]]
    outs = gen(prefixes, [10, 11, 12, 13, 14])
    adds = [c for c in eng.calls if c[0] == "add"]
    forks = [c for c in eng.calls if c[0] == "fork"]
    if share:
        assert adds == [("add", 10), ("add", 12)]
        assert forks == [("fork", 10, 11), ("fork", 10, 13), ("fork", 12, 14)]     # call order
        assert gen.prefills == 2
    else:
        assert len(adds) == 5 and not forks and gen.prefills == 5
    assert outs == fake_generate(prefixes, [10, 11, 12, 13, 14])
    assert not eng.live and gen.rounds == 1                  # every stream removed after the call
