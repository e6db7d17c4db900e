"""ToT-BFS reasoning-tree construction (Alg. 2, App. C) -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module.  It writes Alg. 2 out literally:

  S_0 <- {I}
  for i = 1..T:
      S'_i <- {[c, z] | c in S_{i-1}, z in G(p_theta, c, n)}          ("Generate thoughts in Parallel")
      E_i  <- E(p_theta, S'_i)                                        ("Evaluate states in Parallel")
      S_i  <- argmax_{S subset S'_i, |S| = b} sum_{s in S} E_i(s)
  return G(p_theta, argmax_{s in S_T} E_T(s), 1)

The arg-max over subsets is enumerated by brute force (itertools.combinations in creation order;
the first maximum wins -- DESIGN R25 tie rule), not by sorting, so it pins the product driver's
top-b selection independently.  The evaluator's value strategy (App. D: "a scalar value
(e.g., '1-10') or a classification (e.g., 'good/bad') which can be heuristically converted into a
value") is read as DESIGN R26: the first token of the response inside the digit range
[digit_base, digit_base + 10) gives its offset, or the classifier table maps the first token found
in it; no such token -> the default value.

`generate(prefixes, gids)` is any callable returning one token list per prefix (the oracle's
SeedOracle run for parity; an injected heuristic for the brute-force pins).  Stream ids are drawn
from one counter in call order (R27), so the Philox streams of both sides agree.
"""
import itertools


def parse_value(response, digit_base=None, table=None, default=0.0):
    """R26: App. D value strategy on token ids."""
    for t in response:
        if table is not None and t in table:
            return float(table[t])
        if digit_base is not None and digit_base <= t < digit_base + 10:
            return float(t - digit_base)
    return float(default)


def seed_bfs(prompt, generate, T, n, b, eval_prefix, eval_suffix, digit_base=None, table=None, default=0.0,
             first_gid=0):
    """Alg. 2 step by step.  Returns (answer tokens, levels, calls)."""
    gid = [first_gid]
    calls = []

    def G(prefixes):
        gids = list(range(gid[0], gid[0] + len(prefixes)))
        gid[0] += len(prefixes)
        outs = generate(prefixes, gids)
        calls.append(("G", len(prefixes)))
        return outs

    def E(states):
        prompts = [list(eval_prefix) + list(s) + list(eval_suffix) for s in states]
        gids = list(range(gid[0], gid[0] + len(prompts)))
        gid[0] += len(prompts)
        outs = generate(prompts, gids)
        calls.append(("E", len(prompts)))
        return [parse_value(o, digit_base, table, default) for o in outs]

    S = [list(prompt)]                                               # S_0 <- {I}
    levels = []
    for i in range(1, T + 1):
        parents = [c for c in S for _ in range(n)]                   # n thoughts per state
        thoughts = G(parents)
        S_prime = [c + z for c, z in zip(parents, thoughts)]         # [c, z_i]
        E_i = E(S_prime)
        k = min(b, len(S_prime))                                     # fewer than b -> keep all
        best, best_sum = None, None
        for comb in itertools.combinations(range(len(S_prime)), k):
            tot = sum(E_i[j] for j in comb)
            if best_sum is None or tot > best_sum:
                best, best_sum = comb, tot
        levels.append({"states": S_prime, "scores": E_i, "keep": list(best),
                       "parent": [j // n for j in range(len(S_prime))]})
        S = [S_prime[j] for j in best]
    scores_T = [levels[-1]["scores"][j] for j in levels[-1]["keep"]]
    s_best = S[max(range(len(S)), key=lambda j: (scores_T[j], -j))]
    answer = G([s_best])[0]
    return answer, levels, calls
