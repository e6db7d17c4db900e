"""CPU oracle for the SeeD draft-then-verify round -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct implementation of what the
hot path computes, written from the paper (arXiv 2406.18200, `PAPER.md`) and
the readings recorded in DESIGN.md.  It exists to prove the CUDA path right.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product path
(`paper_2406_18200_b200`) never imports, links or executes anything here and
fails loudly when its CUDA library is missing.  The oracle shares no code,
tables or constants with the CUDA path; the only common module is `seedgen/`,
which draws the synthetic inputs and holds none of the method's arithmetic.

Modules (each function cites the passage it follows; `P:n` = PAPER.md line n,
`S:n` = SPEC.md line n, "R<k>" = DESIGN.md reading k):
  philox     -- Philox4x32-10 counter-based RNG + the odd-grid uniform (R5, R17)
  sampling   -- speculative sampling: accept test, residual, bonus, race
  llama      -- Llama-2 forward, fp64 and bf16-faithful (R15)
  scheduler  -- FCFS rounds scheduler (Alg. 1)
  seed_round -- one full round per stream and the run loop (Alg. 1)

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Random123 known-answer vectors,
the SPEC worked example, q == p acceptance, exact enumeration losslessness,
chi-square goodness of fit, closed-form E[emitted], HF `LlamaForCausalLM` in
float64, cached == uncached decode, the SPEC scheduler hand trace.
"""
