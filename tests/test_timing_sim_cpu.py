"""Timing model of Fig. 1's strategies (paper_2406_18200_b200.timing_sim): hand traces and invariants.

Hand traces are worked here from the service model (DESIGN R29), not from the module:
  * serial-sd, n=1, alpha=1, k=2, l=4, t_draft=t_verify=1: two rounds of 2*1 + 1 -> 6 ticks;
  * serial, n=3, l=4, t_target_ar=1 -> 12 ticks, target busy 100 %;
  * scheduled-sd, n=2, alpha=1, k=1, l=2, t_draft=2, t_verify=1: both drafts ready at 2, the
    target verifies s0 in [2, 3) and s1 in [3, 4) -> 4 ticks (serial-sd: 2 * (2 + 1) = 6).
"""
import numpy as np
import pytest

from paper_2406_18200_b200.timing_sim import STRATEGIES, TimingParams, simulate, sweep


def test_hand_traces():
    p = TimingParams(t_draft=1, t_verify=1, t_resample=1, n=1, k=2, l=4, alpha=1.0)
    assert simulate("serial-sd", p).makespan == 6
    r = simulate("serial", TimingParams(t_target_ar=1, n=3, l=4))
    assert r.makespan == 12 and r.busy_fraction == 1.0
    p = TimingParams(t_draft=2, t_verify=1, n=2, k=1, l=2, alpha=1.0)
    assert simulate("scheduled-sd", p).makespan == 4
    assert simulate("serial-sd", p).makespan == 6
    assert simulate("parallel", TimingParams(t_target_ar=3, n=5, l=4)).peak_target_instances == 5


def test_rejection_costs_resample():
    p = TimingParams(t_draft=1, t_verify=2, t_resample=3, n=1, k=3, l=1, alpha=0.0)
    assert simulate("serial-sd", p).makespan == 3 * 1 + 2 + 3     # one round, first token rejected


@pytest.mark.parametrize("seed", range(6))
def test_dominance_and_accounting(seed):
    rng = np.random.default_rng(seed)
    p = TimingParams(t_draft=int(rng.integers(1, 4)), t_verify=int(rng.integers(1, 6)),
                     t_resample=int(rng.integers(0, 3)), n=int(rng.integers(1, 9)), k=int(rng.integers(1, 6)),
                     l=int(rng.integers(4, 40)), alpha=float(rng.random()), seed=seed)
    sd, sch = simulate("serial-sd", p), simulate("scheduled-sd", p)
    assert sch.makespan <= sd.makespan
    assert sch.target_busy == sd.target_busy                   # same verifications, common random numbers
    assert sch.makespan >= sch.target_busy                     # one target: busy + idle = makespan
    if p.n == 1:
        assert sch.makespan == sd.makespan


def test_alpha_monotone_with_common_random_numbers():
    ms = [simulate("serial-sd", TimingParams(n=4, k=4, l=32, alpha=a, seed=3)).makespan
          for a in np.linspace(0.05, 0.95, 10)]
    assert all(x >= y for x, y in zip(ms, ms[1:]))


def test_busy_fraction_saturates_in_n():
    fr = [simulate("scheduled-sd", TimingParams(t_draft=2, t_verify=1, t_resample=0, n=n, k=4, l=100,
                                                alpha=1.0)).busy_fraction for n in range(1, 13)]
    assert all(x <= y + 1e-12 for x, y in zip(fr, fr[1:]))
    # n = 1: 20 rounds of 8 + 1 ticks; n = 12 >= (8 + 1) / 1: the target never idles after the
    # first 8-tick draft, so makespan = 8 + 12 * 20 (Fig. 5(b): fixed verification capacity)
    assert fr[0] == 20 / (20 * 9)
    assert fr[-1] == 240 / (8 + 240)


def test_batched_sd_with_batch_cost_and_sweep():
    p = TimingParams(t_draft=1, t_verify=10, t_resample=0, n=4, k=4, l=10, alpha=1.0)
    r = simulate("batched-sd", p, t_verify_batch=lambda m: 10 + m)
    assert r.makespan == 2 * (4 * 1 + 10 + 4)                  # 2 rounds of 5 tokens, 4 streams each
    rows = sweep([p, TimingParams(n=1)])
    assert rows[0].startswith("strategy,") and len(rows) == 1 + 2 * len(STRATEGIES)
    with pytest.raises(ValueError):
        simulate("serial", TimingParams(alpha=2.0))


def test_pipelined_hand_trace():
    # n = 2, alpha = 1, k = 1, l = 2: one round per stream.  A drafts [0, 2); then verify A (3)
    # || draft B (2) -> 3; then verify B (3) -> 3; makespan 2 + 3 + 3 = 8.
    p = TimingParams(t_draft=2, t_verify=3, n=2, k=1, l=2, alpha=1.0)
    r = simulate("pipelined-sd", p)
    assert r.makespan == 8 and r.target_busy == 6
    # when drafting dominates, the overlap hides verification: draft 10, verify 1, two rounds each
    p = TimingParams(t_draft=10, t_verify=1, n=2, k=1, l=4, alpha=1.0)
    assert simulate("pipelined-sd", p).makespan == 10 + 10 + 10 + 10 + 1
    assert simulate("batched-sd", p).makespan == 2 * (10 + 1)
