#!/usr/bin/env python
"""n-sweep of the Fig. 1 strategies with service times taken from this build's B200 measurements.

    python scripts/timing_sweep.py > profiles/r01/timing_sweep.csv

Ticks are microseconds.  Measured (profiles/r01/bench, 68M draft + 7B target, gamma = 4):
draft phase ~284 us per round at N = 3 -> t_draft = 71 us per token; device round 3.19 ms at
N = 3 and 6.00 ms at N = 24 -> batched verification t_verify_batch(m) ~ 2.90 + (m - 3) * 0.1333 ms
(linear between the two measured points).  The paper's scheduled SD verifies one draft at a
time; on B200 a single-stream 7B verification still streams all 13.2 GB of weights, so it costs
~t_verify_batch(1).  t_target_ar: one 7B decode step ~ the same weight stream, 2.0 ms (HBM bound).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_18200_b200.timing_sim import TimingParams, sweep  # noqa: E402


def t_verify_batch(m):
    return int(round(2900 + (m - 3) * (5700 - 2900) / 21))


def main():
    ps = [TimingParams(t_draft=71, t_verify=t_verify_batch(1), t_resample=0, t_target_ar=2000, n=n, k=4, l=64,
                       alpha=a, seed=1) for a in (0.5, 0.8) for n in (1, 3, 6, 12, 24)]
    print("\n".join(sweep(ps, t_verify_batch=t_verify_batch)))


if __name__ == "__main__":
    main()
