"""Oracle pin: Philox4x32-10 against the Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
import os

import numpy as np

from oracle import philox as ph

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kats():
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        yield w[:4], w[4:6], w[6:10]


def test_kat_scalar():
    n = 0
    for ctr, key, out in _kats():
        assert list(ph.philox4x32_10(ctr, key)) == out
        n += 1
    assert n == 3


def test_kat_vectorised():
    for ctr, key, out in _kats():
        got = ph.philox4x32_10_np(*[np.array([c], dtype=np.uint64) for c in ctr], key[0], key[1])
        assert [int(g[0]) for g in got] == out


def test_vectorised_matches_scalar_over_counters():
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64)
    k0, k1 = 0x5EED2406, 0x12345678
    vec = ph.philox4x32_10_np(c[0], c[1], c[2], c[3], k0, k1)
    for i in range(64):
        assert tuple(int(v[i]) for v in vec) == ph.philox4x32_10(tuple(int(x) for x in c[:, i]), (k0, k1))


def test_uniform_grid():
    # R2: u = (2k+1) 2^-24, k in [0, 2^23): never 0 or 1, exact in fp32
    assert ph.u_from_word(0) == 2.0 ** -24
    assert ph.u_from_word(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    xs = np.random.default_rng(1).integers(0, 2**32, size=10000, dtype=np.uint64)
    u = ph.u_from_word_np(xs)
    assert np.all(u > 0) and np.all(u < 1)
    assert np.all(u.astype(np.float32).astype(np.float64) == u)


def test_race_uniform_layout():
    # R17: u_v = word (v & 3) of counter (v >> 2, tag<<24|slot, r, sid)
    seed, sid, r, tag, slot = 0x5EED2406, 7, 3, ph.TAG_RESAMPLE, 2
    u = ph.race_uniforms(seed, sid, r, tag, slot, 11)
    for v in range(11):
        assert u[v] == ph.philox_u(seed, sid, r, tag, slot, v >> 2, v & 3)
