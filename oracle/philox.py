"""Philox4x32-10 (Salmon et al., SC'11) and the uniform/exponential conversion.

Test infrastructure only (see oracle/__init__.py).

The paper fixes no RNG (it only says drafts are accepted "with the probability"
min(1, p_t/p_d)).  The build reads it as a counter-based generator keyed
by (seed, global stream id, stream-local round, tag, slot) -- DESIGN.md R5/R17 --
so that the realisation is independent of batching, scheduling and world size.

Counter layout (R5): c0 = draw block, c1 = tag << 24 | slot, c2 = stream-local
round r_s, c3 = global stream id.  Key = (lo32(seed), hi32(seed)).
Uniform (R2): k = x >> 9 (23 bits), u = (2k + 1) * 2^-24  in [2^-24, 1 - 2^-24].

Pinned by the Random123 known-answer vectors (tests/test_oracle_philox.py).
"""
import numpy as np

M32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85

TAG_DRAFT = 1      # draft race at step j (slot j)
TAG_ACCEPT = 2     # accept uniform for draft position j (slot j, c0 = 0, word 0)
TAG_RESAMPLE = 3   # residual / bonus race (slot a + 1)


def philox4x32_10(ctr, key):
    """Scalar Philox4x32-10: ctr = 4 uint32, key = 2 uint32 -> 4 uint32."""
    c0, c1, c2, c3 = (int(x) & M32 for x in ctr)
    k0, k1 = (int(x) & M32 for x in key)
    for rnd in range(10):
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> 32, p0 & M32
        hi1, lo1 = p1 >> 32, p1 & M32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & M32, lo1, (hi0 ^ c3 ^ k1) & M32, lo0
        if rnd < 9:
            k0 = (k0 + PHILOX_W0) & M32
            k1 = (k1 + PHILOX_W1) & M32
    return (c0, c1, c2, c3)


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over numpy arrays (uint64 carriers of uint32 values).

    Same round function as `philox4x32_10`; broadcasting over the counter words.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & M32
    c1 = np.asarray(c1, dtype=np.uint64) & M32
    c2 = np.asarray(c2, dtype=np.uint64) & M32
    c3 = np.asarray(c3, dtype=np.uint64) & M32
    k0 = np.uint64(int(k0) & M32)
    k1 = np.uint64(int(k1) & M32)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    m0 = np.uint64(PHILOX_M0)
    m1 = np.uint64(PHILOX_M1)
    mask = np.uint64(M32)
    s32 = np.uint64(32)
    for rnd in range(10):
        p0 = m0 * c0            # < 2^64, exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> s32, p0 & mask
        hi1, lo1 = p1 >> s32, p1 & mask
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & mask, lo1, (hi0 ^ c3 ^ k1) & mask, lo0
        if rnd < 9:
            k0 = np.uint64((int(k0) + PHILOX_W0) & M32)
            k1 = np.uint64((int(k1) + PHILOX_W1) & M32)
    return c0, c1, c2, c3


def seed_key(seed):
    """Key = (lo32(seed), hi32(seed)) (R5)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & M32, seed >> 32


def u_from_word(x):
    """Odd-grid uniform (R2): u = (2*(x >> 9) + 1) / 2^24, exact in fp32 and fp64."""
    return (2.0 * (int(x) >> 9) + 1.0) / 16777216.0


def u_from_word_np(x):
    x = np.asarray(x, dtype=np.uint64)
    return (2.0 * (x >> np.uint64(9)).astype(np.float64) + 1.0) / 16777216.0


def philox_u(seed, sid, r, tag, slot, c0, word):
    """One uniform: counter (c0, tag<<24|slot, r, sid), output word `word` (R5)."""
    k0, k1 = seed_key(seed)
    out = philox4x32_10((c0, (tag << 24) | slot, r, sid), (k0, k1))
    return u_from_word(out[word])


def race_uniforms(seed, sid, r, tag, slot, V):
    """Uniforms u_v, v = 0..V-1, for one race: word v & 3 of block c0 = v >> 2 (R17)."""
    k0, k1 = seed_key(seed)
    nblk = (V + 3) // 4
    blk = np.arange(nblk, dtype=np.uint64)
    w = philox4x32_10_np(blk, (tag << 24) | slot, r, sid, k0, k1)
    words = np.stack(w, axis=1).reshape(-1)[:V]
    return u_from_word_np(words)
