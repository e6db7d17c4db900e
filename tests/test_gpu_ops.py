"""GPU parity of the single kernels against the oracle, through the C ABI.

Inputs come from seedgen (and, for drafted ids, from the oracle); nothing flows from the
CUDA path into the oracle.  Tolerances: decisions bit-exact except oracle-flagged near-ties
(|u - rho| < 1e-6, race top-2 gap < 1e-6), flagged < 1e-5 of decisions; probabilities within
1e-5 abs (north_star); GEMM within fp32-accumulation error of the fp64 product.
"""
import os

import numpy as np
import pytest
import torch

import seedgen
from oracle import philox as ph
from oracle import sampling as sp

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")
SEED = seedgen.PHILOX_SEED


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_18200_b200 import ops as o
    return o


def test_philox_kat_and_oracle(ops):
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        got = ops.philox(w[0], w[1], w[2], w[3], w[4], w[5], 1)[0].tolist()
        assert got == w[6:10]
    k0, k1 = ph.seed_key(SEED)
    got = ops.philox(5, (3 << 24) | 2, 7, 123456, k0, k1, 4096)
    ref = np.stack(ph.philox4x32_10_np(np.arange(5, 5 + 4096, dtype=np.uint64), (3 << 24) | 2, 7, 123456, k0, k1),
                   axis=1).astype(np.int64)
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("N,K,M", [(128, 64, 1), (192, 128, 15), (32, 128, 3), (300, 256, 37), (4096, 4096, 15),
                                   (12288, 4096, 120), (4096, 11008, 5), (2304, 768, 48), (1000, 512, 256),
                                   (640, 1024, 300), (32000, 768, 3), (5120, 5120, 72), (5120, 13824, 15),
                                   (4096, 4096, 600), (12288, 4096, 960), (22016, 4096, 513)])
def test_gemm_vs_fp64(ops, N, K, M):
    W = seedgen.bf16_matrix(N, K, seed=N * 7 + K).cuda()
    X = seedgen.bf16_matrix(M, K, seed=M * 13 + K + 1).cuda()
    Y = ops.gemm(W, X).double().cpu()
    ref = X.double().cpu() @ W.double().cpu().T
    # fp32 accumulation of K bf16 products: |err| <= ~K * 2^-24 * sum|x w|; use a relative bound
    scale = (X.double().abs().cpu() @ W.double().abs().cpu().T)
    err = ((Y - ref).abs() / scale.clamp_min(1e-30)).max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("N,K", [(4096, 4096), (4096, 11008), (12288, 4096), (768, 3072), (5120, 13824)])
def test_gemm_batch_invariance(ops, N, K):
    """R19: a row's result does not depend on how many other rows share the launch (the cluster
    split-K reduction order is a function of (N, K) only); repeated launches are bit-identical."""
    W = seedgen.bf16_matrix(N, K, seed=1).cuda()
    X = seedgen.bf16_matrix(120, K, seed=2).cuda()
    Y120 = ops.gemm(W, X)
    assert torch.equal(Y120, ops.gemm(W, X))
    for m in (15, 16, 64):
        assert torch.equal(Y120[:m], ops.gemm(W, X[:m].contiguous())), m
    assert torch.equal(Y120[7:8], ops.gemm(W, X[7:8].contiguous()))
    # several 256-row token tiles: every row reduced in the same order as alone
    X960 = seedgen.bf16_matrix(960, K, seed=3).cuda()
    X960[:120] = X
    Y960 = ops.gemm(W, X960)
    assert torch.equal(Y960[:120], Y120)
    assert torch.equal(Y960[700:701], ops.gemm(W, X960[700:701].contiguous()))


def _oracle_xs(zd, T, sids, rs):
    B, g, V = zd.shape
    xs = np.zeros((B, g), dtype=np.int32)
    for b in range(B):
        for j in range(g):
            xs[b, j] = sp.draft_token(zd[b, j], T, SEED, int(sids[b]), int(rs[b]), j + 1)[0]
    return xs


SETTINGS = [(1.0, 0.3, 1.0), (1.0, 0.1, 1.0), (1.0, 0.02, 1.0), (3.0, 1.0, 0.2), (5.0, 0.5, 0.2)]


@pytest.mark.parametrize("V,gamma,B", [(32, 4, 3000), (32, 1, 1000), (32, 6, 1000), (32000, 4, 96), (32000, 5, 24),
                                       (32000, 6, 5), (32000, 4, 192), (32000, 1, 3)])
def test_verify_vs_oracle(ops, V, gamma, B):
    """P1: accepted lengths and token ids bit-exact except oracle-flagged near-ties."""
    total = mism = flagged = 0
    for si, (sigma, noise, T) in enumerate(SETTINGS):
        zt, zd = seedgen.synthetic_logits(B, gamma, V, sigma, noise, seed=1000 * si + V + gamma)
        sids = np.arange(B, dtype=np.int64) * 7919 + si
        rs = (np.arange(B) % 5).astype(np.int32)
        xs = _oracle_xs(zd, T, sids, rs)
        for bonus in (True, False):
            out = ops.verify(torch.from_numpy(zt).cuda(), torch.from_numpy(zd).cuda(), torch.from_numpy(xs).cuda(),
                             T, SEED, sids, rs, bonus=bonus)
            tok, cnt, a_gpu = out["out_tok"].cpu().numpy(), out["out_cnt"].cpu().numpy(), out["a"].cpu().numpy()
            dbg = out["dbg"].cpu().numpy()
            for b in range(B):
                r = sp.verify_stream(zt[b], zd[b], xs[b].tolist(), T, SEED, int(sids[b]), int(rs[b]), bonus=bonus)
                total += 1
                same = (r.a == a_gpu[b]) and (len(r.emitted) == cnt[b]) and list(tok[b, :cnt[b]]) == r.emitted
                if r.flags:
                    flagged += 1
                elif not same:
                    mism += 1
                # probabilities within 1e-5 abs for the consumed positions
                for j in range(min(r.a + 1, gamma)):
                    x = xs[b, j]
                    lp = sp.logsoftmax_tail(sp.scaled_logits(zt[b, j], T))[x]
                    lq = sp.logsoftmax_tail(sp.scaled_logits(zd[b, j], T))[x]
                    assert abs(np.exp(dbg[b, j, 0]) - np.exp(lp)) < 1e-5
                    assert abs(np.exp(dbg[b, j, 1]) - np.exp(lq)) < 1e-5
                    assert abs(dbg[b, j, 3] - sp.accept_prob(lp, lq)) < 1e-5
    assert mism == 0, f"{mism} unflagged mismatches of {total}"
    assert flagged <= max(1, 1e-5 * total * (gamma + 1)), flagged


def test_q_equals_p_gpu(ops):
    """P3: draft logits := target logits -> a = gamma, n_emit = gamma + 1."""
    B, g, V = 64, 4, 32000
    zt, _ = seedgen.synthetic_logits(B, g, V, 1.0, 0.0, seed=5)
    zd = zt[:, :g].copy()
    xs = np.random.default_rng(0).integers(0, V, size=(B, g)).astype(np.int32)
    for T in (1.0, 0.2):
        out = ops.verify(torch.from_numpy(zt).cuda(), torch.from_numpy(zd).cuda(), torch.from_numpy(xs).cuda(), T,
                         SEED, np.arange(B), np.zeros(B, np.int32))
        assert (out["a"].cpu().numpy() == g).all()
        assert (out["out_cnt"].cpu().numpy() == g + 1).all()


def test_draft_sample_vs_oracle(ops):
    rng = np.random.default_rng(3)
    for V, B, T in ((32, 500, 1.0), (32000, 64, 1.0), (32000, 64, 0.2)):
        z = (rng.standard_normal((B, V)) * 2).astype(np.float32)
        sids = rng.integers(0, 2**31, size=B)
        rs = rng.integers(0, 50, size=B).astype(np.int32)
        got = ops.draft_sample(torch.from_numpy(z).cuda(), T, SEED, sids, rs, 3).cpu().numpy()
        for b in range(B):
            tok, gap = sp.draft_token(z[b], T, SEED, int(sids[b]), int(rs[b]), 3)
            if gap >= 1e-6:
                assert got[b] == tok


def test_gpu_round_chi2(ops):
    """P2: 1e6 GPU rounds (draft sampler + K4) on fixed (p, q): first emitted token ~ p_1
    (df 31) and the first two ~ p_1 x p_2 (df 1023), chi-square at alpha = 0.01."""
    from scipy import stats
    rng = np.random.default_rng(11)
    g, V, n = 4, 32, 1_000_000
    zt1 = rng.standard_normal((g + 1, V)).astype(np.float32)
    zd1 = (zt1[:g] + rng.standard_normal((g, V)) * 0.6).astype(np.float32)
    T = 1.0
    sids = np.arange(n, dtype=np.int64)
    rs = np.zeros(n, dtype=np.int32)
    zd_dev = torch.from_numpy(np.broadcast_to(zd1, (n, g, V)).copy()).cuda()
    xs = torch.empty((n, g), dtype=torch.int32, device="cuda")
    for j in range(g):
        xs[:, j] = ops.draft_sample(zd_dev[:, j].contiguous(), T, SEED, sids, rs, j + 1)
    zt_dev = torch.from_numpy(np.broadcast_to(zt1, (n, g + 1, V)).copy()).cuda()
    out = ops.verify(zt_dev, zd_dev, xs, T, SEED, sids, rs, want_dbg=False)
    tok = out["out_tok"].cpu().numpy()
    p1 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt1[0], T)))
    p2 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt1[1], T)))
    c1 = np.bincount(tok[:, 0], minlength=V).astype(float)
    chi1 = np.sum((c1 - n * p1) ** 2 / (n * p1))
    assert chi1 < stats.chi2.ppf(0.99, V - 1), chi1
    # rounds emitting >= 2 tokens accepted x_1: then t_1 ~ min(p_1, q_1) / alpha_1 and t_2 ~ p_2
    # independently (the rows here do not depend on the prefix)
    q1 = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zd1[0], T)))
    two = out["out_cnt"].cpu().numpy() >= 2
    m = int(two.sum())
    joint = np.bincount(tok[two, 0] * V + tok[two, 1], minlength=V * V).astype(float)
    acc = np.minimum(p1, q1)
    pj = np.outer(acc / acc.sum(), p2).reshape(-1)
    keep = m * pj > 5
    exp_ = m * pj[keep] / pj[keep].sum() * (joint[keep].sum() / m)
    chi2 = np.sum((joint[keep] - exp_) ** 2 / exp_)
    assert chi2 < stats.chi2.ppf(0.99, int(keep.sum()) - 1), chi2


def test_verify_empty_residual_gpu(ops):
    """R3 edge case through rounding (see tests/test_oracle_sampling.py::test_empty_residual_fallback):
    the residual max(0, p - q) is empty in fp64, so K4 falls back to the bonus rule on the same row
    with the same uniforms -- the same token as the oracle's fallback, for every stream."""
    V, g, T = 32000, 1, 1.0
    rng = np.random.default_rng(12)
    zd = rng.standard_normal((g, V)).astype(np.float32)
    x = int(np.argmin(zd[0]))
    zd[0, x] = np.float32(zd[0].max() - 60.0)
    zt = np.zeros((g + 1, V), dtype=np.float32)
    zt[:g] = zd
    zt[0, x] = zd[0, x] - np.float32(5.0)
    zt[g] = rng.standard_normal(V).astype(np.float32)
    B = 64
    ZT = np.broadcast_to(zt, (B, g + 1, V)).copy()
    ZD = np.broadcast_to(zd, (B, g, V)).copy()
    xs = np.full((B, g), x, dtype=np.int32)
    sids = np.arange(B, dtype=np.int64) + 1000
    rs = np.zeros(B, dtype=np.int32)
    out = ops.verify(torch.from_numpy(ZT).cuda(), torch.from_numpy(ZD).cuda(), torch.from_numpy(xs).cuda(), T, SEED,
                     sids, rs)
    tok, cnt, a = out["out_tok"].cpu().numpy(), out["out_cnt"].cpu().numpy(), out["a"].cpu().numpy()
    fallbacks = 0
    for b in range(B):
        r = sp.verify_stream(ZT[b], ZD[b], [x], T, SEED, int(sids[b]), 0)
        assert a[b] == r.a and list(tok[b, :cnt[b]]) == r.emitted, b
        fallbacks += r.fallback
    assert fallbacks > B // 2


def test_gpu_bonus_chi2(ops):
    """R1 on the GPU: over 1e6 K4 launches' streams with q close to p, the bonus tokens of the
    all-accepted rounds follow p_{gamma+1} (chi-square at alpha = 0.01, df 31)."""
    from scipy import stats
    rng = np.random.default_rng(21)
    g, V, n, T = 4, 32, 1_000_000, 1.0
    zt1 = rng.standard_normal((g + 1, V)).astype(np.float32)
    zd1 = (zt1[:g] + rng.standard_normal((g, V)) * 0.15).astype(np.float32)
    sids = np.arange(n, dtype=np.int64)
    rs = np.full(n, 3, dtype=np.int32)
    zd_dev = torch.from_numpy(np.broadcast_to(zd1, (n, g, V)).copy()).cuda()
    xs = torch.empty((n, g), dtype=torch.int32, device="cuda")
    for j in range(g):
        xs[:, j] = ops.draft_sample(zd_dev[:, j].contiguous(), T, SEED, sids, rs, j + 1)
    zt_dev = torch.from_numpy(np.broadcast_to(zt1, (n, g + 1, V)).copy()).cuda()
    out = ops.verify(zt_dev, zd_dev, xs, T, SEED, sids, rs, want_dbg=False)
    a = out["a"].cpu().numpy()
    tok = out["out_tok"].cpu().numpy()
    full = a == g
    assert full.sum() > 50_000
    pb = np.exp(sp.logsoftmax_tail(sp.scaled_logits(zt1[g], T)))
    c = np.bincount(tok[full, g], minlength=V).astype(float)
    m = c.sum()
    chi = np.sum((c - m * pb) ** 2 / (m * pb))
    assert chi < stats.chi2.ppf(0.99, V - 1), chi


def test_near_tie_rate_gpu(ops):
    """north_star: decisions the kernel and the oracle may legitimately take differently (|u - rho| <
    1e-6, R16) must stay below 1e-5 of all decisions -- counted here on 1M accept decisions at
    V = 32000 from the kernel's own (u, rho) (the oracle agrees with every other decision, P1)."""
    B, g, V = 2048, 4, 32000
    total = near = 0
    gen = torch.Generator(device="cuda").manual_seed(11)
    for it in range(128):
        sigma, noise, T = ((1.0, 0.3, 1.0), (3.0, 1.0, 0.2))[it % 2]
        zt = torch.randn((B, g + 1, V), device="cuda", generator=gen) * sigma
        zd = (zt[:, :g] + torch.randn((B, g, V), device="cuda", generator=gen) * noise).contiguous()
        xs = torch.randint(0, V, (B, g), device="cuda", dtype=torch.int32, generator=gen)
        sids = np.arange(B, dtype=np.int64) * 104729 + it
        rs = (np.arange(B) % 7).astype(np.int32)
        dbg = ops.verify(zt, zd, xs, T, SEED, sids, rs)["dbg"]
        near += int((dbg[..., 2] - dbg[..., 3]).abs().lt(1e-6).sum().item())
        total += B * g
    assert total >= 1_000_000
    assert near <= 1e-5 * total, (near, total)
