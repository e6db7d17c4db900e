// vocab_common.cuh -- device building blocks of the vocabulary kernels (K4 chain and tree
// verification, K1 samplers): an 8-CTA cluster holds one vocabulary row per CTA slice; slice
// statistics and race winners meet through distributed shared memory.  Every decision is taken in
// fp64 after the exact fp32 front end (R13, R21), as the oracle takes it.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace seed {
namespace vocab {
namespace {   // internal linkage: included by vocab.cu and tree.cu

constexpr int CS = 8;         // CTAs per cluster (portable maximum): CTA r holds vocabulary slice r
constexpr int VT = 256;       // threads per CTA

struct MaxI {   // fp32 maximum and its first index (-1: empty)
  float m;
  int i;
};
__device__ __forceinline__ MaxI maxi_merge(MaxI A, MaxI B) {
  if (B.i < 0) return A;
  if (A.i < 0) return B;
  return (B.m > A.m || (B.m == A.m && B.i < A.i)) ? B : A;
}

struct Best {  // race winner
  double k;
  int v;
};
__device__ __forceinline__ Best best_merge(Best A, Best B) {
  if (B.v < 0) return A;
  if (A.v < 0) return B;
  return (B.k > A.k || (B.k == A.k && B.v < A.v)) ? B : A;
}

// a CTA's partial log-softmax statistic of one row slice, exchanged through distributed shared memory
struct SliceStat {
  double S;    // sum over the slice minus its own argmax of exp(a_v - m) (fp32 terms, fp64 sum)
  float m;     // slice maximum of a
  int i;       // its first index (-1: empty slice)
};

// block-wide deterministic reductions (warp butterflies, then warps in order)
__device__ MaxI block_maxi(MaxI s, MaxI* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    s = maxi_merge(s, MaxI{__shfl_xor_sync(0xffffffffu, s.m, o), __shfl_xor_sync(0xffffffffu, s.i, o)});
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = s;
  __syncthreads();
  MaxI r = red[0];
#pragma unroll
  for (int i = 1; i < VT / 32; ++i) r = maxi_merge(r, red[i]);
  return r;
}
__device__ double block_sum(double s, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = s;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int i = 1; i < VT / 32; ++i) r += red[i];
  return r;
}
__device__ float block_maxf(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int i = 1; i < VT / 32; ++i) r = fmaxf(r, red[i]);
  return r;
}
__device__ Best block_best(Best b, Best* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    b = best_merge(b, Best{__shfl_xor_sync(0xffffffffu, b.k, o), __shfl_xor_sync(0xffffffffu, b.v, o)});
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = b;
  __syncthreads();
  Best r = red[0];
#pragma unroll
  for (int i = 1; i < VT / 32; ++i) r = best_merge(r, red[i]);
  return r;
}

// a = fl32(z / T) (R4); z / 1 is z exactly
__device__ __forceinline__ float scaled_v(float z, float T) { return T == 1.0f ? z : __fdiv_rn(z, T); }

// -log(E), E = -log1p(-u): the exponential-race offset, fp64
__device__ __forceinline__ double neg_log_exp(double u) { return -log(-log1p(-u)); }

// -log(E) for the fp32 screen: absolute error < 1e-4, far inside RACE_MARGIN / 2 (the rescoring is
// exact): the candidate set of pass B holds every id whose exact key can be the maximum.  The
// logarithms run on the SFU.
__device__ __forceinline__ float neg_log_exp_screen(float u) {
  // u < 2^-7: E = u (1 + u/2 + u^2/3 + u^3/4), truncation < 1e-9 relative; else 1 - u is exact
  // (the uniform grid, R2) and __logf's absolute error (< 4e-7 on [0.5, 1)) is < 5e-5 of E >= 2^-7
  const float E = u < 0.0078125f ? u * (1.0f + u * (0.5f + u * (0.33333334f + u * 0.25f))) : -__logf(1.0f - u);
  return -__logf(E);
}

// Stage rows of this CTA's vocabulary slice into shared memory: one bulk TMA copy per row
// when the slice is 16-byte aligned, coalesced loads otherwise.  All threads call it.
struct Stager {
  float* buf;       // [nbuf][slice]
  uint64_t* bar;
  uint32_t phase;
  int slice, v0, n; // n = valid elements of this CTA's slice
  bool bulk;
  template <class RowPtr>
  __device__ void stage(int first, int k, RowPtr rowptr) {
    if (n <= 0) {
      __syncthreads();
      return;
    }
    if (bulk) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, (uint32_t)(k * n * 4));
        for (int i = 0; i < k; ++i) bulk_g2s(buf + (size_t)i * slice, rowptr(first + i) + v0, (uint32_t)(n * 4), bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
    } else {
      for (int i = 0; i < k; ++i) {
        const float* src = rowptr(first + i) + v0;
        for (int l = threadIdx.x; l < n; l += VT) buf[(size_t)i * slice + l] = __ldg(src + l);
      }
      __syncthreads();
    }
  }
};

// This CTA's slice statistic of the staged row zs: fp32 maximum and first argmax, then
// S'_c = sum over the slice minus the argmax of exp(a_v - m_c), fp32 terms summed in fp64 in a
// fixed thread / warp order (R13, R21).
__device__ SliceStat slice_stat(const float* zs, int v0, int n, float T, MaxI* red_m, double* red_d) {
  MaxI mi{-INFINITY, -1};
  for (int l = threadIdx.x; l < n; l += VT) {
    const float xf = scaled_v(zs[l], T);
    if (mi.i < 0 || xf > mi.m) mi = MaxI{xf, v0 + l};
  }
  mi = block_maxi(mi, red_m);
  // a thread's ~16 terms (each <= 1) summed in fp32 (relative error < 16 ulp, far below the expf
  // terms' own), the 256 partial sums in fp64 in a fixed order
  float s32 = 0.f;
  if (mi.i >= 0)
    for (int l = threadIdx.x; l < n; l += VT) {
      const float t = expf(scaled_v(zs[l], T) - mi.m);
      s32 += v0 + l != mi.i ? t : 0.f;
    }
  const double S = block_sum((double)s32, red_d);
  return SliceStat{S, mi.m, mi.i};
}

// The row's statistic from the CS slice statistics (rank order): m = max, i* = its first index,
// S' = sum_c S'_c e^{m_c - m} + sum_{c != c*} e^{m_c - m}  -- every slice's own maximum re-enters
// except the global argmax (the tail-excluded log-sum-exp of R13, merged in fp64).
struct RowStat {
  double m, l1p;   // m and log1p(S')
};
__device__ RowStat merge_stats(const SliceStat* st) {
  int cs = -1;
  for (int c = 0; c < CS; ++c) {
    if (st[c].i < 0) continue;
    if (cs < 0 || st[c].m > st[cs].m || (st[c].m == st[cs].m && st[c].i < st[cs].i)) cs = c;
  }
  const double m = st[cs].m;
  double S = 0.0;
  for (int c = 0; c < CS; ++c) {
    if (st[c].i < 0) continue;
    const double f = c == cs ? 1.0 : exp((double)st[c].m - m);
    S += st[c].S * f;
    if (c != cs) S += f;
  }
  return RowStat{m, log1p(S)};
}

// Exponential race over this CTA's slice, decided exactly as in fp64 (R21).  Pass A scores every id
// in fp32 (w32 returns NAN where fp32 is not accurate enough: those are scored in fp64); pass B
// rescores in fp64 every id within RACE_MARGIN of the SLICE's best fp32 key and keeps the exact
// slice argmax.  The global exact argmax is within the margin of its own slice's best (the slice
// best is at most the global best), so the maximum of the CS slice results is the exact argmax --
// one exchange, ties to the smallest id (R14).
constexpr float RACE_MARGIN = 1e-3f;

constexpr int RACE_NB = 4;   // register-resident screen keys: 4 blocks of 4 ids per thread (n <= 4096)

// the fp32 screen offsets -log(E) of a thread's ids on the register-resident path: they depend on
// the Philox counters only, so a sampler computes them before its PDL wait, while its predecessor
// (the LM head) still runs
struct ScreenPre {
  float s[RACE_NB][4];
};
__device__ __forceinline__ void screen_precompute(int v0, int n, uint32_t c1, uint32_t r, uint32_t sid, uint32_t k0,
                                                  uint32_t k1, ScreenPre& p) {
#pragma unroll
  for (int i = 0; i < RACE_NB; ++i) {
    const int l = 4 * (int)threadIdx.x + i * 4 * VT;
#pragma unroll
    for (int e = 0; e < 4; ++e) p.s[i][e] = 0.f;
    if (l < n) {
      const Philox4 ph = philox4x32_10((uint32_t)((v0 + l) >> 2), c1, r, sid, k0, k1);
      const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) p.s[i][e] = neg_log_exp_screen((float)philox_uniform(words[e]));
    }
  }
}

template <class W32, class W64>
__device__ Best race_slice(int v0, int n, uint32_t c1, uint32_t r, uint32_t sid, uint32_t k0, uint32_t k1, float* keys,
                           float* red_f, Best* red_b, W32 w32, W64 w64, const ScreenPre* pre = nullptr) {
  Best b{-INFINITY, -1};
  auto rescore = [&](int l) {   // pass B: the exact fp64 key of id v0 + l
    const int g = v0 + l;
    const Philox4 ph = philox4x32_10((uint32_t)(g >> 2), c1, r, sid, k0, k1);
    const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
    const double wd = w64(l);
    if (!(wd > -INFINITY)) return;   // -inf, or NaN (non-finite logits: no finite key, R35)
    const double key = wd + neg_log_exp(philox_uniform(words[g & 3]));
    if (b.v < 0 || key > b.k || (key == b.k && g < b.v)) b = Best{key, g};
  };
  // pass A: fp32 screen keys; an id whose weight fp32 cannot screen (w32 = NaN) is a candidate by
  // construction (+inf) and is scored in pass B only.  The threshold is taken over screened keys:
  // the exact argmax is screened within RACE_MARGIN / 2 of its key, or is an fp64 candidate.
  auto screen = [&](int l, uint32_t word) -> float {
    const float w = w32(l);
    if (w != w) return INFINITY;
    return w != -INFINITY ? w + neg_log_exp_screen((float)philox_uniform(word)) : -INFINITY;
  };
  float best32 = -INFINITY;
  if (n <= 4 * VT * RACE_NB) {
    // the 16 screen keys of a thread stay in registers; pass B walks a candidate bit mask (one
    // out-of-loop copy of the fp64 rescoring code)
    float kr[RACE_NB][4];
#pragma unroll
    for (int i = 0; i < RACE_NB; ++i) {
      const int l = 4 * (int)threadIdx.x + i * 4 * VT;
#pragma unroll
      for (int e = 0; e < 4; ++e) kr[i][e] = -INFINITY;
      if (l < n) {
        if (pre) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (l + e < n) {
              const float w = w32(l + e);
              kr[i][e] = w != w ? INFINITY : (w != -INFINITY ? w + pre->s[i][e] : -INFINITY);
            }
        } else {
          const Philox4 ph = philox4x32_10((uint32_t)((v0 + l) >> 2), c1, r, sid, k0, k1);
          const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (l + e < n) kr[i][e] = screen(l + e, words[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (kr[i][e] != INFINITY) best32 = fmaxf(best32, kr[i][e]);
    }
    const float lmax = block_maxf(best32, red_f);
    const float thr = lmax - RACE_MARGIN;
    uint32_t mask = 0;
#pragma unroll
    for (int i = 0; i < RACE_NB; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (kr[i][e] == INFINITY || (kr[i][e] != -INFINITY && kr[i][e] >= thr)) mask |= 1u << (4 * i + e);
    while (mask) {
      const int bit = __ffs(mask) - 1;
      mask &= mask - 1;
      rescore(4 * (int)threadIdx.x + (bit >> 2) * 4 * VT + (bit & 3));
    }
    return block_best(b, red_b);
  }
  // large slices: screen keys through shared memory
  for (int l = 4 * (int)threadIdx.x; l < n; l += 4 * VT) {
    const Philox4 ph = philox4x32_10((uint32_t)((v0 + l) >> 2), c1, r, sid, k0, k1);
    const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (l + e >= n) break;
      const float key = screen(l + e, words[e]);
      keys[l + e] = key;
      if (key != INFINITY) best32 = fmaxf(best32, key);
    }
  }
  const float lmax = block_maxf(best32, red_f);
  const float thr = lmax - RACE_MARGIN;
  for (int l = threadIdx.x; l < n; l += VT)
    if (keys[l] == INFINITY || (keys[l] != -INFINITY && keys[l] >= thr)) rescore(l);
  return block_best(b, red_b);
}


// push `bytes` (multiple of 4) of this CTA's value into the same shared address of every rank
SEED_DEV void push_all(const void* src, void* dst_local, int bytes) {
  for (int c = 0; c < CS; ++c) {
    const uint32_t dst = dsmem_addr(dst_local, (uint32_t)c);
    for (int o = 0; o < bytes; o += 4)
      asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(dst + o), "r"(*reinterpret_cast<const uint32_t*>(
                       reinterpret_cast<const char*>(src) + o))
                   : "memory");
  }
}

}  // namespace
}  // namespace vocab
}  // namespace seed
