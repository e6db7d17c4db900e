// gemm.cu -- K2: every projection of both models (and the LM heads) on tcgen05.
//
// Y[m][n] = sum_k X[m][k] * W[n][k]  (nn.Linear, W row-major [N][K], bf16 in, fp32 accumulate).
// The method streams every weight once per round with only M = B(gamma+1) tokens
// (M <= 120 sits far below the ridge), so the kernel is built to keep
// HBM busy: swap-AB puts the weight rows on the UMMA M = 128 side and the tokens on
// UMMA N = M_pad (16..256); TMA streams 128 x 64 weight tiles through a deep smem ring
// (evict-first), the token tile rides along (evict-last, L2 resident); one elected
// thread issues tcgen05.mma into a TMEM accumulator; four epilogue warps drain TMEM
// with tcgen05.ld and apply the fused epilogue (store / residual + RMSNorm operand / SwiGLU).
//
// Work split (cluster split-K, below): c CTAs per 128-row weight tile, c a function of (N, K)
// only, never of M, so every output element is reduced in the same order whatever the batch
// (batch invariance, DESIGN R19).
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace seed {

namespace {
constexpr int BLOCK_N = 128;   // weight rows per tile (UMMA M)
constexpr int BLOCK_K = 64;    // one 128-byte swizzle row of bf16
constexpr int W_TILE_BYTES = BLOCK_N * BLOCK_K * 2;
constexpr int MAX_STAGES = 16;
constexpr int TOKEN_TILE = 256;   // rows per CTA (UMMA N <= 256); more rows -> several token tiles

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // K-major operand, 128B swizzle: 8-row x 128B atoms, SBO = 1024 B, LBO unused, version 1
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ============================================================================================
// K2, cluster split-K form (the default): one thread-block cluster of c CTAs per 128-row weight
// tile.  CTA rank r streams k-blocks [r KB / c, (r + 1) KB / c) of the tile into its TMEM
// accumulator; the c partials meet in distributed shared memory, where CTA r sums them in rank
// order 0 .. c-1 -- c is a function of (N, K) only, so every output element is reduced in the same
// order whatever the batch (R19) -- and finishes the tile's tokens [r per, (r + 1) per).  c = 1:
// whole tiles straight from TMEM.  Compared with the stream-K form this replaces the tail (one
// reducer CTA per tile reading every partial back from L2, then the whole tile's epilogue) by a
// c-way parallel reduction and epilogue that never leaves the cluster.
struct SplitArgs {
  int KB, c, per, M, m_pad, stages, N, K, ldY, ymode, ssq_in_ld, pc, pitch;
  int Mtot;                    // rows of the whole launch; a CTA's token tile holds rows [row0, row0 + M)
  float eps;
  float* Y;
  const float* ssq_in;
  const int32_t* yrow;
  float* ssq_out;
  const __nv_bfloat16* nw;
  __nv_bfloat16* hout;
  unsigned long long* timing;
  unsigned long long* cta;
  int keep_w;                  // weights evict-last (small models re-read every draft step stay in L2)
  int tstore;                  // c = 1, ymode 0 without a row map or ymode 2: the whole tile is staged in the
                               // idle ring and leaves by one tensor store (tmY)
};

// rows m0 .. m0 + 15 below mlim of tile column nl (weight row n = 128 t + nl), v = the reduced
// accumulator.  The finished rows are staged in shared memory (`stg`, one of two 12 KB buffers
// used alternately, so one barrier per chunk suffices) and leave as coalesced 16-byte stores, a
// warp per 512-byte row segment.  ymode 0: store (x 1/rms, row map); 1: residual add, x^2 row
// sums per warp, bf16 operand of the next RMSNorm; 2: SwiGLU -- gate (nl < 64) and up (nl >= 64)
// meet in shared memory and all 128 threads form 8 rows each of silu(g) * u               (B4)
__host__ __device__ __forceinline__ int c_dump_bytes(const SplitArgs& a) { return a.c > 1 ? a.c * 128 * a.pitch * 4 : 0; }

SEED_DEV float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int YM>
__device__ __forceinline__ void split_finish16(const SplitArgs& a, int t, int nl, int et, int lane, int m0, int mlim,
                                               const float* v, const float* inv_s, const int* rowmap_s, float* red_s,
                                               const float* xo, float w, uint8_t* stg) {
  const int n = t * BLOCK_N + nl;
  float* sf = reinterpret_cast<float*>(stg);                       // [16][128] fp32 rows
  __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(stg + 8192); // [16][128] | [16][64] bf16 rows
  if constexpr (YM == 0) {
    float sc[16];   // every load before the first store (no load-after-store chains)
#pragma unroll
    for (int i = 0; i < 16; ++i) sc[i] = a.ssq_in ? inv_s[min(m0 + i, 255)] : 1.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) sf[i * 128 + nl] = a.ssq_in ? v[i] * sc[i] : v[i];
  } else if constexpr (YM == 1) {
    float sq[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float xn = xo[i] + v[i];
      sf[i * 128 + nl] = xn;
      sh[i * 128 + nl] = f2bf(xn * w);
      sq[i] = (m0 + i < mlim && n < a.N) ? xn * xn : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) sq[i] = warp_sum(sq[i]);
    if (lane == 0) {
      const int ew = et >> 5;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (m0 + i < mlim) red_s[ew * 256 + m0 + i] = sq[i];
    }
  } else {
    float* xch = red_s;   // [16][128]
    float sc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) sc[i] = inv_s[min(m0 + i, 255)];
#pragma unroll
    for (int i = 0; i < 16; ++i) xch[i * 128 + nl] = v[i] * sc[i];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int j = et & 63, i0 = (et >> 6) * 8;
    float g[8], u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      g[q] = xch[(i0 + q) * 128 + j];
      u[q] = xch[(i0 + q) * 128 + 64 + j];
    }
    // silu(g) u = g u / (1 + e^-g) on the SFU (ex2 / rcp approx; the product is rounded to bf16, B4)
    __nv_bfloat16 hb[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) hb[q] = f2bf(g[q] * rcp_approx(1.0f + __expf(-g[q])) * u[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) sh[(i0 + q) * 64 + j] = hb[q];
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  {
    const int ncols = min(BLOCK_N, a.N - t * BLOCK_N);
    if (YM != 2) {
      // fp32 rows: 16 x 32 float4, a warp per row
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = et + 128 * k, i = q >> 5, c4 = (q & 31) * 4, m = m0 + i;
        if (m < mlim && c4 < ncols) {
          const int row = YM == 0 && a.yrow ? rowmap_s[m] : m;
          if (row >= 0)
            *reinterpret_cast<float4*>(a.Y + (size_t)row * a.ldY + t * BLOCK_N + c4) =
                *reinterpret_cast<const float4*>(sf + i * 128 + c4);
        }
      }
    }
    if (YM == 1) {
      // bf16 rows: 16 x 16 uint4
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = et + 128 * k, i = q >> 4, c8 = (q & 15) * 8, m = m0 + i;
        if (m < mlim && c8 < ncols)
          *reinterpret_cast<uint4*>(a.hout + (size_t)m * a.N + t * BLOCK_N + c8) =
              *reinterpret_cast<const uint4*>(sh + i * 128 + c8);
      }
    } else if (YM == 2) {
      const int i = et >> 3, c8 = (et & 7) * 8, m = m0 + i;
      if (m < mlim)
        *reinterpret_cast<uint4*>(a.hout + (size_t)m * (a.N / 2) + t * 64 + c8) =
            *reinterpret_cast<const uint4*>(sh + i * 64 + c8);
    }
  }
}

// One instantiation per epilogue form (YM = ymode, SPLIT = c > 1, TST = whole-tile tensor store):
// each holds only its own epilogue, so the code a CTA runs after its mainloop stays within the SM's
// instruction cache (the all-forms kernel was ~100 KB of SASS; its epilogue fetched instructions
// from L2 behind the weight stream, ~3 us per CTA at M = 120).
template <int YM, int SPLIT, int TST>
__global__ void __launch_bounds__(192, 2)
gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmY, SplitArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the shared array (the compiler keeps the shared
  // state space: ld/st.shared instead of generic accesses)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.stages;
  const int x_bytes = a.m_pad * BLOCK_K * 2;
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * W_TILE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + S * x_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  float* inv_s = reinterpret_cast<float*>(tmem_slot + 4);   // [256] 1/rms per X row (ssq_in)
  int* rowmap_s = reinterpret_cast<int*>(inv_s + 256);      // [256] output row map (yrow)
  float* red_s = reinterpret_cast<float*>(rowmap_s + 256);  // [4][256] x^2 row sums | [16][128] gate/up
  float* part_s = reinterpret_cast<float*>(smem);           // [128][pitch] accumulator dump (aliases the ring)
  // two 12 KB output staging buffers after the dump (the ring is idle once the accumulator is ready)
  uint8_t* stg0 = smem + (c_dump_bytes(a) + 1023) / 1024 * 1024;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = SPLIT ? a.c : 1, r = blockIdx.x % c, t = blockIdx.y;
  // token tile: rows [row0, row0 + M) of the launch (blockIdx.x / c); every row's reduction order is
  // the same whatever tile it falls in (R19).  The pointers below are rebased to the tile.
  const int row0 = (blockIdx.x / c) * TOKEN_TILE;
  a.M = min(TOKEN_TILE, a.Mtot - row0);
  if (row0 > 0) {
    if (YM == 0 && a.yrow) a.yrow += row0;
    else if (a.Y) a.Y += (size_t)row0 * a.ldY;
    if (a.hout) a.hout += (size_t)row0 * (YM == 2 ? a.N / 2 : a.N);
    if (a.ssq_in) a.ssq_in += row0;
    if (a.ssq_out) a.ssq_out += row0;
  }
  const int kb0 = (int)((long)r * a.KB / c), kb1 = (int)((long)(r + 1) * a.KB / c);
  const int nk = kb1 - kb0;
  pdl_trigger();
  if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[0], globaltimer());
  unsigned long long* ct = a.cta && blockIdx.x < c ? a.cta + (size_t)(t * c + r) * 16 : nullptr;
  if (ct && threadIdx.x == 0) ct[0] = globaltimer();

  uint32_t cols = 32;
  while (cols < (uint32_t)a.m_pad) cols <<= 1;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);   // split-K exchange: the slices this rank reduces have landed
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int mcols = (a.M + 15) / 16 * 16;               // accumulator columns holding real rows
  const int npass = c > 1 ? (mcols + a.pc - 1) / a.pc : 0;

  if (warp == 0) {
    // ---------------- producer (one lane): weight + X k-blocks by TMA; the weights of the first
    // ring fill are requested before the PDL wait (they do not depend on the predecessor)
    if (lane == 0) {
      const uint64_t pol_w = a.keep_w ? l2_policy_evict_last() : l2_policy_evict_first();
      const uint64_t pol_x = l2_policy_evict_last();
      const uint32_t tx = W_TILE_BYTES + x_bytes;
      const int n_pre = min(S, nk);
      for (int i = 0; i < n_pre; ++i) {
        mbar_arrive_expect_tx(&full[i], tx);
        tma_load_2d(sW + i * W_TILE_BYTES, &tmW, &full[i], (kb0 + i) * BLOCK_K, t * BLOCK_N, pol_w);
      }
      pdl_wait();
      if (a.timing) atomicMin(&a.timing[1], globaltimer());
      if (ct) ct[1] = globaltimer();
      for (int i = 0; i < n_pre; ++i)
        tma_load_2d(sX + i * x_bytes, &tmX, &full[i], (kb0 + i) * BLOCK_K, row0, pol_x);
      int stage = n_pre % S;
      uint32_t phase = n_pre == S ? 1u : 0u;
      for (int k = n_pre; k < nk; ++k) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], tx);
        tma_load_2d(sW + stage * W_TILE_BYTES, &tmW, &full[stage], (kb0 + k) * BLOCK_K, t * BLOCK_N, pol_w);
        tma_load_2d(sX + stage * x_bytes, &tmX, &full[stage], (kb0 + k) * BLOCK_K, row0, pol_x);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (ct) ct[2] = globaltimer();
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (one elected lane)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(a.m_pad >> 3) << 17) |
                           ((uint32_t)(BLOCK_N >> 4) << 24);
    const uint32_t sW0 = smem_u32(sW), sX0 = smem_u32(sX);
    int stage = 0;
    uint32_t phase = 0;
    for (int k = 0; k < nk; ++k) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (ct && k == 0 && lane == 0) ct[3] = globaltimer();
      if (elect_one()) {
        const uint32_t wa = sW0 + stage * W_TILE_BYTES, xa = sX0 + stage * x_bytes;
#pragma unroll
        for (int kk = 0; kk < BLOCK_K / 16; ++kk)
          umma_bf16(tmem_base, sw128_desc(wa + kk * 32), sw128_desc(xa + kk * 32), idesc,
                    (k > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[stage]);
        if (k == nk - 1) umma_commit(&tfull[0]);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (ct && lane == 0) ct[4] = globaltimer();
  } else {
    // ---------------- epilogue warps 2..5: thread = weight row nl of the tile (TMEM lane)
    const int lane_grp = warp & 3;
    const int nl = lane_grp * 32 + lane;
    const int n = t * BLOCK_N + nl;
    const int et = threadIdx.x - 64;
    // rows this CTA finishes first (pass 0 for c > 1); 1/rms and the row map cover every row
    const int perp0 = c > 1 ? ((min(a.pc, mcols) / 4) + c - 1) / c * 4 : a.M;
    const int m_lo = c > 1 ? min(a.M, r * perp0) : 0;
    const int m_hi = c > 1 ? min(a.M, min(min(a.pc, mcols), (r + 1) * perp0)) : a.M;
    pdl_wait();   // ssq_in, the residual and the row map are written by predecessors
    // what does not depend on the accumulator is loaded while it is computed
    if (a.ssq_in) {
      const int kt = (a.K + 127) / 128;
      for (int m = et; m < a.M; m += 128) {
        float ss = 0.f;
        for (int i = 0; i < kt; ++i) ss += __ldcg(a.ssq_in + (size_t)i * a.ssq_in_ld + m);
        inv_s[m] = 1.0f / sqrtf(ss / (float)a.K + a.eps);
      }
    }
    if (a.yrow)
      for (int m = et; m < a.M; m += 128) rowmap_s[m] = __ldg(a.yrow + m);
    constexpr bool res = YM == 1;
    const float w = (res && n < a.N) ? bf2f(a.nw[n]) : 0.f;
    float xo[16], xn[16];
    auto load_res = [&](int m0, float* dst) {
#pragma unroll
      for (int i = 0; i < 16; ++i)   // (clamped unconditional loads measured slower: 4.92 vs 5.08 ms at N = 24)
        dst[i] = (m0 + i < a.M && n < a.N) ? a.Y[(size_t)(m0 + i) * a.ldY + n] : 0.f;
    };
    // the first two chunks' residual rows (c > 1: the rest stays one chunk ahead in the loop)
    if (res) load_res(m_lo, xo);
    if (res && c > 1 && m_lo + 16 < m_hi) load_res(m_lo + 16, xn);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    if (ct && et == 0) ct[5] = globaltimer();
    const uint32_t row_addr = tmem_base + ((uint32_t)(lane_grp * 32) << 16);
    int chunk = 0;
    if constexpr (TST != 0) {
      // whole tile: every accumulator column straight into a staging tile in the idle ring (32 columns
      // per TMEM load), one barrier, one tensor store -- no per-chunk barrier or store round trip
      float* sf = reinterpret_cast<float*>(smem);   // ymode 0: fp32 [m_pad][128]; ymode 2: fp32 [m_pad][128] gate | up
      // Branch-free: 32 columns per TMEM load (the allocation holds max(32, m_pad) rounded to a power
      // of two), every row of the 32-row group stored (rows past m_pad land in the idle ring and are
      // never stored out), rows >= M scaled by 1 (a per-element branch here cost ~3x the stores)
      const bool scaled = a.ssq_in != nullptr;
      for (int m0 = 0; m0 < mcols; m0 += 32) {
        float v[32];
        tmem_ld32(row_addr + m0, v);
        float sc[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 s4 = make_float4(1.f, 1.f, 1.f, 1.f);
          if (scaled) s4 = *reinterpret_cast<const float4*>(inv_s + m0 + 4 * q);
          sc[4 * q] = m0 + 4 * q < a.M ? s4.x : 1.f;
          sc[4 * q + 1] = m0 + 4 * q + 1 < a.M ? s4.y : 1.f;
          sc[4 * q + 2] = m0 + 4 * q + 2 < a.M ? s4.z : 1.f;
          sc[4 * q + 3] = m0 + 4 * q + 3 < a.M ? s4.w : 1.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) sf[(m0 + i) * 128 + nl] = v[i] * sc[i];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (ct && et == 0) ct[8] = globaltimer();   // staged
      if constexpr (YM == 2) {
        // SwiGLU: output j (0..63) of row m from gate column j and up column 64 + j (B4)
        __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(smem + (size_t)a.m_pad * 128 * 4);   // bf16 [m_pad][64]
        const int j = et & 63;
        for (int m = et >> 6; m < mcols; m += 2) {
          const float g = sf[m * 128 + j], u = sf[m * 128 + 64 + j];
          sh[m * 64 + j] = f2bf(g * rcp_approx(1.0f + __expf(-g)) * u);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          fence_proxy_async();
          tma_store_2d(&tmY, sh, t * 64, row0);
          bulk_commit();
          bulk_wait_read0();
        }
      } else if (et == 0) {
        fence_proxy_async();
        tma_store_2d(&tmY, sf, t * BLOCK_N, row0);
        bulk_commit();
        bulk_wait_read0();
      }
      if (ct && et == 0) ct[11] = globaltimer();
    } else if constexpr (!SPLIT) {
      for (int m0 = 0; m0 < a.M; m0 += 16) {
        float v[16];
        tmem_ld16(row_addr + m0, v);
        if (res && m0 + 16 < a.M) load_res(m0 + 16, xn);
        split_finish16<YM>(a, t, nl, et, lane, m0, min(m0 + 16, a.M), v, inv_s, rowmap_s, red_s, xo, w,
                       stg0 + (chunk++ & 1) * 12288);
        if (ct && et == 0 && m0 == 0) ct[11] = globaltimer();
        if (res) {
#pragma unroll
          for (int i = 0; i < 16; ++i) xo[i] = xn[i];
        }
      }
    } else {
      for (int pass = 0; pass < npass; ++pass) {
        const int pb = pass * a.pc, pe = min(pb + a.pc, mcols);
        const int perp = ((pe - pb) / 4 + c - 1) / c * 4;   // tokens each rank reduces in this pass
        // the slots alias the peers' rings: every rank's MMAs have finished reading its ring
        if (pass == 0) cluster_sync_relaxed();
        // push: every 4-token group of this CTA's partial goes straight into the shared memory of
        // the rank that reduces it, slot [my rank][group][nl] of float4 (a warp's store covers 512
        // contiguous bytes, the owner's 16-byte reads of consecutive lanes are conflict-free), by
        // asynchronous remote stores that complete on the owner's mbarrier: the owner waits for
        // exactly its bytes -- no cluster barrier, so no GPU-scope fence behind the epilogue's
        // global stores
        const int ng = perp / 4;   // token groups per rank
        const int mine = max(0, min((pe - pb) / 4, (r + 1) * ng) - r * ng);
        if (et == 0) mbar_arrive_expect_tx(&tfull[1], (uint32_t)(c * mine * 128 * 16));
        for (int col = pb; col < pe; col += 16) {
          float v[16];
          tmem_ld16(row_addr + col, v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = col + 4 * j - pb, owner = cc / perp, grp = (cc - owner * perp) / 4;
            st_async_f4(dsmem_addr(part_s + (((size_t)r * ng + grp) * 128 + nl) * 4, (uint32_t)owner),
                        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]),
                        dsmem_addr(&tfull[1], (uint32_t)owner));
          }
        }
        if (ct && et == 0) ct[8] = globaltimer();
        mbar_wait(&tfull[1], (uint32_t)(pass & 1));   // every rank's slices have landed
        if (ct && et == 0) ct[9] = globaltimer();
        const int lo = min(a.M, pb + r * perp), hi = min(a.M, min(pe, pb + (r + 1) * perp));
        if (res && pass > 0 && lo < hi) {
          load_res(lo, xo);
          if (lo + 16 < hi) load_res(lo + 16, xn);
        }
        for (int m0 = lo; m0 < hi; m0 += 16) {
          float v[16];
          const float* src = part_s + ((size_t)((m0 - lo) / 4) * 128 + nl) * 4;   // [rank][group][nl][4]
          // ranks in order 0 .. c-1 (R19); all loads of the chunk first
          const int nq = (min(16, hi - m0) + 3) / 4;
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
          for (int s0 = 0; s0 < c; s0 += 4) {
            float4 q[4][4];
#pragma unroll
            for (int ss = 0; ss < 4; ++ss)
#pragma unroll
              for (int j = 0; j < 4; ++j)
              {   // every slot inside the (idle) ring: load unconditionally, keep the valid ones
                const float4 t4 = *reinterpret_cast<const float4*>(src + ((size_t)(s0 + ss) * ng + j) * 128 * 4);
                q[ss][j] = (s0 + ss < c && j < nq) ? t4 : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
            for (int ss = 0; ss < 4; ++ss) {
              if (s0 + ss >= c) break;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                v[4 * j] += q[ss][j].x;
                v[4 * j + 1] += q[ss][j].y;
                v[4 * j + 2] += q[ss][j].z;
                v[4 * j + 3] += q[ss][j].w;
              }
            }
          }
          if (ct && et == 0) ct[10] = globaltimer() + (v[0] == 1.2345e-30f ? 1 : 0);
            // (the next chunk's residual rows are already in flight)
          split_finish16<YM>(a, t, nl, et, lane, m0, min(m0 + 16, hi), v, inv_s, rowmap_s, red_s, xo, w,
                         stg0 + (chunk++ & 1) * 12288);
          if (res) {
#pragma unroll
            for (int i = 0; i < 16; ++i) xo[i] = xn[i];
            if (m0 + 32 < hi) load_res(m0 + 32, xn);   // two chunks ahead of its use
          }
        }
        if (res) {
          // per-tile sums of squares of this rank's rows, warps in a fixed order
          asm volatile("bar.sync 1, 128;" ::: "memory");
          for (int m = lo + et; m < hi; m += 128)
            a.ssq_out[(size_t)t * a.Mtot + m] = ((red_s[m] + red_s[256 + m]) + red_s[512 + m]) + red_s[768 + m];
        }
        if (pass + 1 < npass) cluster_sync();   // slots are rewritten by the next pass
      }
    }
    if (res && c == 1) {
      // per-tile sums of squares of the updated residual rows, warps in a fixed order
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int m = m_lo + et; m < m_hi; m += 128)
        a.ssq_out[(size_t)t * a.Mtot + m] = ((red_s[m] + red_s[256 + m]) + red_s[512 + m]) + red_s[768 + m];
    }
    if (ct && et == 0) ct[6] = globaltimer();
  }
  if (warp < 2 && npass > 0) {
    cluster_sync_relaxed();
    for (int p = 0; p < npass - 1; ++p) cluster_sync();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, cols);
  if (ct && threadIdx.x == 0) ct[7] = globaltimer();
  if (a.timing && threadIdx.x == 0) {
    atomicMax(&a.timing[2], globaltimer());
    a.timing[3] = 1;
  }
}

using GemmKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, SplitArgs);
constexpr GemmKernel kGemmKernels[7] = {gemm_splitk_kernel<0, 0, 0>, gemm_splitk_kernel<1, 0, 0>, gemm_splitk_kernel<2, 0, 0>,
                                        gemm_splitk_kernel<0, 1, 0>, gemm_splitk_kernel<1, 1, 0>, gemm_splitk_kernel<2, 1, 0>,
                                        gemm_splitk_kernel<0, 0, 1>};
GemmKernel gemm_kernel_for(int ymode, bool split, bool tstore) {
  return tstore ? kGemmKernels[6] : kGemmKernels[(split ? 3 : 0) + ymode];
}
void gemm_kernel_attrs() {
  static bool done = false;
  if (done) return;
  for (GemmKernel k : kGemmKernels) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) cudaGetLastError();
  }
  done = true;
}

// GEMM records (kind 1): acc[0] += end - release (ns on the critical path), acc[1] += 1,
// acc[2] += end - start (span, including the PDL overlap with the predecessor); copies all records
// to `last` (the most recent round, for the trace ABI) and resets them
__global__ void timing_accumulate_kernel(unsigned long long* rec, int n, unsigned long long* acc,
                                         unsigned long long* last) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long s = rec[4 * i], r = rec[4 * i + 1], e = rec[4 * i + 2];
    if (rec[4 * i + 3] == 1 && e > s && s != ~0ull) {
      atomicAdd(&acc[0], e - (r != ~0ull && r < e ? r : s));
      atomicAdd(&acc[1], 1ull);
      atomicAdd(&acc[2], e - s);
    }
    if (last) {
      last[4 * i] = rec[4 * i];
      last[4 * i + 1] = rec[4 * i + 1];
      last[4 * i + 2] = rec[4 * i + 2];
      last[4 * i + 3] = rec[4 * i + 3];
    }
    rec[4 * i] = ~0ull;
    rec[4 * i + 1] = ~0ull;
    rec[4 * i + 2] = 0ull;
    rec[4 * i + 3] = 0ull;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

void load_encode() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<EncodeTiledFn>(fn);
}
}  // namespace

int gemm_mpad(int M) { return std::min(((M + 15) / 16) * 16, TOKEN_TILE); }

bool encode_tmap_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                    uint32_t box_outer, int swizzle_bytes) {
  std::call_once(g_encode_once, load_encode);
  if (!g_encode) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_tmap_kv_halves(CUtensorMap* map, const void* ptr, uint64_t rows, uint32_t box_rows) {
  // bf16 rows of 128 elements seen as (64 elements, row, half): one box = box_rows rows x both 64-element
  // halves, laid out in shared memory as [half][row][64] with the 128-byte swizzle
  std::call_once(g_encode_once, load_encode);
  if (!g_encode) return false;
  cuuint64_t dims[3] = {64, rows, 2};
  cuuint64_t strides[2] = {256, 128};
  cuuint32_t box[3] = {64, box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_tmap_store(CUtensorMap* map, const void* ptr, bool fp32, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer) {
  std::call_once(g_encode_once, load_encode);
  if (!g_encode) return false;
  const int es = fp32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_elems * es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// clusters of c gemm_splitk_kernel CTAs (smem_kb each) the device can hold at once
int split_cluster_capacity(int c, int smem_kb) {
  gemm_kernel_attrs();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c, 1024);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = (size_t)smem_kb * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel_for(0, true, false), &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void gemm_plan(GemmPlan* p, const void* W, int N, int K, int min_units) {
  p->N = N;
  p->K = K;
  p->KB = K / BLOCK_K;
  p->tiles = (N + BLOCK_N - 1) / BLOCK_N;
  // c CTAs per tile, c a function of (N, K) only (R19).  Enough clusters to fill two CTAs per SM,
  // at most 8 (portable cluster), at least min_units k-blocks per CTA; more tiles than SMs: whole
  // tiles.  Env SEED_SPLIT_C caps c (experiments).
  int c = 1;
  if (p->tiles < kNumSMs) c = std::min(8, (2 * kNumSMs) / p->tiles);
  c = std::min(c, std::max(1, p->KB / std::max(1, min_units)));
  const char* e = getenv("SEED_SPLIT_C");
  if (e && atoi(e) > 0) c = std::min(c, atoi(e));
  c = std::max(1, c);
  // every cluster of the grid must be resident at once (one wave): a cluster is placed inside
  // one GPC, so fewer c-CTA clusters fit than SMs / c (measured: 15 clusters of 8 at 2 CTAs per
  // SM); shrink c until the device reports room for all tiles
  for (; c > 1; --c) {
    const int smem_kb = p->tiles * c <= kNumSMs ? 180 : 112;
    const int cap = split_cluster_capacity(c, smem_kb);
    if (getenv("SEED_GEMM_VERBOSE")) fprintf(stderr, "[seed] gemm N=%d K=%d try c=%d smem=%dKB capacity=%d\n", N, K, c, smem_kb, cap);
    if (cap >= p->tiles) break;
  }
  p->c = c;
  // one CTA per SM with the deep ring while the grid fits the SMs, else two per SM (gate/up and
  // the LM heads: 172 / 250 whole tiles)
  p->split_smem_kb = p->tiles * p->c <= kNumSMs ? 180 : 112;
  if (getenv("SEED_GEMM_VERBOSE"))
    fprintf(stderr, "[seed] gemm N=%d K=%d tiles=%d c=%d smem=%dKB cluster capacity=%d\n", N, K, p->tiles, p->c,
            p->split_smem_kb, p->c > 1 ? split_cluster_capacity(p->c, p->split_smem_kb) : -1);
  encode_tmap_2d(&p->tmW, W, (uint64_t)K, (uint64_t)N, BLOCK_K, BLOCK_N);
}

void gemm_plan_free(GemmPlan*) {}


void carveout_once(const void* kern) {
  static std::vector<const void*> done;
  for (const void* k : done)
    if (k == kern) return;
  done.push_back(kern);
  const char* e = getenv("SEED_CARVEOUT");
  const int pct = e ? atoi(e) : 100;
  if (pct >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SEED_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

cudaError_t timing_accumulate(unsigned long long* rec, int n, unsigned long long* acc, unsigned long long* last,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  timing_accumulate_kernel<<<1, 256, 0, st>>>(rec, n, acc, last);
  return cudaGetLastError();
}

cudaError_t gemm_run(const GemmPlan& p, int M, const GemmIO& io, cudaStream_t st, unsigned long long* timing,
                     unsigned long long* cta) {
  const int m_pad = std::min(gemm_mpad(M), TOKEN_TILE);
  const int ttiles = (M + TOKEN_TILE - 1) / TOKEN_TILE;
  if (M < 1 || !io.tmX) return cudaErrorInvalidValue;
  if (io.ymode == 1 && (!io.Y || !io.ssq_out || !io.nw || !io.hout)) return cudaErrorInvalidValue;
  if (io.ymode == 2 && (!io.ssq_in || !io.hout || p.N % BLOCK_N)) return cudaErrorInvalidValue;
  if (io.ymode == 0 && !io.Y) return cudaErrorInvalidValue;
  // rows leave by 16-byte stores
  if (p.N % 4 || (io.ymode == 1 && p.N % 8) || (io.ymode != 2 && io.ldY % 4)) return cudaErrorInvalidValue;
  SplitArgs b{};
  b.KB = p.KB;
  b.c = p.c;
  b.M = std::min(M, TOKEN_TILE);
  b.Mtot = M;
  b.m_pad = m_pad;
  b.per = (m_pad / 4 + p.c - 1) / p.c * 4;
  b.N = p.N;
  b.K = p.K;
  b.ldY = io.ldY;
  b.ymode = io.ymode;
  b.ssq_in_ld = io.ssq_in_ld;
  b.pc = std::min(m_pad, 128);
  b.pitch = (b.pc / 4 + p.c - 1) / p.c * 4 + 4;   // [rank][128][tokens per rank + 4] slots
  b.eps = io.eps;
  b.Y = io.Y;
  b.ssq_in = io.ssq_in;
  b.yrow = io.yrow;
  b.ssq_out = io.ssq_out;
  b.nw = io.nw;
  b.hout = io.hout;
  b.timing = timing;
  b.cta = cta;
  b.tstore = 0;
  b.keep_w = p.keep_w;
  const int stage_bytes = W_TILE_BYTES + m_pad * BLOCK_K * 2;
  const int extra = (256 + 256 + 2048) * 4 + 64;   // inv_s, rowmap_s, red_s | xch, barriers
  const char* e = getenv("SEED_SPLIT_SMEM_KB");
  const int budget = (e ? atoi(e) : p.split_smem_kb) * 1024;
  int stages = (budget - 1024 - extra - 16 * 16) / stage_bytes;
  if (stages > MAX_STAGES) stages = MAX_STAGES;
  // the accumulator dump (c > 1) and the two output staging buffers alias the ring
  while (stages * stage_bytes < (c_dump_bytes(b) + 1023) / 1024 * 1024 + 2 * 12288) ++stages;
  if (stages < 2) stages = 2;
  b.stages = stages;
  // whole-tile staging + one tensor store (c = 1): the staging tile must fit the idle ring
  if (p.c == 1 && io.tmY && io.ymode == 0 && !io.yrow &&
      (size_t)((m_pad + 31) / 32 * 32) * 512 <= (size_t)stages * stage_bytes && !getenv("SEED_GEMM_NO_TSTORE"))
    b.tstore = 1;
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 2) * 8 + 16 + extra;
  gemm_kernel_attrs();
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  return launch_clustered(gemm_kernel_for(io.ymode, p.c > 1, b.tstore != 0), dim3(p.c * ttiles, p.tiles), dim3(192), smem, st, dim3(p.c, 1, 1), p.tmW,
                          *io.tmX, b.tstore ? *io.tmY : p.tmW, b);
}

}  // namespace seed
