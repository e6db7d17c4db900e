// vocab.cu -- K4 fused vocabulary kernel, the K1 draft sampler, K7 Philox fill, K5 rollback.
//
// K4 computes, for one stream per 8-CTA thread-block cluster (each CTA owns a 1/8 slice of
// the vocabulary, partial results meet through distributed shared memory in rank order):
//   a_v = fl32(z_v / T)                                     (R4)
//   log-softmax statistics with the argmax kept out of the sum: m, log1p(S')  (R13)
//   rho_j = exp(min(0, lp_j(x_j) - lq_j(x_j))), accept iff u_j < rho_j        (R2, R13)
//   a = number of leading accepts
//   y = exponential race over norm(max(0, p_{a+1} - q_{a+1})), or over p_{g+1} on full
//       acceptance (bonus, R1); ties to the smallest id (R14)                 (R3)
// Every decision is taken in fp64 after the exact fp32 front end, exactly as the oracle takes
// it (DESIGN "decision precision"), so accepted lengths and token ids match bit for bit.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace seed {

namespace {
constexpr int CS = 8;         // CTAs per cluster (portable maximum)
constexpr int VT = 256;       // threads per CTA
constexpr int MAX_ROWS = 2 * 16 + 1;

struct Stat {  // log-softmax running statistic over a set of indices
  double m;    // max of a (as fp64)
  double S;    // sum over the set minus the argmax of exp(a - m)
  int i;       // first argmax (-1: empty)
};

__device__ __forceinline__ Stat stat_merge(Stat A, Stat B) {
  if (B.i < 0) return A;
  if (A.i < 0) return B;
  if (B.m > A.m || (B.m == A.m && B.i < A.i)) {
    Stat t = A;
    A = B;
    B = t;
  }
  A.S = A.S + (B.S + 1.0) * exp(B.m - A.m);
  return A;
}

__device__ __forceinline__ Stat stat_shfl(const Stat& s, int o) {
  Stat r;
  r.m = __shfl_xor_sync(0xffffffffu, s.m, o);
  r.S = __shfl_xor_sync(0xffffffffu, s.S, o);
  r.i = __shfl_xor_sync(0xffffffffu, s.i, o);
  return r;
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
__device__ __forceinline__ Best best_shfl(const Best& b, int o) {
  return Best{__shfl_xor_sync(0xffffffffu, b.k, o), __shfl_xor_sync(0xffffffffu, b.v, o)};
}

// block-wide deterministic reductions (warp butterflies, then warps in order)
__device__ Stat block_stat(Stat s, Stat* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = stat_merge(s, stat_shfl(s, o));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = s;
  __syncthreads();
  Stat r = red[0];
  for (int i = 1; i < VT / 32; ++i) r = stat_merge(r, red[i]);
  return r;
}
__device__ Best block_best(Best b, Best* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = best_merge(b, best_shfl(b, o));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = b;
  __syncthreads();
  Best r = red[0];
  for (int i = 1; i < VT / 32; ++i) r = best_merge(r, red[i]);
  return r;
}

__device__ __forceinline__ float scaled(const float* z, int v, float T) { return __fdiv_rn(__ldg(z + v), T); }

// -log(E), E = -log1p(-u): the exponential-race offset, fp64
__device__ __forceinline__ double neg_log_exp(double u) { return -log(-log1p(-u)); }

// race over this CTA's slice with weights given by `wfn(v)` (fp64, -inf = excluded)
template <class WFn>
__device__ Best race_slice(int v0, int v1, uint32_t c1, uint32_t r, uint32_t sid, uint32_t k0, uint32_t k1,
                           WFn wfn) {
  Best b{-INFINITY, -1};
  for (int g = v0 + 4 * (int)threadIdx.x; g < v1; g += 4 * VT) {
    const Philox4 ph = philox4x32_10((uint32_t)(g >> 2), c1, r, sid, k0, k1);
    const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int v = g + e;
      if (v >= v1) break;
      const double w = wfn(v);
      if (w == -INFINITY) continue;
      const double key = w + neg_log_exp(philox_uniform(words[e]));
      if (b.v < 0 || key > b.k) b = Best{key, v};
    }
  }
  return b;
}

__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
vocab_verify_kernel(VerifyArgs A) {
  __shared__ Stat red_s[VT / 32];
  __shared__ Best red_b[VT / 32];
  __shared__ Stat cta_stat[MAX_ROWS];
  __shared__ Stat glob[MAX_ROWS];
  __shared__ Best cta_best;
  __shared__ int s_a, s_y;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  const int g = A.gamma, V = A.V;
  const int R = 2 * g + 1;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const int v0 = min(V, rank * slice), v1 = min(V, v0 + slice);
  const float* zt = A.zt + (size_t)b * A.zt_stride_b;
  const float* zd = A.zd + (size_t)b * A.zd_stride_b;
  const uint32_t sid = A.sids[b], rr = (uint32_t)A.rs[b];

  // ---- phase 1: per-row statistics over the slice (rows 0..g target, g+1..2g draft)
  for (int row = 0; row < R; ++row) {
    const float* z = row <= g ? zt + (size_t)row * V : zd + (size_t)(row - g - 1) * V;
    Stat s{-INFINITY, 0.0, -1};
    for (int v = v0 + threadIdx.x; v < v1; v += VT) {
      const double x = (double)scaled(z, v, A.T);
      if (s.i < 0) {
        s = Stat{x, 0.0, v};
      } else if (x > s.m) {
        s.S = (s.S + 1.0) * exp(s.m - x);  // the old maximum joins the tail
        s.m = x;
        s.i = v;
      } else {
        s.S += exp(x - s.m);
      }
    }
    const Stat t = block_stat(s, red_s);
    if (threadIdx.x == 0) cta_stat[row] = t;
  }
  cluster.sync();
  // ---- cluster merge in rank order (identical result in every CTA)
  for (int row = threadIdx.x; row < R; row += VT) {
    Stat acc = *cluster.map_shared_rank(&cta_stat[row], 0);
    for (int c = 1; c < CS; ++c) acc = stat_merge(acc, *cluster.map_shared_rank(&cta_stat[row], c));
    glob[row] = acc;
  }
  __syncthreads();

  // ---- phase 2: accept / reject chain
  if (threadIdx.x == 0) {
    int a = 0;
    bool alive = true;
    for (int j = 1; j <= g; ++j) {
      const int x = A.xs[(size_t)b * g + (j - 1)];
      const Stat st = glob[j - 1], sq = glob[g + j];
      const double lp = ((double)scaled(zt + (size_t)(j - 1) * V, x, A.T) - st.m) - log1p(st.S);
      const double lq = ((double)scaled(zd + (size_t)(j - 1) * V, x, A.T) - sq.m) - log1p(sq.S);
      const double rho = exp(fmin(0.0, lp - lq));
      const Philox4 ph = philox4x32_10(0u, (kTagAccept << 24) | (uint32_t)j, rr, sid, A.k0, A.k1);
      const double u = philox_uniform(ph.x);
      if (alive && u < rho) ++a;
      else alive = false;
      if (A.dbg && rank == 0) {
        float* d = A.dbg + ((size_t)b * g + (j - 1)) * 4;
        d[0] = (float)lp;
        d[1] = (float)lq;
        d[2] = (float)u;
        d[3] = (float)rho;
      }
    }
    s_a = a;
  }
  __syncthreads();
  const int a = s_a;

  // ---- phase 3: residual race on row a (0-based) or bonus race on row g
  const uint32_t c1 = (kTagResample << 24) | (uint32_t)(a + 1);
  int y = -1;
  if (a < g || A.bonus) {
    Best bb;
    if (a < g) {
      const Stat st = glob[a], sq = glob[g + 1 + a];
      const double l1t = log1p(st.S), l1q = log1p(sq.S);
      const float* zta = zt + (size_t)a * V;
      const float* zda = zd + (size_t)a * V;
      bb = race_slice(v0, v1, c1, rr, sid, A.k0, A.k1, [&](int v) -> double {
        const double lp = ((double)scaled(zta, v, A.T) - st.m) - l1t;
        const double lq = ((double)scaled(zda, v, A.T) - sq.m) - l1q;
        return lq < lp ? lp + log(-expm1(lq - lp)) : -INFINITY;
      });
    } else {
      const float* ztg = zt + (size_t)g * V;
      bb = race_slice(v0, v1, c1, rr, sid, A.k0, A.k1, [&](int v) -> double { return (double)scaled(ztg, v, A.T); });
    }
    bb = block_best(bb, red_b);
    if (threadIdx.x == 0) cta_best = bb;
    cluster.sync();
    if (threadIdx.x == 0) {
      Best acc = *cluster.map_shared_rank(&cta_best, 0);
      for (int c = 1; c < CS; ++c) acc = best_merge(acc, *cluster.map_shared_rank(&cta_best, c));
      s_y = acc.v;
    }
    __syncthreads();
    y = s_y;
    if (y < 0 && a < g) {
      // empty residual (rounding only): bonus rule on the same row, same uniforms
      const float* zta = zt + (size_t)a * V;
      Best fb = race_slice(v0, v1, c1, rr, sid, A.k0, A.k1, [&](int v) -> double { return (double)scaled(zta, v, A.T); });
      fb = block_best(fb, red_b);
      cluster.sync();   // everyone finished reading cta_best
      if (threadIdx.x == 0) cta_best = fb;
      cluster.sync();
      if (threadIdx.x == 0) {
        Best acc = *cluster.map_shared_rank(&cta_best, 0);
        for (int c = 1; c < CS; ++c) acc = best_merge(acc, *cluster.map_shared_rank(&cta_best, c));
        s_y = acc.v;
      }
      __syncthreads();
      y = s_y;
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    int32_t* ot = A.out_tok + (size_t)b * (g + 1);
    for (int j = 0; j < a; ++j) ot[j] = A.xs[(size_t)b * g + j];
    int n = a;
    if (y >= 0) ot[n++] = y;
    for (int j = n; j <= g; ++j) ot[j] = -1;
    if (A.out_cnt) A.out_cnt[b] = n;
    if (A.out_acc) A.out_acc[b] = a;
  }
  if (A.stats && rank == 0) {
    for (int row = threadIdx.x; row < R; row += VT) {
      A.stats[((size_t)b * R + row) * 2] = glob[row].m;
      A.stats[((size_t)b * R + row) * 2 + 1] = log1p(glob[row].S);
    }
  }
  cluster.sync();  // keep shared memory alive until every peer has read it
}

// K1 sampler: one cluster per row
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
draft_sample_kernel(const float* z, long ld, int V, float T, uint32_t k0, uint32_t k1, const uint32_t* sids,
                    const int32_t* rs, int j, int32_t* out, int out_stride, int32_t* out2, int out2_stride) {
  __shared__ Best red_b[VT / 32];
  __shared__ Best cta_best;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const int v0 = min(V, rank * slice), v1 = min(V, v0 + slice);
  const float* zr = z + (size_t)b * ld;
  Best bb = race_slice(v0, v1, (kTagDraft << 24) | (uint32_t)j, (uint32_t)rs[b], sids[b], k0, k1,
                       [&](int v) -> double { return (double)scaled(zr, v, T); });
  bb = block_best(bb, red_b);
  if (threadIdx.x == 0) cta_best = bb;
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) {
    Best acc = *cluster.map_shared_rank(&cta_best, 0);
    for (int c = 1; c < CS; ++c) acc = best_merge(acc, *cluster.map_shared_rank(&cta_best, c));
    out[(size_t)b * out_stride] = acc.v;
    if (out2) out2[(size_t)b * out2_stride] = acc.v;
  }
  cluster.sync();
}

__global__ void philox_fill_kernel(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int n,
                                   uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Philox4 p = philox4x32_10(c0 + (uint32_t)i, c1, c2, c3, k0, k1);
  reinterpret_cast<uint4*>(out)[i] = make_uint4(p.x, p.y, p.z, p.w);
}

// K5: commit the emitted tokens, truncate to l, roll both KV lengths back (R6, R7).
__global__ void rollback_commit_kernel(StreamState s, const int32_t* batch_slots, int B, int gamma,
                                       const int32_t* out_tok, const int32_t* out_cnt, int max_new, int32_t* records,
                                       const uint32_t* gids) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int slot = batch_slots[b];
  const int t_before = s.tlen[slot];
  const int room = max_new - s.L[slot];
  const int c = min(out_cnt[b], max(room, 0));
  int32_t* h = s.hist + (size_t)slot * s.max_ctx;
  for (int i = 0; i < c; ++i) h[t_before + i] = out_tok[(size_t)b * (gamma + 1) + i];
  const int t_new = t_before + c;
  s.tlen[slot] = t_new;
  s.L[slot] += c;
  s.r[slot] += 1;
  s.len_t[slot] = t_new - 1;                              // keep T'[:-1]
  s.len_d[slot] = min(t_new - 1, t_before + gamma - 1);   // draft wrote up to |T| + gamma - 2
  s.done[slot] = s.L[slot] >= max_new ? 1 : 0;
  if (records) {
    int32_t* rec = records + (size_t)b * (gamma + 3);
    rec[0] = (int32_t)gids[b];
    rec[1] = c;
    for (int i = 0; i <= gamma; ++i) rec[2 + i] = i < c ? out_tok[(size_t)b * (gamma + 1) + i] : -1;
  }
}
}  // namespace

cudaError_t vocab_verify(const VerifyArgs& a, cudaStream_t st) {
  if (2 * a.gamma + 1 > MAX_ROWS) return cudaErrorInvalidValue;
  vocab_verify_kernel<<<a.B * CS, VT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t draft_sample(const float* z, long ld, int B, int V, float T, uint32_t k0, uint32_t k1,
                         const uint32_t* sids, const int32_t* rs, int j, int32_t* out, int out_stride, int32_t* out2,
                         int out2_stride, cudaStream_t st) {
  draft_sample_kernel<<<B * CS, VT, 0, st>>>(z, ld, V, T, k0, k1, sids, rs, j, out, out_stride, out2, out2_stride);
  return cudaGetLastError();
}

cudaError_t philox_fill(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int n,
                        uint32_t* out, cudaStream_t st) {
  philox_fill_kernel<<<(n + 255) / 256, 256, 0, st>>>(c0, c1, c2, c3, k0, k1, n, out);
  return cudaGetLastError();
}

cudaError_t rollback_commit(const StreamState& s, const int32_t* batch_slots, int B, int gamma,
                            const int32_t* out_tok, const int32_t* out_cnt, int max_new, int32_t* records,
                            const uint32_t* gids, cudaStream_t st) {
  rollback_commit_kernel<<<(B + 127) / 128, 128, 0, st>>>(s, batch_slots, B, gamma, out_tok, out_cnt, max_new,
                                                          records, gids);
  return cudaGetLastError();
}

}  // namespace seed
