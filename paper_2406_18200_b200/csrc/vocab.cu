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
#include <algorithm>

#include "vocab_common.cuh"

namespace seed {

namespace {
using namespace vocab;

// Work area of K4 per launch (vocab_verify_work_bytes): tickets int32 [B] (zero between launches, the
// kernel re-zeroes them), accept flags int32 [B][gamma], then (8-aligned) row statistics fp64
// [B][2 gamma + 1][2] = (m, log1p(S')) of target rows 0..gamma and draft rows 0..gamma-1.
struct K4Work {
  int32_t* ticket;
  int32_t* acc;
  double* stats;
};
__host__ __device__ inline K4Work k4_work(void* base, int B, int g) {
  K4Work w;
  w.ticket = reinterpret_cast<int32_t*>(base);
  w.acc = w.ticket + B;
  const size_t off = (((size_t)B * (g + 1) * 4) + 7) & ~(size_t)7;
  w.stats = reinterpret_cast<double*>(reinterpret_cast<char*>(base) + off);
  return w;
}

// K4, two phases in one launch.  Phase 1: one 8-CTA cluster per (stream b, position j = 0..gamma)
// computes the log-softmax statistics of target row j and draft row j (R13) -- every CTA pushes its
// slice statistics into every peer's shared memory, one cluster barrier, every CTA merges them --
// and the accept decision for x_{j+1} (j < gamma), and publishes them.  Phase 2: the
// stream's last cluster to finish (ticket) counts the leading accepts a and runs the ONE race Alg. 1
// needs: the residual race over norm(max(0, p_{a+1} - q_{a+1})) (a < gamma, slot a + 1; R3) or the
// bonus race over p_{gamma+1} (a = gamma, R1) -- staging rows a again if they are not its own -- then
// emits x_1..x_a, y.  The same decisions, counters and races as the sequential Alg. 1.
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
vocab_verify_kernel(VerifyArgs A) {
  extern __shared__ __align__(128) float rows_s[];  // [2][slice] target / draft row, [slice] race keys
  __shared__ float red_f[VT / 32];
  __shared__ MaxI red_m[VT / 32];
  __shared__ double red_d[VT / 32];
  __shared__ Best red_b[VT / 32];
  __shared__ SliceStat xst[2][CS];   // the cluster's slice statistics (pushed by every rank)
  __shared__ Best xbest[CS];         // the race's slice winners (pushed to rank 0)
  __shared__ int last_s, a_s;
  __shared__ __align__(8) uint64_t bar;
  const int rank = (int)cluster_ctarank();
  const int g = A.gamma, V = A.V;
  const int cid = blockIdx.x / CS;
  const int b = cid / (g + 1), j = cid % (g + 1);
  const bool has_d = j < g;                          // draft row j exists
  const int nrows = has_d ? 2 : 1;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const int v0 = min(V, rank * slice), n = min(V, v0 + slice) - v0;
  const float* zt = A.zt + (size_t)b * A.zt_stride_b;
  const float* zd = A.zd + (size_t)b * A.zd_stride_b;
  const uint32_t sid = A.sids[b], rr = (uint32_t)A.rs[b];
  const K4Work W = k4_work(A.work, A.B, g);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  rec_start(A.timing);
  pdl_wait();   // the logits are written by the previous kernels
  rec_release(A.timing);
  Stager sg{rows_s, &bar, 0u, slice, v0, n, (V % 4 == 0) && (n % 4 == 0)};
  float* keys_s = rows_s + (size_t)2 * slice;
  sg.stage(0, nrows, [&](int row) -> const float* { return row == 0 ? zt + (size_t)j * V : zd + (size_t)j * V; });

  // ---- phase 1: slice statistics of both rows, pushed to every rank, one cluster barrier
  SliceStat my[2];
  for (int i = 0; i < nrows; ++i) my[i] = slice_stat(rows_s + (size_t)i * slice, v0, n, A.T, red_m, red_d);
  if (threadIdx.x < nrows * CS) {
    const int i = threadIdx.x / CS, c = threadIdx.x % CS;
    const SliceStat v = my[i];
    const uint32_t dst = dsmem_addr(&xst[i][rank], (uint32_t)c);
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(v.S) : "memory");
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst + 8), "f"(v.m) : "memory");
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dst + 12), "r"(v.i) : "memory");
  }
  cluster_sync();
  const RowStat st = merge_stats(xst[0]);

  double* stt = W.stats + (size_t)b * (2 * g + 1) * 2;
  if (rank == 0 && threadIdx.x == 0) {
    stt[2 * j] = st.m;
    stt[2 * j + 1] = st.l1p;
    if (has_d) {
      // accept decision for x_{j+1}: u < min(1, p / q) in log space (R2, R13)
      const RowStat sq = merge_stats(xst[1]);
      stt[2 * (g + 1 + j)] = sq.m;
      stt[2 * (g + 1 + j) + 1] = sq.l1p;
      const int x = A.xs[(size_t)b * g + j];
      double lp = -INFINITY, lq = 0.0, rho = 0.0;
      if (x >= 0 && x < V) {
        lp = ((double)scaled_v(__ldg(zt + (size_t)j * V + x), A.T) - st.m) - st.l1p;
        lq = ((double)scaled_v(__ldg(zd + (size_t)j * V + x), A.T) - sq.m) - sq.l1p;
        rho = exp(fmin(0.0, lp - lq));
      } else if (A.err) {
        atomicOr(&A.err[0], 1);   // contract violation: a drafted id outside the vocabulary is rejected
      }
      const Philox4 ph = philox4x32_10(0u, (kTagAccept << 24) | (uint32_t)(j + 1), rr, sid, A.k0, A.k1);
      const double u = philox_uniform(ph.x);
      W.acc[(size_t)b * g + j] = u < rho ? 1 : 0;
      if (A.dbg) {
        float* d = A.dbg + ((size_t)b * g + j) * 4;
        d[0] = (float)lp;
        d[1] = (float)lq;
        d[2] = (float)u;
        d[3] = (float)rho;
      }
      if (A.stats) {
        A.stats[((size_t)b * (2 * g + 1) + g + 1 + j) * 2] = sq.m;
        A.stats[((size_t)b * (2 * g + 1) + g + 1 + j) * 2 + 1] = sq.l1p;
      }
    }
    if (A.stats) {
      A.stats[((size_t)b * (2 * g + 1) + j) * 2] = st.m;
      A.stats[((size_t)b * (2 * g + 1) + j) * 2 + 1] = st.l1p;
    }
    // publish; the stream's last cluster runs phase 2 (the flag goes to every rank's shared memory)
    fence_acq_rel_gpu();
    const int t = atomicAdd(&W.ticket[b], 1);
    if (t == g) {
      fence_acq_rel_gpu();   // acquire every cluster's flags and statistics
      W.ticket[b] = 0;       // ready for the next launch (graph replay)
    }
    for (int c = 0; c < CS; ++c)
      asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsmem_addr(&last_s, (uint32_t)c)), "r"(t == g ? 1 : 0)
                   : "memory");
  }
  cluster_sync();   // the flag has landed; every peer is done reading xst
  if (!last_s) {
    rec_end(A.timing, 3);
    return;
  }

  // ---- phase 2 (the stream's last cluster): a, then the one race Alg. 1 needs
  if (threadIdx.x == 0) {
    const volatile int32_t* acc = W.acc + (size_t)b * g;
    int a = 0;
    while (a < g && acc[a]) ++a;
    a_s = a;
  }
  __syncthreads();
  const int a = a_s;
  int y = -1;
  if (a < g || A.bonus) {
    const int row = a;                          // residual on rows a (slot a + 1), or bonus on target row gamma
    const bool res = a < g;
    if (row != j) {
      // rows `row` were staged by another cluster: stage them here (L2-resident logits); the
      // generic reads of phase 1 are ordered before the bulk copies overwrite the buffers
      if (threadIdx.x == 0) fence_proxy_async();
      sg.stage(0, res ? 2 : 1, [&](int i) -> const float* { return i == 0 ? zt + (size_t)row * V : zd + (size_t)row * V; });
    }
    const volatile double* sv = W.stats + (size_t)b * (2 * g + 1) * 2;
    const double mt = sv[2 * row], l1t = sv[2 * row + 1];
    const float mtf = (float)mt, l1tf = (float)l1t;
    const float* zt_s = rows_s;
    const float* zd_s = rows_s + slice;
    const uint32_t c1 = (kTagResample << 24) | (uint32_t)(row + 1);
    auto bonus32 = [&](int l) -> float { return scaled_v(zt_s[l], A.T); };
    auto bonus64 = [&](int l) -> double { return (double)scaled_v(zt_s[l], A.T); };
    auto exchange = [&](Best mine) -> Best {   // slice winners to every rank, one barrier, merged by each
      if (threadIdx.x < CS) {
        const uint32_t dst = dsmem_addr(&xbest[rank], (uint32_t)threadIdx.x);
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(mine.k) : "memory");
        asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dst + 8), "r"(mine.v) : "memory");
      }
      cluster_sync();
      Best r{-INFINITY, -1};
      for (int c = 0; c < CS; ++c) r = best_merge(r, xbest[c]);
      return r;
    };
    if (res) {
      const double mq = sv[2 * (g + 1 + row)], l1q = sv[2 * (g + 1 + row) + 1];
      const double cq = (mq + l1q) - (mt + l1t);   // lq - lp = (a_q - a_t) - cq
      auto res32 = [&](int l) -> float {
        // lq - lp from the two fp32 logits in fp64 (their difference is exact there), so the fp32
        // screen below holds to ~1e-6 for any sign-definite difference; only |lq - lp| < 1e-12 is
        // left to fp64 (pass B).  Screen only: pass B is exact.
        const float at = scaled_v(zt_s[l], A.T);
        const double d = ((double)scaled_v(zd_s[l], A.T) - (double)at) - cq;
        if (d > -1e-12) return d >= 1e-12 ? -INFINITY : NAN;
        return ((at - mtf) - l1tf) + __logf(-expm1f((float)d));
      };
      auto res64 = [&](int l) -> double {
        const double lp = ((double)scaled_v(zt_s[l], A.T) - mt) - l1t;
        const double lq = ((double)scaled_v(zd_s[l], A.T) - mq) - l1q;
        return lq < lp ? lp + log(-expm1(lq - lp)) : -INFINITY;
      };
      y = exchange(race_slice(v0, n, c1, rr, sid, A.k0, A.k1, keys_s, red_f, red_b, res32, res64)).v;
      // empty residual (rounding only): bonus rule on the same row, same uniforms (every rank merged
      // the same winners, so the decision is uniform); the slice winners are rewritten only after
      // every rank has read them
      if (y < 0) {
        cluster_sync_relaxed();
        y = exchange(race_slice(v0, n, c1, rr, sid, A.k0, A.k1, keys_s, red_f, red_b, bonus32, bonus64)).v;
        if (A.err && rank == 0 && threadIdx.x == 0) atomicAdd(&A.err[1], 1);
      }
    } else {
      y = exchange(race_slice(v0, n, c1, rr, sid, A.k0, A.k1, keys_s, red_f, red_b, bonus32, bonus64)).v;
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    if (y < 0 && (a < g || A.bonus) && A.err) atomicOr(&A.err[0], 2);   // no finite key (non-finite logits)
    int32_t* ot = A.out_tok + (size_t)b * (g + 1);
    for (int q = 0; q < a; ++q) ot[q] = A.xs[(size_t)b * g + q];
    int cnt = a;
    if (y >= 0) ot[cnt++] = y;
    for (int q = cnt; q <= g; ++q) ot[q] = -1;
    if (A.out_cnt) A.out_cnt[b] = cnt;
    if (A.out_acc) A.out_acc[b] = a;
  }
  rec_end(A.timing, 3);
}

// K1 sampler: one cluster per row; slice winners pushed to rank 0, one barrier
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
draft_sample_kernel(const float* z, long ld, int V, float T, uint32_t k0, uint32_t k1, const uint32_t* sids,
                    const int32_t* rs, int j, int32_t* out, int out_stride, int32_t* out2, int out2_stride,
                    int32_t* err, unsigned long long* rec, EmbedNext en) {
  extern __shared__ __align__(128) float rows_s[];  // [slice] row, then [slice] race keys
  __shared__ float red_f[VT / 32];
  __shared__ float red_e[VT / 32];
  __shared__ Best red_b[VT / 32];
  __shared__ Best xbest[CS];
  __shared__ __align__(8) uint64_t bar;
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / CS;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const int v0 = min(V, rank * slice), n = min(V, v0 + slice) - v0;
  const float* zr = z + (size_t)b * ld;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  rec_start(rec);
  // the race's screen offsets before the wait (they need only the counters: sids / rs are uploaded
  // before the round's first kernel)
  const uint32_t c1 = (kTagDraft << 24) | (uint32_t)j, rr = (uint32_t)rs[b], sid = sids[b];
  ScreenPre pre;
  const bool use_pre = n <= 4 * VT * RACE_NB;
  if (use_pre) screen_precompute(v0, n, c1, rr, sid, k0, k1, pre);
  pdl_wait();
  rec_release(rec);
  Stager sg{rows_s, &bar, 0u, slice, v0, n, (V % 4 == 0) && (n % 4 == 0) && (ld % 4 == 0)};
  sg.stage(0, 1, [&](int) { return zr; });
  auto w32 = [&](int l) -> float { return scaled_v(rows_s[l], T); };
  auto w64 = [&](int l) -> double { return (double)scaled_v(rows_s[l], T); };
  const Best mine = race_slice(v0, n, c1, rr, sid, k0, k1, rows_s + slice, red_f, red_b, w32, w64,
                               use_pre ? &pre : nullptr);
  // slice winners to rank 0 (to every rank when the next step's embedding is fused: each merges)
  const int npush = en.emb ? CS : 1;
  if (threadIdx.x < npush) {
    const uint32_t dst = dsmem_addr(&xbest[rank], (uint32_t)threadIdx.x);
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(mine.k) : "memory");
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dst + 8), "r"(mine.v) : "memory");
  }
  cluster_sync();
  if (rank == 0 && threadIdx.x == 0) {
    Best acc{-INFINITY, -1};
    for (int c = 0; c < CS; ++c) acc = best_merge(acc, xbest[c]);
    out[(size_t)b * out_stride] = acc.v;
    if (out2) out2[(size_t)b * out2_stride] = acc.v;
    if (acc.v < 0 && err) atomicOr(err, 2);   // no finite key (non-finite logits)
  }
  if (en.emb) {
    // the next draft step's embedding of row b, 128-column tiles rank, rank + CS, ...: the same
    // values, warp sums and warp order as embed_stats (a token outside the table reads row 0)
    Best acc{-INFINITY, -1};
    for (int c = 0; c < CS; ++c) acc = best_merge(acc, xbest[c]);
    const int id = acc.v >= 0 && acc.v < V ? acc.v : 0;
    const int nt = (en.d + 127) / 128, w = threadIdx.x >> 5;
    for (int t0 = rank * 2; t0 < nt; t0 += 2 * CS) {   // two tiles per pass: warps 0-3 and 4-7
      const int tile = t0 + (w >> 2), n = tile * 128 + (threadIdx.x & 127);
      float v = 0.f;
      if (tile < nt && n < en.d) {
        v = bf2f(en.emb[(size_t)id * en.d + n]);
        en.x[(size_t)b * en.d + n] = v;
        en.h[(size_t)b * en.d + n] = f2bf(v * bf2f(en.nw[n]));
      }
      const float sq = warp_sum(v * v);
      if ((threadIdx.x & 31) == 0) red_e[w] = sq;
      __syncthreads();
      if ((threadIdx.x & 127) == 0 && tile < nt) {
        const int q = w & ~3;
        en.ssq[(size_t)tile * en.ssq_ld + b] = ((red_e[q] + red_e[q + 1]) + red_e[q + 2]) + red_e[q + 3];
      }
      __syncthreads();
    }
  }
  rec_end(rec, 4);
}

__global__ void philox_fill_kernel(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int n,
                                   uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Philox4 p = philox4x32_10(c0 + (uint32_t)i, c1, c2, c3, k0, k1);
  reinterpret_cast<uint4*>(out)[i] = make_uint4(p.x, p.y, p.z, p.w);
}

// K5: commit the emitted tokens, truncate to l, roll both KV lengths back (R6, R7), and write this
// rank's exchange block (a6): one record [gid, c, tokens] per stream, then the number of this rank's
// streams still undone after the round (*outside = undone streams not in the batch).  One CTA.
constexpr int K5_THREADS = 256;
__global__ void __launch_bounds__(K5_THREADS)
rollback_commit_kernel(StreamState s, const int32_t* batch_slots, int B, int gamma, const int32_t* out_tok,
                       const int32_t* out_cnt, int max_new, int32_t* records, int cap, const uint32_t* gids,
                       const int32_t* outside, unsigned long long* rec) {
  __shared__ int red[K5_THREADS / 32];
  pdl_trigger();
  rec_start(rec);
  pdl_wait();
  rec_release(rec);
  int undone = 0;
  for (int b = threadIdx.x; b < B; b += K5_THREADS) {
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
    const int done = s.L[slot] >= max_new ? 1 : 0;
    s.done[slot] = done;
    undone += 1 - done;
    int32_t* rec = records + (size_t)b * (gamma + 3);
    rec[0] = (int32_t)gids[b];
    rec[1] = c;
    for (int i = 0; i <= gamma; ++i) rec[2 + i] = i < c ? out_tok[(size_t)b * (gamma + 1) + i] : -1;
  }
  // the block's unused records read as empty (-1): written here rather than by a memset before the
  // kernel, which would break the PDL chain from K4 (a graph memset node waits for K4 to finish)
  for (int i = B * (gamma + 3) + threadIdx.x; i < cap * (gamma + 3); i += K5_THREADS) records[i] = -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) undone += __shfl_xor_sync(0xffffffffu, undone, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = undone;
  __syncthreads();
  if (threadIdx.x == 0) {
    int u = *outside;
    for (int w = 0; w < K5_THREADS / 32; ++w) u += red[w];
    records[(size_t)cap * (gamma + 3)] = u;
  }
  rec_end(rec, 6);
}
}  // namespace

size_t vocab_verify_work_bytes(int B, int gamma) {
  return ((((size_t)B * (gamma + 1) * 4) + 7) & ~(size_t)7) + (size_t)B * (2 * gamma + 1) * 2 * sizeof(double);
}

cudaError_t vocab_verify(const VerifyArgs& a, cudaStream_t st) {
  if (!a.work || a.gamma < 1) return cudaErrorInvalidValue;
  const int slice = ((a.V + CS - 1) / CS + 3) & ~3;
  const size_t smem = (size_t)3 * slice * 4;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(vocab_verify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  return launch(vocab_verify_kernel, dim3(a.B * (a.gamma + 1) * CS), dim3(VT), smem, st, a);
}

cudaError_t draft_sample(const float* z, long ld, int B, int V, float T, uint32_t k0, uint32_t k1,
                         const uint32_t* sids, const int32_t* rs, int j, int32_t* out, int out_stride, int32_t* out2,
                         int out2_stride, int32_t* err, cudaStream_t st, unsigned long long* timing,
                         const EmbedNext& en) {
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const size_t smem = (size_t)2 * slice * 4;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(draft_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  return launch(draft_sample_kernel, dim3(B * CS), dim3(VT), smem, st, z, ld, V, T, k0, k1, sids, rs, j, out,
                out_stride, out2, out2_stride, err, timing, en);
}

cudaError_t philox_fill(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int n,
                        uint32_t* out, cudaStream_t st) {
  philox_fill_kernel<<<(n + 255) / 256, 256, 0, st>>>(c0, c1, c2, c3, k0, k1, n, out);
  return cudaGetLastError();
}

cudaError_t rollback_commit(const StreamState& s, const int32_t* batch_slots, int B, int gamma,
                            const int32_t* out_tok, const int32_t* out_cnt, int max_new, int32_t* records, int cap,
                            const uint32_t* gids, const int32_t* outside, cudaStream_t st,
                            unsigned long long* timing) {
  return launch(rollback_commit_kernel, dim3(1), dim3(K5_THREADS), 0, st, s, batch_slots, B, gamma, out_tok, out_cnt,
                max_new, records, cap, gids, outside, timing);
}

}  // namespace seed
