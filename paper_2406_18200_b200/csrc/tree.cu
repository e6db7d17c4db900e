// tree.cu -- k_config tree drafting and verification on the vocabulary side (
// PAPER.md §3.2, App. B; R36).
//
//   K1T  draft_topk_kernel   node n's m children: the m largest keys of the exponential race over
//                            the draft row conditioned on n's path (tag DRAFT, slot n + 1) -- a draw
//                            without replacement (the chain's K1 is m = 1)
//   K4T  verify_tree_kernel  walks the tree from the root: at node n, candidates in their drawn order
//                            are accepted with min(1, p(c) / q(c)); a rejection updates
//                            p <- norm(max(0, p - q)), q <- q without c; the first accepted child
//                            becomes the path; all rejected -> correction from the residual (slot
//                            n + 1); a leaf reached -> bonus from p (slot n + 1).
// One 8-CTA cluster per stream; every rank makes every decision from the same exchanged values
// (uniform control flow).  fp64 decisions after the exact fp32 front end, like oracle/tree.py.
#include "vocab_common.cuh"

namespace seed {

namespace {
using namespace vocab;

constexpr int MAXC = 8;        // children per node
constexpr int CAND = 64;       // exact-rescoring candidates per slice (top-m)

struct TopEntry {
  double k;
  int v;
  int pad;
};

__device__ __forceinline__ bool key_before(double ka, int va, double kb, int vb) {
  return ka > kb || (ka == kb && va < vb);
}

// top-m race over this CTA's slice of one row, exact (fp32 screen within RACE_MARGIN of the slice's
// m-th best screened key, fp64 rescoring); every rank pushes its slice top-m to every rank and
// merges: out[0..m) is the global top-m (decreasing keys, ties -> smaller id).  Returns the count.
template <class W32, class W64>
__device__ int race_topm(int v0, int n, int m, uint32_t c1, uint32_t r, uint32_t sid, uint32_t k0, uint32_t k1,
                         float* keys, float* red_f, TopEntry* cand, int* ncand, TopEntry* xtop, TopEntry* out,
                         int32_t* err, W32 w32, W64 w64) {
  for (int l = 4 * (int)threadIdx.x; l < n; l += 4 * VT) {
    const int g = v0 + l;
    const Philox4 ph = philox4x32_10((uint32_t)(g >> 2), c1, r, sid, k0, k1);
    const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (l + e >= n) break;
      const float w = w32(l + e);
      float key = -INFINITY;
      if (w != w) {
        const double wd = w64(l + e);
        if (wd != -INFINITY) key = (float)(wd + neg_log_exp(philox_uniform(words[e])));
      } else if (w != -INFINITY) {
        key = w + neg_log_exp_screen((float)philox_uniform(words[e]));
      }
      keys[l + e] = key;
    }
  }
  __syncthreads();
  // the m-th largest screened key of the slice: m rounds of a block max over the keys above it
  float thr = INFINITY, kth = -INFINITY;
  for (int q = 0; q < m; ++q) {
    float best = -INFINITY;
    for (int l = threadIdx.x; l < n; l += VT)
      if (keys[l] < thr) best = fmaxf(best, keys[l]);
    kth = block_maxf(best, red_f);
    if (kth == -INFINITY) break;
    thr = kth;
  }
  if (threadIdx.x == 0) *ncand = 0;
  __syncthreads();
  const float cut = kth == -INFINITY ? -INFINITY : kth - RACE_MARGIN;
  for (int l = threadIdx.x; l < n; l += VT) {
    if (!(keys[l] >= cut) || keys[l] == -INFINITY) continue;
    const int g = v0 + l;
    const Philox4 ph = philox4x32_10((uint32_t)(g >> 2), c1, r, sid, k0, k1);
    const uint32_t words[4] = {ph.x, ph.y, ph.z, ph.w};
    const double wd = w64(l);
    if (wd == -INFINITY) continue;
    const int slot = atomicAdd(ncand, 1);
    if (slot < CAND) cand[slot] = TopEntry{wd + neg_log_exp(philox_uniform(words[g & 3])), g, 0};
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nc = *ncand;
    if (nc > CAND) {
      nc = CAND;
      if (err) atomicOr(err, 4);   // more near-ties than the rescoring list holds (never observed)
    }
    // slice top-m by selection (nc <= 64, m <= 8)
    TopEntry mine[MAXC];
    for (int q = 0; q < m; ++q) {
      int bi = -1;
      for (int i = 0; i < nc; ++i) {
        if (cand[i].v < 0) continue;
        if (bi < 0 || key_before(cand[i].k, cand[i].v, cand[bi].k, cand[bi].v)) bi = i;
      }
      mine[q] = bi >= 0 ? cand[bi] : TopEntry{-INFINITY, -1, 0};
      if (bi >= 0) cand[bi].v = -1;
    }
    for (int q = 0; q < m; ++q) push_all(&mine[q], &xtop[cluster_ctarank() * MAXC + q], sizeof(TopEntry));
  }
  cluster_sync();
  int cnt = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < m; ++q) {
      int bi = -1;
      for (int i = 0; i < CS * m; ++i) {
        const TopEntry& e = xtop[(i / m) * MAXC + i % m];
        if (e.v < 0) continue;
        bool used = false;
        for (int j = 0; j < q; ++j) used |= out[j].v == e.v;
        if (used) continue;
        if (bi < 0 || key_before(e.k, e.v, xtop[(bi / m) * MAXC + bi % m].k, xtop[(bi / m) * MAXC + bi % m].v)) bi = i;
      }
      if (bi < 0) break;
      out[q] = xtop[(bi / m) * MAXC + bi % m];
      ++cnt;
    }
    out[MAXC].v = cnt;
  }
  __syncthreads();
  return out[MAXC].v;
}

// K1T: one cluster per (stream b, node row); out[b][first + q] = the q-th child's token
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
draft_topk_kernel(const float* z, long ld, int V, float T, uint32_t k0, uint32_t k1, const uint32_t* sids,
                  const int32_t* rs, int node, int m, int32_t* out, int out_stride, int first, int32_t* out2,
                  int out2_stride, int32_t* err, unsigned long long* rec) {
  extern __shared__ __align__(128) float rows_s[];  // [slice] row, then [slice] race keys
  __shared__ float red_f[VT / 32];
  __shared__ TopEntry cand[CAND];
  __shared__ int ncand;
  __shared__ TopEntry xtop[CS * MAXC];
  __shared__ TopEntry top[MAXC + 1];
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
  pdl_wait();
  rec_release(rec);
  Stager sg{rows_s, &bar, 0u, slice, v0, n, (V % 4 == 0) && (n % 4 == 0) && (ld % 4 == 0)};
  sg.stage(0, 1, [&](int) { return zr; });
  auto w32 = [&](int l) -> float { return scaled_v(rows_s[l], T); };
  auto w64 = [&](int l) -> double { return (double)scaled_v(rows_s[l], T); };
  const int cnt = race_topm(v0, n, m, (kTagDraft << 24) | (uint32_t)(node + 1), (uint32_t)rs[b], sids[b], k0, k1,
                            rows_s + slice, red_f, cand, &ncand, xtop, top, err, w32, w64);
  if (rank == 0 && threadIdx.x < m) {
    const int v = threadIdx.x < cnt ? top[threadIdx.x].v : -1;
    out[(size_t)b * out_stride + first + threadIdx.x] = v;
    if (out2) out2[(size_t)b * out2_stride + first + threadIdx.x] = v;
    if (v < 0 && err) atomicOr(err, 2);
  }
  cluster_sync_relaxed();   // peers' pushes into xtop are complete before any rank exits
  rec_end(rec, 4);
}

// K4T.  tree: ch_first[node], ch_cnt[node] (breadth-first, children contiguous); zt / zd rows are
// per node (row n: the distributions of n's children, or at a leaf the bonus row); tok [B][n + 1].
struct TreeArgs {
  const float* zt;
  const float* zd;
  long zt_stride_b, zd_stride_b;
  const int32_t* tok;
  int tok_stride;
  const int32_t* ch_first;
  const int32_t* ch_cnt;
  int B, K, V;
  float T;
  uint32_t k0, k1;
  const uint32_t* sids;
  const int32_t* rs;
  int bonus;
  int32_t* out_tok;    // [B][K + 1]: path tokens, y, -1 pad
  int32_t* out_cnt;    // [B]
  int32_t* out_node;   // [B][K]: accepted node indices, -1 pad (optional)
  int32_t* err;
  unsigned long long* timing;
};

struct Lse {   // log-sum-exp partial: max and sum of exp(w - max)
  double m, s;
};

__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(VT)
verify_tree_kernel(TreeArgs A) {
  extern __shared__ __align__(128) float rows_s[];  // [2][slice] fp32 rows, [slice] keys, then fp64 w [slice]
  __shared__ float red_f[VT / 32];
  __shared__ MaxI red_m[VT / 32];
  __shared__ double red_d[VT / 32];
  __shared__ Best red_b[VT / 32];
  __shared__ SliceStat xst[2][CS];
  __shared__ Lse xl[CS];
  __shared__ double xw, xw_keep;   // the next candidate's new / kept residual weight (pushed by its owner)
  __shared__ Best xbest[CS];
  __shared__ __align__(8) uint64_t bar;
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / CS;
  const int V = A.V;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const int v0 = min(V, rank * slice), n = min(V, v0 + slice) - v0;
  const float* zt = A.zt + (size_t)b * A.zt_stride_b;
  const float* zd = A.zd + (size_t)b * A.zd_stride_b;
  const int32_t* tok = A.tok + (size_t)b * A.tok_stride;
  const uint32_t sid = A.sids[b], rr = (uint32_t)A.rs[b];
  float* zt_s = rows_s;
  float* zd_s = rows_s + slice;
  float* keys_s = rows_s + 2 * (size_t)slice;
  double* w_buf = reinterpret_cast<double*>(rows_s + 3 * (size_t)slice + (slice & 1));   // [2][slice]
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  rec_start(A.timing);
  pdl_wait();
  rec_release(A.timing);
  Stager sg{rows_s, &bar, 0u, slice, v0, n, (V % 4 == 0) && (n % 4 == 0)};
  auto race_all = [&](auto w32, auto w64, int node) -> int {   // exact race, winners to every rank
    const Best mine = race_slice(v0, n, (kTagResample << 24) | (uint32_t)(node + 1), rr, sid, A.k0, A.k1, keys_s, red_f,
                                 red_b, w32, w64);
    if (threadIdx.x == 0) push_all(&mine, &xbest[rank], sizeof(Best));
    cluster_sync();
    Best r{-INFINITY, -1};
    for (int c = 0; c < CS; ++c) r = best_merge(r, xbest[c]);
    cluster_sync_relaxed();   // xbest is rewritten only after every rank has read it
    return r.v;
  };
  int node = 0, a = 0, y = -1;
  int path[16];
  sg.stage(0, 2, [&](int i) -> const float* { return i == 0 ? zt : zd; });
  for (;;) {
    // ---- statistics of this node's target and draft rows (R13), one exchange
    SliceStat my[2];
    my[0] = slice_stat(zt_s, v0, n, A.T, red_m, red_d);
    my[1] = slice_stat(zd_s, v0, n, A.T, red_m, red_d);
    if (threadIdx.x < 2) push_all(&my[threadIdx.x], &xst[threadIdx.x][rank], sizeof(SliceStat));
    cluster_sync();
    const RowStat st = merge_stats(xst[0]), sq = merge_stats(xst[1]);
    cluster_sync_relaxed();   // xst is rewritten at the next node only after every rank read it
    const int c0 = __ldg(A.ch_first + node), m = __ldg(A.ch_cnt + node);
    // ---- recursive rejection over the candidates (oracle.tree.rejection_chain): the current p is
    // the row's log-softmax while `fresh`, else w_cur - N; q is the row's minus the removed mass Sq,
    // with the rejected candidates excluded
    double Sq = 0.0, N = 0.0;
    bool fresh = true, last_fb = false, any_fb = false;
    int cur = 0;
    int excl[MAXC];
    int nex = 0, accepted = -1;
    const float* zt_node = zt + (size_t)node * V;
    const float* zd_node = zd + (size_t)node * V;
    auto lp_of = [&](int v, int l) -> double {   // l: index in this slice
      if (fresh) return ((double)scaled_v(zt_s[l], A.T) - st.m) - st.l1p;
      return w_buf[(size_t)cur * slice + l] - N;
    };
    auto lq_of = [&](int v, int l) -> double {   // l < 0: read the row from global memory
      for (int e = 0; e < nex; ++e)
        if (excl[e] == v) return -INFINITY;
      return (((double)scaled_v(l >= 0 ? zd_s[l] : __ldg(zd_node + v), A.T) - sq.m) - sq.l1p) - Sq;
    };
    for (int i = 0; i < m; ++i) {
      const int c = c0 + i, x = tok[c];
      const bool xin = x >= 0 && x < V;
      if (!xin && A.err && rank == 0 && threadIdx.x == 0) atomicOr(&A.err[0], 1);   // rejected: bad id
      const double lpx = !xin ? -INFINITY
                              : (fresh ? ((double)scaled_v(__ldg(zt_node + x), A.T) - st.m) - st.l1p : xw - N);
      const double lqx = !xin ? 0.0 : lq_of(x, -1);
      const double rho = xin ? exp(fmin(0.0, lpx - lqx)) : 0.0;
      const double u = philox_uniform(philox4x32_10(0u, (kTagAccept << 24) | (uint32_t)c, rr, sid, A.k0, A.k1).x);
      if (u < rho) {
        accepted = c;
        break;
      }
      // rejected: w <- log max(0, p - q) over the slice (into the other buffer), its log-sum-exp
      // exchanged together with the next candidate's weight
      double* w_nxt = w_buf + (size_t)(cur ^ 1) * slice;
      double lm = -INFINITY;
      for (int l = threadIdx.x; l < n; l += VT) {
        const int v = v0 + l;
        const double lp = lp_of(v, l), lq = lq_of(v, l);
        const double w = lq < lp ? lp + log(-expm1(lq - lp)) : -INFINITY;
        w_nxt[l] = w;
        lm = fmax(lm, w);
      }
      __shared__ double red_x[VT / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
      __syncthreads();
      if ((threadIdx.x & 31) == 0) red_x[threadIdx.x >> 5] = lm;
      __syncthreads();
      double bm = red_x[0];
      for (int k = 1; k < VT / 32; ++k) bm = fmax(bm, red_x[k]);
      double ls = 0.0;
      if (bm != -INFINITY)
        for (int l = threadIdx.x; l < n; l += VT)
          if (w_nxt[l] != -INFINITY) ls += exp(w_nxt[l] - bm);
      ls = block_sum(ls, red_d);   // (its barriers also order w_nxt before the reads below)
      if (threadIdx.x == 0) {
        const Lse mine{bm, ls};
        push_all(&mine, &xl[rank], sizeof(Lse));
        if (i + 1 < m) {   // the owner of the next candidate pushes its new weight
          const int xn = tok[c + 1];
          if (xn >= v0 && xn < v0 + n) {
            const double wn[2] = {w_nxt[xn - v0], fresh ? 0.0 : w_buf[(size_t)cur * slice + (xn - v0)]};
            push_all(&wn[0], &xw, sizeof(double));
            push_all(&wn[1], &xw_keep, sizeof(double));
          }
        }
      }
      cluster_sync();
      double gm = -INFINITY;
      for (int k = 0; k < CS; ++k) gm = fmax(gm, xl[k].m);
      double gs = 0.0;
      if (gm != -INFINITY)
        for (int k = 0; k < CS; ++k)
          if (xl[k].m != -INFINITY) gs += xl[k].s * exp(xl[k].m - gm);
      last_fb = gm == -INFINITY;
      if (last_fb) {
        // empty residual (rounding only): p is kept (the oracle's fallback), flagged; the next
        // candidate's weight is its kept one (fresh: read from the row again)
        any_fb = true;
        __syncthreads();
        if (threadIdx.x == 0) xw = xw_keep;
        __syncthreads();
      } else {
        N = gm + log(gs);
        fresh = false;
        cur ^= 1;
      }
      const double rest = -expm1(lqx);   // 1 - q(x)
      Sq += rest > 0.0 ? log(rest) : INFINITY;
      if (nex < MAXC) excl[nex++] = x;
      cluster_sync_relaxed();   // xl / xw are rewritten only after every rank read them
    }
    if (accepted < 0) {
      // every candidate rejected: the correction from the residual (slot node + 1)
      if (A.err && any_fb && rank == 0 && threadIdx.x == 0) atomicAdd(&A.err[1], 1);
      if (last_fb && (m == 1 || fresh)) {   // the chain's fallback: the bonus rule on this row
        y = race_all([&](int l) -> float { return scaled_v(zt_s[l], A.T); },
                     [&](int l) -> double { return (double)scaled_v(zt_s[l], A.T); }, node);
      } else if (last_fb) {                  // the kept (normalised) p
        const double* wc = w_buf + (size_t)cur * slice;
        y = race_all([&](int l) -> float { return (float)(wc[l] - N); }, [&](int l) -> double { return wc[l] - N; },
                     node);
      } else {
        const double* wc = w_buf + (size_t)cur * slice;
        y = race_all([&](int l) -> float { return (float)wc[l]; }, [&](int l) -> double { return wc[l]; }, node);
      }
      break;
    }
    node = accepted;
    path[a++] = node;
    if (__ldg(A.ch_cnt + node) == 0) {   // a leaf: the bonus token from its target row (R1)
      if (A.bonus) {
        if (threadIdx.x == 0) fence_proxy_async();
        sg.stage(0, 1, [&](int) -> const float* { return zt + (size_t)node * V; });
        y = race_all([&](int l) -> float { return scaled_v(zt_s[l], A.T); },
                     [&](int l) -> double { return (double)scaled_v(zt_s[l], A.T); }, node);
      }
      break;
    }
    if (threadIdx.x == 0) fence_proxy_async();
    sg.stage(0, 2, [&](int i) -> const float* { return i == 0 ? zt + (size_t)node * V : zd + (size_t)node * V; });
  }
  if (rank == 0 && threadIdx.x == 0) {
    int32_t* ot = A.out_tok + (size_t)b * (A.K + 1);
    for (int q = 0; q < a; ++q) ot[q] = tok[path[q]];
    int cnt = a;
    if (y >= 0) ot[cnt++] = y;
    for (int q = cnt; q <= A.K; ++q) ot[q] = -1;
    A.out_cnt[b] = cnt;
    if (A.out_node)
      for (int q = 0; q < A.K; ++q) A.out_node[(size_t)b * A.K + q] = q < a ? path[q] : -1;
    if (y < 0 && (a < A.K || A.bonus) && A.err) atomicOr(&A.err[0], 2);
  }
  rec_end(A.timing, 3);
}
}  // namespace

cudaError_t draft_topk(const float* z, long ld, int B, int V, float T, uint32_t k0, uint32_t k1, const uint32_t* sids,
                       const int32_t* rs, int node, int m, int32_t* out, int out_stride, int first, int32_t* out2,
                       int out2_stride, int32_t* err, cudaStream_t st, unsigned long long* timing) {
  if (m < 1 || m > MAXC) return cudaErrorInvalidValue;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const size_t smem = (size_t)2 * slice * 4;
  if (smem > 180 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(draft_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  return launch(draft_topk_kernel, dim3(B * CS), dim3(VT), smem, st, z, ld, V, T, k0, k1, sids, rs, node, m, out,
                out_stride, first, out2, out2_stride, err, timing);
}

cudaError_t verify_tree(const float* zt, long zt_stride_b, const float* zd, long zd_stride_b, const int32_t* tok,
                        int tok_stride, const int32_t* ch_first, const int32_t* ch_cnt, int B, int K, int V, float T,
                        uint32_t k0, uint32_t k1, const uint32_t* sids, const int32_t* rs, int bonus, int32_t* out_tok,
                        int32_t* out_cnt, int32_t* out_node, int32_t* err, cudaStream_t st,
                        unsigned long long* timing) {
  if (K < 1 || K > 15) return cudaErrorInvalidValue;
  const int slice = ((V + CS - 1) / CS + 3) & ~3;
  const size_t smem = (size_t)3 * slice * 4 + 8 + (size_t)2 * slice * 8;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(verify_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  TreeArgs a{};
  a.zt = zt;
  a.zd = zd;
  a.zt_stride_b = zt_stride_b;
  a.zd_stride_b = zd_stride_b;
  a.tok = tok;
  a.tok_stride = tok_stride;
  a.ch_first = ch_first;
  a.ch_cnt = ch_cnt;
  a.B = B;
  a.K = K;
  a.V = V;
  a.T = T;
  a.k0 = k0;
  a.k1 = k1;
  a.sids = sids;
  a.rs = rs;
  a.bonus = bonus;
  a.out_tok = out_tok;
  a.out_cnt = out_cnt;
  a.out_node = out_node;
  a.err = err;
  a.timing = timing;
  return launch(verify_tree_kernel, dim3(B * CS), dim3(VT), smem, st, a);
}

}  // namespace seed
