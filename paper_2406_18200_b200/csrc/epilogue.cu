// epilogue.cu -- the fused consumers of the K2 partial sums, plus embedding and RoPE table.
//
// Each consumer sums the split-K partials of its output element in CTA order (fixed,
// M-independent: R19) and applies the layer step that follows the projection in the
// Llama-2 block (R15), storing bf16 exactly where DESIGN.md "bf16 rounding points" says:
//   QKV   -> RoPE(q), RoPE(k), v -> bf16 Q buffer, K/V appended to the paged cache (B2)
//   O     -> residual add (fp32, F1) -> RMSNorm(mlp_norm) -> bf16 operand (B1)
//   gate/up (interleaved 64-row blocks) -> silu(g) * u -> bf16 operand (B4)
//   down  -> residual add (F1) -> RMSNorm(next attn_norm / final_norm) -> bf16 (B1)
//   LM head -> fp32 logits (F2)
// Row-wide RMSNorm runs on an 8-CTA cluster per row: each CTA owns d/8 columns, the
// sums of squares meet through distributed shared memory in rank order.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace seed {

namespace {

// sum over the CTAs that covered tile n / 128, in CTA order (precomputed table).  Up to 8
// segments are loaded with independent, predicated loads so they are all in flight at once.
__device__ __forceinline__ float partial_sum(const PartialView& v, int m, int n) {
  const int t = n >> 7, nl = n & 127;
  const int* s = v.seg + t * (v.maxseg + 1);
  const int cnt = __ldg(s);
  constexpr int K = 8;
  float vals[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int id = k < cnt ? __ldg(s + 1 + k) : 0;
    vals[k] = k < cnt ? __ldg(v.p + ((size_t)id * v.M + m) * 128 + nl) : 0.f;
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) acc += vals[k];
  for (int k = K; k < cnt; ++k) acc += __ldg(v.p + ((size_t)__ldg(s + 1 + k) * v.M + m) * 128 + nl);
  return acc;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

__global__ void epi_store_kernel(PartialView v, int N, float* Y, int ldY, const int32_t* row_map) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int dst = row_map ? row_map[m] : m;
  if (dst < 0) return;
  Y[(size_t)dst * ldY + n] = partial_sum(v, m, n);
}

constexpr int NORM_THREADS = 256;
constexpr int RCS = 8;            // CTAs per row (cluster)
constexpr int RN_THREADS = 128;

__global__ void __launch_bounds__(NORM_THREADS)
embed_rmsnorm_kernel(const __nv_bfloat16* __restrict__ embed, const int32_t* __restrict__ tok, int tok_stride, int d,
                     const __nv_bfloat16* __restrict__ w, float eps, float* __restrict__ x,
                     __nv_bfloat16* __restrict__ h) {
  __shared__ float red[NORM_THREADS / 32];
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const __nv_bfloat16* e = embed + (size_t)tok[(size_t)m * tok_stride] * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += NORM_THREADS) {
    const float xv = bf2f(e[i]);
    x[(size_t)m * d + i] = xv;
    ss += xv * xv;
  }
  const float tot = block_sum<NORM_THREADS>(ss, red);
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += NORM_THREADS)
    h[(size_t)m * d + i] = f2bf(x[(size_t)m * d + i] * inv * bf2f(w[i]));
}

// x[m] += sum of partials (or nothing when v.p == nullptr); h = bf16(rmsnorm(x[m]) * w).
// grid (M * RCS), cluster (RCS): CTA `rank` owns columns [rank * cw, (rank + 1) * cw).
__global__ void __cluster_dims__(RCS, 1, 1) __launch_bounds__(RN_THREADS)
residual_rmsnorm_kernel(PartialView v, int d, float* __restrict__ x, const __nv_bfloat16* __restrict__ w, float eps,
                        __nv_bfloat16* __restrict__ h, const int32_t* __restrict__ compact_map,
                        __nv_bfloat16* __restrict__ h_compact) {
  __shared__ float red[RN_THREADS / 32];
  __shared__ float cta_ss;
  pdl_trigger();
  pdl_wait();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int m = blockIdx.x / RCS;
  const int cw = (d + RCS - 1) / RCS;
  const int c0 = rank * cw, c1 = min(d, c0 + cw);
  float* xr = x + (size_t)m * d;
  // up to CPT columns per thread, all loads issued before any store (ILP)
  constexpr int CPT = 6;
  float vals[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = c0 + threadIdx.x + k * RN_THREADS;
    vals[k] = 0.f;
    if (i < c1) vals[k] = xr[i] + (v.p ? partial_sum(v, m, i) : 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = c0 + threadIdx.x + k * RN_THREADS;
    if (i < c1) {
      if (v.p) xr[i] = vals[k];
      ss += vals[k] * vals[k];
    }
  }
  for (int i = c0 + threadIdx.x + CPT * RN_THREADS; i < c1; i += RN_THREADS) {  // very wide rows
    float nv = xr[i];
    if (v.p) {
      nv += partial_sum(v, m, i);
      xr[i] = nv;
    }
    ss += nv * nv;
  }
  const float t = block_sum<RN_THREADS>(ss, red);
  if (threadIdx.x == 0) cta_ss = t;
  cluster.sync();
  float tot = 0.f;
  for (int c = 0; c < RCS; ++c) tot += *cluster.map_shared_rank(&cta_ss, c);
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  const int cm = compact_map ? compact_map[m] : -1;
  for (int i = c0 + threadIdx.x; i < c1; i += RN_THREADS) {
    const __nv_bfloat16 o = f2bf(xr[i] * inv * bf2f(w[i]));
    if (h) h[(size_t)m * d + i] = o;
    if (cm >= 0) h_compact[(size_t)cm * d + i] = o;
  }
  cluster.sync();
}

__global__ void epi_swiglu_kernel(PartialView v, int ff, __nv_bfloat16* __restrict__ act) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ff) return;
  const int b = i >> 6, r = i & 63;
  const float g = partial_sum(v, m, b * 128 + r);
  const float u = partial_sum(v, m, b * 128 + 64 + r);
  const float s = g / (1.0f + expf(-g));
  act[(size_t)m * ff + i] = f2bf(s * u);
}

// grid (M, H + 2*Hk), block Dh/2: thread i rotates dims (i, i + Dh/2) of one head
__global__ void epi_qkv_rope_kernel(PartialView v, int H, int Hk, int Dh, RowInfo rows, const float2* __restrict__ rope,
                                    int layer, KVLayout kv, __nv_bfloat16* __restrict__ q_out,
                                    __nv_bfloat16* __restrict__ k_dbg, __nv_bfloat16* __restrict__ v_dbg) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x, head = blockIdx.y, i = threadIdx.x;
  const int half = Dh >> 1;
  const int base = head * Dh;
  float a = partial_sum(v, m, base + i);
  float b = partial_sum(v, m, base + i + half);
  const int pos = rows.pos[m];
  if (head < H + Hk) {  // q or k: rotate-half RoPE
    const float2 cs = rope[(size_t)pos * half + i];
    const float ra = a * cs.x - b * cs.y;
    const float rb = b * cs.x + a * cs.y;
    a = ra;
    b = rb;
  }
  const __nv_bfloat16 ba = f2bf(a), bb = f2bf(b);
  if (head < H) {
    __nv_bfloat16* q = q_out + ((size_t)m * H + head) * Dh;
    q[i] = ba;
    q[i + half] = bb;
    return;
  }
  const int is_v = head >= H + Hk;
  const int h = head - H - (is_v ? Hk : 0);
  const int slot = rows.slot[m];
  const int page = kv.page_table[(size_t)slot * kv.max_pages + pos / kv.P];
  __nv_bfloat16* dst = kv.pool + kv.offset(page, layer, is_v, h, pos % kv.P);
  dst[i] = ba;
  dst[i + half] = bb;
  __nv_bfloat16* dbg = is_v ? v_dbg : k_dbg;
  if (dbg) {
    dbg[((size_t)m * Hk + h) * Dh + i] = ba;
    dbg[((size_t)m * Hk + h) * Dh + i + half] = bb;
  }
}

// cos/sin(pos * theta^(-2i/Dh)) computed in fp64 on the device, stored fp32
__global__ void rope_table_kernel(float2* table, int max_pos, int Dh, double theta) {
  const int half = Dh / 2;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)max_pos * half) return;
  const int pos = (int)(idx / half), i = (int)(idx % half);
  const double inv = pow(theta, -2.0 * (double)i / (double)Dh);
  double s, c;
  sincos((double)pos * inv, &s, &c);
  table[idx] = make_float2((float)c, (float)s);
}

// dense [n][Hk][Dh] K and V -> pages of `slot`, positions 0..n-1 (test / debug path)
__global__ void kv_write_dense_kernel(KVLayout kv, int layer, int slot, int n, const __nv_bfloat16* __restrict__ k,
                                      const __nv_bfloat16* __restrict__ v) {
  pdl_trigger();
  pdl_wait();
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long per_tok = (long)kv.Hk * kv.Dh;
  if (idx >= (long)n * per_tok) return;
  const int pos = (int)(idx / per_tok);
  const int h = (int)((idx % per_tok) / kv.Dh), d = (int)(idx % kv.Dh);
  const int page = kv.page_table[(size_t)slot * kv.max_pages + pos / kv.P];
  kv.pool[kv.offset(page, layer, 0, h, pos % kv.P) + d] = k[idx];
  kv.pool[kv.offset(page, layer, 1, h, pos % kv.P) + d] = v[idx];
}

}  // namespace

cudaError_t epi_store(const PartialView& v, int N, float* Y, int ldY, const int32_t* row_map, int M, cudaStream_t st) {
  return launch(epi_store_kernel, dim3((N + 255) / 256, M), dim3(256), 0, st, v, N, Y, ldY, row_map);
}

cudaError_t embed_rmsnorm(const __nv_bfloat16* embed, const int32_t* tok, int tok_stride, int M, int d,
                          const __nv_bfloat16* w, float eps, float* x, __nv_bfloat16* h, cudaStream_t st) {
  return launch(embed_rmsnorm_kernel, dim3(M), dim3(NORM_THREADS), 0, st, embed, tok, tok_stride, d, w, eps, x, h);
}

cudaError_t epi_qkv_rope(const PartialView& v, int M, int H, int Hk, int Dh, const RowInfo& rows, const float2* rope,
                         int layer, const KVLayout& kv, __nv_bfloat16* q_out, __nv_bfloat16* k_dbg,
                         __nv_bfloat16* v_dbg, cudaStream_t st) {
  return launch(epi_qkv_rope_kernel, dim3(M, H + 2 * Hk), dim3(Dh / 2), 0, st, v, H, Hk, Dh, rows, rope, layer, kv,
                q_out, k_dbg, v_dbg);
}

cudaError_t epi_residual_rmsnorm(const PartialView& v, int M, int d, float* x, const __nv_bfloat16* w, float eps,
                                 __nv_bfloat16* h, const int32_t* compact_map, __nv_bfloat16* h_compact,
                                 cudaStream_t st) {
  return launch(residual_rmsnorm_kernel, dim3(M * RCS), dim3(RN_THREADS), 0, st, v, d, x, w, eps, h, compact_map,
                h_compact);
}

cudaError_t epi_swiglu(const PartialView& v, int M, int ff, __nv_bfloat16* act, cudaStream_t st) {
  return launch(epi_swiglu_kernel, dim3((ff + 255) / 256, M), dim3(256), 0, st, v, ff, act);
}

cudaError_t rmsnorm_rows(const float* x, int M, int d, const __nv_bfloat16* w, float eps, __nv_bfloat16* h,
                         cudaStream_t st) {
  PartialView none{nullptr, nullptr, 0, M};
  return launch(residual_rmsnorm_kernel, dim3(M * RCS), dim3(RN_THREADS), 0, st, none, d, const_cast<float*>(x), w,
                eps, h, (const int32_t*)nullptr, (__nv_bfloat16*)nullptr);
}

cudaError_t kv_write_dense(const KVLayout& kv, int layer, int slot, int n, const __nv_bfloat16* k,
                           const __nv_bfloat16* v, cudaStream_t st) {
  const long tot = (long)n * kv.Hk * kv.Dh;
  if (tot == 0) return cudaSuccess;
  return launch(kv_write_dense_kernel, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, kv, layer, slot, n, k, v);
}

cudaError_t rope_table_init(float2* table, int max_pos, int Dh, double theta, cudaStream_t st) {
  const long n = (long)max_pos * (Dh / 2);
  rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(table, max_pos, Dh, theta);
  return cudaGetLastError();
}

}  // namespace seed
