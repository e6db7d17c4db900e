// epilogue.cu -- the small kernels left around the projections: embedding + row statistics,
// the RoPE table, and a dense-KV writer for tests.
//
// Everything else between the projections is fused (DESIGN "kernels"): the residual adds and
// the per-tile sums of squares run in the O / down GEMM epilogues, RMSNorm and SwiGLU in the
// X-producer of the next GEMM, the QKV epilogue in the attention kernel.
#include "common.cuh"
#include "kernels.h"

namespace seed {

namespace {

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

// x[m] = embed[tok[m]] (fp32, exact) -- or x given -- and the per-128-column-tile sums of
// squares ssq[t][m] and h = bf16(x * nw) the next GEMM consumes (RMSNorm scale 1/rms applied
// in its epilogue, R24).  grid (ceil(d / 1024), M), 128 threads: a CTA covers eight 128-column
// tiles of one row, every load issued before the first use, one barrier.
constexpr int EMB_TILES = 8;
__global__ void __launch_bounds__(128)
embed_stats_kernel(const __nv_bfloat16* __restrict__ embed, const int32_t* __restrict__ tok, int tok_stride, int d,
                   int V, float* __restrict__ x, float* __restrict__ ssq, const __nv_bfloat16* __restrict__ nw,
                   __nv_bfloat16* __restrict__ h, int32_t* err, int M, unsigned long long* rec) {
  __shared__ float red[EMB_TILES][4];
  pdl_trigger();
  rec_start(rec);
  pdl_wait();
  rec_release(rec);
  const int m = blockIdx.y, t0 = blockIdx.x * EMB_TILES, tid = threadIdx.x;
  int id = 0;
  if (embed) {
    id = tok[(size_t)m * tok_stride];
    if (id < 0 || id >= V) {   // contract violation (SEED_EDEVICE): never read outside the table
      if (err && tid == 0 && blockIdx.x == 0) atomicOr(err, 1);
      id = 0;
    }
  }
  float v[EMB_TILES];
#pragma unroll
  for (int k = 0; k < EMB_TILES; ++k) {
    const int n = (t0 + k) * 128 + tid;
    v[k] = 0.f;
    if (n < d) v[k] = embed ? bf2f(embed[(size_t)id * d + n]) : x[(size_t)m * d + n];
  }
#pragma unroll
  for (int k = 0; k < EMB_TILES; ++k) {
    const int n = (t0 + k) * 128 + tid;
    if (n < d) {
      if (embed) x[(size_t)m * d + n] = v[k];
      if (h) h[(size_t)m * d + n] = f2bf(v[k] * bf2f(nw[n]));
    }
    const float sq = warp_sum(v[k] * v[k]);
    if ((tid & 31) == 0) red[k][tid >> 5] = sq;
  }
  __syncthreads();
  const int nt = (d + 127) / 128;
  if (tid < EMB_TILES && t0 + tid < nt)
    ssq[(size_t)(t0 + tid) * M + m] = ((red[tid][0] + red[tid][1]) + red[tid][2]) + red[tid][3];
  rec_end(rec, 5);
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

// one block per (stream, layer x K|V x kv head); threads over the head dim
__global__ void kv_compact_kernel(KVLayout kv, const int32_t* __restrict__ slots, const int32_t* __restrict__ tlen,
                                  const int32_t* __restrict__ node, int node_stride, int max_depth,
                                  unsigned long long* rec) {
  pdl_trigger();
  rec_start(rec);
  pdl_wait();
  rec_release(rec);
  const int b = blockIdx.x;
  const int lkh = blockIdx.y;                       // (layer * 2 + kv) * Hk + h
  const int h = lkh % kv.Hk, lk = lkh / kv.Hk, layer = lk / 2, which = lk % 2;
  const int slot = slots[b];
  const int root = tlen[slot] - 1;
  const int32_t* pt = kv.page_table + (size_t)slot * kv.max_pages;
  for (int d = 1; d <= max_depth; ++d) {
    const int nd = node[(size_t)b * node_stride + d - 1];
    if (nd < 0) break;
    if (nd == d) continue;
    const int src = root + nd, dst = root + d;
    const __nv_bfloat16* s = kv.pool + kv.offset(pt[src / kv.P], layer, which, h, src % kv.P);
    __nv_bfloat16* t = kv.pool + kv.offset(pt[dst / kv.P], layer, which, h, dst % kv.P);
    for (int e = threadIdx.x; e < kv.Dh / 2; e += blockDim.x)
      reinterpret_cast<uint32_t*>(t)[e] = reinterpret_cast<const uint32_t*>(s)[e];
  }
  rec_end(rec, 7);
}

}  // namespace

cudaError_t kv_compact(const KVLayout& kv, const int32_t* slots, const int32_t* tlen, const int32_t* node,
                       int node_stride, int max_depth, int B, cudaStream_t st, unsigned long long* timing) {
  if (B <= 0 || max_depth <= 0) return cudaSuccess;
  return launch(kv_compact_kernel, dim3(B, kv.n_layers * 2 * kv.Hk), dim3(64), 0, st, kv, slots, tlen, node,
                node_stride, max_depth, timing);
}

cudaError_t embed_stats(const __nv_bfloat16* embed, const int32_t* tok, int tok_stride, int M, int d, int V, float* x,
                        float* ssq, const __nv_bfloat16* nw, __nv_bfloat16* h, int32_t* err, cudaStream_t st,
                        unsigned long long* timing) {
  const int nt = (d + 127) / 128;
  return launch(embed_stats_kernel, dim3((nt + EMB_TILES - 1) / EMB_TILES, M), dim3(128), 0, st, embed, tok, tok_stride,
                d, V, x, ssq, nw, h, err, M, timing);
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
