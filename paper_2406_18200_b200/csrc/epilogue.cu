// epilogue.cu -- the small kernels between the projections: embedding + RMSNorm, residual +
// RMSNorm, SwiGLU, and the RoPE table.
//
// They consume the GEMMs' final fp32 outputs Y (split-K already reduced inside the GEMM in a
// fixed order, R19) and store bf16 exactly where DESIGN.md "bf16 rounding points" says:
//   O / down -> residual add (fp32, F1) -> RMSNorm(mlp_norm / next attn_norm / final_norm) -> bf16 (B1)
//   gate/up (interleaved 64-row blocks) -> silu(g) * u -> bf16 operand of down (B4)
//   QKV -> fused into the attention kernel (attention.cu); LM head -> logits written by the GEMM (F2)
// Every kernel launches with PDL: it becomes resident while its predecessor runs and waits
// in pdl_wait(); they are small enough (threads, registers, no dynamic smem) to sit next to a
// running GEMM CTA.
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

constexpr int NT = 512;  // threads per row
constexpr int CPT = 10;  // columns per thread held in registers (d <= 5120)

// x[m] (+)= Y[m]; h = bf16(rmsnorm(x[m]) * w); one CTA per row, fixed-order reduction
__global__ void __launch_bounds__(NT)
residual_rmsnorm_kernel(const float* __restrict__ Y, int d, float* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                        float eps, __nv_bfloat16* __restrict__ h, const int32_t* __restrict__ compact_map,
                        __nv_bfloat16* __restrict__ h_compact) {
  __shared__ float red[NT / 32];
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  float* xr = x + (size_t)m * d;
  const float* yr = Y ? Y + (size_t)m * d : nullptr;
  float vals[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = threadIdx.x + k * NT;
    vals[k] = 0.f;
    if (i < d) vals[k] = xr[i] + (yr ? yr[i] : 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = threadIdx.x + k * NT;
    if (i < d) {
      if (yr) xr[i] = vals[k];
      ss += vals[k] * vals[k];
    }
  }
  const float tot = block_sum<NT>(ss, red);
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  const int cm = compact_map ? compact_map[m] : -1;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = threadIdx.x + k * NT;
    if (i < d) {
      const __nv_bfloat16 o = f2bf(vals[k] * inv * bf2f(w[i]));
      if (h) h[(size_t)m * d + i] = o;
      if (cm >= 0) h_compact[(size_t)cm * d + i] = o;
    }
  }
}

__global__ void __launch_bounds__(NT)
embed_rmsnorm_kernel(const __nv_bfloat16* __restrict__ embed, const int32_t* __restrict__ tok, int tok_stride, int d,
                     const __nv_bfloat16* __restrict__ w, float eps, float* __restrict__ x,
                     __nv_bfloat16* __restrict__ h) {
  __shared__ float red[NT / 32];
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const __nv_bfloat16* e = embed + (size_t)tok[(size_t)m * tok_stride] * d;
  float vals[CPT];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = threadIdx.x + k * NT;
    vals[k] = i < d ? bf2f(e[i]) : 0.f;
    if (i < d) x[(size_t)m * d + i] = vals[k];
    ss += vals[k] * vals[k];
  }
  const float tot = block_sum<NT>(ss, red);
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int i = threadIdx.x + k * NT;
    if (i < d) h[(size_t)m * d + i] = f2bf(vals[k] * inv * bf2f(w[i]));
  }
}

__global__ void swiglu_kernel(const float* __restrict__ Y, int ff, __nv_bfloat16* __restrict__ act) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ff) return;
  const int b = i >> 6, r = i & 63;
  const float* yr = Y + (size_t)m * 2 * ff;
  const float g = yr[b * 128 + r];
  const float u = yr[b * 128 + 64 + r];
  const float s = g / (1.0f + expf(-g));
  act[(size_t)m * ff + i] = f2bf(s * u);
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

cudaError_t embed_rmsnorm(const __nv_bfloat16* embed, const int32_t* tok, int tok_stride, int M, int d,
                          const __nv_bfloat16* w, float eps, float* x, __nv_bfloat16* h, cudaStream_t st) {
  if (d > NT * CPT) return cudaErrorInvalidValue;
  return launch(embed_rmsnorm_kernel, dim3(M), dim3(NT), 0, st, embed, tok, tok_stride, d, w, eps, x, h);
}

cudaError_t residual_rmsnorm(const float* Y, int M, int d, float* x, const __nv_bfloat16* w, float eps,
                             __nv_bfloat16* h, const int32_t* compact_map, __nv_bfloat16* h_compact,
                             cudaStream_t st) {
  if (d > NT * CPT) return cudaErrorInvalidValue;
  return launch(residual_rmsnorm_kernel, dim3(M), dim3(NT), 0, st, Y, d, x, w, eps, h, compact_map, h_compact);
}

cudaError_t swiglu(const float* Y, int M, int ff, __nv_bfloat16* act, cudaStream_t st) {
  return launch(swiglu_kernel, dim3((ff + 255) / 256, M), dim3(256), 0, st, Y, ff, act);
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
