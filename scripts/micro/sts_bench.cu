// Shared-memory store throughput of the GEMM epilogue's staging pattern (4 warps, thread nl writes
// column nl of rows 0..M-1 of an fp32 [M][128] tile): cycles per CTA, one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(192, 1) sts_kernel(int M, int reps, long long* out, float* sink) {
  extern __shared__ float sf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) return;
  const int nl = (warp & 3) * 32 + lane;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = nl * 0.5f + i;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int m0 = 0; m0 < M; m0 += 32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int m = m0 + i;
        if (m < M) sf[m * 128 + nl] = v[i] + r;
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 64 && blockIdx.x == 0) out[0] = (t1 - t0) / reps;
  if (sf[(threadIdx.x * 7) % (M * 128)] == 12345.f) sink[0] = 1;
}
int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 4);
  cudaFuncSetAttribute(sts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  for (int M : {16, 64, 120, 128}) {
    for (int grid : {1, 148}) {
      sts_kernel<<<grid, 192, 180 * 1024>>>(M, 100, d, s);
      long long c;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("M=%d grid=%d: %lld cycles per staging pass (%.2f us at 1.965 GHz), %.1f B/cycle\n", M, grid, c,
             c / 1965.0, M * 128 * 4.0 / c);
    }
  }
  return 0;
}
