// Compute cost of the vocabulary building blocks (vocab_common.cuh) on one 4000-element slice in
// shared memory, 256 threads: slice_stat, and the exponential race (bonus form: fp32 keys; residual
// form: near-equal p, q through the fp64 path, or well separated).  Cycles per call, one CTA per SM.
#include <cstdio>
#include "vocab_common.cuh"
using namespace seed;
using namespace seed::vocab;
__global__ void __launch_bounds__(VT) race_bench(int mode, int reps, long long* out, int* sink) {
  extern __shared__ float sm[];
  __shared__ float red_f[VT / 32];
  __shared__ MaxI red_m[VT / 32];
  __shared__ double red_d[VT / 32];
  __shared__ Best red_b[VT / 32];
  const int n = 4000;
  float* zt = sm;
  float* zd = sm + n;
  float* keys = sm + 2 * n;
  for (int l = threadIdx.x; l < n; l += VT) {
    const float x = 0.001f * (float)((l * 7919) % 1000);
    zt[l] = x;
    zd[l] = mode == 2 ? x + 0.3f * (float)(((l * 31) % 7) - 3) : x + 1e-3f * (float)((l * 13) % 5);
  }
  __syncthreads();
  long long t0 = clock64();
  int acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) {
      const SliceStat s = slice_stat(zt, 0, n, 1.0f, red_m, red_d);
      acc += s.i;
    } else {
      const float mt = 1.0f, l1t = 10.3f, mq = 1.0f, l1q = 10.31f;
      auto w32 = [&](int l) -> float {
        if (mode == 3) return zt[l];
        const double d = ((double)zd[l] - (double)zt[l]) - ((double)(mq + l1q) - (double)(mt + l1t));
        if (d > -1e-12) return d >= 1e-12 ? -INFINITY : NAN;
        return ((zt[l] - mt) - l1t) + __logf(-expm1f((float)d));
      };
      auto w64 = [&](int l) -> double {
        if (mode == 3) return (double)zt[l];
        const double lp = ((double)zt[l] - mt) - l1t, lq = ((double)zd[l] - mq) - l1q;
        return lq < lp ? lp + log(-expm1(lq - lp)) : -INFINITY;
      };
      const Best b = race_slice(0, n, 0x03000001u, (uint32_t)r, 12345u, 0x5EED2406u, 0u, keys, red_f, red_b, w32, w64);
      acc += b.v;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = (t1 - t0) / reps;
    sink[blockIdx.x] = acc;
  }
}
int main() {
  long long* d;
  int* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 148 * 4);
  cudaFuncSetAttribute(race_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4000 * 4);
  const char* names[] = {"slice_stat", "race residual near-equal (fp64 path)", "race residual separated", "race bonus"};
  for (int mode = 0; mode < 4; ++mode)
    for (int grid : {1, 148}) {
      race_bench<<<grid, VT, 3 * 4000 * 4>>>(mode, 20, d, s);
      long long c;
      cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      printf("%-40s grid %3d: %8lld cycles per call (%.2f us)\n", names[mode], grid, c, c / 1965.0);
    }
  return 0;
}
