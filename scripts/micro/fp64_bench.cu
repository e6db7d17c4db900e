// Latency / throughput of the fp64 transcendentals the races use, one warp vs a full CTA.
#include <cstdio>
__global__ void k(int mode, int n, double* out, long long* cyc) {
  double x = 0.3 + threadIdx.x * 1e-6, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (mode == 0) x = -log(-log1p(-x * 0.5)) * 1e-3 + 0.3;
    else if (mode == 1) x = log(x + 1.0) * 0.5 + 0.1;
    else if (mode == 2) x = x * 1.0000001 + 1e-9;
    else x = (double)(-__logf(-log1pf(-(float)x * 0.5f))) * 1e-3 + 0.3;
    acc += x;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / n;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 148 * 256 * 8);
  cudaMalloc(&c, 148 * 8);
  const char* nm[] = {"fp64 -log(-log1p(-u))", "fp64 log", "fp64 fma", "fp32 screen"};
  for (int mode = 0; mode < 4; ++mode)
    for (int th : {32, 256}) {
      k<<<1, th>>>(mode, 200, o, c);
      long long v;
      cudaMemcpy(&v, c, 8, cudaMemcpyDeviceToHost);
      printf("%-24s threads %3d: %5lld cycles per dependent call\n", nm[mode], th, v);
    }
  return 0;
}
