// Microbenchmark: cost of the split-K publish / reduce chain on B200 (diagnostics only).
// 148 CTAs x 128 threads; groups of G CTAs share a "tile"; CTA 0 of a group reduces.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
  return t;
}

__global__ void tail_kernel(float* part, int* counters, float* out, unsigned long long* ts, int G, int mode,
                            const float* warm) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const int grp = c / G, r = c % G;
  unsigned long long* T = ts + c * 8;
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = (float)(c * 16 + i + tid);
  if (tid == 0) T[0] = gt();
  if (r != 0) {
    float* dst = part + (size_t)c * 16 * 128 + tid;
    for (int i = 0; i < 16; ++i) dst[i * 128] = v[i];
    if (tid == 0) T[1] = gt();
    __syncthreads();
    if (tid == 0) {
      if (mode == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(&counters[grp], 1);
      } else {
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&counters[grp]) : "memory");
      }
      T[2] = gt();
    }
  } else {
    // baseline: latency of loading 16 L2-resident values (warm buffer written by the host)
    float w[16];
    unsigned long long a = gt();
    for (int i = 0; i < 16; ++i) w[i] = __ldcg(warm + (size_t)c * 16 * 128 + i * 128 + tid);
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += w[i];
    unsigned long long b = gt() + (s == 1.2345f ? 1 : 0);
    if (tid == 0) { T[1] = a; T[2] = b; }
    if (tid == 0) {
      volatile int* ctr = counters + grp;
      while (*ctr < G - 1) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      *ctr = 0;
      T[3] = gt();
    }
    __syncthreads();
    float acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = v[i];
    for (int k = 1; k < G; ++k) {
      const float* src = part + (size_t)(c + k) * 16 * 128 + tid;
      for (int i = 0; i < 16; ++i) acc[i] += __ldcg(src + i * 128);
    }
    float s2 = 0.f;
    for (int i = 0; i < 16; ++i) s2 += acc[i];
    if (tid == 0) T[4] = gt() + (s2 == 1.2345f ? 1 : 0);
    for (int i = 0; i < 16; ++i) out[(size_t)c * 16 * 128 + i * 128 + tid] = acc[i];
    if (tid == 0) T[5] = gt();
  }
}

int main() {
  const int N = 148;
  float *part, *out, *warm;
  int* counters;
  unsigned long long* ts;
  cudaMalloc(&part, N * 16 * 128 * 4);
  cudaMalloc(&out, N * 16 * 128 * 4);
  cudaMalloc(&warm, N * 16 * 128 * 4);
  cudaMemset(warm, 0, N * 16 * 128 * 4);
  cudaMalloc(&counters, N * 4);
  cudaMemset(counters, 0, N * 4);
  cudaMalloc(&ts, N * 8 * 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int G : {2, 5, 8}) {
      std::vector<double> pub, spin, red, base;
      for (int it = 0; it < 20; ++it) {
        cudaMemset(ts, 0, N * 64);
        tail_kernel<<<N / G * G, 128>>>(part, counters, out, ts, G, mode, warm);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(N * 8);
        cudaMemcpy(h.data(), ts, N * 64, cudaMemcpyDeviceToHost);
        if (it < 5) continue;
        for (int c = 0; c < N / G * G; ++c) {
          auto* T = &h[c * 8];
          if (c % G) pub.push_back((T[2] - T[1]) / 1e3);
          else {
            base.push_back((T[2] - T[1]) / 1e3);
            red.push_back((T[4] - T[3]) / 1e3);
            unsigned long long last = 0;
            for (int k = 1; k < G; ++k) last = std::max(last, h[(c + k) * 8 + 2]);
            spin.push_back(((double)T[3] - (double)last) / 1e3);
          }
        }
      }
      auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
      auto mx = [](std::vector<double> v) { return *std::max_element(v.begin(), v.end()); };
      printf("mode %d G %d: publish(fence+atomic) med %.2f max %.2f | flag seen after last publish med %.2f max %.2f |"
             " reduce loads med %.2f max %.2f | warm L2 16 loads med %.2f us\n",
             mode, G, med(pub), mx(pub), med(spin), mx(spin), med(red), mx(red), med(base));
    }
  return 0;
}
