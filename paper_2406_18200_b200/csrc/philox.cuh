// philox.cuh -- K7: Philox4x32-10 (Salmon et al. SC'11) and the odd-grid uniform (R2, R5, R17).
//
// Counter layout (R5): c0 = draw block, c1 = tag << 24 | slot, c2 = stream-local round,
// c3 = global stream id; key = (lo32(seed), hi32(seed)).  u = (2*(x >> 9) + 1) * 2^-24.
#pragma once
#include <stdint.h>

namespace seed {

enum : uint32_t { kTagDraft = 1, kTagAccept = 2, kTagResample = 3 };

struct Philox4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// exact in fp32 and fp64: (2k + 1) / 2^24, k = x >> 9
__device__ __forceinline__ double philox_uniform(uint32_t x) {
  return (double)(2u * (x >> 9) + 1u) * (1.0 / 16777216.0);
}

}  // namespace seed
