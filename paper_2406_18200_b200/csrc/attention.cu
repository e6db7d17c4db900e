// attention.cu -- K3: the QKV epilogue, causal attention over the paged KV cache, and the
// split-KV merge, fused in one kernel.
//
// For each sequence of the ragged batch, rows q_start .. q_start + q_len - 1 sit at positions
// kv_len - q_len .. kv_len - 1 and attend to keys 0 .. pos (R15: causal MHA).  One CTA of 4
// warps owns (sequence x 16-row query block, head, 128-key chunk):
//   * it reads the QKV GEMM's fp32 output for its query rows, applies RoPE and rounds Q to bf16
//     (B2) -- no separate epilogue kernel;
//   * cached keys/values stream into shared memory with cp.async; the new rows' K (RoPE) and V
//     are formed from the QKV output straight into the tiles and appended to the cache pages
//     (one writer per position);
//   * warp w owns the 32-key tile c_begin + 32 w: S = Q K^T and O = P V run as bf16
//     mma.sync.m16n8k16 tiles (Q padded to 16 rows; ldmatrix from padded, conflict-free tiles;
//     P re-packed from the S accumulators as the A operand, B5);
//   * the 4 warps merge (m, l, O) in a fixed order; with several chunks the last CTA of a
//     (sequence block, head) to finish (atomic ticket) merges the chunk partials in chunk
//     order; the output is rounded to bf16 (B3).
// The chunk grid is fixed (128 keys), so a row's result never depends on the batch (R19).
// Memory-bound on the cached K/V.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace seed {

namespace {
constexpr int WARPS = 4;
constexpr int CHUNK = WARPS * 32;        // keys per CTA
constexpr int QB = 16;                   // query rows per CTA (one m16 MMA tile)

// KV1 = false: K and V tiles resident together (64 KB at Dh = 128, three CTAs per SM).
// KV1 = true (blocks of <= 8 query rows): one tile buffer, K first, then V into the same buffer
// after the scores -- half the shared memory, five CTAs per SM; the arithmetic is identical.
template <int DH, bool KV1 = false>
struct Smem {
  static constexpr int PITCH = DH + 8;   // bf16 row pitch of Q (16-byte pad: conflict-free ldmatrix)
  static constexpr int RB = (DH >= 64 ? 64 : DH) * 2;   // bytes per swizzled K/V row segment (<= 128)
  static constexpr int OP = DH + 4;      // fp32 row pitch of the warp-merge scratch (conflict-free float2)
  static constexpr int QR = KV1 ? 8 : QB;  // query rows a block may hold
  static constexpr size_t TILE = (size_t)32 * DH * 2;                 // one warp's 32 K (or V) rows
  static constexpr size_t K = 0;                                      // bf16 [WARPS] tiles, 128B swizzle
  static constexpr size_t V = KV1 ? K : K + WARPS * TILE;
  static constexpr size_t Q = V + WARPS * TILE;                       // bf16 [16][PITCH]
  static constexpr size_t OWN = Q + (size_t)QB * PITCH * 2;          // KV1: fp32 [QR][DH] reducer's own o,
                                                                     // own max / sum [2][QB], others [splits][QB][2]
  static constexpr size_t ML = KV1 ? OWN + (size_t)QR * DH * 4 + 2 * QB * 4 : OWN;
  static constexpr size_t TK = ML + (size_t)(3 * WARPS + 2) * QB * 4; // ticket
  static constexpr size_t BAR = TK + 16;                             // mbarrier per warp (K / V tile)
  static constexpr size_t OML = BAR + WARPS * 8;                      // KV1: other chunks' (max, sum)
  static size_t bytes(int splits) { return OML + (KV1 ? (size_t)splits * QB * 2 * 4 : 0) + 1024; }
  // KV1 = false: o merge scratch fp32 [WARPS][QB][OP], own, max / sum and others alias K|V after
  // the MMAs; KV1: only the scratch [WARPS][QR][OP] aliases the tile buffer
};

// K / V tiles hold 32 rows per warp in the TMA swizzle of their row size (RB = 128 B: 16-byte chunk
// bits [4:6] of the shared address XOR bits [7:9]; RB = 64 B: bits [4:5] XOR bits [7:8]), so page
// blocks land by one tensor copy each and ldmatrix stays conflict-free.  Byte address of element e
// of tile row `row` (tile 1024-aligned):
template <int DH>
SEED_DEV uint32_t tile_addr(uint32_t tile, int row, int e) {
  constexpr int RB = Smem<DH, false>::RB, EH = RB / 2;
  constexpr uint32_t MASK = RB == 128 ? 0x70u : 0x30u;
  const uint32_t a = tile + (uint32_t)((e / EH) * 32 * RB + row * RB + (e % EH) * 2);
  return a ^ ((a >> 3) & MASK);
}

SEED_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
SEED_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
SEED_DEV void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 2^x on the SFU (ex2.approx: ~2 ulp; the attention probabilities are rounded to bf16 anyway, B5)
SEED_DEV float exp2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SEED_DEV uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// ---- one warp's 32-key tile (keys kt .. kt + 31 of a chunk ending at c_end): S = Q K^T (two
// accumulator chains), mask, base-2 softmax -> P in s (rows g, g + 8; lane holds keys 8 nt + 2 t4, +1),
// the tile's row max and sum.  Shared by the chunk-parallel and the sequential kernel, so a chunk's
// result is bit-identical in both (R19).
template <int DH>
SEED_DEV void warp_scores(const __nv_bfloat16* q_s, uint32_t kb, int kt, int c_end, int nr, int pos0,
                          float scale, int lane, float (&s)[4][4], float* m_row, float* l_row) {
  constexpr int P = DH + 8;
  const int g = lane >> 2, t4 = lane & 3;
  float s2[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    s[j][0] = s[j][1] = s[j][2] = s[j][3] = s2[j][0] = s2[j][1] = s2[j][2] = s2[j][3] = 0.f;
  const uint32_t qa = smem_u32(q_s);
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
    uint32_t a0, a1, a2, a3;
    ldsm_x4(qa + ((lane & 15) * P + ks * 16 + (lane >> 4) * 8) * 2, a0, a1, a2, a3);
    float (*acc)[4] = (ks & 1) ? s2 : s;
#pragma unroll
    for (int nt = 0; nt < 4; nt += 2) {
      uint32_t b0, b1, b2, b3;
      const int key = nt * 8 + (lane >> 4) * 8 + (lane & 7);
      ldsm_x4(tile_addr<DH>(kb, key, ks * 16 + ((lane >> 3) & 1) * 8), b0, b1, b2, b3);
      mma_bf16(acc[nt], a0, a1, a2, a3, b0, b1);
      mma_bf16(acc[nt + 1], a0, a1, a2, a3, b2, b3);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int c = 0; c < 4; ++c) s[j][c] += s2[j][c];
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int r = g + 8 * h2;
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int key = kt + nt * 8 + 2 * t4 + c;
        const bool ok = r < nr && key < c_end && key <= pos0 + r;
        float& v = s[nt][2 * h2 + c];
        v = ok ? v * scale : -INFINITY;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    float sum = 0.f;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float& v = s[nt][2 * h2 + c];
        v = (mx == -INFINITY) ? 0.f : exp2_approx(v - mx);
        sum += v;
      }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    m_row[h2] = mx;
    l_row[h2] = sum;
  }
}

// ---- O += P V for the tile: P (bf16, B5) re-packed from the score accumulators; V via ldmatrix.trans
template <int DH>
SEED_DEV void warp_pv(uint32_t vb, int lane, const float (&s)[4][4], float (*o_acc)[4]) {
  constexpr int DT = DH / 8;
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {   // keys 16 kc .. 16 kc + 15
    const uint32_t pa0 = pack_bf16(s[2 * kc][0], s[2 * kc][1]);
    const uint32_t pa1 = pack_bf16(s[2 * kc][2], s[2 * kc][3]);
    const uint32_t pa2 = pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]);
    const uint32_t pa3 = pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
    for (int dt = 0; dt < DT; dt += 2) {
      uint32_t b0, b1, b2, b3;
      const int key = kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int dim = dt * 8 + (lane >> 4) * 8;
      ldsm_x4_t(tile_addr<DH>(vb, key, dim), b0, b1, b2, b3);
      mma_bf16(o_acc[dt], pa0, pa1, pa2, pa3, b0, b1);
      mma_bf16(o_acc[dt + 1], pa0, pa1, pa2, pa3, b2, b3);
    }
  }
}

template <int DH, bool KV1>
// minimum CTAs per SM = what shared memory allows (caps the registers accordingly; the
// single-buffer form at Dh = 128 spills ~140 bytes at five per SM and is still faster: 55 vs 59 us
// per layer at N = 24)
__global__ void __launch_bounds__(WARPS * 32, KV1 ? 5 : (DH >= 128 ? 3 : 4))
attn_fused_kernel(const __grid_constant__ CUtensorMap tmKV, const float* __restrict__ qkv, int H, int Hk,
                  SeqInfo seqs, const float2* __restrict__ rope, KVLayout kv, int layer, int n_qblk, float scale,
                  AttnWorkspace ws, int M, __nv_bfloat16* __restrict__ out, int clustered) {
  using L = Smem<DH, KV1>;
  constexpr int QR = L::QR;
  constexpr int P = L::PITCH;
  constexpr int OP = L::OP;
  constexpr int HALF = DH / 2;
  constexpr int NT = WARPS * 32;
  constexpr int DT = DH / 8;             // 8-dim n-tiles of the output
  constexpr int EH = L::RB / 2;          // elements per swizzled row segment (TMA box width)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __nv_bfloat16* q_s = reinterpret_cast<__nv_bfloat16*>(smem + L::Q);
  __nv_bfloat16* k_s = reinterpret_cast<__nv_bfloat16*>(smem + L::K);
  __nv_bfloat16* v_s = reinterpret_cast<__nv_bfloat16*>(smem + L::V);
  float* m_s = reinterpret_cast<float*>(smem + L::ML);
  float* l_s = m_s + WARPS * QB;
  float* o_s = reinterpret_cast<float*>(smem + L::K);
  float* fw_s = l_s + WARPS * QB;                 // [WARPS][QB] warp merge factors
  float* rm_s = fw_s + WARPS * QB;                // [QB] row max, then row sum
  float* rl_s = rm_s + QB;
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::BAR);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmKV);
    for (int w = 0; w < WARPS; ++w) mbar_init(&bar_s[w], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  if (ws.timing && threadIdx.x == 0) atomicMin(&ws.timing[0], globaltimer_ns());
  unsigned long long* ct =
      ws.cta ? ws.cta + 8 * (size_t)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) : nullptr;
  auto stamp = [&](int k) {
    if (ct && threadIdx.x == 0) ct[k] = globaltimer_ns();
  };
  stamp(0);
  const int seq = blockIdx.x / n_qblk, qb = blockIdx.x % n_qblk;
  const int head = blockIdx.y, split = blockIdx.z, nsplit = gridDim.z;
  const int kvh = head / (H / Hk);
  // the descriptors were uploaded before the round's first kernel: safe before pdl_wait()
  const int q0 = seqs.q_start[seq], ql = seqs.q_len[seq], kvl = seqs.kv_len[seq];
  const int slot = seqs.slot[seq];
  const int r0 = qb * QB;
  const bool active = r0 < ql;                     // this query block holds rows of the sequence
  const int nr = min(QB, ql - r0);
  const int new_first = kvl - ql;                  // position of the sequence's first new row
  const int pos0 = new_first + r0;                 // position of the first row of this block
  const int key_end = pos0 + nr;                   // keys [0, key_end) are visible to some row
  const int c_begin = split * CHUNK;
  const int c_end = min(c_begin + CHUNK, key_end);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;          // MMA fragment coordinates
  const size_t ws_row = (size_t)(q0 + r0);
  const int ldq = (H + 2 * Hk) * DH;               // row stride of the QKV GEMM output
  const bool has_keys = active && c_begin < key_end;
  // ---- cached keys of this warp's 32-key tile: one 2D tensor copy (TMA) per page block of BR
  // rows, K and V, each 64-dim half, completing on the warp's mbarrier.  Blocks whose rows were all
  // written before this round (< `stable`) are requested while the predecessor (the QKV GEMM)
  // still runs; the rest after the dependency wait.  Rows of a block past the cached keys are
  // rewritten below (new keys, or zero past the chunk) once the copies landed.
  const int kt = c_begin + warp * 32;
  const int old_end = min(c_end, new_first);
  const int stable = seqs.stable ? min(seqs.stable[seq], old_end) : 0;
  const int BR = min(kv.P, 32);                    // rows per tensor copy (a page, or 32 of it)
  const uint32_t kw = smem_u32(k_s) + (uint32_t)(warp * L::TILE);
  const uint32_t vw = smem_u32(v_s) + (uint32_t)(warp * L::TILE);
  // page of block b in lane b (page-table rows are uploaded before the round: safe before the
  // PDL wait), all blocks' loads in flight together
  int pg = 0;
  if (has_keys && lane < 32 / BR && kt + lane * BR < old_end)
    pg = __ldg(kv.page_table + (size_t)slot * kv.max_pages + (kt + lane * BR) / kv.P);
  // pre: blocks written before the round (-1: every block); which: 1 K, 2 V, 3 both
  auto copy_blocks = [&](int pre, int which) {     // whole warp; lane 0 issues
    for (int b = 0; b < 32 / BR; ++b) {
      const int k0 = kt + b * BR;
      const int page = __shfl_sync(0xffffffffu, pg, b);
      if (k0 >= old_end || (pre >= 0 && (k0 + BR <= stable) != (pre == 1)) || lane != 0) continue;
      const int row = (((page * kv.n_layers + layer) * 2) * kv.Hk + kvh) * kv.P + (k0 % kv.P);
#pragma unroll
      for (int h = 0; h < DH / EH; ++h) {
        const uint32_t o = (uint32_t)(h * 32 * L::RB + b * BR * L::RB);
        if (which & 1) tma_load_2d_u32(kw + o, &tmKV, &bar_s[warp], h * EH, row);
        if (which & 2) tma_load_2d_u32(vw + o, &tmKV, &bar_s[warp], h * EH, row + kv.Hk * kv.P);
      }
    }
  };
  const int nblk = old_end > kt ? (min(kt + 32, old_end) - kt + BR - 1) / BR : 0;
  if (has_keys) {
    if (lane == 0) mbar_arrive_expect_tx(&bar_s[warp], (uint32_t)nblk * BR * DH * 2 * (KV1 ? 1 : 2));
    copy_blocks(1, KV1 ? 1 : 3);
  }
  pdl_wait();
  if (ws.timing && threadIdx.x == 0) atomicMin(&ws.timing[1], globaltimer_ns());
  stamp(1);
  auto done = [&]() {
    stamp(5);
    if (ws.timing && threadIdx.x == 0) {
      atomicMax(&ws.timing[2], globaltimer_ns());
      ws.timing[3] = 2;  // record kind: attention
    }
  };
  // chunks holding keys of this block: 0 .. n_ne - 1.  Outside a cluster an empty chunk has nothing
  // to publish (the merge would skip its -inf maximum anyway): it leaves at once, unless it is the
  // reducer (the last chunk of the grid)
  const int n_ne = (key_end + CHUNK - 1) / CHUNK;
  if (!active || (!clustered && !has_keys && split != nsplit - 1)) {
    done();
    return;
  }

  float o_acc[DT][4];
  float m_row[2] = {-INFINITY, -INFINITY}, l_row[2] = {0.f, 0.f};   // rows g, g + 8
#pragma unroll
  for (int j = 0; j < DT; ++j) o_acc[j][0] = o_acc[j][1] = o_acc[j][2] = o_acc[j][3] = 0.f;

  if (has_keys) {
    copy_blocks(0, KV1 ? 1 : 3);
    // ---- Q of this block's rows and head: RoPE, bf16 rounding (B2); padding rows are zero.
    // Items of 4 rotation pairs; every load of the loop is issued before the first use.
    {
      constexpr int QI = QB * HALF / 4, QIT = (QI + NT - 1) / NT;
      float4 x0[QIT], x1[QIT], c0[QIT], c1[QIT];
#pragma unroll
      for (int k = 0; k < QIT; ++k) {
        const int it = tid + k * NT, r = it / (HALF / 4), i = (it % (HALF / 4)) * 4;
        x0[k] = x1[k] = c0[k] = c1[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (it < QI && r < nr) {
          const float* yr = qkv + (size_t)(q0 + r0 + r) * ldq + head * DH;
          const float4* cs = reinterpret_cast<const float4*>(rope + (size_t)(pos0 + r) * HALF + i);
          x0[k] = *reinterpret_cast<const float4*>(yr + i);
          x1[k] = *reinterpret_cast<const float4*>(yr + i + HALF);
          c0[k] = __ldg(cs);
          c1[k] = __ldg(cs + 1);
        }
      }
#pragma unroll
      for (int k = 0; k < QIT; ++k) {
        const int it = tid + k * NT, r = it / (HALF / 4), i = (it % (HALF / 4)) * 4;
        if (it < QI) {
          // c0 = (cos_i, sin_i, cos_i+1, sin_i+1), c1 = (cos_i+2, sin_i+2, cos_i+3, sin_i+3)
          const float a0 = x0[k].x * c0[k].x - x1[k].x * c0[k].y, b0 = x1[k].x * c0[k].x + x0[k].x * c0[k].y;
          const float a1 = x0[k].y * c0[k].z - x1[k].y * c0[k].w, b1 = x1[k].y * c0[k].z + x0[k].y * c0[k].w;
          const float a2 = x0[k].z * c1[k].x - x1[k].z * c1[k].y, b2 = x1[k].z * c1[k].x + x0[k].z * c1[k].y;
          const float a3 = x0[k].w * c1[k].z - x1[k].w * c1[k].w, b3 = x1[k].w * c1[k].z + x0[k].w * c1[k].w;
          *reinterpret_cast<uint2*>(q_s + r * P + i) = make_uint2(pack_bf16(a0, a1), pack_bf16(a2, a3));
          *reinterpret_cast<uint2*>(q_s + r * P + i + HALF) = make_uint2(pack_bf16(b0, b1), pack_bf16(b2, b3));
        }
      }
    }
    // every warp's tensor copies have landed before any thread rewrites rows of the tiles
    auto rewrite_rows = [&](bool do_k, bool do_v, uint32_t parity) {
      for (int w = 0; w < WARPS; ++w) mbar_wait(&bar_s[w], parity);
      // ---- rows past the chunk: zero (each lane its own row of its warp's tiles)
      if (kt + lane >= c_end) {
#pragma unroll
        for (int e = 0; e < DH; e += 8) {
          if (do_k) st_shared_v4(tile_addr<DH>(kw, lane, e), make_uint4(0, 0, 0, 0));
          if (do_v) st_shared_v4(tile_addr<DH>(vw, lane, e), make_uint4(0, 0, 0, 0));
        }
      }
      // ---- new rows of the sequence inside this chunk: K (RoPE) and V from the QKV output into
      // the tiles; the owning query block appends them to the cache (one writer per kv head and
      // position).  Same 4-pair items, loads first.
      const int nk0 = max(c_begin, new_first), nk1 = c_end;
      const int NI = (nk1 - nk0) * (HALF / 4);
      for (int base = 0; base < NI; base += 2 * NT) {
        float4 ka[2], kb[2], va[2], vb[2], c0[2], c1[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int it = base + tid + k * NT;
          ka[k] = kb[k] = va[k] = vb[k] = c0[k] = c1[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (it < NI) {
            const int key = nk0 + it / (HALF / 4), i = (it % (HALF / 4)) * 4;
            const int m = q0 + (key - new_first);
            const float* yk = qkv + (size_t)m * ldq + (H + kvh) * DH;
            const float* yv = qkv + (size_t)m * ldq + (H + Hk + kvh) * DH;
            if (do_k) {
              const float4* cs = reinterpret_cast<const float4*>(rope + (size_t)key * HALF + i);
              ka[k] = *reinterpret_cast<const float4*>(yk + i);
              kb[k] = *reinterpret_cast<const float4*>(yk + i + HALF);
              c0[k] = __ldg(cs);
              c1[k] = __ldg(cs + 1);
            }
            if (do_v) {
              va[k] = *reinterpret_cast<const float4*>(yv + i);
              vb[k] = *reinterpret_cast<const float4*>(yv + i + HALF);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int it = base + tid + k * NT;
          if (it >= NI) continue;
          const int key = nk0 + it / (HALF / 4), i = (it % (HALF / 4)) * 4;
          const int w = (key - c_begin) >> 5, kk = (key - c_begin) & 31;
          const bool own_row = head % (H / Hk) == 0 && qb == (key - new_first) / QB;
          __nv_bfloat16* kdst = nullptr;
          if (own_row) {
            const int page = __ldg(kv.page_table + (size_t)slot * kv.max_pages + key / kv.P);
            kdst = kv.pool + kv.offset(page, layer, 0, kvh, key % kv.P);
          }
          if (do_k) {
            const float4 x0 = ka[k], x1 = kb[k];
            const uint2 klo = make_uint2(pack_bf16(x0.x * c0[k].x - x1.x * c0[k].y, x0.y * c0[k].z - x1.y * c0[k].w),
                                         pack_bf16(x0.z * c1[k].x - x1.z * c1[k].y, x0.w * c1[k].z - x1.w * c1[k].w));
            const uint2 khi = make_uint2(pack_bf16(x1.x * c0[k].x + x0.x * c0[k].y, x1.y * c0[k].z + x0.y * c0[k].w),
                                         pack_bf16(x1.z * c1[k].x + x0.z * c1[k].y, x1.w * c1[k].z + x0.w * c1[k].w));
            const uint32_t kt_w = smem_u32(k_s) + (uint32_t)(w * L::TILE);
            st_shared_v2(tile_addr<DH>(kt_w, kk, i), klo);
            st_shared_v2(tile_addr<DH>(kt_w, kk, i + HALF), khi);
            if (own_row) {
              *reinterpret_cast<uint2*>(kdst + i) = klo;
              *reinterpret_cast<uint2*>(kdst + i + HALF) = khi;
            }
          }
          if (do_v) {
            const uint2 vlo = make_uint2(pack_bf16(va[k].x, va[k].y), pack_bf16(va[k].z, va[k].w));
            const uint2 vhi = make_uint2(pack_bf16(vb[k].x, vb[k].y), pack_bf16(vb[k].z, vb[k].w));
            const uint32_t vt_w = smem_u32(v_s) + (uint32_t)(w * L::TILE);
            st_shared_v2(tile_addr<DH>(vt_w, kk, i), vlo);
            st_shared_v2(tile_addr<DH>(vt_w, kk, i + HALF), vhi);
            if (own_row) {
              *reinterpret_cast<uint2*>(kdst + kv.vofs() + i) = vlo;
              *reinterpret_cast<uint2*>(kdst + kv.vofs() + i + HALF) = vhi;
            }
          }
        }
      }
      __syncthreads();
    };
    rewrite_rows(true, !KV1, 0);
    stamp(2);

    float sc[4][4];
    if (kt < c_end) warp_scores<DH>(q_s, kw, kt, c_end, nr, pos0, scale, lane, sc, m_row, l_row);
    if (KV1) {
      // V into the buffer the scores were read from
      if (max(c_begin, new_first) < c_end) {
        // the chunk holds new keys, whose V rows every thread helps to form: every warp is done
        // with K first
        __syncthreads();
        fence_proxy_async();
        if (lane == 0) mbar_arrive_expect_tx(&bar_s[warp], (uint32_t)nblk * BR * DH * 2);
        copy_blocks(-1, 2);
        rewrite_rows(false, true, 1);
      } else {
        // only cached keys (and no rows past the chunk): a warp's K rows are read by that warp
        // alone, so each warp requests its V rows as soon as its scores are done
        __syncwarp();
        fence_proxy_async();
        if (lane == 0) mbar_arrive_expect_tx(&bar_s[warp], (uint32_t)nblk * BR * DH * 2);
        copy_blocks(-1, 2);
        mbar_wait(&bar_s[warp], 1);
      }
    }
    if (kt < c_end) warp_pv<DH>(vw, lane, sc, o_acc);
  }

  // ---- merge the 4 warps (fixed order) into this chunk's result
  __syncthreads();   // o_s aliases the K / V tiles
  if (t4 == 0) {
    m_s[warp * QB + g] = m_row[0];
    m_s[warp * QB + g + 8] = m_row[1];
    l_s[warp * QB + g] = l_row[0];
    l_s[warp * QB + g + 8] = l_row[1];
  }
  // rows g, g + 8 of the fragments (only the block's real rows), row pitch OP: conflict-free float2
  if (g < nr) {
#pragma unroll
    for (int dt = 0; dt < DT; ++dt)
      *reinterpret_cast<float2*>(o_s + ((size_t)warp * QR + g) * OP + dt * 8 + 2 * t4) =
          make_float2(o_acc[dt][0], o_acc[dt][1]);
  }
  if (!KV1 && g + 8 < nr) {
#pragma unroll
    for (int dt = 0; dt < DT; ++dt)
      *reinterpret_cast<float2*>(o_s + ((size_t)warp * QR + g + 8) * OP + dt * 8 + 2 * t4) =
          make_float2(o_acc[dt][2], o_acc[dt][3]);
  }
  __syncthreads();
  const bool single = nsplit == 1;
  // With several chunks: launched as one thread-block cluster per (sequence block, head)
  // (clustered, <= 8 chunks), every chunk keeps its result in shared memory and the cluster
  // merges through distributed shared memory; otherwise the last chunk (it holds the new keys)
  // merges from global memory after the others published theirs.
  const bool reducer = clustered || split == nsplit - 1;
  // [QR][DH] own result, [QB] own chunk max and sum, [nsplit - 1][QB][2] other chunks' (max, sum)
  float* own = KV1 ? reinterpret_cast<float*>(smem + L::OWN) : o_s + (size_t)WARPS * QB * OP;
  float* cm = own + QR * DH;
  float* cl = cm + QB;
  float* oml = KV1 ? reinterpret_cast<float*>(smem + L::OML) : cl + QB;
  // per row: the 4 warps' merge factors exp(m_w - m) and the row sum, warps in a fixed order
  if (tid < nr) {
    const int r = tid;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) mx = fmaxf(mx, m_s[w * QB + r]);
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float mw = m_s[w * QB + r];
      const float f = (mx == -INFINITY || mw == -INFINITY) ? 0.f : exp2_approx(mw - mx);
      fw_s[w * QB + r] = f;
      l += l_s[w * QB + r] * f;
    }
    rm_s[r] = mx;
    rl_s[r] = l;
    if (!single && reducer) {
      cm[r] = mx;
      cl[r] = l;
    } else if (!single) {
      float* ml = ws.ml_part + (((size_t)split * M + ws_row + r) * H + head) * 2;
      ml[0] = mx;
      ml[1] = l;
    }
  }
  __syncthreads();
  for (int e = tid; e < nr * (DH / 4); e += NT) {
    const int r = e / (DH / 4), d = (e % (DH / 4)) * 4;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float f = fw_s[w * QB + r];
      const float4 v = *reinterpret_cast<const float4*>(o_s + ((size_t)w * QR + r) * OP + d);
      o.x += v.x * f;
      o.y += v.y * f;
      o.z += v.z * f;
      o.w += v.w * f;
    }
    const size_t row = ws_row + r;
    if (single) {
      const float l = rl_s[r];
      *reinterpret_cast<uint2*>(out + (row * H + head) * DH + d) =
          make_uint2(pack_bf16(o.x / l, o.y / l), pack_bf16(o.z / l, o.w / l));
    } else if (reducer) {
      *reinterpret_cast<float4*>(own + r * DH + d) = o;
    } else {
      *reinterpret_cast<float4*>(ws.o_part + (((size_t)split * M + row) * H + head) * DH + d) = o;
    }
  }
  stamp(3);
  if (single) {
    done();
    return;
  }
  if (clustered) {
    // every rank merges a slice of the (row, 4-dim) items from all ranks' results, chunk order
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();   // release this CTA's result, acquire the peers'
    stamp(4);
    for (int e = tid + split * NT; e < nr * (DH / 4); e += NT * nsplit) {
      const int r = e / (DH / 4), d = (e % (DH / 4)) * 4;
      // every rank's (max, sum, o) loaded at once (one DSMEM round trip), then merged in rank order
      float msv[8], lsv[8];
      float4 ov[8];
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        if (sp < nsplit) {
          msv[sp] = *cluster.map_shared_rank(cm + r, sp);
          lsv[sp] = *cluster.map_shared_rank(cl + r, sp);
          ov[sp] = *reinterpret_cast<const float4*>(cluster.map_shared_rank(own + r * DH + d, sp));
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int sp = 0; sp < 8; ++sp)
        if (sp < nsplit) mx = fmaxf(mx, msv[sp]);
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
      float l = 0.f;
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        if (sp >= nsplit || msv[sp] == -INFINITY) continue;
        const float f = exp2_approx(msv[sp] - mx);
        o.x += ov[sp].x * f;
        o.y += ov[sp].y * f;
        o.z += ov[sp].z * f;
        o.w += ov[sp].w * f;
        l += lsv[sp] * f;
      }
      const size_t row = ws_row + r;
      *reinterpret_cast<uint2*>(out + (row * H + head) * DH + d) =
          make_uint2(pack_bf16(o.x / l, o.y / l), pack_bf16(o.z / l, o.w / l));
    }
    cluster_sync_relaxed();   // peers finished reading this CTA's shared memory (execution order only:
                              // the reads completed when their values were used)
    done();
    return;
  }
  int* ctr = ws.counters + ((size_t)(seq * n_qblk + qb) * H + head);
  if (!reducer) {
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel_gpu();   // release this chunk's partial (bar.sync + cumulativity)
      atomicAdd(ctr, 1);
    }
    done();
    return;
  }
  if (tid == 0) {
    volatile int* vc = ctr;
    while (*vc < min(nsplit - 1, n_ne)) {
    }
    fence_acq_rel_gpu();     // acquire the other chunks' partials
    *vc = 0;                 // ready for the next launch (graph replay)
  }
  __syncthreads();
  stamp(4);
  const int n_oth = min(nsplit - 1, n_ne);   // published chunks (the reducer's own excluded)
  for (int e = tid; e < n_oth * nr; e += NT) {
    const int sp = e / nr, r = e % nr;
    const float2 v = __ldcg(reinterpret_cast<const float2*>(ws.ml_part + (((size_t)sp * M + ws_row + r) * H + head) * 2));
    oml[(sp * QB + r) * 2] = v.x;
    oml[(sp * QB + r) * 2 + 1] = v.y;
  }
  __syncthreads();
  // chunks in chunk order 0 .. nsplit - 1 (this one last), as one fixed sum (R19); items of 4 dims
  constexpr int MI = QB * DH / 4, MIT = (MI + NT - 1) / NT;
#pragma unroll
  for (int k = 0; k < MIT; ++k) {
    const int it = tid + k * NT, r = it / (DH / 4), d = (it % (DH / 4)) * 4;
    if (it >= MI || r >= nr) continue;
    float mx = cm[r];
    for (int sp = 0; sp < n_oth; ++sp) mx = fmaxf(mx, oml[(sp * QB + r) * 2]);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.f;
    const size_t row = ws_row + r;
    for (int s0 = 0; s0 < n_oth; s0 += 4) {
      float4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = s0 + q < n_oth
                   ? __ldcg(reinterpret_cast<const float4*>(ws.o_part + (((size_t)(s0 + q) * M + row) * H + head) * DH + d))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (s0 + q >= n_oth) break;
        const float ms = oml[((s0 + q) * QB + r) * 2];
        if (ms == -INFINITY) continue;
        const float f = exp2_approx(ms - mx);
        o.x += v[q].x * f;
        o.y += v[q].y * f;
        o.z += v[q].z * f;
        o.w += v[q].w * f;
        l += oml[((s0 + q) * QB + r) * 2 + 1] * f;
      }
    }
    if (cm[r] != -INFINITY) {
      const float f = exp2_approx(cm[r] - mx);
      o.x += own[r * DH + d] * f;
      o.y += own[r * DH + d + 1] * f;
      o.z += own[r * DH + d + 2] * f;
      o.w += own[r * DH + d + 3] * f;
      l += cl[r] * f;
    }
    *reinterpret_cast<uint2*>(out + (row * H + head) * DH + d) =
        make_uint2(pack_bf16(o.x / l, o.y / l), pack_bf16(o.z / l, o.w / l));
  }
  done();
}

// env SEED_ATTN_CLUSTER: 0 global-memory merge, 1 DSMEM merge (<= 8 chunks), default: DSMEM merge
// while the grid fits one wave of three CTAs per SM -- thread-block clusters must be co-scheduled
// inside a GPC, which costs occupancy once the grid is larger (measured at N = 24 streams: 96 us
// per layer clustered vs 74 us global).  Both give identical results (R19).
int attn_cluster_mode() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("SEED_ATTN_CLUSTER");
    mode = e ? atoi(e) : -1;
  }
  return mode;
}

template <int DH, bool KV1>
cudaError_t launch_form(int M, int n_seq, int n_qblk, int splits, int H, int Hk, const CUtensorMap& tmkv,
                        const float* qkv, const SeqInfo& seqs, const float2* rope, const KVLayout& kv, int layer,
                        const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st, int clustered) {
  using L = Smem<DH, KV1>;
  const size_t smem = L::bytes(splits);
  // warp-merge scratch (and, two-tile form, the reducer's own result and every chunk's (max, sum))
  // alias the tiles
  const size_t kv_bytes = (KV1 ? 1 : 2) * WARPS * L::TILE;
  const size_t alias = KV1 ? (size_t)WARPS * L::QR * L::OP * 4
                           : ((size_t)WARPS * QB * L::OP + (size_t)QB * DH + 2 * QB + (size_t)2 * QB * splits) * 4;
  if (alias > kv_bytes || smem > 227 * 1024) return cudaErrorInvalidValue;
  static int attr = 0;
  if (attr < (int)smem) {
    cudaFuncSetAttribute(attn_fused_kernel<DH, KV1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = (int)smem;
  }
  // scores are kept in the base-2 domain: s = q.k / sqrt(Dh) * log2(e), p = 2^(s - max)
  const float scale = 1.0f / sqrtf((float)DH) * 1.4426950408889634f;
  return launch_clustered(attn_fused_kernel<DH, KV1>, dim3(n_seq * n_qblk, H, splits), dim3(WARPS * 32), smem, st,
                          dim3(1, 1, clustered ? splits : 1), tmkv, qkv, H, Hk, seqs, rope, kv, layer, n_qblk, scale,
                          ws, M, out, clustered);
}

// env SEED_ATTN_KV1: 0 never, 1 whenever possible, default: blocks of <= 8 rows and a grid beyond one
// wave of the two-tile form (results identical, R19)
int attn_kv1_mode() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("SEED_ATTN_KV1");
    mode = e ? atoi(e) : -1;
  }
  return mode;
}

template <int DH>
cudaError_t launch_dh(int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, const CUtensorMap& tmkv,
                      const float* qkv, const SeqInfo& seqs, const float2* rope, const KVLayout& kv, int layer,
                      const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st) {
  const int n_qblk = (max_q_len + QB - 1) / QB;
  const int splits = (max_kv + CHUNK - 1) / CHUNK;
  // tensor copies of whole page blocks into the swizzled tiles: blocks of >= 16 rows (1 KB atoms)
  if (kv.P < 16 || (kv.P & (kv.P - 1))) return cudaErrorInvalidValue;
  const int cm = attn_cluster_mode();
  const long ctas = (long)n_seq * n_qblk * H * splits;
  const int clustered = (splits > 1 && splits <= 8 && (cm == 1 || (cm < 0 && ctas <= 3 * kNumSMs))) ? 1 : 0;
  const int k1 = attn_kv1_mode();
  if (max_q_len <= 8 && !clustered && (k1 == 1 || (k1 < 0 && ctas > 3 * kNumSMs)))
    return launch_form<DH, true>(M, n_seq, n_qblk, splits, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st, 0);
  return launch_form<DH, false>(M, n_seq, n_qblk, splits, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st,
                                clustered);
}
}  // namespace

int attn_chunk_tokens() { return CHUNK; }
int attn_query_block() { return QB; }

bool attn_kv_tmap(CUtensorMap* map, const KVLayout& kv, size_t n_pages) {
  const uint64_t rows = (uint64_t)n_pages * kv.n_layers * 2 * kv.Hk * kv.P;
  // rows of 128 B (Dh >= 64: 64-dim halves) in the 128-byte swizzle, 64-byte rows (Dh = 32) in the 64-byte one
  return encode_tmap_2d(map, kv.pool, (uint64_t)kv.Dh, rows, (uint32_t)(kv.Dh >= 64 ? 64 : kv.Dh),
                        (uint32_t)(kv.P < 32 ? kv.P : 32), kv.Dh >= 64 ? 128 : 64);
}

cudaError_t attention(const float* qkv, int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, int Dh,
                      const SeqInfo& seqs, const float2* rope, const KVLayout& kv, const CUtensorMap& tmkv, int layer,
                      const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st) {
  const int splits = (max_kv + CHUNK - 1) / CHUNK;
  if (splits > ws.max_splits) return cudaErrorInvalidValue;
  if ((size_t)n_seq * ((max_q_len + QB - 1) / QB) * H > (size_t)ws.max_counters) return cudaErrorInvalidValue;
  if (Dh == 128) return launch_dh<128>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  if (Dh == 64) return launch_dh<64>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  if (Dh == 32) return launch_dh<32>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  return cudaErrorInvalidValue;
}

}  // namespace seed
