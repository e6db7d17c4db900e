// attention.cu -- K3: the QKV epilogue, causal attention over the paged KV cache, and the
// split-KV merge, fused in one kernel.
//
// For each sequence of the ragged batch, rows q_start .. q_start + q_len - 1 sit at positions
// kv_len - q_len .. kv_len - 1 and attend to keys 0 .. pos (R15: causal MHA).  One CTA of W
// warps (4 at Dh = 128, 8 below: attn_warps) owns (sequence x 16-row query block, head, split of
// SPLIT keys, R33) and streams the split's keys as 16-key tiles:
//   * it reads the QKV GEMM's fp32 output for its query rows, applies RoPE and rounds Q to bf16
//     (B2) -- no separate epilogue kernel;
//   * warp w owns tiles w, w + W, w + 2W, ... of the split, each through its own two-stage ring in
//     shared memory: cached K/V page blocks (16 keys of one head) land by 2-D tensor copies (TMA)
//     in the 128-byte swizzle ldmatrix reads conflict-free; the warp requests its tile j + 2 as
//     soon as tile j is consumed, so every warp keeps two tiles in flight with no CTA barrier;
//     blocks written before the round are requested before the PDL wait (while the QKV GEMM
//     still runs);
//   * the sequence's new rows (K with RoPE, V) are formed from the QKV output straight into the
//     tiles by the warp that owns them, and appended to the cache pages by one writer per key;
//   * S = Q K^T and O = P V run as bf16 mma.sync.m16n8k16 (Q padded to 16 rows; P re-packed from
//     the S accumulators as the A operand, B5) with an online base-2 softmax per warp;
//   * the W warps merge (m, l, O) in warp order; with several splits every split publishes its
//     partial and the last to finish (atomic ticket) merges them in split order; the output is
//     rounded to bf16 (B3).
// Tile-to-warp assignment, split boundaries and every merge order are functions of the key
// positions only, so a row's result never depends on the batch (R19).  Memory-bound on the
// cached K/V: 2 * Dh * 2 bytes per key and head.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace seed {

namespace {
constexpr int STAGES = 2;               // tiles in flight per warp (3 and 4 measured: no gain, §7)
constexpr int TK = 16;                   // keys per tile (one page block: P >= 16, P % 16 == 0)
constexpr int QB = 16;                   // query rows per CTA (one m16 MMA tile)

template <int DH, int WARPS>
struct Smem {
  static constexpr int PITCH = DH + 8;                       // bf16 row pitch of Q (conflict-free ldmatrix)
  static constexpr int RB = (DH >= 64 ? 64 : DH) * 2;        // bytes per swizzled row segment (TMA box width)
  static constexpr int OP = DH + 4;                          // fp32 row pitch of the merge scratch
  static constexpr size_t TILE = (size_t)TK * DH * 2;        // K (or V) of one 16-key tile
  static constexpr size_t STAGE = 2 * TILE;                  // K then V
  static constexpr size_t RING = 0;                          // [WARPS][STAGES] stages, 1024-aligned
  static constexpr size_t Q = RING + (size_t)WARPS * STAGES * STAGE;   // bf16 [16][PITCH]
  static constexpr size_t ML = Q + (size_t)QB * PITCH * 2;   // fp32 m, l [WARPS][QB] each, factors [WARPS][QB], row l [QB]
  static constexpr size_t TKT = ML + (size_t)(3 * WARPS + 1) * QB * 4;  // ticket broadcast
  static constexpr size_t BAR = TKT + 16;                    // mbarriers [WARPS][STAGES]
  static constexpr size_t PG = BAR + WARPS * STAGES * 8;     // int [WARPS][32]: page of each of a warp's tiles
  static constexpr size_t BYTES = PG + WARPS * 32 * 4 + 1024;
  static constexpr int PER_SM = (int)((227 * 1024) / (BYTES + 1024)) < 1 ? 1 : (int)((227 * 1024) / (BYTES + 1024));
  // merge scratch fp32 [WARPS][QB][OP] aliases the ring after the loop
  static_assert((size_t)WARPS * QB * OP * 4 <= (size_t)WARPS * STAGES * STAGE, "merge scratch must fit the ring");
};

// Byte address of element e of row `row` in a 16-row K / V tile (tile base 1024-aligned), in the
// TMA swizzle of its row size (RB = 128 B: 16-byte chunk bits [4:6] XOR bits [7:9]; RB = 64 B:
// bits [4:5] XOR bits [7:8]); a row of Dh > 64 is split into 64-element halves, 16 rows each.
template <int DH>
SEED_DEV uint32_t tile_addr(uint32_t tile, int row, int e) {
  constexpr int RB = (DH >= 64 ? 64 : DH) * 2, EH = RB / 2;
  constexpr uint32_t MASK = RB == 128 ? 0x70u : 0x30u;
  const uint32_t a = tile + (uint32_t)((e / EH) * TK * RB + row * RB + (e % EH) * 2);
  return a ^ ((a >> 3) & MASK);
}

// tile_addr(tile, row, e) for e = e0 + E, E a multiple of 16 (compile-time after unrolling) and e0 < 16
// the lane's part, given x = tile_addr(0, row, e0): with 128-byte rows the swizzle XORs bits [4:6]
// with the row's bits [0:2], E's in-row part only touches bits [5:6] and the tile base is 1024-aligned,
// so the address is ((tile + x) ^ ((E % 64) * 2)) + (E / 64) * 16 rows * 128 B -- one XOR per ldmatrix
template <int DH>
SEED_DEV uint32_t tile_at(uint32_t tile, uint32_t x, int row, int e, int E) {
  if constexpr (DH >= 64) {
    return ((tile + x) ^ (uint32_t)((E % 64) * 2)) + (uint32_t)((E / 64) * TK * 128);
  } else {
    return tile_addr<DH>(tile, row, e);
  }
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


// MINB: resident CTAs per SM the registers are budgeted for (launch_w picks it per launch; register
// allocation does not change the arithmetic)
template <int DH, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
attn_stream_kernel(const __grid_constant__ CUtensorMap tmKV, const float* __restrict__ qkv, int H, int Hk,
                   SeqInfo seqs, const float2* __restrict__ rope, KVLayout kv, int layer, int n_qblk, float scale,
                   AttnWorkspace ws, int M, __nv_bfloat16* __restrict__ out, int SPLIT, int kv3d) {
  using L = Smem<DH, WARPS>;
  constexpr int NT = WARPS * 32;
  constexpr int P = L::PITCH;
  constexpr int OP = L::OP;
  constexpr int HALF = DH / 2;
  constexpr int DT = DH / 8;             // 8-dim n-tiles of the output
  constexpr int EH = L::RB / 2;          // elements per swizzled row segment (TMA box width)
  constexpr uint32_t TX = (uint32_t)(2 * TK * DH * 2);   // bytes of one tile's K and V
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __nv_bfloat16* q_s = reinterpret_cast<__nv_bfloat16*>(smem + L::Q);
  float* m_s = reinterpret_cast<float*>(smem + L::ML);   // [WARPS][QB]
  float* l_s = m_s + WARPS * QB;                          // [WARPS][QB]
  float* fw_s = l_s + WARPS * QB;                         // [WARPS][QB] warp merge factors
  float* rl_s = fw_s + WARPS * QB;                        // [QB] row sums
  int* tkt_s = reinterpret_cast<int*>(smem + L::TKT);
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::BAR);
  float* o_s = reinterpret_cast<float*>(smem + L::RING);  // merge scratch (after the loop)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    prefetch_tmap(&tmKV);
    for (int i = 0; i < WARPS * STAGES; ++i) mbar_init(&bar_s[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (ws.timing && tid == 0) atomicMin(&ws.timing[0], globaltimer_ns());
  unsigned long long* ct =
      ws.cta ? ws.cta + 8 * (size_t)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) : nullptr;
  auto stamp = [&](int k) {
    if (ct && tid == 0) ct[k] = globaltimer_ns();
  };
  auto done = [&]() {
    stamp(5);
    if (ws.timing && tid == 0) {
      atomicMax(&ws.timing[2], globaltimer_ns());
      ws.timing[3] = 2;  // record kind: attention
    }
  };
  stamp(0);
  const int seq = blockIdx.x / n_qblk, qb = blockIdx.x % n_qblk;
  const int head = blockIdx.y, split = blockIdx.z;
  const int kvh = head / (H / Hk);
  // the descriptors were uploaded before the round's first kernel: safe before pdl_wait()
  const int q0 = seqs.q_start[seq], ql = seqs.q_len[seq], kvl = seqs.kv_len[seq];
  const int slot = seqs.slot[seq];
  const int r0 = qb * QB;
  const int nr = min(QB, ql - r0);
  const int new_first = kvl - ql;                  // position of the sequence's first new row
  const int pos0 = new_first + r0;                 // position of the first row of this block
  const int key_end = pos0 + nr;                   // keys [0, key_end) are visible to some row
  const int k_lo = split * SPLIT, k_hi = min(k_lo + SPLIT, key_end);
  if (r0 >= ql || k_lo >= key_end) {               // nothing to do (grid sized by the longest sequence)
    done();
    return;                                        // (an exited CTA counts as having triggered)
  }
  const int nsplit = (key_end + SPLIT - 1) / SPLIT;  // splits of this query block (all CTAs agree)
  const int old_end = new_first;                   // keys [0, old_end) come from the cache
  const int stable = seqs.stable ? min(seqs.stable[seq], old_end) : 0;  // written before the round
  const int n_tiles = (k_hi - k_lo + TK - 1) / TK;
  const int my_tiles = warp < n_tiles ? (n_tiles - warp + WARPS - 1) / WARPS : 0;
  const int ldq = (H + 2 * Hk) * DH;               // row stride of the QKV GEMM output
  const uint32_t ring = smem_u32(smem + L::RING) + (uint32_t)(warp * STAGES * L::STAGE);

  // ---- this warp's j-th tile: keys [t0, t0 + 16); the cached part by tensor copies (lane 0)
  auto tile_t0 = [&](int j) { return k_lo + (warp + j * WARPS) * TK; };
  auto cached = [&](int j) { return tile_t0(j) < old_end; };
  // the page of each of this warp's tiles, one lane per tile, before any request: the issue path
  // below reads shared memory instead of waiting on a global load per tile (page-table rows are
  // uploaded before the round: safe before the PDL wait)
  int* pg_s = reinterpret_cast<int*>(smem + L::PG) + warp * 32;
  for (int j = lane; j < my_tiles; j += 32)
    if (cached(j)) pg_s[j] = __ldg(kv.page_table + (size_t)slot * kv.max_pages + tile_t0(j) / kv.P);
  __syncwarp();
  auto issue = [&](int j) {   // lane 0
    const int t0 = tile_t0(j);
    const int page = pg_s[j];
    const int row = (((page * kv.n_layers + layer) * 2) * kv.Hk + kvh) * kv.P + (t0 % kv.P);
    const uint32_t st = ring + (uint32_t)((j % STAGES) * L::STAGE);
    uint64_t* bar = &bar_s[warp * STAGES + j % STAGES];
    mbar_arrive_expect_tx(bar, TX);
    const uint64_t pol = kv.kv_once ? l2_policy_evict_first() : l2_policy_evict_normal();
    if (kv3d) {
      tma_load_3d_u32_hint(st, &tmKV, bar, 0, row, 0, pol);
      tma_load_3d_u32_hint(st + (uint32_t)L::TILE, &tmKV, bar, 0, row + kv.Hk * kv.P, 0, pol);
    } else {
#pragma unroll
      for (int h = 0; h < DH / EH; ++h) {
        tma_load_2d_u32_hint(st + (uint32_t)(h * TK * L::RB), &tmKV, bar, h * EH, row, pol);
        tma_load_2d_u32_hint(st + (uint32_t)(L::TILE + h * TK * L::RB), &tmKV, bar, h * EH, row + kv.Hk * kv.P, pol);
      }
    }
  };
  // tiles whose cached keys were all written before the round: requested before the PDL wait
  bool pre[STAGES];
#pragma unroll
  for (int j = 0; j < STAGES; ++j) {
    pre[j] = j < my_tiles && cached(j) && min(tile_t0(j) + TK, old_end) <= stable;
    if (pre[j] && lane == 0) issue(j);
  }
  pdl_wait();
  if (ws.timing && tid == 0) atomicMin(&ws.timing[1], globaltimer_ns());
  stamp(1);
#pragma unroll
  for (int j = 0; j < STAGES; ++j)
    if (!pre[j] && j < my_tiles && cached(j) && lane == 0) issue(j);

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
        const int rp = seqs.row_pos ? seqs.row_pos[q0 + r0 + r] : pos0 + r;   // tree rows: depth positions
        const float4* cs = reinterpret_cast<const float4*>(rope + (size_t)rp * HALF + i);
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
  __syncthreads();
#if ATTN_STAMPS
  stamp(6);
#endif

  // ---- the warp's tiles, online softmax over them (rows g, g + 8 of the MMA fragments)
  const int g = lane >> 2, t4 = lane & 3;
  // tree rows: the tree rows each row attends to (rows g, g + 8 of the fragments; 0 = causal row);
  // bit j = cache slot tbase + j
  const int tbase = seqs.tree_base ? seqs.tree_base[seq] : new_first;
  uint64_t anc_rows[2] = {0ull, 0ull};
  if (seqs.anc) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
      if (g + 8 * h2 < nr) anc_rows[h2] = seqs.anc[q0 + r0 + g + 8 * h2];
  }
  float o_acc[DT][4];
  float m_row[2] = {-INFINITY, -INFINITY}, l_row[2] = {0.f, 0.f};
#pragma unroll
  for (int j = 0; j < DT; ++j) o_acc[j][0] = o_acc[j][1] = o_acc[j][2] = o_acc[j][3] = 0.f;
  // this lane's swizzled ldmatrix offsets in a tile (K: key row, column 8 x bit 3 of the lane; V: the
  // transposed read), element 0 of the tile's first 64-column half (tile_at)
  const uint32_t kx = tile_addr<DH>(0u, (lane >> 4) * 8 + (lane & 7), ((lane >> 3) & 1) * 8);
  const uint32_t vx = tile_addr<DH>(0u, (lane & 7) + ((lane >> 3) & 1) * 8, (lane >> 4) * 8);
  uint32_t phase = 0;   // bit s: parity of stage s's next completion
  const uint32_t qa = smem_u32(q_s);
  const bool own_head = head % (H / Hk) == 0;
  // at most 256 threads per SM (MINB x warps): registers to spare, so Q's MMA fragments are loaded
  // once instead of once per tile (the same values: bit-identical)
  constexpr bool QREG = WARPS * 32 * MINB <= 256;
  uint32_t qf[QREG ? DH / 16 : 1][4];
  if constexpr (QREG) {
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks)
      ldsm_x4(qa + ((lane & 15) * P + ks * 16 + (lane >> 4) * 8) * 2, qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }
  for (int j = 0; j < my_tiles; ++j) {
    const int t0 = tile_t0(j), s = j % STAGES;
    const uint32_t kb = ring + (uint32_t)(s * L::STAGE), vb = kb + (uint32_t)L::TILE;
    if (t0 < old_end) {
      mbar_wait(&bar_s[warp * STAGES + s], (phase >> s) & 1u);
      phase ^= 1u << s;
    }
    // rows past the split's keys: zero (lane r its row r)
    if (lane < TK && t0 + lane >= k_hi) {
#pragma unroll
      for (int e = 0; e < DH; e += 8) {
        st_shared_v4(tile_addr<DH>(kb, lane, e), make_uint4(0, 0, 0, 0));
        st_shared_v4(tile_addr<DH>(vb, lane, e), make_uint4(0, 0, 0, 0));
      }
    }
    // the sequence's new keys in this tile: K (RoPE) and V from the QKV output into the tile; the
    // owning query block appends them to the cache (one writer per kv head and position)
    const int nk0 = max(t0, new_first), nk1 = min(t0 + TK, k_hi);
    if (nk0 < nk1) {
      const int NI = (nk1 - nk0) * (HALF / 4);
      for (int it = lane; it < NI; it += 32) {
        const int key = nk0 + it / (HALF / 4), i = (it % (HALF / 4)) * 4;
        const int m = q0 + (key - new_first);
        const float* yk = qkv + (size_t)m * ldq + (H + kvh) * DH;
        const float* yv = qkv + (size_t)m * ldq + (H + Hk + kvh) * DH;
        const int kp = seqs.row_pos ? seqs.row_pos[m] : key;
        const float4* cs = reinterpret_cast<const float4*>(rope + (size_t)kp * HALF + i);
        const float4 x0 = *reinterpret_cast<const float4*>(yk + i), x1 = *reinterpret_cast<const float4*>(yk + i + HALF);
        const float4 va = *reinterpret_cast<const float4*>(yv + i), vv = *reinterpret_cast<const float4*>(yv + i + HALF);
        const float4 c0 = __ldg(cs), c1 = __ldg(cs + 1);
        const uint2 klo = make_uint2(pack_bf16(x0.x * c0.x - x1.x * c0.y, x0.y * c0.z - x1.y * c0.w),
                                     pack_bf16(x0.z * c1.x - x1.z * c1.y, x0.w * c1.z - x1.w * c1.w));
        const uint2 khi = make_uint2(pack_bf16(x1.x * c0.x + x0.x * c0.y, x1.y * c0.z + x0.y * c0.w),
                                     pack_bf16(x1.z * c1.x + x0.z * c1.y, x1.w * c1.z + x0.w * c1.w));
        const uint2 vlo = make_uint2(pack_bf16(va.x, va.y), pack_bf16(va.z, va.w));
        const uint2 vhi = make_uint2(pack_bf16(vv.x, vv.y), pack_bf16(vv.z, vv.w));
        const int kk = key - t0;
        st_shared_v2(tile_addr<DH>(kb, kk, i), klo);
        st_shared_v2(tile_addr<DH>(kb, kk, i + HALF), khi);
        st_shared_v2(tile_addr<DH>(vb, kk, i), vlo);
        st_shared_v2(tile_addr<DH>(vb, kk, i + HALF), vhi);
        if (own_head && qb == (key - new_first) / QB) {
          const int page = __ldg(kv.page_table + (size_t)slot * kv.max_pages + key / kv.P);
          __nv_bfloat16* kdst = kv.pool + kv.offset(page, layer, 0, kvh, key % kv.P);
          *reinterpret_cast<uint2*>(kdst + i) = klo;
          *reinterpret_cast<uint2*>(kdst + i + HALF) = khi;
          *reinterpret_cast<uint2*>(kdst + kv.vofs() + i) = vlo;
          *reinterpret_cast<uint2*>(kdst + kv.vofs() + i + HALF) = vhi;
        }
      }
    }
    __syncwarp();
    // S = Q K^T (two accumulator chains), scaled and masked
    float sc[2][4], s2[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = s2[nt][0] = s2[nt][1] = s2[nt][2] = s2[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
      if constexpr (QREG) {
        a0 = qf[ks][0];
        a1 = qf[ks][1];
        a2 = qf[ks][2];
        a3 = qf[ks][3];
      } else {
        ldsm_x4(qa + ((lane & 15) * P + ks * 16 + (lane >> 4) * 8) * 2, a0, a1, a2, a3);
      }
      ldsm_x4(tile_at<DH>(kb, kx, (lane >> 4) * 8 + (lane & 7), ks * 16 + ((lane >> 3) & 1) * 8, ks * 16), b0, b1, b2,
              b3);
      float (*acc)[4] = (ks & 1) ? s2 : sc;
      mma_bf16(acc[0], a0, a1, a2, a3, b0, b1);
      mma_bf16(acc[1], a0, a1, a2, a3, b2, b3);
    }
    // a tile of cached keys below every row's position (and below the tree) needs no mask; padding
    // rows then score finite values that only their own, discarded, outputs see
    const bool interior = t0 + TK <= min(k_hi, new_first) && (!seqs.anc || t0 + TK <= tbase);
    float f_row[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = g + 8 * h2;
      const uint64_t anc_r = anc_rows[h2];
      float mx = -INFINITY;
      if (interior) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            float& v = sc[nt][2 * h2 + c];
            v = (v + s2[nt][2 * h2 + c]) * scale;
            mx = fmaxf(mx, v);
          }
      } else {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int key = t0 + nt * 8 + 2 * t4 + c;
            const bool ok = r < nr && key < k_hi &&
                            (anc_r ? (key < tbase || ((anc_r >> (key - tbase)) & 1ull)) : key <= pos0 + r);
            float& v = sc[nt][2 * h2 + c];
            v = ok ? (v + s2[nt][2 * h2 + c]) * scale : -INFINITY;
            mx = fmaxf(mx, v);
          }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(m_row[h2], mx);
      f_row[h2] = (m_row[h2] == -INFINITY) ? 0.f : exp2_approx(m_row[h2] - mn);
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float& v = sc[nt][2 * h2 + c];
          v = (mn == -INFINITY) ? 0.f : exp2_approx(v - mn);
          sum += v;
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      m_row[h2] = mn;
      l_row[h2] = l_row[h2] * f_row[h2] + sum;
    }
    // O = O * f + P V (P rounded to bf16 as the A operand, B5); V via ldmatrix.trans.  Once the
    // running maxima settle f = 1 exactly (ex2(0)) and the warp skips the rescaling (bit-identical)
    const uint32_t pa0 = pack_bf16(sc[0][0], sc[0][1]), pa1 = pack_bf16(sc[0][2], sc[0][3]);
    const uint32_t pa2 = pack_bf16(sc[1][0], sc[1][1]), pa3 = pack_bf16(sc[1][2], sc[1][3]);
    if (__any_sync(0xffffffffu, f_row[0] != 1.f || f_row[1] != 1.f)) {
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        o_acc[dt][0] *= f_row[0];
        o_acc[dt][1] *= f_row[0];
        o_acc[dt][2] *= f_row[1];
        o_acc[dt][3] *= f_row[1];
      }
    }
#pragma unroll
    for (int dt = 0; dt < DT; dt += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(tile_at<DH>(vb, vx, (lane & 7) + ((lane >> 3) & 1) * 8, dt * 8 + (lane >> 4) * 8, dt * 8), b0, b1, b2,
                b3);
      mma_bf16(o_acc[dt], pa0, pa1, pa2, pa3, b0, b1);
      mma_bf16(o_acc[dt + 1], pa0, pa1, pa2, pa3, b2, b3);
    }
    // stage s is free: request this warp's tile j + 2 into it
    __syncwarp();
#if ATTN_STAMPS
    if (j == 1) stamp(7);
#endif
    if (j + STAGES < my_tiles && cached(j + STAGES) && lane == 0) {
      fence_proxy_async();   // the generic reads / writes of the stage before the tensor copy
      issue(j + STAGES);
    }
  }
  stamp(2);
  // The successor (the O projection) may launch once every CTA got here: triggering at the start
  // would let its CTAs (one per SM, 175 KB of shared memory each) take the SMs this grid's later
  // waves need while they wait for this grid to finish.
  pdl_trigger();

  // ---- merge the W warps (fixed order) into this split's result
  __syncthreads();   // o_s aliases the ring
  if (t4 == 0) {
    m_s[warp * QB + g] = m_row[0];
    m_s[warp * QB + g + 8] = m_row[1];
    l_s[warp * QB + g] = l_row[0];
    l_s[warp * QB + g + 8] = l_row[1];
  }
  if (g < nr) {
#pragma unroll
    for (int dt = 0; dt < DT; ++dt)
      *reinterpret_cast<float2*>(o_s + ((size_t)warp * QB + g) * OP + dt * 8 + 2 * t4) =
          make_float2(o_acc[dt][0], o_acc[dt][1]);
  }
  if (g + 8 < nr) {
#pragma unroll
    for (int dt = 0; dt < DT; ++dt)
      *reinterpret_cast<float2*>(o_s + ((size_t)warp * QB + g + 8) * OP + dt * 8 + 2 * t4) =
          make_float2(o_acc[dt][2], o_acc[dt][3]);
  }
  __syncthreads();
  const size_t ws_row = (size_t)(q0 + r0);
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
    rl_s[r] = l;
    if (nsplit > 1) {
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
      const float4 v = *reinterpret_cast<const float4*>(o_s + ((size_t)w * QB + r) * OP + d);
      o.x += v.x * f;
      o.y += v.y * f;
      o.z += v.z * f;
      o.w += v.w * f;
    }
    const size_t row = ws_row + r;
    if (nsplit == 1) {
      const float l = rl_s[r];
      *reinterpret_cast<uint2*>(out + (row * H + head) * DH + d) =
          make_uint2(pack_bf16(o.x / l, o.y / l), pack_bf16(o.z / l, o.w / l));
    } else {
      *reinterpret_cast<float4*>(ws.o_part + (((size_t)split * M + row) * H + head) * DH + d) = o;
    }
  }
  stamp(3);
  if (nsplit == 1) {
    done();
    return;
  }
  // ---- several splits: publish, the last to finish merges every split in split order (R19)
  __syncthreads();
  int* ctr = ws.counters + ((size_t)(seq * n_qblk + qb) * H + head);
  if (tid == 0) {
    fence_acq_rel_gpu();   // release this split's partial (bar.sync + cumulativity)
    const int t = atomicAdd(ctr, 1);
    if (t == nsplit - 1) {
      fence_acq_rel_gpu(); // acquire the other splits' partials
      *ctr = 0;            // ready for the next launch (graph replay)
    }
    *tkt_s = t;
  }
  __syncthreads();
  if (*tkt_s != nsplit - 1) {
    done();
    return;
  }
  stamp(4);
  for (int e = tid; e < nr * (DH / 4); e += NT) {
    const int r = e / (DH / 4), d = (e % (DH / 4)) * 4;
    const size_t row = ws_row + r;
    float mx = -INFINITY;
    for (int sp = 0; sp < nsplit; ++sp)
      mx = fmaxf(mx, __ldcg(ws.ml_part + (((size_t)sp * M + row) * H + head) * 2));
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float2 ml = __ldcg(reinterpret_cast<const float2*>(ws.ml_part + (((size_t)sp * M + row) * H + head) * 2));
      if (ml.x == -INFINITY) continue;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(ws.o_part + (((size_t)sp * M + row) * H + head) * DH + d));
      const float f = exp2_approx(ml.x - mx);
      o.x += v.x * f;
      o.y += v.y * f;
      o.z += v.z * f;
      o.w += v.w * f;
      l += ml.y * f;
    }
    *reinterpret_cast<uint2*>(out + (row * H + head) * DH + d) =
        make_uint2(pack_bf16(o.x / l, o.y / l), pack_bf16(o.z / l, o.w / l));
  }
  done();
}

// warps per CTA (each with its own tile ring), a function of the head size only (R19)
// (measured per round, §7: the 68M draft at 8 warps 13.8 -> 11.7 us per layer at N = 24, 9.7 -> 7.9
// at N = 3; the 7B at 6 / 8 / 12 warps wins at N = 3..12 but loses at N = 24, where 4-warp CTAs
// three per SM keep the most warps resident)
int attn_warps(int Dh) { return Dh >= 128 ? 4 : 8; }

template <int DH, int W, int MINB>
cudaError_t launch_wm(dim3 grid, int M, int H, int Hk, const CUtensorMap& tmkv, const float* qkv, const SeqInfo& seqs,
                      const float2* rope, const KVLayout& kv, int layer, int n_qblk, int SPLIT, const AttnWorkspace& ws,
                      __nv_bfloat16* out, cudaStream_t st) {
  const size_t smem = Smem<DH, W>::BYTES;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_stream_kernel<DH, W, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return cudaErrorInvalidValue;
    attr = true;
  }
  // scores are kept in the base-2 domain: s = q.k / sqrt(Dh) * log2(e), p = 2^(s - max)
  const float scale = 1.0f / sqrtf((float)DH) * 1.4426950408889634f;
  return launch(attn_stream_kernel<DH, W, MINB>, grid, dim3(W * 32), smem, st, tmkv, qkv, H, Hk, seqs, rope, kv, layer,
                n_qblk, scale, ws, M, out, SPLIT, kv.kv3d);
}

template <int DH, int W>
cudaError_t launch_w(int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, const CUtensorMap& tmkv,
                     const float* qkv, const SeqInfo& seqs, const float2* rope, const KVLayout& kv, int layer,
                     const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st) {
  const int n_qblk = (max_q_len + QB - 1) / QB;
  const int SPLIT = attn_chunk_tokens(DH);
  const int splits = (max_kv + SPLIT - 1) / SPLIT;
  if (SPLIT / (TK * W) > 32) return cudaErrorInvalidValue;   // tiles per warp held in pg_s
  const dim3 grid(n_seq * n_qblk, H, splits);
  constexpr int per_sm = Smem<DH, W>::PER_SM > 4 ? 4 : Smem<DH, W>::PER_SM;
  // 8 warps: when the grid fits two CTAs per SM, the variant with twice the registers (the 68M
  // draft at N = 24: 128 registers, no spill, 9.5 vs 10.3 us per layer); larger grids (the 160M
  // draft's longer contexts) keep the resident count shared memory allows
  if constexpr (W == 8 && per_sm > 2) {
    if ((long)grid.x * grid.y * grid.z <= 2L * kNumSMs)
      return launch_wm<DH, W, 2>(grid, M, H, Hk, tmkv, qkv, seqs, rope, kv, layer, n_qblk, SPLIT, ws, out, st);
  }
  // 4 warps: a grid within one or two CTAs per SM takes a variant with Q held in registers (the 7B
  // at N = 3 / 5 / 6 / 8: 96-256 CTAs; GSM8K 12.5 -> 11.6 us per layer, rounds -0.8 %, CW -1.3 %,
  // N = 6 -2 %); the N = 24 grid (768 CTAs) keeps three per SM
  if constexpr (W == 4 && per_sm > 1) {
    if ((long)grid.x * grid.y * grid.z <= (long)kNumSMs)
      return launch_wm<DH, W, 1>(grid, M, H, Hk, tmkv, qkv, seqs, rope, kv, layer, n_qblk, SPLIT, ws, out, st);
    if constexpr (per_sm > 2)
      if ((long)grid.x * grid.y * grid.z <= 2L * kNumSMs)
        return launch_wm<DH, W, 2>(grid, M, H, Hk, tmkv, qkv, seqs, rope, kv, layer, n_qblk, SPLIT, ws, out, st);
  }
  return launch_wm<DH, W, per_sm>(grid, M, H, Hk, tmkv, qkv, seqs, rope, kv, layer, n_qblk, SPLIT, ws, out, st);
}

// warps per CTA: a function of the head size only (R19); env SEED_ATTN_WARPS (Dh = 128) /
// SEED_ATTN_WARPS_SMALL (below) override it for experiments (4, 8; 16 below Dh = 128)
template <int DH>
cudaError_t launch_dh(int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, const CUtensorMap& tmkv,
                      const float* qkv, const SeqInfo& seqs, const float2* rope, const KVLayout& kv, int layer,
                      const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st) {
  // page blocks of 16 keys land by one tensor copy each: 16 | P
  if (kv.P < TK || kv.P % TK) return cudaErrorInvalidValue;
  static int w = -1;
  if (w < 0) {
    const char* e = getenv(DH >= 128 ? "SEED_ATTN_WARPS" : "SEED_ATTN_WARPS_SMALL");
    w = e ? atoi(e) : attn_warps(DH);
  }
  if (w == 8)
    return launch_w<DH, 8>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  if constexpr (DH < 128) {
    if (w == 16)
      return launch_w<DH, 16>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  } else {
    if (w == 6)
      return launch_w<DH, 6>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
    if (w == 12)
      return launch_w<DH, 12>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  }
  return launch_w<DH, 4>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
}

}  // namespace

// keys per CTA: a fixed split grid, a function of the head size only (R19): 1024 keys at Dh = 128,
// 512 below.  Fewer, longer CTAs keep more bytes in flight and merge less (measured per round: the
// 68M draft at 128-key splits 5.29 ms -> 5.07 at 512 on the N = 24 sweep; the 7B / 13B targets at
// 512 -> 1024: sweep 5.07 -> 5.03, 13B BW shape 10.33 -> 10.09; N = 3 / 5 unchanged).  Env
// SEED_ATTN_SPLIT / SEED_ATTN_SPLIT_SMALL (Dh >= 128 / < 128, multiples of 16) for experiments.
int attn_chunk_tokens(int Dh) {
  static int big = -1, small = -1;
  if (big < 0) {
    const char* e = getenv("SEED_ATTN_SPLIT");
    big = e ? std::max(16, atoi(e) / 16 * 16) : 1024;
    const char* f = getenv("SEED_ATTN_SPLIT_SMALL");
    small = f ? std::max(16, atoi(f) / 16 * 16) : 512;
  }
  return Dh >= 128 ? big : small;
}

bool attn_kv_tmap(CUtensorMap* map, const KVLayout& kv, size_t n_pages, int* kv3d) {
  const uint64_t rows = (uint64_t)n_pages * kv.n_layers * 2 * kv.Hk * kv.P;
  // Dh = 128: one 3D box per 16-row block (both 64-element halves: 4 KB contiguous in the pool);
  // otherwise boxes of 16 rows of 128 B (Dh = 64, 128-byte swizzle) or 64 B (Dh = 32, 64-byte swizzle)
  *kv3d = 0;
  const char* e = getenv("SEED_ATTN_KV3D");
  if (kv.Dh == 128 && !(e && e[0] == '0') && encode_tmap_kv_halves(map, kv.pool, rows, (uint32_t)TK)) {
    *kv3d = 1;
    return true;
  }
  return encode_tmap_2d(map, kv.pool, (uint64_t)kv.Dh, rows, (uint32_t)(kv.Dh >= 64 ? 64 : kv.Dh), (uint32_t)TK,
                        kv.Dh >= 64 ? 128 : 64);
}

cudaError_t attention(const float* qkv, int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, int Dh,
                      const SeqInfo& seqs, const float2* rope, const KVLayout& kv, const CUtensorMap& tmkv, int layer,
                      const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st) {
  const int splits = (max_kv + attn_chunk_tokens(Dh) - 1) / attn_chunk_tokens(Dh);
  if (splits > ws.max_splits) return cudaErrorInvalidValue;
  if ((size_t)n_seq * ((max_q_len + QB - 1) / QB) * H > (size_t)ws.max_counters) return cudaErrorInvalidValue;
  if (Dh == 128) return launch_dh<128>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  if (Dh == 64) return launch_dh<64>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  if (Dh == 32) return launch_dh<32>(M, n_seq, max_q_len, max_kv, H, Hk, tmkv, qkv, seqs, rope, kv, layer, ws, out, st);
  return cudaErrorInvalidValue;
}

}  // namespace seed
