// attention.cu -- K3: causal attention of the verify / draft / prefill rows over the paged KV cache.
//
// For each sequence of the ragged batch, rows q_start .. q_start + q_len - 1 sit at positions
// kv_len - q_len .. kv_len - 1 and attend to keys 0 .. pos (R15: causal MHA).  The new rows'
// K/V were already appended to the pages by the QKV epilogue, so every key is read from the
// cache the same way.  Memory-bound on K/V; the work is split over
// (sequence x 8-row query block, head, 128-key chunk) so that N = 3 streams still fill the
// GPU ("flash-decoding"), with a fixed chunk grid so a row's result never depends on the
// batch (R19).  Each warp stages a 32-key K/V tile in shared memory, scores it with fp32
// FMAs (lane = key), keeps an online softmax per row and accumulates P.V (lane = dims).
// A second kernel merges the chunk partials in chunk order and rounds the output to bf16 (B3).
#include "common.cuh"
#include "kernels.h"

namespace seed {

namespace {
constexpr int CHUNK = 128;      // keys per CTA (4 warps x 32)
constexpr int WARPS = 4;
constexpr int QB = 8;           // query rows per CTA

template <int DH, int NR>
__global__ void __launch_bounds__(128)
attn_chunk_kernel(const __nv_bfloat16* __restrict__ q, int H, int Hk, SeqInfo seqs, KVLayout kv, int layer,
                  int n_qblk, float scale, AttnWorkspace ws, int M) {
  constexpr int DPL = DH / 32;          // dims per lane in P.V
  constexpr int KPAD = DH + 8;          // bf16 row pitch of the K tile (16-byte pad)
  extern __shared__ __align__(16) uint8_t attn_smem[];
  // carve: K tiles | V tiles (aliased by o_s after the key loop) | q | p | m, l
  auto k_s = reinterpret_cast<__nv_bfloat16(*)[32][KPAD]>(attn_smem);
  auto v_s = reinterpret_cast<__nv_bfloat16(*)[32][DH]>(attn_smem + WARPS * 32 * KPAD * 2);
  auto o_s = reinterpret_cast<float(*)[QB][DH]>(attn_smem);
  uint8_t* tail = attn_smem + WARPS * 32 * (KPAD + DH) * 2;
  auto q_s = reinterpret_cast<float(*)[DH]>(tail);
  auto p_s = reinterpret_cast<float(*)[QB][32]>(tail + QB * DH * 4);
  auto m_s = reinterpret_cast<float(*)[QB]>(tail + QB * DH * 4 + WARPS * QB * 32 * 4);
  auto l_s = reinterpret_cast<float(*)[QB]>(tail + QB * DH * 4 + WARPS * QB * 32 * 4 + WARPS * QB * 4);

  pdl_trigger();
  pdl_wait();
  const int seq = blockIdx.x / n_qblk, qb = blockIdx.x % n_qblk;
  const int head = blockIdx.y, split = blockIdx.z;
  const int kvh = head / (H / Hk);
  const int q0 = seqs.q_start[seq], ql = seqs.q_len[seq], kvl = seqs.kv_len[seq];
  const int slot = seqs.slot[seq];
  const int r0 = qb * QB;
  if (r0 >= ql) return;
  const int nr = min(QB, ql - r0);
  const int pos0 = kvl - ql + r0;                  // position of the first row of this block
  const int key_end = pos0 + nr;                   // keys [0, key_end) are visible to some row
  const int c_begin = split * CHUNK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t ws_row = (size_t)(q0 + r0);

  if (c_begin >= key_end) {
    // empty chunk for this block: mark the partials invalid
    for (int e = tid; e < nr; e += 128) {
      float* ml = ws.ml_part + (((size_t)split * M + ws_row + e) * H + head) * 2;
      ml[0] = -INFINITY;
      ml[1] = 0.f;
    }
    return;
  }

  for (int e = tid; e < QB * DH; e += 128) {
    const int r = e / DH, d = e % DH;
    q_s[r][d] = r < nr ? bf2f(q[((size_t)(q0 + r0 + r) * H + head) * DH + d]) : 0.f;
  }
  __syncthreads();

  float m_r[NR], l_r[NR], o_r[NR][DPL];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    m_r[r] = -INFINITY;
    l_r[r] = 0.f;
#pragma unroll
    for (int j = 0; j < DPL; ++j) o_r[r][j] = 0.f;
  }

  const int c_end = min(c_begin + CHUNK, key_end);
  for (int kt = c_begin + warp * 32; kt < c_end; kt += WARPS * 32) {
    // ---- stage the K and V tile of keys kt .. kt+31 (16-byte vectors)
    constexpr int VPR = DH / 8;   // 16-byte vectors per key row
    // all 16-byte pieces of the tile in flight at once (cp.async, no register staging); the
    // tile's page ids (kt is a multiple of 32, P divides 32 or vice versa) are read once
    const int pg_first = kt / kv.P;
    const int npg = (min(kt + 31, c_end - 1)) / kv.P - pg_first + 1;
    const int my_page = lane < npg ? __ldg(kv.page_table + (size_t)slot * kv.max_pages + pg_first + lane) : 0;
#pragma unroll 8
    for (int e = lane; e < 32 * VPR; e += 32) {
      const int kk = e / VPR, c16 = e % VPR;
      const int key = kt + kk;
      const int page = __shfl_sync(0xffffffffu, my_page, min(31, key / kv.P - pg_first));
      if (key < c_end) {
        const size_t ko = kv.offset(page, layer, 0, kvh, key % kv.P);
        cp_async16(&k_s[warp][kk][c16 * 8], reinterpret_cast<const uint4*>(kv.pool + ko) + c16);
        cp_async16(&v_s[warp][kk][c16 * 8], reinterpret_cast<const uint4*>(kv.pool + ko + kv.vofs()) + c16);
      } else {
        *reinterpret_cast<uint4*>(&k_s[warp][kk][c16 * 8]) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(&v_s[warp][kk][c16 * 8]) = make_uint4(0, 0, 0, 0);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    // ---- scores: lane = key
    const int key = kt + lane;
    float s[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) s[r] = 0.f;
#pragma unroll 4
    for (int d = 0; d < DH; d += 8) {
      float kf[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(&k_s[warp][lane][d]), kf);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float4 qa = *reinterpret_cast<const float4*>(&q_s[r][d]);
        const float4 qc = *reinterpret_cast<const float4*>(&q_s[r][d + 4]);
        s[r] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qc.x * kf[4] + qc.y * kf[5] +
                qc.z * kf[6] + qc.w * kf[7];
      }
    }
    // ---- online softmax per row (causal mask: key <= pos(row))
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const bool valid = (r < nr) && (key < c_end) && (key <= pos0 + r);
      const float sc = valid ? s[r] * scale : -INFINITY;
      const float tmax = warp_max(sc);
      const float m_new = fmaxf(m_r[r], tmax);
      float p = 0.f, corr = 1.f;
      if (m_new != -INFINITY) {
        p = valid ? expf(sc - m_new) : 0.f;
        corr = (m_r[r] == -INFINITY) ? 0.f : expf(m_r[r] - m_new);
      }
      l_r[r] = l_r[r] * corr + warp_sum(p);
      m_r[r] = m_new;
#pragma unroll
      for (int j = 0; j < DPL; ++j) o_r[r][j] *= corr;
      p_s[warp][r][lane] = p;
    }
    __syncwarp();
    // ---- P.V: lane owns dims lane*DPL .. +DPL
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      float vf[DPL];
      if constexpr (DPL == 4) {
        const uint2 raw = *reinterpret_cast<const uint2*>(&v_s[warp][kk][lane * 4]);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
        vf[0] = a.x; vf[1] = a.y; vf[2] = b.x; vf[3] = b.y;
      } else if constexpr (DPL == 2) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v_s[warp][kk][lane * 2]));
        vf[0] = a.x; vf[1] = a.y;
      } else {
        vf[0] = bf2f(v_s[warp][kk][lane]);
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float p = p_s[warp][r][kk];
#pragma unroll
        for (int j = 0; j < DPL; ++j) o_r[r][j] += p * vf[j];
      }
    }
    __syncwarp();
  }
  // ---- merge the 4 warps of the CTA (fixed order); o_s aliases the K/V tiles
  __syncthreads();
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (lane == 0) {
      m_s[warp][r] = m_r[r];
      l_s[warp][r] = l_r[r];
    }
#pragma unroll
    for (int j = 0; j < DPL; ++j) o_s[warp][r][lane * DPL + j] = o_r[r][j];
  }
  __syncthreads();
  for (int e = tid; e < nr * DH; e += 128) {
    const int r = e / DH, d = e % DH;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) mx = fmaxf(mx, m_s[w][r]);
    float o = 0.f, l = 0.f;
    if (mx != -INFINITY) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        if (m_s[w][r] == -INFINITY) continue;
        const float f = expf(m_s[w][r] - mx);
        o += o_s[w][r][d] * f;
        l += l_s[w][r] * f;
      }
    }
    const size_t row = ws_row + r;
    ws.o_part[(((size_t)split * M + row) * H + head) * DH + d] = o;
    if (d == 0) {
      float* ml = ws.ml_part + (((size_t)split * M + row) * H + head) * 2;
      ml[0] = mx;
      ml[1] = l;
    }
  }
}

// merge chunk partials in chunk order; grid (M, H), block Dh
__global__ void attn_combine_kernel(AttnWorkspace ws, int M, int H, int Dh, int splits, const int32_t* row_nsplit,
                                    __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, head = blockIdx.y, d = threadIdx.x;
  const int ns = row_nsplit ? row_nsplit[row] : splits;
  float mx = -INFINITY;
  for (int s = 0; s < ns; ++s) mx = fmaxf(mx, ws.ml_part[(((size_t)s * M + row) * H + head) * 2]);
  float o = 0.f, l = 0.f;
  for (int s = 0; s < ns; ++s) {
    const float* ml = ws.ml_part + (((size_t)s * M + row) * H + head) * 2;
    if (ml[0] == -INFINITY) continue;
    const float f = expf(ml[0] - mx);
    o += ws.o_part[(((size_t)s * M + row) * H + head) * Dh + d] * f;
    l += ml[1] * f;
  }
  out[((size_t)row * H + head) * Dh + d] = f2bf(o / l);
}


template <int DH>
constexpr size_t attn_smem_bytes() {
  return (size_t)WARPS * 32 * (DH + 8 + DH) * 2 + QB * DH * 4 + WARPS * QB * 32 * 4 + 2 * WARPS * QB * 4;
}

template <int DH, int NR>
struct ChunkLauncher {
  static cudaError_t go(dim3 grid, size_t smem, cudaStream_t st, const __nv_bfloat16* q, int H, int Hk,
                        const SeqInfo& seqs, const KVLayout& kv, int layer, int n_qblk, float scale,
                        const AttnWorkspace& ws, int M) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(attn_chunk_kernel<DH, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    return launch(attn_chunk_kernel<DH, NR>, grid, dim3(128), smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws,
                  M);
  }
};

template <int DH>
cudaError_t launch_chunks(const __nv_bfloat16* q, int M, int n_seq, int max_q_len, int max_kv, int H, int Hk,
                          const SeqInfo& seqs, const KVLayout& kv, int layer, const AttnWorkspace& ws,
                          cudaStream_t st) {
  const int n_qblk = (max_q_len + QB - 1) / QB;
  const int splits = (max_kv + CHUNK - 1) / CHUNK;
  dim3 grid(n_seq * n_qblk, H, splits);
  const float scale = 1.0f / sqrtf((float)DH);
  const size_t smem = attn_smem_bytes<DH>();
  if (max_q_len == 1)
    return ChunkLauncher<DH, 1>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else if (max_q_len == 2)
    return ChunkLauncher<DH, 2>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else if (max_q_len <= 4)
    return ChunkLauncher<DH, 4>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else if (max_q_len <= 5)
    return ChunkLauncher<DH, 5>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else if (max_q_len <= 6)
    return ChunkLauncher<DH, 6>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else if (max_q_len <= 7)
    return ChunkLauncher<DH, 7>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
  else
    return ChunkLauncher<DH, 8>::go(grid, smem, st, q, H, Hk, seqs, kv, layer, n_qblk, scale, ws, M);
}
}  // namespace

int attn_chunk_tokens() { return CHUNK; }

cudaError_t attention(const __nv_bfloat16* q, int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, int Dh,
                      const SeqInfo& seqs, const KVLayout& kv, int layer, const AttnWorkspace& ws,
                      __nv_bfloat16* out, cudaStream_t st) {
  const int splits = (max_kv + CHUNK - 1) / CHUNK;
  if (splits > ws.max_splits) return cudaErrorInvalidValue;
  cudaError_t e;
  if (Dh == 128) e = launch_chunks<128>(q, M, n_seq, max_q_len, max_kv, H, Hk, seqs, kv, layer, ws, st);
  else if (Dh == 64) e = launch_chunks<64>(q, M, n_seq, max_q_len, max_kv, H, Hk, seqs, kv, layer, ws, st);
  else if (Dh == 32) e = launch_chunks<32>(q, M, n_seq, max_q_len, max_kv, H, Hk, seqs, kv, layer, ws, st);
  else return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return launch(attn_combine_kernel, dim3(M, H), dim3(Dh), 0, st, ws, M, H, Dh, splits, (const int32_t*)nullptr, out);
}

}  // namespace seed
