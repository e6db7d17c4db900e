// kernels.h -- host-side launch interface between the engine and the CUDA kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

namespace seed {

// ------------------------------------------------------------------ paged KV cache layout
// pool: bf16 [num_pages][n_layers][2 (K,V)][Hk][P][Dh]; page table: int32 [slots][max_pages]
struct KVLayout {
  __nv_bfloat16* pool;
  const int32_t* page_table;
  int32_t max_pages;  // per slot
  int32_t n_layers, Hk, Dh, P;
  int32_t kv3d;       // the pool's tensor map is the 3D (64, rows, halves) form (Dh = 128)
  int32_t kv_once;    // the cache is read once per round (the target): K/V tiles loaded evict-first
  __host__ __device__ size_t page_elems() const { return (size_t)n_layers * 2 * Hk * P * Dh; }
  __host__ __device__ size_t vofs() const { return (size_t)Hk * P * Dh; }  // K -> V of the same layer
  __host__ __device__ size_t offset(int page, int layer, int kv, int h, int slot_in_page) const {
    return (size_t)page * page_elems() + ((size_t)(layer * 2 + kv) * Hk + h) * P * Dh + (size_t)slot_in_page * Dh;
  }
};

// ------------------------------------------------------------------ K2: cluster split-K GEMM
// Y[m][n] = sum_k X[m][k] W[n][k]; W [N][K] bf16, X [Mcap][K] bf16 (rows >= M ignored).
struct GemmPlan {
  int N, K, KB, tiles;
  int c;                         // CTAs (k-ranges) per 128-row weight tile, a function of (N, K)
  int split_smem_kb;             // dynamic shared memory per CTA
  int keep_w = 0;                // weights streamed with the L2 evict-last policy (a draft model re-read every step)
  CUtensorMap tmW;
};

// bf16 2D tensor map, swizzle 128 B (default) or 64 B
bool encode_tmap_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                    uint32_t box_outer, int swizzle_bytes = 128);
// KV pool rows of 128 bf16 as a 3D map (64 elements, rows, 2 halves): one tensor copy per 16-row block
bool encode_tmap_kv_halves(CUtensorMap* map, const void* ptr, uint64_t rows, uint32_t box_rows);
// 2D store map (fp32 or bf16) without swizzle, rows of row_stride_elems elements
bool encode_tmap_store(CUtensorMap* map, const void* ptr, bool fp32, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer);

void gemm_plan(GemmPlan* plan, const void* W, int N, int K, int min_units = 4);
void gemm_plan_free(GemmPlan* plan);
// Operands and epilogue of one GEMM launch (see gemm.cu):
// Y = epilogue(X W^T): X is a bf16 [M][K] operand read by TMA (tmX, box 64 x m_pad).
// ssq_in (optional, [ceil(K/128)][ssq_in_ld]) scales output row m by 1/rms(x_m) = 1/sqrt(sum/K + eps):
// the RMSNorm of x_m applied after the GEMM, on X = bf16(x * w_norm) (R24).
//   ymode 0: Y[yrow ? yrow[m] : m][n] = acc (* 1/rms), rows with yrow[m] < 0 skipped
//   ymode 1: residual: Y[m][n] += acc; ssq_out[n/128][m] = tile sums of the new Y^2;
//            hout[m][n] = bf16(Y[m][n] * nw[n]) (the next RMSNorm's operand)
//   ymode 2: SwiGLU on interleaved gate/up tiles (64 + 64 rows of W per 128-row tile):
//            hout[m][j] = bf16(silu(g_j) * u_j), g, u scaled by 1/rms; hout is [M][N/2]
struct GemmIO {
  const CUtensorMap* tmX = nullptr;
  const float* ssq_in = nullptr;
  int ssq_in_ld = 0;
  float eps = 1e-5f;
  int ymode = 0;
  float* Y = nullptr;
  int ldY = 0;
  const int32_t* yrow = nullptr;
  float* ssq_out = nullptr;
  const __nv_bfloat16* nw = nullptr;
  __nv_bfloat16* hout = nullptr;
  // optional tensor map of the output for whole-tile stores (c = 1): ymode 0 -> Y (fp32, exactly M rows,
  // boxes of 128 x m_pad), ymode 2 -> hout (bf16, exactly M rows, boxes of 64 x m_pad); no swizzle
  const CUtensorMap* tmY = nullptr;
};
// timing: optional [4] launch record (kind 1); cta: optional [G][16] per-CTA globaltimer ns:
// start, producer release, producer done, first stage full, MMA done, first accumulator ready,
// epilogue done, end, last partial stored, last ticket taken, reduce done, finish done
cudaError_t gemm_run(const GemmPlan& plan, int M, const GemmIO& io, cudaStream_t st,
                     unsigned long long* timing = nullptr, unsigned long long* cta = nullptr);
cudaError_t timing_accumulate(unsigned long long* rec, int n, unsigned long long* acc, unsigned long long* last,
                              cudaStream_t st);
int gemm_mpad(int M);

// ------------------------------------------------------------------ epilogues / elementwise
struct RowInfo {         // per row of the ragged batch
  const int32_t* tok;    // [M] token ids
  const int32_t* pos;    // [M] absolute positions
  const int32_t* slot;   // [M] stream slot (page table row)
};
// x = embed[tok] (or x as given when embed == nullptr), ssq[t][m] = sum of x^2 over 128-column
// tile t, h = bf16(x * nw) (the first RMSNorm's GEMM operand, R24)
// err (optional): bit 1 is set when a token id is outside [0, V) (the row then reads id 0)
cudaError_t embed_stats(const __nv_bfloat16* embed, const int32_t* tok, int tok_stride, int M, int d, int V, float* x,
                        float* ssq, const __nv_bfloat16* nw, __nv_bfloat16* h, int32_t* err, cudaStream_t st,
                        unsigned long long* timing = nullptr);
cudaError_t rope_table_init(float2* table, int max_pos, int Dh, double theta, cudaStream_t st);
// tree rounds: the accepted path's K/V rows of every layer move to consecutive slots -- for
// stream b (stream slot slots[b], root at cache position tlen[slots[b]] - 1 before the commit) and
// depth d = 1 .. max_depth while node[b][d - 1] >= 0: position root + node -> root + d (a node's
// index is at least its depth, so in-order copies never overwrite a later source)
cudaError_t kv_compact(const KVLayout& kv, const int32_t* slots, const int32_t* tlen, const int32_t* node,
                       int node_stride, int max_depth, int B, cudaStream_t st, unsigned long long* timing = nullptr);
cudaError_t kv_write_dense(const KVLayout& kv, int layer, int slot, int n, const __nv_bfloat16* k,
                           const __nv_bfloat16* v, cudaStream_t st);

// ------------------------------------------------------------------ K3: paged attention
struct SeqInfo {          // per sequence of the ragged batch (device arrays)
  const int32_t* q_start; // first row
  const int32_t* q_len;   // rows
  const int32_t* kv_len;  // keys after append = pos(last row) + 1
  const int32_t* slot;
  const int32_t* stable;  // keys written before the round (safe to prefetch early); may be null
  // tree rows (k_config verification, R36; both null for causal rows): per chunk row, the RoPE
  // position and the bit mask of the sequence's new rows it attends to (bit j = new row j; the
  // cached keys are always visible).  A sequence then has at most 64 new rows.
  const int32_t* row_pos = nullptr;
  const uint64_t* anc = nullptr;
  const int32_t* tree_base = nullptr;  // per sequence: cache slot of bit 0 of anc (default: its first new row)
};
struct AttnWorkspace {
  float* o_part;   // [splits][M][H][Dh]
  float* ml_part;  // [splits][M][H][2]
  int* counters;   // [max_counters] chunk tickets per (sequence block, head), zero between launches
  int max_splits, max_counters;
  unsigned long long* timing;  // optional profile record [4] (start, release, end)
  unsigned long long* cta = nullptr;  // optional per-block phase words [grid][8] (diagnostics)
};
int attn_chunk_tokens(int Dh);   // keys per attention CTA (split grid) for head size Dh
int attn_query_block();
// fused: QKV epilogue (RoPE, bf16, KV append) + paged attention + split-KV merge; qkv = Y [M][(H+2Hk)Dh]
// tmkv: 2D tensor map of the KV pool (attn_kv_tmap): rows of Dh elements, boxes of min(Dh, 64) x
// min(P, 32) with the 128-byte swizzle
bool attn_kv_tmap(CUtensorMap* map, const KVLayout& kv, size_t n_pages, int* kv3d);
// qkv: the QKV projection's fp32 output; ws.counters holds max_counters split tickets, zero between launches
cudaError_t attention(const float* qkv, int M, int n_seq, int max_q_len, int max_kv, int H, int Hk, int Dh,
                      const SeqInfo& seqs, const float2* rope, const KVLayout& kv, const CUtensorMap& tmkv, int layer,
                      const AttnWorkspace& ws, __nv_bfloat16* out, cudaStream_t st);

// ------------------------------------------------------------------ K4 / K1 sampler / K5
struct VerifyArgs {
  const float* zt; const float* zd; const int32_t* xs;
  long zt_stride_b, zd_stride_b;  // floats between streams
  int B, gamma, V;
  float T;
  uint32_t k0, k1;
  const uint32_t* sids; const int32_t* rs;
  int bonus;
  int32_t* out_tok; int32_t* out_cnt; int32_t* out_acc;
  float* dbg; double* stats;
  void* work;      // device scratch of vocab_verify_work_bytes(B, gamma): tickets, accept flags, row statistics;
                   // zero before the first launch (the kernel re-zeroes the tickets)
  int32_t* err;    // optional error word: [0] |= 2 when a race has no finite key, [1] += empty-residual fallbacks
  unsigned long long* timing;   // optional launch record (kind 3)
};
size_t vocab_verify_work_bytes(int B, int gamma);
cudaError_t vocab_verify(const VerifyArgs& a, cudaStream_t st);
// K1's fused successor work: the next draft step's embedding of the sampled token (what
// embed_stats computes for that step's rows, bit for bit): x[b] = E[y_b] (fp32), ssq[tile][b]
// (ld = rows of the next step), h[b] = bf16(x * nw); emb == nullptr: none
struct EmbedNext {
  const __nv_bfloat16* emb = nullptr;
  int d = 0;
  float* x = nullptr;
  float* ssq = nullptr;
  int ssq_ld = 0;
  const __nv_bfloat16* nw = nullptr;
  __nv_bfloat16* h = nullptr;
};
cudaError_t draft_sample(const float* z, long ld, int B, int V, float T, uint32_t k0, uint32_t k1,
                         const uint32_t* sids, const int32_t* rs, int j, int32_t* out, int out_stride, int32_t* out2,
                         int out2_stride, int32_t* err, cudaStream_t st, unsigned long long* timing = nullptr,
                         const EmbedNext& en = EmbedNext{});
// K1T / K4T (tree.cu): k_config tree drafting and verification (DESIGN R36)
cudaError_t draft_topk(const float* z, long ld, int B, int V, float T, uint32_t k0, uint32_t k1, const uint32_t* sids,
                       const int32_t* rs, int node, int m, int32_t* out, int out_stride, int first, int32_t* out2,
                       int out2_stride, int32_t* err, cudaStream_t st, unsigned long long* timing = nullptr);
cudaError_t verify_tree(const float* zt, long zt_stride_b, const float* zd, long zd_stride_b, const int32_t* tok,
                        int tok_stride, const int32_t* ch_first, const int32_t* ch_cnt, int B, int K, int V, float T,
                        uint32_t k0, uint32_t k1, const uint32_t* sids, const int32_t* rs, int bonus, int32_t* out_tok,
                        int32_t* out_cnt, int32_t* out_node, int32_t* err, cudaStream_t st,
                        unsigned long long* timing = nullptr);
cudaError_t philox_fill(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int n,
                        uint32_t* out, cudaStream_t st);

struct StreamState {     // device per-slot state (K5)
  int32_t* tlen;         // |T_s|
  int32_t* len_t;        // target KV entries
  int32_t* len_d;        // draft KV entries
  int32_t* L;            // new tokens
  int32_t* r;            // stream-local round
  int32_t* done;
  int32_t* hist;         // [slots][max_ctx] validated tokens
  int32_t max_ctx;
};
// K5 (one CTA): commit + KV lengths (R6, R7) and this rank's exchange block: records [cap][gamma + 3]
// (padding pre-filled with -1 by the caller) and, after them, *outside + the batch's undone streams
cudaError_t rollback_commit(const StreamState& s, const int32_t* batch_slots, int B, int gamma,
                            const int32_t* out_tok, const int32_t* out_cnt, int max_new, int32_t* records, int cap,
                            const uint32_t* gids, const int32_t* outside, cudaStream_t st,
                            unsigned long long* timing = nullptr);

}  // namespace seed
