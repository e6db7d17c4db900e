/*
 * seed_ops.h -- op-level C ABI of libseed: the individual hot-path kernels, exported so
 * each can be checked element by element against the oracle (tests/test_gpu_*.py).
 * The round API in seed.h composes exactly these kernels; nothing here has a CPU path.
 *
 * All pointers are DEVICE pointers unless named *_host; all calls are asynchronous on
 * `stream` (cudaStream_t as void*) and return seed_status (see seed.h).
 */
#ifndef SEED_OPS_H_
#define SEED_OPS_H_

#include "seed.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K7 Philox4x32-10 (R5): out[4*i + w] = word w of Philox(ctr = (c0_base + i, c1, c2, c3),
 * key = (k0, k1)), i = 0..n-1.  out: device uint32 [4n]. */
SEED_API seed_status seed_op_philox(uint32_t c0_base, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                           uint32_t k1, int32_t n, uint32_t* out, void* stream);

/* K2 GEMM on tcgen05: Y[M][N] = X[M][K] * W[N][K]^T with bf16 operands and fp32
 * accumulation (swap-AB: W rows are the UMMA M=128 side).  K % 64 == 0, 1 <= M.
 * Split over the SMs stream-K style with a fixed, M-independent reduction order
 * (batch invariance, R19).  Y: fp32 row-major [M][N]. */
SEED_API seed_status seed_op_gemm(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* Y,
                         void* stream);

/* K4 fused vocabulary kernel, given logits (R1-R4, R13, R14):
 *   zt [B][gamma+1][V], zd [B][gamma][V] fp32; xs [B][gamma] drafted ids;
 *   sids [B] global stream ids; rs [B] stream-local round counters.
 * out_tok [B][gamma+1] (x_1..x_a, y, -1 pad), out_cnt [B] (a + 1, or gamma if bonus = 0 and
 * a = gamma), out_acc [B] (= a).  dbg (optional) [B][gamma][4] fp32:
 * lp(x_j), lq(x_j), u_j, rho_j (unconsumed positions included).  stats (optional)
 * [B][2*gamma+1][2] fp64: (m, log1p(S')) for target rows 0..gamma then draft rows. */
SEED_API seed_status seed_op_verify(const float* zt, const float* zd, const int32_t* xs, int32_t B, int32_t gamma,
                           int32_t V, float temperature, uint64_t seed, const uint32_t* sids,
                           const int32_t* rs, int32_t bonus, int32_t* out_tok, int32_t* out_cnt,
                           int32_t* out_acc, float* dbg, double* stats, void* stream);

/* K1 sampler: draft race x = argmax_v (fl32(z_v / T) - log(-log1p(-u_v))) per row
 * (tag DRAFT, slot j; R5, R14).  z [B][V] fp32 (row stride ld floats); out [B]. */
SEED_API seed_status seed_op_draft_sample(const float* z, int32_t ld, int32_t B, int32_t V, float temperature,
                                 uint64_t seed, const uint32_t* sids, const int32_t* rs, int32_t j,
                                 int32_t* out, void* stream);

/* k_config trees (§3.2, App. B; SPEC.md S:90-134;
 * DESIGN.md R36).  A tree of K = n_counts levels is laid out breadth-first: node 0 is the root (the
 * context), each depth-(d-1) node has counts[d-1] children, children are contiguous.
 *
 * K1T: the children of node `node` for every row: the `m` largest keys of the exponential race
 * over z [B][V] (row stride ld floats) with tag DRAFT, slot node + 1 -- m distinct ids drawn without
 * replacement from softmax(fl32(z / T)), in draw order.  out: device int32, row b written at
 * out[b * out_stride + first .. + m).  1 <= m <= 8. */
SEED_API seed_status seed_op_draft_topk(const float* z, int32_t ld, int32_t B, int32_t V, float temperature,
                                        uint64_t seed, const uint32_t* sids, const int32_t* rs, int32_t node,
                                        int32_t m, int32_t* out, int32_t out_stride, int32_t first, void* stream);

/* K4T: verification of a drafted tree by recursive rejection (DESIGN R36): zt, zd [B][n+1][V] fp32 --
 * row i = the target / draft logits after node i's path (zd rows of leaves unused); tok [B][n+1]
 * node tokens (tok[.][0] unused); counts_host [n_counts] the k_config (each 1..8, n_counts <= 15).
 * out_tok [B][K+1]: the accepted path's tokens, then the correction or bonus token, -1 padding;
 * out_cnt [B]; out_node [B][K] (optional): accepted node indices, -1 padding. */
SEED_API seed_status seed_op_verify_tree(const float* zt, const float* zd, const int32_t* tok, int32_t B,
                                         const int32_t* counts_host, int32_t n_counts, int32_t V, float temperature,
                                         uint64_t seed, const uint32_t* sids, const int32_t* rs, int32_t bonus,
                                         int32_t* out_tok, int32_t* out_cnt, int32_t* out_node, void* stream);

/* One decoder layer of `shape` on hidden states (per-layer parity).
 * w: host array of the 9 device pointers of seed_model_weights.layers for one layer.
 * x_in/x_out: fp32 [M][d]; the M rows are q_len consecutive positions
 * ctx .. ctx + M - 1 of one sequence whose earlier keys/values are k_prev/v_prev
 * (bf16 [ctx][Hk][Dh], may be NULL when ctx == 0).  k_new/v_new (optional): bf16
 * [M][Hk][Dh] as appended to the cache. */
SEED_API seed_status seed_op_decoder_layer(const seed_model_shape* shape, const void* const* w, const float* x_in,
                                  int32_t M, int32_t ctx, const void* k_prev, const void* v_prev,
                                  float* x_out, void* k_new, void* v_new, void* stream);

/* The same layer over a TREE of M <= 64 rows (k_config verification, §3.2 P:107-113 and
 * Figure 7 of App. B; R36): parent (host int32 [M]): parent[0] = -1 (the root,
 * the sequence's next token at position ctx), 0 <= parent[i] < i otherwise.  Row i is rotated at
 * position ctx + depth(i) and attends to the ctx cached keys and to its ancestors and itself only,
 * so every row equals the last row of the causal layer over its root-to-row path.  k_new/v_new: the
 * rows' K/V as appended (row i at cache slot ctx + i, rotated at its tree position; the accepted
 * path compacts into consecutive slots without re-rotation).  Errors: SEED_EINVAL on a malformed
 * parent array or M > 64. */
SEED_API seed_status seed_op_decoder_layer_tree(const seed_model_shape* shape, const void* const* w, const float* x_in,
                                       int32_t M, int32_t ctx, const int32_t* parent, const void* k_prev,
                                       const void* v_prev, float* x_out, void* k_new, void* v_new, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SEED_OPS_H_ */
