/*
 * seed.h -- C ABI of libseed: SeeD's rounds-scheduled draft-then-verify round on B200 (sm_100a).
 *
 * Paper: "SeeD: Accelerating Reasoning Tree Construction via Scheduled Speculative
 * Decoding", arXiv 2406.18200.  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, Rk = reading k in DESIGN.md ("Readings of the paper").
 *
 * One round (Alg. 1, in the lock-step batched reading R9):
 *   seed_schedule_round  a1  FCFS pop of <= C ready, undone streams
 *   seed_draft_round     a2  gamma autoregressive draft steps per stream
 *   seed_verify          a3  one batched target forward over B(gamma+1)
 *                        a4  fused accept / resample / bonus              (R1-R4)
 *                        a5  commit + KV rollback                         (R6, R7)
 *                        a6  all-gather of emitted tokens (world > 1)
 *
 * Conventions (all calls):
 *   - Every call returns seed_status; no C++ exception crosses the ABI.
 *   - Device work is enqueued on the caller's CUDA stream (`stream`, a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Outputs are valid after the
 *     stream is synchronised.
 *   - Ownership: the caller owns the weights it passes to seed_init only for the
 *     duration of seed_init (the library packs them into its own layout, R18), and
 *     owns every output buffer.  The library owns its packed weights, the KV pool,
 *     scratch and the scheduler and frees them in seed_destroy.
 *   - A CUDA or NCCL failure poisons the context: every later call returns
 *     SEED_ESTATE until seed_destroy.  seed_last_error() gives the message.
 *   - Threading: one context per GPU; calls on one context are serialised by the caller.
 *   - There is no CPU fallback: without a usable sm_100a device seed_init fails
 *     with SEED_ECUDA.
 */
#ifndef SEED_H_
#define SEED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEED_ABI_VERSION 1

#if defined(__GNUC__)
#define SEED_API __attribute__((visibility("default")))
#else
#define SEED_API
#endif

typedef struct seed_ctx_s* seed_ctx;

typedef enum {
  SEED_OK = 0,
  SEED_EINVAL = 1,     /* bad argument: shape, id >= vocab, vocab mismatch */
  SEED_ENOMEM = 2,     /* device or host allocation failed, KV pool exhausted */
  SEED_ECUDA = 3,      /* CUDA runtime / driver error (context poisoned) */
  SEED_ENCCL = 4,      /* NCCL error (context poisoned) */
  SEED_ESTATE = 5,     /* context poisoned, or call out of order (verify before draft) */
  SEED_ECAPACITY = 6,  /* more streams than max_streams, batch larger than max_batch */
  SEED_EDEVICE = 7,    /* device contract violation reported through the error word */
  SEED_ENOTFOUND = 8   /* unknown global stream id */
} seed_status;

/* Llama-2 shape (R15: RMSNorm eps, RoPE theta 1e4 rotate-half, SwiGLU, untied head, no bias).
 * Constraints: d_model % 64 == 0, d_ff % 64 == 0, head_dim = d_model / n_heads in {32, 64, 128},
 * n_kv_heads divides n_heads (0 = n_heads). */
typedef struct {
  int32_t vocab, d_model, n_layers, n_heads, n_kv_heads, d_ff;
  float rms_eps;     /* 1e-5 */
  float rope_theta;  /* 1e4 */
} seed_model_shape;

/* Device pointers to bf16 tensors in the HF layout (row-major [out][in]).
 * layers[9*l + i] for layer l, i = 0..8:
 *   0 wq [H*Dh][d]   1 wk [Hk*Dh][d]   2 wv [Hk*Dh][d]   3 wo [d][H*Dh]
 *   4 w_gate [ff][d] 5 w_up [ff][d]    6 w_down [d][ff]  7 attn_norm [d]  8 mlp_norm [d] */
typedef struct {
  const void* embed;        /* [V][d] */
  const void* const* layers;/* host array of 9*n_layers device pointers */
  const void* final_norm;   /* [d] */
  const void* lm_head;      /* [V][d] */
} seed_model_weights;

#define SEED_FLAG_PROFILE 1u  /* bracket every GEMM launch with CUDA events (seed_get_profile) */

typedef struct {
  seed_model_shape draft, target;        /* draft.vocab must equal target.vocab */
  seed_model_weights draft_w, target_w;
  int32_t gamma;                         /* draft length gamma >= 1 (the paper's k) */
  float temperature;                     /* T > 0: softmax(z / T) for both models (R4) */
  uint64_t seed;                         /* Philox key (R5) */
  int32_t bonus;                         /* 1 = bonus token on full acceptance (R1), 0 = Alg. 1 literal */
  int32_t max_new_tokens;                /* l; streams stop at exactly l new tokens (R7) */
  int32_t max_streams;                   /* resident streams (stream slots) */
  int32_t max_batch;                     /* capacity C per round (R11) */
  int32_t max_ctx;                       /* longest |T_s| + gamma + 1 supported */
  int32_t page_tokens;                   /* KV page size in tokens: 16 (if 0), 32, 64, 128 or 256 -- a page
                                            holds whole 16-key attention tiles; anything else: EINVAL */
  int64_t kv_pool_bytes;                 /* KV pool size; 0 = enough for max_streams x max_ctx */
  int32_t rank, world;                   /* data-parallel replica index / count (replicas, R20) */
  const void* nccl_id;                   /* 128-byte ncclUniqueId (same on all ranks) or NULL if world == 1 */
  uint32_t flags;                        /* SEED_FLAG_* */
  /* k_config tree rounds (§3.2, App. B; R36): n_tree = 0 runs
   * the chain; n_tree = K > 0 drafts a tree with tree_counts[d] candidates per node at depth d
   * (1..8 each), verified by one target pass with tree attention and recursive rejection.  gamma
   * must equal K; the tree holds at most 64 rows (root + nodes).  Tokens are emitted like the chain's
   * (at most K + 1 per round) and the accepted path's KV is compacted in place. */
  int32_t n_tree;
  int32_t tree_counts[8];
} seed_config;

/* Validates shapes, packs weights (R18), allocates the KV pool and scratch, builds TMA
 * descriptors, creates the NCCL communicator when world > 1. */
SEED_API seed_status seed_init(const seed_config* cfg, seed_ctx* out);

/* Alg. 1 "Initialize": prefill both models with the prefix and enqueue the stream
 * FCFS with ready = 1.  prefix_host: host int32 token ids, len >= 2 (R30), ids < vocab;
 * global_id < 2^31, not already present on this rank (a removed id may be added again).
 * Synchronous with respect to `stream`.  ESTATE between seed_draft_round and seed_verify. */
SEED_API seed_status seed_add_stream(seed_ctx ctx, uint32_t global_id, const int32_t* prefix_host,
                            int32_t len, void* stream);

/* ToT siblings (Alg. 2 line P:738: the n thoughts of a state share its prefix; §4.1 "the input
 * instructions are the same"): adds stream `global_id` with the same prefix as `src_global_id`
 * from src's prefilled K/V instead of recomputing the prefill: pages holding only positions
 * < len-2 (index < (len-2)/page_tokens) are SHARED (refcounted; rounds write positions >= len-2:
 * the draft's first step rewrites len-2, R22), the page holding position len-2 is copied on the
 * device (cudaMemcpyAsync on `stream`).  The new stream is bit-identical to seed_add_stream(global_id, same prefix); both
 * streams run and are removed independently (a page returns to the pool with its last
 * reference).  Errors: unknown src or
 * duplicate id -> EINVAL; src has already run a round -> ESTATE (not poisoning); no free slot ->
 * ECAPACITY; no free pages -> ENOMEM.  Synchronous with respect to `stream`. */
SEED_API seed_status seed_fork_stream(seed_ctx ctx, uint32_t src_global_id, uint32_t global_id, void* stream);

/* a1: completes the previous round on the host (waits for its counts), re-enqueues undone
 * streams at the tail in batch order, then pops up to min(cap, max_batch)
 * ready, undone streams FCFS (ties -> lowest global id, R10).
 * batch_ids: host buffer of `cap` int32 (global ids).  *n = 0 when every own stream is done.
 * Returns SEED_EDEVICE (after scheduling normally) when the completed round raised the device
 * error word (seed_device_status). */
SEED_API seed_status seed_schedule_round(seed_ctx ctx, int32_t* batch_ids, int32_t cap, int32_t* n);

/* a2: gamma draft steps for the batch (K1: batched draft forward + Philox race sampler).
 * batch_ids: host array of n global ids returned by seed_schedule_round; n = 0 is allowed (a
 * rank whose streams are done still takes part in the round's exchange, world > 1). */
SEED_API seed_status seed_draft_round(seed_ctx ctx, const int32_t* batch_ids, int32_t n, void* stream);

/* a3-a6: target verify forward, fused vocabulary kernel, rollback, all-gather.
 * World > 1: EVERY rank calls seed_draft_round + seed_verify EVERY round (n = 0 once its own
 * streams are done: it then contributes an empty exchange block) until seed_global_pending
 * reports 0 -- the all-gather is collective.
 * out_tok: device int32 [n][gamma+1]: x_1..x_a, y, then -1 padding (R1; Alg. 1 emits
 *          x_1..x_gamma only when bonus = 0 and a = gamma).
 * out_cnt: device int32 [n]: tokens emitted this round (before truncation to l).
 * Either may be NULL.  Returns SEED_ESTATE if seed_draft_round was not called for this batch. */
SEED_API seed_status seed_verify(seed_ctx ctx, const int32_t* batch_ids, int32_t n,
                        int32_t* out_tok, int32_t* out_cnt, void* stream);

/* Convenience for end-to-end measurement: one whole round with HOST outputs.
 * out_tok_host [n][gamma+1], out_cnt_host [n]; includes the device->host copies. */
SEED_API seed_status seed_round_host(seed_ctx ctx, const int32_t* batch_ids, int32_t n,
                            int32_t* out_tok_host, int32_t* out_cnt_host, void* stream);

/* Validated new tokens of a stream (after the last completed round), truncated to l.
 * Works for any global id known to this rank (own or gathered from peers). */
SEED_API seed_status seed_get_tokens(seed_ctx ctx, uint32_t global_id, int32_t* dst_host, int32_t cap,
                            int32_t* len);

/* info[0..7] = |T_s|, L_s, r_s, done, len_t (target KV entries), len_d (draft KV entries),
 * pages held, slot. */
SEED_API seed_status seed_stream_info(seed_ctx ctx, uint32_t global_id, int32_t* info);

/* Frees the stream's pages and slot (pruned ToT node) and forgets the id (scheduler entry and
 * tokens: read them with seed_get_tokens first).  ESTATE between seed_draft_round and seed_verify. */
SEED_API seed_status seed_remove_stream(seed_ctx ctx, uint32_t global_id);

/* Streams not yet done on ALL ranks after the last completed round (the sum of the undone counts
 * every rank posted in its exchange block); world == 1 before any round: this rank's count.
 * Completes the pending round first.  The loop of a multi-GPU run:
 *   do { n = schedule(); draft(n); verify(n); } while (global_pending() > 0)
 * stops on the same round on every rank. */
SEED_API seed_status seed_global_pending(seed_ctx ctx, int64_t* n);

/* Device error word (SEED_EDEVICE, cumulative since seed_init): bit 0 (1) a token id outside
 * [0, vocab) reached an embedding gather (the row read id 0 instead); bit 1 (2) a sampling race
 * found no finite key (non-finite logits).  fallbacks: K4 empty-residual fallbacks (R3: p <= q
 * everywhere after rounding; the bonus rule on the same row is used, as in the oracle). */
SEED_API seed_status seed_device_status(seed_ctx ctx, uint32_t* bits, int64_t* fallbacks);

/* Forward of one model over `tokens` from an empty cache (debug / parity; ESTATE between
 * seed_draft_round and seed_verify):
 * which = 0 draft, 1 target; logits_dev: device fp32 [n][vocab]. Synchronous w.r.t. stream. */
SEED_API seed_status seed_forward_logits(seed_ctx ctx, int32_t which, const int32_t* tokens_host, int32_t n,
                                float* logits_dev, void* stream);

/* Last-round diagnostics (device pointers, valid until the next seed_verify):
 * target logits [n][gamma+1][V], draft logits [n][gamma][V] (fp32), draft tokens [n][gamma]. */
SEED_API seed_status seed_last_round_buffers(seed_ctx ctx, const float** tgt_logits, const float** drf_logits,
                                    const int32_t** draft_tokens);

/* Profiling (SEED_FLAG_PROFILE), since the last reset, measured on the device with %globaltimer
 * inside the GEMM kernel (launches inside CUDA graphs with PDL have no stream events between them):
 * gemm_ms = sum over GEMM launches of (last CTA end - dependency release), i.e. the time each GEMM
 * holds the critical path; gemm_span_ms = sum of (last CTA end - first CTA start), which also
 * counts the weight prefetch overlapped with the predecessor; gemm_bytes = algorithmic bytes
 * (weights + activations + fp32 outputs); kernel_launches = libseed kernels launched. */
SEED_API seed_status seed_get_profile(seed_ctx ctx, double* gemm_ms, int64_t* gemm_launches,
                             double* gemm_bytes, int64_t* kernel_launches, double* gemm_span_ms);
SEED_API seed_status seed_reset_profile(seed_ctx ctx);
/* Switch the device timing records on or off between rounds (the context must have been created
 * with SEED_FLAG_PROFILE; the timing atomics cost ~2% of a round, so a benchmark times its
 * rounds with profiling off).  SEED_ESTATE between seed_draft_round and seed_verify. */
SEED_API seed_status seed_set_profile(seed_ctx ctx, int32_t on);
/* GEMM trace of the most recent round (SEED_FLAG_PROFILE): out[4*i..4*i+3] = globaltimer ns of
 * launch i: first CTA start, dependency release (PDL wait returned), last CTA end, 0.
 * out: host buffer of 4*cap uint64; *n = launches written (in round launch order). */
SEED_API seed_status seed_gemm_trace(seed_ctx ctx, uint64_t* out, int32_t cap, int32_t* n);
/* Diagnostics (SEED_FLAG_PROFILE and env SEED_CTA_TRACE=1 at seed_init): per-CTA phase
 * timestamps (globaltimer ns) of launch `launch` (index as in seed_gemm_trace) of the most recent
 * round.  out: host buffer of 8192 uint64.  GEMM launches: row c (16 words) = CTA c: start,
 * producer release, producer done, first stage full, MMA done, first accumulator ready, epilogue
 * done, end, partial stored, contributors seen, reduce done, finish done, ring consumed, first
 * refill.  Attention launches: row b (8 words) = linear block b: start, release, tiles ready,
 * chunk result stored, merge ticket, end.  Words a launch did not reach are 0 or stale.
 * *n_cta = 8192 (words written), or 0 when tracing is off. */
SEED_API seed_status seed_gemm_cta_trace(seed_ctx ctx, int32_t launch, uint64_t* out, int32_t* n_cta);

SEED_API const char* seed_last_error(seed_ctx ctx);
SEED_API void seed_destroy(seed_ctx ctx);

/* 128-byte NCCL unique id for world > 1 (call on rank 0, broadcast, pass in seed_config). */
SEED_API seed_status seed_nccl_unique_id(void* out128);

/* ---- host-only pieces (no GPU needed; tested on CPU) ------------------------------- */

/* FCFS rounds scheduler (H1): the object seed_schedule_round drives. */
typedef struct seed_sched_s* seed_sched;
SEED_API seed_status seed_sched_create(const int32_t* ids, int32_t n, seed_sched* out);
SEED_API seed_status seed_sched_add(seed_sched s, int32_t id);
/* pop <= cap ready, undone ids FCFS; *n = 0 and SEED_ESTATE if nothing is ready but work remains */
SEED_API seed_status seed_sched_pop(seed_sched s, int32_t* out, int32_t cap, int32_t* n);
/* after verification: ready = 1; undone ids re-enter at the tail in batch order */
SEED_API seed_status seed_sched_complete(seed_sched s, const int32_t* batch, const int32_t* done, int32_t n);
SEED_API int32_t seed_sched_all_done(seed_sched s);
/* forget an id entirely (queue entry, ready / done flags): a removed stream's id may be re-added */
SEED_API seed_status seed_sched_remove(seed_sched s, int32_t id);
SEED_API void seed_sched_destroy(seed_sched s);

/* Token table merged from per-rank round records (a6).  Record layout (int32):
 *   [0] global id  [1] emitted count c (after truncation)  [2..2+c) tokens ; stride gamma + 3. */
typedef struct seed_table_s* seed_table;
SEED_API seed_status seed_table_create(int32_t record_stride, seed_table* out);
SEED_API seed_status seed_table_merge(seed_table t, const int32_t* records, int32_t n_records);
SEED_API seed_status seed_table_get(seed_table t, uint32_t global_id, int32_t* dst, int32_t cap, int32_t* len);
SEED_API seed_status seed_table_erase(seed_table t, uint32_t global_id);
SEED_API void seed_table_destroy(seed_table t);

/* Round book of one rank (H1 + a5 + a6): the host state seed_schedule_round /
 * seed_verify drive inside a context, exported so the multi-rank protocol runs on CPU too.
 *   own streams: validated tokens T, L (new tokens, done at l = max_new, R7), r (stream-local
 *   round, R5); the FCFS scheduler; the token table of other ranks' streams.
 * Exchange block (int32, seed_book_block_ints() = cap * (gamma + 3) + 1 words): cap records
 *   [gid, c, tok_0 .. tok_gamma] (c tokens committed this round after truncation to l; padding
 *   records have gid = -1), then one word: this rank's streams still undone after the round.
 * Protocol (every rank, every round, in lock step): schedule (a batch, possibly empty) ->
 *   the round -> pack (device: K5) -> all-gather of the blocks in rank order -> complete.
 *   Stop when seed_book_global_pending() == 0: the same value on every rank (it sums the gathered
 *   tails), so no rank leaves a collective the others still enter. */
typedef struct seed_book_s* seed_book;
SEED_API seed_status seed_book_create(int32_t gamma, int32_t max_new, int32_t cap, int32_t world, int32_t rank,
                                      seed_book* out);
/* register one of this rank's streams (prefix host int32, len >= 1; duplicate id -> EINVAL) */
SEED_API seed_status seed_book_add(seed_book b, uint32_t global_id, const int32_t* prefix, int32_t len);
SEED_API seed_status seed_book_remove(seed_book b, uint32_t global_id);
/* a1: FCFS pop of <= min(cap, book cap) ready, undone own streams; *n = 0 once all are done */
SEED_API seed_status seed_book_schedule(seed_book b, int32_t* ids, int32_t cap, int32_t* n);
/* a5 record formation on the host (the device path's K5 writes the same block): out_tok
 * [n][gamma+1], out_cnt [n] as seed_verify returns them; block: seed_book_block_ints() words.
 * Does not change the book (seed_book_complete applies the round). */
SEED_API seed_status seed_book_pack(seed_book b, const int32_t* ids, int32_t n, const int32_t* out_tok,
                                    const int32_t* out_cnt, int32_t* block);
/* a6: apply the gathered blocks (world blocks, rank order): own records update T / L / r / done
 * and requeue undone streams at the tail in batch order; other ranks' records go
 * to the token table; the tails give the global pending count.  EINVAL on a malformed block. */
SEED_API seed_status seed_book_complete(seed_book b, const int32_t* blocks, int32_t n_blocks);
/* streams undone on all ranks after the last completed exchange; -1 before the first */
SEED_API seed_status seed_book_global_pending(seed_book b, int64_t* n);
SEED_API seed_status seed_book_tokens(seed_book b, uint32_t global_id, int32_t* dst, int32_t cap, int32_t* len);
/* info[0..4] = |T|, L, r, done, prompt length (own streams; ENOTFOUND otherwise) */
SEED_API seed_status seed_book_info(seed_book b, uint32_t global_id, int32_t* info);
SEED_API int32_t seed_book_block_ints(seed_book b);
SEED_API void seed_book_destroy(seed_book b);

#ifdef __cplusplus
}
#endif
#endif /* SEED_H_ */
