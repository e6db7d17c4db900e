// engine.cu -- the C ABI of seed.h / seed_ops.h: models, paged KV pool, the round, NCCL.
//
// Host orchestration of one round (Alg. 1 in the lock-step batched reading, DESIGN R9):
//   seed_schedule_round  -> completes round r-1 on the host mirrors, FCFS pop (H1)
//   seed_draft_round     -> gamma batched draft forwards + K1 sampler
//   seed_verify          -> batched target forward, K4, K5, all-gather
// Every arithmetic step runs in the kernels of gemm.cu / epilogue.cu / attention.cu /
// vocab.cu; this file only plans, allocates, uploads descriptors and launches.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/seed.h"
#include "../../include/seed_ops.h"
#include "host_book.h"
#include "kernels.h"

using seed::GemmPlan;
using seed::KVLayout;
typedef __nv_bfloat16 bf16;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen'd, a6 only)
struct Id128 {
  char b[128];
};
typedef int (*InitRankFn)(void**, int, Id128, int);
struct Nccl {
  void* lib = nullptr;
  int (*get_id)(Id128*) = nullptr;
  InitRankFn init = nullptr;
  int (*allgather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*destroy)(void*) = nullptr;
  bool load() {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!lib) lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) return false;
    get_id = (int (*)(Id128*))dlsym(lib, "ncclGetUniqueId");
    init = (InitRankFn)dlsym(lib, "ncclCommInitRank");
    allgather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(lib, "ncclAllGather");
    destroy = (int (*)(void*))dlsym(lib, "ncclCommDestroy");
    return get_id && init && allgather && destroy;
  }
};
Nccl g_nccl;
constexpr int kNcclInt32 = 2;

// ------------------------------------------------------------------ descriptor arena
// pinned host staging + device mirror; one H2D copy per upload
struct Arena {
  int32_t* host = nullptr;
  int32_t* dev = nullptr;
  size_t cap = 0, used = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
  cudaError_t init(size_t ints) {
    cap = ints;
    cudaError_t e = cudaMallocHost(&host, cap * 4);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&dev, cap * 4);
    if (e != cudaSuccess) return e;
    return cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  }
  void begin() {
    if (pending) cudaEventSynchronize(done);
    pending = false;
    used = 0;
  }
  size_t alloc(size_t n) {  // returns offset (ints), 16-byte aligned
    size_t off = (used + 3) & ~size_t(3);
    if (off + n > cap) return (size_t)-1;
    used = off + n;
    return off;
  }
  cudaError_t upload(cudaStream_t st) {
    if (!used) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(dev, host, used * 4, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    pending = true;
    return cudaEventRecord(done, st);
  }
  void destroy() {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    if (done) cudaEventDestroy(done);
  }
};

struct Segment {  // rows of one sequence in a forward chunk
  int slot, pos0, q_len;
  int tok_off;    // offset of host tokens in the arena (-1: tokens from a device source)
  int stable = 0; // cache positions written before this round (attention may prefetch them early)
};

struct TokSrc {   // device token source for rows (row m reads dev[m * stride])
  const int32_t* dev;
  int stride;
};

struct Model {
  seed_model_shape sh{};
  int d = 0, H = 0, Hk = 0, Dh = 0, ff = 0, V = 0, L = 0, nqkv = 0;
  bf16 *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  std::vector<bf16*> wqkv, wo, wgu, wdown, an, mn;
  std::vector<GemmPlan> pq, po, pgu, pd;
  GemmPlan plm{};
  // paged KV
  KVLayout kv{};
  CUtensorMap tmkv;                 // 2D tensor map of the KV pool (attention's page-block copies)
  int32_t* page_table_dev = nullptr;
  int32_t* page_table = nullptr;          // pinned host mirror [slots][max_pages]
  std::vector<int32_t> free_pages;
  std::vector<int32_t> refs;              // slots referencing each page (ToT siblings share full prefix pages)
  std::vector<int32_t> held;              // pages held per slot
  size_t n_pages = 0;
  float2* rope = nullptr;
  // activations for up to m_cap rows per forward chunk
  int m_cap = 0;
  float* x = nullptr;
  float* y = nullptr;    // fp32 QKV output [m_cap][nqkv]
  float *ssq_a = nullptr, *ssq_b = nullptr;  // per-tile sums of squares of the residual [d/128][m_cap]
  bf16* h = nullptr;     // bf16(x * w_norm): operand of QKV / gate-up / LM head (B1, R24)
  bf16* act = nullptr;   // bf16(silu(g) * u): operand of the down projection (B4)
  bf16* attn = nullptr;  // attention output (bf16 operand of the O projection, B3)
  seed::AttnWorkspace aws{};
  std::vector<bf16*> owned;
};

struct SlotState {  // one stream slot; the validated tokens live in the round book (host_book.h)
  uint32_t gid = 0;
  bool used = false;
  int len_t = 0, len_d = 0;   // KV entries of the target / draft cache (R6)
};

struct ChunkDesc {
  int M, n_seq, max_q_len, max_kv;
  const int32_t *pos, *slot, *q_start, *q_len, *kv_len, *seq_slot, *seq_stable, *compact;  // device (slot: per row)
  const int32_t* row_pos = nullptr;   // tree rows (R36): per-row RoPE positions and attended tree rows
  const uint64_t* anc = nullptr;
  const int32_t* tree_base = nullptr; // per sequence: cache slot of the tree's root (bit 0 of anc)
  bool rowmap = false;                // logits rows through `compact` even when every row has logits
  bool pre_embedded = false;          // x, ssq and h of the rows were written by the previous step's K1
  TokSrc tok;
  int n_logits;
  const int32_t* logit_rows;  // device [n_logits]: chunk row of each logits row
  float* Y;       // logits destination for compact row 0
  int ldY;
};

struct RoundPlan {  // descriptors of one round at batch-size-determined arena offsets
  int n = 0;
  int64_t key_draft = 0, key_verify = 0;  // graph keys: batch size and attention chunk counts
  int dk_raw = 0, vk_raw = 0;             // longest draft / target context of the round (unrounded)
  size_t o_sid = 0, o_r = 0, o_sl = 0, o_last = 0, o_out = 0;  // o_out: undone own streams outside the batch
  std::vector<ChunkDesc> draft, verify;
  std::vector<int> verify_b0;
};

struct RoundGraphEntry {
  cudaGraphExec_t exec = nullptr;
  double gemm_bytes = 0;
  int64_t gemms = 0, kernels = 0;
};

constexpr int kMaxChunkRows = 1024;   // rows per forward chunk (the GEMM runs token tiles of 256)
constexpr size_t kCtaRec = 8192;  // per-launch per-CTA trace words (GEMM: 148 x 16, attention: grid x 8)

}  // namespace

struct seed_ctx_s {
  seed_config cfg{};
  std::string err;
  bool poisoned = false;
  int dev = 0;
  Model dm, tm;                   // draft, target
  int P = 16, max_pages = 0, n_slots = 0;
  std::map<std::tuple<const void*, int, int>, CUtensorMap> xmaps;
  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> ymaps;
  Arena arena;
  // stream registry
  std::vector<SlotState> slots;
  std::unordered_map<uint32_t, int> gid2slot;
  seed_book book = nullptr;       // FCFS scheduler, own streams' tokens, other ranks' tokens (a1, a5, a6)
  // device state (K5)
  seed::StreamState ds{};
  // per-round buffers (capacity C = max_batch)
  int C = 0, G = 0;
  float *tgt_logits = nullptr, *drf_logits = nullptr;
  int32_t *xs = nullptr, *vtok = nullptr, *out_tok = nullptr, *out_cnt = nullptr, *out_acc = nullptr;
  void* verify_work = nullptr;     // K4 scratch (vocab_verify_work_bytes; tickets zero between launches)
  int32_t *records = nullptr, *records_all = nullptr, *records_host = nullptr;   // exchange blocks (a6)
  int32_t* out_host = nullptr;   // pinned staging of seed_round_host's results: [C][gamma + 1] tokens, [C] counts
  int block_ints = 0;             // words per rank's block: C records of gamma + 3, then the undone count
  // device error word (SEED_EDEVICE): [0] contract-violation bits, [1] empty-residual fallbacks (K4)
  int32_t* dev_err = nullptr;
  int32_t* err_host = nullptr;    // pinned copy, refreshed at the end of every verify
  uint32_t err_bits_seen = 0;
  int64_t fallbacks = 0;
  uint32_t* sids_dev = nullptr;
  int32_t* rs_dev = nullptr;
  int32_t* slots_dev = nullptr;
  cudaEvent_t round_done = nullptr;
  std::vector<int32_t> last_batch;  // global ids of the batch in flight
  std::vector<int32_t> drafted;     // batch drafted and not yet verified
  bool draft_called = false;        // seed_draft_round called for `drafted` (n may be 0 when world > 1)
  RoundPlan plan;
  bool round_pending = false;
  // k_config tree rounds (R36; tree.n == 0: chain rounds)
  struct Tree {
    int n = 0, nn = 1;                       // levels K, rows per stream (root + nodes)
    std::vector<int> counts, parent, depth, first, cnt, lvl_start, lvl_len;
    std::vector<uint64_t> anc;
    int32_t* ch_dev = nullptr;               // device [2][nn]: first child, child count (K4T)
    int32_t* tok_lvl = nullptr;              // device: draft input tokens of levels 2..K, level-major [B][len]
    std::vector<size_t> lvl_off;             // offset of level d's block in tok_lvl
    int32_t* tree_tok = nullptr;             // device [C][nn]: root + node tokens (verify input)
    int32_t* out_node = nullptr;             // device [C][K]: accepted nodes (-1 pad)
  } tree;
  // NCCL
  void* comm = nullptr;
  // CUDA graphs of the round, one pair per batch size (R23)
  bool use_graphs = true;
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::map<int64_t, RoundGraphEntry> round_graphs;   // draft + verify of a round, one graph (R23)
  bool draft_deferred = false;                   // seed_draft_round planned a round, not launched
  // profiling: per-GEMM globaltimer records accumulated on the device
  bool profile = false, in_round = false;
  unsigned long long *timing_rec = nullptr, *timing_acc = nullptr, *timing_last = nullptr;
  unsigned long long* cta_rec = nullptr;  // SEED_CTA_TRACE=1: [rec_cap][kCtaRec] per-CTA phases
  int last_draft_recs = 0, last_verify_recs = 0;
  std::map<int, int> draft_recs;  // records of the draft phase per batch size
  int rec_cap = 0, rec_used = 0;
  double round_gemm_bytes = 0, gemm_bytes = 0;
  int64_t round_gemms = 0, gemm_launches = 0, kernel_launches = 0;
};

namespace {

#define CK(expr)                                                                  \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) return fail(ctx, SEED_ECUDA, #expr, cudaGetErrorString(_e)); \
  } while (0)

seed_status fail(seed_ctx ctx, seed_status s, const char* what, const char* detail) {
  if (ctx) {
    ctx->err = std::string(what) + ": " + (detail ? detail : "");
    if (s == SEED_ECUDA || s == SEED_ENCCL) ctx->poisoned = true;
  }
  return s;
}

int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

const CUtensorMap* xmap(seed_ctx ctx, const bf16* buf, int K, int rows_cap, int M) {
  const int m_pad = seed::gemm_mpad(M);
  auto key = std::make_tuple((const void*)buf, K, m_pad);
  auto it = ctx->xmaps.find(key);
  if (it != ctx->xmaps.end()) return &it->second;
  CUtensorMap m;
  if (!seed::encode_tmap_2d(&m, buf, (uint64_t)K, (uint64_t)rows_cap, 64, (uint32_t)m_pad)) return nullptr;
  return &(ctx->xmaps[key] = m);
}

// the next device timing record of the round being enqueued (profiling), else null; cta: the
// launch's per-CTA trace words (SEED_CTA_TRACE=1)
unsigned long long* next_rec(seed_ctx ctx, unsigned long long** cta = nullptr) {
  if (!(ctx->profile && ctx->in_round && ctx->rec_used < ctx->rec_cap)) return nullptr;
  if (cta && ctx->cta_rec) *cta = ctx->cta_rec + (size_t)ctx->rec_used * kCtaRec;
  return ctx->timing_rec + 4 * ctx->rec_used++;
}

seed_status run_gemm(seed_ctx ctx, const GemmPlan& p, int M, const seed::GemmIO& io, cudaStream_t st) {
  unsigned long long* cta = nullptr;
  unsigned long long* rec = next_rec(ctx, &cta);
  CK(seed::gemm_run(p, M, io, st, rec, cta));
  if (ctx->in_round) {
    // algorithmic bytes: weights + bf16 X + output (fp32 Y; residual: read + write x, write bf16 h;
    // SwiGLU: bf16 act of half the width)
    const double yout = io.ymode == 0 ? 4.0 : (io.ymode == 1 ? 10.0 : 1.0);
    ctx->round_gemm_bytes += (double)p.N * p.K * 2 + (double)M * p.K * 2 + (double)M * p.N * yout;
    ctx->round_gemms++;
  }
  ctx->kernel_launches++;
  return SEED_OK;
}

// X operand from a bf16 activation buffer by TMA
// the output's store map (whole-tile tensor stores, gemm.cu): exactly M rows starting at `ptr`
const CUtensorMap* ymap(seed_ctx ctx, const void* ptr, bool fp32, int cols, int ld, int M) {
  const int m_pad = seed::gemm_mpad(M);
  if (m_pad > 256) return nullptr;
  auto key = std::make_tuple(ptr, (int)fp32 * (1 << 30) + cols, ld, M);
  auto it = ctx->ymaps.find(key);
  if (it != ctx->ymaps.end()) return &it->second;
  CUtensorMap m;
  if (!seed::encode_tmap_store(&m, ptr, fp32, (uint64_t)cols, (uint64_t)M, (uint64_t)ld, fp32 ? 128 : 64, (uint32_t)m_pad))
    return nullptr;
  return &(ctx->ymaps[key] = m);
}

seed::GemmIO io_tma(seed_ctx ctx, const bf16* X, int K, int rows_cap, int M, float* Y, int ldY) {
  seed::GemmIO io;
  io.tmX = xmap(ctx, X, K, rows_cap, M);
  io.Y = Y;
  io.ldY = ldY;
  return io;
}

// ------------------------------------------------------------------ model setup
seed_status check_shape(const seed_model_shape& s) {
  if (s.vocab <= 0 || s.d_model <= 0 || s.n_layers <= 0 || s.n_heads <= 0 || s.d_ff <= 0) return SEED_EINVAL;
  if (s.d_model % 64 || s.d_ff % 64 || s.d_model % s.n_heads) return SEED_EINVAL;
  const int hk = s.n_kv_heads ? s.n_kv_heads : s.n_heads;
  if (s.n_heads % hk) return SEED_EINVAL;
  const int dh = s.d_model / s.n_heads;
  if (dh != 32 && dh != 64 && dh != 128) return SEED_EINVAL;
  return SEED_OK;
}

seed_status copy_rows(seed_ctx ctx, bf16* dst, const void* src, size_t elems) {
  CK(cudaMemcpy(dst, src, elems * 2, cudaMemcpyDeviceToDevice));
  return SEED_OK;
}

// pack weights into the library layout (R18): QKV stacked, gate/up interleaved in 64-row blocks
seed_status build_model(seed_ctx ctx, Model& m, const seed_model_shape& sh, const seed_model_weights& w, int m_cap,
                        int slots, int max_pages, size_t pool_pages, int max_pos) {
  seed_status s = check_shape(sh);
  if (s != SEED_OK) return fail(ctx, s, "seed_init", "bad model shape");
  if (!w.embed || !w.layers || !w.final_norm || !w.lm_head) return fail(ctx, SEED_EINVAL, "seed_init", "null weight");
  m.sh = sh;
  m.d = sh.d_model;
  m.H = sh.n_heads;
  m.Hk = sh.n_kv_heads ? sh.n_kv_heads : sh.n_heads;
  m.Dh = m.d / m.H;
  m.ff = sh.d_ff;
  m.V = sh.vocab;
  m.L = sh.n_layers;
  m.nqkv = (m.H + 2 * m.Hk) * m.Dh;
  // k-blocks per CTA at least: small models (the draft) trade split-K parallelism for fewer
  // partial reductions (env SEED_MIN_UNITS_SMALL for models with d_model < 2048); a function of
  // the shape only, so batch invariance (R19) holds
  int min_units = 4;
  if (m.d < 2048) {
    const char* e = getenv("SEED_MIN_UNITS_SMALL");
    // measured (GSM8K round, 68M draft): stream-K GEMM 12 best; cluster split-K 6 (two CTAs per
    // 768-wide k-row: draft phase 311 -> 287 us; 3 and 4 within noise of 6)
    min_units = e ? atoi(e) : 6;
  }
  const size_t d = m.d, ff = m.ff, V = m.V, dkv = (size_t)m.Hk * m.Dh, dq = (size_t)m.H * m.Dh;
  auto alloc = [&](size_t elems) -> bf16* {
    bf16* p = nullptr;
    if (cudaMalloc(&p, elems * 2) != cudaSuccess) return nullptr;
    m.owned.push_back(p);
    return p;
  };
  m.embed = alloc(V * d);
  m.final_norm = alloc(d);
  m.lm_head = alloc(V * d);
  if (!m.embed || !m.final_norm || !m.lm_head) return fail(ctx, SEED_ENOMEM, "seed_init", "weights");
  if ((s = copy_rows(ctx, m.embed, w.embed, V * d)) != SEED_OK) return s;
  if ((s = copy_rows(ctx, m.final_norm, w.final_norm, d)) != SEED_OK) return s;
  if ((s = copy_rows(ctx, m.lm_head, w.lm_head, V * d)) != SEED_OK) return s;
  for (int l = 0; l < m.L; ++l) {
    const void* const* lw = w.layers + 9 * l;
    for (int i = 0; i < 9; ++i)
      if (!lw[i]) return fail(ctx, SEED_EINVAL, "seed_init", "null layer weight");
    bf16* qkv = alloc((dq + 2 * dkv) * d);
    bf16* o = alloc(d * dq);
    bf16* gu = alloc(2 * ff * d);
    bf16* dn = alloc(d * ff);
    bf16* a = alloc(d);
    bf16* mm = alloc(d);
    if (!qkv || !o || !gu || !dn || !a || !mm) return fail(ctx, SEED_ENOMEM, "seed_init", "weights");
    CK(cudaMemcpy(qkv, lw[0], dq * d * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(qkv + dq * d, lw[1], dkv * d * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(qkv + (dq + dkv) * d, lw[2], dkv * d * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(o, lw[3], d * dq * 2, cudaMemcpyDeviceToDevice));
    // gate/up interleave: rows [128b, 128b+64) = gate [64b, 64b+64), rows [128b+64, 128b+128) = up
    CK(cudaMemcpy2D(gu, 128 * d * 2, lw[4], 64 * d * 2, 64 * d * 2, ff / 64, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy2D(gu + 64 * d, 128 * d * 2, lw[5], 64 * d * 2, 64 * d * 2, ff / 64, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(dn, lw[6], d * ff * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(a, lw[7], d * 2, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(mm, lw[8], d * 2, cudaMemcpyDeviceToDevice));
    m.wqkv.push_back(qkv);
    m.wo.push_back(o);
    m.wgu.push_back(gu);
    m.wdown.push_back(dn);
    m.an.push_back(a);
    m.mn.push_back(mm);
    GemmPlan pq, po, pg, pd;
    seed::gemm_plan(&pq, qkv, m.nqkv, m.d, min_units);
    seed::gemm_plan(&po, o, m.d, (int)dq, min_units);
    seed::gemm_plan(&pg, gu, 2 * m.ff, m.d, min_units);
    seed::gemm_plan(&pd, dn, m.d, m.ff, min_units);
    m.pq.push_back(pq);
    m.po.push_back(po);
    m.pgu.push_back(pg);
    m.pd.push_back(pd);
  }
  seed::gemm_plan(&m.plm, m.lm_head, m.V, m.d, min_units);
  {   // a small model (the draft) runs every draft step: its weights stay L2-resident between steps
    const double layer_bytes = (double)m.L * ((double)m.nqkv * m.d + (double)m.d * dq + 3.0 * m.ff * m.d) * 2;
    if (layer_bytes <= 64e6) {   // (and its LM head, re-read every step: GSM8K -9 us per round)
      for (auto* v : {&m.pq, &m.po, &m.pgu, &m.pd})
        for (auto& p : *v) p.keep_w = 1;
      m.plm.keep_w = 1;
    }
    // a large model's cache is streamed once per round and would only displace what is re-read:
    // its K/V tiles are loaded evict-first (7B at N = 24: attention 38.3 -> 35.7 us per layer)
    m.kv.kv_once = layer_bytes > 64e6 ? 1 : 0;
  }
  // KV pool
  m.kv.n_layers = m.L;
  m.kv.Hk = m.Hk;
  m.kv.Dh = m.Dh;
  m.kv.P = ctx->P;
  m.kv.max_pages = max_pages;
  m.n_pages = pool_pages;
  CK(cudaMalloc(&m.kv.pool, m.kv.page_elems() * pool_pages * 2));
  CK(cudaMalloc(&m.page_table_dev, (size_t)slots * max_pages * 4));
  CK(cudaMallocHost(&m.page_table, (size_t)slots * max_pages * 4));
  std::memset(m.page_table, 0, (size_t)slots * max_pages * 4);
  CK(cudaMemset(m.page_table_dev, 0, (size_t)slots * max_pages * 4));
  m.kv.page_table = m.page_table_dev;
  if (!seed::attn_kv_tmap(&m.tmkv, m.kv, pool_pages, &m.kv.kv3d)) return fail(ctx, SEED_ECUDA, "seed_init", "KV tensor map");
  m.held.assign(slots, 0);
  for (size_t i = pool_pages; i-- > 0;) m.free_pages.push_back((int32_t)i);
  m.refs.assign(pool_pages, 0);
  CK(cudaMalloc(&m.rope, (size_t)max_pos * (m.Dh / 2) * sizeof(float2)));
  CK(seed::rope_table_init(m.rope, max_pos, m.Dh, sh.rope_theta > 0 ? sh.rope_theta : 10000.0, 0));
  // activations (rows rounded to >= 256 so every TMA box fits)
  m.m_cap = std::max(m_cap, 256);
  const size_t mc = m.m_cap;
  CK(cudaMalloc(&m.x, mc * d * 4));
  CK(cudaMalloc(&m.ssq_a, ((d + 127) / 128) * mc * 4));
  CK(cudaMalloc(&m.ssq_b, ((d + 127) / 128) * mc * 4));
  CK(cudaMalloc(&m.y, mc * (size_t)m.nqkv * 4));   // QKV output
  m.attn = alloc(mc * dq);
  m.h = alloc(mc * d);
  m.act = alloc(mc * ff);
  if (!m.attn || !m.h || !m.act) return fail(ctx, SEED_ENOMEM, "seed_init", "activations");
  m.aws.max_splits = (max_pos + seed::attn_chunk_tokens(m.Dh) - 1) / seed::attn_chunk_tokens(m.Dh);
  CK(cudaMalloc(&m.aws.o_part, (size_t)m.aws.max_splits * mc * dq * 4));
  CK(cudaMalloc(&m.aws.ml_part, (size_t)m.aws.max_splits * mc * m.H * 2 * 4));
  m.aws.max_counters = (int)(mc * m.H);
  CK(cudaMalloc(&m.aws.counters, (size_t)m.aws.max_counters * 4));
  CK(cudaMemset(m.aws.counters, 0, (size_t)m.aws.max_counters * 4));
  return SEED_OK;
}

void free_model(Model& m) {
  for (auto* v : {&m.pq, &m.po, &m.pgu, &m.pd})
    for (auto& p : *v) seed::gemm_plan_free(&p);
  seed::gemm_plan_free(&m.plm);
  if (m.page_table) cudaFreeHost(m.page_table);
  m.page_table = nullptr;
  for (bf16* p : m.owned) cudaFree(p);
  m.owned.clear();
  if (m.kv.pool) cudaFree(m.kv.pool);
  if (m.page_table_dev) cudaFree(m.page_table_dev);
  if (m.rope) cudaFree(m.rope);
  if (m.x) cudaFree(m.x);
  if (m.y) cudaFree(m.y);
  if (m.ssq_a) cudaFree(m.ssq_a);
  if (m.ssq_b) cudaFree(m.ssq_b);
  if (m.aws.o_part) cudaFree(m.aws.o_part);
  if (m.aws.ml_part) cudaFree(m.aws.ml_part);
  if (m.aws.counters) cudaFree(m.aws.counters);
}

// make sure `slot` holds pages for positions [0, n_tokens)
// cache positions a round may write past |T| - 1: gamma + 1 (chain) or every tree row
int round_rows(seed_ctx ctx) { return ctx->tree.n > 0 ? std::max(ctx->tree.nn, ctx->cfg.gamma + 1) : ctx->cfg.gamma + 1; }

seed_status ensure_pages(seed_ctx ctx, Model& m, int slot, int n_tokens, cudaStream_t st) {
  const int need = (n_tokens + ctx->P - 1) / ctx->P;
  if (need > ctx->max_pages) return fail(ctx, SEED_ECAPACITY, "KV", "context longer than max_ctx");
  int& held = m.held[slot];
  if (need <= held) return SEED_OK;
  const int first = held;
  while (held < need) {
    if (m.free_pages.empty()) return fail(ctx, SEED_ENOMEM, "KV", "page pool exhausted");
    m.page_table[(size_t)slot * ctx->max_pages + held] = m.free_pages.back();
    m.refs[m.free_pages.back()] = 1;
    m.free_pages.pop_back();
    ++held;
  }
  // pinned mirror: entries change again only after release_pages, which synchronises first
  CK(cudaMemcpyAsync(m.page_table_dev + (size_t)slot * ctx->max_pages + first,
                     m.page_table + (size_t)slot * ctx->max_pages + first, (size_t)(need - first) * 4,
                     cudaMemcpyHostToDevice, st));
  return SEED_OK;
}

void release_pages(Model& m, int slot, int max_pages) {
  for (int i = 0; i < m.held[slot]; ++i) {
    const int32_t pg = m.page_table[(size_t)slot * max_pages + i];
    if (--m.refs[pg] == 0) m.free_pages.push_back(pg);
  }
  m.held[slot] = 0;
}

// ------------------------------------------------------------------ forward over one chunk

seed_status forward_chunk(seed_ctx ctx, Model& m, const ChunkDesc& c, cudaStream_t st, int first_layer = 0,
                          int last_layer = -1, bool embed = true) {
  const float eps = m.sh.rms_eps > 0 ? m.sh.rms_eps : 1e-5f;
  if (last_layer < 0) last_layer = m.L;
  const int M = c.M;
  seed_status s;
  // the RMSNorm weight applied to the residual after layer l (B1, R24)
  auto next_norm = [&](int l) { return l + 1 < m.L ? m.an[l + 1] : m.final_norm; };
  // embedding (or the given residual), its per-tile sums of squares and h = bf16(x * attn_norm)
  if (!(embed && c.pre_embedded)) {   // (the previous draft step's K1 already wrote them: EmbedNext)
    CK(seed::embed_stats(embed ? m.embed : nullptr, c.tok.dev, c.tok.stride, M, m.d, m.V, m.x, m.ssq_b,
                         first_layer < m.L ? m.an[first_layer] : m.final_norm, m.h, ctx->dev_err, st,
                         next_rec(ctx)));
    ctx->kernel_launches++;
  }
  seed::SeqInfo seqs{c.q_start, c.q_len, c.kv_len, c.seq_slot, c.seq_stable, c.row_pos, c.anc, c.tree_base};
  const CUtensorMap* tm_h = xmap(ctx, m.h, m.d, m.m_cap, M);
  const CUtensorMap* tm_attn = xmap(ctx, m.attn, m.H * m.Dh, m.m_cap, M);
  const CUtensorMap* tm_act = xmap(ctx, m.act, m.ff, m.m_cap, M);
  if (!tm_h || !tm_attn || !tm_act) return fail(ctx, SEED_ECUDA, "cuTensorMapEncodeTiled", "activations");
  // X = h, output rows scaled by 1/rms from the per-tile sums of squares `ssq`
  auto norm_io = [&](const float* ssq) {
    seed::GemmIO io;
    io.tmX = tm_h;
    io.ssq_in = ssq;
    io.ssq_in_ld = M;
    io.eps = eps;
    return io;
  };
  for (int l = first_layer; l < last_layer; ++l) {
    // QKV: y = (h Wqkv^T) / rms(x)
    {
      seed::GemmIO io = norm_io(m.ssq_b);
      io.Y = m.y;
      io.ldY = m.nqkv;
      io.tmY = ymap(ctx, m.y, true, m.nqkv, m.nqkv, M);
      if ((s = run_gemm(ctx, m.pq[l], M, io, st)) != SEED_OK) return s;
    }
    {
      seed::AttnWorkspace aws = m.aws;
      aws.cta = nullptr;
      aws.timing = next_rec(ctx, &aws.cta);
      CK(seed::attention(m.y, M, c.n_seq, c.max_q_len, c.max_kv, m.H, m.Hk, m.Dh, seqs, m.rope, m.kv, m.tmkv, l, aws,
                         m.attn, st));
    }
    // O: x += attn Wo^T; sums of squares -> ssq_a; h = bf16(x * mlp_norm)
    {
      seed::GemmIO io;
      io.tmX = tm_attn;
      io.ymode = 1;
      io.Y = m.x;
      io.ldY = m.d;
      io.ssq_out = m.ssq_a;
      io.nw = m.mn[l];
      io.hout = m.h;
      if ((s = run_gemm(ctx, m.po[l], M, io, st)) != SEED_OK) return s;
    }
    // gate/up: act = bf16(silu(g) * u), g | u = (h Wgu^T) / rms(x)
    {
      seed::GemmIO io = norm_io(m.ssq_a);
      io.ymode = 2;
      io.hout = m.act;
      if ((s = run_gemm(ctx, m.pgu[l], M, io, st)) != SEED_OK) return s;
    }
    // down: x += act Wd^T; sums of squares -> ssq_b; h = bf16(x * next norm weight)
    {
      seed::GemmIO io;
      io.tmX = tm_act;
      io.ymode = 1;
      io.Y = m.x;
      io.ldY = m.d;
      io.ssq_out = m.ssq_b;
      io.nw = next_norm(l);
      io.hout = m.h;
      if ((s = run_gemm(ctx, m.pd[l], M, io, st)) != SEED_OK) return s;
    }
    ctx->kernel_launches += 1;
  }
  if (last_layer == m.L && c.n_logits > 0) {
    // LM head over all chunk rows; fp32 logits of the logits rows (compact index) straight into
    // the caller's rows (F2)
    seed::GemmIO io = norm_io(m.ssq_b);
    io.Y = c.Y;
    io.ldY = c.ldY;
    io.yrow = c.n_logits == M && !c.rowmap ? nullptr : c.compact;
    if (!io.yrow) io.tmY = ymap(ctx, c.Y, true, m.V, c.ldY, M);
    if ((s = run_gemm(ctx, m.plm, M, io, st)) != SEED_OK) return s;
  }
  return SEED_OK;
}

// Build the descriptors of one chunk into the arena. Segments must fit kMaxChunkRows rows.
// logits: 0 none, 1 all rows, 2 last row of each segment.
bool pack_chunk(seed_ctx ctx, const std::vector<Segment>& segs, int logits_mode, ChunkDesc* c,
                size_t* host_tok_off) {
  Arena& A = ctx->arena;
  int M = 0, mq = 0, mkv = 0;
  for (auto& s : segs) {
    M += s.q_len;
    mq = std::max(mq, s.q_len);
    mkv = std::max(mkv, s.pos0 + s.q_len);
  }
  const size_t o_pos = A.alloc(M), o_slot = A.alloc(M), o_cmp = A.alloc(M), o_tok = A.alloc(M), o_lr = A.alloc(M);
  const size_t n = segs.size();
  const size_t o_qs = A.alloc(n), o_ql = A.alloc(n), o_kv = A.alloc(n), o_ss = A.alloc(n), o_st = A.alloc(n);
  if (o_st == (size_t)-1) return false;
  int r = 0, nl = 0;
  for (size_t i = 0; i < n; ++i) {
    const Segment& s = segs[i];
    A.host[o_qs + i] = r;
    A.host[o_ql + i] = s.q_len;
    A.host[o_kv + i] = s.pos0 + s.q_len;
    A.host[o_ss + i] = s.slot;
    A.host[o_st + i] = s.stable;
    for (int j = 0; j < s.q_len; ++j, ++r) {
      A.host[o_pos + r] = s.pos0 + j;
      A.host[o_slot + r] = s.slot;
      const bool lg = logits_mode == 1 || (logits_mode == 2 && j == s.q_len - 1);
      if (lg) A.host[o_lr + nl] = r;
      A.host[o_cmp + r] = lg ? nl++ : -1;
      A.host[o_tok + r] = s.tok_off >= 0 ? A.host[s.tok_off + j] : 0;
    }
  }
  c->M = M;
  c->n_seq = (int)n;
  c->max_q_len = mq;
  c->max_kv = mkv;
  c->pos = A.dev + o_pos;
  c->slot = A.dev + o_slot;
  c->seq_slot = A.dev + o_ss;
  c->seq_stable = A.dev + o_st;
  c->compact = A.dev + o_cmp;
  c->logit_rows = A.dev + o_lr;
  c->q_start = A.dev + o_qs;
  c->q_len = A.dev + o_ql;
  c->kv_len = A.dev + o_kv;
  c->tok = TokSrc{A.dev + o_tok, 1};
  c->n_logits = nl;
  *host_tok_off = o_tok;
  return true;
}

// Prefill-style forward of host tokens into `slot` starting at position pos0 (chunked).
seed_status prefill(seed_ctx ctx, Model& m, int slot, const int32_t* toks, int n, int pos0, float* logits,
                    cudaStream_t st) {
  int done = 0;
  while (done < n) {
    const int q = std::min(std::min(kMaxChunkRows, m.m_cap), n - done);
    ctx->arena.begin();
    const size_t to = ctx->arena.alloc(q);
    if (to == (size_t)-1) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    std::memcpy(ctx->arena.host + to, toks + done, (size_t)q * 4);
    std::vector<Segment> segs{{slot, pos0 + done, q, (int)to}};
    ChunkDesc c;
    size_t tok_off;
    if (!pack_chunk(ctx, segs, logits ? 1 : 0, &c, &tok_off)) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    c.Y = logits ? logits + (size_t)done * m.V : nullptr;
    c.ldY = m.V;
    CK(ctx->arena.upload(st));
    seed_status s = forward_chunk(ctx, m, c, st);
    if (s != SEED_OK) return s;
    done += q;
  }
  return SEED_OK;
}

seed_status check_ctx(seed_ctx ctx) {
  if (!ctx) return SEED_EINVAL;
  if (ctx->poisoned) return SEED_ESTATE;
  return SEED_OK;
}

seed::BookStream& stream_of(seed_ctx ctx, uint32_t gid) { return ctx->book->own.at(gid); }

// a5 / a6 on the host, once round r's work completed on the device: the gathered exchange
// blocks (K5 wrote this rank's, the all-gather the others') go to the round book -- own streams
// commit their tokens and are requeued FCFS, other ranks' tokens go to the token
// table, the undone counts give the global pending count -- and the KV lengths follow (R6).
// A device contract violation (error word) is reported here as SEED_EDEVICE, without poisoning.
seed_status complete_round(seed_ctx ctx) {
  if (!ctx->round_pending) return SEED_OK;
  CK(cudaEventSynchronize(ctx->round_done));
  ctx->round_pending = false;
  const int g = ctx->cfg.gamma;
  const int world = std::max(ctx->cfg.world, 1);
  std::vector<int> t_before;
  t_before.reserve(ctx->last_batch.size());
  for (int32_t gid : ctx->last_batch) t_before.push_back((int)stream_of(ctx, (uint32_t)gid).T.size());
  seed_status st = seed_book_complete(ctx->book, ctx->records_host, world);
  if (st != SEED_OK) return fail(ctx, SEED_ESTATE, "seed_book_complete", "malformed exchange block");
  for (size_t b = 0; b < ctx->last_batch.size(); ++b) {
    const uint32_t gid = (uint32_t)ctx->last_batch[b];
    const int T = (int)stream_of(ctx, gid).T.size();
    SlotState& ss = ctx->slots[ctx->gid2slot[gid]];
    ss.len_t = T - 1;                                  // keep T'[:-1]
    ss.len_d = std::min(T - 1, t_before[b] + g - 1);   // the draft wrote up to |T| + gamma - 2
  }
  ctx->last_batch.clear();
  const uint32_t bits = (uint32_t)ctx->err_host[0];
  ctx->fallbacks = ctx->err_host[1];
  if (bits) {
    ctx->err_bits_seen |= bits;
    CK(cudaMemset(ctx->dev_err, 0, sizeof(int32_t)));
    ctx->err_host[0] = 0;
    char msg[256];
    snprintf(msg, sizeof(msg),
             "device contract violation (error word 0x%x): 1 = token id out of range at an embedding gather (read "
             "as id 0), 2 = a race over no finite key (non-finite logits)", bits);
    ctx->err = msg;
    return SEED_EDEVICE;
  }
  return SEED_OK;
}

// finish any round work in flight before the descriptor arena is reused outside a round
// (a device error word found here stays visible through seed_device_status)
seed_status quiesce(seed_ctx ctx) {
  if (ctx->gstream) CK(cudaStreamSynchronize(ctx->gstream));
  if (ctx->round_pending) {
    const seed_status s = complete_round(ctx);
    return s == SEED_EDEVICE ? SEED_OK : s;
  }
  return SEED_OK;
}

seed_status map_batch(seed_ctx ctx, const int32_t* ids, int n, std::vector<int>& slots) {
  if (n < 0 || n > ctx->C || (n > 0 && !ids)) return fail(ctx, n > ctx->C ? SEED_ECAPACITY : SEED_EINVAL, "batch", "size");
  slots.resize(n);
  for (int i = 0; i < n; ++i) {
    auto it = ctx->gid2slot.find((uint32_t)ids[i]);
    if (it == ctx->gid2slot.end()) return fail(ctx, SEED_ENOTFOUND, "batch", "unknown stream id");
    slots[i] = it->second;
    if (stream_of(ctx, (uint32_t)ids[i]).done) return fail(ctx, SEED_EINVAL, "batch", "stream already done");
    for (int k = 0; k < i; ++k)
      if (ids[k] == ids[i]) return fail(ctx, SEED_EINVAL, "batch", "duplicate stream id");
  }
  return SEED_OK;
}

// ------------------------------------------------------------------ one round
// All descriptors of a round (draft steps and verify chunks) are packed into the arena at
// offsets that depend on the batch size only, so the captured graph of a batch size can be
// replayed with fresh descriptor contents (R23).
// Tree round descriptors (R36): level 1 = the chain's draft step 1 (T[-2], T[-1]: the root's draft
// row); level d = 2..K = the depth d - 1 nodes of every stream as tree rows (RoPE at the root's
// position + depth, attention to the context and the row's ancestors; the node's K/V at cache
// position root + node); the verify chunk = root + every node as tree rows.  Node logits rows go to
// [stream][node][V] through the row map.
seed_status build_tree_plan(seed_ctx ctx, const std::vector<const seed::BookStream*>& bs, const std::vector<int>& slots,
                            RoundPlan& P, int max_pos) {
  auto& TR = ctx->tree;
  Arena& A = ctx->arena;
  const int n = P.n, K = TR.n, nn = TR.nn, V = ctx->cfg.target.vocab;
  size_t tok_off;
  // tree-row descriptors of a chunk whose segment b holds the tree rows [row0, row0 + len) of stream b
  auto tree_rows = [&](ChunkDesc& c, int row0, int len, bool map_logits) -> bool {
    const int M = n * len;
    const size_t o_p = A.alloc(M), o_b = A.alloc(n), o_a = A.alloc(2 * M + 2);
    if (o_a == (size_t)-1) return false;
    const size_t o_a8 = (o_a + 1) & ~(size_t)1;
    for (int b = 0; b < n; ++b) {
      const int root = (int)bs[b]->T.size() - 1;
      A.host[o_b + b] = root;
      for (int k = 0; k < len; ++k) {
        const int node = row0 + k, r = b * len + k;
        A.host[o_p + r] = root + TR.depth[node];
        std::memcpy(A.host + o_a8 + 2 * r, &TR.anc[node], 8);
      }
    }
    c.row_pos = A.dev + o_p;
    c.tree_base = A.dev + o_b;
    c.anc = reinterpret_cast<const uint64_t*>(A.dev + o_a8);
    if (map_logits) {   // chunk row (b, k) -> logits row b * nn + row0 + k
      const size_t o_c = A.alloc(M);
      if (o_c == (size_t)-1) return false;
      for (int b = 0; b < n; ++b)
        for (int k = 0; k < len; ++k) A.host[o_c + b * len + k] = b * nn + row0 + k;
      c.compact = A.dev + o_c;
      c.rowmap = true;
    }
    return true;
  };
  P.draft.assign(K, ChunkDesc{});
  std::vector<Segment> segs(n);
  for (int b = 0; b < n; ++b) {
    const int T = (int)bs[b]->T.size();
    const size_t to = A.alloc(2);
    if (to == (size_t)-1) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    A.host[to] = bs[b]->T[T - 2];
    A.host[to + 1] = bs[b]->T[T - 1];
    segs[b] = Segment{slots[b], T - 2, 2, (int)to, T - 2};
  }
  if (2 * n > ctx->tm.m_cap || 2 * n > ctx->dm.m_cap || !pack_chunk(ctx, segs, 2, &P.draft[0], &tok_off))
    return fail(ctx, SEED_ECAPACITY, "seed_draft_round", "batch too large");
  P.draft[0].Y = ctx->drf_logits;               // the root's draft row: [b][node 0]
  P.draft[0].ldY = nn * V;
  for (int d = 2; d <= K; ++d) {
    const int row0 = TR.lvl_start[d - 1], len = TR.lvl_len[d - 1];
    if (n * len > ctx->dm.m_cap) return fail(ctx, SEED_ECAPACITY, "seed_draft_round", "tree level too wide");
    for (int b = 0; b < n; ++b) {
      const int T = (int)bs[b]->T.size();
      segs[b] = Segment{slots[b], T - 1 + row0, len, -1, T - 2};
    }
    ChunkDesc& c = P.draft[d - 1];
    if (!pack_chunk(ctx, segs, 1, &c, &tok_off) || !tree_rows(c, row0, len, true))
      return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    c.tok = TokSrc{TR.tok_lvl + TR.lvl_off[d], 1};
    c.Y = ctx->drf_logits;
    c.ldY = V;
  }
  // verify chunks of whole streams: root + nodes
  const int per_chunk = std::max(1, ctx->tm.m_cap / nn);
  for (int b0 = 0; b0 < n; b0 += per_chunk) {
    const int nb = std::min(per_chunk, n - b0);
    std::vector<Segment> vs(nb);
    for (int b = 0; b < nb; ++b) {
      const int T = (int)bs[b0 + b]->T.size();
      vs[b] = Segment{slots[b0 + b], T - 1, nn, -1, T - 1};
    }
    ChunkDesc c;
    std::vector<const seed::BookStream*> sub(bs.begin() + b0, bs.begin() + b0 + nb);
    if (!pack_chunk(ctx, vs, 1, &c, &tok_off)) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    {
      const int M = nb * nn;
      const size_t o_p = A.alloc(M), o_b = A.alloc(nb), o_a = A.alloc(2 * M + 2);
      if (o_a == (size_t)-1) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
      const size_t o_a8 = (o_a + 1) & ~(size_t)1;
      for (int b = 0; b < nb; ++b) {
        const int root = (int)sub[b]->T.size() - 1;
        A.host[o_b + b] = root;
        for (int k = 0; k < nn; ++k) {
          A.host[o_p + b * nn + k] = root + TR.depth[k];
          std::memcpy(A.host + o_a8 + 2 * (b * nn + k), &TR.anc[k], 8);
        }
      }
      c.row_pos = A.dev + o_p;
      c.tree_base = A.dev + o_b;
      c.anc = reinterpret_cast<const uint64_t*>(A.dev + o_a8);
    }
    c.tok = TokSrc{TR.tree_tok + (size_t)b0 * nn, 1};
    c.Y = ctx->tgt_logits + (size_t)b0 * nn * V;
    c.ldY = V;
    P.verify.push_back(c);
    P.verify_b0.push_back(b0);
  }
  const int chd = seed::attn_chunk_tokens(ctx->dm.Dh), cht = seed::attn_chunk_tokens(ctx->tm.Dh);
  int dk = 0, vk = 0;
  for (auto& c : P.draft) dk = std::max(dk, c.max_kv);
  for (auto& c : P.verify) vk = std::max(vk, c.max_kv);
  P.dk_raw = dk;
  P.vk_raw = vk;
  dk = std::min(max_pos, (dk + chd - 1) / chd * chd);
  vk = std::min(max_pos, (vk + cht - 1) / cht * cht);
  for (auto& c : P.draft) c.max_kv = dk;
  for (auto& c : P.verify) c.max_kv = vk;
  P.key_draft = ((int64_t)n << 32) | (dk / chd);
  P.key_verify = ((int64_t)n << 32) | (vk / cht);
  return SEED_OK;
}

seed_status build_round_plan(seed_ctx ctx, const std::vector<int32_t>& ids, const std::vector<int>& slots,
                             RoundPlan& P) {
  const int g = ctx->cfg.gamma, n = (int)ids.size();
  Arena& A = ctx->arena;
  A.begin();
  P.n = n;
  P.o_sid = A.alloc(n);
  P.o_r = A.alloc(n);
  P.o_sl = A.alloc(n);
  P.o_last = A.alloc(n);
  P.o_out = A.alloc(1);
  if (P.o_out == (size_t)-1) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
  std::vector<const seed::BookStream*> bs(n);
  for (int b = 0; b < n; ++b) {
    bs[b] = &stream_of(ctx, (uint32_t)ids[b]);
    A.host[P.o_sid + b] = ids[b];
    A.host[P.o_r + b] = bs[b]->r;
    A.host[P.o_sl + b] = slots[b];
    A.host[P.o_last + b] = bs[b]->T.back();
  }
  A.host[P.o_out] = (int32_t)(ctx->book->undone - n);   // K5 adds the batch's undone streams
  P.draft.clear();
  P.verify.clear();
  P.verify_b0.clear();
  P.key_draft = P.key_verify = 0;
  if (n == 0) return SEED_OK;   // a rank with nothing to run still joins the exchange (world > 1)
  const int max_pos = ctx->cfg.max_ctx + std::max(g, ctx->tree.n > 0 ? ctx->tree.nn : g + 1) + 2;
  if (ctx->tree.n > 0) return build_tree_plan(ctx, bs, slots, P, max_pos);
  // draft step 1 feeds (T[-2], T[-1]); when one token is pending the first row rewrites an
  // existing entry with identical values (R22), so M = 2n every round
  P.draft.assign(g, ChunkDesc{});
  std::vector<Segment> segs(n);
  for (int b = 0; b < n; ++b) {
    const int T = (int)bs[b]->T.size();
    const size_t to = A.alloc(2);
    if (to == (size_t)-1) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    A.host[to] = bs[b]->T[T - 2];
    A.host[to + 1] = bs[b]->T[T - 1];
    segs[b] = Segment{slots[b], T - 2, 2, (int)to, T - 2};
  }
  size_t tok_off;
  if (2 * n > ctx->tm.m_cap || 2 * n > ctx->dm.m_cap || !pack_chunk(ctx, segs, 2, &P.draft[0], &tok_off))
    return fail(ctx, SEED_ECAPACITY, "seed_draft_round", "batch too large");
  for (int j = 2; j <= g; ++j) {
    for (int b = 0; b < n; ++b) {
      const int T = (int)bs[b]->T.size();
      segs[b] = Segment{slots[b], T + j - 2, 1, -1, T - 2};
    }
    if (!pack_chunk(ctx, segs, 2, &P.draft[j - 1], &tok_off)) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    P.draft[j - 1].tok = TokSrc{ctx->xs + (j - 2), g};  // x_{j-1} of every stream ([B][g] layout)
  }
  // verify chunks of whole streams
  const int per_chunk = std::max(1, ctx->tm.m_cap / (g + 1));
  for (int b0 = 0; b0 < n; b0 += per_chunk) {
    const int nb = std::min(per_chunk, n - b0);
    std::vector<Segment> vs(nb);
    for (int b = 0; b < nb; ++b) {
      const int T = (int)bs[b0 + b]->T.size();
      vs[b] = Segment{slots[b0 + b], T - 1, g + 1, -1, T - 1};
    }
    ChunkDesc c;
    if (!pack_chunk(ctx, vs, 1, &c, &tok_off)) return fail(ctx, SEED_ENOMEM, "arena", "descriptors");
    c.tok = TokSrc{ctx->vtok + (size_t)b0 * (g + 1), 1};
    c.Y = ctx->tgt_logits + (size_t)b0 * (g + 1) * ctx->cfg.target.vocab;
    c.ldY = ctx->cfg.target.vocab;
    P.verify.push_back(c);
    P.verify_b0.push_back(b0);
  }
  // attention grids sized by the round's longest context, rounded up to whole splits; the
  // graphs are keyed by (batch size, split counts), so a graph is re-captured only when a
  // context crosses a split boundary (R23)
  const int chd = seed::attn_chunk_tokens(ctx->dm.Dh), cht = seed::attn_chunk_tokens(ctx->tm.Dh);
  int dk = 0, vk = 0;
  for (auto& c : P.draft) dk = std::max(dk, c.max_kv);
  for (auto& c : P.verify) vk = std::max(vk, c.max_kv);
  P.dk_raw = dk;
  P.vk_raw = vk;
  dk = std::min(max_pos, (dk + chd - 1) / chd * chd);
  vk = std::min(max_pos, (vk + cht - 1) / cht * cht);
  for (auto& c : P.draft) c.max_kv = dk;
  for (auto& c : P.verify) c.max_kv = vk;
  P.key_draft = ((int64_t)n << 32) | (dk / chd);
  P.key_verify = ((int64_t)n << 32) | (vk / cht);
  return SEED_OK;
}

seed_status enqueue_draft(seed_ctx ctx, cudaStream_t st) {
  RoundPlan& P = ctx->plan;
  const int n = P.n, g = ctx->cfg.gamma, V = ctx->cfg.target.vocab;
  Arena& A = ctx->arena;
  seed_status s;
  CK(cudaMemcpyAsync(A.dev, A.host, A.used * 4, cudaMemcpyHostToDevice, st));
  if (n == 0) return SEED_OK;
  CK(cudaMemcpyAsync(ctx->sids_dev, A.dev + P.o_sid, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(ctx->rs_dev, A.dev + P.o_r, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(ctx->slots_dev, A.dev + P.o_sl, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  const uint32_t k0 = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu), k1 = (uint32_t)(ctx->cfg.seed >> 32);
  if (ctx->tree.n > 0) {
    // tree drafting (R36): level by level, every node's children are the top-m of its draft row's
    // race (K1T, slot node + 1), written as the next level's input and into the verify rows
    auto& TR = ctx->tree;
    const int nn = TR.nn, K = TR.n;
    CK(cudaMemcpy2DAsync(TR.tree_tok, (size_t)nn * 4, A.dev + P.o_last, 4, 4, n, cudaMemcpyDeviceToDevice, st));
    for (int d = 1; d <= K; ++d) {
      if ((s = forward_chunk(ctx, ctx->dm, P.draft[d - 1], st)) != SEED_OK) return s;
      const int row0 = TR.lvl_start[d - 1], len = TR.lvl_len[d - 1], m = TR.counts[d - 1];
      for (int k = 0; k < len; ++k) {
        const int node = row0 + k;
        int32_t* nxt = d < K ? TR.tok_lvl + TR.lvl_off[d + 1] : nullptr;   // level d + 1 rows: [b][len * m]
        int32_t* vrow = TR.tree_tok + TR.first[node];                      // verify rows: children of `node`
        if (nxt) {
          CK(seed::draft_topk(ctx->drf_logits + (size_t)node * V, (long)nn * V, n, V, ctx->cfg.temperature, k0, k1,
                              ctx->sids_dev, ctx->rs_dev, node, m, nxt, len * m, k * m, vrow - k * m, nn,
                              ctx->dev_err, st, next_rec(ctx)));
        } else {
          CK(seed::draft_topk(ctx->drf_logits + (size_t)node * V, (long)nn * V, n, V, ctx->cfg.temperature, k0, k1,
                              ctx->sids_dev, ctx->rs_dev, node, m, vrow, nn, 0, nullptr, 0, ctx->dev_err, st,
                              next_rec(ctx)));
        }
        ctx->kernel_launches++;
      }
    }
    return SEED_OK;
  }
  // verify input column 0 = T[-1]
  CK(cudaMemcpy2DAsync(ctx->vtok, (size_t)(g + 1) * 4, A.dev + P.o_last, 4, 4, n, cudaMemcpyDeviceToDevice, st));
  for (int j = 1; j <= g; ++j) {
    ChunkDesc& c = P.draft[j - 1];
    c.Y = ctx->drf_logits + (size_t)(j - 1) * V;
    c.ldY = g * V;
    if ((s = forward_chunk(ctx, ctx->dm, c, st)) != SEED_OK) return s;
    // K1 sampler: x_j -> xs[b][j-1] and the verify input vtok[b][j]; below the last step it also
    // embeds x_j as the next step's rows (that step's chunk: one row per stream, in batch order)
    seed::EmbedNext en;
    if (j < g) {
      Model& dm = ctx->dm;
      en.emb = dm.embed;
      en.d = dm.d;
      en.x = dm.x;
      en.ssq = dm.ssq_b;
      en.ssq_ld = P.draft[j].M;
      en.nw = dm.an[0];
      en.h = dm.h;
      P.draft[j].pre_embedded = P.draft[j].M == n;
      if (!P.draft[j].pre_embedded) en.emb = nullptr;
    }
    CK(seed::draft_sample(c.Y, (long)g * V, n, V, ctx->cfg.temperature, k0, k1, ctx->sids_dev, ctx->rs_dev, j,
                          ctx->xs + (j - 1), g, ctx->vtok + j, g + 1, ctx->dev_err, st, next_rec(ctx), en));
    ctx->kernel_launches++;
  }
  return SEED_OK;
}

seed_status enqueue_verify(seed_ctx ctx, cudaStream_t st) {
  RoundPlan& P = ctx->plan;
  const int n = P.n, g = ctx->cfg.gamma, V = ctx->cfg.target.vocab;
  seed_status s;
  for (auto& c : P.verify)
    if ((s = forward_chunk(ctx, ctx->tm, c, st)) != SEED_OK) return s;
  if (n > 0 && ctx->tree.n > 0) {
    // a4 on a tree: K4T (recursive rejection over each node's candidates), then the accepted path's
    // K/V compacted into consecutive positions of both caches (the draft holds nodes to depth K - 1)
    auto& TR = ctx->tree;
    CK(seed::verify_tree(ctx->tgt_logits, (long)TR.nn * V, ctx->drf_logits, (long)TR.nn * V, TR.tree_tok, TR.nn,
                         TR.ch_dev, TR.ch_dev + TR.nn, n, TR.n, V, ctx->cfg.temperature,
                         (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu), (uint32_t)(ctx->cfg.seed >> 32), ctx->sids_dev,
                         ctx->rs_dev, ctx->cfg.bonus, ctx->out_tok, ctx->out_cnt, TR.out_node, ctx->dev_err, st,
                         next_rec(ctx)));
    CK(seed::kv_compact(ctx->tm.kv, ctx->slots_dev, ctx->ds.tlen, TR.out_node, TR.n, TR.n, n, st, next_rec(ctx)));
    if (TR.n > 1)
      CK(seed::kv_compact(ctx->dm.kv, ctx->slots_dev, ctx->ds.tlen, TR.out_node, TR.n, TR.n - 1, n, st, next_rec(ctx)));
    ctx->kernel_launches += TR.n > 1 ? 3 : 2;
  } else if (n > 0) {
    // a4: K4 fused vocabulary kernel
    seed::VerifyArgs a{};
    a.zt = ctx->tgt_logits;
    a.zd = ctx->drf_logits;
    a.xs = ctx->xs;
    a.zt_stride_b = (long)(g + 1) * V;
    a.zd_stride_b = (long)g * V;
    a.B = n;
    a.gamma = g;
    a.V = V;
    a.T = ctx->cfg.temperature;
    a.k0 = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu);
    a.k1 = (uint32_t)(ctx->cfg.seed >> 32);
    a.sids = ctx->sids_dev;
    a.rs = ctx->rs_dev;
    a.bonus = ctx->cfg.bonus;
    a.out_tok = ctx->out_tok;
    a.out_cnt = ctx->out_cnt;
    a.out_acc = ctx->out_acc;
    a.work = ctx->verify_work;
    a.err = ctx->dev_err;
    a.timing = next_rec(ctx);
    CK(seed::vocab_verify(a, st));
    ctx->kernel_launches++;
  }
  // a5: K5 commit + rollback and this rank's exchange block (records, then the undone count)
  const int world = std::max(ctx->cfg.world, 1);
  const size_t blk_bytes = (size_t)ctx->block_ints * 4;
  CK(seed::rollback_commit(ctx->ds, ctx->slots_dev, n, g, ctx->out_tok, ctx->out_cnt, ctx->cfg.max_new_tokens,
                           ctx->records, ctx->C, ctx->sids_dev, ctx->arena.dev + P.o_out, st, next_rec(ctx)));
  ctx->kernel_launches++;
  if (ctx->profile) {
    // draft records live in [0, half), verify records in [half, ...)
    const int half = ctx->rec_cap / 2;
    const int nd = ctx->draft_recs[n], nv = ctx->rec_used - half;
    ctx->last_draft_recs = nd;
    ctx->last_verify_recs = nv;
    CK(seed::timing_accumulate(ctx->timing_rec, nd, ctx->timing_acc, ctx->timing_last, st));
    CK(seed::timing_accumulate(ctx->timing_rec + 4 * (size_t)half, nv, ctx->timing_acc,
                               ctx->timing_last + 4 * (size_t)half, st));
    ctx->kernel_launches += 2;
  }
  // the device error word travels with the round's results
  CK(cudaMemcpyAsync(ctx->err_host, ctx->dev_err, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  // a6: all-gather of the per-rank exchange blocks over NVLink (world > 1)
  if (world > 1) {
    if (g_nccl.allgather(ctx->records, ctx->records_all, (size_t)ctx->block_ints, kNcclInt32, ctx->comm, st) != 0)
      return fail(ctx, SEED_ENCCL, "ncclAllGather", "exchange blocks");
    CK(cudaMemcpyAsync(ctx->records_host, ctx->records_all, blk_bytes * world, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(ctx->records_host, ctx->records, blk_bytes, cudaMemcpyDeviceToHost, st));
  }
  return SEED_OK;
}

// Captures and instantiates the round graph of the current plan (draft + verify phases).
seed_status capture_round(seed_ctx ctx, int n, RoundGraphEntry& G) {
  const int64_t k0 = ctx->kernel_launches;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal));
  ctx->in_round = true;
  ctx->rec_used = 0;
  ctx->round_gemm_bytes = 0;
  ctx->round_gemms = 0;
  seed_status s = enqueue_draft(ctx, ctx->gstream);
  if (s == SEED_OK) {
    ctx->draft_recs[n] = ctx->rec_used;
    ctx->rec_used = ctx->rec_cap / 2;
    s = enqueue_verify(ctx, ctx->gstream);
  }
  cudaError_t e = cudaStreamEndCapture(ctx->gstream, &graph);
  if (s != SEED_OK) return s;
  CK(e);
  e = cudaGraphInstantiate(&G.exec, graph, 0);
  cudaGraphDestroy(graph);
  CK(e);
  G.kernels = ctx->kernel_launches - k0;
  ctx->kernel_launches = k0;
  G.gemm_bytes = ctx->round_gemm_bytes;
  G.gemms = ctx->round_gemms;
  return SEED_OK;
}

// A context crossing an attention split boundary needs the graph of the next chunk count (R23).
// Each round adds at most gamma + 1 keys per stream, so when the round just launched could be
// followed by one that crosses, that graph is captured and uploaded now, on the host, while the
// device runs the round: the crossing round launches it like any other (no capture between rounds).
seed_status precapture_next(seed_ctx ctx, int n, int64_t pbit) {
  RoundPlan& P = ctx->plan;
  if (n == 0 || getenv("SEED_NO_PRECAPTURE")) return SEED_OK;
  const int g = ctx->cfg.gamma;
  const int max_pos = ctx->cfg.max_ctx + g + 2;
  const int chd = seed::attn_chunk_tokens(ctx->dm.Dh), cht = seed::attn_chunk_tokens(ctx->tm.Dh);
  const int dk = std::min(max_pos, (P.dk_raw + g + 1 + chd - 1) / chd * chd);
  const int vk = std::min(max_pos, (P.vk_raw + g + 1 + cht - 1) / cht * cht);
  const int64_t kd = ((int64_t)n << 32) | (dk / chd), kv = ((int64_t)n << 32) | (vk / cht);
  if (kd == P.key_draft && kv == P.key_verify) return SEED_OK;
  const int64_t key = ((int64_t)n << 40) | ((kd & 0xFFFFF) << 20) | (kv & 0xFFFFF) | pbit;
  auto& G = ctx->round_graphs[key];
  if (G.exec) return SEED_OK;
  // the plan with the next rounds' grids; everything else of a graph is a function of the batch size
  std::vector<int> dsave, vsave;
  for (auto& c : P.draft) dsave.push_back(c.max_kv), c.max_kv = dk;
  for (auto& c : P.verify) vsave.push_back(c.max_kv), c.max_kv = vk;
  const int64_t sd = P.key_draft, sv = P.key_verify;
  const int ru = ctx->rec_used, dr = ctx->draft_recs[n];
  const double gb = ctx->round_gemm_bytes;
  const int64_t gl = ctx->round_gemms;
  P.key_draft = kd;
  P.key_verify = kv;
  seed_status s = capture_round(ctx, n, G);
  for (size_t i = 0; i < P.draft.size(); ++i) P.draft[i].max_kv = dsave[i];
  for (size_t i = 0; i < P.verify.size(); ++i) P.verify[i].max_kv = vsave[i];
  P.key_draft = sd;
  P.key_verify = sv;
  ctx->rec_used = ru;
  ctx->draft_recs[n] = dr;
  ctx->round_gemm_bytes = gb;
  ctx->round_gemms = gl;
  ctx->in_round = false;
  if (s != SEED_OK) return s;
  CK(cudaGraphUpload(G.exec, ctx->gstream));
  return SEED_OK;
}

// Runs the draft (draft = true) or verify phase of the planned round: directly on the caller's
// stream, or as a CUDA graph captured once per batch size on the library's stream.
seed_status run_phase(seed_ctx ctx, int n, bool draft, cudaStream_t st) {
  seed_status s;
  const int64_t k0 = ctx->kernel_launches;
  ctx->in_round = true;
  ctx->rec_used = draft ? 0 : ctx->rec_cap / 2;
  ctx->round_gemm_bytes = 0;
  ctx->round_gemms = 0;
  if (!ctx->use_graphs) {
    s = draft ? enqueue_draft(ctx, st) : enqueue_verify(ctx, st);
    if (s != SEED_OK) return s;
    ctx->gemm_bytes += ctx->round_gemm_bytes;
    ctx->gemm_launches += ctx->round_gemms;
    if (draft) {
      ctx->draft_recs[n] = ctx->rec_used;
    } else {
      ctx->in_round = false;
      CK(cudaEventRecord(ctx->round_done, st));
    }
    return SEED_OK;
  }
  // With graphs the draft phase is not launched on its own: seed_verify launches one graph holding
  // the draft and verify phases of the round, so PDL overlaps their boundary too (R23: keyed by
  // batch size, both phases' attention chunk counts and the profiling state).
  if (draft) {
    ctx->draft_deferred = true;
    ctx->in_round = false;
    return SEED_OK;
  }
  if (!ctx->draft_deferred) return fail(ctx, SEED_ESTATE, "seed_verify", "batch was not drafted");
  ctx->draft_deferred = false;
  const int64_t pbit = ctx->profile ? (int64_t)1 << 62 : 0;
  const int64_t key = ((int64_t)n << 40) | ((ctx->plan.key_draft & 0xFFFFF) << 20) | (ctx->plan.key_verify & 0xFFFFF) | pbit;
  auto& G = ctx->round_graphs[key];
  if (!G.exec && (s = capture_round(ctx, n, G)) != SEED_OK) return s;
  cudaGraphExec_t& ex = G.exec;
  CK(cudaEventRecord(ctx->ev_in, st));
  CK(cudaStreamWaitEvent(ctx->gstream, ctx->ev_in, 0));
  CK(cudaGraphLaunch(ex, ctx->gstream));
  ctx->kernel_launches = k0 + G.kernels;
  CK(cudaEventRecord(ctx->round_done, ctx->gstream));
  ctx->gemm_bytes += G.gemm_bytes;
  ctx->gemm_launches += G.gemms;
  ctx->in_round = false;
  CK(cudaEventRecord(ctx->ev_out, ctx->gstream));
  CK(cudaStreamWaitEvent(st, ctx->ev_out, 0));
  return precapture_next(ctx, n, pbit);
}

seed_status install_slot(seed_ctx ctx, int slot, uint32_t gid, const int32_t* prefix, int len, cudaStream_t st) {
  SlotState& ss = ctx->slots[slot];
  ss = SlotState();
  ss.used = true;
  ss.gid = gid;
  ss.len_t = ss.len_d = len - 1;
  // device state (K5 reads/writes it)
  int32_t vals[6] = {len, len - 1, len - 1, 0, 0, 0};
  int32_t* dst[6] = {ctx->ds.tlen, ctx->ds.len_t, ctx->ds.len_d, ctx->ds.L, ctx->ds.r, ctx->ds.done};
  for (int i = 0; i < 6; ++i) CK(cudaMemcpyAsync(dst[i] + slot, &vals[i], 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->ds.hist + (size_t)slot * ctx->ds.max_ctx, prefix, (size_t)len * 4, cudaMemcpyHostToDevice,
                     st));
  CK(cudaStreamSynchronize(st));
  seed_status s = seed_book_add(ctx->book, gid, prefix, len);
  if (s != SEED_OK) return fail(ctx, s, "seed_book_add", "");
  ctx->gid2slot[gid] = slot;
  return SEED_OK;
}

// calls that change streams or reuse the descriptor arena must not fall between seed_draft_round
// and seed_verify (the planned round's descriptors and pages are in flight)
seed_status check_between(seed_ctx ctx, const char* what) {
  if (ctx->draft_called) return fail(ctx, SEED_ESTATE, what, "a drafted batch is not verified");
  return SEED_OK;
}

int free_slot(seed_ctx ctx) {
  for (int i = 0; i < ctx->cfg.max_streams; ++i)
    if (!ctx->slots[i].used) return i;
  return -1;
}

}  // namespace

// ====================================================================== C ABI
namespace {
seed_status decoder_layer_impl(const seed_model_shape* shape, const void* const* w, const float* x_in, int32_t M,
                               int32_t ctx_len, const int32_t* parent, const void* k_prev, const void* v_prev,
                               float* x_out, void* k_new, void* v_new, void* stream);
}  // namespace

extern "C" {

const char* seed_last_error(seed_ctx ctx) { return ctx ? ctx->err.c_str() : "null context"; }

seed_status seed_nccl_unique_id(void* out128) {
  if (!out128) return SEED_EINVAL;
  if (!g_nccl.load()) return SEED_ENCCL;
  Id128 id;
  if (g_nccl.get_id(&id) != 0) return SEED_ENCCL;
  std::memcpy(out128, &id, 128);
  return SEED_OK;
}

seed_status seed_init(const seed_config* cfg, seed_ctx* out) {
  if (!cfg || !out) return SEED_EINVAL;
  *out = nullptr;
  if (cfg->draft.vocab != cfg->target.vocab) return SEED_EINVAL;
  if (cfg->gamma < 1 || cfg->gamma > 16 || !(cfg->temperature > 0.f) || cfg->max_new_tokens < 1 ||
      cfg->max_streams < 1 || cfg->max_batch < 1 || cfg->max_ctx < 8)
    return SEED_EINVAL;
  // KV pages hold whole 16-key attention tiles (one tensor copy each): 16, 32, ..., 256 tokens
  const int P = cfg->page_tokens > 0 ? cfg->page_tokens : 16;
  if (P < 16 || P > 256 || (P & (P - 1))) return SEED_EINVAL;
  if (cfg->world < 0 || (cfg->world > 1 && (cfg->rank < 0 || cfg->rank >= cfg->world))) return SEED_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SEED_ECUDA;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major < 10) return SEED_ECUDA;

  seed_ctx ctx = new seed_ctx_s;
  ctx->cfg = *cfg;
  ctx->dev = dev;
  ctx->P = P;
  ctx->C = std::min(cfg->max_batch, cfg->max_streams);
  ctx->profile = (cfg->flags & SEED_FLAG_PROFILE) != 0;
  const int g = cfg->gamma;
  // k_config tree (R36): breadth-first shape, ancestor masks, level spans
  auto& TR = ctx->tree;
  if (cfg->n_tree < 0 || cfg->n_tree > 8 || (cfg->n_tree > 0 && cfg->n_tree != g)) {
    delete ctx;
    return SEED_EINVAL;
  }
  if (cfg->n_tree > 0) {
    TR.n = cfg->n_tree;
    TR.parent = {-1};
    TR.depth = {0};
    TR.lvl_start = {0};
    TR.lvl_len = {1};
    std::vector<int> level{0};
    for (int d = 0; d < TR.n; ++d) {
      const int m = cfg->tree_counts[d];
      if (m < 1 || m > 8) {
        delete ctx;
        return SEED_EINVAL;
      }
      TR.counts.push_back(m);
      std::vector<int> nxt;
      TR.lvl_start.push_back((int)TR.parent.size());
      for (int p : level)
        for (int i = 0; i < m; ++i) {
          TR.parent.push_back(p);
          TR.depth.push_back(d + 1);
          nxt.push_back((int)TR.parent.size() - 1);
        }
      TR.lvl_len.push_back((int)nxt.size());
      level = nxt;
      if (TR.parent.size() > 64) {
        delete ctx;
        return SEED_EINVAL;
      }
    }
    TR.nn = (int)TR.parent.size();
    TR.first.assign(TR.nn, 0);
    TR.cnt.assign(TR.nn, 0);
    TR.anc.assign(TR.nn, 0);
    for (int i = 0; i < TR.nn; ++i) {
      TR.anc[i] = (i == 0 ? 0ull : TR.anc[TR.parent[i]]) | (1ull << i);
      if (i > 0) {
        const int p = TR.parent[i];
        if (TR.cnt[p]++ == 0) TR.first[p] = i;
      }
    }
  }
  const int rows = TR.n > 0 ? TR.nn : g + 1;   // verify rows per stream
  const int max_pos = cfg->max_ctx + std::max(g, rows) + 2;
  ctx->max_pages = (max_pos + ctx->P - 1) / ctx->P;
  ctx->n_slots = cfg->max_streams + 1;  // + one scratch slot for seed_forward_logits / ops
  const int m_cap = std::min(kMaxChunkRows, std::max(ctx->C * rows, 2 * ctx->C));
  auto pool_pages_for = [&](const seed_model_shape& sh) -> size_t {
    const size_t full = (size_t)ctx->n_slots * ctx->max_pages;
    if (cfg->kv_pool_bytes <= 0) return full;
    const int hk = sh.n_kv_heads ? sh.n_kv_heads : sh.n_heads;
    const size_t page_bytes = (size_t)sh.n_layers * 2 * hk * ctx->P * (sh.d_model / sh.n_heads) * 2;
    return std::max<size_t>(ctx->max_pages, std::min(full, (size_t)cfg->kv_pool_bytes / page_bytes));
  };
  seed_status s = build_model(ctx, ctx->tm, cfg->target, cfg->target_w, m_cap, ctx->n_slots, ctx->max_pages,
                              pool_pages_for(cfg->target), max_pos);
  if (s == SEED_OK)
    s = build_model(ctx, ctx->dm, cfg->draft, cfg->draft_w, m_cap, ctx->n_slots, ctx->max_pages,
                    pool_pages_for(cfg->draft), max_pos);
  if (s != SEED_OK) {
    std::string e = ctx->err;
    seed_destroy(ctx);
    return s;
  }
  auto fail_init = [&](seed_status st) {
    seed_destroy(ctx);
    return st;
  };
  if (ctx->arena.init(1 << 20) != cudaSuccess) return fail_init(SEED_ENOMEM);
  const int V = cfg->target.vocab, C = ctx->C, S = ctx->n_slots;
  ctx->slots.resize(S);
  bool ok = true;
  ok &= cudaMalloc(&ctx->tgt_logits, (size_t)C * rows * V * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->drf_logits, (size_t)C * (TR.n > 0 ? TR.nn : g) * V * 4) == cudaSuccess;
  if (TR.n > 0) {
    size_t lvl = 0;
    TR.lvl_off.assign(TR.n + 2, 0);
    for (int d = 2; d <= TR.n; ++d) {   // level d's draft rows: the depth d - 1 nodes
      TR.lvl_off[d] = lvl;
      lvl += (size_t)C * TR.lvl_len[d - 1];
    }
    ok &= cudaMalloc(&TR.tok_lvl, std::max<size_t>(lvl, 1) * 4) == cudaSuccess;
    ok &= cudaMalloc(&TR.tree_tok, (size_t)C * TR.nn * 4) == cudaSuccess;
    ok &= cudaMalloc(&TR.out_node, (size_t)C * TR.n * 4) == cudaSuccess;
    ok &= cudaMalloc(&TR.ch_dev, (size_t)2 * TR.nn * 4) == cudaSuccess;
    if (ok) {
      ok &= cudaMemcpy(TR.ch_dev, TR.first.data(), (size_t)TR.nn * 4, cudaMemcpyHostToDevice) == cudaSuccess;
      ok &= cudaMemcpy(TR.ch_dev + TR.nn, TR.cnt.data(), (size_t)TR.nn * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    }
  }
  ok &= cudaMalloc(&ctx->xs, (size_t)C * g * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->vtok, (size_t)C * (g + 1) * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->out_tok, (size_t)C * (g + 1) * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->out_cnt, (size_t)C * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->out_acc, (size_t)C * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->verify_work, seed::vocab_verify_work_bytes(C, g)) == cudaSuccess;
  if (ok) ok &= cudaMemset(ctx->verify_work, 0, seed::vocab_verify_work_bytes(C, g)) == cudaSuccess;
  const int world = std::max(cfg->world, 1);
  ctx->block_ints = C * (g + 3) + 1;
  ok &= cudaMalloc(&ctx->records, (size_t)ctx->block_ints * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->records_all, (size_t)world * ctx->block_ints * 4) == cudaSuccess;
  ok &= cudaMallocHost(&ctx->records_host, (size_t)world * ctx->block_ints * 4) == cudaSuccess;
  ok &= cudaMallocHost(&ctx->out_host, (size_t)C * (g + 2) * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->dev_err, 2 * sizeof(int32_t)) == cudaSuccess;
  if (ok) ok &= cudaMemset(ctx->dev_err, 0, 2 * sizeof(int32_t)) == cudaSuccess;
  ok &= cudaMallocHost(&ctx->err_host, 2 * sizeof(int32_t)) == cudaSuccess;
  if (ok) ctx->err_host[0] = ctx->err_host[1] = 0;
  ok &= cudaMalloc(&ctx->sids_dev, (size_t)C * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->rs_dev, (size_t)C * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->slots_dev, (size_t)C * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.tlen, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.len_t, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.len_d, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.L, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.r, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.done, (size_t)S * 4) == cudaSuccess;
  ok &= cudaMalloc(&ctx->ds.hist, (size_t)S * max_pos * 4) == cudaSuccess;
  ctx->ds.max_ctx = max_pos;
  ok &= cudaEventCreateWithFlags(&ctx->round_done, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) == cudaSuccess;
  {
    const char* e = getenv("SEED_GRAPHS");
    ctx->use_graphs = !(e && e[0] == '0');
  }
  if (ctx->profile) {
    ctx->rec_cap = 8192;
    ok &= cudaMalloc(&ctx->timing_rec, (size_t)ctx->rec_cap * 4 * 8) == cudaSuccess;
    ok &= cudaMalloc(&ctx->timing_last, (size_t)ctx->rec_cap * 4 * 8) == cudaSuccess;
    ok &= cudaMalloc(&ctx->timing_acc, 4 * 8) == cudaSuccess;
    const char* ce = getenv("SEED_CTA_TRACE");
    if (ce && ce[0] == '1') ok &= cudaMalloc(&ctx->cta_rec, (size_t)ctx->rec_cap * kCtaRec * 8) == cudaSuccess;
    if (ok) {
      std::vector<unsigned long long> init((size_t)ctx->rec_cap * 4);
      for (int i = 0; i < ctx->rec_cap; ++i) {
        init[4 * i] = ~0ull;
        init[4 * i + 1] = ~0ull;
        init[4 * i + 2] = 0ull;
        init[4 * i + 3] = 0ull;
      }
      ok &= cudaMemcpy(ctx->timing_rec, init.data(), init.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess;
      ok &= cudaMemset(ctx->timing_acc, 0, 32) == cudaSuccess;
    }
  }
  if (!ok) return fail_init(SEED_ENOMEM);
  if (seed_book_create(g, cfg->max_new_tokens, C, world, world > 1 ? cfg->rank : 0, &ctx->book) != SEED_OK)
    return fail_init(SEED_ENOMEM);
  if (world > 1) {
    if (!cfg->nccl_id || !g_nccl.load()) return fail_init(SEED_ENCCL);
    Id128 id;
    std::memcpy(&id, cfg->nccl_id, 128);
    if (g_nccl.init(&ctx->comm, world, id, cfg->rank) != 0) return fail_init(SEED_ENCCL);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return fail_init(SEED_ECUDA);
  *out = ctx;
  return SEED_OK;
}

void seed_destroy(seed_ctx ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  free_model(ctx->tm);
  free_model(ctx->dm);
  void* bufs[] = {ctx->dev_err, ctx->tgt_logits, ctx->drf_logits, ctx->xs, ctx->vtok, ctx->out_tok,
                  ctx->out_cnt, ctx->out_acc, ctx->verify_work, ctx->records, ctx->records_all, ctx->sids_dev, ctx->rs_dev,
                  ctx->slots_dev, ctx->ds.tlen, ctx->ds.len_t, ctx->ds.len_d, ctx->ds.L, ctx->ds.r,
                  ctx->ds.done, ctx->ds.hist, ctx->tree.tok_lvl, ctx->tree.tree_tok, ctx->tree.out_node,
                  ctx->tree.ch_dev};
  for (void* p : bufs)
    if (p) cudaFree(p);
  if (ctx->records_host) cudaFreeHost(ctx->records_host);
  if (ctx->out_host) cudaFreeHost(ctx->out_host);
  if (ctx->err_host) cudaFreeHost(ctx->err_host);
  ctx->arena.destroy();
  if (ctx->round_done) cudaEventDestroy(ctx->round_done);
  for (auto* gm : {&ctx->round_graphs})
    for (auto& kv : *gm)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->timing_rec) cudaFree(ctx->timing_rec);
  if (ctx->timing_acc) cudaFree(ctx->timing_acc);
  if (ctx->timing_last) cudaFree(ctx->timing_last);
  if (ctx->cta_rec) cudaFree(ctx->cta_rec);
  if (ctx->book) seed_book_destroy(ctx->book);
  if (ctx->comm && g_nccl.destroy) g_nccl.destroy(ctx->comm);
  delete ctx;
}

seed_status seed_add_stream(seed_ctx ctx, uint32_t gid, const int32_t* prefix, int32_t len, void* stream) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if ((s = check_between(ctx, "seed_add_stream")) != SEED_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (!prefix || len < 2) return fail(ctx, SEED_EINVAL, "seed_add_stream", "prefix must hold >= 2 tokens");
  if ((int32_t)gid < 0) return fail(ctx, SEED_EINVAL, "seed_add_stream", "global id must be < 2^31");
  if ((s = quiesce(ctx)) != SEED_OK) return s;
  if (len + ctx->cfg.max_new_tokens > ctx->cfg.max_ctx)
    return fail(ctx, SEED_ECAPACITY, "seed_add_stream", "prefix + l exceeds max_ctx");
  for (int i = 0; i < len; ++i)
    if (prefix[i] < 0 || prefix[i] >= ctx->cfg.target.vocab)
      return fail(ctx, SEED_EINVAL, "seed_add_stream", "token id out of range");
  if (ctx->gid2slot.count(gid)) return fail(ctx, SEED_EINVAL, "seed_add_stream", "duplicate global id");
  const int slot = free_slot(ctx);
  if (slot < 0) return fail(ctx, SEED_ECAPACITY, "seed_add_stream", "max_streams reached");
  const int g = ctx->cfg.gamma;
  if ((s = ensure_pages(ctx, ctx->tm, slot, len + round_rows(ctx), st)) != SEED_OK) return s;
  if ((s = ensure_pages(ctx, ctx->dm, slot, len + round_rows(ctx), st)) != SEED_OK) return s;
  // Alg. 1 Initialize: prefill both models with the prefix (all but the last token, R6)
  if ((s = prefill(ctx, ctx->tm, slot, prefix, len - 1, 0, nullptr, st)) != SEED_OK) return s;
  if ((s = prefill(ctx, ctx->dm, slot, prefix, len - 1, 0, nullptr, st)) != SEED_OK) return s;
  return install_slot(ctx, slot, gid, prefix, len, st);
}

seed_status seed_fork_stream(seed_ctx ctx, uint32_t src_gid, uint32_t gid, void* stream) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if ((s = check_between(ctx, "seed_fork_stream")) != SEED_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = quiesce(ctx)) != SEED_OK) return s;
  auto it = ctx->gid2slot.find(src_gid);
  if (it == ctx->gid2slot.end()) return fail(ctx, SEED_EINVAL, "seed_fork_stream", "unknown source id");
  if (ctx->gid2slot.count(gid) || (int32_t)gid < 0)
    return fail(ctx, SEED_EINVAL, "seed_fork_stream", "duplicate or invalid global id");
  const int src = it->second;
  const seed::BookStream& from = stream_of(ctx, src_gid);
  if (from.r != 0 || from.L != 0)  // only a freshly prefilled stream (no round yet)
    return fail(ctx, SEED_ESTATE, "seed_fork_stream", "source stream has already run a round");
  const int slot = free_slot(ctx);
  if (slot < 0) return fail(ctx, SEED_ECAPACITY, "seed_fork_stream", "max_streams reached");
  const std::vector<int32_t> prefix = from.T;
  const int len = (int)prefix.size(), g = ctx->cfg.gamma;
  // The prefilled K/V of positions 0 .. len - 2.  Rounds write positions >= len - 2 (the draft's
  // first step rewrites len - 2, R22; the target writes from len - 1), so pages holding only
  // positions < len - 2 are never written again: the new slot shares them (refcounted).  The page
  // holding position len - 2 is copied on the device; later pages are fresh.  Bit-identical to a
  // fresh prefill (test_fork_stream_equals_add_stream).
  const int shared = (len - 2) / ctx->P;
  for (Model* m : {&ctx->tm, &ctx->dm}) {
    int32_t* pt_src = m->page_table + (size_t)src * ctx->max_pages;
    int32_t* pt_new = m->page_table + (size_t)slot * ctx->max_pages;
    for (int i = 0; i < shared; ++i) {
      pt_new[i] = pt_src[i];
      ++m->refs[pt_new[i]];
    }
    m->held[slot] = shared;
    if (shared > 0)
      CK(cudaMemcpyAsync(m->page_table_dev + (size_t)slot * ctx->max_pages, pt_new, (size_t)shared * 4,
                         cudaMemcpyHostToDevice, st));
    if ((s = ensure_pages(ctx, *m, slot, len + round_rows(ctx), st)) != SEED_OK) {
      release_pages(ctx->tm, slot, ctx->max_pages);  // the slot was never installed: drop its references
      release_pages(ctx->dm, slot, ctx->max_pages);
      return s;
    }
    const size_t elems = m->kv.page_elems();
    CK(cudaMemcpyAsync(m->kv.pool + (size_t)pt_new[shared] * elems, m->kv.pool + (size_t)pt_src[shared] * elems,
                       elems * sizeof(bf16), cudaMemcpyDeviceToDevice, st));
  }
  return install_slot(ctx, slot, gid, prefix.data(), len, st);
}

seed_status seed_schedule_round(seed_ctx ctx, int32_t* batch_ids, int32_t cap, int32_t* n) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if (!n || cap < 0 || (cap > 0 && !batch_ids)) return fail(ctx, SEED_EINVAL, "seed_schedule_round", "args");
  *n = 0;
  if ((s = check_between(ctx, "seed_schedule_round")) != SEED_OK) return s;
  const seed_status done_st = complete_round(ctx);   // SEED_EDEVICE still schedules the next round
  if (done_st != SEED_OK && done_st != SEED_EDEVICE) return done_st;
  s = seed_book_schedule(ctx->book, batch_ids, cap, n);
  if (s != SEED_OK) return fail(ctx, s, "seed_schedule_round", "no ready stream (liveness)");
  return done_st;
}

seed_status seed_global_pending(seed_ctx ctx, int64_t* n) {
  if (!ctx || !n) return SEED_EINVAL;
  seed_status s = complete_round(ctx);
  if (s != SEED_OK && s != SEED_EDEVICE) return s;
  seed_book_global_pending(ctx->book, n);
  if (*n < 0 && std::max(ctx->cfg.world, 1) == 1) *n = ctx->book->undone;   // no exchange yet: own count
  return s;
}

seed_status seed_draft_round(seed_ctx ctx, const int32_t* ids, int32_t n, void* stream) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if ((s = check_between(ctx, "seed_draft_round")) != SEED_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> slots;
  if ((s = map_batch(ctx, ids, n, slots)) != SEED_OK) return s;
  if (ctx->round_pending) {
    s = complete_round(ctx);
    if (s != SEED_OK && s != SEED_EDEVICE) return s;
    if ((s = map_batch(ctx, ids, n, slots)) != SEED_OK) return s;   // the previous round may have finished some
  }
  const int g = ctx->cfg.gamma;
  std::vector<int32_t> batch(ids, ids + n);
  for (int b = 0; b < n; ++b) {
    const int T = (int)stream_of(ctx, (uint32_t)ids[b]).T.size();
    if ((s = ensure_pages(ctx, ctx->tm, slots[b], T + round_rows(ctx), st)) != SEED_OK) return s;
    if ((s = ensure_pages(ctx, ctx->dm, slots[b], T + round_rows(ctx), st)) != SEED_OK) return s;
  }
  RoundPlan& P = ctx->plan;
  if ((s = build_round_plan(ctx, batch, slots, P)) != SEED_OK) return s;
  if ((s = run_phase(ctx, n, true, st)) != SEED_OK) return s;
  ctx->drafted = batch;
  ctx->draft_called = true;
  return SEED_OK;
}

seed_status seed_verify(seed_ctx ctx, const int32_t* ids, int32_t n, int32_t* out_tok, int32_t* out_cnt,
                        void* stream) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (!ctx->draft_called || (int)ctx->drafted.size() != n || (n > 0 && !std::equal(ids, ids + n, ctx->drafted.begin())))
    return fail(ctx, SEED_ESTATE, "seed_verify", "batch was not drafted");
  if ((s = run_phase(ctx, n, false, st)) != SEED_OK) return s;
  const int g = ctx->cfg.gamma;
  if (out_tok && n > 0)
    CK(cudaMemcpyAsync(out_tok, ctx->out_tok, (size_t)n * (g + 1) * 4, cudaMemcpyDeviceToDevice, st));
  if (out_cnt && n > 0) CK(cudaMemcpyAsync(out_cnt, ctx->out_cnt, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  ctx->round_pending = true;
  ctx->last_batch = ctx->drafted;
  ctx->drafted.clear();
  ctx->draft_called = false;
  return SEED_OK;
}

seed_status seed_round_host(seed_ctx ctx, const int32_t* ids, int32_t n, int32_t* out_tok_host, int32_t* out_cnt_host,
                            void* stream) {
  seed_status s = seed_draft_round(ctx, ids, n, stream);
  if (s != SEED_OK) return s;
  if ((s = seed_verify(ctx, ids, n, nullptr, nullptr, stream)) != SEED_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = ctx->cfg.gamma;
  // through pinned staging: both copies queue behind the round, one synchronisation (a copy into
  // pageable memory would block the host per copy)
  int32_t* stage_tok = ctx->out_host;
  int32_t* stage_cnt = ctx->out_host + (size_t)ctx->C * (g + 1);
  if (out_tok_host && n > 0)
    CK(cudaMemcpyAsync(stage_tok, ctx->out_tok, (size_t)n * (g + 1) * 4, cudaMemcpyDeviceToHost, st));
  if (out_cnt_host && n > 0) CK(cudaMemcpyAsync(stage_cnt, ctx->out_cnt, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (out_tok_host && n > 0) std::memcpy(out_tok_host, stage_tok, (size_t)n * (g + 1) * 4);
  if (out_cnt_host && n > 0) std::memcpy(out_cnt_host, stage_cnt, (size_t)n * 4);
  return SEED_OK;
}

seed_status seed_get_tokens(seed_ctx ctx, uint32_t gid, int32_t* dst, int32_t cap, int32_t* len) {
  if (!ctx || !len || cap < 0) return SEED_EINVAL;
  seed_status s = complete_round(ctx);
  if (s != SEED_OK && s != SEED_EDEVICE) return s;
  const seed_status t = seed_book_tokens(ctx->book, gid, dst, cap, len);
  return t != SEED_OK ? t : s;
}

seed_status seed_stream_info(seed_ctx ctx, uint32_t gid, int32_t* info) {
  if (!ctx || !info) return SEED_EINVAL;
  seed_status s = complete_round(ctx);
  if (s != SEED_OK && s != SEED_EDEVICE) return s;
  auto it = ctx->gid2slot.find(gid);
  if (it == ctx->gid2slot.end()) return SEED_ENOTFOUND;
  const seed::BookStream& b = stream_of(ctx, gid);
  const SlotState& ss = ctx->slots[it->second];
  info[0] = (int32_t)b.T.size();
  info[1] = b.L;
  info[2] = b.r;
  info[3] = b.done ? 1 : 0;
  info[4] = ss.len_t;
  info[5] = ss.len_d;
  info[6] = ctx->tm.held[it->second];
  info[7] = it->second;
  return s;
}

seed_status seed_remove_stream(seed_ctx ctx, uint32_t gid) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if ((s = check_between(ctx, "seed_remove_stream")) != SEED_OK) return s;
  if (ctx->round_pending) {
    s = complete_round(ctx);
    if (s != SEED_OK && s != SEED_EDEVICE) return s;
  }
  auto it = ctx->gid2slot.find(gid);
  if (it == ctx->gid2slot.end()) return SEED_ENOTFOUND;
  const int slot = it->second;
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(ctx, SEED_ECUDA, "seed_remove_stream", "sync");
  release_pages(ctx->tm, slot, ctx->max_pages);
  release_pages(ctx->dm, slot, ctx->max_pages);
  ctx->slots[slot] = SlotState();
  ctx->gid2slot.erase(it);
  // forget the id: scheduler entry, tokens (a removed id may be added again)
  seed_book_remove(ctx->book, gid);
  return s;
}

seed_status seed_device_status(seed_ctx ctx, uint32_t* bits, int64_t* fallbacks) {
  if (!ctx) return SEED_EINVAL;
  seed_status s = complete_round(ctx);
  if (s != SEED_OK && s != SEED_EDEVICE) return s;
  if (bits) *bits = ctx->err_bits_seen;
  if (fallbacks) *fallbacks = ctx->fallbacks;
  return SEED_OK;
}

seed_status seed_forward_logits(seed_ctx ctx, int32_t which, const int32_t* tokens, int32_t n, float* logits,
                                void* stream) {
  seed_status s = check_ctx(ctx);
  if (s != SEED_OK) return s;
  if ((s = check_between(ctx, "seed_forward_logits")) != SEED_OK) return s;
  if (!tokens || n < 1 || !logits) return fail(ctx, SEED_EINVAL, "seed_forward_logits", "args");
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = quiesce(ctx)) != SEED_OK) return s;
  Model& m = which ? ctx->tm : ctx->dm;
  const int slot = ctx->n_slots - 1;  // scratch slot
  if ((s = ensure_pages(ctx, m, slot, n, st)) != SEED_OK) return s;
  s = prefill(ctx, m, slot, tokens, n, 0, logits, st);
  CK(cudaStreamSynchronize(st));
  release_pages(m, slot, ctx->max_pages);
  return s;
}

seed_status seed_last_round_buffers(seed_ctx ctx, const float** t, const float** d, const int32_t** x) {
  if (!ctx) return SEED_EINVAL;
  if (t) *t = ctx->tgt_logits;
  if (d) *d = ctx->drf_logits;
  if (x) *x = ctx->tree.n > 0 ? ctx->tree.tree_tok : ctx->xs;   // trees: [n][nodes + 1] root + node tokens
  return SEED_OK;
}

seed_status seed_get_profile(seed_ctx ctx, double* gemm_ms, int64_t* launches, double* bytes, int64_t* kernels,
                             double* gemm_span_ms) {
  if (!ctx) return SEED_EINVAL;
  double ms = 0, span = 0;
  if (ctx->timing_acc) {
    unsigned long long acc[4] = {0, 0, 0, 0};
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(acc, ctx->timing_acc, sizeof(acc), cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(ctx, SEED_ECUDA, "seed_get_profile", "");
    ms = acc[0] * 1e-6;
    span = acc[2] * 1e-6;
  }
  if (gemm_ms) *gemm_ms = ms;
  if (gemm_span_ms) *gemm_span_ms = span;
  if (launches) *launches = ctx->gemm_launches;
  if (bytes) *bytes = ctx->gemm_bytes;
  if (kernels) *kernels = ctx->kernel_launches;
  return SEED_OK;
}

seed_status seed_gemm_trace(seed_ctx ctx, uint64_t* out, int32_t cap, int32_t* n) {
  if (!ctx || !n) return SEED_EINVAL;
  *n = 0;
  if (!ctx->timing_last) return SEED_OK;
  const int nd = std::min(cap, ctx->last_draft_recs);
  const int nv = std::min(cap - nd, ctx->last_verify_recs);
  const size_t half = (size_t)ctx->rec_cap / 2;
  if (cudaDeviceSynchronize() != cudaSuccess ||
      (nd > 0 && cudaMemcpy(out, ctx->timing_last, (size_t)nd * 32, cudaMemcpyDeviceToHost) != cudaSuccess) ||
      (nv > 0 && cudaMemcpy(out + 4 * (size_t)nd, ctx->timing_last + 4 * half, (size_t)nv * 32,
                            cudaMemcpyDeviceToHost) != cudaSuccess))
    return fail(ctx, SEED_ECUDA, "seed_gemm_trace", "");
  *n = nd + nv;
  return SEED_OK;
}

seed_status seed_gemm_cta_trace(seed_ctx ctx, int32_t launch, uint64_t* out, int32_t* n_cta) {
  if (!ctx || !out || !n_cta || launch < 0) return SEED_EINVAL;
  *n_cta = 0;
  if (!ctx->cta_rec) return SEED_OK;
  const int nd = ctx->last_draft_recs, nv = ctx->last_verify_recs;
  if (launch >= nd + nv) return SEED_EINVAL;
  const size_t idx = launch < nd ? (size_t)launch : (size_t)ctx->rec_cap / 2 + (launch - nd);
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(out, ctx->cta_rec + idx * kCtaRec, kCtaRec * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(ctx, SEED_ECUDA, "seed_gemm_cta_trace", "");
  *n_cta = (int32_t)kCtaRec;
  return SEED_OK;
}

seed_status seed_set_profile(seed_ctx ctx, int32_t on) {
  if (!ctx) return SEED_EINVAL;
  if (on && !ctx->timing_rec) return fail(ctx, SEED_ESTATE, "seed_set_profile", "created without SEED_FLAG_PROFILE");
  if (ctx->draft_called) return fail(ctx, SEED_ESTATE, "seed_set_profile", "a drafted batch is not verified");
  ctx->profile = on != 0;
  return SEED_OK;
}

seed_status seed_reset_profile(seed_ctx ctx) {
  if (!ctx) return SEED_EINVAL;
  if (ctx->timing_acc && cudaMemset(ctx->timing_acc, 0, 4 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(ctx, SEED_ECUDA, "seed_reset_profile", "");
  ctx->gemm_bytes = 0;
  ctx->gemm_launches = 0;
  ctx->kernel_launches = 0;
  return SEED_OK;
}

// ====================================================================== op-level ABI
seed_status seed_op_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int32_t n,
                           uint32_t* out, void* stream) {
  if (!out || n < 0) return SEED_EINVAL;
  return seed::philox_fill(c0, c1, c2, c3, k0, k1, n, out, (cudaStream_t)stream) == cudaSuccess ? SEED_OK
                                                                                               : SEED_ECUDA;
}

seed_status seed_op_gemm(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* Y, void* stream) {
  if (!W || !X || !Y || N < 4 || N % 4 || K < 64 || K % 64 || M < 1) return SEED_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GemmPlan p;
  seed::gemm_plan(&p, W, N, K);
  // X read in place: boxes of 64 x m_pad rows per 256-row token tile (rows past M read as zero and
  // only feed accumulator columns that are never stored)
  CUtensorMap tm;
  seed_status s = SEED_OK;
  if (!seed::encode_tmap_2d(&tm, X, (uint64_t)K, (uint64_t)M, 64, (uint32_t)seed::gemm_mpad(M))) s = SEED_ECUDA;
  if (s == SEED_OK) {
    seed::GemmIO io;
    io.tmX = &tm;
    io.Y = Y;
    io.ldY = N;
    if (seed::gemm_run(p, M, io, st) != cudaSuccess) s = SEED_ECUDA;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) s = SEED_ECUDA;
  seed::gemm_plan_free(&p);
  return s;
}

seed_status seed_op_verify(const float* zt, const float* zd, const int32_t* xs, int32_t B, int32_t gamma, int32_t V,
                           float temperature, uint64_t seed, const uint32_t* sids, const int32_t* rs, int32_t bonus,
                           int32_t* out_tok, int32_t* out_cnt, int32_t* out_acc, float* dbg, double* stats,
                           void* stream) {
  if (!zt || !zd || !xs || B < 1 || gamma < 1 || gamma > 16 || V < 1 || !(temperature > 0.f) || !sids || !rs ||
      !out_tok)
    return SEED_EINVAL;
  seed::VerifyArgs a{};
  a.zt = zt;
  a.zd = zd;
  a.xs = xs;
  a.zt_stride_b = (long)(gamma + 1) * V;
  a.zd_stride_b = (long)gamma * V;
  a.B = B;
  a.gamma = gamma;
  a.V = V;
  a.T = temperature;
  a.k0 = (uint32_t)(seed & 0xFFFFFFFFu);
  a.k1 = (uint32_t)(seed >> 32);
  a.sids = sids;
  a.rs = rs;
  a.bonus = bonus;
  a.out_tok = out_tok;
  a.out_cnt = out_cnt;
  a.out_acc = out_acc;
  a.dbg = dbg;
  a.stats = stats;
  const size_t wb = seed::vocab_verify_work_bytes(B, gamma);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMallocAsync(&a.work, wb, st) != cudaSuccess) return SEED_ENOMEM;
  bool ok = cudaMemsetAsync(a.work, 0, wb, st) == cudaSuccess && seed::vocab_verify(a, st) == cudaSuccess;
  ok &= cudaFreeAsync(a.work, st) == cudaSuccess;
  return ok ? SEED_OK : SEED_ECUDA;
}

seed_status seed_op_draft_sample(const float* z, int32_t ld, int32_t B, int32_t V, float temperature, uint64_t seed,
                                 const uint32_t* sids, const int32_t* rs, int32_t j, int32_t* out, void* stream) {
  if (!z || B < 1 || V < 1 || !sids || !rs || !out || !(temperature > 0.f)) return SEED_EINVAL;
  return seed::draft_sample(z, ld, B, V, temperature, (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32), sids,
                            rs, j, out, 1, nullptr, 0, nullptr, (cudaStream_t)stream) == cudaSuccess
             ? SEED_OK
             : SEED_ECUDA;
}

seed_status seed_op_draft_topk(const float* z, int32_t ld, int32_t B, int32_t V, float temperature, uint64_t seed,
                               const uint32_t* sids, const int32_t* rs, int32_t node, int32_t m, int32_t* out,
                               int32_t out_stride, int32_t first, void* stream) {
  if (!z || B < 1 || V < 1 || !sids || !rs || !out || !(temperature > 0.f) || m < 1 || m > 8 || node < 0 || m > V)
    return SEED_EINVAL;
  return seed::draft_topk(z, ld, B, V, temperature, (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32), sids, rs,
                          node, m, out, out_stride, first, nullptr, 0, nullptr, (cudaStream_t)stream) == cudaSuccess
             ? SEED_OK
             : SEED_ECUDA;
}

seed_status seed_op_verify_tree(const float* zt, const float* zd, const int32_t* tok, int32_t B, const int32_t* counts,
                                int32_t n_counts, int32_t V, float temperature, uint64_t seed, const uint32_t* sids,
                                const int32_t* rs, int32_t bonus, int32_t* out_tok, int32_t* out_cnt, int32_t* out_node,
                                void* stream) {
  if (!zt || !zd || !tok || B < 1 || !counts || n_counts < 1 || n_counts > 15 || V < 1 || !(temperature > 0.f) ||
      !sids || !rs || !out_tok || !out_cnt)
    return SEED_EINVAL;
  // breadth-first shape: children of every node contiguous
  std::vector<int32_t> first(1, 0), cnt(1, 0);
  std::vector<int> level{0};
  for (int d = 0; d < n_counts; ++d) {
    if (counts[d] < 1 || counts[d] > 8 || counts[d] > V) return SEED_EINVAL;
    std::vector<int> nxt;
    for (int p : level) {
      first[p] = (int32_t)first.size();
      cnt[p] = counts[d];
      for (int i = 0; i < counts[d]; ++i) {
        first.push_back(0);
        cnt.push_back(0);
        nxt.push_back((int)first.size() - 1);
      }
    }
    level = nxt;
  }
  const int nn = (int)first.size();   // nodes incl. the root
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* dev = nullptr;
  if (cudaMallocAsync(&dev, (size_t)2 * nn * 4, st) != cudaSuccess) return SEED_ENOMEM;
  bool ok = cudaMemcpyAsync(dev, first.data(), (size_t)nn * 4, cudaMemcpyHostToDevice, st) == cudaSuccess &&
            cudaMemcpyAsync(dev + nn, cnt.data(), (size_t)nn * 4, cudaMemcpyHostToDevice, st) == cudaSuccess &&
            seed::verify_tree(zt, (long)nn * V, zd, (long)nn * V, tok, nn, dev, dev + nn, B, n_counts, V, temperature,
                              (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32), sids, rs, bonus, out_tok, out_cnt,
                              out_node, nullptr, st) == cudaSuccess;
  ok &= cudaStreamSynchronize(st) == cudaSuccess;
  cudaFree(dev);
  return ok ? SEED_OK : SEED_ECUDA;
}

seed_status seed_op_decoder_layer_tree(const seed_model_shape* shape, const void* const* w, const float* x_in,
                                       int32_t M, int32_t ctx_len, const int32_t* parent, const void* k_prev,
                                       const void* v_prev, float* x_out, void* k_new, void* v_new, void* stream) {
  return decoder_layer_impl(shape, w, x_in, M, ctx_len, parent, k_prev, v_prev, x_out, k_new, v_new, stream);
}

seed_status seed_op_decoder_layer(const seed_model_shape* shape, const void* const* w, const float* x_in, int32_t M,
                                  int32_t ctx_len, const void* k_prev, const void* v_prev, float* x_out, void* k_new,
                                  void* v_new, void* stream) {
  return decoder_layer_impl(shape, w, x_in, M, ctx_len, nullptr, k_prev, v_prev, x_out, k_new, v_new, stream);
}

}  // extern "C"

namespace {
// one decoder layer on M rows of one sequence after ctx_len cached keys; parent (host, optional):
// the rows form a tree (row 0 the root, parent[i] < i) -- RoPE position ctx_len + depth, attention
// to the cached keys and the row's ancestors and itself (Figure 7, R36)
seed_status decoder_layer_impl(const seed_model_shape* shape, const void* const* w, const float* x_in, int32_t M,
                               int32_t ctx_len, const int32_t* parent, const void* k_prev, const void* v_prev,
                               float* x_out, void* k_new, void* v_new, void* stream) {
  if (!shape || !w || !x_in || !x_out || M < 1 || M > kMaxChunkRows || ctx_len < 0) return SEED_EINVAL;
  if (parent && M > 64) return SEED_EINVAL;
  std::vector<int32_t> tpos;
  std::vector<uint64_t> tanc;
  if (parent) {
    tpos.resize(M);
    tanc.resize(M);
    for (int i = 0; i < M; ++i) {
      if ((i == 0) != (parent[i] < 0) || parent[i] >= i) return SEED_EINVAL;
      tpos[i] = i == 0 ? ctx_len : tpos[parent[i]] + 1;
      tanc[i] = (i == 0 ? 0ull : tanc[parent[i]]) | (1ull << i);
    }
  }
  if (ctx_len > 0 && (!k_prev || !v_prev)) return SEED_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  // a throw-away context holding a one-layer model (weights packed exactly as seed_init does)
  seed_model_shape sh = *shape;
  sh.n_layers = 1;
  seed_ctx ctx = new seed_ctx_s;
  ctx->P = 16;
  const int max_pos = ctx_len + M + 1;
  ctx->max_pages = (max_pos + ctx->P - 1) / ctx->P;
  ctx->n_slots = 1;
  // the model builder needs embed / lm_head: give it zero-size stand-ins by pointing at layer weights
  bf16* dummy = nullptr;
  seed_status s = SEED_OK;
  const size_t Vd = (size_t)sh.vocab * sh.d_model;
  if (cudaMalloc(&dummy, Vd * 2) != cudaSuccess) {
    delete ctx;
    return SEED_ENOMEM;
  }
  cudaMemset(dummy, 0, Vd * 2);
  seed_model_weights mw{dummy, w, w[7], dummy};
  s = build_model(ctx, ctx->tm, sh, mw, M, 1, ctx->max_pages, ctx->max_pages, max_pos);
  Model& m = ctx->tm;
  if (s == SEED_OK && ctx->arena.init(1 << 16) != cudaSuccess) s = SEED_ENOMEM;
  if (s == SEED_OK) s = ensure_pages(ctx, m, 0, ctx_len + M, st);
  if (s == SEED_OK && ctx_len > 0 &&
      seed::kv_write_dense(m.kv, 0, 0, ctx_len, (const bf16*)k_prev, (const bf16*)v_prev, st) != cudaSuccess)
    s = SEED_ECUDA;
  if (s == SEED_OK) {
    ctx->arena.begin();
    std::vector<Segment> segs{{0, ctx_len, M, -1}};
    ChunkDesc c;
    size_t tok_off;
    pack_chunk(ctx, segs, 0, &c, &tok_off);
    if (parent) {   // per-row tree positions and ancestor masks in the descriptor arena
      const size_t o_p = ctx->arena.alloc(M), o_a = ctx->arena.alloc(2 * M + 2);
      if (o_a == (size_t)-1) s = SEED_ENOMEM;
      if (s == SEED_OK) {
        const size_t o_a8 = (o_a + 1) & ~(size_t)1;   // 8-byte aligned
        std::memcpy(ctx->arena.host + o_p, tpos.data(), (size_t)M * 4);
        std::memcpy(ctx->arena.host + o_a8, tanc.data(), (size_t)M * 8);
        c.row_pos = ctx->arena.dev + o_p;
        c.anc = reinterpret_cast<const uint64_t*>(ctx->arena.dev + o_a8);
      }
    }
    if (s == SEED_OK && ctx->arena.upload(st) != cudaSuccess) s = SEED_ECUDA;
    const float eps = sh.rms_eps > 0 ? sh.rms_eps : 1e-5f;
    if (s == SEED_OK && cudaMemcpyAsync(m.x, x_in, (size_t)M * m.d * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      s = SEED_ECUDA;
    (void)eps;
    if (s == SEED_OK) s = forward_chunk(ctx, m, c, st, 0, 1, false);
    if (s == SEED_OK && cudaMemcpyAsync(x_out, m.x, (size_t)M * m.d * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      s = SEED_ECUDA;
    // copy the appended K/V back out (dense) through a scratch pass over the pages
    if (s == SEED_OK && (k_new || v_new)) {
      const size_t per = (size_t)m.Hk * m.Dh;
      std::vector<bf16> hk(per * M), hv(per * M);
      cudaStreamSynchronize(st);
      for (int p = 0; p < M && s == SEED_OK; ++p) {
        const int pos = ctx_len + p;
        const int page = m.page_table[pos / ctx->P];
        for (int h = 0; h < m.Hk; ++h) {
          const size_t ko = m.kv.offset(page, 0, 0, h, pos % ctx->P), vo = m.kv.offset(page, 0, 1, h, pos % ctx->P);
          if (k_new && cudaMemcpy((bf16*)k_new + ((size_t)p * m.Hk + h) * m.Dh, m.kv.pool + ko, m.Dh * 2,
                                  cudaMemcpyDeviceToDevice) != cudaSuccess)
            s = SEED_ECUDA;
          if (v_new && cudaMemcpy((bf16*)v_new + ((size_t)p * m.Hk + h) * m.Dh, m.kv.pool + vo, m.Dh * 2,
                                  cudaMemcpyDeviceToDevice) != cudaSuccess)
            s = SEED_ECUDA;
        }
      }
    }
  }
  cudaStreamSynchronize(st);
  if (s == SEED_OK && cudaGetLastError() != cudaSuccess) s = SEED_ECUDA;
  free_model(ctx->tm);
  ctx->arena.destroy();
  cudaFree(dummy);
  delete ctx;
  return s;
}
}  // namespace
