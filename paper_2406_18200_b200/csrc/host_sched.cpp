// host_sched.cpp -- H1: the FCFS rounds scheduler, the a6 token table and the per-rank round
// book that ties them together (host only, no CUDA; the engine drives the same book).
//
// Scheduler (Alg. 1; lock-step batched reading R9):
//   queue Q of global ids, FCFS; ready flag per stream (the paper's draft label
//   map): 0 after drafting, 1 after verification; undone streams re-enter
//   at the tail in batch order -- the "rounds" of P:206 / P:230; ties at admission -> lowest
//   id (R10); a done stream met in the queue is dropped; an empty pop while work
//   remains is a liveness violation reported as SEED_ESTATE.
#include <algorithm>
#include <new>

#include "host_book.h"

extern "C" {

seed_status seed_sched_create(const int32_t* ids, int32_t n, seed_sched* out) {
  if (!out || n < 0 || (n > 0 && !ids)) return SEED_EINVAL;
  seed_sched s = new (std::nothrow) seed_sched_s;
  if (!s) return SEED_ENOMEM;
  std::vector<int32_t> v(ids, ids + n);
  std::sort(v.begin(), v.end());
  for (int32_t id : v) {
    if (s->ready.count(id)) {
      delete s;
      return SEED_EINVAL;
    }
    s->queue.push_back(id);
    s->ready[id] = 1;
    s->done[id] = 0;
  }
  *out = s;
  return SEED_OK;
}

seed_status seed_sched_add(seed_sched s, int32_t id) {
  if (!s) return SEED_EINVAL;
  if (s->ready.count(id) && !s->done[id]) return SEED_EINVAL;
  s->ready[id] = 1;
  s->done[id] = 0;
  s->queue.push_back(id);
  return SEED_OK;
}

seed_status seed_sched_pop(seed_sched s, int32_t* out, int32_t cap, int32_t* n) {
  if (!s || !n || cap < 0 || (cap > 0 && !out)) return SEED_EINVAL;
  int32_t k = 0;
  while (!s->queue.empty() && k < cap) {
    const int32_t id = s->queue.front();
    s->queue.pop_front();
    if (s->done[id]) continue;           // S:211 dropped
    if (!s->ready[id]) return SEED_ESTATE;  // ready-flag safety
    s->ready[id] = 0;
    out[k++] = id;
  }
  *n = k;
  if (k == 0 && cap > 0 && !seed_sched_all_done(s)) return SEED_ESTATE;  // liveness
  return SEED_OK;
}

seed_status seed_sched_complete(seed_sched s, const int32_t* batch, const int32_t* done, int32_t n) {
  if (!s || n < 0 || (n > 0 && (!batch || !done))) return SEED_EINVAL;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t id = batch[i];
    if (!s->ready.count(id)) return SEED_EINVAL;
    s->ready[id] = 1;
    s->done[id] = done[i] ? 1 : 0;
    if (!done[i]) s->queue.push_back(id);  // rounds: back to the tail
  }
  return SEED_OK;
}

int32_t seed_sched_all_done(seed_sched s) {
  if (!s) return 1;
  for (const auto& kv : s->done)
    if (!kv.second) return 0;
  return 1;
}

void seed_sched_destroy(seed_sched s) { delete s; }

seed_status seed_sched_remove(seed_sched s, int32_t id) {
  if (!s) return SEED_EINVAL;
  if (!s->ready.count(id)) return SEED_ENOTFOUND;
  s->queue.erase(std::remove(s->queue.begin(), s->queue.end(), id), s->queue.end());
  s->ready.erase(id);
  s->done.erase(id);
  return SEED_OK;
}

seed_status seed_table_create(int32_t record_stride, seed_table* out) {
  if (!out || record_stride < 3) return SEED_EINVAL;
  seed_table t = new (std::nothrow) seed_table_s;
  if (!t) return SEED_ENOMEM;
  t->stride = record_stride;
  *out = t;
  return SEED_OK;
}

seed_status seed_table_merge(seed_table t, const int32_t* records, int32_t n_records) {
  if (!t || n_records < 0 || (n_records > 0 && !records)) return SEED_EINVAL;
  for (int32_t i = 0; i < n_records; ++i) {
    const int32_t* r = records + (size_t)i * t->stride;
    if (r[0] < 0) continue;  // padding record
    const int32_t c = r[1];
    if (c < 0 || c > t->stride - 2) return SEED_EINVAL;
    auto& v = t->tokens[(uint32_t)r[0]];
    v.insert(v.end(), r + 2, r + 2 + c);
  }
  return SEED_OK;
}

seed_status seed_table_get(seed_table t, uint32_t gid, int32_t* dst, int32_t cap, int32_t* len) {
  if (!t || !len) return SEED_EINVAL;
  auto it = t->tokens.find(gid);
  if (it == t->tokens.end()) return SEED_ENOTFOUND;
  *len = (int32_t)it->second.size();
  if (dst) std::copy(it->second.begin(), it->second.begin() + std::min<int32_t>(cap, *len), dst);
  return SEED_OK;
}

seed_status seed_table_erase(seed_table t, uint32_t gid) {
  if (!t) return SEED_EINVAL;
  return t->tokens.erase(gid) ? SEED_OK : SEED_ENOTFOUND;
}

void seed_table_destroy(seed_table t) { delete t; }

/* ---------------------------------------------------------------- round book (H1 + a5 + a6)
 * One rank's host bookkeeping of the round: its own streams' validated tokens
 * (Alg. 1, R6/R7), the FCFS scheduler, and the exchange block every rank contributes
 * to the per-round all-gather: [cap] records of [gid, c, tok_0 .. tok_gamma] (padding
 * gid = -1) followed by one word, the number of this rank's streams still undone after the
 * round.  The engine's K5 kernel writes the block on the device; seed_book_pack writes the same
 * block on the host (CPU tests, world > 1 without a GPU).  Every rank joins every round's
 * exchange -- with an empty batch once its own streams are done -- until the gathered undone
 * counts sum to zero (seed_book_global_pending), so uneven completion cannot hang a collective. */
namespace {
seed_status book_complete_own(seed_book b, const int32_t* blk, std::vector<int32_t>& batch, std::vector<int32_t>& done) {
  const int stride = b->gamma + 3;
  for (int i = 0; i < b->cap; ++i) {
    const int32_t* r = blk + (size_t)i * stride;
    if (r[0] < 0) continue;
    auto it = b->own.find((uint32_t)r[0]);
    if (it == b->own.end() || it->second.done) return SEED_EINVAL;
    const int32_t c = r[1];
    if (c < 0 || c > b->gamma + 1) return SEED_EINVAL;
    seed::BookStream& st = it->second;
    st.T.insert(st.T.end(), r + 2, r + 2 + c);
    st.L += c;
    st.r += 1;
    st.done = st.L >= b->max_new;
    if (st.done) --b->undone;
    batch.push_back(r[0]);
    done.push_back(st.done ? 1 : 0);
  }
  return SEED_OK;
}
}  // namespace

seed_status seed_book_create(int32_t gamma, int32_t max_new, int32_t cap, int32_t world, int32_t rank,
                             seed_book* out) {
  if (!out || gamma < 1 || max_new < 1 || cap < 1 || world < 1 || rank < 0 || rank >= world) return SEED_EINVAL;
  seed_book b = new (std::nothrow) seed_book_s;
  if (!b) return SEED_ENOMEM;
  b->gamma = gamma;
  b->max_new = max_new;
  b->cap = cap;
  b->world = world;
  b->rank = rank;
  b->table.stride = gamma + 3;
  *out = b;
  return SEED_OK;
}

seed_status seed_book_add(seed_book b, uint32_t gid, const int32_t* prefix, int32_t len) {
  if (!b || !prefix || len < 1 || (int32_t)gid < 0) return SEED_EINVAL;
  if (b->own.count(gid)) return SEED_EINVAL;
  seed_status s = seed_sched_add(&b->sched, (int32_t)gid);
  if (s != SEED_OK) return s;
  seed::BookStream st;
  st.T.assign(prefix, prefix + len);
  st.prompt_len = len;
  b->own.emplace(gid, std::move(st));
  b->table.tokens.erase(gid);   // a reused id starts from an empty record
  ++b->undone;
  return SEED_OK;
}

seed_status seed_book_remove(seed_book b, uint32_t gid) {
  if (!b) return SEED_EINVAL;
  auto it = b->own.find(gid);
  if (it == b->own.end()) return SEED_ENOTFOUND;
  if (!it->second.done) --b->undone;
  b->own.erase(it);
  seed_sched_remove(&b->sched, (int32_t)gid);
  b->table.tokens.erase(gid);
  return SEED_OK;
}

seed_status seed_book_schedule(seed_book b, int32_t* ids, int32_t cap, int32_t* n) {
  if (!b || !n || cap < 0 || (cap > 0 && !ids)) return SEED_EINVAL;
  *n = 0;
  if (seed_sched_all_done(&b->sched)) return SEED_OK;
  return seed_sched_pop(&b->sched, ids, std::min(cap, b->cap), n);
}

seed_status seed_book_pack(seed_book b, const int32_t* ids, int32_t n, const int32_t* out_tok, const int32_t* out_cnt,
                           int32_t* block) {
  if (!b || !block || n < 0 || n > b->cap || (n > 0 && (!ids || !out_tok || !out_cnt))) return SEED_EINVAL;
  const int stride = b->gamma + 3;
  std::fill(block, block + b->block_ints(), -1);
  int64_t pending = b->undone - n;
  for (int i = 0; i < n; ++i) {
    auto it = b->own.find((uint32_t)ids[i]);
    if (it == b->own.end() || it->second.done) return SEED_EINVAL;
    // a5 (R7): commit at most the room left before l
    const int room = std::max(b->max_new - it->second.L, 0);
    const int c = std::min(out_cnt[i], room);
    int32_t* r = block + (size_t)i * stride;
    r[0] = ids[i];
    r[1] = c;
    for (int k = 0; k < c; ++k) r[2 + k] = out_tok[(size_t)i * (b->gamma + 1) + k];
    if (it->second.L + c < b->max_new) ++pending;
  }
  block[b->block_ints() - 1] = (int32_t)pending;
  return SEED_OK;
}

seed_status seed_book_complete(seed_book b, const int32_t* blocks, int32_t n_blocks) {
  if (!b || !blocks || n_blocks != b->world) return SEED_EINVAL;
  const int bi = b->block_ints();
  std::vector<int32_t> batch, done;
  seed_status s = book_complete_own(b, blocks + (size_t)b->rank * bi, batch, done);
  if (s != SEED_OK) return s;
  s = seed_sched_complete(&b->sched, batch.data(), done.data(), (int32_t)batch.size());
  if (s != SEED_OK) return s;
  int64_t pending = 0;
  for (int w = 0; w < n_blocks; ++w) {
    const int32_t* blk = blocks + (size_t)w * bi;
    if (w != b->rank) {
      s = seed_table_merge(&b->table, blk, b->cap);
      if (s != SEED_OK) return s;
    }
    if (blk[bi - 1] < 0) return SEED_EINVAL;
    pending += blk[bi - 1];
  }
  if (pending < b->undone) return SEED_EINVAL;   // the own tail must count the own undone streams
  b->global_pending = pending;
  return SEED_OK;
}

seed_status seed_book_global_pending(seed_book b, int64_t* n) {
  if (!b || !n) return SEED_EINVAL;
  *n = b->global_pending;
  return SEED_OK;
}

seed_status seed_book_tokens(seed_book b, uint32_t gid, int32_t* dst, int32_t cap, int32_t* len) {
  if (!b || !len) return SEED_EINVAL;
  auto it = b->own.find(gid);
  if (it != b->own.end()) {
    const seed::BookStream& st = it->second;
    *len = (int32_t)st.T.size() - st.prompt_len;
    if (dst) std::copy(st.T.begin() + st.prompt_len, st.T.begin() + st.prompt_len + std::min(cap, *len), dst);
    return SEED_OK;
  }
  return seed_table_get(&b->table, gid, dst, cap, len);
}

seed_status seed_book_info(seed_book b, uint32_t gid, int32_t* info) {
  if (!b || !info) return SEED_EINVAL;
  auto it = b->own.find(gid);
  if (it == b->own.end()) return SEED_ENOTFOUND;
  const seed::BookStream& st = it->second;
  info[0] = (int32_t)st.T.size();
  info[1] = st.L;
  info[2] = st.r;
  info[3] = st.done ? 1 : 0;
  info[4] = st.prompt_len;
  return SEED_OK;
}

int32_t seed_book_block_ints(seed_book b) { return b ? b->block_ints() : 0; }

void seed_book_destroy(seed_book b) { delete b; }

}  // extern "C"
