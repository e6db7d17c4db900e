// host_sched.cpp -- H1: the FCFS rounds scheduler and the a6 token table (host only, no CUDA).
//
// Scheduler (Alg. 1; lock-step batched reading R9):
//   queue Q of global ids, FCFS; ready flag per stream (the paper's draft label
//   map): 0 after drafting, 1 after verification; undone streams re-enter
//   at the tail in batch order -- the "rounds" of P:206 / P:230; ties at admission -> lowest
//   id (R10); a done stream met in the queue is dropped; an empty pop while work
//   remains is a liveness violation reported as SEED_ESTATE.
#include <algorithm>
#include <deque>
#include <new>
#include <unordered_map>
#include <vector>

#include "../../include/seed.h"

struct seed_sched_s {
  std::deque<int32_t> queue;
  std::unordered_map<int32_t, int> ready, done;
};

struct seed_table_s {
  int32_t stride;
  std::unordered_map<uint32_t, std::vector<int32_t>> tokens;
};

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

void seed_table_destroy(seed_table t) { delete t; }

}  // extern "C"
