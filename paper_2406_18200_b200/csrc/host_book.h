// host_book.h -- internal C++ view of the host-only round bookkeeping of one rank (H1 + a6),
// shared by host_sched.cpp (which implements it and the seed_book_* C ABI) and engine.cu (which
// drives it every round).  No CUDA here: the same code runs in the CPU tests.
#pragma once
#include <stdint.h>

#include <deque>
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

namespace seed {

struct BookStream {            // validated state of one of this rank's streams (Alg. 1)
  std::vector<int32_t> T;      // prompt + validated new tokens
  int prompt_len = 0;
  int L = 0;                   // new tokens (R7: from 0, done at l)
  int r = 0;                   // stream-local round counter (R5)
  bool done = false;
};

}  // namespace seed

struct seed_book_s {
  int32_t gamma, max_new, cap, world, rank;
  seed_sched_s sched;
  seed_table_s table;
  std::unordered_map<uint32_t, seed::BookStream> own;
  int64_t undone = 0;            // own streams not done
  int64_t global_pending = -1;   // sum over ranks of undone streams after the last exchange (-1: none yet)
  int32_t block_ints() const { return cap * (gamma + 3) + 1; }
};
