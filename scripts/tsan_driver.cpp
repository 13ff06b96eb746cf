// Host-runtime race check (SURVEY.md §5 "race detection"): a ThreadSanitizer build of libsurge driven
// by the documented threading model -- ONE producer thread submits partitions and finishes, while a
// second thread polls and releases pieces concurrently (include/surge.h "Threading") -- on the toy
// encoder (C1 shapes, random bf16 weights).  Every partition must come back exactly once.
//   built and run by scripts/sanitize.sh (g++ -fsanitize=thread, libsurge built with TSAN).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <thread>
#include <vector>

#include "../include/surge.h"

int main() {
  surge_config cfg{};
  cfg.vocab_size = 1024; cfg.max_position = 64; cfg.type_vocab_size = 2;
  cfg.hidden = 64; cfg.layers = 2; cfg.heads = 4; cfg.ffn = 256; cfg.ln_eps = 1e-12f;
  cfg.b_min = 64; cfg.b_max = 96; cfg.world_size = 1; cfg.max_inflight = 2;
  const size_t d = 64, f = 256, L = 2;
  const size_t n_w = (1024 + 64 + 2) * d + 2 * d + L * (4 * (d * d + d) + 2 * d + (f * d + f) + (d * f + d) + 2 * d);
  std::vector<uint16_t> w(n_w);
  std::mt19937 rng(1);
  for (auto& x : w) x = uint16_t(0x3c00 + (rng() % 512) - 256);   // bf16 values near +-0.01
  for (int policy = SURGE_BMAX_LABEL; policy <= SURGE_BMAX_PREFLUSH; ++policy) {
    cfg.bmax_policy = policy;
    surge_handle h = nullptr;
    if (surge_create(&cfg, w.data(), n_w, &h) != SURGE_OK) { std::fprintf(stderr, "create failed\n"); return 2; }
    std::atomic<bool> done{false};
    std::map<uint64_t, int64_t> rows;
    std::thread poller([&] {
      surge_flushed buf[64];
      for (;;) {
        int64_t n = 0;
        if (surge_poll_flushed(h, buf, 64, 5, &n) != SURGE_OK) std::abort();
        for (int64_t i = 0; i < n; ++i) {
          rows[buf[i].partition_id] += buf[i].n_rows;
          surge_release(h, &buf[i]);
        }
        surge_stats st;
        surge_get_stats(h, &st);                 // stats from the non-producer thread
        int64_t pend = 0;
        surge_pending(h, &pend);
        if (n == 0 && done.load() && pend == 0) break;
      }
    });
    std::map<uint64_t, int64_t> want;
    for (uint64_t k = 0; k < 60; ++k) {
      const int64_t n = int64_t(rng() % 200);
      std::vector<int32_t> lens(static_cast<size_t>(n));
      std::vector<int32_t> ids;
      for (auto& l : lens) {
        l = 1 + int32_t(rng() % 32);
        for (int32_t t = 0; t < l; ++t) ids.push_back(int32_t(4 + rng() % 1000));
      }
      want[k] = n;
      if (surge_submit_partition(h, k, ids.data(), lens.data(), n) != SURGE_OK) { std::fprintf(stderr, "submit\n"); return 3; }
    }
    surge_finish(h);
    done = true;
    poller.join();
    surge_destroy(h);
    for (auto& kv : want)
      if (rows[kv.first] != kv.second) { std::fprintf(stderr, "partition %lu: %ld rows, want %ld\n",
                                                      (unsigned long)kv.first, (long)rows[kv.first], (long)kv.second); return 4; }
    std::printf("tsan driver: policy %d ok, %zu partitions\n", policy, want.size());
  }
  return 0;
}
