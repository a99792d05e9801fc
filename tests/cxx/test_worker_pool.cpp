// WorkerPool (include/stengrid/worker_pool.hpp): the reference's host thread
// pool API (worker_pool.hpp:1-47; its tests: test_grid.cpp:136-160,
// test_penta.cpp:306-316). Header-only, no GPU: built and run by
// tests/test_worker_pool_cpu.py.
#include <atomic>
#include <cstdio>
#include <set>
#include <stdexcept>
#include <vector>

#include "stengrid/worker_pool.hpp"

static int g_fail = 0;
#define CHECK(c)                                            \
  do {                                                      \
    if (!(c)) {                                             \
      ++g_fail;                                             \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                       \
  } while (0)

int main() {
  using stengrid::WorkerPool;
  bool threw = false;
  try {
    WorkerPool bad(0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  for (int workers : {1, 2, 3, 8}) {
    WorkerPool pool(workers);
    CHECK(pool.workers() == workers);
    for (int round = 0; round < 200; ++round) {  // many back-to-back batches
      const int jobs = 1 + (round * 37) % 500;
      std::vector<std::atomic<int>> hits(static_cast<size_t>(jobs));
      std::vector<int> slotOf(static_cast<size_t>(jobs), -1);
      pool.run(jobs, [&](int j, int slot) {
        hits[static_cast<size_t>(j)].fetch_add(1);
        slotOf[static_cast<size_t>(j)] = slot;
      });
      for (int j = 0; j < jobs; ++j) {
        CHECK(hits[static_cast<size_t>(j)].load() == 1);
        CHECK(slotOf[static_cast<size_t>(j)] >= 0 && slotOf[static_cast<size_t>(j)] < workers);
      }
    }
    pool.run(0, [&](int, int) { CHECK(false); });
    // exceptions reach the caller; the batch still completes
    std::atomic<int> ran{0};
    bool caught = false;
    try {
      pool.run(64, [&](int j, int) {
        ran.fetch_add(1);
        if (j == 7) throw std::runtime_error("job 7");
      });
    } catch (const std::runtime_error&) {
      caught = true;
    }
    CHECK(caught);
    CHECK(ran.load() == 64);
  }
  // several slots really run concurrently with more than one worker
  {
    WorkerPool pool(4);
    std::atomic<int> inside{0}, peak{0};
    pool.run(64, [&](int, int) {
      const int now = inside.fetch_add(1) + 1;
      int p = peak.load();
      while (now > p && !peak.compare_exchange_weak(p, now)) {
      }
      std::atomic<int> spin{0};
      while (spin.fetch_add(1, std::memory_order_relaxed) < 200000) {
      }
      inside.fetch_sub(1);
    });
    CHECK(peak.load() >= 2);
  }
  std::printf("%s\n", g_fail == 0 ? "worker pool OK" : "worker pool FAILED");
  return g_fail == 0 ? 0 : 1;
}
