// stengrid/worker_pool.hpp — API-compatible stand-in for the reference's
// WorkerPool (worker_pool.hpp:1-47). On the B200 the parallel runtime is the
// GPU itself (streams, CUDA graphs, NCCL across devices); a WorkerPool only
// carries the worker count that create_plan / CHStepper validate
// (stencil.cpp:159-161). run() executes jobs inline on the caller, which is
// what the reference does for one worker (worker_pool.cpp:55-75).
#pragma once

#include <functional>
#include <stdexcept>

namespace stengrid {

class WorkerPool {
 public:
  explicit WorkerPool(int workers = 1) : workers_(workers) {
    if (workers < 1) throw std::invalid_argument("WorkerPool: workers must be >= 1");
  }
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  int workers() const { return workers_; }
  void run(int jobCount, const std::function<void(int, int)>& fn) {
    for (int j = 0; j < jobCount; ++j) fn(j, 0);
  }

 private:
  int workers_ = 1;
};

}  // namespace stengrid
