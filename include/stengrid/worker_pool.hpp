// stengrid/worker_pool.hpp — the reference's WorkerPool API
// (worker_pool.hpp:1-47): a fixed set of host threads running batches of
// indexed jobs, the caller taking part as slot 0.
//
// On the B200 the stencil, penta and CH paths do not need it: their
// parallelism is the GPU (kernels, streams, CUDA graphs) and numWorkers maps
// to the GPU count; create_plan / CHStepper only check the pool's size like
// the reference (stencil.cpp:159-161). It remains a working host thread pool
// for user code written against the reference API.
//
// Semantics: run(jobCount, fn) calls fn(job, slot) once for every job in
// [0, jobCount), slot in [0, workers()), and returns when all have finished;
// jobs are claimed through an atomic counter, so which slot runs which job
// varies while results written per job do not. One worker (or one job) runs
// inline. Extension: an exception thrown by a job is rethrown by run() (the
// first one; the batch still completes) instead of terminating the process.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

namespace stengrid {

class WorkerPool {
 public:
  explicit WorkerPool(int workers = 1) : workers_(workers) {
    if (workers < 1) throw std::invalid_argument("WorkerPool: workers must be >= 1");
    for (int slot = 1; slot < workers; ++slot) threads_.emplace_back([this, slot] { serve(slot); });
  }
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    wake_.notify_all();
    for (auto& t : threads_) t.join();
  }

  int workers() const { return workers_; }

  void run(int jobCount, const std::function<void(int, int)>& fn) {
    if (jobCount <= 0) return;
    if (workers_ == 1 || jobCount == 1) {
      std::exception_ptr err;
      for (int j = 0; j < jobCount; ++j) {
        try {
          fn(j, 0);
        } catch (...) {
          if (!err) err = std::current_exception();
        }
      }
      if (err) std::rethrow_exception(err);
      return;
    }
    auto b = std::make_shared<Batch>(&fn, jobCount, workers_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      batch_ = b;
      ++epoch_;
    }
    wake_.notify_all();
    b->work(0);
    // every thread checks in once per batch (so none can miss the next one)
    std::unique_lock<std::mutex> lk(b->m);
    b->cv.wait(lk, [&] { return b->pending == 0; });
    if (b->error) std::rethrow_exception(b->error);
  }

 private:
  struct Batch {
    const std::function<void(int, int)>* fn;
    int count;
    std::atomic<int> next{0};
    int pending;  // participants that have not finished (guarded by m)
    std::exception_ptr error;
    std::mutex m;
    std::condition_variable cv;
    Batch(const std::function<void(int, int)>* f, int c, int participants) : fn(f), count(c), pending(participants) {}
    void work(int slot) {
      std::exception_ptr err;
      for (int j = next.fetch_add(1); j < count; j = next.fetch_add(1)) {
        try {
          (*fn)(j, slot);
        } catch (...) {
          if (!err) err = std::current_exception();
        }
      }
      std::lock_guard<std::mutex> lk(m);
      if (err && !error) error = err;
      if (--pending == 0) cv.notify_all();
    }
  };

  void serve(int slot) {
    std::uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Batch> b;
      {
        std::unique_lock<std::mutex> lk(mu_);
        wake_.wait(lk, [&] { return quit_ || epoch_ != seen; });
        if (quit_) return;
        seen = epoch_;
        b = batch_;
      }
      b->work(slot);
    }
  }

  int workers_ = 1;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable wake_;
  std::shared_ptr<Batch> batch_;
  std::uint64_t epoch_ = 0;
  bool quit_ = false;
};

}  // namespace stengrid
