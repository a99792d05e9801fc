// stengrid/penta.hpp — drop-in replacement for the reference batched
// pentadiagonal API (/root/reference/proj/include/stengrid/penta.hpp:1-125).
// Factorization and solves run on the GPU (one system per thread, sm_100a,
// csrc/penta.cu) with the reference's arithmetic: solutions are bitwise
// identical. Errors: std::invalid_argument, PentaSolveError{system}.
#pragma once

#include <cstring>
#include <utility>

#include "stengrid/grid.hpp"
#include "stengrid/worker_pool.hpp"

namespace stengrid {

namespace detail {
inline void penta_check_shapes(int batchCount, int n) {  // penta.cpp:10-13
  if (batchCount < 1) throw std::invalid_argument("penta: batchCount must be >= 1");
  if (n < 5) throw std::invalid_argument("penta: systems need n >= 5");
}
}  // namespace detail

/// penta.hpp:12-33 — interleaved bands, idx(b, r) = r*batchCount + b.
struct PentaBatch {
  int batchCount = 0;
  int n = 0;
  bool periodic = false;
  ArrayXd secondSub, sub, diag, super, secondSuper;

  PentaBatch() = default;
  PentaBatch(int batchCount_, int n_, bool periodic_) : batchCount(batchCount_), n(n_), periodic(periodic_) {
    detail::penta_check_shapes(batchCount, n);
    const std::ptrdiff_t len = static_cast<std::ptrdiff_t>(batchCount) * n;
    secondSub.setZero(len);
    sub.setZero(len);
    diag.setZero(len);
    super.setZero(len);
    secondSuper.setZero(len);
    detail::note_large_alloc();
  }
  std::ptrdiff_t idx(int b, int r) const { return static_cast<std::ptrdiff_t>(r) * batchCount + b; }
};

/// penta.hpp:36-49
struct RhsBatch {
  int batchCount = 0;
  int n = 0;
  ArrayXd values;

  RhsBatch() = default;
  RhsBatch(int batchCount_, int n_) : batchCount(batchCount_), n(n_) {
    if (batchCount < 1 || n < 1) throw std::invalid_argument("RhsBatch: batchCount and n must be >= 1");
    values.setZero(static_cast<std::ptrdiff_t>(batchCount) * n);
    detail::note_large_alloc();
  }
  std::ptrdiff_t idx(int b, int r) const { return static_cast<std::ptrdiff_t>(r) * batchCount + b; }
  double at(int b, int r) const { return values[idx(b, r)]; }
  double& at(int b, int r) { return values[idx(b, r)]; }
};

namespace detail {
class DevicePentaFactor {
 public:
  DevicePentaFactor(const PentaBatch& m, bool periodic) : B_(m.batchCount), n_(m.n) {
    penta_check_shapes(B_, n_);
    check(sg_penta_create(B_, n_, periodic ? 1 : 0, m.secondSub.data(), m.sub.data(), m.diag.data(),
                          m.super.data(), m.secondSuper.data(), SG_MEM_HOST, &h_));
  }
  DevicePentaFactor(DevicePentaFactor&& o) noexcept : h_(o.h_), B_(o.B_), n_(o.n_) { o.h_ = nullptr; }
  DevicePentaFactor& operator=(DevicePentaFactor&& o) noexcept {
    std::swap(h_, o.h_);
    B_ = o.B_;
    n_ = o.n_;
    return *this;
  }
  DevicePentaFactor(const DevicePentaFactor&) = delete;
  DevicePentaFactor& operator=(const DevicePentaFactor&) = delete;
  ~DevicePentaFactor() {
    if (h_) sg_penta_destroy(&h_);
  }
  int batch_count() const { return B_; }
  int size() const { return n_; }
  void solve(RhsBatch& rhs, const char* who) const {
    if (rhs.batchCount != B_ || rhs.n != n_)
      throw std::invalid_argument(std::string(who) + ": rhs shape does not match the operator");
    check(sg_penta_solve(h_, rhs.values.data(), SG_MEM_HOST, nullptr, 1));
  }

 private:
  sg_penta_t h_ = nullptr;
  int B_ = 0, n_ = 0;
};
}  // namespace detail

/// penta.hpp:57-77 — non-pivoting LU, factored on the device.
class PentaFactor {
 public:
  explicit PentaFactor(const PentaBatch& m) : f_(m, false) {}
  int batch_count() const { return f_.batch_count(); }
  int size() const { return f_.size(); }
  void solve_in_place(RhsBatch& rhs, WorkerPool* pool = nullptr) const {
    (void)pool;
    f_.solve(rhs, "PentaFactor::solve_in_place");
  }

 private:
  detail::DevicePentaFactor f_;
};

/// penta.hpp:79-100 — Woodbury corner correction on the device.
class PeriodicPentaFactor {
 public:
  explicit PeriodicPentaFactor(const PentaBatch& m) : f_(m, true) {}
  int batch_count() const { return f_.batch_count(); }
  int size() const { return f_.size(); }
  void solve_in_place(RhsBatch& rhs, WorkerPool* pool = nullptr) const {
    (void)pool;
    f_.solve(rhs, "PeriodicPentaFactor::solve_in_place");
  }

 private:
  detail::DevicePentaFactor f_;
};

/// penta.cpp:297-303
inline RhsBatch solve_batch(const PentaBatch& m, RhsBatch rhs, WorkerPool* pool = nullptr) {
  if (m.periodic) throw std::invalid_argument("solve_batch: operator is periodic");
  if (rhs.batchCount != m.batchCount || rhs.n != m.n)
    throw std::invalid_argument("solve_batch: rhs shape does not match the operator");
  const PentaFactor f(m);
  f.solve_in_place(rhs, pool);
  return rhs;
}

/// penta.cpp:305-311
inline RhsBatch solve_periodic_batch(const PentaBatch& m, RhsBatch rhs, WorkerPool* pool = nullptr) {
  if (!m.periodic) throw std::invalid_argument("solve_periodic_batch: operator is not periodic");
  if (rhs.batchCount != m.batchCount || rhs.n != m.n)
    throw std::invalid_argument("solve_periodic_batch: rhs shape does not match the operator");
  const PeriodicPentaFactor f(m);
  f.solve_in_place(rhs, pool);
  return rhs;
}

/// penta.cpp:313-335 — rows {s, -4s, 1+6s, -4s, s}, cyclic iff periodic.
inline PentaBatch build_hyperdiffusion_operator(double sigma, int n, int batchCount, bool periodic) {
  if (!(sigma >= 0.0)) throw std::invalid_argument("build_hyperdiffusion_operator: sigma must be >= 0");
  PentaBatch m(batchCount, n, periodic);
  const double second = sigma, first = -4.0 * sigma, center = 1.0 + 6.0 * sigma;
  m.secondSub.setConstant(second);
  m.sub.setConstant(first);
  m.diag.setConstant(center);
  m.super.setConstant(first);
  m.secondSuper.setConstant(second);
  if (!periodic) {
    for (int b = 0; b < batchCount; ++b) {
      m.secondSub[m.idx(b, 0)] = 0.0;
      m.secondSub[m.idx(b, 1)] = 0.0;
      m.sub[m.idx(b, 0)] = 0.0;
      m.super[m.idx(b, n - 1)] = 0.0;
      m.secondSuper[m.idx(b, n - 2)] = 0.0;
      m.secondSuper[m.idx(b, n - 1)] = 0.0;
    }
  }
  return m;
}

enum class Axis { X, Y };

/// penta.cpp:343-360 (layout move)
inline void interleave_into(const Grid2D& g, Axis axis, RhsBatch& out) {
  const int batchCount = axis == Axis::X ? g.ny : g.nx;
  const int n = axis == Axis::X ? g.nx : g.ny;
  if (out.batchCount != batchCount || out.n != n)
    throw std::invalid_argument("interleave_into: batch shape does not match the grid");
  const double* v = g.data();
  double* o = out.values.data();
  if (axis == Axis::X) {
    for (int j = 0; j < g.ny; ++j)
      for (int i = 0; i < g.nx; ++i) o[static_cast<std::ptrdiff_t>(i) * g.ny + j] = v[static_cast<std::ptrdiff_t>(j) * g.nx + i];
  } else {
    std::memcpy(o, v, sizeof(double) * static_cast<std::size_t>(g.size()));
  }
}

inline RhsBatch interleave(const Grid2D& g, Axis axis) {
  RhsBatch out(axis == Axis::X ? g.ny : g.nx, axis == Axis::X ? g.nx : g.ny);
  interleave_into(g, axis, out);
  return out;
}

/// penta.cpp:369-384 (layout move)
inline void deinterleave_into(const RhsBatch& rhs, Axis axis, Grid2D& out) {
  const int nx = axis == Axis::X ? rhs.n : rhs.batchCount;
  const int ny = axis == Axis::X ? rhs.batchCount : rhs.n;
  if (out.nx != nx || out.ny != ny)
    throw std::invalid_argument("deinterleave_into: grid shape does not match the batch");
  const double* v = rhs.values.data();
  double* o = out.data();
  if (axis == Axis::X) {
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) o[static_cast<std::ptrdiff_t>(j) * nx + i] = v[static_cast<std::ptrdiff_t>(i) * ny + j];
  } else {
    std::memcpy(o, v, sizeof(double) * static_cast<std::size_t>(out.size()));
  }
}

inline Grid2D deinterleave(const RhsBatch& rhs, Axis axis, double dx, double dy) {
  Grid2D g(axis == Axis::X ? rhs.n : rhs.batchCount, axis == Axis::X ? rhs.batchCount : rhs.n, dx, dy);
  deinterleave_into(rhs, axis, g);
  return g;
}

}  // namespace stengrid
