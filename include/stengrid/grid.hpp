// stengrid/grid.hpp — drop-in replacement for the reference's grid core
// (/root/reference/proj/include/stengrid/grid.hpp:1-102) on top of the
// B200 C ABI (stengrid/sg.h). Same names, signatures and exceptions.
//
// Storage: the reference uses an Eigen row-major array purely as storage
// (SURVEY.md §8(c)). When <Eigen/Core> is on the include path (or
// STENGRID_USE_EIGEN is defined) `Array2d` / `ArrayXd` ARE the reference's
// Eigen types, so caller code that applies Eigen expressions to
// `Grid2D::values` compiles unchanged; otherwise (this image has no Eigen;
// STENGRID_NO_EIGEN forces it) they are dense row-major containers with the
// members the reference API and its tests use (setZero, setConstant,
// operator()(row, col), data, size, rows, cols, transpose, swap). The library
// itself only exchanges raw pointers (data()) with the C ABI, so both
// storages bind the same libstengrid_b200.so.
#pragma once

#include <algorithm>
#include <atomic>
#include <cassert>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "stengrid/errors.hpp"
#include "stengrid/sg.h"

#if !defined(STENGRID_NO_EIGEN) && (defined(STENGRID_USE_EIGEN) || __has_include(<Eigen/Core>))
#include <Eigen/Core>
#define STENGRID_EIGEN_STORAGE 1
#endif

namespace stengrid {

namespace detail {
inline std::atomic<std::int64_t>& large_alloc_counter() {
  static std::atomic<std::int64_t> c{0};
  return c;
}
/// Count of grid-sized host buffer allocations (grid.hpp:15-20).
inline std::int64_t large_alloc_count() noexcept { return large_alloc_counter().load(); }
inline void note_large_alloc() noexcept { large_alloc_counter().fetch_add(1, std::memory_order_relaxed); }
}  // namespace detail

#ifdef STENGRID_EIGEN_STORAGE
/// The reference's storage types (grid.hpp:13, penta.hpp).
template <typename T>
using DenseArray2 = Eigen::Array<T, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
template <typename T>
using DenseVector = Eigen::Array<T, Eigen::Dynamic, 1>;
#else
/// Dense row-major 2D array of T (the subset of Eigen::Array the reference uses).
template <typename T>
class DenseArray2 {
 public:
  DenseArray2() = default;
  DenseArray2(std::ptrdiff_t r, std::ptrdiff_t c) { setZero(r, c); }

  std::ptrdiff_t rows() const { return rows_; }
  std::ptrdiff_t cols() const { return cols_; }
  std::ptrdiff_t size() const { return static_cast<std::ptrdiff_t>(v_.size()); }
  T* data() { return v_.empty() ? nullptr : v_.data(); }
  const T* data() const { return v_.empty() ? nullptr : v_.data(); }
  T& operator()(std::ptrdiff_t r, std::ptrdiff_t c) { return v_[static_cast<std::size_t>(r * cols_ + c)]; }
  const T& operator()(std::ptrdiff_t r, std::ptrdiff_t c) const {
    return v_[static_cast<std::size_t>(r * cols_ + c)];
  }
  T& operator[](std::ptrdiff_t k) { return v_[static_cast<std::size_t>(k)]; }
  const T& operator[](std::ptrdiff_t k) const { return v_[static_cast<std::size_t>(k)]; }

  void setZero(std::ptrdiff_t r, std::ptrdiff_t c) {
    rows_ = r;
    cols_ = c;
    v_.assign(static_cast<std::size_t>(r * c), T{});
  }
  void setZero() { std::fill(v_.begin(), v_.end(), T{}); }
  void setConstant(const T& x) { std::fill(v_.begin(), v_.end(), x); }
  DenseArray2 transpose() const {
    DenseArray2 t(cols_, rows_);
    for (std::ptrdiff_t r = 0; r < rows_; ++r)
      for (std::ptrdiff_t c = 0; c < cols_; ++c) t(c, r) = (*this)(r, c);
    return t;
  }
  void swap(DenseArray2& o) noexcept {
    v_.swap(o.v_);
    std::swap(rows_, o.rows_);
    std::swap(cols_, o.cols_);
  }

 private:
  std::ptrdiff_t rows_ = 0, cols_ = 0;
  std::vector<T> v_;
};

/// Dense vector of T (the subset of Eigen::ArrayXd the reference uses).
template <typename T>
class DenseVector {
 public:
  DenseVector() = default;
  explicit DenseVector(std::ptrdiff_t n) : v_(static_cast<std::size_t>(n)) {}
  std::ptrdiff_t size() const { return static_cast<std::ptrdiff_t>(v_.size()); }
  T* data() { return v_.empty() ? nullptr : v_.data(); }
  const T* data() const { return v_.empty() ? nullptr : v_.data(); }
  T& operator[](std::ptrdiff_t k) { return v_[static_cast<std::size_t>(k)]; }
  const T& operator[](std::ptrdiff_t k) const { return v_[static_cast<std::size_t>(k)]; }
  T& operator()(std::ptrdiff_t k) { return v_[static_cast<std::size_t>(k)]; }
  const T& operator()(std::ptrdiff_t k) const { return v_[static_cast<std::size_t>(k)]; }
  void setZero(std::ptrdiff_t n) { v_.assign(static_cast<std::size_t>(n), T{}); }
  void setZero() { std::fill(v_.begin(), v_.end(), T{}); }
  void setConstant(const T& x) { std::fill(v_.begin(), v_.end(), x); }

 private:
  std::vector<T> v_;
};

#endif  // STENGRID_EIGEN_STORAGE

/// Row-major storage backing every field: entry (j, i) at j*nx + i.
using Array2d = DenseArray2<double>;
using ArrayXd = DenseVector<double>;

/// grid.hpp:25-49 — a uniform 2D field; (i, j) at values(j, i). The
/// reference stores doubles only (grid.hpp:13); BasicGrid2D<float> (Grid2Df)
/// is this library's FP32 extension (north_star: FP32+FP64 stencils), accepted
/// by create_plan / compute / swap_plan like Grid2D.
template <typename T>
struct BasicGrid2D {
  using value_type = T;
  int nx = 0;
  int ny = 0;
  double dx = 1.0;
  double dy = 1.0;
  DenseArray2<T> values;

  BasicGrid2D() = default;
  BasicGrid2D(int nx_, int ny_, double dx_, double dy_) : nx(nx_), ny(ny_), dx(dx_), dy(dy_) {
    if (nx < 1 || ny < 1) throw std::invalid_argument("Grid2D: nx and ny must be >= 1");
    if (!(dx > 0.0) || !(dy > 0.0)) throw std::invalid_argument("Grid2D: dx and dy must be > 0");
    values.setZero(ny, nx);
    detail::note_large_alloc();
  }
  BasicGrid2D(const BasicGrid2D& o) : nx(o.nx), ny(o.ny), dx(o.dx), dy(o.dy), values(o.values) {
    if (values.size() > 0) detail::note_large_alloc();
  }
  BasicGrid2D& operator=(const BasicGrid2D& o) {
    if (this == &o) return *this;
    if (values.size() != o.values.size() && o.values.size() > 0) detail::note_large_alloc();
    nx = o.nx;
    ny = o.ny;
    dx = o.dx;
    dy = o.dy;
    values = o.values;
    return *this;
  }
  BasicGrid2D(BasicGrid2D&&) noexcept = default;
  BasicGrid2D& operator=(BasicGrid2D&&) noexcept = default;

  T operator()(int i, int j) const { return values(j, i); }
  T& operator()(int i, int j) { return values(j, i); }
  const T* data() const { return values.data(); }
  T* data() { return values.data(); }
  std::ptrdiff_t size() const { return static_cast<std::ptrdiff_t>(nx) * ny; }
  bool same_shape(const BasicGrid2D& o) const { return nx == o.nx && ny == o.ny; }
};

using Grid2D = BasicGrid2D<double>;
using Grid2Df = BasicGrid2D<float>;

/// grid.hpp:53-62
struct Extents {
  int left = 0;
  int right = 0;
  int top = 0;
  int bottom = 0;
  int width() const { return left + right + 1; }
  int height() const { return top + bottom + 1; }
  bool valid() const { return left >= 0 && right >= 0 && top >= 0 && bottom >= 0; }
};

enum class BoundaryMode { Periodic, NonPeriodic };

struct TileRange {
  int jBegin = 0;
  int jEnd = 0;
};

/// grid.hpp:67-81 — on the B200 the tiles are the y-slab decomposition.
struct TilePlan {
  std::vector<TileRange> tiles;
  int haloTop = 0;
  int haloBottom = 0;
  int num_tiles() const { return static_cast<int>(tiles.size()); }
};

inline std::ptrdiff_t linear_index(int i, int j, int nx) {
  assert(nx >= 1 && i >= 0 && i < nx && j >= 0);
  return static_cast<std::ptrdiff_t>(j) * nx + i;
}

/// grid.cpp:42-47 (through sg_wrap).
inline int wrap(std::int64_t i, int n) {
  int out = 0;
  detail::check(sg_wrap(i, n, &out));
  return out;
}

/// grid.cpp:55-60 — exact transposed copy.
inline void transpose_into(const Grid2D& g, Grid2D& out) {
  if (&out == &g) throw std::invalid_argument("transpose_into: output must not alias the input");
  if (out.nx != g.ny || out.ny != g.nx)
    throw std::invalid_argument("transpose_into: output shape must be the transposed input shape");
  out.values = g.values.transpose();
}

inline Grid2D transpose(const Grid2D& g) {
  Grid2D out(g.ny, g.nx, g.dy, g.dx);
  transpose_into(g, out);
  return out;
}

/// grid.cpp:62-82 (through sg_make_tiles).
inline TilePlan make_tiles(int ny, int numTiles, const Extents& ext) {
  if (!ext.valid()) throw std::invalid_argument("make_tiles: negative extents");
  TilePlan plan;
  plan.haloTop = ext.top;
  plan.haloBottom = ext.bottom;
  if (ny >= 1 && numTiles >= 1 && numTiles <= ny) {
    std::vector<int> b(static_cast<std::size_t>(numTiles)), e(static_cast<std::size_t>(numTiles));
    detail::check(sg_make_tiles(ny, numTiles, b.data(), e.data()));
    for (int t = 0; t < numTiles; ++t) plan.tiles.push_back(TileRange{b[t], e[t]});
  } else {
    detail::check(sg_make_tiles(ny, numTiles, nullptr, nullptr));
  }
  return plan;
}

}  // namespace stengrid
