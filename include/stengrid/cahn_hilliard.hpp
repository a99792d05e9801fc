// stengrid/cahn_hilliard.hpp — drop-in replacement for the reference
// Cahn-Hilliard BDF2-ADI API (/root/reference/proj/include/stengrid/
// cahn_hilliard.hpp:1-151). CHStepper keeps both time levels in HBM and runs
// step() as one CUDA-graph replay of five sm_100a kernels (csrc/ch.cu);
// field() / previous_field() download on demand. Results are bitwise
// identical to the reference CHStepper.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <numbers>
#include <vector>

#include "stengrid/grid.hpp"
#include "stengrid/penta.hpp"
#include "stengrid/stencil.hpp"
#include "stengrid/worker_pool.hpp"

namespace stengrid {

/// cahn_hilliard.hpp:23-39 (same defaults).
struct CHParams {
  double D = 1.0;
  double gamma = 0.01;
  int nx = 512;
  int ny = 512;
  double lx = 2.0 * std::numbers::pi;
  double ly = 2.0 * std::numbers::pi;
  double dt = 0.0;
  double T = 0.0;
  std::uint64_t seed = 1;
  double icAmplitude = 0.1;
  bool nonlinearEnabled = true;

  double dx() const { return lx / nx; }
  double dy() const { return ly / ny; }
  sg_ch_params c() const {
    return sg_ch_params{D, gamma, lx, ly, dt, T, icAmplitude, nx, ny, seed, nonlinearEnabled ? 1 : 0};
  }
  /// cahn_hilliard.cpp:56-66
  void validate() const {
    const sg_ch_params p = c();
    detail::check(sg_ch_validate(&p));
  }
};

struct Diagnostics {
  double t = 0.0;
  double s = 0.0;
  double k1Inv = 0.0;
};

/// cahn_hilliard.hpp:47-63 — the reproducible seed-to-field generator.
struct SplitMix64 {
  std::uint64_t state;
  explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

/// cahn_hilliard.cpp:68-76
inline Grid2D initial_condition(const CHParams& params) {
  Grid2D g(params.nx, params.ny, params.dx(), params.dy());
  SplitMix64 rng(params.seed);
  double* v = g.data();
  const double amp = params.icAmplitude;
  for (std::ptrdiff_t k = 0; k < g.size(); ++k) v[k] = amp * (2.0 * rng.next_unit() - 1.0);
  return g;
}

/// cahn_hilliard.cpp:78-83
inline std::vector<double> nonlinear_laplacian_coefficients(double dx, double dy) {
  const double cx = 1.0 / (dx * dx);
  const double cy = 1.0 / (dy * dy);
  const double cc = -2.0 * cx - 2.0 * cy;
  return {0.0, cy, 0.0, cx, cc, cx, 0.0, cy, 0.0};
}

/// cahn_hilliard.cpp:85-114
inline std::vector<double> biharmonic_weights(double dx, double dy) {
  auto pow4 = [](double h) {
    const double h2 = h * h;
    return h2 * h2;
  };
  const double ax = 1.0 / pow4(dx);
  const double ay = 1.0 / pow4(dy);
  const double cr = 2.0 / ((dx * dx) * (dy * dy));
  std::vector<double> w(25, 0.0);
  auto at = [&w](int p, int q) -> double& { return w[static_cast<std::size_t>(q) * 5 + p]; };
  at(0, 2) += ax;
  at(1, 2) += -4.0 * ax;
  at(2, 2) += 6.0 * ax;
  at(3, 2) += -4.0 * ax;
  at(4, 2) += ax;
  at(2, 0) += ay;
  at(2, 1) += -4.0 * ay;
  at(2, 2) += 6.0 * ay;
  at(2, 3) += -4.0 * ay;
  at(2, 4) += ay;
  static constexpr double cross[9] = {1.0, -2.0, 1.0, -2.0, 4.0, -2.0, 1.0, -2.0, 1.0};
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) at(p + 1, q + 1) += cross[q * 3 + p] * cr;
  double prefix = 0.0;
  for (int k = 0; k < 22; ++k) prefix += w[static_cast<std::size_t>(k)];
  at(2, 4) = -prefix;
  return w;
}

/// cahn_hilliard.cpp:116-125 — device 3x3 function stencil.
inline Grid2D nonlinear_term(const Grid2D& c) {
  Grid2D out(c.nx, c.ny, c.dx, c.dy);
  FunctionStencil fs{Extents{1, 1, 1, 1}, &functions::ch_nonlinear_window,
                     nonlinear_laplacian_coefficients(c.dx, c.dy)};
  StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, fs, const_cast<Grid2D&>(c), out, 1, 1);
  compute(plan);
  return out;
}

/// cahn_hilliard.cpp:127-135 — device 5x5 weight stencil.
inline Grid2D biharmonic(const Grid2D& c) {
  if (c.nx < 5 || c.ny < 5) throw std::invalid_argument("biharmonic: need nx, ny >= 5");
  Grid2D out(c.nx, c.ny, c.dx, c.dy);
  WeightStencil ws{Extents{2, 2, 2, 2}, biharmonic_weights(c.dx, c.dy)};
  StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, ws, const_cast<Grid2D&>(c), out, 1, 1);
  compute(plan);
  return out;
}

/// cahn_hilliard.cpp:161-177 — composite Simpson mean, on the device
/// (bitwise identical to the reference).
inline double simpson_mean(const Grid2D& g) {
  double out = 0.0;
  detail::check(sg_simpson_mean(g.data(), g.nx, g.ny, 0, SG_MEM_HOST, &out));
  return out;
}

/// cahn_hilliard.cpp:179-188 — s = 1/(1 - <C^2>); std::domain_error at saturation.
inline double s_metric(const Grid2D& c) {
  double out = 0.0;
  detail::check(sg_s_metric(c.data(), c.nx, c.ny, SG_MEM_HOST, &out));
  return out;
}

/// cahn_hilliard.cpp:190-211 — spectral mean wavenumber (cuFFT on the
/// device); std::domain_error on an all-zero field.
inline double k1_metric(const Grid2D& c) {
  double out = 0.0;
  detail::check(sg_k1_metric(c.data(), c.nx, c.ny, c.dx, c.dy, SG_MEM_HOST, &out));
  return out;
}

/// cahn_hilliard.hpp:104-137 — BDF2-ADI stepper, state in HBM.
class CHStepper {
 public:
  CHStepper(const CHParams& params, int numTiles = 1, int numWorkers = 1)
      : params_(params),
        cCurr_(params.nx >= 1 ? params.nx : 1, params.ny >= 1 ? params.ny : 1, params.dx() > 0 ? params.dx() : 1.0,
               params.dy() > 0 ? params.dy() : 1.0),
        cPrev_(cCurr_) {
    const sg_ch_params p = params.c();
    detail::check(sg_ch_create(&p, numTiles, numWorkers, &h_));
    dirty_ = true;
  }
  CHStepper(const CHStepper&) = delete;
  CHStepper& operator=(const CHStepper&) = delete;
  ~CHStepper() {
    if (h_) sg_ch_destroy(&h_);
  }

  /// cahn_hilliard.cpp:260-328
  void step() { steps(1); }
  /// `n` consecutive steps without host round trips.
  void steps(int n) {
    detail::check(sg_ch_step(h_, n));
    dirty_ = true;
  }
  /// Extension (sg.h: sg_ch_set_partition): partitioned x/y sweeps with
  /// `segments` segments per system — shorter recurrences, results NOT
  /// bitwise the reference's; 0 or 1 restores the bitwise default.
  void set_partition(int segments) { detail::check(sg_ch_set_partition(h_, segments)); }

  /// cahn_hilliard.cpp:251-258
  void set_state(const Grid2D& curr, const Grid2D& prev) {
    if (curr.nx != params_.nx || curr.ny != params_.ny || !curr.same_shape(prev))
      throw std::invalid_argument("CHStepper::set_state: shape mismatch");
    detail::check(sg_ch_set_state(h_, curr.data(), prev.data(), SG_MEM_HOST));
    dirty_ = true;
  }

  /// Restore the step counter (exact checkpoint resume; not in the reference).
  void set_step_index(int step) { detail::check(sg_ch_set_step(h_, step)); }

  int step_index() const {
    int s = 0;
    detail::check(sg_ch_status(h_, &s, nullptr));
    return s;
  }
  double time() const {
    double t = 0.0;
    detail::check(sg_ch_status(h_, nullptr, &t));
    return t;
  }
  const CHParams& params() const { return params_; }
  const Grid2D& field() const {
    refresh();
    return cCurr_;
  }
  const Grid2D& previous_field() const {
    refresh();
    return cPrev_;
  }
  /// cahn_hilliard.cpp:330-340 — computed on the device-resident C^n.
  Diagnostics diagnostics() const {
    Diagnostics d;
    detail::check(sg_ch_diagnostics(h_, &d.t, &d.s, &d.k1Inv));
    return d;
  }

  /// Device pointer of C^n (which = 0) or C^{n-1} (which = 1).
  const double* device_field(int which = 0) const {
    const double* p = nullptr;
    detail::check(sg_ch_device_field(h_, which, &p));
    return p;
  }

 private:
  void refresh() const {
    if (!dirty_) return;
    detail::check(sg_ch_get_field(h_, 0, cCurr_.data(), SG_MEM_HOST));
    detail::check(sg_ch_get_field(h_, 1, cPrev_.data(), SG_MEM_HOST));
    dirty_ = false;
  }

  CHParams params_;
  sg_ch_t h_ = nullptr;
  mutable Grid2D cCurr_, cPrev_;
  mutable bool dirty_ = true;
};

/// cahn_hilliard.hpp:141-146
struct RunSink {
  int diagEvery = 1;
  int snapEvery = 0;
  std::function<void(const Diagnostics&)> onDiagnostics;
  std::function<void(const Grid2D&, int step, double t)> onSnapshot;
};

/// cahn_hilliard.cpp:342-356 — steps between sink emissions run back to
/// back on the device (no host round trips).
inline void run(const CHParams& params, int numTiles, int numWorkers, const RunSink& sink) {
  CHStepper stepper(params, numTiles, numWorkers);
  const bool diag = sink.diagEvery > 0 && sink.onDiagnostics;
  const bool snap = sink.snapEvery > 0 && sink.onSnapshot;
  const auto emit = [&](long step) {
    if (diag && step % sink.diagEvery == 0) sink.onDiagnostics(stepper.diagnostics());
    if (snap && step % sink.snapEvery == 0) sink.onSnapshot(stepper.field(), static_cast<int>(step), stepper.time());
  };
  emit(0);
  const auto steps = static_cast<long>(std::ceil(params.T / params.dt - 1e-9));
  long s = 0;
  while (s < steps) {
    long next = steps;
    if (diag) next = std::min(next, (s / sink.diagEvery + 1) * sink.diagEvery);
    if (snap) next = std::min(next, (s / sink.snapEvery + 1) * sink.snapEvery);
    stepper.steps(static_cast<int>(next - s));
    s = next;
    emit(s);
  }
}

}  // namespace stengrid
