// C++ tests of the drop-in API (include/stengrid/*.hpp), written the way the
// reference's own doctest suites are (tests/test_stencil.cpp,
// tests/test_penta.cpp, tests/test_cahn_hilliard.cpp, tests/acceptance.cpp)
// — same calls, same assertions — but executed by the B200 engine.
// A user of the reference recompiles against these headers and links
// libstengrid_b200.so; nothing else changes. Run via tests/test_cxx_gpu.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "stengrid/cahn_hilliard.hpp"
#include "stengrid/penta.hpp"
#include "stengrid/snapshot.hpp"
#include "stengrid/stencil.hpp"
#include "stengrid/weno.hpp"

using namespace stengrid;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (cond) {                                                              \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, T)          \
  do {                                    \
    bool caught = false;                  \
    try {                                 \
      (void)(expr);                       \
    } catch (const T&) {                  \
      caught = true;                      \
    } catch (...) {                       \
    }                                     \
    CHECK(caught && #T);                  \
  } while (0)

namespace {

constexpr double kTwoPi = 2.0 * std::numbers::pi;

Grid2D random_grid(int nx, int ny, std::uint64_t seed, double lo = -1.0, double hi = 1.0) {
  Grid2D g(nx, ny, 0.1, 0.2);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (std::ptrdiff_t k = 0; k < g.size(); ++k) g.data()[k] = dist(rng);
  return g;
}

std::vector<double> random_weights(int count, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-2.0, 2.0);
  std::vector<double> w(static_cast<std::size_t>(count));
  for (double& x : w) x = dist(rng);
  return w;
}

double oracle_weights_at(const Grid2D& g, const Extents& e, const std::vector<double>& w, int i, int j,
                         bool periodic) {
  const int W = e.left + e.right + 1;
  double acc = 0.0;
  for (int q = 0; q < e.top + e.bottom + 1; ++q)
    for (int p = 0; p < W; ++p) {
      int ii = i - e.left + p, jj = j - e.top + q;
      if (periodic) {
        ii = ((ii % g.nx) + g.nx) % g.nx;
        jj = ((jj % g.ny) + g.ny) % g.ny;
      }
      acc += w[static_cast<std::size_t>(q) * W + p] * g.values(jj, ii);
    }
  return acc;
}

bool grids_equal_bitwise(const Grid2D& a, const Grid2D& b) {
  return a.same_shape(b) &&
         std::memcmp(a.data(), b.data(), sizeof(double) * static_cast<std::size_t>(a.size())) == 0;
}

Grid2D cyclic_shift(const Grid2D& g, int si, int sj) {
  Grid2D out(g.nx, g.ny, g.dx, g.dy);
  for (int j = 0; j < g.ny; ++j)
    for (int i = 0; i < g.nx; ++i) out(wrap(i + si, g.nx), wrap(j + sj, g.ny)) = g(i, j);
  return out;
}

double second_derivative_max_error(int n, const std::vector<double>& coeffs, int hw) {
  Grid2D in(n, 1, kTwoPi / n, 1.0);
  for (int i = 0; i < n; ++i) in(i, 0) = std::sin(i * in.dx);
  Grid2D out(n, 1, in.dx, in.dy);
  std::vector<double> w(coeffs.size());
  const double s = 1.0 / (in.dx * in.dx);
  for (std::size_t k = 0; k < w.size(); ++k) w[k] = coeffs[k] * s;
  StencilPlan plan =
      create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{hw, hw, 0, 0}, w}, in, out, 1, 1);
  compute(plan);
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = std::max(m, std::abs(out(i, 0) + std::sin(i * in.dx)));
  return m;
}

// ---------------------------------------------------------------- stencil

void test_create_plan_rejects_invalid_setups() {  // test_stencil.cpp:134-183
  Grid2D a(16, 8, 1.0, 1.0), b(16, 8, 1.0, 1.0), small(4, 8, 1.0, 1.0);
  const std::vector<double> w3 = {1.0, -2.0, 1.0};
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, w3}, a, a, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic,
                              WeightStencil{Extents{16, 0, 0, 0}, std::vector<double>(17, 1.0)}, a, b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, {}}, a, b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(
      create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, {1.0, 2.0}}, a, b, 1, 1),
      std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic,
                              WeightStencil{Extents{1, 1, 0, 0}, {1.0, NAN, 1.0}}, a, b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic,
                              WeightStencil{Extents{1, 1, 1, 0}, std::vector<double>(6, 1.0)}, a, b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::Y, BoundaryMode::Periodic,
                              WeightStencil{Extents{1, 0, 1, 1}, std::vector<double>(6, 1.0)}, a, b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, w3}, a, small, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic, FunctionStencil{Extents{1, 1, 0, 0}, nullptr, {}}, a,
                              b, 1, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, w3}, a, b, 9, 1),
                  std::invalid_argument);
}

void test_lifecycle() {  // test_stencil.cpp:185-209
  Grid2D in = random_grid(12, 7, 11);
  const Grid2D inCopy = in;
  Grid2D out(12, 7, in.dx, in.dy);
  const std::vector<double> w3 = {0.25, 0.5, 0.25};
  StencilPlan plan = create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, w3}, in, out, 2, 2);
  compute(plan);
  destroy_plan(plan);
  CHECK(!plan.valid());
  destroy_plan(plan);
  CHECK(!plan.valid());
  CHECK_THROWS_AS(compute(plan), std::logic_error);
  CHECK_THROWS_AS(swap_plan(plan), std::logic_error);
  CHECK(grids_equal_bitwise(in, inCopy));
  StencilPlan again = create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, w3}, in, out, 2, 2);
  compute(again);
  CHECK(again.valid());
}

void test_swap_and_two_pass() {  // test_stencil.cpp:211-249
  Grid2D a = random_grid(10, 6, 21), b(10, 6, 0.1, 0.2);
  StencilPlan plan =
      create_plan(Direction::X, BoundaryMode::Periodic, WeightStencil{Extents{1, 1, 0, 0}, {0.25, 0.5, 0.25}}, a, b, 1, 1);
  CHECK(plan.input() == &a && plan.output() == &b);
  swap_plan(plan);
  CHECK(plan.input() == &b && plan.output() == &a);
  swap_plan(plan);
  CHECK(plan.input() == &a && plan.output() == &b);

  Grid2D in = random_grid(14, 9, 31);
  const Grid2D inCopy = in;
  Grid2D out(14, 9, in.dx, in.dy);
  const WeightStencil sten{Extents{1, 1, 0, 0}, {0.5, -1.0, 0.5}};
  StencilPlan p2 = create_plan(Direction::X, BoundaryMode::Periodic, sten, in, out, 3, 2);
  compute(p2);
  swap_plan(p2);
  compute(p2);
  Grid2D ref1(14, 9, inCopy.dx, inCopy.dy), ref2(14, 9, inCopy.dx, inCopy.dy);
  for (int j = 0; j < 9; ++j)
    for (int i = 0; i < 14; ++i) ref1(i, j) = apply_weights_at(inCopy, sten, i, j, BoundaryMode::Periodic);
  for (int j = 0; j < 9; ++j)
    for (int i = 0; i < 14; ++i) ref2(i, j) = apply_weights_at(ref1, sten, i, j, BoundaryMode::Periodic);
  CHECK(grids_equal_bitwise(in, ref2));
}

void test_sine_and_convergence() {  // test_stencil.cpp:263-276, 489-501
  const int n = 1024;
  Grid2D in(n, 1, kTwoPi / n, 1.0);
  for (int i = 0; i < n; ++i) in(i, 0) = std::sin(i * in.dx);
  Grid2D out(n, 1, in.dx, in.dy);
  const double c = 1.0 / (in.dx * in.dx);
  StencilPlan plan = create_plan(Direction::X, BoundaryMode::Periodic,
                                 WeightStencil{Extents{1, 1, 0, 0}, {c, -2.0 * c, c}}, in, out, 1, 1);
  compute(plan);
  double maxErr = 0.0;
  for (int i = 0; i < n; ++i) maxErr = std::max(maxErr, std::abs(out(i, 0) + std::sin(i * in.dx)));
  CHECK(maxErr < 5e-6);
  CHECK(maxErr > 1e-6);
  const std::vector<double> k8 = {-1.0 / 560.0, 8.0 / 315.0, -1.0 / 5.0, 8.0 / 5.0, -205.0 / 72.0,
                                  8.0 / 5.0,    -1.0 / 5.0,  8.0 / 315.0, -1.0 / 560.0};
  const double r2 = second_derivative_max_error(128, {1.0, -2.0, 1.0}, 1) /
                    second_derivative_max_error(256, {1.0, -2.0, 1.0}, 1);
  const double r8 = second_derivative_max_error(32, k8, 4) / second_derivative_max_error(64, k8, 4);
  CHECK(r2 > 3.6 && r2 < 4.4);
  CHECK(r8 > 256.0 * 0.8 && r8 < 256.0 * 1.2);
}

void test_identity_cross_weightsfn() {  // test_stencil.cpp:278-388
  Grid2D in = random_grid(9, 11, 51);
  Grid2D out(9, 11, in.dx, in.dy);
  for (Direction dir : {Direction::X, Direction::Y, Direction::XY})
    for (BoundaryMode mode : {BoundaryMode::Periodic, BoundaryMode::NonPeriodic}) {
      out.values.setZero();
      StencilPlan plan = create_plan(dir, mode, WeightStencil{Extents{}, {1.0}}, in, out, 2, 2);
      compute(plan);
      CHECK(grids_equal_bitwise(out, in));
    }
  Grid2D g(8, 8, 1.0, 1.0);
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 8; ++i) g(i, j) = static_cast<double>(i * i) * static_cast<double>(j * j);
  Grid2D o(8, 8, 1.0, 1.0);
  StencilPlan cp = create_plan(Direction::XY, BoundaryMode::NonPeriodic,
                               WeightStencil{Extents{1, 1, 1, 1}, {1, -2, 1, -2, 4, -2, 1, -2, 1}}, g, o, 1, 1);
  compute(cp);
  for (int j = 2; j <= 5; ++j)
    for (int i = 2; i <= 5; ++i) CHECK(o(i, j) == 4.0);

  Grid2D r = random_grid(9, 6, 101);
  const std::vector<double> w = random_weights(9, 102);
  for (BoundaryMode mode : {BoundaryMode::Periodic, BoundaryMode::NonPeriodic}) {
    Grid2D outW(9, 6, r.dx, r.dy), outF(9, 6, r.dx, r.dy);
    StencilPlan pw = create_plan(Direction::XY, mode, WeightStencil{Extents{1, 1, 1, 1}, w}, r, outW, 3, 2);
    StencilPlan pf = create_plan(Direction::XY, mode, FunctionStencil{Extents{1, 1, 1, 1}, &functions::fn_weighted_3x3, w},
                                 r, outF, 3, 2);
    compute(pw);
    compute(pf);
    CHECK(grids_equal_bitwise(outW, outF));
  }
}

void test_tiles_frame_shift_concurrency() {  // test_stencil.cpp:390-555
  Grid2D in = random_grid(16, 13, 111);
  const std::vector<double> w = random_weights(15, 112);
  const WeightStencil ws{Extents{2, 2, 1, 1}, w};
  Grid2D ref(16, 13, in.dx, in.dy);
  {
    StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, ws, in, ref, 1, 1);
    compute(plan);
  }
  for (int j = 0; j < 13; ++j)
    for (int i = 0; i < 16; ++i) CHECK(ref(i, j) == oracle_weights_at(in, ws.ext, w, i, j, true));
  for (int tiles : {1, 2, 3, 5, 13})
    for (int workers : {1, 2, 4}) {
      Grid2D out(16, 13, in.dx, in.dy);
      StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, ws, in, out, tiles, workers);
      compute(plan);
      CHECK(grids_equal_bitwise(out, ref));
    }
  const double sentinel = -12345.678;
  struct Case {
    Direction dir;
    Extents e;
  };
  for (const Case& c : {Case{Direction::X, {2, 3, 0, 0}}, Case{Direction::Y, {0, 0, 1, 2}}, Case{Direction::XY, {1, 2, 2, 1}}}) {
    Grid2D g = random_grid(11, 9, 121);
    Grid2D out(11, 9, g.dx, g.dy);
    out.values.setConstant(sentinel);
    const int count = c.e.width() * c.e.height();
    StencilPlan plan =
        create_plan(c.dir, BoundaryMode::NonPeriodic, WeightStencil{c.e, random_weights(count, 122)}, g, out, 3, 2);
    compute(plan);
    for (int j = 0; j < 9; ++j)
      for (int i = 0; i < 11; ++i) {
        const bool frame = i < c.e.left || i >= 11 - c.e.right || j < c.e.top || j >= 9 - c.e.bottom;
        CHECK(frame ? out(i, j) == sentinel : out(i, j) != sentinel);
      }
  }
  Grid2D s0 = random_grid(12, 10, 131);
  const WeightStencil w9{Extents{1, 1, 1, 1}, random_weights(9, 132)};
  Grid2D plain(12, 10, s0.dx, s0.dy);
  {
    StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, w9, s0, plain, 2, 2);
    compute(plan);
  }
  for (auto [si, sj] : {std::pair{3, 2}, std::pair{-5, 7}, std::pair{1, 0}}) {
    Grid2D shifted = cyclic_shift(s0, si, sj);
    Grid2D o(12, 10, s0.dx, s0.dy);
    StencilPlan plan = create_plan(Direction::XY, BoundaryMode::Periodic, w9, shifted, o, 2, 2);
    compute(plan);
    CHECK(grids_equal_bitwise(o, cyclic_shift(plain, si, sj)));
  }
  Grid2D inA = random_grid(24, 18, 171), inB = random_grid(24, 18, 172);
  Grid2D outA(24, 18, inA.dx, inA.dy), outB(24, 18, inB.dx, inB.dy);
  Grid2D refA(24, 18, inA.dx, inA.dy), refB(24, 18, inB.dx, inB.dy);
  const WeightStencil w16{Extents{2, 1, 1, 2}, random_weights(16, 173)};
  {
    StencilPlan pa = create_plan(Direction::XY, BoundaryMode::Periodic, w16, inA, refA, 2, 1);
    StencilPlan pb = create_plan(Direction::XY, BoundaryMode::Periodic, w16, inB, refB, 2, 1);
    compute(pa);
    compute(pb);
  }
  StencilPlan pa = create_plan(Direction::XY, BoundaryMode::Periodic, w16, inA, outA, 3, 2);
  StencilPlan pb = create_plan(Direction::XY, BoundaryMode::Periodic, w16, inB, outB, 3, 2);
  std::thread ta([&] {
    for (int rep = 0; rep < 50; ++rep) compute(pa);
  });
  std::thread tb([&] {
    for (int rep = 0; rep < 50; ++rep) compute(pb);
  });
  ta.join();
  tb.join();
  CHECK(grids_equal_bitwise(outA, refA));
  CHECK(grids_equal_bitwise(outB, refB));
}

void test_residency() {  // test_stencil.cpp:515-525: the hint does not change results
  Grid2D in = random_grid(8, 8, 151);
  Grid2D outH(8, 8, in.dx, in.dy), outD(8, 8, in.dx, in.dy);
  const WeightStencil ws{Extents{1, 1, 1, 1}, random_weights(9, 152)};
  StencilPlan ph = create_plan(Direction::XY, BoundaryMode::Periodic, ws, in, outH, 1, 1);
  StencilPlan pd = create_plan(Direction::XY, BoundaryMode::Periodic, ws, in, outD, 1, 1);
  compute(ph, Residency::Host);
  compute(pd, Residency::Device);  // host-coherent on return, no sync needed
  CHECK(grids_equal_bitwise(outH, outD));
  // a second plan reading the Device-hint output sees the fresh host values
  Grid2D out2(8, 8, in.dx, in.dy), out3(8, 8, in.dx, in.dy);
  StencilPlan p2 = create_plan(Direction::XY, BoundaryMode::Periodic, ws, outD, out2, 1, 1);
  StencilPlan p3 = create_plan(Direction::XY, BoundaryMode::Periodic, ws, outH, out3, 1, 1);
  compute(p2);
  compute(p3);
  CHECK(grids_equal_bitwise(out2, out3));
  // the extension: compute_deferred chains stay in HBM until sync_to_host
  Grid2D a = random_grid(16, 12, 153), b(16, 12, a.dx, a.dy);
  Grid2D a2 = a, b2(16, 12, a.dx, a.dy);
  StencilPlan pc = create_plan(Direction::XY, BoundaryMode::Periodic, ws, a, b, 1, 1);
  StencilPlan ps = create_plan(Direction::XY, BoundaryMode::Periodic, ws, a2, b2, 1, 1);
  for (int k = 0; k < 3; ++k) {
    compute_deferred(pc);
    swap_plan(pc);
    compute(ps);
    swap_plan(ps);
  }
  sync_to_host(pc);
  CHECK(grids_equal_bitwise(*pc.input(), *ps.input()));
}

void test_workers_to_gpus() {  // numWorkers -> GPUs; test_stencil.cpp:390-409
  // SG_DEVICE_MAP=modulo (set by tests/test_cxx_gpu.py): G workers on a
  // one-GPU box share the device; the multi-worker path still runs
  const Grid2D in0 = random_grid(64, 40, 161);
  const FunctionStencil fs{Extents{1, 1, 1, 1}, functions::fn_weighted_3x3, random_weights(9, 162)};
  const WeightStencil tall{Extents{1, 2, 3, 1}, random_weights(20, 163)};
  for (const bool periodic : {true, false}) {
    const BoundaryMode mode = periodic ? BoundaryMode::Periodic : BoundaryMode::NonPeriodic;
    std::vector<Grid2D> outs;
    for (const int workers : {1, 2, 4, 8}) {
      Grid2D in = in0, out(64, 40, in0.dx, in0.dy);
      StencilPlan p = create_plan(Direction::XY, mode, fs, in, out, 1, workers);
      compute(p);
      swap_plan(p);
      compute_deferred(p);
      swap_plan(p);
      compute_deferred(p);
      sync_to_host(p);
      StencilPlan q = create_plan(Direction::XY, mode, tall, out, in, 1, workers);
      compute(q);
      outs.push_back(in);
    }
    for (std::size_t k = 1; k < outs.size(); ++k) CHECK(grids_equal_bitwise(outs[0], outs[k]));
  }
  // CHStepper(p, 1, numWorkers): the distributed step over numWorkers GPUs
  CHParams prm;
  prm.nx = prm.ny = 256;
  prm.dt = 0.1 * prm.dx();
  prm.T = 1.0;
  std::vector<Grid2D> fields;
  for (const int workers : {1, 2, 4, 8}) {
    CHStepper st(prm, 1, workers);
    for (int k = 0; k < 7; ++k) st.step();
    fields.push_back(st.field());
    fields.push_back(st.previous_field());
  }
  for (std::size_t k = 2; k < fields.size(); ++k) CHECK(grids_equal_bitwise(fields[k % 2], fields[k]));
}

void test_fp32_dropin() {  // FP32 extension (north_star: FP32+FP64); bar 1e-5 relative
  // Grid2Df through the same create_plan / compute / swap_plan calls: the
  // result is within 1e-5 (normwise, relative) of the FP64 evaluation on the
  // float-rounded input, for weights and device functions, XY/X/Y, periodic
  // and not, one worker and several (numWorkers -> GPUs)
  const int nx = 97, ny = 61;  // odd sizes: the unaligned-row path too
  const Grid2D src = random_grid(nx, ny, 171);
  Grid2D in64(nx, ny, src.dx, src.dy);
  Grid2Df in32(nx, ny, src.dx, src.dy);
  for (std::ptrdiff_t k = 0; k < src.size(); ++k) {
    in32.data()[k] = static_cast<float>(src.data()[k]);
    in64.data()[k] = static_cast<double>(in32.data()[k]);
  }
  struct Case {
    Direction d;
    StencilKind kind;
  };
  const std::vector<Case> cases = {
      {Direction::XY, FunctionStencil{Extents{1, 1, 1, 1}, functions::fn_weighted_3x3, random_weights(9, 172)}},
      {Direction::XY, WeightStencil{Extents{1, 1, 1, 1}, random_weights(9, 173)}},
      {Direction::XY, WeightStencil{Extents{2, 2, 2, 2}, random_weights(25, 174)}},
      {Direction::X, WeightStencil{Extents{2, 2, 0, 0}, {1.0, -4.0, 6.0, -4.0, 1.0}}},
      {Direction::Y, WeightStencil{Extents{0, 0, 3, 1}, random_weights(5, 175)}},
      {Direction::XY, FunctionStencil{Extents{1, 1, 1, 1}, functions::ch_nonlinear_window, random_weights(9, 176)}},
  };
  for (const Case& c : cases)
    for (const bool periodic : {true, false})
      for (const int workers : {1, 3}) {
        const BoundaryMode mode = periodic ? BoundaryMode::Periodic : BoundaryMode::NonPeriodic;
        Grid2Df a = in32, b(nx, ny, src.dx, src.dy);
        Grid2D a64 = in64, b64(nx, ny, src.dx, src.dy);
        StencilPlanF p = create_plan(c.d, mode, c.kind, a, b, 1, workers);
        compute(p);
        StencilPlan q = create_plan(c.d, mode, c.kind, a64, b64, 1, 1);
        compute(q);
        double num = 0.0, den = 0.0;
        for (std::ptrdiff_t k = 0; k < b64.size(); ++k) {
          const double e = static_cast<double>(b.data()[k]) - b64.data()[k];
          num += e * e;
          den += b64.data()[k] * b64.data()[k];
        }
        const double rel = std::sqrt(num / (den > 0.0 ? den : 1.0));
        CHECK(rel <= 1e-5);
        if (rel > 1e-5) std::printf("  fp32 rel %.3e periodic=%d workers=%d\n", rel, periodic, workers);
        swap_plan(p);  // the float plan swaps like the double one
        CHECK(p.input() == &b && p.output() == &a);
        destroy_plan(p);
        CHECK(!p.valid());
      }
  Grid2Df x(8, 8, 1.0, 1.0), y(8, 9, 1.0, 1.0);
  CHECK_THROWS_AS(create_plan(Direction::XY, BoundaryMode::Periodic,
                              WeightStencil{Extents{1, 1, 1, 1}, std::vector<double>(9, 1.0)}, x, y, 1, 1),
                  std::invalid_argument);
}

// A user's own window function (the reference's central feature,
// stencil.hpp:20-25): the host function and its body as source.
double user_fn(const double* window, const double* coe, int rowStride) {
  const double c = window[rowStride + 1];
  double acc = c * c * coe[0];
  acc += (window[0] - window[2 * rowStride + 2]) * coe[1];
  acc += window[rowStride] * window[rowStride + 2] - coe[2];
  return acc;
}

void test_source_function() {
  const char* body = R"(
    const T c = window[rowStride + 1];
    T acc = c * c * coe[0];
    acc += (window[0] - window[2 * rowStride + 2]) * coe[1];
    acc += window[rowStride] * window[rowStride + 2] - coe[2];
    return acc;)";
  const Grid2D in0 = random_grid(97, 45, 181);
  const FunctionStencil fs{Extents{1, 1, 1, 1}, user_fn, {0.5, -1.25, 0.75}};
  // unregistered: there is no CPU path
  {
    Grid2D a = in0, b(97, 45, in0.dx, in0.dy);
    CHECK_THROWS_AS(create_plan(Direction::XY, BoundaryMode::Periodic, fs, a, b, 1, 1), std::invalid_argument);
  }
  CHECK_THROWS_AS(register_device_function_source(user_fn, "return undefined_name;"), std::invalid_argument);
  CHECK(register_device_function_source(user_fn, body, "user_fn") >= SG_FN_JIT_BASE);
  for (const bool periodic : {true, false}) {
    const BoundaryMode mode = periodic ? BoundaryMode::Periodic : BoundaryMode::NonPeriodic;
    Grid2D a = in0, b(97, 45, in0.dx, in0.dy);
    StencilPlan p = create_plan(Direction::XY, mode, fs, a, b, 1, 1);
    compute(p);
    int bad = 0;
    const int lo = periodic ? 0 : 1;
    for (int j = lo; j < 45 - lo; ++j)
      for (int i = lo; i < 97 - lo; ++i) {
        const double want = apply_function_at(a, fs, i, j, mode);  // the host function itself
        if (std::memcmp(&want, &b.values(j, i), sizeof(double)) != 0) ++bad;
      }
    CHECK(bad == 0);
  }
}

void test_acceptance_criterion_2() {  // acceptance.cpp:104-151
  std::mt19937_64 rng(99);
  std::uniform_real_distribution<double> val(-2.0, 2.0);
  int mismatches = 0;
  for (int trial = 0; trial < 200; ++trial) {
    std::uniform_int_distribution<int> dim(1, 9);
    const int nx = dim(rng), ny = dim(rng);
    auto extent = [&](int n) { return std::uniform_int_distribution<int>(0, std::min(2, n - 1))(rng); };
    Extents e;
    const int pick = std::uniform_int_distribution<int>(0, 2)(rng);
    const Direction dir = pick == 0 ? Direction::X : pick == 1 ? Direction::Y : Direction::XY;
    if (dir != Direction::Y) {
      e.left = extent(nx);
      e.right = extent(nx);
    }
    if (dir != Direction::X) {
      e.top = extent(ny);
      e.bottom = extent(ny);
    }
    Grid2D in(nx, ny, 1.0, 1.0);
    for (std::ptrdiff_t k = 0; k < in.size(); ++k) in.data()[k] = val(rng);
    std::vector<double> w(static_cast<std::size_t>(e.width()) * e.height());
    for (double& x : w) x = val(rng);
    Grid2D out(nx, ny, 1.0, 1.0);
    StencilPlan plan = create_plan(dir, BoundaryMode::Periodic, WeightStencil{e, w}, in, out, 1, 1);
    compute(plan);
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const double acc = oracle_weights_at(in, e, w, i, j, true);
        if (std::memcmp(&acc, &out.values(j, i), sizeof(double)) != 0) ++mismatches;
      }
  }
  CHECK(mismatches == 0);
}

// ------------------------------------------------------------------ penta

void test_penta() {  // test_penta.cpp
  const int B = 4, n = 11;
  PentaBatch m(B, n, true);
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (ArrayXd* band : {&m.secondSub, &m.sub, &m.diag, &m.super, &m.secondSuper})
    for (std::ptrdiff_t k = 0; k < band->size(); ++k) (*band)[k] = u(rng);
  for (std::ptrdiff_t k = 0; k < m.diag.size(); ++k) m.diag[k] += 6.0;
  RhsBatch rhs(B, n);
  for (std::ptrdiff_t k = 0; k < rhs.values.size(); ++k) rhs.values[k] = u(rng);
  const RhsBatch x = solve_periodic_batch(m, rhs);
  double worst = 0.0;
  for (int b = 0; b < B; ++b)
    for (int r = 0; r < n; ++r) {
      double ax = m.diag[m.idx(b, r)] * x.at(b, r);
      ax += m.secondSub[m.idx(b, r)] * x.at(b, (r - 2 + n) % n) + m.sub[m.idx(b, r)] * x.at(b, (r - 1 + n) % n);
      ax += m.super[m.idx(b, r)] * x.at(b, (r + 1) % n) + m.secondSuper[m.idx(b, r)] * x.at(b, (r + 2) % n);
      worst = std::max(worst, std::abs(ax - rhs.at(b, r)));
    }
  CHECK(worst <= 1e-10);
  PentaBatch z(3, 6, false);
  z.diag.setConstant(1.0);
  z.diag[z.idx(1, 0)] = 0.0;
  bool right = false;
  try {
    solve_batch(z, RhsBatch(3, 6));
  } catch (const PentaSolveError& e) {
    right = e.system == 1;
  }
  CHECK(right);
  CHECK_THROWS_AS(solve_periodic_batch(z, RhsBatch(3, 6)), std::invalid_argument);
  const PentaBatch id = build_hyperdiffusion_operator(0.0, 16, 5, false);
  RhsBatch r(5, 16);
  for (std::ptrdiff_t k = 0; k < r.values.size(); ++k) r.values[k] = u(rng);
  const RhsBatch xi = solve_batch(id, r);
  CHECK(std::memcmp(xi.values.data(), r.values.data(), sizeof(double) * 80) == 0);
}

// --------------------------------------------------------------------- CH

CHParams small_params(int nx, int ny, double dtFactor = 0.1) {
  CHParams p;
  p.nx = nx;
  p.ny = ny;
  p.T = 1.0;
  p.dt = dtFactor * p.dx();
  return p;
}

void test_ch() {  // test_cahn_hilliard.cpp:56-75, 259-318
  CHParams bad = small_params(64, 64);
  bad.nx = 100;
  CHECK_THROWS_AS(bad.validate(), std::invalid_argument);
  CHECK_THROWS_AS(CHStepper(bad), std::invalid_argument);

  CHParams p = small_params(64, 16);
  p.nonlinearEnabled = false;
  CHStepper stepper(p);
  Grid2D mode(p.nx, p.ny, p.dx(), p.dy());
  for (int j = 0; j < p.ny; ++j)
    for (int i = 0; i < p.nx; ++i) mode(i, j) = std::cos(i * p.dx());
  stepper.set_state(mode, mode);
  const double h = p.dx();
  const double lam4 = (6.0 - 8.0 * std::cos(h) + 2.0 * std::cos(2.0 * h)) / (h * h * h * h);
  const double kb = (2.0 / 3.0) * p.D * p.gamma * p.dt;
  const double lx = 1.0 + kb * lam4;
  double aPrev = 1.0, aCurr = 1.0;
  for (int s = 0; s < 10; ++s) {
    stepper.step();
    const double aBar = 2.0 * aCurr - aPrev;
    const double rhs = -(2.0 / 3.0) * (aCurr - aPrev) - kb * lam4 * aBar;
    const double aNext = aBar + rhs / lx;
    aPrev = aCurr;
    aCurr = aNext;
    double maxErr = 0.0;
    for (int j = 0; j < p.ny; ++j)
      for (int i = 0; i < p.nx; ++i) maxErr = std::max(maxErr, std::abs(stepper.field()(i, j) - aCurr * std::cos(i * h)));
    CHECK(maxErr <= 1e-12);
  }
  CHECK(stepper.step_index() == 10);

  CHParams q = small_params(32, 32);
  q.seed = 21;
  CHStepper ref(q, 1, 1);
  for (int s = 0; s < 3; ++s) ref.step();
  for (int tiles : {1, 2, 4})
    for (int workers : {1, 2}) {
      CHStepper st(q, tiles, workers);
      for (int s = 0; s < 3; ++s) st.step();
      CHECK(grids_equal_bitwise(st.field(), ref.field()));
    }
  CHStepper ic(q);
  CHECK(grids_equal_bitwise(ic.field(), initial_condition(q)));
  Grid2D cst(32, 32, q.dx(), q.dy());
  cst.values.setConstant(0.3);
  ic.set_state(cst, cst);
  ic.steps(10);
  double worst = 0.0;
  for (std::ptrdiff_t k = 0; k < cst.size(); ++k) worst = std::max(worst, std::abs(ic.field().data()[k] - 0.3));
  CHECK(worst <= 0.3 * 1e-13);
}

void test_diagnostics_and_run() {  // test_cahn_hilliard.cpp:320-366, 475-505
  Grid2D c(64, 64, kTwoPi / 64, kTwoPi / 64);
  c.values.setConstant(0.77);
  CHECK(std::abs(simpson_mean(c) - 0.77) <= 0.77 * 1e-13);
  Grid2D zero(16, 16, kTwoPi / 16, kTwoPi / 16);
  CHECK(s_metric(zero) == 1.0);
  Grid2D one(16, 16, kTwoPi / 16, kTwoPi / 16);
  one.values.setConstant(1.0);
  CHECK_THROWS_AS(s_metric(one), std::domain_error);
  CHParams p = small_params(64, 64);
  Grid2D cx(64, 64, p.dx(), p.dy());
  for (int j = 0; j < 64; ++j)
    for (int i = 0; i < 64; ++i) cx(i, j) = std::cos(i * p.dx());
  CHECK(std::abs(k1_metric(cx) - 1.0) <= 1e-12);
  CHECK_THROWS_AS(k1_metric(Grid2D(64, 64, p.dx(), p.dy())), std::domain_error);
  CHParams q = small_params(16, 16);
  q.T = q.dt;
  q.icAmplitude = 0.0;
  std::vector<Diagnostics> rows;
  RunSink sink;
  sink.diagEvery = 1;
  sink.onDiagnostics = [&](const Diagnostics& d) { rows.push_back(d); };
  run(q, 1, 1, sink);
  CHECK(rows.size() == 2);
  CHECK(rows.size() == 2 && rows[0].t == 0.0 && rows[1].t == q.dt);
  q.T = 10.5 * q.dt;
  int snaps = 0;
  RunSink s2;
  s2.diagEvery = 0;
  s2.snapEvery = 5;
  s2.onSnapshot = [&](const Grid2D& g, int, double) {
    CHECK(g.nx == 16);
    ++snaps;
  };
  run(q, 1, 1, s2);
  CHECK(snaps == 3);
}

void test_snapshot_and_checkpoint() {  // test_io.cpp:26-93 + exact BDF2 resume
  Grid2D g = random_grid(13, 7, 5);
  const std::string path = "/tmp/stengrid_cxx_test.csg";
  write_snapshot(g, path);
  const Grid2D back = read_snapshot(path);
  CHECK(grids_equal_bitwise(back, g) && back.dx == g.dx && back.dy == g.dy);
  CHECK(format_diagnostics_row(Diagnostics{0.5, 1.25, 0.0}) == "0.5,1.25,0");
  CHParams p = small_params(32, 16);
  CHStepper a(p);
  a.steps(7);
  const std::string ck = "/tmp/stengrid_cxx_test.ck";
  save_checkpoint(a, ck);
  a.steps(9);
  CHStepper b(p);
  load_checkpoint(b, ck);
  CHECK(b.step_index() == 7);
  b.steps(9);
  CHECK(grids_equal_bitwise(a.field(), b.field()));
  CHECK(b.time() == a.time());
}

void test_weno() {  // test_weno.cpp: constant field, shape errors
  const int n = 64;
  const double dx = kTwoPi / n;
  Grid2D c(n, n, dx, dx);
  c.values.setConstant(0.7);
  VelocityField vel{Grid2D(n, n, dx, dx), Grid2D(n, n, dx, dx)};
  vel.u.values.setConstant(1.0);
  vel.v.values.setConstant(-0.5);
  const Grid2D o = weno_advect(c, vel);
  bool zero = true;
  for (std::ptrdiff_t k = 0; k < o.size(); ++k) zero = zero && o.data()[k] == 0.0;
  CHECK(zero);
  Grid2D s(n, n, dx, dx);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) s(i, j) = std::sin(i * dx);
  vel.v.values.setZero();
  const Grid2D d = weno_advect(s, vel);
  double err = 0.0;
  for (int i = 0; i < n; ++i) err = std::max(err, std::abs(d(i, 3) + std::cos(i * dx)));
  CHECK(err < 1e-5);
  CHECK_THROWS_AS(weno_advect(Grid2D(6, 8, 1.0, 1.0), VelocityField{Grid2D(6, 8, 1.0, 1.0), Grid2D(6, 8, 1.0, 1.0)}),
                  std::invalid_argument);
}

}  // namespace

void run_test(const char* name, void (*fn)()) {
  std::printf("[ %s ]\n", name);
  std::fflush(stdout);
  fn();
}

int main() {
  run_test("test_create_plan_rejects_invalid_setups", test_create_plan_rejects_invalid_setups);
  run_test("test_lifecycle", test_lifecycle);
  run_test("test_swap_and_two_pass", test_swap_and_two_pass);
  run_test("test_sine_and_convergence", test_sine_and_convergence);
  run_test("test_identity_cross_weightsfn", test_identity_cross_weightsfn);
  run_test("test_tiles_frame_shift_concurrency", test_tiles_frame_shift_concurrency);
  run_test("test_residency", test_residency);
  run_test("test_workers_to_gpus", test_workers_to_gpus);
  run_test("test_fp32_dropin", test_fp32_dropin);
  run_test("test_source_function", test_source_function);
  run_test("test_acceptance_criterion_2", test_acceptance_criterion_2);
  run_test("test_penta", test_penta);
  run_test("test_ch", test_ch);
  run_test("test_diagnostics_and_run", test_diagnostics_and_run);
  run_test("test_snapshot_and_checkpoint", test_snapshot_and_checkpoint);
  run_test("test_weno", test_weno);
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
