// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on
// the product path). A thin extern "C" shim over the UNMODIFIED reference
// library (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libstengrid_ref.so) so that Python tests, the golden-fixture
// generator and bench.py's cpu_baseline / --impl reference legs can call the
// real reference code with plain pointers.
//
// Every entry point copies caller buffers into reference Grid2D / RhsBatch
// objects, runs the reference's own public API, and copies results back.
// Errors are mapped to integer codes (1 invalid_argument, 2 logic_error,
// 3 PentaSolveError, 4 domain_error, 9 other) with the message and the
// PentaSolveError system index retrievable via ref_last_error().
//
// The six window functions below restate, with identical arithmetic order,
// the functions the reference defines in anonymous namespaces of its tests,
// CLI and CH solver (they are not exported by the library):
//   ch_nonlinear_window        cahn_hilliard.cpp:36-47
//   central_difference_window  tools/main.cpp:47-49
//   fn_center                  tests/test_stencil.cpp:68
//   fn_central_second          tests/test_stencil.cpp:70-77
//   fn_lap_cube_diff_first     tests/test_stencil.cpp:79-85
//   fn_weighted_3x3            tests/test_stencil.cpp:88-93
#include "stengrid/cahn_hilliard.hpp"
#include "stengrid/grid.hpp"
#include "stengrid/penta.hpp"
#include "stengrid/snapshot.hpp"
#include "stengrid/stencil.hpp"
#include "stengrid/weno.hpp"

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

using namespace stengrid;

namespace {

thread_local std::string g_msg;
thread_local int g_system = -1;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_msg.clear();
    return 0;
  } catch (const PentaSolveError& e) {
    g_msg = e.what();
    g_system = e.system;
    return 3;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_msg = e.what();
    return 4;
  } catch (const std::logic_error& e) {
    g_msg = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 9;
  }
}

double w_ch_nonlinear(const double* window, const double* coe, int rs) {
  double acc = 0.0;
  for (int q = 0; q < 3; ++q) {
    const double* row = window + static_cast<std::ptrdiff_t>(q) * rs;
    const double* cr = coe + q * 3;
    for (int p = 0; p < 3; ++p) {
      const double v = row[p];
      acc += cr[p] * (v * v * v - v);
    }
  }
  return acc;
}
double w_central_difference(const double* w, const double* coe, int) {
  return (w[0] - 2.0 * w[1] + w[2]) * coe[0];
}
double w_center(const double* w, const double*, int rs) { return w[rs + 1]; }
double w_central_second(const double* w, const double* coe, int) {
  double acc = 0.0;
  acc += coe[0] * w[0];
  acc += (-2.0 * coe[0]) * w[1];
  acc += coe[0] * w[2];
  return acc;
}
double w_lap_cube_diff_first(const double* w, const double* coe, int rs) {
  auto g = [](double v) { return v * v * v - v; };
  const double gm = g(w[rs + 1]);
  const double x = (g(w[rs]) - 2.0 * gm) + g(w[rs + 2]);
  const double y = (g(w[1]) - 2.0 * gm) + g(w[2 * rs + 1]);
  return coe[0] * x + coe[1] * y;
}
double w_weighted_3x3(const double* w, const double* coe, int rs) {
  double acc = 0.0;
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) acc += coe[q * 3 + p] * w[q * rs + p];
  return acc;
}

// Function ids shared with include/stengrid/sg.h (SG_FN_*).
StencilFunction fn_by_id(int id) {
  switch (id) {
    case 1: return &w_ch_nonlinear;
    case 2: return &w_central_difference;
    case 3: return &w_center;
    case 4: return &w_central_second;
    case 5: return &w_lap_cube_diff_first;
    case 6: return &w_weighted_3x3;
    default: return nullptr;
  }
}

Direction dir_of(int d) { return d == 0 ? Direction::X : d == 1 ? Direction::Y : Direction::XY; }
BoundaryMode mode_of(int periodic) { return periodic ? BoundaryMode::Periodic : BoundaryMode::NonPeriodic; }

Grid2D grid_from(const double* v, int nx, int ny) {
  Grid2D g(nx, ny, 1.0, 1.0);
  std::memcpy(g.data(), v, sizeof(double) * static_cast<std::size_t>(g.size()));
  return g;
}

StencilKind make_kind(int fnId, const int* ext, const double* w, int nw) {
  Extents e{ext[0], ext[1], ext[2], ext[3]};
  if (fnId == 0) return WeightStencil{e, std::vector<double>(w, w + nw)};
  return FunctionStencil{e, fn_by_id(fnId), std::vector<double>(w, w + nw)};
}

CHParams ch_params(const double* dp, const long long* ip) {
  CHParams p;
  p.D = dp[0];
  p.gamma = dp[1];
  p.lx = dp[2];
  p.ly = dp[3];
  p.dt = dp[4];
  p.T = dp[5];
  p.icAmplitude = dp[6];
  p.nx = static_cast<int>(ip[0]);
  p.ny = static_cast<int>(ip[1]);
  p.seed = static_cast<std::uint64_t>(ip[2]);
  p.nonlinearEnabled = ip[3] != 0;
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error(int* system) {
  if (system) *system = g_system;
  return g_msg.c_str();
}

int ref_wrap(long long i, int n, int* out) {
  return guarded([&] { *out = wrap(i, n); });
}

int ref_make_tiles(int ny, int numTiles, int* begins, int* ends) {
  return guarded([&] {
    TilePlan t = make_tiles(ny, numTiles, Extents{});
    for (int k = 0; k < t.num_tiles(); ++k) {
      begins[k] = t.tiles[k].jBegin;
      ends[k] = t.tiles[k].jEnd;
    }
  });
}

/// create_plan + compute (+ swap + compute, `applications` times) + destroy.
/// `out` is both the initial content of the output grid (so non-periodic
/// frames keep caller values) and the result buffer. When applications > 1
/// the plan is swapped between applications (stencil.cpp:197-200) and the
/// final result is copied from whichever grid holds it.
int ref_stencil(int dir, int periodic, const int* ext, int fnId, const double* w, int nw,
                const double* in, double* out, int nx, int ny, int numTiles, int numWorkers,
                int applications) {
  return guarded([&] {
    Grid2D gi = grid_from(in, nx, ny);
    Grid2D go = grid_from(out, nx, ny);
    StencilPlan plan = create_plan(dir_of(dir), mode_of(periodic), make_kind(fnId, ext, w, nw), gi,
                                   go, numTiles, numWorkers);
    for (int a = 0; a < applications; ++a) {
      compute(plan);
      if (a + 1 < applications) swap_plan(plan);
    }
    const Grid2D* res = plan.output();
    std::memcpy(out, res->data(), sizeof(double) * static_cast<std::size_t>(res->size()));
    destroy_plan(plan);
  });
}

/// Timed compute loop (steady_clock around compute() only, as bench.cpp:33-40).
/// Returns seconds per application through *secs.
int ref_stencil_timed(int dir, int periodic, const int* ext, int fnId, const double* w, int nw,
                      const double* in, int nx, int ny, int numTiles, int numWorkers, int warmup,
                      int reps, double* secs) {
  return guarded([&] {
    Grid2D gi = grid_from(in, nx, ny);
    Grid2D go(nx, ny, 1.0, 1.0);
    StencilPlan plan = create_plan(dir_of(dir), mode_of(periodic), make_kind(fnId, ext, w, nw), gi,
                                   go, numTiles, numWorkers);
    for (int a = 0; a < warmup; ++a) compute(plan);
    const auto t0 = std::chrono::steady_clock::now();
    for (int a = 0; a < reps; ++a) compute(plan);
    const auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count() / (reps > 0 ? reps : 1);
  });
}

int ref_apply_at(int periodic, const int* ext, int fnId, const double* w, int nw, const double* in,
                 int nx, int ny, int i, int j, double* out) {
  return guarded([&] {
    Grid2D g = grid_from(in, nx, ny);
    Extents e{ext[0], ext[1], ext[2], ext[3]};
    if (fnId == 0)
      *out = apply_weights_at(g, WeightStencil{e, std::vector<double>(w, w + nw)}, i, j, mode_of(periodic));
    else
      *out = apply_function_at(g, FunctionStencil{e, fn_by_id(fnId), std::vector<double>(w, w + nw)},
                               i, j, mode_of(periodic));
  });
}

/// Batched pentadiagonal solve through solve_batch / solve_periodic_batch.
/// Bands and rhs are interleaved (r*B + b) as in penta.hpp:12-20.
int ref_penta_solve(int periodic, int B, int n, const double* e, const double* c, const double* d,
                    const double* a, const double* b, double* rhs, int numWorkers) {
  return guarded([&] {
    PentaBatch m(B, n, periodic != 0);
    const std::size_t len = static_cast<std::size_t>(B) * n;
    std::memcpy(m.secondSub.data(), e, len * sizeof(double));
    std::memcpy(m.sub.data(), c, len * sizeof(double));
    std::memcpy(m.diag.data(), d, len * sizeof(double));
    std::memcpy(m.super.data(), a, len * sizeof(double));
    std::memcpy(m.secondSuper.data(), b, len * sizeof(double));
    RhsBatch r(B, n);
    std::memcpy(r.values.data(), rhs, len * sizeof(double));
    WorkerPool pool(numWorkers);
    RhsBatch x = periodic ? solve_periodic_batch(m, r, &pool) : solve_batch(m, r, &pool);
    std::memcpy(rhs, x.values.data(), len * sizeof(double));
  });
}

int ref_hyperdiffusion_operator(double sigma, int n, int B, int periodic, double* e, double* c,
                                double* d, double* a, double* b) {
  return guarded([&] {
    PentaBatch m = build_hyperdiffusion_operator(sigma, n, B, periodic != 0);
    const std::size_t len = static_cast<std::size_t>(B) * n * sizeof(double);
    std::memcpy(e, m.secondSub.data(), len);
    std::memcpy(c, m.sub.data(), len);
    std::memcpy(d, m.diag.data(), len);
    std::memcpy(a, m.super.data(), len);
    std::memcpy(b, m.secondSuper.data(), len);
  });
}

int ref_ch_weights(double dx, double dy, double* bih25, double* nl9) {
  return guarded([&] {
    const auto b = biharmonic_weights(dx, dy);
    const auto n = nonlinear_laplacian_coefficients(dx, dy);
    std::memcpy(bih25, b.data(), 25 * sizeof(double));
    std::memcpy(nl9, n.data(), 9 * sizeof(double));
  });
}

int ref_ch_initial_condition(const double* dp, const long long* ip, double* out) {
  return guarded([&] {
    const Grid2D g = initial_condition(ch_params(dp, ip));
    std::memcpy(out, g.data(), sizeof(double) * static_cast<std::size_t>(g.size()));
  });
}

/// Construct CHStepper(params, tiles, workers); optionally set_state(curr,
/// prev) when both pointers are non-null on input (flag setState); run
/// `steps` steps; write C^n and C^{n-1} back.
int ref_ch_run(const double* dp, const long long* ip, int numTiles, int numWorkers, int steps,
               int setState, double* curr, double* prev) {
  return guarded([&] {
    const CHParams p = ch_params(dp, ip);
    CHStepper st(p, numTiles, numWorkers);
    if (setState) st.set_state(grid_from(curr, p.nx, p.ny), grid_from(prev, p.nx, p.ny));
    for (int s = 0; s < steps; ++s) st.step();
    const std::size_t cnt = static_cast<std::size_t>(p.nx) * p.ny;
    std::memcpy(curr, st.field().data(), cnt * sizeof(double));
    std::memcpy(prev, st.previous_field().data(), cnt * sizeof(double));
  });
}

/// Timed CH stepping (bench.cpp:33-40 pattern): construct untimed, `warmup`
/// untimed steps, then steady_clock around `steps` steps.
int ref_ch_timed(const double* dp, const long long* ip, int numTiles, int numWorkers, int warmup,
                 int steps, double* secsPerStep) {
  return guarded([&] {
    CHStepper st(ch_params(dp, ip), numTiles, numWorkers);
    for (int s = 0; s < warmup; ++s) st.step();
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) st.step();
    const auto t1 = std::chrono::steady_clock::now();
    *secsPerStep = std::chrono::duration<double>(t1 - t0).count() / (steps > 0 ? steps : 1);
  });
}

int ref_ch_diagnostics(const double* field, int nx, int ny, double dx, double dy, double* s,
                       double* k1Inv) {
  return guarded([&] {
    Grid2D g(nx, ny, dx, dy);
    std::memcpy(g.data(), field, sizeof(double) * static_cast<std::size_t>(g.size()));
    *s = s_metric(g);
    try {
      *k1Inv = 1.0 / k1_metric(g);
    } catch (const std::domain_error&) {
      *k1Inv = 0.0;
    }
  });
}

int ref_write_snapshot(const double* v, int nx, int ny, double dx, double dy, const char* path) {
  return guarded([&] {
    Grid2D g(nx, ny, dx, dy);
    std::memcpy(g.data(), v, sizeof(double) * static_cast<std::size_t>(g.size()));
    write_snapshot(g, std::string(path));
  });
}

int ref_read_snapshot(const char* path, int* nx, int* ny, double* dx, double* dy, double* out, long long cap) {
  return guarded([&] {
    const Grid2D g = read_snapshot(std::string(path));
    *nx = g.nx;
    *ny = g.ny;
    *dx = g.dx;
    *dy = g.dy;
    if (out && cap >= g.size()) std::memcpy(out, g.data(), sizeof(double) * static_cast<std::size_t>(g.size()));
  });
}

int ref_weno_advect(const double* phi, const double* u, const double* v, int nx, int ny, double dx, double dy,
                    int tiles, int workers, double* out) {
  return guarded([&] {
    Grid2D f(nx, ny, dx, dy);
    std::memcpy(f.data(), phi, sizeof(double) * static_cast<std::size_t>(f.size()));
    VelocityField vel{Grid2D(nx, ny, dx, dy), Grid2D(nx, ny, dx, dy)};
    std::memcpy(vel.u.data(), u, sizeof(double) * static_cast<std::size_t>(f.size()));
    std::memcpy(vel.v.data(), v, sizeof(double) * static_cast<std::size_t>(f.size()));
    const Grid2D o = weno_advect(f, vel, tiles, workers);
    std::memcpy(out, o.data(), sizeof(double) * static_cast<std::size_t>(o.size()));
  });
}

int ref_write_diagnostics_csv(const double* rows, int n, const char* path) {
  return guarded([&] {
    std::vector<Diagnostics> v(static_cast<std::size_t>(n));
    for (int k = 0; k < n; ++k) v[k] = Diagnostics{rows[3 * k], rows[3 * k + 1], rows[3 * k + 2]};
    write_diagnostics_csv(v, std::string(path));
  });
}

}  // extern "C"
