// stengrid/stencil.hpp — drop-in replacement for the reference stencil API
// (/root/reference/proj/include/stengrid/stencil.hpp:1-116): the same
// create_plan / compute / swap_plan / destroy_plan over Grid2D fields, the
// same kinds, enums, ownership rules and exceptions — executed by the sm_100a
// kernels of libstengrid_b200.so through the C ABI (stengrid/sg.h).
//
// Differences a caller can observe:
//  * StencilFunction pointers are host code; a FunctionStencil's fn must be
//    registered with a device twin (register_device_function) or with its
//    source (register_device_function_source: compiled at run time). The
//    reference's own window functions are pre-registered (stengrid::functions).
//    An unregistered fn throws std::invalid_argument — there is no CPU path.
//  * compute() is synchronous and host-coherent for both residency hints,
//    like the reference; the extension compute_deferred(plan) is the
//    paper's Residency::Device (output left in HBM until sync_to_host).
//  * numWorkers -> GPUs: a plan with numWorkers > 1 runs one y-slab per GPU.
#pragma once

#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <variant>
#include <vector>

#include "stengrid/grid.hpp"
#include "stengrid/worker_pool.hpp"

namespace stengrid {

/// stencil.hpp:12-18
struct WeightStencil {
  Extents ext;
  std::vector<double> weights;
};

/// stencil.hpp:20-25 — entry (p, q) of the window is window[q*rowStride + p].
using StencilFunction = double (*)(const double* window, const double* coe, int rowStride);

/// stencil.hpp:29-33
struct FunctionStencil {
  Extents ext;
  StencilFunction fn = nullptr;
  std::vector<double> coe;
};

enum class Direction { X, Y, XY };
enum class Residency { Host, Device };
using StencilKind = std::variant<WeightStencil, FunctionStencil>;

/// Host implementations of the reference's window functions (same arithmetic),
/// pre-registered with their device twins.
namespace functions {
inline double ch_nonlinear_window(const double* window, const double* coe, int rowStride) {
  double acc = 0.0;  // cahn_hilliard.cpp:36-47
  for (int q = 0; q < 3; ++q) {
    const double* row = window + static_cast<std::ptrdiff_t>(q) * rowStride;
    const double* cr = coe + q * 3;
    for (int p = 0; p < 3; ++p) {
      const double v = row[p];
      acc += cr[p] * (v * v * v - v);
    }
  }
  return acc;
}
inline double central_difference_window(const double* w, const double* coe, int) {
  return (w[0] - 2.0 * w[1] + w[2]) * coe[0];  // tools/main.cpp:47-49
}
inline double fn_center(const double* w, const double*, int rs) { return w[rs + 1]; }
inline double fn_central_second(const double* w, const double* coe, int) {
  double acc = 0.0;  // tests/test_stencil.cpp:70-77
  acc += coe[0] * w[0];
  acc += (-2.0 * coe[0]) * w[1];
  acc += coe[0] * w[2];
  return acc;
}
inline double fn_lap_cube_diff_first(const double* w, const double* coe, int rs) {
  auto g = [](double v) { return v * v * v - v; };  // tests/test_stencil.cpp:79-85
  const double gm = g(w[rs + 1]);
  const double x = (g(w[rs]) - 2.0 * gm) + g(w[rs + 2]);
  const double y = (g(w[1]) - 2.0 * gm) + g(w[2 * rs + 1]);
  return coe[0] * x + coe[1] * y;
}
inline double fn_weighted_3x3(const double* w, const double* coe, int rs) {
  double acc = 0.0;  // tests/test_stencil.cpp:88-93
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) acc += coe[q * 3 + p] * w[q * rs + p];
  return acc;
}
}  // namespace functions

namespace detail {
inline std::mutex& registry_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<StencilFunction, int>& registry() {
  static std::map<StencilFunction, int> r = {
      {&functions::ch_nonlinear_window, SG_FN_CH_NONLINEAR},
      {&functions::central_difference_window, SG_FN_CENTRAL_DIFFERENCE},
      {&functions::fn_center, SG_FN_CENTER},
      {&functions::fn_central_second, SG_FN_CENTRAL_SECOND},
      {&functions::fn_lap_cube_diff_first, SG_FN_LAP_CUBE_DIFF_FIRST},
      {&functions::fn_weighted_3x3, SG_FN_WEIGHTED_3X3},
  };
  return r;
}
}  // namespace detail

/// Map a host window function to a device twin (an sg_function id). The
/// caller asserts the two compute the same expression in the same order.
inline void register_device_function(StencilFunction hostFn, sg_function deviceFn) {
  if (hostFn == nullptr || deviceFn <= SG_FN_NONE || deviceFn >= SG_FN_COUNT)
    throw std::invalid_argument("register_device_function: bad arguments");
  std::lock_guard<std::mutex> lk(detail::registry_mutex());
  detail::registry()[hostFn] = deviceFn;
}

/// Extension — register a host window function together with its SOURCE:
/// `body` is the body of  T fn(const T* window, const T* coe, int rowStride)
/// (the same statements as the host function, T = double or float), which the
/// library compiles at run time (NVRTC, sm_100a, no FMA contraction) into its
/// stencil kernels (sg.h: sg_register_function_source). After this call
/// FunctionStencil{ext, hostFn, coe} runs on the GPU like the reference's own
/// functions; FP64 results equal the host function's bitwise when the body is
/// the same expression. Throws std::invalid_argument (with the compiler log)
/// if the body does not compile.
inline int register_device_function_source(StencilFunction hostFn, const std::string& body,
                                           const std::string& name = "user_function") {
  if (hostFn == nullptr) throw std::invalid_argument("register_device_function_source: null function");
  int id = -1;
  detail::check(sg_register_function_source(name.c_str(), body.c_str(), &id));
  std::lock_guard<std::mutex> lk(detail::registry_mutex());
  detail::registry()[hostFn] = id;
  return id;
}

inline int device_function_id(StencilFunction fn) {
  if (fn == nullptr) return -1;
  std::lock_guard<std::mutex> lk(detail::registry_mutex());
  auto it = detail::registry().find(fn);
  return it == detail::registry().end() ? -2 : it->second;
}

/// stencil.hpp:42-85 — movable, not copyable; never owns the fields.
/// BasicStencilPlan<double> is the reference's StencilPlan; the float
/// instantiation (StencilPlanF) binds Grid2Df fields and runs the FP32 kernels.
template <typename T>
class BasicStencilPlan;
namespace detail {
template <typename T>
void compute_impl(BasicStencilPlan<T>& plan, bool hostCoherent);
template <typename T>
struct dtype_of;
template <>
struct dtype_of<double> {
  static constexpr sg_dtype value = SG_F64;
};
template <>
struct dtype_of<float> {
  static constexpr sg_dtype value = SG_F32;
};
}  // namespace detail

template <typename T>
class BasicStencilPlan {
 public:
  using grid_type = BasicGrid2D<T>;
  BasicStencilPlan() = default;
  BasicStencilPlan(BasicStencilPlan&& o) noexcept { *this = std::move(o); }
  BasicStencilPlan& operator=(BasicStencilPlan&& o) noexcept {
    if (this != &o) {
      destroy();
      h_ = o.h_;
      o.h_ = nullptr;
      direction_ = o.direction_;
      mode_ = o.mode_;
      ext_ = o.ext_;
      kind_ = std::move(o.kind_);
      tiles_ = std::move(o.tiles_);
      input_ = o.input_;
      output_ = o.output_;
      numWorkers_ = o.numWorkers_;
      numTiles_ = o.numTiles_;
      fnId_ = o.fnId_;
      boundIn_ = o.boundIn_;
      boundOut_ = o.boundOut_;
      o.input_ = o.output_ = nullptr;
    }
    return *this;
  }
  BasicStencilPlan(const BasicStencilPlan&) = delete;
  BasicStencilPlan& operator=(const BasicStencilPlan&) = delete;
  ~BasicStencilPlan() { destroy(); }

  bool valid() const { return input_ != nullptr; }
  Direction direction() const { return direction_; }
  BoundaryMode mode() const { return mode_; }
  const Extents& extents() const { return ext_; }
  const TilePlan& tiles() const { return tiles_; }
  int num_workers() const { return numWorkers_; }
  const grid_type* input() const { return input_; }
  const grid_type* output() const { return output_; }

  /// stencil.cpp:186-193 — idempotent; never touches the grids.
  void destroy() {
    if (h_) sg_plan_destroy(&h_);
    h_ = nullptr;
    input_ = nullptr;
    output_ = nullptr;
    tiles_ = TilePlan{};
  }

  // Internals used by the free functions below (create_plan, swap_plan,
  // compute, sync_to_host); not part of the reference API.
  struct Access;

 private:
  friend struct Access;

  // (Re)bind the C plan to the grids' current host buffers.
  void bind() {
    if (h_) sg_plan_destroy(&h_);
    const double* vals = nullptr;
    size_t count = 0;
    if (const auto* ws = std::get_if<WeightStencil>(&kind_)) {
      vals = ws->weights.data();
      count = ws->weights.size();
    } else {
      const auto& fs = std::get<FunctionStencil>(kind_);
      vals = fs.coe.data();
      count = fs.coe.size();
    }
    const sg_extents e{ext_.left, ext_.right, ext_.top, ext_.bottom};
    detail::check(sg_plan_create(static_cast<sg_direction>(direction_),
                                 mode_ == BoundaryMode::Periodic ? SG_PERIODIC : SG_NONPERIODIC, e,
                                 static_cast<sg_function>(fnId_), vals, count, detail::dtype_of<T>::value,
                                 input_->data(), output_->data(), input_->nx, input_->ny, SG_MEM_HOST, numTiles_,
                                 numWorkers_, &h_));
    boundIn_ = input_->data();
    boundOut_ = output_->data();
  }

  sg_plan_t h_ = nullptr;
  Direction direction_ = Direction::X;
  BoundaryMode mode_ = BoundaryMode::Periodic;
  Extents ext_;
  StencilKind kind_;
  TilePlan tiles_;
  grid_type* input_ = nullptr;
  grid_type* output_ = nullptr;
  int numWorkers_ = 1;
  int numTiles_ = 1;
  int fnId_ = SG_FN_NONE;
  const T* boundIn_ = nullptr;
  const T* boundOut_ = nullptr;
};

template <typename T>
struct BasicStencilPlan<T>::Access {
  static sg_plan_t& handle(BasicStencilPlan& p) { return p.h_; }
  static void bind(BasicStencilPlan& p) { p.bind(); }
  static grid_type*& input(BasicStencilPlan& p) { return p.input_; }
  static grid_type*& output(BasicStencilPlan& p) { return p.output_; }
  static const T*& bound_in(BasicStencilPlan& p) { return p.boundIn_; }
  static const T*& bound_out(BasicStencilPlan& p) { return p.boundOut_; }
  static void init(BasicStencilPlan& p, Direction d, BoundaryMode m, StencilKind&& kind, grid_type& in,
                   grid_type& out, int numTiles, int numWorkers, int fnId) {
    p.direction_ = d;
    p.mode_ = m;
    p.ext_ = std::visit([](const auto& s) { return s.ext; }, kind);
    p.kind_ = std::move(kind);
    p.input_ = &in;
    p.output_ = &out;
    p.numWorkers_ = numWorkers;
    p.numTiles_ = numTiles;
    p.fnId_ = fnId;
  }
  static void set_tiles(BasicStencilPlan& p, TilePlan&& t) { p.tiles_ = std::move(t); }
};

using StencilPlan = BasicStencilPlan<double>;
using StencilPlanF = BasicStencilPlan<float>;

namespace detail {
template <typename T>
BasicStencilPlan<T> create_plan_impl(Direction direction, BoundaryMode mode, StencilKind kind, BasicGrid2D<T>& input,
                                     BasicGrid2D<T>& output, int numTiles, int numWorkers, WorkerPool* sharedPool) {
  using A = typename BasicStencilPlan<T>::Access;
  if (!input.same_shape(output)) throw std::invalid_argument("create_plan: input and output shapes differ");
  if (&input == &output || input.data() == output.data())
    throw std::invalid_argument("create_plan: input and output must be distinct buffers");
  int fnId = SG_FN_NONE;
  if (const auto* fs = std::get_if<FunctionStencil>(&kind)) {
    fnId = device_function_id(fs->fn);
    if (fnId == -2 && fs->ext.valid())
      throw std::invalid_argument(
          "create_plan: stencil function has no registered device twin (register_device_function)");
  }
  if (numWorkers >= 1 && sharedPool != nullptr && sharedPool->workers() != numWorkers)
    throw std::invalid_argument("create_plan: shared pool size does not match numWorkers");
  BasicStencilPlan<T> plan;
  // fnId -1: null function -> invalid_argument from the ABI
  A::init(plan, direction, mode, std::move(kind), input, output, numTiles, numWorkers, fnId < 0 ? -1 : fnId);
  try {
    A::bind(plan);  // full validation (stencil.cpp:128-161) happens in the C ABI
  } catch (...) {
    A::input(plan) = A::output(plan) = nullptr;
    throw;
  }
  A::set_tiles(plan, make_tiles(input.ny, numTiles, plan.extents()));
  return plan;
}
}  // namespace detail

/// stencil.hpp:90-92 / stencil.cpp:152-184.
inline StencilPlan create_plan(Direction direction, BoundaryMode mode, StencilKind kind, Grid2D& input,
                               Grid2D& output, int numTiles, int numWorkers,
                               WorkerPool* sharedPool = nullptr) {
  return detail::create_plan_impl<double>(direction, mode, std::move(kind), input, output, numTiles, numWorkers,
                                          sharedPool);
}

/// FP32 extension: the same plan over float fields (weights / coefficients
/// are given in double, as in the reference's kinds, and rounded to float on
/// the device path; FunctionStencil's fn selects the device twin, which
/// evaluates the same expression in float).
inline StencilPlanF create_plan(Direction direction, BoundaryMode mode, StencilKind kind, Grid2Df& input,
                                Grid2Df& output, int numTiles, int numWorkers,
                                WorkerPool* sharedPool = nullptr) {
  return detail::create_plan_impl<float>(direction, mode, std::move(kind), input, output, numTiles, numWorkers,
                                         sharedPool);
}

template <typename T>
inline void destroy_plan(BasicStencilPlan<T>& plan) {
  plan.destroy();
}

/// stencil.cpp:197-200
template <typename T>
inline void swap_plan(BasicStencilPlan<T>& plan) {
  using A = typename BasicStencilPlan<T>::Access;
  if (!plan.valid()) throw std::logic_error("swap_plan: plan was destroyed");
  detail::check(sg_plan_swap(A::handle(plan)));
  std::swap(A::input(plan), A::output(plan));
  std::swap(A::bound_in(plan), A::bound_out(plan));
}

/// stencil.cpp:202-235 — runs on the GPU, synchronous and host-coherent for
/// BOTH hints: on return the bound output Grid2D holds the result, exactly
/// as in the reference, where the residency hint is a no-op
/// (stencil.cpp:202). A numWorkers > 1 plan runs one y-slab per GPU
/// (sg.h: sg_set_device_map).
template <typename T>
inline void compute(BasicStencilPlan<T>& plan, Residency hint = Residency::Host) {
  (void)hint;
  detail::compute_impl(plan, true);
}

/// Extension — the paper's Residency::Device: returns once
/// the kernel is queued and leaves the output in HBM, so chains of
/// compute_deferred / swap_plan never wait on the host or move the grids
/// over PCIe. The bound host output is stale until sync_to_host(plan) (or a
/// later compute()); do not modify the bound host grids in between.
template <typename T>
inline void compute_deferred(BasicStencilPlan<T>& plan) {
  detail::compute_impl(plan, false);
}

/// Bring compute_deferred results back into the bound host grids.
template <typename T>
inline void sync_to_host(BasicStencilPlan<T>& plan) {
  using A = typename BasicStencilPlan<T>::Access;
  if (!plan.valid()) throw std::logic_error("sync_to_host: plan was destroyed");
  detail::check(sg_plan_sync_to_host(A::handle(plan)));
}

namespace detail {
template <typename T>
void compute_impl(BasicStencilPlan<T>& plan, bool hostCoherent) {
  using A = typename BasicStencilPlan<T>::Access;
  if (!plan.valid()) throw std::logic_error("compute: plan was destroyed");
  BasicGrid2D<T>& in = *A::input(plan);
  BasicGrid2D<T>& out = *A::output(plan);
  if (!in.same_shape(out)) throw std::invalid_argument("compute: bound grids changed shape");
  if (in.data() == out.data()) throw std::invalid_argument("compute: bound grids alias");
  if (in.data() != A::bound_in(plan) || out.data() != A::bound_out(plan)) A::bind(plan);  // storage moved
  detail::check(sg_plan_compute(A::handle(plan), hostCoherent ? SG_RESIDENCY_HOST : SG_RESIDENCY_DEVICE, nullptr,
                                hostCoherent ? 1 : 0));
}
}  // namespace detail

/// stencil.cpp:237-260 — single-point evaluation (host; used as a checker).
inline double apply_weights_at(const Grid2D& input, const WeightStencil& sten, int i, int j,
                               BoundaryMode mode) {
  const Extents& e = sten.ext;
  const int W = e.width(), H = e.height();
  const double* w = sten.weights.data();
  const double* v = input.data();
  double acc = 0.0;
  for (int q = 0; q < H; ++q) {
    const int jj = mode == BoundaryMode::Periodic ? wrap(j - e.top + q, input.ny) : j - e.top + q;
    const std::ptrdiff_t base = static_cast<std::ptrdiff_t>(jj) * input.nx;
    for (int p = 0; p < W; ++p) {
      const int ii = mode == BoundaryMode::Periodic ? wrap(i - e.left + p, input.nx) : i - e.left + p;
      acc += w[q * W + p] * v[base + ii];
    }
  }
  return acc;
}

/// stencil.cpp:262-286
inline double apply_function_at(const Grid2D& input, const FunctionStencil& sten, int i, int j,
                                BoundaryMode mode) {
  const Extents& e = sten.ext;
  const int W = e.width(), H = e.height();
  std::vector<double> window(static_cast<std::size_t>(W) * H);
  for (int q = 0; q < H; ++q) {
    const int jj = mode == BoundaryMode::Periodic ? wrap(j - e.top + q, input.ny) : j - e.top + q;
    for (int p = 0; p < W; ++p) {
      const int ii = mode == BoundaryMode::Periodic ? wrap(i - e.left + p, input.nx) : i - e.left + p;
      window[static_cast<std::size_t>(q) * W + p] = input(ii, jj);
    }
  }
  return sten.fn(window.data(), sten.coe.data(), W);
}

}  // namespace stengrid
