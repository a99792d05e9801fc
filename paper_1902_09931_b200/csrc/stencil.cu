// stencil.cu — sm_100a stencil kernels for the cuSten/stengrid engine.
//
// Replaces the reference's CPU hot loops weights_rows / weights_wrapped_point
// (stencil.cpp:49-85) and function_rows / function_gathered_point
// (stencil.cpp:87-126). Arithmetic is bitwise identical to the reference:
// each output is acc = 0; acc += w[q*W+p] * in(i-left+p, j-top+q) row-major
// over the window (compiled with --fmad=false, the device analogue of the
// reference's -ffp-contract=off, CMakeLists.txt:15-21); function stencils
// receive the window packed with rowStride = W, which the reference's
// contract allows (stencil.hpp:20-25).
//
// Three kernels:
//  * k_tma — the bandwidth path for symmetric windows (extents <= 4 a side)
//    on 16 B-aligned rows: TMA-staged shared-memory row ring, one producer
//    warp, 16 consumer warps holding the window in registers.
//  * k_tma_g — the same pipeline for every other window up to 9 x 9
//    (asymmetric left/right and top/bottom splits) and every row pitch /
//    pointer alignment (nx % V != 0): rows keep their global 16 B phase in
//    shared memory.
//  * k_generic — windows beyond 9 x 9 and device functions on non-natural
//    windows: a shared-memory input tile per 32 x 32 outputs (one thread per
//    point from global memory when the tile would not fit).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "sg_internal.hpp"
#include "stencil_kern.cuh"

namespace sg {

std::atomic<uint64_t> g_launches{0};

namespace {

// -------------------------------------------------------------- dispatch
struct FnInfo {
  const char* name;
  int minW, minH, minCoe;
};
constexpr FnInfo kFn[SG_FN_COUNT] = {
    {"weights", 1, 1, 0},
    {"ch_nonlinear_window", 3, 3, 9},
    {"central_difference_window", 3, 1, 1},
    {"fn_center", 2, 2, 0},
    {"fn_central_second", 3, 1, 1},
    {"fn_lap_cube_diff_first", 3, 3, 2},
    {"fn_weighted_3x3", 3, 3, 9},
};

// Natural window of a device function (the shape its reference test uses);
// the pipelined kernels serve functions on their natural window only.
bool fn_natural(const sg_extents& e, int fn) {
  if (fn == SG_FN_CENTRAL_DIFFERENCE || fn == SG_FN_CENTRAL_SECOND)
    return e.left == 1 && e.right == 1 && e.top == 0 && e.bottom == 0;
  return e.left == 1 && e.right == 1 && e.top == 1 && e.bottom == 1;
}

// k_tma: symmetric weight windows up to 4 a side, natural function windows.
bool strip_supported(const sg_extents& e, int fn) {
  if (fn != SG_FN_NONE) return fn_natural(e, fn);
  return e.left == e.right && e.top == e.bottom && e.left <= 4 && e.top <= 4;
}

// k_tma_g: any weight window up to 9 x 9, natural function windows.
bool general_supported(const sg_extents& e, int fn) {
  if (fn != SG_FN_NONE) return fn_natural(e, fn);
  return e.left + e.right + 1 <= TMA_G_MAXW && e.top + e.bottom + 1 <= TMA_G_MAXW;
}

// 2 = k_tma_g, 1 = k_tma, 0 = k_generic
template <typename T>
int kernel_kind(const sg_slab_desc& d, const sg_extents& e, int fn, size_t count, const void* in,
                const void* out) {
  constexpr int V = VecT<T>::V;
  if (count > static_cast<size_t>(VMAX)) return 0;
  const uintptr_t pin = reinterpret_cast<uintptr_t>(in), pout = reinterpret_cast<uintptr_t>(out);
  const bool aligned = d.nx % V == 0 && (pin | pout) % 16 == 0;
  // SG_STENCIL_KIND=g (experiments): route k_tma's cases to k_tma_g
  static const bool forceG = [] {
    const char* v = std::getenv("SG_STENCIL_KIND");
    return v && v[0] == 'g';
  }();
  if (aligned && strip_supported(e, fn) && !(forceG && general_supported(e, fn))) return 1;
  if ((pin | pout) % sizeof(T) == 0 && general_supported(e, fn)) return 2;
  return 0;
}

template <typename T, int L, int TP, typename Op>
void launch_tma_lt(const KArgs<T>& a, cudaStream_t s) {
  using G = TmaGeom<T, L, L, TP, TP>;
  auto kern = k_tma<T, L, L, TP, TP, Op>;
  static int ctasPerSm = 0;  // per instantiation
  if (ctasPerSm == 0) {
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(G::smem_bytes)));
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctasPerSm, kern, (G::NW + 1) * 32, G::smem_bytes));
    if (ctasPerSm < 1) ctasPerSm = 1;
  }
  const int gx = (a.nx + G::CW - 1) / G::CW;
  const int rows = a.row1 - a.row0;
  KArgs<T> b = a;
  b.segRows = tma_segment_rows(rows, gx, ctasPerSm, G::RPS);
  dim3 g2(gx, static_cast<unsigned>((rows + b.segRows - 1) / b.segRows));
  launch_ex(kern, g2, dim3((G::NW + 1) * 32), G::smem_bytes, s, stencil_pdl(), b);
}

template <typename T, typename Op>
void launch_tma(const KArgs<T>& a, const sg_extents& e, cudaStream_t s) {
#define SG_CASE(LV, TV) \
  if (e.left == LV && e.top == TV) return launch_tma_lt<T, LV, TV, Op>(a, s);
  if constexpr (std::is_same_v<Op, OpWeights>) {
    SG_CASE(0, 0) SG_CASE(1, 0) SG_CASE(2, 0) SG_CASE(3, 0) SG_CASE(4, 0)
    SG_CASE(0, 1) SG_CASE(1, 1) SG_CASE(2, 1) SG_CASE(3, 1) SG_CASE(4, 1)
    SG_CASE(0, 2) SG_CASE(1, 2) SG_CASE(2, 2) SG_CASE(3, 2) SG_CASE(4, 2)
    SG_CASE(0, 3) SG_CASE(1, 3) SG_CASE(2, 3) SG_CASE(3, 3) SG_CASE(4, 3)
    SG_CASE(0, 4) SG_CASE(1, 4) SG_CASE(2, 4) SG_CASE(3, 4) SG_CASE(4, 4)
  } else if constexpr (std::is_same_v<Op, OpCentralDifference> ||
                       std::is_same_v<Op, OpCentralSecond>) {
    SG_CASE(1, 0)
  } else {
    SG_CASE(1, 1)
  }
#undef SG_CASE
  invalid("internal: no k_tma instantiation for these extents");
}

template <typename T>
int launch_typed(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values,
                 size_t count, const void* in, void* out, cudaStream_t s, const PeerRows& peers) {
  const int rows = d.row1 - d.row0;
  const int cols = d.col1 - d.col0;
  const int kind = kernel_kind<T>(d, e, fn, count, in, out);
  if (rows <= 0 || cols <= 0) return kind;
  if (kind == 2) {
    if constexpr (std::is_same_v<T, double>)
      launch_stencil_g_f64(d, e, fn, values, count, in, out, s, peers);
    else
      launch_stencil_g_f32(d, e, fn, values, count, in, out, s, peers);
    check_launch("stencil k_tma_g kernel");
    return 2;
  }
  KArgs<T> a = make_args<T>(d, e, values, count, in, out, peers);
  if (kind == 1) {
    with_op<void>(fn, [&](auto op) { launch_tma<T, decltype(op)>(a, e, s); });
    check_launch("stencil k_tma kernel");
    return 1;
  }

  T* wtmp = nullptr;
  if (fn == SG_FN_NONE && count > static_cast<size_t>(VMAX)) {
    retain_async_pool();
    SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wtmp), count * sizeof(T), s));
    T* hw = new T[count];
    for (size_t k = 0; k < count; ++k) hw[k] = static_cast<T>(values[k]);
    cudaError_t err = cudaMemcpyAsync(wtmp, hw, count * sizeof(T), cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    delete[] hw;
    SG_CUDA(err);
    a.wdev = wtmp;
  }
  dim3 block(32, 8);
  const bool weights = fn == SG_FN_NONE;
  const size_t tileB = generic_tile_bytes<T>(e, weights);
  a.gtile = tileB > 0 ? 1 : 0;
  const int gw = tileB > 0 ? generic_tile_cols(weights) : 32;
  dim3 grid((cols + gw - 1) / gw, tileB > 0 ? (rows + 31) / 32 : (rows + 7) / 8);
  if (weights && tileB > (48u << 10)) {
    static const cudaError_t optin =  // once per T (thread-safe static init)
        cudaFuncSetAttribute(k_generic<T, OpWeights>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(SG_GENERIC_SMEM));
    SG_CUDA(optin);
  }
  with_op<void>(fn, [&](auto op) { k_generic<T, decltype(op)><<<grid, block, tileB, s>>>(a); });
  check_launch("stencil generic kernel");
  if (wtmp) SG_CUDA(cudaFreeAsync(wtmp, s));
  return 0;
}

}  // namespace

bool function_shape(int fn, int* minW, int* minH, int* minCoe) {
  if (jit_function(fn, nullptr)) {  // source functions: any window (the user's contract)
    *minW = *minH = 1;
    *minCoe = 0;
    return true;
  }
  if (fn < 0 || fn >= SG_FN_COUNT) return false;
  *minW = kFn[fn].minW;
  *minH = kFn[fn].minH;
  *minCoe = kFn[fn].minCoe;
  return true;
}

const char* function_name(int fn) {
  if (fn >= SG_FN_JIT_BASE) return jit_function_name(fn);
  return (fn >= 0 && fn < SG_FN_COUNT) ? kFn[fn].name : nullptr;
}

int stencil_kernel_kind(const sg_slab_desc& d, const sg_extents& e, int fn, size_t count,
                        sg_dtype dtype, const void* in, const void* out) {
  if (fn >= SG_FN_JIT_BASE)
    return launch_stencil_jit(d, e, fn, nullptr, count, dtype, in, const_cast<void*>(out), nullptr, PeerRows{}, false);
  return dtype == SG_F64 ? kernel_kind<double>(d, e, fn, count, in, out)
                         : kernel_kind<float>(d, e, fn, count, in, out);
}

int launch_stencil(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values,
                   size_t count, sg_dtype dtype, const void* in, void* out, cudaStream_t stream,
                   const PeerRows& peers) {
  if (fn >= SG_FN_JIT_BASE)
    return launch_stencil_jit(d, e, fn, values, count, dtype, in, out, stream, peers, true);
  if (fn != SG_FN_NONE && (e.left + e.right + 1) * (e.top + e.bottom + 1) > GENERIC_FN_MAX &&
      !general_supported(e, fn))
    invalid("create_plan: device function windows are limited to 256 taps");
  if (dtype == SG_F64) return launch_typed<double>(d, e, fn, values, count, in, out, stream, peers);
  if (dtype == SG_F32) return launch_typed<float>(d, e, fn, values, count, in, out, stream, peers);
  invalid("unknown dtype");
}

}  // namespace sg
