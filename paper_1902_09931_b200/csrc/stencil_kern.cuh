// stencil_kern.cuh — kernel-side definitions shared by the stencil
// translation units (stencil.cu: k_tma, k_generic, dispatch;
// stencil_g64.cu / stencil_g32.cu: k_tma_g). Everything here has internal
// linkage (anonymous namespace): each translation unit instantiates its own
// kernels. See stencil.cu for the design notes.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "sg_internal.hpp"
#include "stencil_dev.cuh"

namespace sg {
namespace {

// Kernel arguments of one slab launch (plain descriptor -> KArgs).
template <typename T>
KArgs<T> make_args(const sg_slab_desc& d, const sg_extents& e, const double* values, size_t count,
                   const void* in, void* out, const PeerRows& peers) {
  KArgs<T> a;
  std::memset(static_cast<void*>(&a), 0, sizeof(a));
  a.in = static_cast<const T*>(in);
  a.out = static_cast<T*>(out);
  a.wdev = nullptr;
  a.nx = d.nx;
  a.inRows = d.inRows;
  a.inShift = d.inShift;
  a.row0 = d.row0;
  a.row1 = d.row1;
  a.col0 = d.col0;
  a.col1 = d.col1;
  a.wrapX = d.wrapX;
  a.wrapY = d.wrapY;
  a.left = e.left;
  a.right = e.right;
  a.top = e.top;
  a.bottom = e.bottom;
  a.count = static_cast<int>(count);
  a.peerUp = static_cast<T*>(peers.up);
  a.peerDn = static_cast<T*>(peers.dn);
  a.upRows = peers.upRows;
  a.dnRow0 = peers.dnRow0;
  const size_t nv = std::min(count, static_cast<size_t>(VMAX));
  for (size_t k = 0; k < nv; ++k) a.v[k] = static_cast<T>(values[k]);
  return a;
}

// Stencil launches as programmatic dependents of the previous kernel on the
// stream (the kernels wait before any global access): back-to-back
// applications overlap launch and prologue with the predecessor's tail.
// SG_STENCIL_PDL=0 disables (A/B).
inline bool stencil_pdl() {
  static const bool v = [] {
    const char* e = std::getenv("SG_STENCIL_PDL");
    return !(e && e[0] == '0') && pdl_enabled();
  }();
  return v;
}

// k_generic's staged input tile (GW + W - 1) x (32 + H - 1) in bytes, or 0
// when it would exceed the limit (taps are then read from global memory); GW
// = generic_tile_cols: 32 x SG_GENERIC_NC output columns per CTA for weight
// windows (SG_GENERIC_NC per thread), 32 for functions. Weight tiles may use
// up to SG_GENERIC_SMEM (the launcher opts in), function tiles 48 KB (the
// NVRTC path launches them without the opt-in).
inline int generic_tile_cols(bool weights) { return weights && SG_GENERIC_ROWS4 ? 32 * SG_GENERIC_NC : 32; }
template <typename T>
size_t generic_tile_bytes(const sg_extents& e, bool weights = false) {
  const size_t b = static_cast<size_t>(generic_tile_cols(weights) + e.left + e.right) * (32 + e.top + e.bottom) *
                   sizeof(T);
  const size_t lim = weights ? static_cast<size_t>(SG_GENERIC_SMEM) : (48u << 10);
  return b <= lim ? b : 0;
}

inline int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Row segments of a TMA-pipelined launch: one wave of CTAs when the grid is
// small (each CTA's pipeline start-up is then paid once), <= 512-row
// segments (several waves) when it is large.
inline int tma_segment_rows(int rows, int gx, int ctasPerSm, int rps) {
  const long long cap = 1LL * sm_count() * ctasPerSm;
  long long seg = (1LL * rows * gx + cap - 1) / cap;
  seg = std::max<long long>(seg, std::min(rows, 2 * rps));
  seg = std::min<long long>(seg, 512);
  // rounding up twice (rows per segment, then segments per column) can
  // leave a handful of CTAs past the last full wave (16384^2 FP32 3x3:
  // 9 x 33 = 297 CTAs on 296 slots, the 297th running its 499 rows alone);
  // take the segment length with the fewest waves x rows per CTA
  auto cost = [&](long long s) {
    const long long ctas = 1LL * gx * ((rows + s - 1) / s);
    return ((ctas + cap - 1) / cap) * s;
  };
  long long best = seg;
  for (long long s = seg + 1; s <= std::min<long long>(rows, seg + seg / 4 + 1); ++s)
    if (cost(s) < cost(best)) best = s;
  return static_cast<int>(best);
}

template <typename Op, typename F>
bool with_op(int fn, F&& f) {
  switch (fn) {
    case SG_FN_NONE: f(OpWeights{}); return true;
    case SG_FN_CH_NONLINEAR: f(OpChNonlinear{}); return true;
    case SG_FN_CENTRAL_DIFFERENCE: f(OpCentralDifference{}); return true;
    case SG_FN_CENTER: f(OpCenter{}); return true;
    case SG_FN_CENTRAL_SECOND: f(OpCentralSecond{}); return true;
    case SG_FN_LAP_CUBE_DIFF_FIRST: f(OpLapCubeDiffFirst{}); return true;
    case SG_FN_WEIGHTED_3X3: f(OpWeighted3x3{}); return true;
    default: return false;
  }
}

}  // namespace
}  // namespace sg
