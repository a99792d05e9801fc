// stencil_g.cuh — k_tma_g, the general-shape / general-alignment member of
// the TMA-staged stencil family (stencil.cu has the design notes of k_tma).
// Included by stencil_g64.cu and stencil_g32.cu with SG_G_T = double / float
// (two translation units: the 81 window shapes compile in parallel).
//
// The reference serves every window with one loop nest (weights_rows /
// function_rows, stencil.cpp:61-126), asymmetric ones included
// (tests/test_stencil.cpp:557-568). k_tma covers symmetric windows on
// 16 B-aligned rows; k_tma_g covers everything else up to 9 x 9:
//  * any split of the window: W = left + right + 1 and H = top + bottom + 1
//    are template parameters, left and top are runtime. The register ring of
//    H rows depends on H alone (output row j completes when input row
//    j + bottom arrives), so the vertical split only moves the producer's
//    first row; the horizontal split moves each lane's window start in the
//    staged row (window columns are read with scalar shared loads);
//  * any row pitch and any element-aligned pointers (nx % V != 0, e.g. odd
//    grids): a staged row keeps the 16 B phase of its global address — input
//    row r, column c sits at srow[HP + ph(r) + c - cx0] with
//    ph(r) = (in + r*nx) mod V elements — so the aligned middle of the row
//    still moves as ONE bulk copy (cp.async.bulk) and only the unaligned
//    head/tail elements and the halo columns use 4/8 B cp.async;
//  * outputs are stored as 16 B vectors where the output row is 16 B
//    aligned, element by element otherwise.
// Arithmetic per output is k_tma's: acc = 0; acc += w[q*W+p] * x row-major,
// or Op::apply(window, coe, W) — bitwise the reference's.
#pragma once

#include "stencil_kern.cuh"

namespace sg {
namespace {

template <typename T, int W, int H, typename Op>
void launch_g_wh(const KArgs<T>& a, cudaStream_t s) {
  using G = TmaGGeom<T, W, H>;
  auto kern = k_tma_g<T, W, H, Op>;
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

// Weight windows: every W x H up to 9 x 9 (runtime dispatch over the 81
// instantiations).
template <typename T, int W>
void launch_g_w(const KArgs<T>& a, int H, cudaStream_t s) {
  switch (H) {
    case 1: return launch_g_wh<T, W, 1, OpWeights>(a, s);
    case 2: return launch_g_wh<T, W, 2, OpWeights>(a, s);
    case 3: return launch_g_wh<T, W, 3, OpWeights>(a, s);
    case 4: return launch_g_wh<T, W, 4, OpWeights>(a, s);
    case 5: return launch_g_wh<T, W, 5, OpWeights>(a, s);
    case 6: return launch_g_wh<T, W, 6, OpWeights>(a, s);
    case 7: return launch_g_wh<T, W, 7, OpWeights>(a, s);
    case 8: return launch_g_wh<T, W, 8, OpWeights>(a, s);
    case 9: return launch_g_wh<T, W, 9, OpWeights>(a, s);
    default: invalid("internal: k_tma_g window height");
  }
}

template <typename T>
void launch_g(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values, size_t count,
              const void* in, void* out, cudaStream_t s, const PeerRows& peers) {
  const KArgs<T> a = make_args<T>(d, e, values, count, in, out, peers);
  const int W = e.left + e.right + 1, H = e.top + e.bottom + 1;
  if (fn == SG_FN_NONE) {
    switch (W) {
      case 1: return launch_g_w<T, 1>(a, H, s);
      case 2: return launch_g_w<T, 2>(a, H, s);
      case 3: return launch_g_w<T, 3>(a, H, s);
      case 4: return launch_g_w<T, 4>(a, H, s);
      case 5: return launch_g_w<T, 5>(a, H, s);
      case 6: return launch_g_w<T, 6>(a, H, s);
      case 7: return launch_g_w<T, 7>(a, H, s);
      case 8: return launch_g_w<T, 8>(a, H, s);
      case 9: return launch_g_w<T, 9>(a, H, s);
      default: invalid("internal: k_tma_g window width");
    }
  }
  // device functions on their natural windows (3 x 3, or 3 x 1)
  bool ok = with_op<void>(fn, [&](auto op) {
    using Op = decltype(op);
    if constexpr (std::is_same_v<Op, OpCentralDifference> || std::is_same_v<Op, OpCentralSecond>)
      launch_g_wh<T, 3, 1, Op>(a, s);
    else if constexpr (!std::is_same_v<Op, OpWeights>)
      launch_g_wh<T, 3, 3, Op>(a, s);
  });
  if (!ok) invalid("internal: k_tma_g function");
}

}  // namespace
}  // namespace sg
