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

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(sizeof(T))
               : "memory");
}

template <typename T, int W, int H>
struct TmaGGeom {
  static constexpr int V = VecT<T>::V;
  static constexpr int SW = 32 * V;
  static constexpr int CW = TMA_WARPS * SW;
  static constexpr int HP = ((W - 1 + V - 1) / V) * V;  // halo room either side (any split of W - 1)
  static constexpr int ROW = HP + CW + V + HP;          // + V: the row's 16 B phase
  static constexpr int RPS = H >= 2 ? H : 2;
  static constexpr int STAGES = (9 + RPS - 1) / RPS >= 2 ? (9 + RPS - 1) / RPS : 2;
  static constexpr size_t stage_bytes = static_cast<size_t>(RPS) * ROW * sizeof(T);
  static constexpr size_t smem_bytes = STAGES * stage_bytes + 2 * STAGES * sizeof(uint64_t);
};

// Source row of the t-th staged row of a CTA: rows wrap (periodic y) or
// clamp to the grid (rows past a non-periodic edge feed only outputs that
// are never stored).
struct RowWalk {
  long long r;  // unclamped row of the next staged row
  int cur;      // its source row
  __device__ void init(long long r0, int inRows, int wrapY) {
    r = r0;
    cur = wrapY ? wrap_idx(r0, inRows) : static_cast<int>(r0 < 0 ? 0 : (r0 >= inRows ? inRows - 1 : r0));
  }
  __device__ void next(int inRows, int wrapY) {
    ++r;
    if (wrapY) {
      cur = cur + 1 == inRows ? 0 : cur + 1;
    } else {
      cur = static_cast<int>(r < 0 ? 0 : (r >= inRows ? inRows - 1 : r));
    }
  }
};

// CTAs per SM the register allocation is sized for (launch bounds): two
// for narrow windows (W <= 3, H <= 6: spill-free in 56 registers) where two
// rings fit in shared memory, else one (the compiler's choice). Measured at
// 16384^2 FP64 (scripts/exp/stencil_shapes.py, A/B of whole builds): 3x3 on
// odd rows 0.59 -> 0.83 of HBM, 1x5 odd 0.76 -> 0.91; wider windows lost
// 4-13 % with two (spills / fewer registers for the FP64 chains).
// SG_TMAG_MINB2=1 forces two wherever the rings fit, =0 one everywhere.
#ifndef SG_TMAG_MINB2
#define SG_TMAG_MINB2 -1
#endif
template <typename T, int W, int H>
constexpr int tmag_min_blocks() {
  constexpr bool fits2 = 2 * TmaGGeom<T, W, H>::smem_bytes <= 227 * 1024;
  if (SG_TMAG_MINB2 == 0 || !fits2) return 1;
  if (SG_TMAG_MINB2 == 1) return 2;
  return W <= 3 && H <= 6 ? 2 : 1;
}

template <typename T, int W, int H, typename Op>
__global__ void __launch_bounds__((TMA_WARPS + 1) * 32, (tmag_min_blocks<T, W, H>())) k_tma_g(const __grid_constant__ KArgs<T> a) {
  using G = TmaGGeom<T, W, H>;
  using VT = typename VecT<T>::type;
  constexpr int V = G::V, SW = G::SW, CW = G::CW, HP = G::HP, ROW = G::ROW;
  constexpr int RPS = G::RPS, STAGES = G::STAGES;
  constexpr int E = W - 1 + V;  // window columns of a lane's V outputs
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * G::stage_bytes);
  uint64_t* empty = full + STAGES;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nx = a.nx;
  const int cx0 = blockIdx.x * CW;
  const int ra = a.row0 + blockIdx.y * a.segRows;
  const int rb = min(ra + a.segRows, a.row1);
  if (ra >= rb) return;  // CTA-uniform
  const int nIn = (rb - ra) + H - 1;
  const int nStages = (nIn + RPS - 1) / RPS;
  // element phase of global row r: (in + r*nx) mod V (low bits only)
  const unsigned inOff = static_cast<unsigned>(reinterpret_cast<uintptr_t>(a.in) / sizeof(T));
  const unsigned unx = static_cast<unsigned>(nx);
  const long long r0 = static_cast<long long>(ra) + a.inShift - a.top;

  if (threadIdx.x == 0) {
    for (int k = 0; k < STAGES; ++k) {
      mbar_init(&full[k], 2);  // expect_tx arrival + cp.async arrival
      mbar_init(&empty[k], TMA_WARPS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == TMA_WARPS) {
    // ---------------- producer (lane 0): per row, the 16 B-aligned middle
    // of the CTA's columns as one bulk copy, head/tail elements and halo
    // columns (wrapped in index math) as element cp.async
    if (lane != 0) return;
    const int validC = min(CW, nx - cx0);
    const int l = a.left, r = a.right;
    const T* __restrict__ in = a.in;
    RowWalk rw;
    rw.init(r0, a.inRows, a.wrapY);
    for (int g = 0; g < nStages; ++g) {
      const int slot = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[slot], ((g / STAGES) + 1) & 1);
      int src[RPS];
      uint32_t tx = 0;
      RowWalk w2 = rw;
#pragma unroll
      for (int k = 0; k < RPS; ++k) {
        src[k] = w2.cur;
        const int ph = static_cast<int>((inOff + static_cast<unsigned>(w2.cur) * unx) & (V - 1));
        const int head = ph ? min(V - ph, validC) : 0;
        tx += static_cast<uint32_t>(((validC - head) / V) * V * sizeof(T));
        w2.next(a.inRows, a.wrapY);
      }
      if (tx) mbar_expect_tx(&full[slot], tx);
      else mbar_arrive(&full[slot]);
      T* sstage = ring + slot * (RPS * ROW);
#pragma unroll
      for (int k = 0; k < RPS; ++k) {
        const T* grow = in + static_cast<long long>(src[k]) * nx;
        const int ph = static_cast<int>((inOff + static_cast<unsigned>(src[k]) * unx) & (V - 1));
        T* srow = sstage + k * ROW + HP + ph;  // column cx0 of this row
        const int head = ph ? min(V - ph, validC) : 0;
        const int mid = ((validC - head) / V) * V;
        for (int t = 0; t < head; ++t) cp_async_elem(srow + t, grow + cx0 + t);
        if (mid) bulk_g2s(srow + head, grow + cx0 + head, static_cast<uint32_t>(mid * sizeof(T)), &full[slot]);
        for (int t = head + mid; t < validC; ++t) cp_async_elem(srow + t, grow + cx0 + t);
        for (int p = 1; p <= l; ++p) {
          const int c = cx0 - p;
          if (c >= 0) cp_async_elem(srow - p, grow + c);
          else if (a.wrapX) cp_async_elem(srow - p, grow + c + nx);
        }
        for (int p = 0; p < r; ++p) {
          const int c = cx0 + validC + p;
          if (c < nx) cp_async_elem(srow + validC + p, grow + c);
          else if (a.wrapX) cp_async_elem(srow + validC + p, grow + c - nx);
        }
      }
      rw = w2;
      cp_async_mbar_arrive(&full[slot]);
    }
    return;
  }

  // ---------------- consumers
  const int xo = warp * SW + lane * V;  // lane's first output column - cx0
  const int xb = cx0 + xo;
  const bool laneValid = xb < nx;
  const bool laneFull = laneValid && xb >= a.col0 && xb + V <= a.col1;
  const unsigned outOff = static_cast<unsigned>(reinterpret_cast<uintptr_t>(a.out) / sizeof(T));
  const bool peers = a.peerUp != nullptr || a.peerDn != nullptr;
  const bool peerVec = nx % V == 0;  // peer rows share the output rows' phase only then
  constexpr bool ACC = std::is_same_v<Op, OpWeights> && H >= 5;
  T win[ACC ? 1 : H][E];   // ring: input row t lives in win[t % H]
  T pend[ACC ? H : 1][V];  // ACC: output started at local input row u lives in pend[u % H]
  RowWalk rw;
  rw.init(r0, a.inRows, a.wrapY);
  int j = ra - (H - 1);  // output row completed by the current input row
  for (int g = 0; g < nStages; ++g) {
    const int slot = g % STAGES;
    mbar_wait(&full[slot], (g / STAGES) & 1);
    const T* sbase = ring + slot * (RPS * ROW) + HP + xo - a.left;
#pragma unroll
    for (int k = 0; k < RPS; ++k) {
      const int ph = static_cast<int>((inOff + static_cast<unsigned>(rw.cur) * unx) & (V - 1));
      rw.next(a.inRows, a.wrapY);
      const T* srow = sbase + k * ROW + ph;  // window column 0 of the lane's first output
      T* e = win[ACC ? 0 : k % H];
#pragma unroll
      for (int p = 0; p < E; ++p) e[p] = srow[p];
      T res[V];
      if constexpr (ACC) {
#pragma unroll
        for (int q = 0; q < H; ++q) {
          T* acc = pend[((k - q) % H + H) % H];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (q == 0) acc[v] = T(0);
#pragma unroll
            for (int p = 0; p < W; ++p) acc[v] += a.v[q * W + p] * e[v + p];
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = pend[(k + 1) % H][v];
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if constexpr (std::is_same_v<Op, OpWeights>) {
            T acc = T(0);
#pragma unroll
            for (int q = 0; q < H; ++q)
#pragma unroll
              for (int p = 0; p < W; ++p) acc += a.v[q * W + p] * win[(k + 1 + q) % H][v + p];
            res[v] = acc;
          } else {
            T w[H * W];
#pragma unroll
            for (int q = 0; q < H; ++q)
#pragma unroll
              for (int p = 0; p < W; ++p) w[q * W + p] = win[(k + 1 + q) % H][v + p];
            res[v] = Op::template apply<T>(w, a.v, W);
          }
        }
      }
      if (j >= ra && j < rb) {  // warp-uniform
        const long long jo = static_cast<long long>(j) * nx;
        const bool rowVec = ((outOff + static_cast<unsigned>(j) * unx) & (V - 1)) == 0;
        if (laneFull && rowVec && (!peers || peerVec)) {
          VT o;
          if constexpr (V == 2) {
            o.x = res[0];
            o.y = res[1];
          } else {
            o.x = res[0];
            o.y = res[1];
            o.z = res[2];
            o.w = res[3];
          }
          *reinterpret_cast<VT*>(a.out + jo + xb) = o;
          if (a.peerUp && j < a.upRows) *reinterpret_cast<VT*>(a.peerUp + jo + xb) = o;
          if (a.peerDn && j >= a.dnRow0)
            *reinterpret_cast<VT*>(a.peerDn + static_cast<long long>(j - a.dnRow0) * nx + xb) = o;
        } else if (laneValid) {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (xb + v >= a.col0 && xb + v < a.col1) put_out(a, j, xb + v, res[v]);
        }
      }
      ++j;
    }
    mbar_arrive(&empty[slot]);  // each thread releases its own reads of the slot
  }
}

template <typename T, int W, int H, typename Op>
void launch_g_wh(const KArgs<T>& a, cudaStream_t s) {
  using G = TmaGGeom<T, W, H>;
  auto kern = k_tma_g<T, W, H, Op>;
  static int ctasPerSm = 0;  // per instantiation
  if (ctasPerSm == 0) {
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(G::smem_bytes)));
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctasPerSm, kern, (TMA_WARPS + 1) * 32, G::smem_bytes));
    if (ctasPerSm < 1) ctasPerSm = 1;
  }
  const int gx = (a.nx + G::CW - 1) / G::CW;
  const int rows = a.row1 - a.row0;
  KArgs<T> b = a;
  b.segRows = tma_segment_rows(rows, gx, ctasPerSm, G::RPS);
  dim3 g2(gx, static_cast<unsigned>((rows + b.segRows - 1) / b.segRows));
  kern<<<g2, (TMA_WARPS + 1) * 32, G::smem_bytes, s>>>(b);
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
