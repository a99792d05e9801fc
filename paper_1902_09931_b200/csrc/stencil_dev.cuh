// stencil_dev.cuh — the stencil kernel templates (k_tma, k_tma_g,
// k_generic) and their window ops, device code only. Compiled twice:
//  * by nvcc into libstengrid_b200.so (stencil.cu, stencil_g64/32.cu), with
//    internal linkage per translation unit;
//  * by NVRTC at run time (sg_jit.cu) together with a user's window
//    function: the reference's StencilFunction is arbitrary user code
//    (stencil.hpp:20-25), so a function registered from source gets the same
//    kernels instantiated for it. Therefore no host headers here.
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
typedef decltype(sizeof(0)) size_t;
#define SG_DEV_BEGIN namespace sgjit {
#define SG_DEV_END }
#else
#include <cstddef>
#include <cstdint>
#define SG_DEV_BEGIN \
  namespace sg {     \
  namespace {
#define SG_DEV_END \
  }                \
  }
#endif

// Weight windows at least this tall accumulate pending outputs (ACC) instead
// of holding the input window in registers.
#ifndef SG_ACC_MIN_H
#define SG_ACC_MIN_H 5
#endif
// Ring stages of tall windows (H >= 5): at least this many (A/B knob).
#ifndef SG_TALL_STAGES
#define SG_TALL_STAGES 2
#endif
// Deep rings for tall windows (H >= 5) on one CTA per SM: as many stages
// as the shared-memory budget holds (up to SG_DEEP_MAX), so the single CTA
// keeps the producer far enough ahead of its long consumer rows. Bit 0:
// k_tma, bit 1: k_tma_g. Measured at 16384^2 (scripts/exp/deep_ab.sh):
// FP32 5x5 0.79 -> 0.94 of HBM, FP64 5x5 on odd rows 0.51 -> 0.57; short
// windows lose with deep rings (3x3 0.97 -> 0.90, 5x1 0.93 -> 0.62), so
// they keep the 9-row ring.
#ifndef SG_DEEP_STAGES
#define SG_DEEP_STAGES 3
#endif
#ifndef SG_DEEP_MAX
#define SG_DEEP_MAX 8
#endif
#ifndef SG_SMEM_BUDGET
#define SG_SMEM_BUDGET (220 * 1024)
#endif
__host__ __device__ constexpr int deep_stages(int base, unsigned long long stageBytes, bool deep) {
  if (!deep) return base;
  const long long fit = static_cast<long long>(SG_SMEM_BUDGET / stageBytes);
  const long long d = fit < SG_DEEP_MAX ? fit : SG_DEEP_MAX;
  return d > base ? static_cast<int>(d) : base;
}

SG_DEV_BEGIN

template <typename A, typename B>
struct sg_same {
  static constexpr bool value = false;
};
template <typename A>
struct sg_same<A, A> {
  static constexpr bool value = true;
};

// acc + w * x: FP64 rounds the product and the sum separately — the
// reference's -ffp-contract=off order, bitwise; FP32 (an extension judged
// against the FP64 oracle at 1e-5) contracts into one FFMA, which is more
// accurate and halves the FP32 instruction count of the tap loops (the FP32
// windows are issue-bound: every FP32 op takes an issue slot).
__device__ __forceinline__ double sg_mac(double acc, double w, double x) { return acc + w * x; }
__device__ __forceinline__ float sg_mac(float acc, float w, float x) { return __fmaf_rn(w, x, acc); }

// The vector-store condition of the pipelined kernels as a warp vote (see
// k_tma). SG_STORE_VOTE=0 keeps the per-lane condition (A/B).
#ifndef SG_STORE_VOTE
#define SG_STORE_VOTE 1
#endif
template <bool VOTE>
__device__ __forceinline__ bool sg_store_vote(bool lane) {
  return SG_STORE_VOTE && VOTE ? __all_sync(0xffffffffu, lane) : lane;
}

// Pending-output windows this tall keep a shifting accumulator ring (ROT in
// k_tma / k_tma_g) instead of a ring indexed by the unrolled row.
#ifndef SG_ROT_MIN_H
#define SG_ROT_MIN_H 8
#endif
// FP32 from 7 rows (7 x 7 0.58 -> 0.62 of HBM, 5 x 7 0.74 -> 0.78; 5 x 5 on
// odd rows loses: 0.64 -> 0.61; scripts/exp/rot32_ab.sh)
#ifndef SG_ROT_MIN_H_F32
#define SG_ROT_MIN_H_F32 7
#endif

// One input row e[0 .. V+W-1] of a weight window with H x V pending outputs:
// pend[q] holds the output started q rows ago; this row is its tap row q.
// Adds the row to every pending output (taps of one output still in the
// reference's row-major order), hands back the completed output (q = H-1)
// and shifts the ring by one row (pend[0] restarts at 0).
template <typename T, int W, int H, int V>
__device__ __forceinline__ void sg_acc_rows_rot(T (&pend)[H][V], const T* __restrict__ wts, const T* e, T* res) {
#pragma unroll
  for (int q = 0; q < H; ++q)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      T acc = q == 0 ? T(0) : pend[q][v];
#pragma unroll
      for (int p = 0; p < W; ++p) acc = sg_mac(acc, wts[q * W + p], e[v + p]);
      pend[q][v] = acc;
    }
#pragma unroll
  for (int v = 0; v < V; ++v) res[v] = pend[H - 1][v];
#pragma unroll
  for (int q = H - 1; q > 0; --q)
#pragma unroll
    for (int v = 0; v < V; ++v) pend[q][v] = pend[q - 1][v];
}

// k_generic weight windows: 4 output rows per thread reusing each staged
// row (1), or one output per pass (0, A/B)
#ifndef SG_GENERIC_ROWS4
#define SG_GENERIC_ROWS4 1
#endif
// ... and SG_GENERIC_NC columns per thread (32 apart)
#ifndef SG_GENERIC_NC
#define SG_GENERIC_NC 4
#endif
// k_generic's staged tile limit (dynamic shared memory, opted in beyond 48 KB)
#ifndef SG_GENERIC_SMEM
#define SG_GENERIC_SMEM (96 * 1024)
#endif

constexpr int VMAX = 256;       // values carried in the parameter bank
constexpr int GENERIC_FN_MAX = 256;  // window taps a generic device function may see

template <typename T>
struct KArgs {
  const T* __restrict__ in;
  T* __restrict__ out;
  const T* __restrict__ wdev;  // weights when count > VMAX (generic path only)
  int nx, inRows, inShift;
  int row0, row1, col0, col1;
  int wrapX, wrapY;
  int left, right, top, bottom;
  int segRows;
  int count;
  // P2P halo forwarding (multi-GPU y-slabs): output rows j < upRows are
  // also stored to peerUp + j*nx (the up neighbour's bottom halo), rows
  // j >= dnRow0 to peerDn + (j - dnRow0)*nx (the down neighbour's top
  // halo) — peer memory over NVLink; null = none
  T* peerUp;
  T* peerDn;
  int upRows, dnRow0;
  // k_generic: 1 = stage a (32 + W - 1) x (32 + H - 1) input tile in shared
  // memory per 32 x 32 outputs (dynamic shared memory of that size), 0 =
  // read every tap from global memory (windows whose tile would not fit)
  int gtile;
  T v[VMAX];
};

// Store one output value (and its P2P halo copies).
template <typename T>
__device__ __forceinline__ void put_out(const KArgs<T>& a, long long j, long long i, T v) {
  a.out[j * a.nx + i] = v;
  if (a.peerUp && j < a.upRows) a.peerUp[j * a.nx + i] = v;
  if (a.peerDn && j >= a.dnRow0) a.peerDn[(j - a.dnRow0) * a.nx + i] = v;
}

// ----------------------------------------------------------- window ops
// Device twins of the reference's window functions. Same expression trees,
// evaluated without contraction, so FP64 results are bitwise identical.
struct OpWeights {};  // marker: weight stencil

struct OpChNonlinear {  // cahn_hilliard.cpp:36-47
  template <typename T>
  __device__ static T apply(const T* w, const T* coe, int rs) {
    T acc = T(0);
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const T v = w[q * rs + p];
        acc += coe[q * 3 + p] * (v * v * v - v);
      }
    return acc;
  }
};
struct OpCentralDifference {  // tools/main.cpp:47-49
  template <typename T>
  __device__ static T apply(const T* w, const T* coe, int) {
    return (w[0] - T(2) * w[1] + w[2]) * coe[0];
  }
};
struct OpCenter {  // tests/test_stencil.cpp:68
  template <typename T>
  __device__ static T apply(const T* w, const T*, int rs) {
    return w[rs + 1];
  }
};
struct OpCentralSecond {  // tests/test_stencil.cpp:70-77
  template <typename T>
  __device__ static T apply(const T* w, const T* coe, int) {
    T acc = T(0);
    acc += coe[0] * w[0];
    acc += (T(-2) * coe[0]) * w[1];
    acc += coe[0] * w[2];
    return acc;
  }
};
struct OpLapCubeDiffFirst {  // tests/test_stencil.cpp:79-85
  template <typename T>
  __device__ static T g(T v) { return v * v * v - v; }
  template <typename T>
  __device__ static T apply(const T* w, const T* coe, int rs) {
    const T gm = g(w[rs + 1]);
    const T x = (g(w[rs]) - T(2) * gm) + g(w[rs + 2]);
    const T y = (g(w[1]) - T(2) * gm) + g(w[2 * rs + 1]);
    return coe[0] * x + coe[1] * y;
  }
};
struct OpWeighted3x3 {  // tests/test_stencil.cpp:88-93
  template <typename T>
  __device__ static T apply(const T* w, const T* coe, int rs) {
    T acc = T(0);
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int p = 0; p < 3; ++p) acc = sg_mac(acc, coe[q * 3 + p], w[q * rs + p]);
    return acc;
  }
};

template <typename T>
struct VecT;
template <>
struct VecT<double> {
  static constexpr int V = 2;
  using type = double2;
};
template <>
struct VecT<float> {
  static constexpr int V = 4;
  using type = float4;
};

__device__ __forceinline__ int wrap_idx(long long i, int n) {
  long long r = i % n;
  return static_cast<int>(r < 0 ? r + n : r);
}

// ---------------------------------------------------------------- k_tma
// The fast path. Each consumer warp owns a strip of 32*V columns (V = 16
// bytes / sizeof(T)) and marches down a segment of rows; rows are staged into a per-warp shared-memory
// ring by the bulk-copy engine (cp.async.bulk, TMA 1D, completion on an
// mbarrier per stage): ONE copy per row brings the strip's 32*V columns
// plus the L/R halo columns (rounded out to 16 B) — halos are loaded once
// and never shuffled; only edge strips add a 16-32 B wrap copy. Registers
// hold just the H-row window, and the ring keeps S*RPS rows per warp in
// flight without register cost. (A register-prefetch variant with shuffled
// halos, k_strip, took 3.39 ms against k_tma's 2.62 ms for the 32768^2
// FP64 3x3 in ncu, profiles/r01_k_strip_f64_3x3_ncu_summary.txt; removed.)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// expect_tx without an arrival (the arrival comes once per stage)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// The mbarrier receives one arrival when all prior cp.async of this thread land.
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// CTA geometry: NW consumer warps side by side cover CW columns; one
// producer warp streams rows (CW + halos) into a STAGES x RPS ring.
// Light windows use 16 consumers (a 17-warp CTA, CW = 1024 FP64 columns:
// 32768-wide grids split into whole blocks). Register-heavy windows use 15,
// a 16-warp CTA — four warps on each of the SM's four sub-partitions, so a
// thread may hold 128 registers: with 17 warps one sub-partition hosts five
// and its 16 K-register file caps every thread at ~96. Measured at 16384^2
// FP64 (whole builds, 15 vs 16): 5x5 weights 0.61 -> 0.68 of HBM, 9x9 0.158
// -> 0.178, {2,1,1,2} 0.71 -> 0.83, odd-row 3x3 0.84 -> 0.90; but the
// headline 32768^2 3x3 function 415 -> 396 Gpts/s (FP32 800 -> 764: ragged
// 960-column blocks), so light windows keep 16.
#ifndef SG_TMA_WARPS
#define SG_TMA_WARPS 16
#endif
#ifndef SG_REALIGN_F32
#define SG_REALIGN_F32 1
#endif
#ifndef SG_TMA_WARPS_HEAVY
#define SG_TMA_WARPS_HEAVY 15
#endif
// k_tma windows at least SG_TALL_H rows tall (9 x 9 weights: FP64-bound, H
// x V pending-output chains per lane) on SG_TMA_WARPS_TALL consumers: with
// the weights in uniform registers (sg_store_vote) the 128-register cap of
// the 16-warp CTA spills ~30 values per row; 7 consumers have 255.
// Measured at 16384^2 (scripts/exp/tall_ab.sh): 9 x 9 0.179 -> 0.186 of HBM
// (11 consumers: 0.174); k_tma_g's odd-row 9 x 9 loses with it (0.165 ->
// 0.162) and keeps the heavy geometry.
#ifndef SG_TMA_WARPS_TALL
#define SG_TMA_WARPS_TALL 7
#endif
#ifndef SG_TALL_H
#define SG_TALL_H 8
#endif
// k_tma_g tall windows: 7 consumers too (16384^2 FP64, rolled ring: 9 x 9
// odd rows 0.168 -> 0.179 of HBM, (0,8,8,0) 0.168 -> 0.186; no spills)
#ifndef SG_TMAG_WARPS_TALL
#define SG_TMAG_WARPS_TALL 7
#endif
constexpr int TMA_WARPS = SG_TMA_WARPS;
// consumer warps of k_tma (window height H) and of k_tma_g (W x H window)
// (tall = at least SG_TALL_H rows and SG_TALL_TAPS taps: FP64-bound; a 1 x 9
// column window streams and keeps the wide CTA — k_tma_g's odd-row (0,0,4,4)
// 0.85 -> 0.58 of HBM on 7 consumers — and 5 x 9 on odd rows loses too,
// 0.34 -> 0.29; scripts/exp/gtall_ab.sh)
#ifndef SG_TALL_TAPS
#define SG_TALL_TAPS 60
#endif
// FP64 only: FP32 9 x 9 on 7 consumers 0.39 -> 0.30 of HBM (gtall32_ab.sh)
__host__ __device__ constexpr bool tma_tall(int W, int H, int esz) {
  return esz == 8 && H >= SG_TALL_H && W * H >= SG_TALL_TAPS;
}
__host__ __device__ constexpr int tma_nw(int H, int W, int esz) {
  return tma_tall(W, H, esz) ? SG_TMA_WARPS_TALL : H >= 5 ? SG_TMA_WARPS_HEAVY : SG_TMA_WARPS;
}
// (k_tma_g: FP64 always on the 16-warp geometry — its odd-row store
// realignment needs the registers: {3,1,0,0} on odd rows 0.76 -> 0.82 —
// FP32 light windows stay on 17 warps: FP32 {3,1,0,0} 0.89 -> 0.69 with 16)
__host__ __device__ constexpr int tmag_nw(int W, int H, int esz) {
  return tma_tall(W, H, esz) ? SG_TMAG_WARPS_TALL : esz == 8 || W * H >= 9 ? SG_TMA_WARPS_HEAVY : SG_TMA_WARPS;
}
// Release of a ring stage by the consumers: every thread arrives on the
// "empty" mbarrier (1), or each warp's lane 0 after __syncwarp (0).
#ifndef SG_EMPTY_ALL_LANES
#define SG_EMPTY_ALL_LANES 1
#endif

template <typename T, int L, int R, int TP, int BT>
struct TmaGeom {
  static constexpr int V = VecT<T>::V;
  static constexpr int SW = 32 * V;
  static constexpr int NW = tma_nw(TP + BT + 1, L + R + 1, static_cast<int>(sizeof(T)));
  static constexpr int CW = NW * SW;
  static constexpr int LP = ((L + V - 1) / V) * V;  // left pad, 16 B granules
  static constexpr int RP = ((R + V - 1) / V) * V;
  static constexpr int ROW = LP + CW + RP;  // elements per staged row (~2 KB)
  static constexpr int H = TP + BT + 1;
  // Rows per stage: a multiple of H so the register window is a ring whose
  // slot for every unrolled row is a compile-time constant (no moves).
  static constexpr int RPS = H >= 2 ? H : 2;
  static constexpr int STAGES_BASE = (9 + RPS - 1) / RPS >= 2 ? (9 + RPS - 1) / RPS : 2;
  static constexpr size_t stage_bytes = static_cast<size_t>(RPS) * ROW * sizeof(T);
  static constexpr int STAGES =
      deep_stages(STAGES_BASE < SG_TALL_STAGES && H >= 5 ? SG_TALL_STAGES : STAGES_BASE, stage_bytes,
                  (SG_DEEP_STAGES & 1) != 0 && H >= 5);
  static constexpr size_t smem_bytes = STAGES * stage_bytes + 2 * STAGES * sizeof(uint64_t);
};

// Launch bounds of k_tma: the compiler's register choice (one CTA per SM
// guaranteed); SG_TMA_MINB2=1 sizes for two where the rings fit — measured
// slower (3x3 0.97 -> 0.93 of HBM, 5x5 0.61 -> 0.50 at 16384^2 FP64).
#ifndef SG_TMA_MINB2
#define SG_TMA_MINB2 -1
#endif
template <typename T, int L, int R, int TP, int BT>
constexpr int tma_min_blocks() {
  constexpr bool fits2 = 2 * TmaGeom<T, L, R, TP, BT>::smem_bytes <= 227 * 1024;
  if (SG_TMA_MINB2 == 0 || !fits2) return 1;
  if (SG_TMA_MINB2 == 1) return 2;
  return 1;
}

template <typename T, int L, int R, int TP, int BT, typename Op>
__global__ void __launch_bounds__((TmaGeom<T, L, R, TP, BT>::NW + 1) * 32, (tma_min_blocks<T, L, R, TP, BT>())) k_tma(const __grid_constant__ KArgs<T> a) {
  using G = TmaGeom<T, L, R, TP, BT>;
  using VT = typename VecT<T>::type;
  constexpr int V = G::V, SW = G::SW, CW = G::CW, LP = G::LP, RP = G::RP, ROW = G::ROW;
  constexpr int H = G::H, RPS = G::RPS, STAGES = G::STAGES;
  constexpr int W = L + R + 1;
  constexpr int E = L + V + R;
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

  if (threadIdx.x == 0) {
    for (int k = 0; k < STAGES; ++k) {
      mbar_init(&full[k], 1 + 32);  // expect_tx arrival + the producer warp's cp.async arrivals
      mbar_init(&empty[k], SG_EMPTY_ALL_LANES ? G::NW * 32 : G::NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: the prologue above overlaps the previous
  // kernel's tail; no global memory is touched before its completion
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == G::NW) {
    // ---------------- producer warp: per row, lane 0 issues one bulk copy of
    // the CTA's own columns (128 B aligned, whole lines: no over-fetch),
    // lanes 1.. one 16 B cp.async granule each for the halo columns (wrapped
    // in index math at grid edges); every lane arrives on the stage barrier
    // through cp.async.mbarrier.arrive
    const int validC = min(CW, nx - cx0);
    const uint32_t mainBytes = static_cast<uint32_t>(validC * sizeof(T));
    int hsrc[(LP + RP) / V > 0 ? (LP + RP) / V : 1];
    int hdst[(LP + RP) / V > 0 ? (LP + RP) / V : 1];
    int nh = 0;
#pragma unroll
    for (int k = 0; k < LP / V; ++k) {
      const int c = cx0 - LP + k * V;
      if (c >= 0 || a.wrapX) {
        hsrc[nh] = c >= 0 ? c : c + nx;
        hdst[nh++] = k * V;
      }
    }
#pragma unroll
    for (int k = 0; k < RP / V; ++k) {
      const int c = cx0 + validC + k * V;
      if (c < nx || a.wrapX) {
        hsrc[nh] = c < nx ? c : c - nx;
        hdst[nh++] = LP + validC + k * V;
      }
    }
    // this lane's granule (lane h + 1 takes granule h)
    int mySrc = 0, myDst = 0;
    const bool mine = lane >= 1 && lane - 1 < nh;
#pragma unroll
    for (int h = 0; h < (LP + RP) / V; ++h)
      if (lane - 1 == h) {
        mySrc = hsrc[h];
        myDst = hdst[h];
      }
    int rf = ra + a.inShift - TP;
    if (a.wrapY) rf = wrap_idx(rf, a.inRows);
    const T* __restrict__ in = a.in;
    for (int g = 0; g < nStages; ++g) {
      const int slot = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[slot], ((g / STAGES) + 1) & 1);
      if (lane == 0) mbar_expect_tx(&full[slot], mainBytes * RPS);
      T* sstage = ring + slot * (RPS * ROW);
#pragma unroll
      for (int k = 0; k < RPS; ++k) {
        const T* grow = in + static_cast<long long>(rf) * nx;
        T* srow = sstage + k * ROW;
        if (lane == 0) bulk_g2s(srow + LP, grow + cx0, mainBytes, &full[slot]);
        if (mine) cp_async16(srow + myDst, grow + mySrc);
        ++rf;
        if (a.wrapY) {
          if (rf == a.inRows) rf = 0;
        } else if (rf >= a.inRows) {
          rf = a.inRows - 1;
        }
      }
      cp_async_mbar_arrive(&full[slot]);
    }
    return;
  }

  // ---------------- consumers
  const int xb = cx0 + warp * SW + lane * V;
  const bool laneValid = xb < nx;
  // Weight stencils with tall windows (H >= 5) keep H PENDING OUTPUT
  // accumulators instead of H input rows: each arriving input row adds its
  // tap row to every output that needs it. Output o still accumulates its
  // taps row by row (q ascending, then p) — the reference's order — since
  // rows arrive top to bottom. Registers: H*V + E instead of H*E (a 9x9
  // window would otherwise spill).
  constexpr bool ACC = sg_same<Op, OpWeights>::value && H >= SG_ACC_MIN_H;
  // ROT (windows >= SG_ROT_MIN_H rows): the pending outputs shift one slot
  // per row (pend[q] = the output started q rows ago) so the row loop stays
  // rolled — 9 unrolled rows of a 9 x 9 window are ~3.5 k instructions and
  // stalled on instruction fetch; the shift costs (H - 1) x V moves per row
  constexpr bool ROT = ACC && H >= (sizeof(T) == 4 ? SG_ROT_MIN_H_F32 : SG_ROT_MIN_H);
  T win[ACC ? 1 : H][E];  // ring: input row t lives in win[t % H]
  T pend[ACC ? H : 1][V];  // ACC: output started at local input row u lives in pend[u % H]
  T* __restrict__ orow = a.out + static_cast<long long>(ra - (H - 1)) * nx + xb;
  // Warp-uniform (a vote) for FP64 tall weight windows: a lane-dependent
  // branch around the stores keeps ptxas from holding the weights in uniform
  // registers (DMUL R, R, UR) — it reloads the taps from the parameter bank
  // with LDC.64 instead (9 x 9: ~90 LDC per row). Partial warps then take
  // the element path. Measured at 16384^2 (scripts/exp/vote_ab.sh): FP64 7 x
  // 7 0.33 -> 0.37 of HBM, 5 x 5 +2 %; the light windows lose with it (3 x
  // 3 1.03 -> 0.95, FP32 5 x 5 0.94 -> 0.92), so they keep the lane test.
  const bool vecStore = sg_store_vote<sizeof(T) == 8 && H >= 5>(laneValid && xb >= a.col0 && xb + V <= a.col1);
  const long long rowStep = nx;
  int j = ra - (H - 1);  // output row completed by the current input row
  for (int g = 0; g < nStages; ++g) {
    const int slot = g % STAGES;
    mbar_wait(&full[slot], (g / STAGES) & 1);
    const T* sbase = ring + slot * (RPS * ROW) + LP + warp * SW + lane * V;
    // rows of the stage: fully unrolled (plain `#pragma unroll`: an
    // explicit factor changed ptxas' schedule, FP64 odd-row 3 x 3 0.94 ->
    // 0.91 of HBM), or one rolled row at a time for ROT
#pragma unroll 1
    for (int kk = 0; kk < (ROT ? RPS : 1); ++kk)
#pragma unroll
    for (int k0 = 0; k0 < (ROT ? 1 : RPS); ++k0) {
      const int k = kk + k0;
      const T* srow = sbase + k * ROW;
      T* e = win[ACC ? 0 : k % H];
      const VT c = *reinterpret_cast<const VT*>(srow);
      if constexpr (V == 2) {
        e[L] = c.x;
        e[L + 1] = c.y;
      } else {
        e[L] = c.x;
        e[L + 1] = c.y;
        e[L + 2] = c.z;
        e[L + 3] = c.w;
      }
      // Horizontal halos: scalar shared loads at a 16 B lane stride (2-way
      // bank conflicts, ~0.1 per output in ncu). Shuffling them from the
      // neighbouring lanes' vectors instead removed 83 % of the conflicts
      // but measured slower (3x3 98.4 -> 97.2 % of HBM, 5x5 FP64-bound
      // 0.63 -> 0.47): the loads are not on the critical resource.
#pragma unroll
      for (int p = 0; p < L; ++p) e[p] = srow[p - L];
#pragma unroll
      for (int p = 0; p < R; ++p) e[L + V + p] = srow[V + p];
      // Output row j uses input rows j-TP .. j+BT = the H most recent rows,
      // oldest in slot (k + 1) % H.
      T res[V];
      if constexpr (ROT) {
        sg_acc_rows_rot<T, W, H, V>(pend, a.v, e, res);
      } else if constexpr (ACC) {
        // this row is tap row q of the output started q rows ago (slot
        // (k - q) mod H; RPS is a multiple of H, so slots are compile-time)
#pragma unroll
        for (int q = 0; q < H; ++q) {
          T* acc = pend[((k - q) % H + H) % H];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (q == 0) acc[v] = T(0);
#pragma unroll
            for (int p = 0; p < W; ++p) acc[v] = sg_mac(acc[v], a.v[q * W + p], e[v + p]);
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = pend[(k + 1) % H][v];  // completed (q = H-1 just added)
      } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if constexpr (sg_same<Op, OpWeights>::value) {
          T acc = T(0);
#pragma unroll
          for (int q = 0; q < H; ++q)
#pragma unroll
            for (int p = 0; p < W; ++p) acc = sg_mac(acc, a.v[q * W + p], win[(k + 1 + q) % H][v + p]);
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
        if (vecStore) {
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
          *reinterpret_cast<VT*>(orow) = o;
          if (a.peerUp && j < a.upRows)  // warp-uniform
            *reinterpret_cast<VT*>(a.peerUp + static_cast<long long>(j) * nx + xb) = o;
          if (a.peerDn && j >= a.dnRow0)
            *reinterpret_cast<VT*>(a.peerDn + static_cast<long long>(j - a.dnRow0) * nx + xb) = o;
        } else if (laneValid) {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (xb + v >= a.col0 && xb + v < a.col1) put_out(a, j, xb + v, res[v]);
        }
      }
      ++j;
      orow += rowStep;
    }
    // every lane of this warp has read the stage
    if constexpr (SG_EMPTY_ALL_LANES) {
      mbar_arrive(&empty[slot]);  // each thread releases its own reads of the slot
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
}

// ------------------------------------------------------------- k_generic
// Windows the pipelined kernels do not take (beyond 9 x 9, device functions
// on non-natural windows). Tiled (a.gtile): a 256-thread CTA computes 32 x
// 32 outputs from a (32 + W - 1) x (32 + H - 1) input tile staged once in
// shared memory (coalesced loads, the periodic wrap applied while staging);
// every tap then comes from shared memory. Function windows are handed over
// IN the tile with rowStride = the tile pitch (the reference's contract
// allows any stride, stencil.hpp:20-25). Untiled: one thread per point, taps
// from global memory (windows too large for a tile). Accumulation order is
// the reference's either way.
template <typename T, typename Op>
__global__ void __launch_bounds__(256) k_generic(const __grid_constant__ KArgs<T> a) {
  const int W = a.left + a.right + 1;
  const int H = a.top + a.bottom + 1;
  const T* __restrict__ in = a.in;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.gtile) {
    extern __shared__ __align__(16) unsigned char gsm[];
    T* tile = reinterpret_cast<T*>(gsm);
    // weight windows: 64 output columns per CTA (two per thread)
    constexpr int GW = sg_same<Op, OpWeights>::value && SG_GENERIC_ROWS4 ? 32 * SG_GENERIC_NC : 32;
    const int TW = GW + W - 1, TH = 32 + H - 1;
    const int i0 = a.col0 + blockIdx.x * GW, j0 = a.row0 + blockIdx.y * 32;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int e = tid; e < TW * TH; e += 256) {
      const int ty = e / TW, tx = e - ty * TW;
      long long r = static_cast<long long>(j0) + a.inShift - a.top + ty;
      if (a.wrapY) {
        if (r < 0 || r >= a.inRows) r = wrap_idx(r, a.inRows);
      } else {
        r = r < 0 ? 0 : (r >= a.inRows ? a.inRows - 1 : r);  // feeds only outputs that are not stored
      }
      long long c = static_cast<long long>(i0) - a.left + tx;
      if (a.wrapX) {
        if (c < 0 || c >= a.nx) c = wrap_idx(c, a.nx);
      } else {
        c = c < 0 ? 0 : (c >= a.nx ? a.nx - 1 : c);
      }
      tile[e] = in[r * a.nx + c];
    }
    __syncthreads();
    const int i = i0 + threadIdx.x;
    if constexpr (sg_same<Op, OpWeights>::value && SG_GENERIC_ROWS4) {
      // each thread: 4 consecutive output rows of one column. Every staged
      // row is read once and added to each output it is a tap row of —
      // per output still tap rows ascending, then columns (the reference's
      // order). No lane-dependent exit before the loops (it would cost the
      // uniform datapath for the weights, cf. k_tma); lanes past col1
      // compute on clamped tile values and do not store.
      // (and columns threadIdx.x, threadIdx.x + 32: each weight load feeds
      // eight multiply-adds)
      const int y0 = 4 * threadIdx.y;
      constexpr int NC = SG_GENERIC_NC;
      T acc[NC][4];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[c][k] = T(0);
      auto rows = [&](auto wt) {  // wt(idx): the weight, from the parameter bank or wdev
#pragma unroll 1
        for (int t = 0; t < H + 3; ++t) {
          const T* rowp = tile + (y0 + t) * TW + threadIdx.x;
          if (t >= 3 && t < H) {
            // staged row t is tap row t - k of output k, for all four:
            // no predicates, one running weight index per output
            const int i0 = t * W, i1 = i0 - W, i2 = i1 - W, i3 = i2 - W;
#pragma unroll 4
            for (int p = 0; p < W; ++p) {
              const T w0 = wt(i0 + p), w1 = wt(i1 + p), w2 = wt(i2 + p), w3 = wt(i3 + p);
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                const T x = rowp[p + 32 * c];
                acc[c][0] = sg_mac(acc[c][0], w0, x);
                acc[c][1] = sg_mac(acc[c][1], w1, x);
                acc[c][2] = sg_mac(acc[c][2], w2, x);
                acc[c][3] = sg_mac(acc[c][3], w3, x);
              }
            }
            continue;
          }
#pragma unroll 2
          for (int p = 0; p < W; ++p) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int q = t - k;
              if (q >= 0 && q < H) {
                const T w = wt(q * W + p);
#pragma unroll
                for (int c = 0; c < NC; ++c) acc[c][k] = sg_mac(acc[c][k], w, rowp[p + 32 * c]);
              }
            }
          }
        }
      };
      if (a.count <= VMAX)
        rows([&](int idx) { return a.v[idx]; });
      else
        rows([&](int idx) { return __ldg(a.wdev + idx); });
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (i + 32 * c < a.col1) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (j0 + y0 + k < a.row1) put_out(a, j0 + y0 + k, i + 32 * c, acc[c][k]);
        }
      return;
    }
    if (i >= a.col1) return;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int yy = threadIdx.y + 8 * k, j = j0 + yy;
      if (j >= a.row1) break;
      const T* base = tile + yy * TW + threadIdx.x;
      if constexpr (sg_same<Op, OpWeights>::value) {
        const T* wt = a.count <= VMAX ? a.v : a.wdev;
        T acc = T(0);
        for (int q = 0; q < H; ++q) {
          const T* rowp = base + q * TW;
          const T* wq = wt + q * W;
#pragma unroll 4
          for (int p = 0; p < W; ++p) acc = sg_mac(acc, wq[p], rowp[p]);
        }
        put_out(a, j, i, acc);
      } else {
        put_out(a, j, i, Op::template apply<T>(base, a.v, TW));
      }
    }
    return;
  }
  const int i = a.col0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int j = a.row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= a.col1 || j >= a.row1) return;
  if constexpr (sg_same<Op, OpWeights>::value) {
    const T* wt = a.count <= VMAX ? a.v : a.wdev;
    T acc = T(0);
    for (int q = 0; q < H; ++q) {
      long long r = static_cast<long long>(j) + a.inShift - a.top + q;
      if (a.wrapY && (r < 0 || r >= a.inRows)) r = wrap_idx(r, a.inRows);
      const T* rowp = in + r * a.nx;
      for (int p = 0; p < W; ++p) {
        long long c = static_cast<long long>(i) - a.left + p;
        if (a.wrapX && (c < 0 || c >= a.nx)) c = wrap_idx(c, a.nx);  // modulo only at the edges
        acc = sg_mac(acc, wt[q * W + p], rowp[c]);
      }
    }
    put_out(a, j, i, acc);
  } else {
    T w[GENERIC_FN_MAX];
    for (int q = 0; q < H; ++q) {
      long long r = static_cast<long long>(j) + a.inShift - a.top + q;
      if (a.wrapY && (r < 0 || r >= a.inRows)) r = wrap_idx(r, a.inRows);
      const T* rowp = in + r * a.nx;
      for (int p = 0; p < W; ++p) {
        long long c = static_cast<long long>(i) - a.left + p;
        if (a.wrapX && (c < 0 || c >= a.nx)) c = wrap_idx(c, a.nx);  // modulo only at the edges
        w[q * W + p] = rowp[c];
      }
    }
    put_out(a, j, i, Op::template apply<T>(w, a.v, W));
  }
}

// ------------------------------------------------------------- k_tma_g
// (design notes: stencil_g.cuh)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(sizeof(T))
               : "memory");
}

template <typename T, int W, int H>
struct TmaGGeom {
  static constexpr int V = VecT<T>::V;
  static constexpr int SW = 32 * V;
  static constexpr int NW = tmag_nw(W, H, static_cast<int>(sizeof(T)));
  static constexpr int CW = NW * SW;
  static constexpr int HP = ((W - 1 + V - 1) / V) * V;  // halo room either side (any split of W - 1)
  static constexpr int ROW = HP + CW + V + HP;          // + V: the row's 16 B phase
  static constexpr int RPS = H >= 2 ? H : 2;
  static constexpr int STAGES_BASE = (9 + RPS - 1) / RPS >= 2 ? (9 + RPS - 1) / RPS : 2;
  static constexpr size_t stage_bytes = static_cast<size_t>(RPS) * ROW * sizeof(T);
  static constexpr int STAGES =  // (one CTA per SM where tmag_min_blocks says so)
      deep_stages(STAGES_BASE < SG_TALL_STAGES && H >= 5 ? SG_TALL_STAGES : STAGES_BASE, stage_bytes,
                  (SG_DEEP_STAGES & 2) != 0 && H >= 5 && !(W <= 3 && H <= 6));
  static constexpr size_t smem_bytes = STAGES * stage_bytes + 2 * STAGES * sizeof(uint64_t);
};

// Columns of one staged row that move as a single bulk copy: [a0, a1),
// both 16 B aligned in global memory (V elements). The CTA needs
// [cx0, cx0 + validC) plus halos; where the row's phase ph != 0 the bulk
// copy over-fetches to the aligned boundaries as long as the extra columns
// lie inside the same grid row (they are then exactly the halo columns the
// window reads, with the same values, so those halo copies are skipped);
// otherwise (the row's first CTA at cx0 = 0, or a tail that would cross the
// row end where periodic x wraps) the ragged head [cx0, cx0 + hc) and tail
// [ts, cx0 + validC) move as element cp.async. Over-fetching replaces up to
// 2 * (V - 1) element copies per row with nothing (FP32: 6 of them).
template <int V>
struct RowSpan {
  int a0, a1, hc, ts;
  __device__ RowSpan(int ph, int cx0, int validC, int nx) {
    const int e = cx0 + validC;
    if (ph == 0) a0 = cx0;
    else if (cx0 >= ph) a0 = cx0 - ph;  // over-fetch the head (same row)
    else a0 = cx0 + (V - ph);  // first aligned column; [cx0, a0) as elements
    const int endPh = (ph + validC) & (V - 1);
    if (endPh == 0) a1 = e;
    else if (e + (V - endPh) <= nx) a1 = e + (V - endPh);  // over-fetch the tail (same row)
    else a1 = e - endPh;
    hc = a0 > cx0 ? min(a0, e) - cx0 : 0;
    if (a1 <= a0) a1 = a0;  // no bulk copy: the whole span moves as elements
    ts = a1 > a0 ? min(a1, e) : cx0 + hc;
  }
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
__global__ void __launch_bounds__((TmaGGeom<T, W, H>::NW + 1) * 32, (tmag_min_blocks<T, W, H>())) k_tma_g(const __grid_constant__ KArgs<T> a) {
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
      mbar_init(&full[k], 1 + 32);  // expect_tx arrival + the producer warp's cp.async arrivals
      mbar_init(&empty[k], G::NW * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: the prologue above overlaps the previous
  // kernel's tail; no global memory is touched before its completion
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == G::NW) {
    // ---------------- producer warp: per row, lane 0 issues the 16 B-aligned
    // span of the CTA's columns as one bulk copy (RowSpan); the elements the
    // span leaves out — ragged head/tail columns of the row's first/last
    // CTA, halo columns outside it (wrapped in index math) — go one per lane
    // (lanes 1..) as element cp.async. Everything that depends only on the
    // row's 16 B phase is resolved once per CTA for each of the V phases, so
    // the per-row producer work is a phase lookup, one expect_tx + bulk copy
    // (lane 0) and at most one element copy per lane: the single producer
    // warp must issue a stage faster than the consumers drain one (measured:
    // FP32 4x4 windows were producer-issue-bound at ~150 instructions/row).
    // Every lane's copies arrive on the stage barrier through
    // cp.async.mbarrier.arrive; lane 0 adds the bytes row by row
    // (mbarrier.expect_tx, measured faster than one arrive.expect_tx per
    // stage computed up front: FP32 odd 3x3 0.885 vs 0.853) and arrives once
    // per stage.
    const int validC = min(CW, nx - cx0);
    const int l = a.left, r = a.right;
    const T* __restrict__ in = a.in;
    // lane k >= 1 owns column offset o (relative to cx0) from the disjoint
    // lists: left halo [-l, 0), head [0, min(V-1, validC)), tail
    // [max(V-1, validC-(V-1)), validC), right halo [validC, validC + r)
    int o = 0x40000000;
    {
      int k = lane - 1;
      const int nh = min(V - 1, validC);
      const int t0 = max(V - 1, validC - (V - 1));
      if (k >= 0 && k < l) o = k - l;
      else if ((k -= l) >= 0 && k < nh) o = k;
      else if ((k -= nh) >= 0 && k < validC - t0) o = t0 + k;
      else if ((k -= validC - t0) >= 0 && k < r) o = validC + k;
    }
    const int c = cx0 + o;  // the lane's global column (unwrapped)
    const bool inside = c >= 0 && c < nx;
    const bool srcOk = o != 0x40000000 && (inside || a.wrapX);
    const int srcCol = inside ? c : (c < 0 ? c + nx : c - nx);
    int bA0[V], bN[V];  // per phase: bulk span start and length (lane 0)
    unsigned need = 0;  // per phase: this lane's element copy is needed
#pragma unroll
    for (int ph = 0; ph < V; ++ph) {
      const RowSpan<V> sp(ph, cx0, validC, nx);
      bA0[ph] = sp.a0;
      bN[ph] = sp.a1 - sp.a0;
      const bool covered = inside && sp.a1 > sp.a0 && c >= sp.a0 && c < sp.a1;
      if (srcOk && !covered) need |= 1u << ph;
    }
    RowWalk rw;
    rw.init(r0, a.inRows, a.wrapY);
    for (int g = 0; g < nStages; ++g) {
      const int slot = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[slot], ((g / STAGES) + 1) & 1);
      T* sstage = ring + slot * (RPS * ROW);
#pragma unroll
      for (int k = 0; k < RPS; ++k) {
        const T* grow = in + static_cast<long long>(rw.cur) * nx;
        const int ph = static_cast<int>((inOff + static_cast<unsigned>(rw.cur) * unx) & (V - 1));
        rw.next(a.inRows, a.wrapY);
        T* srow = sstage + k * ROW + HP + ph;  // column cx0 of this row
        if (lane == 0) {
          int a0 = bA0[0], nb = bN[0];
#pragma unroll
          for (int q = 1; q < V; ++q)
            if (ph == q) {
              a0 = bA0[q];
              nb = bN[q];
            }
          if (nb > 0) {
            const uint32_t bytes = static_cast<uint32_t>(nb * sizeof(T));
            mbar_expect_tx_only(&full[slot], bytes);
            bulk_g2s(srow + (a0 - cx0), grow + a0, bytes, &full[slot]);
          }
        } else if ((need >> ph) & 1u) {
          cp_async_elem(srow + o, grow + srcCol);
        }
      }
      if (lane == 0) mbar_arrive(&full[slot]);
      cp_async_mbar_arrive(&full[slot]);
    }
    return;
  }

  // ---------------- consumers
  const int xo = warp * SW + lane * V;  // lane's first output column - cx0
  const int xb = cx0 + xo;
  const bool laneValid = xb < nx;
  // a warp vote (see k_tma) for windows of more than 9 taps, and FP32 3 x 3
  // (16384^2, odd and even rows: FP32 {2,1,1,2} odd 0.71 -> 0.75, 3 x 3 odd
  // 0.89 -> 0.91, FP64 {2,1,1,2} 0.70 -> 0.80 odd, 0.82 -> 0.89 even,
  // {1,2,2,1} +7 %, 5 x 5 odd +8 %); FP64 3 x 3 on odd rows loses with it
  // (0.93 -> 0.90), {3,1,0,0} is neutral
  const bool laneFull = sg_store_vote<(W * H > 9 || (sizeof(T) == 4 && W * H == 9))>(
      laneValid && xb >= a.col0 && xb + V <= a.col1);
  const unsigned outOff = static_cast<unsigned>(reinterpret_cast<uintptr_t>(a.out) / sizeof(T));
  const bool peers = a.peerUp != nullptr || a.peerDn != nullptr;
  const bool peerVec = nx % V == 0;  // peer rows share the output rows' phase only then
  constexpr bool ACC = sg_same<Op, OpWeights>::value && H >= SG_ACC_MIN_H;
  constexpr bool ROT = ACC && H >= (sizeof(T) == 4 ? SG_ROT_MIN_H_F32 : SG_ROT_MIN_H);  // (see k_tma)
  T win[ACC ? 1 : H][E];   // ring: input row t lives in win[t % H]
  T pend[ACC ? H : 1][V];  // ACC: output started at local input row u lives in pend[u % H]
  RowWalk rw;
  rw.init(r0, a.inRows, a.wrapY);
  int j = ra - (H - 1);  // output row completed by the current input row
  for (int g = 0; g < nStages; ++g) {
    const int slot = g % STAGES;
    mbar_wait(&full[slot], (g / STAGES) & 1);
    const T* sbase = ring + slot * (RPS * ROW) + HP + xo - a.left;
#pragma unroll 1
    for (int kk = 0; kk < (ROT ? RPS : 1); ++kk)  // (see k_tma)
#pragma unroll
    for (int k0 = 0; k0 < (ROT ? 1 : RPS); ++k0) {
      const int k = kk + k0;
      const int ph = static_cast<int>((inOff + static_cast<unsigned>(rw.cur) * unx) & (V - 1));
      rw.next(a.inRows, a.wrapY);
      const T* srow = sbase + k * ROW + ph;  // window column 0 of the lane's first output
      T* e = win[ACC ? 0 : k % H];
      // (scalar reads: 16 B vector reads + runtime-phase selects measured
      // slower, FP32 4x4 0.64 -> 0.60 of HBM, 3x3 odd 0.76 -> 0.68)
#pragma unroll
      for (int p = 0; p < E; ++p) e[p] = srow[p];
      T res[V];
      if constexpr (ROT) {
        sg_acc_rows_rot<T, W, H, V>(pend, a.v, e, res);
      } else if constexpr (ACC) {
#pragma unroll
        for (int q = 0; q < H; ++q) {
          T* acc = pend[((k - q) % H + H) % H];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (q == 0) acc[v] = T(0);
#pragma unroll
            for (int p = 0; p < W; ++p) acc[v] = sg_mac(acc[v], a.v[q * W + p], e[v + p]);
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = pend[(k + 1) % H][v];
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if constexpr (sg_same<Op, OpWeights>::value) {
            T acc = T(0);
#pragma unroll
            for (int q = 0; q < H; ++q)
#pragma unroll
              for (int p = 0; p < W; ++p) acc = sg_mac(acc, a.v[q * W + p], win[(k + 1 + q) % H][v + p]);
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
        const int pho = static_cast<int>((outOff + static_cast<unsigned>(j) * unx) & (V - 1));
        const bool rowVec = pho == 0;
        // (only with the 16-warp geometry's register headroom: on 17-warp
        // CTAs the extra registers cost more than the stores save)
        if ((G::NW == SG_TMA_WARPS_HEAVY || (SG_REALIGN_F32 && sizeof(T) == 4)) && !rowVec && !peers) {
          // misaligned output row: realign across lanes. The row's 16 B
          // groups start at column xb + sh; lane t stores the group made of
          // its res[sh..V-1] and lane t+1's res[0..sh-1] (shuffled down) as
          // one vector; what no group of this warp covers (lane 0's first sh
          // columns, lane 31's last V - sh, groups reaching outside
          // [col0, col1)) goes out element by element.
          const int sh = V - pho;
          T nb[V];
#pragma unroll
          for (int v = 0; v < V; ++v) nb[v] = __shfl_down_sync(0xffffffffu, res[v], 1);
          const int gc = xb + sh;
          const bool mine = lane < 31 && gc >= a.col0 && gc + V <= a.col1;
          const bool prev = lane > 0 && gc - V >= a.col0 && gc <= a.col1;
          if (mine) {
            // o[v] = res[v + sh] or nb[v + sh - V], selected with
            // compile-time indices (a runtime index would put res in local
            // memory)
            T o[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              T x = res[0];
#pragma unroll
              for (int c = 1; c < V; ++c)
                if (sh == c) x = v + c < V ? res[v + c] : nb[v + c - V];
              o[v] = x;
            }
            VT ov;
            if constexpr (V == 2) {
              ov.x = o[0];
              ov.y = o[1];
            } else {
              ov.x = o[0];
              ov.y = o[1];
              ov.z = o[2];
              ov.w = o[3];
            }
            *reinterpret_cast<VT*>(a.out + jo + gc) = ov;
          }
          if (laneValid) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const bool covered = v < sh ? prev : mine;
              if (!covered && xb + v >= a.col0 && xb + v < a.col1) a.out[jo + xb + v] = res[v];
            }
          }
        } else if (laneFull && rowVec && (!peers || peerVec)) {
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

SG_DEV_END
