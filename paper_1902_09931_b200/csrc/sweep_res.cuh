// sweep_res.cuh — the resident-turn uniform pentadiagonal sweep (k_sweep_res)
// and its TMA plumbing (tensor maps, the transposed-input preparation),
// included by penta.cu. A device-function body (sweep_res_body) so that a
// CTA of another kernel can run a sweep (tried for a merged CH RHS + x-sweep
// grid). Internal linkage.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <type_traits>

#include "penta.cuh"
#include "sg_internal.hpp"

namespace sg {
namespace {

struct alignas(64) SweepMaps {
  CUtensorMap z;     // 2D {B, n}, box {32, RS}
  CUtensorMap t[5];  // m1, m2, dInv, ap, bp: uniform 1D {n} box {RS}; else 2D like z
  CUtensorMap yc[1]; // XIN 1: the previous sweep's Woodbury coefficients y_k[r], 2D {n, 4} box {RS, 4}
  CUtensorMap zt;    // XIN (k_sweep_res): the input read TRANSPOSED, system-major:
                     // 3D {ztInner, B, n / ztInner} box {16, 32, 1}, 128 B swizzle —
                     // unknown r of system b at ((r % ztInner), b, r / ztInner): one
                     // block per source rank on the distributed y-sweep, else one
  CUtensorMap pz[8]; // P2P: the final (backward) results of unknowns [d*prow, (d+1)*prow)
                     // go to destination d's buffer (box {32, RS}, at (b, r - d*prow))
  int ztInner = 0;
  int ztBox = 0;     // 1: zt is the 4D view {16, B, ztInner / 16, n / ztInner}, box {16, 32, RS/16, 1}
  int npeer = 0;     // 0: final results stay in z
  int prow = 0;
  // Partitioned (SPIKE-type) sweep: each system's unknowns are segments of
  // segRows rows, segment blockIdx.y of a CTA's 32 systems solved as an
  // independent non-periodic system with the segment-local factor (the
  // `n` of the kernel is then segRows; z / zt / yc rows are offset by
  // blockIdx.y * segRows). The interface values g[0], g[1], g[m-2], g[m-1]
  // of every (segment, system) go to y4[(seg * 4 + k) * B + b].
  int segRows = 0;
  // XIN 1 after a partitioned sweep: yc holds one [4][n] plane of
  // coefficients per segment of THAT sweep (ycSeg rows each, along this
  // sweep's systems); 3D map {n, 4, planes}, box {RS, 4, 1}
  int ycSeg = 0;
};

// Fusions of the transposed-input sweep (k_sweep_res XIN, the CH step):
//  Wc/yc (XIN 1): the input is another sweep's UNcorrected result; its
//         Woodbury correction is applied on load: z(b, r) -= Wc0[b] yc0[r] +
//         ... + Wc3[b] yc3[r] (penta.cpp:279-286, same expression).
struct SweepFuse {
  const double* Wc[4] = {nullptr, nullptr, nullptr, nullptr};
  const double* yc = nullptr;  // XIN: yc[k*n + r], the previous sweep's y_k
  // P2P: y (this sweep's Woodbury coefficients) also written to every
  // destination: py4[d][k*y4Stride + y4Off + b]
  double* py4[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int y4Stride = 0, y4Off = 0;
};

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void s_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void s_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void s_mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(s_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}
// Non-blocking phase test: issued one stage ahead so its latency hides
// behind the current stage's recurrence.
__device__ __forceinline__ bool s_mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(s_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void s_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void s_mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void s_tma_2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ void s_tma_3d(void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ void s_tma_4d(void* dst, const CUtensorMap* m, int x, int y, int z, int w, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(s_u32(dst)),
      "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ void s_tma_1d(void* dst, const CUtensorMap* m, int x, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
          s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(s_u32(bar))
      : "memory");
}

// ------------------------------------------------------------ k_sweep_res
// Uniform-operator sweep with a RESIDENT TURN (the production path for the
// CH sweeps and every uniform batch). Warp 0 runs the recurrence of 32
// systems; warp 1 (one lane) owns ALL data movement, so the chain warp only
// computes:
//  * stages of RR_RS rows of z plus the five factor boxes stream in by
//    tensor TMA into an RR_NSTG-slot ring (full mbarriers);
//  * the consumer writes each result back into its slot (st.shared, constant
//    offsets), fences it to the async proxy and arrives on the slot's `done`
//    mbarrier; the producer then stores the slot with ONE tensor-TMA store
//    (shared -> global) before it reuses the slot for a later load;
//  * the last RR_NSTG forward stages are never stored: the backward pass
//    starts on them straight from shared memory while the producer refetches
//    the older stages (their stores completed: same thread, bulk wait_group),
//    so the forward->backward round trip through memory leaves the chain;
//  * operands are loaded RG rows ahead of the chain (software pipelined,
//    pinned by compiler barriers), so shared-memory latency stays off it.
// Arithmetic per row is penta.cpp:171-196 exactly, as in k_sweep_tma.
// Stage height RS: 64 rows (two 95 KB CTAs per SM: large batches) or 128
// rows (one 190 KB CTA per SM: batches of at most one CTA per SM, where
// halving the number of stage hand-offs shortens the chain's critical path:
// CH 1024^2 97.8 -> 92.4 us/step; 256-row stages (three slots) measured
// slower, 95.3 us — the backward group loop slows down).
constexpr int RR_RS = 64;    // rows per stage (default geometry)
constexpr int RR_RS_WIDE = 128;
constexpr int RR_NSTG = 5;   // ring slots (= stages resident at the turn)
// Rows per software-pipelined operand group (>= 2: the first group of a
// system holds its special rows 0 and 1). Measured (sweep_trace, 1024
// rows): RG 8 -> 27.3 / 36.3 cycles per row forward / backward, RG 4 ->
// 26.5 / 34.8, RG 2 -> 25.7 / 34.9 (chain floor 24.6 / 32.8); in the CH
// step (transposed-input sweeps) RG 4 is fastest: 88.4 us/step at 1024^2
// against 92.3 (RG 2) and 90.5 (RG 8).
#ifndef SG_SWEEP_RG
#define SG_SWEEP_RG 4
#endif
constexpr int RG = SG_SWEEP_RG;
static_assert(RG >= 2, "the first operand group must cover rows 0 and 1");
// XIN 1 (the CH y-sweep): the forward input is the x-sweep's output zT in
// ITS layout (zT[b*n + r]: system-major), fetched as 128 B-swizzled 16 x 32
// tensor boxes into two raw buffers; warp 1's 32 lanes transpose each stage
// into the slot while applying the x Woodbury correction — the separate
// transpose/correct pass (16 B/pt of traffic and a launch) disappears.
// XIN 2 (the CH x-sweep): the same transposed read with no correction — the
// RHS kernel then writes its output row-major (coalesced) instead of
// transposed. Four ring slots instead of five pay for the raw buffers; the
// TMA traffic moves to a fifth warp (the transform warps only transform).
// (CH step with 2 / 3 / 4 transform warps: 87.1 / 87.2 / 89.7 us at 1024^2,
// 1.154 / 1.152 / 1.157 ms at 8192^2.)
#ifndef SG_XIN_TW
#define SG_XIN_TW 3
#endif
constexpr int XIN_TW = SG_XIN_TW;  // transform warps (1..XIN_TW) of the XIN sweep
// Raw zT buffers of the XIN sweep (ring slots: 4 with two raw buffers, 3
// with three). With the TMA producer in its own warp, two suffice:
// sweep_trace at 8192^2 y / x-sweep 375 / 352 us (two) against 379 / 362
// (three), at 1024^2 70.5 k / 68.7 k cycles against 71.3 k / 69.7 k.
#ifndef SG_XIN_NRAW
#define SG_XIN_NRAW 2
#endif

template <int RS, int XIN = 0>
struct RRGeom {
  static constexpr int FAC = RS;  // doubles per uniform factor slot
  static constexpr int STAGE = RS * 32 + 5 * FAC;  // doubles per slot
  static_assert((STAGE * 8) % 128 == 0 && (FAC * 8) % 128 == 0, "TMA destinations must be 128 B aligned");
  static_assert(RS % RG == 0 && RS % 16 == 0, "stage = whole operand groups / swizzle boxes");
  // XIN: NRAW raw buffers (NRAW - 1 stages of zT in flight ahead of the
  // transform) and NST ring slots, within the two-CTAs-per-SM budget
  static constexpr int NRAW = XIN ? SG_XIN_NRAW : 0;
  static constexpr int NST = XIN ? (NRAW > 2 ? 3 : 4) : RR_NSTG;
  // doubles per raw buffer: RS/16 swizzled zT boxes of 4 KB, then the
  // stage's four y_k row vectors (1D TMA)
  static constexpr int RAW = XIN ? RS * 32 + 4 * RS : 0;
  static constexpr size_t RAW_OFF = static_cast<size_t>(NST) * STAGE * 8;  // bytes, before alignment
  static constexpr size_t SMEM =
      RAW_OFF + (XIN ? NRAW * RAW * 8 + 1024 : 0) + (XIN ? 3 * NST + 2 * NRAW : 2 * NST) * 8;
};

__device__ __forceinline__ void s_tma_store_2d(const CUtensorMap* m, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(x), "r"(y), "r"(s_u32(src))
               : "memory");
}

#ifdef SG_SWEEP_TRACE  // scripts/micro/sweep_trace.cu: per-stage clock64 of CTA 0's consumer
__device__ long long g_sweep_trace[8192];
#define SG_TRACE(i)                                                   \
  do {                                                                \
    if (blockIdx.x == 0 && lane == 0) g_sweep_trace[(i)] = clock64(); \
  } while (0)
#define SG_TRACE_X(i)                                                                  \
  do {                                                                                 \
    if (blockIdx.x == 0 && warp == 1 && lane == 0) g_sweep_trace[4096 + (i)] = clock64(); \
  } while (0)
#else
#define SG_TRACE_X(i) \
  do {                \
  } while (0)
#define SG_TRACE(i) \
  do {              \
  } while (0)
#endif

// Threads of one k_sweep_res CTA.
template <int XIN>
__host__ __device__ constexpr int sweep_res_threads() {
  return XIN ? 32 * (2 + XIN_TW) : 64;
}

// The sweep of one CTA (systems [32 cta, 32 cta + 32)). Called by every
// thread of a CTA of at least sweep_res_threads<XIN>() threads: surplus
// threads take part in the barrier that publishes the mbarrier
// initialisation, then leave. rr_smem: RRGeom<RS, XIN>::SMEM bytes of
// dynamic shared memory.
template <bool PERIODIC, int RS, int XIN>
__device__ __forceinline__ void sweep_res_body(const PentaTables& f, const SweepMaps& maps, int B, int n,
                                               double* __restrict__ y4, const SweepFuse& fuse, int cta,
                                               double* rr_smem) {
  using GEO = RRGeom<RS, XIN>;
  constexpr int NST = GEO::NST, FAC = GEO::FAC, STG = GEO::STAGE;
  constexpr uint32_t TX = RS * 32 * 8 + 5 * RS * 8;  // bytes per stage load
  constexpr uint32_t FTX = 5 * RS * 8;               // factor boxes only (XIN forward)
  // XIN raw buffers: 1024 B aligned (the 128 B swizzle pattern is a function
  // of the shared-memory address bits 4-9)
  double* raw = nullptr;
  uint64_t* full;
  if constexpr (XIN) {
    const uint32_t a = s_u32(rr_smem) + static_cast<uint32_t>(GEO::RAW_OFF);
    raw = rr_smem + (GEO::RAW_OFF + ((1024u - (a & 1023u)) & 1023u)) / 8;
    full = reinterpret_cast<uint64_t*>(rr_smem + (GEO::RAW_OFF + 1024 + GEO::NRAW * GEO::RAW * 8) / 8);
  } else {
    full = reinterpret_cast<uint64_t*>(rr_smem + NST * STG);
  }
  uint64_t* done = full + NST;
  uint64_t* rawfull = done + NST;             // XIN only: raw buffer loaded
  uint64_t* rawfree = rawfull + GEO::NRAW;     // XIN: raw buffer read by the transform
  uint64_t* slotfree = rawfree + GEO::NRAW;    // XIN: forward slot stored, writable
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = cta * 32;
  const int seg = maps.segRows ? static_cast<int>(blockIdx.y) : 0;
  const int rb0 = seg * maps.segRows;  // first row of this CTA's segment in z / zt / yc
  const int nS = (n + RS - 1) / RS;
  const int keep = nS < NST ? nS : NST;  // forward stages resident at the turn
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) {
      // XIN: every load of a slot completes on the TMA bytes AND a plain
      // arrival (the transform in the forward pass, immediate in backward)
      s_mbar_init(&full[k], XIN ? 1 + 32 * XIN_TW : 1);  // XIN: every transform thread arrives
      s_mbar_init(&done[k], 1);
    }
    if constexpr (XIN) {
      for (int k = 0; k < GEO::NRAW; ++k) {
        s_mbar_init(&rawfull[k], 1);
        s_mbar_init(&rawfree[k], 32 * XIN_TW);
      }
      for (int k = 0; k < NST; ++k) s_mbar_init(&slotfree[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= sweep_res_threads<XIN>()) return;
  // programmatic dependent launch: everything above touches only shared
  // memory; z and y4 belong to the predecessor kernels
  pdl_wait();
  // forward uses of ring slot s. full[s] completes once per load into s;
  // done[s] once per consumer use of s EXCEPT the resident forward stage
  auto uses = [&](int s) { return s < nS ? (nS - s + NST - 1) / NST : 0; };

  if (warp >= 1) {
    // ------------------------------------------------------------ producer
    // (warp 1 lane 0; with XIN, warp XIN_TW + 1 lane 0, while warps 1-3
    // run the forward transform)
    auto load = [&](int s, int G) {
      double* st = rr_smem + s * STG;
      s_mbar_expect_tx(&full[s], TX);
      s_tma_2d(st, &maps.z, b0, rb0 + G * RS, &full[s]);
      for (int k = 0; k < 5; ++k) s_tma_1d(st + RS * 32 + k * FAC, &maps.t[k], G * RS, &full[s]);
      if constexpr (XIN)  // no transform on refetched rows: the transform arrivals now
        s_mbar_arrive_cnt(&full[s], 32 * XIN_TW);
    };
    auto store = [&](int s, int G) {
      s_tma_store_2d(&maps.z, b0, rb0 + G * RS, rr_smem + s * STG);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };
    if constexpr (XIN) {
      constexpr int NR = GEO::NRAW;
      if (warp <= XIN_TW) {
        // forward stages, transform warps 1-3 (three SMSPs: the transform's
        // FP64 work is ~2x the consumer's per row): transpose (+ correct) the
        // raw zT boxes of stage g into slot g % NST (k_transpose_correct's
        // expression: z - (W0 y0 + W1 y1 + W2 y2 + W3 y3), penta.cpp:283-284)
        const int tw = warp - 1;  // transform warp 0..XIN_TW-1
        const int bl = b0 + lane;
        double Wb[4] = {0.0, 0.0, 0.0, 0.0};
        if constexpr (XIN == 1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) Wb[k] = bl < B ? __ldg(fuse.Wc[k] + bl) : 0.0;
        }
        for (int g = 0; g < nS; ++g) {
          const int s = g % NST;
          SG_TRACE_X(4 * g);
          // the slot's previous stage has been stored (read out by the TMA)
          if (g >= NST) s_mbar_wait(&slotfree[s], ((g / NST) - 1) & 1);
          SG_TRACE_X(4 * g + 1);
          s_mbar_wait(&rawfull[g % NR], (g / NR) & 1);
          SG_TRACE_X(4 * g + 2);
          const double* rb = raw + (g % NR) * GEO::RAW;
          double* zs = rr_smem + s * STG;
          // batches of TB row pairs, dealt round-robin to the transform warps:
          // all loads first, then the arithmetic (independent chains
          // interleave), then the stores
          constexpr int TB = 4;
          for (int jb = tw * TB; jb < RS / 2; jb += XIN_TW * TB) {
            double2 v[TB], y[TB][4];
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              const int jp = jb + t;
              // rows 2jp, 2jp+1 of system bl: box jp/8, 16 B chunk jp%8 of
              // smem row `lane`, XOR-swizzled by lane % 8
              v[t] = *reinterpret_cast<const double2*>(rb + (jp >> 3) * 512 + lane * 16 +
                                                       (((jp & 7) ^ (lane & 7)) << 1));
              if constexpr (XIN == 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // broadcast: every lane reads the same pair
                  y[t][k] = *reinterpret_cast<const double2*>(rb + RS * 32 + k * RS + 2 * jp);
              }
            }
            double o[TB][2];
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              if constexpr (XIN == 1) {
                const double c0 = Wb[0] * y[t][0].x + Wb[1] * y[t][1].x + Wb[2] * y[t][2].x + Wb[3] * y[t][3].x;
                const double c1 = Wb[0] * y[t][0].y + Wb[1] * y[t][1].y + Wb[2] * y[t][2].y + Wb[3] * y[t][3].y;
                o[t][0] = v[t].x - c0;
                o[t][1] = v[t].y - c1;
              } else {
                o[t][0] = v[t].x;
                o[t][1] = v[t].y;
              }
            }
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              zs[(2 * (jb + t)) * 32 + lane] = o[t][0];
              zs[(2 * (jb + t) + 1) * 32 + lane] = o[t][1];
            }
          }
          s_mbar_arrive(&full[s]);         // each thread releases its own slot writes
          s_mbar_arrive(&rawfree[g % NR]);  // ... and its reads of the raw buffer
          SG_TRACE_X(4 * g + 3);
        }
        return;
      }
      // warp XIN_TW + 1, lane 0: every TMA operation of the CTA. Forward
      // stage g: store slot g % NST (stage g - NST, once the consumer is
      // done with it) and hand it to the transform; the stage's factor rows;
      // the raw zT (+ y_k) rows of stage g + NR - 1 into the buffer that
      // stage g - 1's transform has released. (Issuing from a transform warp
      // serialised ~100 cycles per TMA operation and the store's smem read
      // into the transform loop: the chain waited 20 % of the 8192^2 y-sweep.)
      if (lane != 0) return;
      auto load_raw = [&](int g) {
        double* rb = raw + (g % NR) * GEO::RAW;
        s_mbar_expect_tx(&rawfull[g % NR], (RS * 32 + (XIN == 1 ? 4 * RS : 0)) * 8);
        if (maps.ztBox) {  // one 4D box: RS/16 chunks of 16 unknowns x 32 systems
          const int r = rb0 + g * RS;
          s_tma_4d(rb, &maps.zt, 0, b0, (r % maps.ztInner) / 16, r / maps.ztInner, &rawfull[g % NR]);
        } else {
          for (int x = 0; x < RS / 16; ++x) {
            const int r = rb0 + g * RS + x * 16;
            s_tma_3d(rb + x * 512, &maps.zt, r % maps.ztInner, b0, r / maps.ztInner, &rawfull[g % NR]);
          }
        }
        if constexpr (XIN == 1) {
          if (maps.ycSeg)  // the coefficient plane of the segment holding these systems
            s_tma_3d(rb + RS * 32, &maps.yc[0], rb0 + g * RS, 0, b0 / maps.ycSeg, &rawfull[g % NR]);
          else
            s_tma_2d(rb + RS * 32, &maps.yc[0], rb0 + g * RS, 0, &rawfull[g % NR]);
        }
      };
      for (int g = 0; g < NR - 1 && g < nS; ++g) load_raw(g);
      for (int g = 0; g < nS; ++g) {
        const int s = g % NST;
        if (g >= NST) {
          s_mbar_wait(&done[s], ((g / NST) + 1) & 1);
          store(s, g - NST);
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          s_mbar_arrive(&slotfree[s]);
        }
        s_mbar_expect_tx(&full[s], FTX);
        for (int k = 0; k < 5; ++k) s_tma_1d(rr_smem + s * STG + RS * 32 + k * FAC, &maps.t[k], g * RS, &full[s]);
        if (g + NR - 1 < nS) {
          if (g >= 1) s_mbar_wait(&rawfree[(g - 1) % NR], ((g - 1) / NR) & 1);
          load_raw(g + NR - 1);
        }
      }
    } else {
      if (lane != 0) return;
      // forward: loading stage g reuses the slot of stage g - NST, which is
      // stored first (it is never resident: g - NST < nS - NST)
      for (int g = 0; g < nS; ++g) {
        const int s = g % NST;
        if (g >= NST) {
          s_mbar_wait(&done[s], ((g / NST) + 1) & 1);
          store(s, g - NST);
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        load(s, g);
      }
    }
    // turn: every forward store has landed before those rows are refetched
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    // final (backward) results: into z, or (P2P) straight into the buffer of
    // the destination owning those unknowns — the distributed CH's
    // all-to-all, overlapped with the recurrence stage by stage
    auto fstore = [&](int s, int G) {
      if (maps.npeer == 0) {
        store(s, G);
        return;
      }
      const int r = G * RS, d = r / maps.prow;
      s_tma_store_2d(&maps.pz[d], b0, r - d * maps.prow, rr_smem + s * STG);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };
    // backward stage h (rows of forward stage G = nS-1-h) reuses the slot of
    // backward stage h - NST, which is stored first
    for (int h = keep; h < nS; ++h) {
      const int G = nS - 1 - h, s = G % NST;
      s_mbar_wait(&done[s], (uses(s) + h / NST) & 1);
      fstore(s, G + NST);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(s, G);
    }
    // the last NST backward stages (or all, for short systems)
    for (int h = nS - keep; h < nS; ++h) {
      const int G = nS - 1 - h, s = G % NST;
      s_mbar_wait(&done[s], (uses(s) + h / NST + 1) & 1);
      fstore(s, G);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }

  // -------------------------------------------------------------- consumer
  // Results go back with st.shared through asm WITHOUT a memory clobber (they
  // never alias a pending operand load); `finish` makes the slot's writes
  // visible to the async proxy and hands it to the producer.
  auto put = [&](uint32_t base, int k, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(base + k * 256), "d"(v));
  };
  auto finish = [&](int s) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) s_mbar_arrive(&done[s]);
  };
  // ---- forward (penta.cpp:171-181)
  double y2 = 0.0, y1 = 0.0;
  bool ready = false;  // stage known complete (tested one stage early)
  for (int g = 0; g < nS; ++g) {
    const int s = g % NST;
    SG_TRACE(3 * g);
    if (!ready) s_mbar_wait(&full[s], (g / NST) & 1);
    ready = g + 1 < nS && s_mbar_test(&full[(g + 1) % NST], ((g + 1) / NST) & 1);
    SG_TRACE(3 * g + 1);
    double* st = rr_smem + s * STG;
    const uint32_t sb = s_u32(st) + lane * 8;
    const double* m1 = st + RS * 32;
    const double* m2 = m1 + FAC;
    const int r0 = g * RS;
    // groups of RG rows from group J0 on: the operands of group j+1 are
    // loaded (and pinned there by the barrier) before group j's chain
    auto groups = [&](auto j0) {
      constexpr int J0 = decltype(j0)::value;
      double zr[2][RG], f0[2][RG], f1[2][RG];
#pragma unroll
      for (int k = 0; k < RG; ++k) {
        zr[J0 & 1][k] = st[(J0 * RG + k) * 32 + lane];
        f0[J0 & 1][k] = m1[J0 * RG + k];
        f1[J0 & 1][k] = m2[J0 * RG + k];
      }
#pragma unroll
      for (int j = J0; j < RS / RG; ++j) {
        const int c = j & 1;
        if (j + 1 < RS / RG) {
#pragma unroll
          for (int k = 0; k < RG; ++k) {
            const int kk = (j + 1) * RG + k;
            zr[c ^ 1][k] = st[kk * 32 + lane];
            f0[c ^ 1][k] = m1[kk];
            f1[c ^ 1][k] = m2[kk];
          }
        }
        asm volatile("" ::: "memory");
#pragma unroll
        for (int k = 0; k < RG; ++k) {
          const double yr = zr[c][k] - (f0[c][k] * y2 + f1[c][k] * y1);  // penta.cpp:180
          put(sb, j * RG + k, yr);
          y2 = y1;
          y1 = yr;
        }
      }
    };
    if (r0 >= 2 && r0 + RS <= n) {
      groups(std::integral_constant<int, 0>{});
    } else if (r0 == 0 && RS <= n) {
      // rows 0 and 1 are special (penta.cpp:173-175): first group scalar
#pragma unroll
      for (int k = 0; k < RG; ++k) {
        const double zr = st[k * 32 + lane];
        double yr;
        if (k >= 2) yr = zr - (m1[k] * y2 + m2[k] * y1);
        else if (k == 1) yr = zr - m2[k] * y1;  // y1 holds y[0]
        else yr = zr;
        put(sb, k, yr);
        y2 = y1;
        y1 = yr;
      }
      groups(std::integral_constant<int, 1>{});
    } else {
#pragma unroll 8
      for (int k = 0; k < RS; ++k) {
        const int r = r0 + k;
        const double zr = st[k * 32 + lane];
        double yr;
        if (r >= 2) yr = zr - (m1[k] * y2 + m2[k] * y1);
        else if (r == 1) yr = zr - m2[k] * y1;  // y1 holds y[0]
        else yr = zr;
        put(sb, k, yr);
        y2 = y1;
        y1 = yr;
      }
    }
    SG_TRACE(3 * g + 2);
    // resident stages (the last `keep`) stay with the consumer
    if (g < nS - keep) finish(s);
  }
  __syncwarp();
  // ---- backward (penta.cpp:183-196), resident stages first
  double s1 = 0.0, s2 = 0.0, zn1 = 0.0, zn2 = 0.0, zz0 = 0.0, zz1 = 0.0;
  ready = false;
  for (int h = 0; h < nS; ++h) {
    const int G = nS - 1 - h, s = G % NST;
    SG_TRACE(3 * (nS + h));
    if (h >= keep && !ready) s_mbar_wait(&full[s], (uses(s) + h / NST + 1) & 1);
    if (h + 1 >= keep && h + 1 < nS) {
      const int sn = (nS - 2 - h) % NST;
      ready = s_mbar_test(&full[sn], (uses(sn) + (h + 1) / NST + 1) & 1);
    }
    SG_TRACE(3 * (nS + h) + 1);
    double* st = rr_smem + s * STG;
    const uint32_t sb = s_u32(st) + lane * 8;
    const double* dI = st + RS * 32 + 2 * FAC;
    const double* ap = dI + FAC;
    const double* bp = ap + FAC;
    const int r0 = G * RS;
    // groups of RG rows from the top of the stage down (group J0 on),
    // pipelined as in the forward pass
    auto groups = [&](auto j0) {
      constexpr int J0 = decltype(j0)::value;
      double yv[2][RG], di[2][RG], fa[2][RG], fb[2][RG];
#pragma unroll
      for (int k = 0; k < RG; ++k) {
        const int kk = RS - 1 - (J0 * RG + k);
        yv[J0 & 1][k] = st[kk * 32 + lane];
        di[J0 & 1][k] = dI[kk];
        fa[J0 & 1][k] = ap[kk];
        fb[J0 & 1][k] = bp[kk];
      }
#pragma unroll
      for (int j = J0; j < RS / RG; ++j) {
        const int c = j & 1;
        if (j + 1 < RS / RG) {
#pragma unroll
          for (int k = 0; k < RG; ++k) {
            const int kk = RS - 1 - ((j + 1) * RG + k);
            yv[c ^ 1][k] = st[kk * 32 + lane];
            di[c ^ 1][k] = dI[kk];
            fa[c ^ 1][k] = ap[kk];
            fb[c ^ 1][k] = bp[kk];
          }
        }
        asm volatile("" ::: "memory");
#pragma unroll
        for (int k = 0; k < RG; ++k) {
          const double yr = (yv[c][k] - fa[c][k] * s1 - fb[c][k] * s2) * di[c][k];  // penta.cpp:193-195
          put(sb, RS - 1 - (j * RG + k), yr);
          s2 = s1;
          s1 = yr;
        }
      }
      if (r0 == 0) {  // rows 0 and 1 closed the chain: the Woodbury inputs
        zz0 = s1;
        zz1 = s2;
      }
    };
    if (r0 + RS <= n - 2) {
      groups(std::integral_constant<int, 0>{});
    } else if (r0 + RS == n && n >= RG + 2) {
      // rows n-1 and n-2 are special (penta.cpp:184-186): top group scalar
#pragma unroll
      for (int k = RS - 1; k >= RS - RG; --k) {
        const double yv = st[k * 32 + lane];
        double yr;
        if (k == RS - 1) {
          yr = yv * dI[k];
          zn1 = yr;
        } else if (k == RS - 2) {
          yr = (yv - ap[k] * s1) * dI[k];
          zn2 = yr;
        } else {
          yr = (yv - ap[k] * s1 - bp[k] * s2) * dI[k];
        }
        put(sb, k, yr);
        s2 = s1;
        s1 = yr;
      }
      groups(std::integral_constant<int, 1>{});
    } else {
#pragma unroll 8
      for (int k = RS - 1; k >= 0; --k) {
        const int r = r0 + k;
        if (r >= n) continue;
        const double yv = st[k * 32 + lane];
        double yr;
        if (r == n - 1) {
          yr = yv * dI[k];
          zn1 = yr;
        } else if (r == n - 2) {
          yr = (yv - ap[k] * s1) * dI[k];
          zn2 = yr;
        } else {
          yr = (yv - ap[k] * s1 - bp[k] * s2) * dI[k];
        }
        if (r == 1) zz1 = yr;
        if (r == 0) zz0 = yr;
        put(sb, k, yr);
        s2 = s1;
        s1 = yr;
      }
    }
    SG_TRACE(3 * (nS + h) + 2);
    finish(s);
  }
  if constexpr (PERIODIC) {
    const int b = b0 + lane;
    if (b >= B) return;
    const double* cw = f.cw;
    double y[4];
    y[0] = cw[0] * zn2 + cw[1] * zn1;
    y[1] = cw[2] * zn1;
    y[2] = cw[3] * zz0;
    y[3] = cw[4] * zz0 + cw[5] * zz1;
    lu4_solve_dev(f.K, f.piv, y);
    const long long sB = B;
#pragma unroll
    for (int k = 0; k < 4; ++k) y4[k * sB + b] = y[k];
    for (int d = 0; d < maps.npeer; ++d)
      if (fuse.py4[d])
#pragma unroll
        for (int k = 0; k < 4; ++k) fuse.py4[d][static_cast<long long>(k) * fuse.y4Stride + fuse.y4Off + b] = y[k];
  } else {
    if (maps.segRows) {  // interface values of this (segment, system)
      const int b = b0 + lane;
      if (b >= B) return;
      const long long sB = B, o = static_cast<long long>(seg) * 4 * sB + b;
      y4[o] = zz0;
      y4[o + sB] = zz1;
      y4[o + 2 * sB] = zn2;
      y4[o + 3 * sB] = zn1;
    }
  }
}

template <bool PERIODIC, int RS, int XIN>
__global__ void __launch_bounds__(sweep_res_threads<XIN>()) k_sweep_res(const PentaTables f,
                                                                       const __grid_constant__ SweepMaps maps, int B,
                                                                       int n, double* __restrict__ y4,
                                                                       const SweepFuse fuse) {
  extern __shared__ __align__(128) double rr_smem[];
  sweep_res_body<PERIODIC, RS, XIN>(f, maps, B, n, y4, fuse, blockIdx.x, rr_smem);
}

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return encode;
}

inline bool encode_map(CUtensorMap* m, const double* p, int rank, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1,
                bool swizzle128 = false) {
  auto enc = tensor_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {d0 * 8};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// zT (system-major, blocks of ztInner unknowns per system) as 4D {16, B,
// ztInner / 16, n / ztInner}, box {16, 32, rs / 16, 1}, 128 B swizzle: the
// box lands as rs/16 consecutive 4 KB [32 systems][16 unknowns] chunks.
inline bool encode_map4_zt(CUtensorMap* m, const double* p, int ztInner, int B, int n, int rs) {
  auto enc = tensor_encoder();
  if (!enc) return false;
  const cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(B), static_cast<cuuint64_t>(ztInner / 16),
                              static_cast<cuuint64_t>(n / ztInner)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ztInner) * 8, 128,
                                 static_cast<cuuint64_t>(B) * ztInner * 8};
  const cuuint32_t box[4] = {16, 32, static_cast<cuuint32_t>(rs / 16), 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool encode_map3(CUtensorMap* m, const double* p, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                 uint32_t b2, bool swizzle128) {
  auto enc = tensor_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA path needs 16 B aligned rows (B even, aligned pointers) and a driver
// tensor-map encoder; otherwise the register-prefetch k_sweep runs.
inline bool sweep_maps(const PentaTables& f, int B, int n, const double* z, SweepMaps* maps, int rows = 32) {
  if (B % 2 != 0 || (reinterpret_cast<uintptr_t>(z) & 15)) return false;
  if (std::getenv("SG_SWEEP_KERNEL") && std::strcmp(std::getenv("SG_SWEEP_KERNEL"), "reg") == 0) return false;
  *maps = SweepMaps{};
  if (!encode_map(&maps->z, z, 2, B, n, 32, rows)) return false;
  const double* t[5] = {f.m1, f.m2, f.dInv, f.ap, f.bp};
  for (int k = 0; k < 5; ++k) {
    if (reinterpret_cast<uintptr_t>(t[k]) & 15) return false;
    const bool ok = f.uniform ? encode_map(&maps->t[k], t[k], 1, n, 1, rows, 1)
                              : encode_map(&maps->t[k], t[k], 2, B, n, 32, rows);
    if (!ok) return false;
  }
  return true;
}

// Stage height for a batch of B systems (one CTA per 32 systems).
inline int sweep_res_rows(int B) {
  static const int sms = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  const char* e = std::getenv("SG_SWEEP_RS");
  if (e) return std::atoi(e) == RR_RS_WIDE ? RR_RS_WIDE : RR_RS;
  return (B + 31) / 32 <= sms ? RR_RS_WIDE : RR_RS;
}

// Tensor maps and fusion arguments of a transposed-input sweep
// (penta_sweep_xin). Returns false if the path is unavailable.
inline bool xin_prepare(const PentaTables& f, int B, int n, double* z, const double* zT, const double* const* Wc,
                        const double* yc, int ztInner, const SweepPeers* peers, SweepMaps* maps, SweepFuse* fuse,
                        int* rsOut) {
  // Uniform periodic operator, resident-turn sweep only (the CH sweeps).
  if (!f.uniform) return false;
  if (ztInner <= 0) ztInner = n;
  if ((reinterpret_cast<uintptr_t>(zT) & 15) || (n & 1) || n % ztInner || ztInner % 16) return false;
  if (Wc && (reinterpret_cast<uintptr_t>(yc) & 15)) return false;
  const int rs = sweep_res_rows(B);
  *rsOut = rs;
  if (!sweep_maps(f, B, n, z, maps, rs)) return false;
  // zT: unknown r of system b at ((r % ztInner), b, r / ztInner) — dims
  // {ztInner, B, n / ztInner}, box {16 unknowns, 32 systems, 1}, 128 B swizzle
  // One 4D box per stage where the stage's rows lie in one block: the view
  // {16 unknowns, B systems, ztInner / 16 chunks, n / ztInner blocks}
  // (strides 8 B, ztInner * 8, 128 B, B * ztInner * 8). Else RS/16 3D boxes.
  maps->ztBox = ztInner % rs == 0 && encode_map4_zt(&maps->zt, zT, ztInner, B, n, rs) ? 1 : 0;
  if (!maps->ztBox && !encode_map3(&maps->zt, zT, ztInner, B, n / ztInner, 16, 32, 1, true)) return false;
  maps->ztInner = ztInner;
  if (peers && peers->npeer > 0) {
    if (peers->npeer > 8 || peers->prow % rs || n != peers->npeer * peers->prow) return false;
    for (int d = 0; d < peers->npeer; ++d) {
      if (reinterpret_cast<uintptr_t>(peers->dst[d]) & 15) return false;
      if (!encode_map(&maps->pz[d], peers->dst[d], 2, B, peers->prow, 32, rs)) return false;
    }
    maps->npeer = peers->npeer;
    maps->prow = peers->prow;
  }
  if (peers && peers->npeer > 0) {
    for (int d = 0; d < peers->npeer; ++d) fuse->py4[d] = peers->y4[d];
    fuse->y4Stride = peers->y4Stride;
    fuse->y4Off = peers->y4Off;
  }
  if (Wc) {
    if (!encode_map(&maps->yc[0], yc, 2, n, 4, rs, 4)) return false;
    for (int k = 0; k < 4; ++k) fuse->Wc[k] = Wc[k];
    fuse->yc = yc;
  }
  return true;
}

}  // namespace
}  // namespace sg
