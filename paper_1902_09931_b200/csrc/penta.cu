// penta.cu — batched (cyclic) pentadiagonal solves on sm_100a.
//
// Replaces PentaFactor / PeriodicPentaFactor (penta.cpp:93-295). Layout is
// the reference's interleaved one, idx(b, r) = r*B + b (penta.hpp:12-32), so
// with ONE SYSTEM PER THREAD every row access of a warp is a coalesced
// 32-system segment. Arithmetic is the reference's, term for term, compiled
// without FMA contraction: solutions are bitwise identical.
//
// Uniform operators (every system has the same bands — the Cahn-Hilliard
// case, penta.cpp:313-335) keep the factor as n-vectors read by all threads
// as warp-uniform broadcasts; otherwise factor arrays are per system.
//
// Kernels:
//   k_factor        non-pivoting LU per system (penta.cpp:93-158); records the
//                   first zero-pivot row per system.
//   k_periodic_setup W_k = P^{-1} e_{0,1,n-2,n-1} (penta.cpp:219-227),
//                   capacitance K = I + V^T W and its 4x4 partial-pivot LU
//                   (penta.cpp:229-250, lu4_factor :37-59).
//   k_sweep         forward + backward substitution (penta.cpp:160-197) with a
//                   register prefetch ring (the recurrence is latency-bound,
//                   loads are not on the dependency chain); periodic systems
//                   then compute y = K^{-1} V^T z (penta.cpp:262-274) and either
//                   apply z -= W y in place (penta.cpp:279-286) or hand y to a
//                   fused consumer (the CH transpose/combine kernels).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "penta.cuh"
#include "sg_internal.hpp"
#include "sweep_res.cuh"

namespace sg {

namespace {

constexpr int SWEEP_THREADS = 32;  // one warp per CTA: spreads the few systems over SMs

// penta.cpp:93-158, one thread per system. bands interleaved with stride B.
__global__ void k_factor(int B, int n, const double* __restrict__ e, const double* __restrict__ c,
                         const double* __restrict__ d, const double* __restrict__ a,
                         const double* __restrict__ bb, double* __restrict__ m1,
                         double* __restrict__ m2, double* __restrict__ dInv,
                         double* __restrict__ ap, double* __restrict__ bp, int* __restrict__ badRow) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int bad = n;
  // r = 0
  double dp2 = d[b];
  double ap2 = a[b];
  double bp2 = bb[b];
  if (dp2 == 0.0 && bad == n) bad = 0;
  m1[b] = 0.0;
  m2[b] = 0.0;
  ap[b] = ap2;
  bp[b] = bp2;
  dInv[b] = 1.0 / dp2;
  // r = 1
  const long long r1 = B + b;
  const double mm = c[r1] / dp2;
  double dp1 = d[r1] - mm * ap2;
  double ap1 = a[r1] - mm * bp2;
  double bp1 = bb[r1];
  if (dp1 == 0.0 && bad == n) bad = 1;
  m1[r1] = 0.0;
  m2[r1] = mm;
  ap[r1] = ap1;
  bp[r1] = bp1;
  dInv[r1] = 1.0 / dp1;
  // the next row's bands are loaded one row ahead: the chain (two dependent
  // divisions per row) then never waits on a global load
  double ne = 0.0, nc = 0.0, nd = 0.0, na = 0.0, nb = 0.0;
  if (n > 2) {
    const long long r2 = 2LL * B + b;
    ne = e[r2], nc = c[r2], nd = d[r2], na = a[r2], nb = bb[r2];
  }
#pragma unroll 2
  for (int r = 2; r < n; ++r) {
    const long long cur = static_cast<long long>(r) * B + b;
    const double ec = ne, cc = nc, dc = nd, ac = na, bc = nb;
    if (r + 1 < n) {
      const long long nx = cur + B;
      ne = e[nx], nc = c[nx], nd = d[nx], na = a[nx], nb = bb[nx];
    }
    const double mm1 = ec / dp2;
    const double cbar = cc - mm1 * ap2;
    const double mm2 = cbar / dp1;
    const double dpc = dc - mm1 * bp2 - mm2 * ap1;
    const double apc = ac - mm2 * bp1;
    const double bpc = bc;
    m1[cur] = mm1;
    m2[cur] = mm2;
    ap[cur] = apc;
    bp[cur] = bpc;
    dInv[cur] = 1.0 / dpc;
    if (dpc == 0.0 && bad == n) bad = r;
    dp2 = dp1;
    ap2 = ap1;
    bp2 = bp1;
    dp1 = dpc;
    ap1 = apc;
    bp1 = bpc;
  }
  badRow[b] = bad;
}

// Table element for system b, row r.
__device__ __forceinline__ double tab(const double* __restrict__ t, int r, int b, int B, bool uniform) {
  return uniform ? __ldg(t + r) : __ldg(t + static_cast<long long>(r) * B + b);
}

// One substitution pass pair on a strided vector (used for setup only): the
// same expressions as the sweeps (penta.cpp:171-196), the two previous
// unknowns carried in registers (re-reading them from global memory put a
// load round trip on every row: 2.25 ms for the n = 8192 setup).
__device__ void substitute(const PentaTables& f, int B, int b, double* y, long long s, int n) {
  const bool u = f.uniform;
  double y2 = y[0];
  double y1 = y[s] - tab(f.m2, 1, b, B, u) * y2;
  y[s] = y1;
#pragma unroll 4
  for (int r = 2; r < n; ++r) {
    const double yr = y[r * s] - (tab(f.m1, r, b, B, u) * y2 + tab(f.m2, r, b, B, u) * y1);
    y[r * s] = yr;
    y2 = y1;
    y1 = yr;
  }
  double s1 = y1 * tab(f.dInv, n - 1, b, B, u);
  y[(n - 1) * s] = s1;
  double s2 = s1;
  s1 = (y[(n - 2) * s] - tab(f.ap, n - 2, b, B, u) * s2) * tab(f.dInv, n - 2, b, B, u);
  y[(n - 2) * s] = s1;
#pragma unroll 4
  for (int r = n - 3; r >= 0; --r) {
    const double yr = (y[r * s] - tab(f.ap, r, b, B, u) * s1 - tab(f.bp, r, b, B, u) * s2) * tab(f.dInv, r, b, B, u);
    y[r * s] = yr;
    s2 = s1;
    s1 = yr;
  }
}

// lu4_factor, penta.cpp:37-59. Returns false if singular.
__device__ bool lu4_factor(double* K, int* piv) {
  for (int c = 0; c < 4; ++c) {
    int pr = c;
    double best = fabs(K[c * 4 + c]);
    for (int r = c + 1; r < 4; ++r) {
      const double cand = fabs(K[r * 4 + c]);
      if (cand > best) {
        best = cand;
        pr = r;
      }
    }
    if (best == 0.0) return false;
    piv[c] = pr;
    if (pr != c)
      for (int cc = 0; cc < 4; ++cc) {
        const double t = K[c * 4 + cc];
        K[c * 4 + cc] = K[pr * 4 + cc];
        K[pr * 4 + cc] = t;
      }
    const double inv = 1.0 / K[c * 4 + c];
    for (int r = c + 1; r < 4; ++r) {
      const double m = K[r * 4 + c] * inv;
      K[r * 4 + c] = m;
      for (int cc = c + 1; cc < 4; ++cc) K[r * 4 + cc] -= m * K[c * 4 + cc];
    }
  }
  return true;
}

// penta.cpp:204-251, one thread per system (uniform: a single thread).
// The four core solves W_k = P^{-1} e_{0,1,n-2,n-1} of every system
// (penta.cpp:219-227) are independent: blockIdx.y = k, one thread per
// system and k (4x the parallelism of one thread per system).
__global__ void k_periodic_core(PentaTables f, int B, int n, double* W0, double* W1, double* W2, double* W3) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int k = blockIdx.y;
  const long long s = B;
  double* Wk = (k == 0 ? W0 : k == 1 ? W1 : k == 2 ? W2 : W3) + b;
  const int row = k == 0 ? 0 : k == 1 ? 1 : k == 2 ? n - 2 : n - 1;
  for (int r = 0; r < n; ++r) Wk[r * s] = 0.0;
  Wk[row * s] = 1.0;
  substitute(f, B, b, Wk, s, n);
}

// Corner coefficients, capacitance K = I + V^T W and its 4x4 LU
// (penta.cpp:210-217, 229-250) from the W_k of k_periodic_core.
__global__ void k_periodic_setup(PentaTables f, int B, int n, const double* __restrict__ e,
                                 const double* __restrict__ c, const double* __restrict__ a,
                                 const double* __restrict__ bb, double* W0, double* W1, double* W2,
                                 double* W3, double* cw, double* K, int* piv, int* singular) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int nsys = f.uniform ? 1 : B;
  if (b >= nsys) return;
  const long long s = f.uniform ? 1 : B;
  double* Wk[4] = {W0 + b, W1 + b, W2 + b, W3 + b};
  double cwl[6] = {e[b], c[b], e[s + b], bb[(n - 2) * s + b], a[(n - 1) * s + b], bb[(n - 1) * s + b]};
  for (int k = 0; k < 6; ++k) cw[b * 6 + k] = cwl[k];
  double Kl[16];
  for (int k = 0; k < 4; ++k) {
    const double w0 = Wk[k][0], w1 = Wk[k][s], wn2 = Wk[k][(n - 2) * s], wn1 = Wk[k][(n - 1) * s];
    Kl[0 * 4 + k] = cwl[0] * wn2 + cwl[1] * wn1;
    Kl[1 * 4 + k] = cwl[2] * wn1;
    Kl[2 * 4 + k] = cwl[3] * w0;
    Kl[3 * 4 + k] = cwl[4] * w0 + cwl[5] * w1;
  }
  for (int r = 0; r < 4; ++r) Kl[r * 4 + r] += 1.0;
  int pv[4] = {0, 1, 2, 3};
  singular[b] = lu4_factor(Kl, pv) ? 0 : 1;
  for (int k = 0; k < 16; ++k) K[b * 16 + k] = Kl[k];
  for (int k = 0; k < 4; ++k) piv[b * 4 + k] = pv[k];
}

// Uniform operator: the four core solves W_k = P^{-1} e_{0,1,n-2,n-1} are
// independent — one thread each — then thread 0 builds K (penta.cpp:204-251).
__global__ void k_periodic_setup_uniform(PentaTables f, int n, const double* __restrict__ e,
                                         const double* __restrict__ c, const double* __restrict__ a,
                                         const double* __restrict__ bb, double* W0, double* W1, double* W2,
                                         double* W3, double* cw, double* K, int* piv, int* singular) {
  const int k = threadIdx.x;
  double* Wk[4] = {W0, W1, W2, W3};
  const int rowOf[4] = {0, 1, n - 2, n - 1};
  if (k < 4) {
    for (int r = 0; r < n; ++r) Wk[k][r] = 0.0;
    Wk[k][rowOf[k]] = 1.0;
    substitute(f, 1, 0, Wk[k], 1, n);
  }
  __syncthreads();
  if (k != 0) return;
  double cwl[6] = {e[0], c[0], e[1], bb[n - 2], a[n - 1], bb[n - 1]};
  for (int q = 0; q < 6; ++q) cw[q] = cwl[q];
  double Kl[16];
  for (int q = 0; q < 4; ++q) {
    const double w0 = Wk[q][0], w1 = Wk[q][1], wn2 = Wk[q][n - 2], wn1 = Wk[q][n - 1];
    Kl[0 * 4 + q] = cwl[0] * wn2 + cwl[1] * wn1;
    Kl[1 * 4 + q] = cwl[2] * wn1;
    Kl[2 * 4 + q] = cwl[3] * w0;
    Kl[3 * 4 + q] = cwl[4] * w0 + cwl[5] * w1;
  }
  for (int r = 0; r < 4; ++r) Kl[r * 4 + r] += 1.0;
  int pv[4] = {0, 1, 2, 3};
  singular[0] = lu4_factor(Kl, pv) ? 0 : 1;
  for (int q = 0; q < 16; ++q) K[q] = Kl[q];
  for (int q = 0; q < 4; ++q) piv[q] = pv[q];
}

}  // namespace

namespace {

constexpr int PF = 16;  // prefetch distance (rows) of the substitution sweeps

// Forward + backward substitution for system b over z (stride B), then the
// periodic correction. MODE 0: in place; MODE 1: write y (4 per system,
// layout y4[k*B + b]) for a fused consumer.
template <bool UNIFORM, bool PERIODIC, int MODE>
__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep(const PentaTables f, int B, int n,
                                                          double* __restrict__ z,
                                                          double* __restrict__ y4) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const long long sB = B;
  double* zc = z + b;
  // ---- forward: y[r] -= m1[r]*y[r-2] + m2[r]*y[r-1]
  double y2 = zc[0];
  double y1 = zc[sB] - tab(f.m2, 1, b, B, UNIFORM) * y2;
  zc[sB] = y1;
  const double z0 = y2;
  double ring[PF];
  double rm1[PF], rm2[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int r = 2 + k;
    if (r < n) {
      ring[k] = zc[r * sB];
      rm1[k] = tab(f.m1, r, b, B, UNIFORM);
      rm2[k] = tab(f.m2, r, b, B, UNIFORM);
    }
  }
  for (int r0 = 2; r0 < n; r0 += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int r = r0 + k;
      if (r < n) {
        const double yr = ring[k] - (rm1[k] * y2 + rm2[k] * y1);
        zc[r * sB] = yr;
        const int rn = r + PF;
        if (rn < n) {
          ring[k] = zc[rn * sB];
          rm1[k] = tab(f.m1, rn, b, B, UNIFORM);
          rm2[k] = tab(f.m2, rn, b, B, UNIFORM);
        }
        y2 = y1;
        y1 = yr;
      }
    }
  }
  // ---- backward
  const double zn1 = y1 * tab(f.dInv, n - 1, b, B, UNIFORM);
  zc[(n - 1) * sB] = zn1;
  const double zn2 = (y2 - tab(f.ap, n - 2, b, B, UNIFORM) * zn1) * tab(f.dInv, n - 2, b, B, UNIFORM);
  zc[(n - 2) * sB] = zn2;
  double s1 = zn2, s2 = zn1;  // y[r+1], y[r+2]
  double rap[PF], rbp[PF], rdi[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int r = n - 3 - k;
    if (r >= 0) {
      ring[k] = zc[r * sB];
      rap[k] = tab(f.ap, r, b, B, UNIFORM);
      rbp[k] = tab(f.bp, r, b, B, UNIFORM);
      rdi[k] = tab(f.dInv, r, b, B, UNIFORM);
    }
  }
  for (int r0 = n - 3; r0 >= 0; r0 -= PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int r = r0 - k;
      if (r >= 0) {
        const double yr = (ring[k] - rap[k] * s1 - rbp[k] * s2) * rdi[k];
        zc[r * sB] = yr;
        const int rn = r - PF;
        if (rn >= 0) {
          ring[k] = zc[rn * sB];
          rap[k] = tab(f.ap, rn, b, B, UNIFORM);
          rbp[k] = tab(f.bp, rn, b, B, UNIFORM);
          rdi[k] = tab(f.dInv, rn, b, B, UNIFORM);
        }
        s2 = s1;
        s1 = yr;
      }
    }
  }
  (void)z0;
  if constexpr (PERIODIC) {
    // y = K^{-1} V^T z (penta.cpp:262-274)
    const double zz0 = s1, zz1 = s2;  // final y[0], y[1]
    const int sys = UNIFORM ? 0 : b;
    const double* cw = f.cw + sys * 6;
    double y[4];
    y[0] = cw[0] * zn2 + cw[1] * zn1;
    y[1] = cw[2] * zn1;
    y[2] = cw[3] * zz0;
    y[3] = cw[4] * zz0 + cw[5] * zz1;
    lu4_solve_dev(f.K + sys * 16, f.piv + sys * 4, y);
    if constexpr (MODE == 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) y4[k * sB + b] = y[k];
    } else {
      // z -= W0 y0 + W1 y1 + W2 y2 + W3 y3 (penta.cpp:279-286)
      for (int r = 0; r < n; ++r) {
        const long long idx = r * sB;
        const double w0 = tab(f.W[0], r, b, B, UNIFORM), w1 = tab(f.W[1], r, b, B, UNIFORM),
                     w2 = tab(f.W[2], r, b, B, UNIFORM), w3 = tab(f.W[3], r, b, B, UNIFORM);
        zc[idx] -= w0 * y[0] + w1 * y[1] + w2 * y[2] + w3 * y[3];
      }
    }
  }
}

// ------------------------------------------------------------ k_sweep_tma
// The latency-bound recurrence path, TMA-fed: one warp = 32 systems; the
// rows of z (and of the factor tables) stream into a shared-memory ring of
// NSTG stages x RS rows through 2D/1D tensor copies (one elected lane, one
// mbarrier per stage), NSTG*RS = 64 rows ahead of the dependency chain, so
// each unknown costs only the FP64 latency of its 3 (forward) or 4
// (backward) dependent ops. Forward results go to z with coalesced stores
// and come back through the same ring for the backward pass (a proxy fence
// orders the generic stores before the async-proxy reads).
constexpr int SW_RS = 32;   // rows per stage
constexpr int SW_NSTG = 4;  // stages in flight

struct SweepSmem {
  // doubles per factor table per stage (per-system tables: one RS x 32 box)
  static constexpr int FAC = SW_RS * 32;
  static constexpr int STAGE = SW_RS * 32 + 3 * FAC;
  static constexpr int STAGE_PAD = (STAGE * 8 + 127) / 128 * 16;  // doubles, 128 B aligned stride
  static constexpr size_t bytes = static_cast<size_t>(SW_NSTG) * STAGE_PAD * 8 + 2 * SW_NSTG * 8;
};

template <bool PERIODIC, int MODE>
__global__ void __launch_bounds__(64) k_sweep_tma(const PentaTables f, const __grid_constant__ SweepMaps maps,
                                                  int B, int n, double* __restrict__ z, double* __restrict__ y4) {
  // Warp 0: consumer (32 systems, the dependency chain). Warp 1 lane 0:
  // producer (tensor-TMA issue), so the chain never stalls on issue code.
  using SM = SweepSmem;
  extern __shared__ __align__(128) double sw_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sw_smem + SW_NSTG * SM::STAGE_PAD);
  uint64_t* empty = full + SW_NSTG;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int b0 = blockIdx.x * 32;
  const int b = b0 + lane;
  const bool active = b < B;
  constexpr int FAC = SM::FAC;
  constexpr int RS = SW_RS;
  constexpr uint32_t ZB = RS * 32 * 8;
  constexpr uint32_t FB = RS * 32 * 8;  // bytes per factor box
  const int nS = (n + RS - 1) / RS;  // stages per pass
  const int total = 2 * nS;
  if (threadIdx.x == 0) {
    for (int k = 0; k < SW_NSTG; ++k) {
      s_mbar_init(&full[k], 1);
      s_mbar_init(&empty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == 1) {
    // ------------------------------------------------------------ producer
    for (int g = 0; g < total; ++g) {
      const int slot = g % SW_NSTG;
      if (g == nS) {
        // backward stages read the forward results: wait until the consumer
        // has stored them all and fenced them to the async proxy
        // non-.aligned form: lane 0 ran the issue code (independent thread
        // scheduling); every one of the 64 threads arrives individually
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      if (lane == 0) {
        if (g >= SW_NSTG) s_mbar_wait(&empty[slot], ((g / SW_NSTG) + 1) & 1);
        const int pass = g < nS ? 0 : 1;
        const int gg = g < nS ? g : g - nS;
        double* st = sw_smem + slot * SM::STAGE_PAD;
        const int r0 = pass == 0 ? gg * RS : n - (gg + 1) * RS;
        const int nt = pass == 0 ? 2 : 3;
        s_mbar_expect_tx(&full[slot], ZB + nt * FB);
        s_tma_2d(st, &maps.z, b0, r0, &full[slot]);
        for (int k = 0; k < nt; ++k) {
          const CUtensorMap* m = &maps.t[pass == 0 ? k : 2 + k];  // fwd: m1, m2; bwd: dInv, ap, bp
          s_tma_2d(st + RS * 32 + k * FAC, m, b0, r0, &full[slot]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumer
  auto fac = [&](const double* st, int k, int row) -> double {
    return st[RS * 32 + k * FAC + row * 32 + lane];
  };
  auto zin = [&](const double* st, int k) -> double { return st[k * 32 + lane]; };
  double* zc = z + b;
  const long long sB = B;
  // ---- forward (penta.cpp:171-181): stage 0 peeled (rows 0, 1 special)
  double y2 = 0.0, y1 = 0.0;
  {
    s_mbar_wait(&full[0], 0);
    const double* st = sw_smem;
#pragma unroll
    for (int k = 0; k < RS; ++k) {
      const double zr = zin(st, k);
      double yr;
      if (k >= 2)
        yr = zr - (fac(st, 0, k) * y2 + fac(st, 1, k) * y1);
      else if (k == 1)
        yr = zr - fac(st, 1, k) * y1;  // y1 holds y[0]
      else
        yr = zr;
      if (active && k >= 1 && k < n) zc[k * sB] = yr;  // row 0 is unchanged by the forward pass
      y2 = y1;
      y1 = yr;
    }
    __syncwarp();
    if (lane == 0) s_mbar_arrive(&empty[0]);
  }
  // Full stages run branch-free with a walking store pointer (the loop is
  // issue-bound: one warp per SM sub-partition, every instruction counts).
  double* zp = zc + RS * sB;
  const long long step = sB;
  bool ready = false;  // stage g known complete (tested one stage early)
  for (int g = 1; g < nS; ++g) {
    const int slot = g % SW_NSTG;
    if (!ready) s_mbar_wait(&full[slot], (g / SW_NSTG) & 1);
    ready = g + 1 < nS && s_mbar_test(&full[(g + 1) % SW_NSTG], ((g + 1) / SW_NSTG) & 1);
    const double* st = sw_smem + slot * SM::STAGE_PAD;
    const int r0 = g * RS;
    if (r0 + RS <= n) {
      // all operands of the stage first (the compiler may not sink these
      // loads into the dependency chain: shared-memory latency stays off it)
      double zr[RS], f0[RS], f1[RS];
#pragma unroll
      for (int k = 0; k < RS; ++k) {
        zr[k] = zin(st, k);
        f0[k] = fac(st, 0, k);
        f1[k] = fac(st, 1, k);
      }
      asm volatile("" ::: "memory");
#pragma unroll
      for (int k = 0; k < RS; ++k) {
        const double yr = zr[k] - (f0[k] * y2 + f1[k] * y1);  // penta.cpp:180
        if (active) *zp = yr;
        zp += step;
        y2 = y1;
        y1 = yr;
      }
    } else {
#pragma unroll
      for (int k = 0; k < RS; ++k) {
        const double yr = zin(st, k) - (fac(st, 0, k) * y2 + fac(st, 1, k) * y1);
        if (active && r0 + k < n) *zp = yr;
        zp += step;
        y2 = y1;
        y1 = yr;
      }
    }
    __syncwarp();
    if (lane == 0) s_mbar_arrive(&empty[slot]);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("barrier.sync 1, 64;" ::: "memory");  // non-.aligned: see the producer side
  // ---- backward (penta.cpp:183-196): stage 0 (rows n-RS..n-1) peeled
  double s1 = 0.0, s2 = 0.0, zn1 = 0.0, zn2 = 0.0, zz0 = 0.0, zz1 = 0.0;
  auto put = [&](int, int r, double yr, double* zq) {
    if (active && r >= 0) *zq = yr;
  };
  ready = false;
  for (int g = nS; g < total; ++g) {
    const int slot = g % SW_NSTG;
    if (!ready) s_mbar_wait(&full[slot], (g / SW_NSTG) & 1);
    ready = g + 1 < total && s_mbar_test(&full[(g + 1) % SW_NSTG], ((g + 1) / SW_NSTG) & 1);
    const double* st = sw_smem + slot * SM::STAGE_PAD;
    const int r0 = n - (g - nS + 1) * RS;
    double* zq = zc + static_cast<long long>(r0 + RS - 1) * sB;
    if (g == nS) {
#pragma unroll
      for (int k = RS - 1; k >= 0; --k) {
        const int r = r0 + k;
        const double yv = st[k * 32 + lane];
        double yr;
        if (k == RS - 1) {
          yr = yv * fac(st, 0, k);
          zn1 = yr;
        } else if (k == RS - 2) {
          yr = (yv - fac(st, 1, k) * s1) * fac(st, 0, k);
          zn2 = yr;
        } else {
          yr = (yv - fac(st, 1, k) * s1 - fac(st, 2, k) * s2) * fac(st, 0, k);
        }
        put(k, r, yr, zq);
        zq -= sB;
        if (r == 1) zz1 = yr;
        if (r == 0) zz0 = yr;
        s2 = s1;
        s1 = yr;
      }
    } else if (r0 >= 2) {
      // full stage above row 1: operands first, then the branch-free chain
      double yv[RS], di[RS], ap[RS], bp[RS];
#pragma unroll
      for (int k = 0; k < RS; ++k) {
        yv[k] = st[k * 32 + lane];
        di[k] = fac(st, 0, k);
        ap[k] = fac(st, 1, k);
        bp[k] = fac(st, 2, k);
      }
      asm volatile("" ::: "memory");
#pragma unroll
      for (int k = RS - 1; k >= 0; --k) {
        const double yr = (yv[k] - ap[k] * s1 - bp[k] * s2) * di[k];
        put(k, r0 + k, yr, zq);
        zq -= sB;
        s2 = s1;
        s1 = yr;
      }
    } else {
#pragma unroll
      for (int k = RS - 1; k >= 0; --k) {
        const int r = r0 + k;
        const double yr = (st[k * 32 + lane] - fac(st, 1, k) * s1 - fac(st, 2, k) * s2) * fac(st, 0, k);
        put(k, r, yr, zq);
        zq -= sB;
        zz1 = r == 1 ? yr : zz1;
        zz0 = r == 0 ? yr : zz0;
        s2 = s1;
        s1 = yr;
      }
    }
    __syncwarp();
    if (lane == 0) s_mbar_arrive(&empty[slot]);
  }
  if constexpr (PERIODIC) {
    const int sys = b;
    if (!active) return;
    const double* cw = f.cw + sys * 6;
    double y[4];
    y[0] = cw[0] * zn2 + cw[1] * zn1;
    y[1] = cw[2] * zn1;
    y[2] = cw[3] * zz0;
    y[3] = cw[4] * zz0 + cw[5] * zz1;
    lu4_solve_dev(f.K + sys * 16, f.piv + sys * 4, y);
    if constexpr (MODE == 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) y4[k * sB + b] = y[k];
    } else {
#pragma unroll 4
      for (int r = 0; r < n; ++r) {
        const long long idx = r * sB;
        const double w0 = tab(f.W[0], r, b, B, false), w1 = tab(f.W[1], r, b, B, false),
                     w2 = tab(f.W[2], r, b, B, false), w3 = tab(f.W[3], r, b, B, false);
        zc[idx] -= w0 * y[0] + w1 * y[1] + w2 * y[2] + w3 * y[3];
      }
    }
  }
}

template <bool P, int M>
void launch_sweep_tma(const PentaTables& f, const SweepMaps& maps, int B, int n, double* z, double* y4,
                      cudaStream_t s) {
  auto kern = k_sweep_tma<P, M>;
  using SM = SweepSmem;
  static bool configured = false;
  if (!configured) {
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SM::bytes)));
    configured = true;
  }
  const int blocks = (B + 31) / 32;
  kern<<<blocks, 64, SM::bytes, s>>>(f, maps, B, n, z, y4);
}

template <int RS, int XIN>
void launch_sweep_res_t(bool periodic, const PentaTables& f, const SweepMaps& maps, int B, int n, double* y4,
                        cudaStream_t s, bool pdl, const SweepFuse& fuse, int segs = 1) {
  constexpr size_t smem = RRGeom<RS, XIN>::SMEM;
  static bool configured = false;
  if (!configured) {
    SG_CUDA(cudaFuncSetAttribute(k_sweep_res<true, RS, XIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    SG_CUDA(cudaFuncSetAttribute(k_sweep_res<false, RS, XIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    configured = true;
  }
  const int blocks = (B + 31) / 32;
  launch_ex(periodic ? k_sweep_res<true, RS, XIN> : k_sweep_res<false, RS, XIN>, dim3(blocks, segs),
            dim3(XIN ? 32 * (2 + XIN_TW) : 64), smem, s, pdl, f, maps, B, n, y4, fuse);
}

void launch_sweep_res(bool periodic, const PentaTables& f, const SweepMaps& maps, int B, int n, double* y4,
                      cudaStream_t s, bool pdl, int rs, int xin = 0, const SweepFuse& fuse = SweepFuse{},
                      int segs = 1) {
  const bool wide = rs == RR_RS_WIDE;
  if (xin == 1) {
    if (wide) launch_sweep_res_t<RR_RS_WIDE, 1>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
    else launch_sweep_res_t<RR_RS, 1>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
  } else if (xin == 2) {
    if (wide) launch_sweep_res_t<RR_RS_WIDE, 2>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
    else launch_sweep_res_t<RR_RS, 2>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
  } else {
    if (wide) launch_sweep_res_t<RR_RS_WIDE, 0>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
    else launch_sweep_res_t<RR_RS, 0>(periodic, f, maps, B, n, y4, s, pdl, fuse, segs);
  }
}

template <bool U, bool P, int M>
void launch_sweep_t(const PentaTables& f, int B, int n, double* z, double* y4, cudaStream_t s) {
  const int blocks = (B + SWEEP_THREADS - 1) / SWEEP_THREADS;
  k_sweep<U, P, M><<<blocks, SWEEP_THREADS, 0, s>>>(f, B, n, z, y4);
}

}  // namespace

// 2D FP64 tile map (no swizzle, zero OOB fill) for other kernels (ch.cu).
bool encode_tile_map(void* m, const double* p, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1) {
  return encode_map(static_cast<CUtensorMap*>(m), p, 2, d0, d1, b0, b1);
}

namespace {
// z[r*B + b] -= W0[r] y0[b] + W1[r] y1[b] + W2[r] y2[b] + W3[r] y3[b]
// (penta.cpp:279-286) as one fully parallel pass: the recurrence kernels
// hand y = K^{-1} V^T z over in y4[k*B + b].
__global__ void __launch_bounds__(256) k_penta_correct(const PentaTables f, int B, int n, double* __restrict__ z,
                                                       const double* __restrict__ y4) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (b >= B) return;
  const bool u = f.uniform;
  const long long idx = static_cast<long long>(r) * B + b;
  const double w0 = tab(f.W[0], r, b, B, u), w1 = tab(f.W[1], r, b, B, u), w2 = tab(f.W[2], r, b, B, u),
               w3 = tab(f.W[3], r, b, B, u);
  z[idx] -= w0 * __ldg(y4 + b) + w1 * __ldg(y4 + B + b) + w2 * __ldg(y4 + 2LL * B + b) + w3 * __ldg(y4 + 3LL * B + b);
}
}  // namespace

void penta_sweep(const PentaTables& f, int B, int n, double* z, double* y4, bool periodic,
                 bool fusedCorrection, cudaStream_t s, bool pdl) {
  if (periodic && !fusedCorrection && y4 != nullptr) {
    // recurrence with y handed over, then the correction as a parallel pass
    penta_sweep(f, B, n, z, y4, true, true, s);
    k_penta_correct<<<dim3((B + 255) / 256, n), 256, 0, s>>>(f, B, n, z, y4);
    check_launch("penta correction kernel");
    return;
  }
  SweepMaps maps;
  const int rs = sweep_res_rows(B);
  if (f.uniform && (!periodic || fusedCorrection) && sweep_maps(f, B, n, z, &maps, rs)) {
    launch_sweep_res(periodic, f, maps, B, n, y4, s, pdl, rs);
    check_launch("penta sweep (TMA, resident turn) kernel");
    return;
  }
  // general per-system tables: the streaming TMA sweep (uniform operators
  // that reach here — odd batches, unaligned rhs, SG_SWEEP_KERNEL=reg — take
  // the register-prefetch sweep below)
  if (!f.uniform && sweep_maps(f, B, n, z, &maps)) {
    if (!periodic) launch_sweep_tma<false, 0>(f, maps, B, n, z, y4, s);
    else if (fusedCorrection) launch_sweep_tma<true, 1>(f, maps, B, n, z, y4, s);
    else launch_sweep_tma<true, 0>(f, maps, B, n, z, y4, s);
    check_launch("penta sweep (TMA) kernel");
    return;
  }
  if (f.uniform) {
    if (!periodic) launch_sweep_t<true, false, 0>(f, B, n, z, y4, s);
    else if (fusedCorrection) launch_sweep_t<true, true, 1>(f, B, n, z, y4, s);
    else launch_sweep_t<true, true, 0>(f, B, n, z, y4, s);
  } else {
    if (!periodic) launch_sweep_t<false, false, 0>(f, B, n, z, y4, s);
    else if (fusedCorrection) launch_sweep_t<false, true, 1>(f, B, n, z, y4, s);
    else launch_sweep_t<false, true, 0>(f, B, n, z, y4, s);
  }
  check_launch("penta sweep kernel");
}

bool penta_sweep_xin(const PentaTables& f, int B, int n, double* z, const double* zT, const double* const* Wc,
                     const double* yc, double* y4, cudaStream_t s, bool pdl, bool launch, int ztInner,
                     const SweepPeers* peers) {
  SweepMaps maps;
  SweepFuse fuse;
  int rs = 0;
  if (!xin_prepare(f, B, n, z, zT, Wc, yc, ztInner, peers, &maps, &fuse, &rs)) return false;
  if (!launch) return true;
  launch_sweep_res(true, f, maps, B, n, y4, s, pdl, rs, Wc ? 1 : 2, fuse);
  check_launch("penta sweep (TMA, resident turn, transposed input) kernel");
  return true;
}


// ------------------------------------------------ partitioned sweep (SegPenta)

bool penta_sweep_seg(const SegPenta& sp, int B, double* z, const double* zT, const double* const* Wc,
                     const double* yc, int ycSeg, double* gIf, cudaStream_t s, bool pdl, bool launch) {
  const int n = sp.n, m = sp.m, P = sp.P;
  if (P < 1 || !sp.local.t.uniform) return false;
  if ((reinterpret_cast<uintptr_t>(zT) & 15) || (reinterpret_cast<uintptr_t>(z) & 15) || (B & 1) || n % 16) return false;
  int rs = sweep_res_rows(B * P);
  if (m % rs) rs = RR_RS;
  if (m % rs || m < rs) return false;
  SweepMaps maps = SweepMaps{};
  if (!encode_map(&maps.z, z, 2, B, n, 32, rs)) return false;
  const double* t[5] = {sp.local.t.m1, sp.local.t.m2, sp.local.t.dInv, sp.local.t.ap, sp.local.t.bp};
  for (int k = 0; k < 5; ++k)
    if ((reinterpret_cast<uintptr_t>(t[k]) & 15) || !encode_map(&maps.t[k], t[k], 1, m, 1, rs, 1)) return false;
  maps.ztBox = n % rs == 0 && encode_map4_zt(&maps.zt, zT, n, B, n, rs) ? 1 : 0;
  if (!maps.ztBox && !encode_map3(&maps.zt, zT, n, B, 1, 16, 32, 1, true)) return false;
  maps.ztInner = n;
  maps.segRows = m;
  SweepFuse fuse;
  if (Wc) {
    if (reinterpret_cast<uintptr_t>(yc) & 15) return false;
    if (ycSeg) {
      if (ycSeg % 32 || B % ycSeg) return false;
      if (!encode_map3(&maps.yc[0], yc, n, 4, B / ycSeg, rs, 4, 1, false)) return false;
      maps.ycSeg = ycSeg;
    } else if (!encode_map(&maps.yc[0], yc, 2, n, 4, rs, 4)) {
      return false;
    }
    for (int k = 0; k < 4; ++k) fuse.Wc[k] = Wc[k];
    fuse.yc = yc;
  }
  if (!launch) return true;
  launch_sweep_res(false, sp.local.t, maps, B, m, gIf, s, pdl, rs, Wc ? 1 : 2, fuse, P);
  check_launch("penta partitioned sweep kernel");
  return true;
}

namespace {
// z = Rinv * G for every system (G: the 4P interface values of system b,
// segment-major as gIf), one thread per (system b, interface unknown i =
// 4j + q): a dot product of length 4P (Rinv row i is warp-uniform: a
// broadcast). z_i is the t_{j,q} (q < 2) or b_{j,q-2} (q >= 2) of segment
// j: coefficient slot q of segment j - 1 (as its t_{k+1}) or j + 1 (as its
// b_{k-1}).
template <int P>
__global__ void __launch_bounds__(128) k_seg_reduce(const double* __restrict__ gIf, const double* __restrict__ Rinv,
                                                    int B, double* __restrict__ coef) {
  constexpr int N = 4 * P;
  const int b = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  pdl_wait();
  if (b >= B) return;
  // all N loads in flight before the dot product (N is compile-time)
  double g[N];
#pragma unroll
  for (int jj = 0; jj < N; ++jj) g[jj] = __ldg(gIf + static_cast<long long>(jj) * B + b);
  const double* row = Rinv + static_cast<long long>(i) * N;
  double acc = 0.0;
#pragma unroll
  for (int jj = 0; jj < N; ++jj) acc += __ldg(row + jj) * g[jj];
  const int j = i / 4, q = i % 4;
  const int k = q < 2 ? (j + P - 1) % P : (j + 1) % P;
  coef[static_cast<long long>(k * 4 + q) * B + b] = acc;
}

// The interface solve fused with the correction of a ROW-MAJOR result
// (w[j*B + i]: row j = unknown, column i = system; the CH y-sweep's output):
// a CTA takes 128 systems and `rows` rows of one segment, computes the 4
// coefficients of its (segment, system) once — the dot products of
// k_seg_reduce, same order — and applies them to its rows:
// w -= V0 c0 + V1 c1 + W0 c2 + W1 c3 (penta.cpp:283-284's expression).
template <int P>
__global__ void __launch_bounds__(128) k_seg_finish_rows(double* __restrict__ w, int B, const double* __restrict__ vec,
                                                         int n, const double* __restrict__ gIf,
                                                         const double* __restrict__ Rinv, int m, int rows) {
  constexpr int N = 4 * P;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j0 = blockIdx.y * rows;
  pdl_wait();
  if (i >= B) return;
  const int seg = j0 / m, kp = (seg + 1) % P, km = (seg + P - 1) % P;
  const int zi[4] = {4 * kp, 4 * kp + 1, 4 * km + 2, 4 * km + 3};
  double g[N];
#pragma unroll
  for (int jj = 0; jj < N; ++jj) g[jj] = __ldg(gIf + static_cast<long long>(jj) * B + i);
  double c[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double* row = Rinv + static_cast<long long>(zi[q]) * N;
    double acc = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) acc += __ldg(row + jj) * g[jj];
    c[q] = acc;
  }
#pragma unroll 4
  for (int r = 0; r < rows; ++r) {
    const int j = j0 + r;
    double* p = w + static_cast<long long>(j) * B + i;
    *p -= __ldg(vec + j) * c[0] + __ldg(vec + n + j) * c[1] + __ldg(vec + 2LL * n + j) * c[2] +
          __ldg(vec + 3LL * n + j) * c[3];
  }
}

template <typename F>
void with_segs(int P, F&& f) {
  switch (P) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 16: return f(std::integral_constant<int, 16>{});
    default: invalid("partitioned sweep: segments must be 1, 2, 4, 8 or 16");
  }
}
}  // namespace

void penta_seg_finish_rows(const SegPenta& sp, int B, double* w, const double* gIf, cudaStream_t s, bool pdl) {
  static const int rowsPer = [] {
    const char* e = std::getenv("SG_SEG_ROWS");
    return e ? std::atoi(e) : 8;
  }();
  const int rows = sp.m % rowsPer == 0 ? rowsPer : sp.m;
  with_segs(sp.P, [&](auto pc) {
    launch_ex(k_seg_finish_rows<decltype(pc)::value>, dim3((B + 127) / 128, sp.n / rows), dim3(128), 0, s, pdl, w,
              B, static_cast<const double*>(sp.vec), sp.n, gIf, static_cast<const double*>(sp.Rinv), sp.m, rows);
  });
  check_launch("penta partitioned interface solve + row correction kernel");
}

void penta_seg_reduce(const SegPenta& sp, int B, const double* gIf, double* coef, cudaStream_t s, bool pdl) {
  with_segs(sp.P, [&](auto pc) {
    launch_ex(k_seg_reduce<decltype(pc)::value>, dim3((B + 127) / 128, 4 * sp.P), dim3(128), 0, s, pdl, gIf,
              static_cast<const double*>(sp.Rinv), B, coef);
  });
  check_launch("penta partitioned interface solve kernel");
}

SegPenta::~SegPenta() {
  for (void* q : allocs) cudaFree(q);
}

void SegPenta::build(double e, double c, double d, double a, double b, int n_, int P_, cudaStream_t s) {
  if ((P_ & (P_ - 1)) || P_ < 1 || P_ > 16 || n_ % P_ || n_ / P_ < 8)
    invalid("partitioned sweep: need P in {1, 2, 4, 8, 16}, P | n, n / P >= 8");
  n = n_;
  P = P_;
  m = n / P;
  auto dalloc = [&](size_t cnt) {
    void* q = nullptr;
    SG_CUDA(cudaMalloc(&q, cnt * sizeof(double)));
    allocs.push_back(q);
    return static_cast<double*>(q);
  };
  // local factor: the m x m leading block (no corners)
  std::vector<double> hb(5 * static_cast<size_t>(m));
  const double bv[5] = {e, c, d, a, b};
  for (int k = 0; k < 5; ++k)
    for (int r = 0; r < m; ++r) hb[static_cast<size_t>(k) * m + r] = bv[k];
  double* bands = dalloc(5 * static_cast<size_t>(m));
  SG_CUDA(cudaMemcpyAsync(bands, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  local.build(1, m, false, true, bands, bands + m, bands + 2 * m, bands + 3 * m, bands + 4 * m, s);
  // spikes: A_loc [V0 V1 W0 W1] = [B0 B1 C0 C1], four systems interleaved (r*4 + col)
  std::vector<double> hz(4 * static_cast<size_t>(m), 0.0);
  hz[(m - 2) * 4 + 0] = b;  // row m-2 couples to the next segment's row 0 (coefficient b)
  hz[(m - 1) * 4 + 0] = a;  // row m-1: a * next row 0 + b * next row 1
  hz[(m - 1) * 4 + 1] = b;
  hz[0 * 4 + 2] = e;        // row 0: e * prev row m-2 + c * prev row m-1
  hz[0 * 4 + 3] = c;
  hz[1 * 4 + 3] = e;        // row 1: e * prev row m-1
  double* zs = dalloc(hz.size());
  SG_CUDA(cudaMemcpyAsync(zs, hz.data(), hz.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  penta_sweep(local.t, 4, m, zs, nullptr, false, true, s);
  SG_CUDA(cudaMemcpyAsync(hz.data(), zs, hz.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  std::vector<double> hv(4 * static_cast<size_t>(n));
  for (int q = 0; q < 4; ++q)
    for (int r = 0; r < n; ++r) hv[static_cast<size_t>(q) * n + r] = hz[static_cast<size_t>(r % m) * 4 + q];
  vec = dalloc(hv.size());
  SG_CUDA(cudaMemcpyAsync(vec, hv.data(), hv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  // reduced system R z = G over z = (t_k0, t_k1, b_k0, b_k1)_k:
  //   rows {0, 1, m-2, m-1} of  x_k + V t_{k+1} + W b_{k-1} = g_k
  const int N = 4 * P;
  std::vector<double> R(static_cast<size_t>(N) * N, 0.0), I(static_cast<size_t>(N) * N, 0.0);
  const int rowsOf[4] = {0, 1, m - 2, m - 1};
  for (int k = 0; k < P; ++k) {
    const int kp = (k + 1) % P, km = (k + P - 1) % P;
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * k + q, r = rowsOf[q];
      R[static_cast<size_t>(i) * N + i] += 1.0;
      R[static_cast<size_t>(i) * N + 4 * kp + 0] += hz[static_cast<size_t>(r) * 4 + 0];
      R[static_cast<size_t>(i) * N + 4 * kp + 1] += hz[static_cast<size_t>(r) * 4 + 1];
      R[static_cast<size_t>(i) * N + 4 * km + 2] += hz[static_cast<size_t>(r) * 4 + 2];
      R[static_cast<size_t>(i) * N + 4 * km + 3] += hz[static_cast<size_t>(r) * 4 + 3];
    }
    (void)km;
  }
  for (int i = 0; i < N; ++i) I[static_cast<size_t>(i) * N + i] = 1.0;
  // Gauss-Jordan with partial pivoting
  for (int col = 0; col < N; ++col) {
    int piv = col;
    for (int r = col + 1; r < N; ++r)
      if (std::fabs(R[static_cast<size_t>(r) * N + col]) > std::fabs(R[static_cast<size_t>(piv) * N + col])) piv = r;
    if (R[static_cast<size_t>(piv) * N + col] == 0.0) throw Error(SG_ERR_PENTA_SOLVE, "partitioned sweep: singular interface system", 0);
    if (piv != col)
      for (int j = 0; j < N; ++j) {
        std::swap(R[static_cast<size_t>(piv) * N + j], R[static_cast<size_t>(col) * N + j]);
        std::swap(I[static_cast<size_t>(piv) * N + j], I[static_cast<size_t>(col) * N + j]);
      }
    const double inv = 1.0 / R[static_cast<size_t>(col) * N + col];
    for (int j = 0; j < N; ++j) {
      R[static_cast<size_t>(col) * N + j] *= inv;
      I[static_cast<size_t>(col) * N + j] *= inv;
    }
    for (int r = 0; r < N; ++r) {
      if (r == col) continue;
      const double f = R[static_cast<size_t>(r) * N + col];
      if (f == 0.0) continue;
      for (int j = 0; j < N; ++j) {
        R[static_cast<size_t>(r) * N + j] -= f * R[static_cast<size_t>(col) * N + j];
        I[static_cast<size_t>(r) * N + j] -= f * I[static_cast<size_t>(col) * N + j];
      }
    }
  }
  Rinv = dalloc(I.size());
  SG_CUDA(cudaMemcpyAsync(Rinv, I.data(), I.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------ peer TMA store self-check

// One 32 x 2 box written by a TMA tensor store from shared memory into
// `dst` (another device's buffer over NVLink, or IPC-mapped memory), then
// read back through generic loads. *ok = 1 iff every value arrived. The
// pattern depends on `salt`, so a stale earlier probe cannot pass.
__global__ void k_peer_tma_probe(const __grid_constant__ CUtensorMap map, const double* dst, unsigned salt,
                                 int* ok) {
  __shared__ alignas(128) double box[64];
  const int t = threadIdx.x;
  box[t] = static_cast<double>(salt) * 64.0 + t;
  box[t + 32] = -(static_cast<double>(salt) * 64.0 + t + 32);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    s_tma_store_2d(&map, 0, 0, box);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
  }
  __syncthreads();
  const volatile double* v = dst;
  const bool good = v[t] == box[t] && v[t + 32] == box[t + 32];
  const int all = __syncthreads_and(good ? 1 : 0);
  if (t == 0) *ok = all;
}

bool peer_tma_probe(double* dst, unsigned salt, cudaStream_t s) {
  if (reinterpret_cast<uintptr_t>(dst) & 15) return false;
  CUtensorMap m;
  if (!encode_map(&m, dst, 2, 32, 2, 32, 2)) return false;
  int* d_ok = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&d_ok), sizeof(int), s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int ok = 0;
  k_peer_tma_probe<<<1, 32, 0, s>>>(m, dst, salt, d_ok);
  bool good = cudaGetLastError() == cudaSuccess &&
              cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
              cudaStreamSynchronize(s) == cudaSuccess;
  cudaFreeAsync(d_ok, s);
  cudaStreamSynchronize(s);
  cudaGetLastError();
  return good && ok == 1;
}


// ------------------------------------------------------------ PentaFactor

DevicePenta::~DevicePenta() {
  for (void* p : allocs) cudaFree(p);
}

double* DevicePenta::alloc(size_t count) {
  void* p = nullptr;
  SG_CUDA(cudaMalloc(&p, count * sizeof(double)));
  allocs.push_back(p);
  return static_cast<double*>(p);
}

void DevicePenta::build(int B_, int n_, bool periodic_, bool uniform, const double* e,
                        const double* c, const double* d, const double* a, const double* b,
                        cudaStream_t s) {
  B = B_;
  n = n_;
  periodic = periodic_;
  const int nsys = uniform ? 1 : B;
  const size_t len = static_cast<size_t>(nsys) * n;
  t.uniform = uniform ? 1 : 0;
  double* m1 = alloc(len);
  double* m2 = alloc(len);
  double* dInv = alloc(len);
  double* ap = alloc(len);
  double* bp = alloc(len);
  t.m1 = m1;
  t.m2 = m2;
  t.dInv = dInv;
  t.ap = ap;
  t.bp = bp;
  int* dBad = nullptr;
  SG_CUDA(cudaMalloc(&dBad, sizeof(int) * nsys));
  allocs.push_back(dBad);
  k_factor<<<(nsys + 127) / 128, 128, 0, s>>>(nsys, n, e, c, d, a, b, m1, m2, dInv, ap, bp, dBad);
  check_launch("penta factor kernel");
  std::vector<int> bad(nsys);
  SG_CUDA(cudaMemcpyAsync(bad.data(), dBad, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  // PentaSolveError for the first zero pivot in the reference's row-major
  // scan order (penta.cpp:119-123): smallest row, then smallest system.
  int bestRow = n, bestSys = -1;
  for (int k = 0; k < nsys; ++k)
    if (bad[k] < bestRow) {
      bestRow = bad[k];
      bestSys = k;
    }
  if (bestSys >= 0) throw Error(SG_ERR_PENTA_SOLVE, "penta: zero pivot during elimination", bestSys);
  if (!periodic) return;
  double* W[4];
  for (int k = 0; k < 4; ++k) W[k] = alloc(len);
  double* cw = alloc(static_cast<size_t>(nsys) * 6);
  double* K = alloc(static_cast<size_t>(nsys) * 16);
  int* piv = nullptr;
  SG_CUDA(cudaMalloc(&piv, sizeof(int) * 4 * nsys));
  allocs.push_back(piv);
  for (int k = 0; k < 4; ++k) t.W[k] = W[k];
  t.cw = cw;
  t.K = K;
  t.piv = piv;
  // For the uniform case the setup thread reads the bands of system 0 with
  // stride 1: pass the single-system bands.
  if (uniform)
    k_periodic_setup_uniform<<<1, 4, 0, s>>>(t, n, e, c, a, b, W[0], W[1], W[2], W[3], cw, K, piv, dBad);
  else {
    k_periodic_core<<<dim3((nsys + 127) / 128, 4), 128, 0, s>>>(t, B, n, W[0], W[1], W[2], W[3]);
    check_launch("penta periodic core-solve kernel");
    k_periodic_setup<<<(nsys + 127) / 128, 128, 0, s>>>(t, B, n, e, c, a, b, W[0], W[1], W[2], W[3], cw, K,
                                                      piv, dBad);
  }
  check_launch("penta periodic setup kernel");
  SG_CUDA(cudaMemcpyAsync(bad.data(), dBad, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < nsys; ++k)
    if (bad[k]) throw Error(SG_ERR_PENTA_SOLVE, "penta: singular capacitance matrix", k);
}

}  // namespace sg
