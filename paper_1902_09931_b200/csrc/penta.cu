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
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "penta.cuh"
#include "sg_internal.hpp"

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
  for (int r = 2; r < n; ++r) {
    const long long cur = static_cast<long long>(r) * B + b;
    const double mm1 = e[cur] / dp2;
    const double cbar = c[cur] - mm1 * ap2;
    const double mm2 = cbar / dp1;
    const double dpc = d[cur] - mm1 * bp2 - mm2 * ap1;
    const double apc = a[cur] - mm2 * bp1;
    const double bpc = bb[cur];
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

// One substitution pass pair on a strided vector (used for setup only).
__device__ void substitute(const PentaTables& f, int B, int b, double* y, long long s, int n) {
  const bool u = f.uniform;
  y[s] -= tab(f.m2, 1, b, B, u) * y[0];
  for (int r = 2; r < n; ++r)
    y[r * s] -= tab(f.m1, r, b, B, u) * y[(r - 2) * s] + tab(f.m2, r, b, B, u) * y[(r - 1) * s];
  y[(n - 1) * s] *= tab(f.dInv, n - 1, b, B, u);
  y[(n - 2) * s] = (y[(n - 2) * s] - tab(f.ap, n - 2, b, B, u) * y[(n - 1) * s]) * tab(f.dInv, n - 2, b, B, u);
  for (int r = n - 3; r >= 0; --r)
    y[r * s] = (y[r * s] - tab(f.ap, r, b, B, u) * y[(r + 1) * s] - tab(f.bp, r, b, B, u) * y[(r + 2) * s]) *
               tab(f.dInv, r, b, B, u);
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
__global__ void k_periodic_setup(PentaTables f, int B, int n, const double* __restrict__ e,
                                 const double* __restrict__ c, const double* __restrict__ a,
                                 const double* __restrict__ bb, double* W0, double* W1, double* W2,
                                 double* W3, double* cw, double* K, int* piv, int* singular) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int nsys = f.uniform ? 1 : B;
  if (b >= nsys) return;
  const long long s = f.uniform ? 1 : B;
  double* Wk[4] = {W0 + b, W1 + b, W2 + b, W3 + b};
  const int rowOf[4] = {0, 1, n - 2, n - 1};
  for (int k = 0; k < 4; ++k) {
    for (int r = 0; r < n; ++r) Wk[k][r * s] = 0.0;
    Wk[k][rowOf[k] * s] = 1.0;
    substitute(f, B, b, Wk[k], s, n);
  }
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

template <bool U, bool P, int M>
void launch_sweep_t(const PentaTables& f, int B, int n, double* z, double* y4, cudaStream_t s) {
  const int blocks = (B + SWEEP_THREADS - 1) / SWEEP_THREADS;
  k_sweep<U, P, M><<<blocks, SWEEP_THREADS, 0, s>>>(f, B, n, z, y4);
}

}  // namespace

void penta_sweep(const PentaTables& f, int B, int n, double* z, double* y4, bool periodic,
                 bool fusedCorrection, cudaStream_t s) {
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
  k_periodic_setup<<<(nsys + 127) / 128, 128, 0, s>>>(t, B, n, e, c, a, b, W[0], W[1], W[2], W[3], cw, K,
                                                    piv, dBad);
  check_launch("penta periodic setup kernel");
  SG_CUDA(cudaMemcpyAsync(bad.data(), dBad, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < nsys; ++k)
    if (bad[k]) throw Error(SG_ERR_PENTA_SOLVE, "penta: singular capacitance matrix", k);
}

}  // namespace sg
