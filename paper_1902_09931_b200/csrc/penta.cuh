// penta.cuh — device pentadiagonal factor tables and sweeps (see penta.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include <vector>

namespace sg {

// Factor tables. uniform: every array holds one system (n entries, W_k n
// entries, cw 6, K 16, piv 4); otherwise interleaved per system (r*B + b;
// cw/K/piv system-major).
struct PentaTables {
  const double* m1 = nullptr;
  const double* m2 = nullptr;
  const double* dInv = nullptr;
  const double* ap = nullptr;
  const double* bp = nullptr;
  const double* W[4] = {nullptr, nullptr, nullptr, nullptr};
  const double* cw = nullptr;
  const double* K = nullptr;
  const int* piv = nullptr;
  int uniform = 0;
};

// Encodes a 2D FP64 tensor map (CUtensorMap*, dims d0 x d1, box b0 x b1,
// no swizzle, OOB elements read as zero); false without a driver encoder.
bool encode_tile_map(void* m, const double* p, uint64_t d0, uint64_t d1, uint32_t b0, uint32_t b1);

// Owns the device factor of one (periodic or not) batch.
struct DevicePenta {
  int B = 0, n = 0;
  bool periodic = false;
  PentaTables t;
  std::vector<void*> allocs;

  DevicePenta() = default;
  DevicePenta(const DevicePenta&) = delete;
  DevicePenta& operator=(const DevicePenta&) = delete;
  ~DevicePenta();

  // Bands are DEVICE pointers; uniform => single-system bands of length n,
  // else interleaved B*n. Throws Error(SG_ERR_PENTA_SOLVE, system) exactly
  // where the reference throws PentaSolveError.
  void build(int B, int n, bool periodic, bool uniform, const double* e, const double* c,
             const double* d, const double* a, const double* b, cudaStream_t s);
  double* alloc(size_t count);
};

// Forward/back substitution (+ periodic correction) of B interleaved systems
// in z. fusedCorrection: skip z -= W y and write y (y4[k*B + b]) instead.
// pdl: launch the resident-turn sweep as a programmatic dependent of the
// previous kernel on `s` (the kernel waits before touching global memory).
void penta_sweep(const PentaTables& f, int B, int n, double* z, double* y4, bool periodic,
                 bool fusedCorrection, cudaStream_t s, bool pdl = false);

// Uniform periodic sweep reading its input TRANSPOSED: zT[b*n + r] (system-
// major for this batch), e.g. the other sweep's output or a row-major RHS.
// With Wc (the CH y-sweep) the previous sweep's Woodbury correction is
// applied on load: zT - (Wc0[b] yc0[r] + ... + Wc3[b] yc3[r]) (yc[k*n + r]);
// Wc = nullptr reads zT as is (the CH x-sweep). Results (uncorrected,
// y -> y4) go to the interleaved z. launch = false only checks
// availability. Returns false if the path is unavailable.
// P2P destinations of the final results (the distributed CH sweeps): the
// unknowns [d*prow, (d+1)*prow) of all B systems go to dst[d] laid out
// [unknown - d*prow][system] (row length B) — peer memory over NVLink in
// production; y (the Woodbury coefficients) also goes to
// y4[d][k*y4Stride + y4Off + b].
struct SweepPeers {
  int npeer = 0;
  int prow = 0;
  double* dst[8] = {};
  double* y4[8] = {};
  int y4Stride = 0, y4Off = 0;
};

// Runtime self-check of the P2P path: one TMA tensor store into `dst`
// (peer / IPC-mapped memory) plus a read-back; false if either fails.
bool peer_tma_probe(double* dst, unsigned salt, cudaStream_t s);

// ztInner: the input's unknowns are stored in blocks of ztInner per system
// (zT[(r / ztInner)*(B*ztInner) + b*ztInner + r % ztInner]; 0 = n: plain
// system-major) — the distributed y-sweep reads one block per source rank.
bool penta_sweep_xin(const PentaTables& f, int B, int n, double* z, const double* zT, const double* const* Wc,
                     const double* yc, double* y4, cudaStream_t s, bool pdl, bool launch = true, int ztInner = 0,
                     const SweepPeers* peers = nullptr);

// Partitioned (SPIKE-type) solve of a uniform CYCLIC pentadiagonal operator
// — an opt-in alternative to the bitwise sweep for latency-bound batches
// (few systems, long chains: CH 1024^2 on one GPU, config 5's 1024 systems
// of 8192 per GPU): every system's n unknowns form P segments of m = n / P
// rows, solved independently (B * P chains of m rows instead of B of n) with
// the factor of the segment-local operator A_loc (non-periodic, m x m); the
// segments couple through the operator's 2 x 2 corner blocks, so
//   x_k = g_k - (V0 t_{k+1,0} + V1 t_{k+1,1} + W0 b_{k-1,0} + W1 b_{k-1,1})
// with g_k = A_loc^{-1} f_k, the spikes [V0 V1] = A_loc^{-1} B and
// [W0 W1] = A_loc^{-1} C (B, C the couplings to the next / previous
// segment), and (t_k, b_k) the first / last two unknowns of segment k: the
// 4P interface unknowns solve a reduced system R z = G (G the interface
// values of the g_k), identical for all systems, inverted once on the host.
// P = 1 is the Woodbury form of the periodic sweep. Not bitwise equal to the
// reference's order of operations (penta.cpp:160-295); see DESIGN.md.
struct SegPenta {
  int n = 0, P = 0, m = 0;
  DevicePenta local;          // factor of A_loc (non-periodic, length m)
  double* vec = nullptr;      // [4][n]: V0, V1, W0, W1, tiled over the n unknowns (row r: local row r % m)
  double* Rinv = nullptr;     // [4P][4P], row-major; interface unknowns per segment: t0, t1, b0, b1
  std::vector<void*> allocs;
  SegPenta() = default;
  SegPenta(const SegPenta&) = delete;
  SegPenta& operator=(const SegPenta&) = delete;
  ~SegPenta();
  // Uniform bands (row r: e x_{r-2} + c x_{r-1} + d x_r + a x_{r+1} + b x_{r+2},
  // cyclic) given on the host; builds the local factor, the spikes and R^{-1}.
  void build(double e, double c, double d, double a, double b, int n, int P, cudaStream_t s);
};
// Sweep of B systems (one CTA per 32 systems and segment) reading its input
// transposed (zT[b*n + r], as penta_sweep_xin; Wc/yc: the previous sweep's
// correction applied on load, yc holding one [4][n] plane per ycSeg systems
// when that sweep was partitioned, ycSeg = 0 otherwise). Writes the local
// solutions g (uncorrected) to z (interleaved) and the interface values to
// gIf[(k*4 + q)*B + b] (q: g[0], g[1], g[m-2], g[m-1]). False if unavailable.
bool penta_sweep_seg(const SegPenta& sp, int B, double* z, const double* zT, const double* const* Wc,
                     const double* yc, int ycSeg, double* gIf, cudaStream_t s, bool pdl, bool launch = true);
// Interface solve: coef[(k*4 + q)*B + b] = (t_{k+1,0}, t_{k+1,1}, b_{k-1,0},
// b_{k-1,1}) of segment k from gIf — the coefficients of the correction.
void penta_seg_reduce(const SegPenta& sp, int B, const double* gIf, double* coef, cudaStream_t s, bool pdl);
// The interface solve fused with the correction of a row-major result
// w[r*B + b] (rows = the unknowns; the CH y-sweep's output) in place.
void penta_seg_finish_rows(const SegPenta& sp, int B, double* w, const double* gIf, cudaStream_t s, bool pdl);

// lu4_solve, penta.cpp:61-70.
__device__ __forceinline__ void lu4_solve_dev(const double* K, const int* piv, double* y) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int p = piv[c];
    if (p != c) {
      double t = y[c];
      // y[c] <-> y[p] with a runtime p: select chain keeps y in registers
      double yp = p == 1 ? y[1] : p == 2 ? y[2] : y[3];
      y[c] = yp;
      if (p == 1) y[1] = t;
      else if (p == 2) y[2] = t;
      else y[3] = t;
    }
  }
#pragma unroll
  for (int r = 1; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < r; ++c) y[r] -= K[r * 4 + c] * y[c];
#pragma unroll
  for (int r = 3; r >= 0; --r) {
#pragma unroll
    for (int c = r + 1; c < 4; ++c) y[r] -= K[r * 4 + c] * y[c];
    y[r] /= K[r * 4 + r];
  }
}


}  // namespace sg
