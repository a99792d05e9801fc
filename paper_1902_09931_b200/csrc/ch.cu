// ch.cu — Cahn-Hilliard BDF2-ADI stepper, end to end on the GPU.
//
// Replaces CHStepper (cahn_hilliard.cpp:213-328). One step is five kernels,
// captured once into a CUDA graph per time-level parity:
//
//   k_rhs        Cbar = 2C^n - C^{n-1} (on the fly), nl = lap(C^3 - C) over
//                3x3 of C^n, bih = 5x5 biharmonic over Cbar, and
//                rhs = kDiff (C^n - C^{n-1}) - kBih bih + kNl nl
//                (cahn_hilliard.cpp:264-297) — one fused pass, written
//                TRANSPOSED (rhsT[i*ny + j]) through a shared-memory tile so
//                the x-sweep sees interleaved systems (the reference's
//                interleave_into(rhs, X), penta.cpp:343-360, for free).
//   x-sweep      ny periodic systems of nx unknowns, one per thread,
//                coalesced (penta.cu k_sweep); the Woodbury correction is
//                NOT applied in place — y = K^{-1} V^T z goes to y4x.
//   k_transpose_correct
//                w(i,j) = zT(i,j) - (W0[i] y0[j] + ... + W3[i] y3[j]) fused
//                with the transpose back to row-major (the reference's
//                correct_range + deinterleave + transpose + interleave,
//                penta.cpp:253-287, 369-384, grid.cpp:55-60).
//   y-sweep      nx periodic systems of ny unknowns on row-major w (already
//                interleaved for Axis::Y, penta.cpp:356-358); y -> y4y.
//   k_combine    C^{n+1} = Cbar + (w - W·y) written over C^{n-1} in place;
//                the time levels then swap roles (cahn_hilliard.cpp:311-324).
//
// Arithmetic is the reference's term for term (no FMA contraction), so the
// fields are bitwise identical to the CPU reference. The only liberty: taps
// whose weight is exactly 0.0 (4 of the 9 nonlinear coefficients, 12 of the
// 25 biharmonic weights — verified at construction) are skipped; for finite
// fields acc + 0*x == acc exactly (acc starts at +0 and is never -0).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "penta.cuh"
#include "sg_internal.hpp"

namespace sg {
namespace {

constexpr double kTwoThirds = 2.0 / 3.0;  // cahn_hilliard.cpp:12

double pow4(double h) {  // cahn_hilliard.cpp:14-17
  const double h2 = h * h;
  return h2 * h2;
}

// biharmonic_weights (cahn_hilliard.cpp:85-114), host setup constant.
void biharmonic_weights(double dx, double dy, double* w) {
  const double ax = 1.0 / pow4(dx);
  const double ay = 1.0 / pow4(dy);
  const double cr = 2.0 / ((dx * dx) * (dy * dy));
  for (int k = 0; k < 25; ++k) w[k] = 0.0;
  auto at = [w](int p, int q) -> double& { return w[q * 5 + p]; };
  at(0, 2) += ax;
  at(1, 2) += -4.0 * ax;
  at(2, 2) += 6.0 * ax;
  at(3, 2) += -4.0 * ax;
  at(4, 2) += ax;
  at(2, 0) += ay;
  at(2, 1) += -4.0 * ay;
  at(2, 2) += 6.0 * ay;
  at(2, 3) += -4.0 * ay;
  at(2, 4) += ay;
  static constexpr double cross[9] = {1.0, -2.0, 1.0, -2.0, 4.0, -2.0, 1.0, -2.0, 1.0};
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) at(p + 1, q + 1) += cross[q * 3 + p] * cr;
  double prefix = 0.0;
  for (int k = 0; k < 22; ++k) prefix += w[k];
  at(2, 4) = -prefix;
}

// Non-zero taps of the two CH windows (row-major positions q*W + p).
#define SG_BIH_TAPS {2, 6, 7, 8, 10, 11, 12, 13, 14, 16, 17, 18, 22}
#define SG_NL_TAPS {1, 3, 4, 5, 7}

struct RhsParams {
  double bw[25];
  double nl[9];
  double kDiff, kBih, kNl;
};

__global__ void k_init(unsigned long long seed, double amp, long long count, double* __restrict__ out) {
  // SplitMix64 (cahn_hilliard.hpp:47-63) in counter form: draw k uses state
  // seed + (k+1)*golden, so every element is independent.
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= count) return;
  unsigned long long z = seed + static_cast<unsigned long long>(k + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z = z ^ (z >> 31);
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  out[k] = amp * (2.0 * u - 1.0);  // initial_condition, cahn_hilliard.cpp:74
}

constexpr int TS = 32;  // output tile edge
constexpr int HALO = 2;

__device__ __forceinline__ int wrapi(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

// Input geometry of the RHS kernel: output row jl (0..outRows) reads input
// rows jl + inShift + dy, dy in [-2, 2], wrapped modulo inRows iff wrapY
// (full periodic grid: inShift 0, wrapY 1; a y-slab with 2 halo rows above
// and below: inShift 2, wrapY 0). Columns always wrap (periodic in x).
struct RhsGeom {
  int nx, outRows, inRows, inShift, wrapY;
  // k_rhs_v only: write the RHS row-major (rhs[j*nx + i]) instead of
  // transposed — the single-GPU step, whose x-sweep reads it transposed
  int rowOut = 0;
};

__device__ __forceinline__ int wrap_once(int i, int n) {  // i in [-n, 2n)
  return i < 0 ? i + n : (i >= n ? i - n : i);
}

// Output tile: RX = 64 columns (i) x RY = 32 rows (j); 256 threads, each
// computes 2 columns x 4 rows. Inputs are staged with a 2-point halo
// (68 x 36: 1.2x redundancy) through a flattened, coalesced load loop.
constexpr int RX = 64, RY = 32;
constexpr int RXE = RX + 2 * HALO, RYE = RY + 2 * HALO;

template <bool NONLINEAR>
__global__ void __launch_bounds__(256) k_rhs(const double* __restrict__ cc, const double* __restrict__ cp,
                                             double* __restrict__ rhsT, const RhsGeom G,
                                             const __grid_constant__ RhsParams P) {
  extern __shared__ __align__(16) double rsm[];
  double (*sc)[RXE + 1] = reinterpret_cast<double (*)[RXE + 1]>(rsm);              // C^n
  double (*sb)[RXE + 1] = reinterpret_cast<double (*)[RXE + 1]>(rsm + RYE * (RXE + 1));  // Cbar
  double (*sp)[RX + 1] = reinterpret_cast<double (*)[RX + 1]>(rsm + 2 * RYE * (RXE + 1));  // C^{n-1}
  const int nx = G.nx;
  const int i0 = blockIdx.x * RX, j0 = blockIdx.y * RY;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  pdl_wait();
  for (int e = tid; e < RYE * RXE; e += 256) {
    const int y = e / RXE, x = e - y * RXE;
    int j = j0 - HALO + y + G.inShift;
    j = G.wrapY ? (G.inRows >= RYE ? wrap_once(j, G.inRows) : wrapi(j, G.inRows)) : min(max(j, 0), G.inRows - 1);
    const int i = nx >= RXE ? wrap_once(i0 - HALO + x, nx) : wrapi(i0 - HALO + x, nx);
    const long long idx = static_cast<long long>(j) * nx + i;
    const double c = __ldg(cc + idx), p = __ldg(cp + idx);
    sc[y][x] = c;
    sb[y][x] = 2.0 * c - p;  // cahn_hilliard.cpp:273
    if (y >= HALO && y < HALO + RY && x >= HALO && x < HALO + RX) sp[y - HALO][x - HALO] = p;
  }
  __syncthreads();
  constexpr int kBihTaps[13] = SG_BIH_TAPS;
  constexpr int kNlTaps[5] = SG_NL_TAPS;
  const int tx = threadIdx.x, ty = threadIdx.y;
  double res[2][4];
#pragma unroll
  for (int cx = 0; cx < 2; ++cx)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int y = ty + 8 * k;   // output row within the tile
      const int x = tx + 32 * cx;  // output column within the tile
      double bh = 0.0;
#pragma unroll
      for (int t = 0; t < 13; ++t) {
        const int q = kBihTaps[t] / 5, p = kBihTaps[t] % 5;
        bh += P.bw[kBihTaps[t]] * sb[y + q][x + p];
      }
      const double c = sc[y + HALO][x + HALO];
      const double pr = sp[y][x];
      double r;
      if constexpr (NONLINEAR) {
        double nl = 0.0;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int q = kNlTaps[t] / 3, p = kNlTaps[t] % 3;
          const double v = sc[y + 1 + q][x + 1 + p];
          nl += P.nl[kNlTaps[t]] * (v * v * v - v);
        }
        r = P.kDiff * (c - pr) - P.kBih * bh + P.kNl * nl;  // cahn_hilliard.cpp:292
      } else {
        r = P.kDiff * (c - pr) - P.kBih * bh;  // cahn_hilliard.cpp:294
      }
      res[cx][k] = r;
    }
  __syncthreads();
  // stage transposed ([i][j], reusing sc/sb) and write rhsT[i*outRows + j],
  // one 256 B row segment per warp instruction
  double (*tt)[RY + 1] = reinterpret_cast<double (*)[RY + 1]>(rsm);
#pragma unroll
  for (int cx = 0; cx < 2; ++cx)
#pragma unroll
    for (int k = 0; k < 4; ++k) tt[tx + 32 * cx][ty + 8 * k] = res[cx][k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RX / 8; ++k) {
    const int x = ty + 8 * k;  // i within the tile
    const int i = i0 + x, j = j0 + tx;
    if (i < nx && j < G.outRows) rhsT[static_cast<long long>(i) * G.outRows + j] = tt[x][tx];
  }
}

constexpr size_t kRhsSmem = (2 * RYE * (RXE + 1) + RY * (RX + 1)) * sizeof(double);

// k_rhs_v: the production RHS kernel for nx a multiple of 64 (every CH grid
// with nx >= 64; CHParams requires powers of two). Same output tile (64 i x
// 32 j), restructured for bytes in flight and shared-memory bandwidth:
//  * loads: every 16 B granule (2 columns) of C^n and C^{n-1} in the 68 x 36
//    halo tile is fetched by exactly one thread with independent 16 B loads
//    issued back to back (4 "own" granules per thread + <= 1 halo granule),
//    and transformed on the way into shared memory: sb = 2c - p (Cbar) and
//    sf = c^3 - c (the nonlinear window's per-point term, cahn_hilliard.cpp:
//    36-47); d = c - p of the thread's own outputs stays in registers;
//  * compute: each thread produces a 2-column x 4-row block. Input rows are
//    streamed once (3 x 16 B shared loads per row) and every output row
//    that a row touches accumulates its taps in the reference's row-major tap
//    order, so each sum is the same sequence of operations as before;
//  * store: the 4 consecutive j of one column are 32 B contiguous in rhsT
//    (one full sector) — the transposed layout needs no staging pass.
struct CorrTables {
  const double* W[4];
  const double* y4;  // y4[k*B + b]
};

constexpr int VR = 4;  // output rows per thread
constexpr int VG = RXE / 2;  // 16 B granules per tile row (34)

//
// FUSE (k_rhs_v<NL, true>, the steady-state single-GPU step): the PREVIOUS
// step's combine is folded into the load. Inputs are C^n (cc), C^{n-1} (cp),
// that step's y-sweep output w and its Woodbury coefficients (ty); every
// loaded point first becomes C^{n+1} = (2C^n - C^{n-1}) + (w - W·y) — k_combine's
// expression, term for term — which is written to cnew (own points only)
// and then plays C^n's role in this step's RHS, with C^n as C^{n-1}.
// 40 B/pt instead of k_combine's 32 + k_rhs_v's 24.
template <bool NONLINEAR, bool FUSE>
__global__ void __launch_bounds__(256, FUSE ? 2 : 4) k_rhs_v(const double* __restrict__ cc, const double* __restrict__ cp,
                                                              double* __restrict__ rhsT, const RhsGeom G,
                                                              const __grid_constant__ RhsParams P,
                                                              const double* __restrict__ wv, const CorrTables cy,
                                                              double* __restrict__ cnew) {
  __shared__ __align__(16) double sb[RYE][RXE];
  __shared__ __align__(16) double sf[NONLINEAR ? RYE : 1][RXE];
  const int nx = G.nx;
  const int i0 = blockIdx.x * RX, j0 = blockIdx.y * RY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * 32 + tx;
  pdl_wait();
  auto in_row = [&](int y) {  // tile row y (0..RYE) -> input row
    int j = j0 - HALO + y + G.inShift;
    if (G.wrapY) return G.inRows >= RYE ? wrap_once(j, G.inRows) : wrapi(j, G.inRows);
    return min(max(j, 0), G.inRows - 1);
  };
  auto put = [&](int y, int g, double2 c, double2 p) {
    double2 b, f;
    b.x = 2.0 * c.x - p.x;  // cahn_hilliard.cpp:273
    b.y = 2.0 * c.y - p.y;
    *reinterpret_cast<double2*>(&sb[y][2 * g]) = b;
    if constexpr (NONLINEAR) {
      f.x = c.x * c.x * c.x - c.x;
      f.y = c.y * c.y * c.y - c.y;
      *reinterpret_cast<double2*>(&sf[y][2 * g]) = f;
    }
  };
  // ---- loads: 4 own granules (rows 2 + 4ty + r, granule tx + 1) + 1 halo
  double2 oc[VR], op[VR], ow[VR], hc, hp, hw;
  int hy = 0, hg = 0, hi = 0;
  const bool halo = tid < 2 * VG * 2 + 2 * RY;  // 136 edge-row + 64 edge-column granules
  long long oidx[VR];
#pragma unroll
  for (int r = 0; r < VR; ++r) {
    oidx[r] = static_cast<long long>(in_row(HALO + VR * ty + r)) * nx + i0 + 2 * tx;
    oc[r] = __ldg(reinterpret_cast<const double2*>(cc + oidx[r]));
    op[r] = __ldg(reinterpret_cast<const double2*>(cp + oidx[r]));
    if constexpr (FUSE) ow[r] = __ldg(reinterpret_cast<const double2*>(wv + oidx[r]));
  }
  if (halo) {
    if (tid < 4 * VG) {
      const int k = tid / VG;
      hy = k < 2 ? k : RY + k;  // rows 0, 1, RY+2, RY+3
      hg = tid - k * VG;
    } else {
      const int h = tid - 4 * VG;
      hy = HALO + (h >> 1);
      hg = (h & 1) ? VG - 1 : 0;
    }
    hi = i0 - HALO + 2 * hg;
    hi = hi < 0 ? hi + nx : (hi >= nx ? hi - nx : hi);
    const long long idx = static_cast<long long>(in_row(hy)) * nx + hi;
    hc = __ldg(reinterpret_cast<const double2*>(cc + idx));
    hp = __ldg(reinterpret_cast<const double2*>(cp + idx));
    if constexpr (FUSE) hw = __ldg(reinterpret_cast<const double2*>(wv + idx));
  }
  if constexpr (FUSE) {
    // C^{n+1} at granule (row, columns i, i+1): k_combine's arithmetic
    // (penta.cpp:283-284 correction, cahn_hilliard.cpp:273,320)
    auto advance = [&](int row, int i, double2 c, double2 p, double2 w) {
      const double W0 = __ldg(cy.W[0] + row), W1 = __ldg(cy.W[1] + row), W2 = __ldg(cy.W[2] + row),
                   W3 = __ldg(cy.W[3] + row);
      const double2 y0 = __ldg(reinterpret_cast<const double2*>(cy.y4 + i));
      const double2 y1 = __ldg(reinterpret_cast<const double2*>(cy.y4 + nx + i));
      const double2 y2 = __ldg(reinterpret_cast<const double2*>(cy.y4 + 2LL * nx + i));
      const double2 y3 = __ldg(reinterpret_cast<const double2*>(cy.y4 + 3LL * nx + i));
      double2 r;
      r.x = (2.0 * c.x - p.x) + (w.x - (W0 * y0.x + W1 * y1.x + W2 * y2.x + W3 * y3.x));
      r.y = (2.0 * c.y - p.y) + (w.y - (W0 * y0.y + W1 * y1.y + W2 * y2.y + W3 * y3.y));
      return r;
    };
#pragma unroll
    for (int r = 0; r < VR; ++r) {
      const double2 cn = advance(in_row(HALO + VR * ty + r), i0 + 2 * tx, oc[r], op[r], ow[r]);
      if (j0 + VR * ty + r < G.outRows) *reinterpret_cast<double2*>(cnew + oidx[r]) = cn;
      op[r] = oc[r];  // this step's C^{n-1} is the loaded C^n
      oc[r] = cn;
    }
    if (halo) {
      const double2 cn = advance(in_row(hy), hi, hc, hp, hw);
      hp = hc;
      hc = cn;
    }
  }
  double d[VR][2];
#pragma unroll
  for (int r = 0; r < VR; ++r) {
    put(HALO + VR * ty + r, tx + 1, oc[r], op[r]);
    d[r][0] = oc[r].x - op[r].x;
    d[r][1] = oc[r].y - op[r].y;
  }
  if (halo) put(hy, hg, hc, hp);
  __syncthreads();

  // ---- compute: outputs (x0 + cx, y0 + r), cx < 2, r < 4
  const int x0 = 2 * tx, y0 = VR * ty;
  double bh[VR][2], nl[VR][2];
#pragma unroll
  for (int r = 0; r < VR; ++r) bh[r][0] = bh[r][1] = nl[r][0] = nl[r][1] = 0.0;
#pragma unroll
  for (int yy = 0; yy < VR + 4; ++yy) {  // Cbar rows y0 .. y0 + 7
    double b[6];
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      const double2 v = *reinterpret_cast<const double2*>(&sb[y0 + yy][x0 + 2 * g]);
      b[2 * g] = v.x;
      b[2 * g + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < VR; ++r) {
      const int q = yy - r;
      if (q < 0 || q > 4) continue;
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        constexpr unsigned kMask = (1u << 2) | (1u << 6) | (1u << 7) | (1u << 8) | (1u << 10) | (1u << 11) |
                                   (1u << 12) | (1u << 13) | (1u << 14) | (1u << 16) | (1u << 17) | (1u << 18) |
                                   (1u << 22);  // SG_BIH_TAPS
        if (!((kMask >> (q * 5 + p)) & 1u)) continue;
        bh[r][0] += P.bw[q * 5 + p] * b[p];
        bh[r][1] += P.bw[q * 5 + p] * b[p + 1];
      }
    }
  }
  if constexpr (NONLINEAR) {
#pragma unroll
    for (int yy = 0; yy < VR + 2; ++yy) {  // f rows y0 + 1 .. y0 + 6
      double f[6];
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        const double2 v = *reinterpret_cast<const double2*>(&sf[y0 + 1 + yy][x0 + 2 * g]);
        f[2 * g] = v.x;
        f[2 * g + 1] = v.y;
      }
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        const int q = yy - r;
        if (q < 0 || q > 2) continue;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          constexpr unsigned kMask = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);  // SG_NL_TAPS
          if (!((kMask >> (q * 3 + p)) & 1u)) continue;
          nl[r][0] += P.nl[q * 3 + p] * f[1 + p];
          nl[r][1] += P.nl[q * 3 + p] * f[2 + p];
        }
      }
    }
  }
  // ---- combine (cahn_hilliard.cpp:292/294) and store 4 consecutive j per column
  const int jb = j0 + y0;
  if (G.rowOut) {  // row-major: 16 B per lane, 512 B per warp and row
    double res[2][VR];
#pragma unroll
    for (int cx = 0; cx < 2; ++cx)
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        if constexpr (NONLINEAR)
          res[cx][r] = P.kDiff * d[r][cx] - P.kBih * bh[r][cx] + P.kNl * nl[r][cx];
        else
          res[cx][r] = P.kDiff * d[r][cx] - P.kBih * bh[r][cx];
      }
#pragma unroll
    for (int r = 0; r < VR; ++r)
      if (jb + r < G.outRows)
        *reinterpret_cast<double2*>(rhsT + static_cast<long long>(jb + r) * nx + i0 + x0) =
            make_double2(res[0][r], res[1][r]);
    return;
  }
#pragma unroll
  for (int cx = 0; cx < 2; ++cx) {
    double res[VR];
#pragma unroll
    for (int r = 0; r < VR; ++r) {
      if constexpr (NONLINEAR)
        res[r] = P.kDiff * d[r][cx] - P.kBih * bh[r][cx] + P.kNl * nl[r][cx];
      else
        res[r] = P.kDiff * d[r][cx] - P.kBih * bh[r][cx];
    }
    double* dst = rhsT + static_cast<long long>(i0 + x0 + cx) * G.outRows + jb;
    if (jb + VR <= G.outRows && (G.outRows & 1) == 0) {
      reinterpret_cast<double2*>(dst)[0] = make_double2(res[0], res[1]);
      reinterpret_cast<double2*>(dst)[1] = make_double2(res[2], res[3]);
    } else {
#pragma unroll
      for (int r = 0; r < VR; ++r)
        if (jb + r < G.outRows) dst[r] = res[r];
    }
  }
}

// SG_CH_RHS=legacy selects the scalar-load k_rhs (A/B); default k_rhs_v.
// (Measured and not kept, 8192^2 fused: a persistent cp.async-pipelined
// variant with one 117 KB CTA per SM, 1.55x slower; a non-persistent
// cp.async-staged variant at 80 registers / three CTAs per SM, 1.4 % slower
// than k_rhs_v's two 128-register CTAs per SM.)
int rhs_kind() {
  static const int v = [] {
    const char* e = std::getenv("SG_CH_RHS");
    return e && std::strcmp(e, "legacy") == 0 ? 0 : 1;
  }();
  return v;
}

// ------------------------------------------------------------ k_rhs_tp
// k_rhs_tp<NL>: the steady-state fused combine + RHS (k_rhs_v<NL, true>'s
// arithmetic, term for term) as a persistent tile pipeline. k_rhs_v holds
// its loads in registers (128 per thread, two CTAs per SM) and a CTA
// alternates between a load phase and an FP64 phase, so DRAM idles while
// both CTAs of an SM compute (4.7 TB/s at 8192^2). Here one CTA per SM
// walks the 64 x 32 output tiles round-robin:
//  * one producer thread streams each tile's 68 x 36 halo windows of C^n,
//    C^{n-1} and w, the window's 36 rows of the four y Woodbury vectors and
//    its 68 columns of y4 into a 3-stage shared-memory ring: five 2D tensor
//    TMA boxes per tile, completion on a per-stage mbarrier. (One bulk copy
//    per window row — 116 per tile — measured 2x slower than k_rhs_v: small
//    copies serialise in the TMA unit.) Boxes reaching past the grid edge
//    read zeros there; the consumers of such a tile (2 % at 8192^2) patch
//    the periodic wrap from global memory before the transform;
//  * two consumer groups of eight warps take alternate tiles: the
//    transform (C^{n+1}, Cbar = 2C^{n+1} - C^n, c^3 - c) is done in place in
//    the stage (Cbar over the C^{n-1} window, c^3 - c over the w window),
//    then the 13-tap biharmonic and 5-tap nonlinear sums run as in k_rhs_v;
//    the stage is released through an "empty" mbarrier.
// No registers hold loads, so the ring keeps ~60-120 KB per SM in flight
// through the FP64 phase.
constexpr int TP_NST = 3;  // ring stages
constexpr int TP_NG = 2;   // consumer groups (8 warps each)
constexpr int TP_THREADS = 32 * (8 * TP_NG + 1);

struct TpStage {
  double c[RYE][RXE];  // C^n window, then (in place) nothing
  double p[RYE][RXE];  // C^{n-1} window, then Cbar
  double w[RYE][RXE];  // w window, then c^3 - c
  double W[4][RYE];    // y Woodbury vectors, the window's rows
  double y[4][RXE];    // y4, the window's columns
};
constexpr uint32_t kTpStageBytes = sizeof(TpStage);
struct TpMaps {
  CUtensorMap c, p, w;  // (nx, ny) fields, box (RXE, RYE)
  CUtensorMap W;        // y Woodbury vectors (ny, 4), box (RYE, 4)
  CUtensorMap y;        // y4 (nx, 4), box (RXE, 4)
};
constexpr size_t kTpSmem = TP_NST * sizeof(TpStage) + 2 * TP_NST * sizeof(uint64_t);
static_assert(sizeof(TpStage) % 16 == 0 && offsetof(TpStage, W) % 16 == 0 && offsetof(TpStage, y) % 16 == 0,
              "bulk-copy destinations must be 16 B aligned");

__device__ __forceinline__ uint32_t ch_s32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ch_mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(ch_s32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void ch_tma_2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          ch_s32(dst)),
      "l"(m), "r"(x), "r"(y), "r"(ch_s32(bar))
      : "memory");
}

// Tile t's origin: row-major over tiles (band 0), or bands of `band` tile
// rows walked column by column (vertical neighbours run in the same wave).
__device__ __forceinline__ void tp_tile_origin(int t, int tilesX, int band, int& i0, int& j0) {
  if (band <= 0) {
    i0 = (t % tilesX) * RX;
    j0 = (t / tilesX) * RY;
    return;
  }
  const int per = tilesX * band, b = t / per, r = t - b * per;
  i0 = (r / band) * RX;
  j0 = (b * band + r % band) * RY;
}

// The pipeline of one CTA (index cta of nCta walking the tiles).
template <bool NONLINEAR>
__device__ __forceinline__ void rhs_tp_body(const double* __restrict__ cc, const double* __restrict__ cp,
                                            const double* __restrict__ wv, const CorrTables& cy,
                                            double* __restrict__ cnew, double* __restrict__ rhs, int nx, int ny,
                                            int band, const RhsParams& P, const TpMaps& M, int cta, int nCta,
                                            unsigned char* tp_raw) {
  TpStage* st = reinterpret_cast<TpStage*>(tp_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(tp_raw + TP_NST * sizeof(TpStage));
  uint64_t* empty = full + TP_NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tilesX = nx / RX, nTiles = tilesX * (ny / RY);
  if (threadIdx.x == 0) {
    for (int s = 0; s < TP_NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ch_s32(full + s)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;" ::"r"(ch_s32(empty + s)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  const int myTiles = cta < nTiles ? (nTiles - 1 - cta) / nCta + 1 : 0;

  if (warp == 8 * TP_NG) {  // ---- producer (one thread)
    if (lane != 0) return;
    for (int k = 0; k < myTiles; ++k) {
      const int s = k % TP_NST;
      if (k >= TP_NST) ch_mbar_wait(empty + s, ((k / TP_NST) - 1) & 1);
      const int tile = cta + k * nCta;
      int i0, j0;
      tp_tile_origin(tile, tilesX, band, i0, j0);
      TpStage& S = st[s];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ch_s32(full + s)),
                   "r"(kTpStageBytes)
                   : "memory");
      ch_tma_2d(S.c, &M.c, i0 - HALO, j0 - HALO, full + s);
      ch_tma_2d(S.p, &M.p, i0 - HALO, j0 - HALO, full + s);
      ch_tma_2d(S.w, &M.w, i0 - HALO, j0 - HALO, full + s);
      ch_tma_2d(S.W, &M.W, j0 - HALO, 0, full + s);
      ch_tma_2d(S.y, &M.y, i0 - HALO, 0, full + s);
    }
    return;
  }

  // ---- consumers: group g takes tiles g, g + NG, ...
  const int g = warp >> 3, ty = warp & 7, tx = lane, tid = ty * 32 + tx;
  const int x0 = 2 * tx, y0 = VR * ty;
  // halo granule of this thread (k_rhs_v's assignment): rows 0, 1, RY+2,
  // RY+3 (34 granules each), then the two edge granules of rows 2..RY+1
  const bool halo = tid < 2 * VG * 2 + 2 * RY;
  int hy = 0, hg = 0;
  if (tid < 4 * VG) {
    const int k = tid / VG;
    hy = k < 2 ? k : RY + k;
    hg = tid - k * VG;
  } else {
    const int h = tid - 4 * VG;
    hy = HALO + (h >> 1);
    hg = (h & 1) ? VG - 1 : 0;
  }
  for (int k = g; k < myTiles; k += TP_NG) {
    const int s = k % TP_NST;
    // Consecutive uses of a stage alternate between the groups, so this
    // group may reach tile k while the stage's previous tile (k - NST, the
    // other group's) is not even loaded: a parity wait on `full` alone would
    // then match that older phase. Waiting for the release of tile k - NST
    // first pins the phase (tile k - 2 NST was this group's own release).
    if (k >= TP_NST) ch_mbar_wait(empty + s, ((k / TP_NST) - 1) & 1);
    ch_mbar_wait(full + s, (k / TP_NST) & 1);
    const int tile = cta + k * nCta;
    int i0, j0;
    tp_tile_origin(tile, tilesX, band, i0, j0);
    TpStage& S = st[s];
    const bool ex = i0 == 0 || i0 + RX == nx, ey = j0 == 0 || j0 + RY == ny;
    if (ex || ey) {  // periodic wrap of the boxes' out-of-grid parts
      for (int e = tid; e < RYE * RXE; e += 256) {
        const int y = e / RXE, x = e - y * RXE;
        const int j = j0 - HALO + y, i = i0 - HALO + x;
        if (j >= 0 && j < ny && i >= 0 && i < nx) continue;
        const long long idx = static_cast<long long>(wrap_once(j, ny)) * nx + wrap_once(i, nx);
        S.c[y][x] = __ldg(cc + idx);
        S.p[y][x] = __ldg(cp + idx);
        S.w[y][x] = __ldg(wv + idx);
      }
      if (ey)
        for (int e = tid; e < 4 * RYE; e += 256) {
          const int q = e / RYE, y = e - q * RYE, j = j0 - HALO + y;
          if (j < 0 || j >= ny) S.W[q][y] = __ldg(cy.W[0] + static_cast<long long>(q) * ny + wrap_once(j, ny));
        }
      if (ex)
        for (int e = tid; e < 4 * RXE; e += 256) {
          const int q = e / RXE, x = e - q * RXE, i = i0 - HALO + x;
          if (i < 0 || i >= nx) S.y[q][x] = __ldg(cy.y4 + static_cast<long long>(q) * nx + wrap_once(i, nx));
        }
      asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
    }
    // C^{n+1} at window granule (y, gc): k_combine's arithmetic
    // (penta.cpp:283-284 correction, cahn_hilliard.cpp:273,320), then
    // Cbar and c^3 - c in place; returns C^{n+1}, leaves C^n in cOld
    auto advance = [&](int y, int gc, double2& cOld) {
      const double2 c = *reinterpret_cast<const double2*>(&S.c[y][2 * gc]);
      const double2 p = *reinterpret_cast<const double2*>(&S.p[y][2 * gc]);
      const double2 w = *reinterpret_cast<const double2*>(&S.w[y][2 * gc]);
      const double W0 = S.W[0][y], W1 = S.W[1][y], W2 = S.W[2][y], W3 = S.W[3][y];
      const double2 y0v = *reinterpret_cast<const double2*>(&S.y[0][2 * gc]);
      const double2 y1v = *reinterpret_cast<const double2*>(&S.y[1][2 * gc]);
      const double2 y2v = *reinterpret_cast<const double2*>(&S.y[2][2 * gc]);
      const double2 y3v = *reinterpret_cast<const double2*>(&S.y[3][2 * gc]);
      double2 r;
      r.x = (2.0 * c.x - p.x) + (w.x - (W0 * y0v.x + W1 * y1v.x + W2 * y2v.x + W3 * y3v.x));
      r.y = (2.0 * c.y - p.y) + (w.y - (W0 * y0v.y + W1 * y1v.y + W2 * y2v.y + W3 * y3v.y));
      double2 b;
      b.x = 2.0 * r.x - c.x;  // cahn_hilliard.cpp:273 (this step's Cbar)
      b.y = 2.0 * r.y - c.y;
      *reinterpret_cast<double2*>(&S.p[y][2 * gc]) = b;
      if constexpr (NONLINEAR) {
        double2 f;
        f.x = r.x * r.x * r.x - r.x;
        f.y = r.y * r.y * r.y - r.y;
        *reinterpret_cast<double2*>(&S.w[y][2 * gc]) = f;
      }
      cOld = c;
      return r;
    };
    double d[VR][2];
#pragma unroll
    for (int r = 0; r < VR; ++r) {
      double2 c;
      const double2 cn = advance(HALO + y0 + r, tx + 1, c);
      *reinterpret_cast<double2*>(cnew + static_cast<long long>(j0 + y0 + r) * nx + i0 + x0) = cn;
      d[r][0] = cn.x - c.x;
      d[r][1] = cn.y - c.y;
    }
    if (halo) {
      double2 c;
      advance(hy, hg, c);
    }
    asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");

    double bh[VR][2], nl[VR][2];
#pragma unroll
    for (int r = 0; r < VR; ++r) bh[r][0] = bh[r][1] = nl[r][0] = nl[r][1] = 0.0;
#pragma unroll
    for (int yy = 0; yy < VR + 4; ++yy) {  // Cbar rows y0 .. y0 + 7
      double b[6];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(&S.p[y0 + yy][x0 + 2 * q]);
        b[2 * q] = v.x;
        b[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        const int q = yy - r;
        if (q < 0 || q > 4) continue;
#pragma unroll
        for (int p = 0; p < 5; ++p) {
          constexpr unsigned kMask = (1u << 2) | (1u << 6) | (1u << 7) | (1u << 8) | (1u << 10) | (1u << 11) |
                                     (1u << 12) | (1u << 13) | (1u << 14) | (1u << 16) | (1u << 17) | (1u << 18) |
                                     (1u << 22);  // SG_BIH_TAPS
          if (!((kMask >> (q * 5 + p)) & 1u)) continue;
          bh[r][0] += P.bw[q * 5 + p] * b[p];
          bh[r][1] += P.bw[q * 5 + p] * b[p + 1];
        }
      }
    }
    if constexpr (NONLINEAR) {
#pragma unroll
      for (int yy = 0; yy < VR + 2; ++yy) {  // c^3 - c rows y0 + 1 .. y0 + 6
        double f[6];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(&S.w[y0 + 1 + yy][x0 + 2 * q]);
          f[2 * q] = v.x;
          f[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < VR; ++r) {
          const int q = yy - r;
          if (q < 0 || q > 2) continue;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            constexpr unsigned kMask = (1u << 1) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7);  // SG_NL_TAPS
            if (!((kMask >> (q * 3 + p)) & 1u)) continue;
            nl[r][0] += P.nl[q * 3 + p] * f[1 + p];
            nl[r][1] += P.nl[q * 3 + p] * f[2 + p];
          }
        }
      }
    }
    // this thread's last shared-memory access of the stage: release it
    // (generic-proxy writes above precede the next bulk copy into it)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ch_s32(empty + s)) : "memory");
#pragma unroll
    for (int r = 0; r < VR; ++r) {
      double2 o;
      if constexpr (NONLINEAR) {  // cahn_hilliard.cpp:292
        o.x = P.kDiff * d[r][0] - P.kBih * bh[r][0] + P.kNl * nl[r][0];
        o.y = P.kDiff * d[r][1] - P.kBih * bh[r][1] + P.kNl * nl[r][1];
      } else {  // cahn_hilliard.cpp:294
        o.x = P.kDiff * d[r][0] - P.kBih * bh[r][0];
        o.y = P.kDiff * d[r][1] - P.kBih * bh[r][1];
      }
      *reinterpret_cast<double2*>(rhs + static_cast<long long>(j0 + y0 + r) * nx + i0 + x0) = o;
    }
  }
}

template <bool NONLINEAR>
__global__ void __launch_bounds__(TP_THREADS, 1) k_rhs_tp(const double* __restrict__ cc, const double* __restrict__ cp,
                                                         const double* __restrict__ wv, const CorrTables cy,
                                                         double* __restrict__ cnew, double* __restrict__ rhs,
                                                         int nx, int ny, int band,
                                                         const __grid_constant__ RhsParams P,
                                                         const __grid_constant__ TpMaps M) {
  extern __shared__ __align__(128) unsigned char tp_raw[];
  rhs_tp_body<NONLINEAR>(cc, cp, wv, cy, cnew, rhs, nx, ny, band, P, M, blockIdx.x, gridDim.x, tp_raw);
}

int ch_sm_count() {
  static const int v = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

// Tensor maps of the pipeline, cached by (pointer, shape): the CH buffers
// are long-lived and a map only encodes the address and the shape.
bool tp_map(CUtensorMap* m, const double* p, int d0, int d1, int b0, int b1) {
  static std::mutex mu;
  static std::map<std::tuple<const double*, int, int, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(p, d0, d1, b0, b1);
  auto it = cache.find(key);
  if (it == cache.end()) {
    CUtensorMap enc;
    if (!encode_tile_map(&enc, p, d0, d1, b0, b1)) return false;
    it = cache.emplace(key, enc).first;
  }
  *m = it->second;
  return true;
}

// SG_CH_RHS_TP=0 keeps k_rhs_v<NL, true> for the steady-state step (A/B);
// =2 uses the pipeline on every eligible grid, however few tiles (tests).
int rhs_tp_mode() {
  static const int v = [] {
    const char* e = std::getenv("SG_CH_RHS_TP");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
// SG_CH_RHS_TP_CTAS=n caps the pipeline's grid (tests: many tiles per CTA,
// so the ring wraps on small grids).
int rhs_tp_ctas() {
  static const int v = [] {
    const char* e = std::getenv("SG_CH_RHS_TP_CTAS");
    const int n = e ? std::atoi(e) : 0;
    return n > 0 ? std::min(n, ch_sm_count()) : ch_sm_count();
  }();
  return v;
}

// The steady-state step's first kernel: previous combine + this RHS (k_rhs_v
// FUSE). Single GPU (full periodic grid), nx a multiple of 64.
void launch_rhs_fused(bool nonlinear, const double* cc, const double* cp, const double* w, const CorrTables& ty,
                      double* cnew, double* rhsT, const RhsGeom& g, const RhsParams& rp, cudaStream_t s, bool pdl) {
  // the pipeline needs the y Woodbury vectors contiguous ([4][ny], ChState's
  // wyCat copy) and boxes no larger than the grid
  const bool wcat = ty.W[1] == ty.W[0] + g.outRows && ty.W[2] == ty.W[1] + g.outRows && ty.W[3] == ty.W[2] + g.outRows;
  TpMaps maps;
  // (below ~4 tiles per SM the ring never fills: 1024^2 measured 1 % slower)
  const long long tiles = static_cast<long long>(g.nx / RX) * (g.outRows / RY);
  const int mode = rhs_tp_mode();
  if (mode != 0 && wcat && g.rowOut && g.outRows % RY == 0 && g.nx % RX == 0 && g.nx >= 2 * RX &&
      g.outRows >= 2 * RY && (mode == 2 || tiles >= 4LL * ch_sm_count()) && tp_map(&maps.c, cc, g.nx, g.outRows, RXE, RYE) &&
      tp_map(&maps.p, cp, g.nx, g.outRows, RXE, RYE) && tp_map(&maps.w, w, g.nx, g.outRows, RXE, RYE) &&
      tp_map(&maps.W, ty.W[0], g.outRows, 4, RYE, 4) && tp_map(&maps.y, ty.y4, g.nx, 4, RXE, 4)) {
    static bool configured = false;
    if (!configured) {
      SG_CUDA(cudaFuncSetAttribute(k_rhs_tp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kTpSmem)));
      SG_CUDA(cudaFuncSetAttribute(k_rhs_tp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kTpSmem)));
      configured = true;
    }
    const int grid = static_cast<int>(std::min<long long>(tiles, rhs_tp_ctas()));
    // tiles walked in bands of two tile rows, column by column: 8192^2
    // 796 -> 835 steps/s against row-major order (SG_CH_RHS_TP_BAND=1;
    // bands of 4 / 8: 830 / 828), 4096^2 and 2048^2 within 1 %
    static const int band = [] {
      const char* e = std::getenv("SG_CH_RHS_TP_BAND");
      return e ? std::atoi(e) : 2;
    }();
    launch_ex(nonlinear ? k_rhs_tp<true> : k_rhs_tp<false>, dim3(grid), dim3(TP_THREADS), kTpSmem, s, pdl, cc, cp,
              w, ty, cnew, rhsT, g.nx, g.outRows, band > 0 && (g.outRows / RY) % band == 0 ? band : 0, rp, maps);
    check_launch("ch fused combine+rhs pipeline kernel");
    return;
  }
  dim3 tb(32, 8), tg(g.nx / RX, (g.outRows + RY - 1) / RY);
  launch_ex(nonlinear ? k_rhs_v<true, true> : k_rhs_v<false, true>, tg, tb, 0, s, pdl, cc, cp, rhsT, g, rp, w, ty,
            cnew);
  check_launch("ch fused combine+rhs kernel");
}

void launch_rhs(bool nonlinear, const double* cc, const double* cp, double* rhsT, const RhsGeom& g,
                const RhsParams& rp, cudaStream_t s, bool pdl = false) {
  static bool configured = false;
  if (!configured) {
    SG_CUDA(cudaFuncSetAttribute(k_rhs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kRhsSmem)));
    SG_CUDA(cudaFuncSetAttribute(k_rhs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kRhsSmem)));
    configured = true;
  }
  dim3 tb(32, 8), tg((g.nx + RX - 1) / RX, (g.outRows + RY - 1) / RY);
  const bool legacy = rhs_kind() == 0;
  if (g.nx % RX == 0 && !legacy) {
    launch_ex(nonlinear ? k_rhs_v<true, false> : k_rhs_v<false, false>, tg, tb, 0, s, pdl, cc, cp, rhsT, g, rp,
              static_cast<const double*>(nullptr), CorrTables{}, static_cast<double*>(nullptr));
    check_launch("ch rhs kernel");
    return;
  }
  if (nonlinear)
    k_rhs<true><<<tg, tb, kRhsSmem, s>>>(cc, cp, rhsT, g, rp);
  else
    k_rhs<false><<<tg, tb, kRhsSmem, s>>>(cc, cp, rhsT, g, rp);
  check_launch("ch rhs kernel");
}

// w(i,jl) = zT[i*own + jl] - (Wx0[i] y0[jl] + Wx1[i] y1[jl] + Wx2[i] y2[jl] + Wx3[i] y3[jl]),
// stored PACKED for the all-to-all: block q = i / nxq holds own x nxq
// (row jl, column i % nxq). With one rank (nxq = nx) this is row-major w.
__global__ void __launch_bounds__(256) k_transpose_correct(const double* __restrict__ zT,
                                                           double* __restrict__ w, int nx, int own, int nxq,
                                                           const CorrTables t) {
  __shared__ double tile[TS][TS + 1];
  const int i0 = blockIdx.x * TS, j0 = blockIdx.y * TS;
  const int tx = threadIdx.x, ty = threadIdx.y;
  pdl_wait();
#pragma unroll
  for (int k = 0; k < TS / 8; ++k) {
    const int i = i0 + ty + 8 * k, j = j0 + tx;
    if (i < nx && j < own) {
      const double z = zT[static_cast<long long>(i) * own + j];
      const double corr = __ldg(t.W[0] + i) * __ldg(t.y4 + j) + __ldg(t.W[1] + i) * __ldg(t.y4 + own + j) +
                          __ldg(t.W[2] + i) * __ldg(t.y4 + 2LL * own + j) +
                          __ldg(t.W[3] + i) * __ldg(t.y4 + 3LL * own + j);
      tile[ty + 8 * k][tx] = z - corr;  // penta.cpp:283-284
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < TS / 8; ++k) {
    const int j = j0 + ty + 8 * k, i = i0 + tx;
    if (i < nx && j < own) {
      const int q = i / nxq, c = i - q * nxq;
      w[static_cast<long long>(q) * own * nxq + static_cast<long long>(j) * nxq + c] = tile[tx][ty + 8 * k];
    }
  }
}

// Same operation on 64 x 64 tiles (nx, own multiples of 64): 512 B row
// segments on both sides of the transpose (DRAM page locality), the four
// y4 values of a thread's two j columns loaded once, 16 independent zT loads
// per thread in flight.
constexpr int TT = 64;
__global__ void __launch_bounds__(256) k_transpose_correct_v(const double* __restrict__ zT,
                                                             double* __restrict__ w, int nx, int own, int nxq,
                                                             const CorrTables t) {
  __shared__ double tile[TT][TT + 1];
  const int i0 = blockIdx.x * TT, j0 = blockIdx.y * TT;
  const int tx = threadIdx.x, ty = threadIdx.y;
  pdl_wait();
  double y4[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < 4; ++k) y4[h][k] = __ldg(t.y4 + static_cast<long long>(k) * own + j0 + tx + 32 * h);
  double z[TT / 8][2];
#pragma unroll
  for (int k = 0; k < TT / 8; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      z[k][h] = zT[static_cast<long long>(i0 + ty + 8 * k) * own + j0 + tx + 32 * h];
#pragma unroll
  for (int k = 0; k < TT / 8; ++k) {
    const int i = i0 + ty + 8 * k;
    const double w0 = __ldg(t.W[0] + i), w1 = __ldg(t.W[1] + i), w2 = __ldg(t.W[2] + i), w3 = __ldg(t.W[3] + i);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double corr = w0 * y4[h][0] + w1 * y4[h][1] + w2 * y4[h][2] + w3 * y4[h][3];
      tile[ty + 8 * k][tx + 32 * h] = z[k][h] - corr;  // penta.cpp:283-284
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < TT / 8; ++k) {
    const int j = j0 + ty + 8 * k;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = i0 + tx + 32 * h;
      const int q = i / nxq, c = i - q * nxq;
      w[static_cast<long long>(q) * own * nxq + static_cast<long long>(j) * nxq + c] = tile[tx + 32 * h][ty + 8 * k];
    }
  }
}

void launch_transpose_correct(const double* zT, double* w, int nx, int own, int nxq, const CorrTables& t,
                              cudaStream_t s, bool pdl = false) {
  if (nx % TT == 0 && own % TT == 0 && nxq % 32 == 0) {
    launch_ex(k_transpose_correct_v, dim3(nx / TT, own / TT), dim3(32, 8), 0, s, pdl, zT, w, nx, own, nxq, t);
  } else {
    k_transpose_correct<<<dim3((nx + TS - 1) / TS, (own + TS - 1) / TS), dim3(32, 8), 0, s>>>(zT, w, nx, own,
                                                                                             nxq, t);
  }
  check_launch("ch transpose kernel");
}

// Single GPU: C^{n+1} = (2 C^n - C^{n-1}) + (w - (Wy0[j] y0[i] + ... + Wy3[j] y3[i])), over C^{n-1}.
__global__ void __launch_bounds__(256) k_combine(const double* __restrict__ cc, double* __restrict__ cpNext,
                                                 const double* __restrict__ w, int nx, int ny,
                                                 const CorrTables t) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  pdl_wait();
  if (i >= nx) return;
  const long long idx = static_cast<long long>(j) * nx + i;
  const double v = w[idx] - (__ldg(t.W[0] + j) * __ldg(t.y4 + i) + __ldg(t.W[1] + j) * __ldg(t.y4 + nx + i) +
                             __ldg(t.W[2] + j) * __ldg(t.y4 + 2LL * nx + i) +
                             __ldg(t.W[3] + j) * __ldg(t.y4 + 3LL * nx + i));
  const double cb = 2.0 * cc[idx] - cpNext[idx];
  cpNext[idx] = cb + v;  // cahn_hilliard.cpp:320
}

// y-slab: C^{n+1} = (2 C^n - C^{n-1}) + v with v the (already corrected)
// y-sweep result received PACKED from the all-to-all; fields are ext slabs
// (2 halo rows above the own rows).
__global__ void __launch_bounds__(256) k_combine_packed(const double* __restrict__ ccExt, double* __restrict__ cpExt,
                                                        const double* __restrict__ v, int nx, int own, int nxq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y;
  if (i >= nx) return;
  const long long idx = static_cast<long long>(jl + HALO) * nx + i;
  const int q = i / nxq, c = i - q * nxq;
  const double vv = v[static_cast<long long>(q) * own * nxq + static_cast<long long>(jl) * nxq + c];
  const double cb = 2.0 * ccExt[idx] - cpExt[idx];
  cpExt[idx] = cb + vv;  // cahn_hilliard.cpp:320
}

// y-slab, P2P path: the y-sweep results arrive UNcorrected (packed blocks
// [q][jl][i_local], each straight from rank q's sweep) with every rank's y
// coefficients in y4All[k*nx + i]; the correction and the update are
// k_combine's expression (penta.cpp:283-284, cahn_hilliard.cpp:273,320).
// peerUp / peerDn (optional): the neighbours' ext slabs of the same time
// level — the first HALO rows of C^{n+1} are also stored into the up
// neighbour's bottom halo, the last HALO rows into the down neighbour's top
// halo (peer memory over NVLink), so no halo exchange precedes the next step.
__global__ void __launch_bounds__(256) k_combine_packed_corr(const double* __restrict__ ccExt,
                                                             double* __restrict__ cpExt,
                                                             const double* __restrict__ v, int nx, int own, int nxq,
                                                             int r0, const CorrTables t, double* peerUp,
                                                             double* peerDn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y;
  pdl_wait();
  if (i >= nx) return;
  const int j = r0 + jl;
  const long long idx = static_cast<long long>(jl + HALO) * nx + i;
  const int q = i / nxq, c = i - q * nxq;
  const double w = v[static_cast<long long>(q) * own * nxq + static_cast<long long>(jl) * nxq + c];
  const double vv = w - (__ldg(t.W[0] + j) * __ldg(t.y4 + i) + __ldg(t.W[1] + j) * __ldg(t.y4 + nx + i) +
                         __ldg(t.W[2] + j) * __ldg(t.y4 + 2LL * nx + i) + __ldg(t.W[3] + j) * __ldg(t.y4 + 3LL * nx + i));
  const double cb = 2.0 * ccExt[idx] - cpExt[idx];
  const double cn = cb + vv;  // cahn_hilliard.cpp:320
  cpExt[idx] = cn;
  if (peerUp && jl < HALO) peerUp[static_cast<long long>(HALO + own + jl) * nx + i] = cn;
  if (peerDn && jl >= own - HALO) peerDn[static_cast<long long>(jl - (own - HALO)) * nx + i] = cn;
}

// initial_condition on a slab: global element index k = (r0 + jl)*nx + i.
__global__ void k_init_slab(unsigned long long seed, double amp, int nx, int own, int r0, double* __restrict__ ext) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y;
  if (i >= nx) return;
  const long long k = static_cast<long long>(r0 + jl) * nx + i;
  unsigned long long z = seed + static_cast<unsigned long long>(k + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z = z ^ (z >> 31);
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  ext[static_cast<long long>(jl + HALO) * nx + i] = amp * (2.0 * u - 1.0);
}

// Bands of the uniform hyperdiffusion operator (penta.cpp:313-335) for one
// periodic system: {sigma, -4 sigma, 1 + 6 sigma, -4 sigma, sigma}.
__global__ void k_fill_bands(double sigma, int n, double* e, double* c, double* d, double* a, double* b) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  e[r] = sigma;
  c[r] = -4.0 * sigma;
  d[r] = 1.0 + 6.0 * sigma;
  a[r] = -4.0 * sigma;
  b[r] = sigma;
}

}  // namespace

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SG_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

static void k_init_slab_launch(unsigned long long seed, double amp, int nx, int own, int r0, double* ext,
                        cudaStream_t s) {
  k_init_slab<<<dim3((nx + 255) / 256, own), 256, 0, s>>>(seed, amp, nx, own, r0, ext);
  check_launch("ch slab init kernel");
}

static void ch_phase_x(const sg_ch_params& p, const RhsParams& rp, const PentaTables& fx, int own, int nxq,
                const double* cur, const double* prev, double* rhsT, double* y4x, double* send, cudaStream_t s) {
  const int nx = p.nx;
  const RhsGeom geom{nx, own, own + 2 * HALO, HALO, 0};
  launch_rhs(p.nonlinearEnabled, cur, prev, rhsT, geom, rp, s);
  penta_sweep(fx, own, nx, rhsT, y4x, true, true, s);
  CorrTables tx{{fx.W[0], fx.W[1], fx.W[2], fx.W[3]}, y4x};
  launch_transpose_correct(rhsT, send, nx, own, nxq, tx, s);
}

static void ch_combine_packed(int nx, int own, int nxq, const double* cur, double* prev, const double* recv,
                       cudaStream_t s) {
  k_combine_packed<<<dim3((nx + 255) / 256, own), 256, 0, s>>>(cur, prev, recv, nx, own, nxq);
  check_launch("ch slab combine kernel");
}

namespace {

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// (An earlier design applied the x correction inside the y-sweep's chain
// warp and wrote the x results transposed from the chain warp: measured
// slower than the separate pass at 1024^2 and 8192^2 and removed; the XIN
// sweeps move that work to three transform warps instead.)

}  // namespace

void ch_validate(const sg_ch_params& p) {  // CHParams::validate, cahn_hilliard.cpp:56-66
  if (!(p.D > 0.0)) invalid("CHParams: D must be > 0");
  if (!(p.gamma > 0.0)) invalid("CHParams: gamma must be > 0");
  if (!(p.dt > 0.0)) invalid("CHParams: dt must be > 0");
  if (!(p.T > 0.0)) invalid("CHParams: T must be > 0");
  if (!(p.lx > 0.0) || !(p.ly > 0.0)) invalid("CHParams: lx, ly must be > 0");
  if (!is_pow2(p.nx) || !is_pow2(p.ny)) invalid("CHParams: nx and ny must be powers of two");
  if (p.nx < 8 || p.ny < 8) invalid("CHParams: grid too small (need >= 8)");
  if (!(p.icAmplitude >= 0.0)) invalid("CHParams: icAmplitude must be >= 0");
}

struct ChState {
  sg_ch_params p{};
  int device = 0;
  cudaStream_t stream = nullptr;
  // Three time-level buffers: field[ic] = C^n, field[ip] = C^{n-1}, the third
  // receives C^{n+1} in the fused steady-state step (its RHS kernel reads a
  // halo around every point, so C^{n+1} cannot overwrite C^{n-1} in place).
  double* field[3] = {nullptr, nullptr, nullptr};
  int ic = 0, ip = 1;
  double *rhsT = nullptr, *w = nullptr, *y4x = nullptr, *y4y = nullptr;
  // the y factor's four Woodbury vectors copied contiguously ([4][ny]): one
  // tensor map for the steady-state RHS pipeline (k_rhs_tp)
  double* wyCat = nullptr;
  // xpipe: the RHS is written row-major into rhsT, the x-sweep reads it
  // transposed and writes its interleaved result to xT, the y-sweep reads xT
  // transposed with the x Woodbury correction (no transpose kernel)
  double* xT = nullptr;
  bool xpipe = false;
  // Opt-in partitioned sweeps (sg_ch_set_partition, SegPenta): P segments
  // per system; gx/gy interface values, cx the x correction coefficients
  // ([P][4][systems]). 0 = the bitwise default.
  int partP = 0;
  std::unique_ptr<SegPenta> sx, sy;
  double *gx = nullptr, *cx = nullptr, *gy = nullptr;

  DevicePenta fx, fy;
  RhsParams rp{};
  // CUDA graphs keyed by (kind, ic, ip): kind 0 = full step, 1 = head (step
  // without its combine), 2 = steady (previous combine fused into this
  // step's RHS), 3 = three steady steps (the buffer rotation closes), 4 =
  // tail (the pending combine alone), 5 = twelve steady steps.
  std::map<int, cudaGraphExec_t> graphs;
  int solveK = -1;  // kernels one solve launches (counted once, by capture)
  int step = 0;
  std::vector<void*> allocs;

  double* dalloc(size_t n) {
    void* q = nullptr;
    SG_CUDA(cudaMalloc(&q, n * sizeof(double)));
    allocs.push_back(q);
    return static_cast<double*>(q);
  }

  ~ChState() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    for (void* q : allocs) cudaFree(q);
    if (stream) cudaStreamDestroy(stream);
  }

  double* cur() const { return field[ic]; }
  double* prev() const { return field[ip]; }
  int spare() const { return 3 - ic - ip; }

  void build_factor(DevicePenta& f, double sigma, int n) {
    double* bands = dalloc(5 * static_cast<size_t>(n));
    k_fill_bands<<<(n + 255) / 256, 256, 0, stream>>>(sigma, n, bands, bands + n, bands + 2 * n, bands + 3 * n,
                                                      bands + 4 * n);
    check_launch("ch bands kernel");
    f.build(1, n, true, true, bands, bands + n, bands + 2 * n, bands + 3 * n, bands + 4 * n, stream);
    f.B = 0;  // batch count is supplied per sweep
  }

  void init() {
    SG_CUDA(cudaGetDevice(&device));
    // a BLOCKING stream: ordered after work the caller queued on the legacy
    // default stream (e.g. torch kernels producing device inputs)
    SG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamDefault));
    const size_t cnt = static_cast<size_t>(p.nx) * p.ny;
    for (auto& f : field) f = dalloc(cnt);
    rhsT = dalloc(cnt);
    w = dalloc(cnt);
    y4x = dalloc(4 * static_cast<size_t>(p.ny));
    y4y = dalloc(4 * static_cast<size_t>(p.nx));
    const double dx = p.lx / p.nx, dy = p.ly / p.ny;
    // hyperdiffusion_sigma (cahn_hilliard.cpp:19-21), RhsCoeffs (:25-34)
    const double sx = kTwoThirds * p.D * p.gamma * p.dt / pow4(dx);
    const double sy = kTwoThirds * p.D * p.gamma * p.dt / pow4(dy);
    build_factor(fx, sx, p.nx);
    build_factor(fy, sy, p.ny);
    wyCat = dalloc(4 * static_cast<size_t>(p.ny));
    for (int k = 0; k < 4; ++k)
      SG_CUDA(cudaMemcpyAsync(wyCat + static_cast<size_t>(k) * p.ny, fy.t.W[k], p.ny * sizeof(double),
                              cudaMemcpyDeviceToDevice, stream));
    rp.kDiff = -kTwoThirds;
    rp.kBih = kTwoThirds * p.D * p.gamma * p.dt;
    rp.kNl = kTwoThirds * p.D * p.dt;
    biharmonic_weights(dx, dy, rp.bw);
    // nonlinear_laplacian_coefficients (cahn_hilliard.cpp:78-83)
    const double cx = 1.0 / (dx * dx), cy = 1.0 / (dy * dy), cc = -2.0 * cx - 2.0 * cy;
    const double nl[9] = {0.0, cy, 0.0, cx, cc, cx, 0.0, cy, 0.0};
    std::memcpy(rp.nl, nl, sizeof nl);
    // the skipped taps must be exactly zero
    bool keep[25] = {};
    constexpr int kBihTaps[13] = SG_BIH_TAPS;
    for (int t : kBihTaps) keep[t] = true;
    for (int k = 0; k < 25; ++k)
      if (!keep[k] && rp.bw[k] != 0.0) throw Error(SG_ERR_CUDA, "internal: biharmonic zero pattern");
    // the transposed-input sweep pipeline (see xpipe)
    if (xin_ok() && rhs_kind() == 1 && p.nx % RX == 0) {
      xT = dalloc(cnt);

      xpipe = penta_sweep_xin(fx.t, p.ny, p.nx, xT, rhsT, nullptr, nullptr, y4x, stream, false, false) &&
              penta_sweep_xin(fy.t, p.nx, p.ny, w, xT, fx.t.W, y4x, y4y, stream, false, false);
    }
    // initial_condition (cahn_hilliard.cpp:68-76); C^{n-1} := C^n (:218)
    const long long n = static_cast<long long>(cnt);
    k_init<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(p.seed, p.icAmplitude, n, field[0]);
    check_launch("ch init kernel");
    SG_CUDA(cudaMemcpyAsync(field[1], field[0], cnt * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    ic = 0;
    ip = 1;
    step = 0;
    SG_CUDA(cudaStreamSynchronize(stream));
  }

  // The fused steady-state step needs the vectorised RHS kernel (nx a
  // multiple of 64); SG_CH_STEADY=0 disables it (A/B measurements).
  bool steady_ok() const {
    static const bool off = [] {
      const char* e = std::getenv("SG_CH_STEADY");
      return e && e[0] == '0';
    }();
    return !off && p.nx % RX == 0 && rhs_kind() != 0;
  }

  // RHS (or, steady, the fused previous combine + RHS writing C^{n+1} into
  // field[in]), the two sweeps and the transpose/correct between them.
  // Leaves the step's combine pending: C^{n+1} = 2C^n - C^{n-1} + (w - W·y4y).
  void enqueue_solve(int c, int q, int in, cudaStream_t s) {
    const int nx = p.nx, ny = p.ny;
    const RhsGeom geom{nx, ny, ny, 0, 1, xpipe ? 1 : 0};
    const bool pdl = pdl_enabled();
    if (in >= 0) {
      CorrTables ty{{wyCat, wyCat + ny, wyCat + 2LL * ny, wyCat + 3LL * ny}, y4y};
      launch_rhs_fused(p.nonlinearEnabled, field[c], field[q], w, ty, field[in], rhsT, geom, rp, s, pdl);
    } else {
      launch_rhs(p.nonlinearEnabled, field[c], field[q], rhsT, geom, rp, s, pdl);
    }
    if (partP) {
      // partitioned: local solves, interface solves, corrections (the x
      // correction on the y-sweep's load, the y correction in place on w;
      // y4y stays zero, so the combine's W . y4y term adds exactly 0)
      const double* wc[4] = {sx->vec, sx->vec + nx, sx->vec + 2LL * nx, sx->vec + 3LL * nx};
      if (!penta_sweep_seg(*sx, ny, xT, rhsT, nullptr, nullptr, 0, gx, s, pdl))
        throw Error(SG_ERR_CUDA, "internal: partitioned x-sweep unavailable");
      penta_seg_reduce(*sx, ny, gx, cx, s, pdl);
      if (!penta_sweep_seg(*sy, nx, w, xT, wc, cx, sx->m, gy, s, pdl))
        throw Error(SG_ERR_CUDA, "internal: partitioned y-sweep unavailable");
      penta_seg_finish_rows(*sy, nx, w, gy, s, pdl);
      return;
    }
    if (xpipe) {
      // x-sweep: rhs (row-major) read transposed -> xT (interleaved);
      // y-sweep: xT read transposed + x-corrected -> w (row-major)
      if (!penta_sweep_xin(fx.t, ny, nx, xT, rhsT, nullptr, nullptr, y4x, s, pdl) ||
          !penta_sweep_xin(fy.t, nx, ny, w, xT, fx.t.W, y4x, y4y, s, pdl))
        throw Error(SG_ERR_CUDA, "internal: transposed-input sweep unavailable");
      return;
    }
    penta_sweep(fx.t, ny, nx, rhsT, y4x, true, true, s, pdl);
    CorrTables tx{{fx.t.W[0], fx.t.W[1], fx.t.W[2], fx.t.W[3]}, y4x};
    launch_transpose_correct(rhsT, w, nx, ny, nx, tx, s, pdl);
    penta_sweep(fy.t, nx, ny, w, y4y, true, true, s, pdl);
  }

  // SG_CH_XIN=0 keeps the separate transpose/correct kernel (A/B).
  static bool xin_ok() {
    static const bool v = [] {
      const char* e = std::getenv("SG_CH_XIN");
      return !(e && e[0] == '0');
    }();
    return v;
  }

  // The pending combine: C^{n+1} written over C^{n-1} (field[q]) in place.
  void enqueue_combine(int c, int q, cudaStream_t s) {
    const int nx = p.nx, ny = p.ny;
    CorrTables ty{{fy.t.W[0], fy.t.W[1], fy.t.W[2], fy.t.W[3]}, y4y};
    launch_ex(k_combine, dim3((nx + 255) / 256, ny), dim3(256), 0, s, pdl_enabled(),
              static_cast<const double*>(field[c]), field[q], static_cast<const double*>(w), nx, ny, ty);
    check_launch("ch combine kernel");
  }

  // Opt-in partitioned sweeps (P >= 2 segments per system; P <= 1: the
  // bitwise default). Results differ from the reference's operation order;
  // DESIGN.md gives the measured deviation.
  void set_partition(int P) {
    SG_CUDA(cudaStreamSynchronize(stream));
    for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    graphs.clear();
    solveK = -1;
    if (P <= 1) {
      partP = 0;
      return;
    }
    if (!xpipe) invalid("CHStepper: partitioned sweeps need the transposed-input pipeline (nx % 64 == 0)");
    const double dx = p.lx / p.nx, dy = p.ly / p.ny;
    const double sxg = kTwoThirds * p.D * p.gamma * p.dt / pow4(dx);
    const double syg = kTwoThirds * p.D * p.gamma * p.dt / pow4(dy);
    auto mk = [&](double sig, int n) {
      auto sp = std::make_unique<SegPenta>();  // k_fill_bands' values
      sp->build(sig, -4.0 * sig, 1.0 + 6.0 * sig, -4.0 * sig, sig, n, P, stream);
      return sp;
    };
    auto nx_ = mk(sxg, p.nx), ny_ = mk(syg, p.ny);
    if (!gx) {
      gx = dalloc(16 * static_cast<size_t>(p.ny) * 4);
      cx = dalloc(16 * static_cast<size_t>(p.ny) * 4);
      gy = dalloc(16 * static_cast<size_t>(p.nx) * 4);
    }
    const double* wc[4] = {nx_->vec, nx_->vec + p.nx, nx_->vec + 2LL * p.nx, nx_->vec + 3LL * p.nx};
    if (!penta_sweep_seg(*nx_, p.ny, xT, rhsT, nullptr, nullptr, 0, gx, stream, false, false) ||
        !penta_sweep_seg(*ny_, p.nx, w, xT, wc, cx, nx_->m, gy, stream, false, false))
      invalid("CHStepper: partitioned sweeps unavailable for this grid (segments must be multiples of 64 rows)");
    sx = std::move(nx_);
    sy = std::move(ny_);
    SG_CUDA(cudaMemsetAsync(y4y, 0, 4 * static_cast<size_t>(p.nx) * sizeof(double), stream));
    SG_CUDA(cudaStreamSynchronize(stream));
    partP = P;
  }

  cudaGraphExec_t graph(int kind, int c, int q) {
    const int key = kind * 16 + c * 4 + q;
    auto it = graphs.find(key);
    if (it != graphs.end()) return it->second;
    cudaGraph_t g;
    SG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    const uint64_t before = g_launches.load();
    switch (kind) {
      case 0:
        enqueue_solve(c, q, -1, stream);
        enqueue_combine(c, q, stream);
        break;
      case 1:
        enqueue_solve(c, q, -1, stream);
        break;
      case 2:
        enqueue_solve(c, q, 3 - c - q, stream);
        break;
      case 3:
      case 5:  // 3 or 12 steady steps (the rotation closes every 3)
        for (int k = 0, a = c, b = q; k < (kind == 3 ? 3 : 12); ++k) {
          const int n = 3 - a - b;
          enqueue_solve(a, b, n, stream);
          b = a;
          a = n;
        }
        break;
      default:
        enqueue_combine(c, q, stream);
    }
    g_launches.store(before);  // captured, not launched
    SG_CUDA(cudaStreamEndCapture(stream, &g));
    cudaGraphExec_t e;
    SG_CUDA(cudaGraphInstantiate(&e, g, 0));
    SG_CUDA(cudaGraphDestroy(g));
    graphs[key] = e;
    return e;
  }

  void launch(int kind, int kernels) {
    SG_CUDA(cudaGraphLaunch(graph(kind, ic, ip), stream));
    count_launch(kernels);
  }

  // `steps` steps; the state (field[ic], field[ip]) is complete on return.
  // Steady state (nx % 64 == 0, steps >= 2): head, then steps-1 fused
  // steps (each applies the previous combine inside its RHS kernel), then
  // the last combine alone — one kernel fewer per step.
  void run(int steps) {
    if (steps <= 0) return;
    // kernels per solve: RHS + x-sweep + y-sweep (+ transpose/correct when
    // the y-sweep cannot read the x output transposed). Captured launches
    // are not counted, so count what one graph replays.
    if (solveK < 0) {
      const uint64_t before = g_launches.load();
      cudaGraph_t g;
      SG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      enqueue_solve(ic, ip, -1, stream);
      SG_CUDA(cudaStreamEndCapture(stream, &g));
      SG_CUDA(cudaGraphDestroy(g));
      solveK = static_cast<int>(g_launches.load() - before);
      g_launches.store(before);
    }
    if (steps == 1 || !steady_ok()) {
      for (int k = 0; k < steps; ++k) {
        launch(0, solveK + 1);
        std::swap(ic, ip);  // C^{n+1} was written over C^{n-1}
        ++step;
      }
      return;
    }
    launch(1, solveK);
    int left = steps - 1;
    while (left >= 12) {  // one graph launch per 12 steps
      launch(5, 12 * solveK);
      left -= 12;
    }
    while (left >= 3) {
      launch(3, 3 * solveK);
      left -= 3;  // three rotations of (ic, ip, spare) restore it
    }
    for (; left > 0; --left) {
      launch(2, solveK);
      const int n = spare();
      ip = ic;
      ic = n;
    }
    launch(4, 1);
    std::swap(ic, ip);
    step += steps;
  }
};

// ------------------------------------------------------------------------
// Distributed CH (one process per GPU, y-slabs). The host orchestrates:
//   halo exchange (2 rows of C^n, C^{n-1}) -> phase_x -> all-to-all ->
//   phase_y -> all-to-all -> combine
// (paper_1902_09931_b200/ch_dist.py). Each phase is the single-GPU step's
// arithmetic on the rank's share, so results are bitwise identical for
// every world size.
struct ChDist {
  sg_ch_params p{};
  int world = 1, rank = 0, own = 0, nxq = 0, r0 = 0;
  int device = 0;
  DevicePenta fx, fy;
  RhsParams rp{};
  double *rhsT = nullptr, *y4x = nullptr, *ybuf = nullptr;
  // P2P path (the all-to-alls fused into the sweeps' final stores): local
  // scratch + the four buffers the peers write into
  double *xloc = nullptr, *ycol = nullptr, *recvX = nullptr, *recvY = nullptr, *y4xAll = nullptr,
         *y4yAll = nullptr;
  SweepPeers px, py;  // destinations of the x- and y-sweep results
  bool p2p = false;
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;

  void alloc_p2p() {
    if (recvX) return;
    const size_t slab = static_cast<size_t>(own) * p.nx;
    xloc = dalloc(slab);
    ycol = dalloc(static_cast<size_t>(p.ny) * nxq);
    recvX = dalloc(slab);
    recvY = dalloc(slab);
    y4xAll = dalloc(4 * static_cast<size_t>(p.ny));
    y4yAll = dalloc(4 * static_cast<size_t>(p.nx));
  }

  // Peer buffers in rank order (device pointers valid in this process:
  // IPC-mapped peer memory, or other simulated ranks' buffers). Returns
  // whether the P2P path can run (tile/box divisibility, alignment, TMA).
  bool set_peers(double* const* rx, double* const* ry, double* const* y4xa, double* const* y4ya) {
    if (world > 8 || p.nx % 64) return false;
    px = SweepPeers{};
    py = SweepPeers{};
    px.npeer = py.npeer = world;
    px.prow = nxq;  // x-sweep unknowns i -> the rank owning column block i / nxq
    py.prow = own;  // y-sweep unknowns j -> the rank owning row block j / own
    for (int d = 0; d < world; ++d) {
      px.dst[d] = rx[d] + static_cast<size_t>(rank) * nxq * own;  // my block [i_local][jl]
      px.y4[d] = y4xa[d];
      py.dst[d] = ry[d] + static_cast<size_t>(rank) * own * nxq;  // my block [jl][i_local]
      py.y4[d] = y4ya[d];
    }
    px.y4Stride = p.ny;
    px.y4Off = rank * own;
    py.y4Stride = p.nx;
    py.y4Off = rank * nxq;
    const double* wx[4];
    for (int k = 0; k < 4; ++k) wx[k] = fx.t.W[k] + static_cast<size_t>(rank) * nxq;
    p2p = penta_sweep_xin(fx.t, own, p.nx, xloc, rhsT, nullptr, nullptr, y4x, stream, false, false, 0, &px) &&
          penta_sweep_xin(fy.t, nxq, p.ny, ycol, recvX, wx, y4xAll, ybuf, stream, false, false, own, &py);
    // Runtime self-check: a TMA tensor store into every peer's receive
    // buffers (the exact mechanism the sweeps use), read back through the
    // mapping. A transport that maps but does not carry TMA stores (or a
    // stale/broken mapping) leaves the caller on the collective form.
    for (int d = 0; p2p && d < world; ++d)
      p2p = peer_tma_probe(rx[d] + static_cast<size_t>(rank) * nxq * own, 0x5a00u + 16u * rank + d, stream) &&
            peer_tma_probe(ry[d] + static_cast<size_t>(rank) * own * nxq, 0x6b00u + 16u * rank + d, stream);
    return p2p;
  }

  void phase_x_p2p(const double* cur, const double* prev, cudaStream_t s) {
    const RhsGeom geom{p.nx, own, own + 2 * HALO, HALO, 0, 1};  // row-major RHS
    launch_rhs(p.nonlinearEnabled, cur, prev, rhsT, geom, rp, s);
    if (!penta_sweep_xin(fx.t, own, p.nx, xloc, rhsT, nullptr, nullptr, y4x, s, false, true, 0, &px))
      throw Error(SG_ERR_CUDA, "internal: P2P x-sweep unavailable");
  }

  void phase_y_p2p(cudaStream_t s) {
    const double* wx[4];
    for (int k = 0; k < 4; ++k) wx[k] = fx.t.W[k] + static_cast<size_t>(rank) * nxq;
    if (!penta_sweep_xin(fy.t, nxq, p.ny, ycol, recvX, wx, y4xAll, ybuf, s, false, true, own, &py))
      throw Error(SG_ERR_CUDA, "internal: P2P y-sweep unavailable");
  }

  void combine_p2p(const double* cur, double* prev, double* peerUp, double* peerDn, cudaStream_t s) {
    CorrTables ty{{fy.t.W[0], fy.t.W[1], fy.t.W[2], fy.t.W[3]}, y4yAll};
    k_combine_packed_corr<<<dim3((p.nx + 255) / 256, own), 256, 0, s>>>(cur, prev, recvY, p.nx, own, nxq, r0, ty,
                                                                        peerUp, peerDn);
    check_launch("ch slab combine (P2P) kernel");
  }

  double* dalloc(size_t n) {
    void* q = nullptr;
    SG_CUDA(cudaMalloc(&q, n * sizeof(double)));
    allocs.push_back(q);
    return static_cast<double*>(q);
  }
  ~ChDist() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* q : allocs) cudaFree(q);
    if (stream) cudaStreamDestroy(stream);
  }
  void build_factor(DevicePenta& f, double sigma, int n) {
    double* bands = dalloc(5 * static_cast<size_t>(n));
    k_fill_bands<<<(n + 255) / 256, 256, 0, stream>>>(sigma, n, bands, bands + n, bands + 2 * n, bands + 3 * n,
                                                      bands + 4 * n);
    check_launch("ch bands kernel");
    f.build(1, n, true, true, bands, bands + n, bands + 2 * n, bands + 3 * n, bands + 4 * n, stream);
  }
  void init() {
    SG_CUDA(cudaGetDevice(&device));
    // a BLOCKING stream: ordered after work the caller queued on the legacy
    // default stream (e.g. torch kernels producing device inputs)
    SG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamDefault));
    own = p.ny / world;
    nxq = p.nx / world;
    r0 = rank * own;
    rhsT = dalloc(static_cast<size_t>(own) * p.nx);
    y4x = dalloc(4 * static_cast<size_t>(own));
    ybuf = dalloc(4 * static_cast<size_t>(nxq));
    const double dx = p.lx / p.nx, dy = p.ly / p.ny;
    build_factor(fx, kTwoThirds * p.D * p.gamma * p.dt / pow4(dx), p.nx);
    build_factor(fy, kTwoThirds * p.D * p.gamma * p.dt / pow4(dy), p.ny);
    rp.kDiff = -kTwoThirds;
    rp.kBih = kTwoThirds * p.D * p.gamma * p.dt;
    rp.kNl = kTwoThirds * p.D * p.dt;
    biharmonic_weights(dx, dy, rp.bw);
    const double cx = 1.0 / (dx * dx), cy = 1.0 / (dy * dy), cc = -2.0 * cx - 2.0 * cy;
    const double nl[9] = {0.0, cy, 0.0, cx, cc, cx, 0.0, cy, 0.0};
    std::memcpy(rp.nl, nl, sizeof nl);
    SG_CUDA(cudaStreamSynchronize(stream));
  }
};

// CHStepper(params, numTiles, numWorkers) with numWorkers = G > 1: the
// distributed step (config 5's y-slabs) driven from ONE process over G GPUs
// (worker w on device w % visible GPUs), each rank a ChDist with its own
// stream. The P2P form stores the all-to-all blocks and halo rows straight
// into the peers' buffers (cudaDeviceEnablePeerAccess, no IPC); the
// barriers between phases are cross-device event joins. When the P2P
// geometry does not fit, the copy-engine form runs: halos and the two
// all-to-alls as cudaMemcpyPeerAsync blocks (the layout all_to_all_single
// produces). Bitwise identical to the one-GPU stepper (same kernels).
struct ChMulti {
  sg_ch_params p{};
  struct Rank {
    std::unique_ptr<ChDist> d;
    double* ext[2] = {nullptr, nullptr};  // time levels, (own + 4) x nx
    double *send = nullptr, *ycol = nullptr, *recv = nullptr;  // copy-engine form
    cudaEvent_t ev = nullptr;
  };
  std::vector<Rank> ranks;
  int G = 1;
  bool p2p = false;
  bool halosValid = false;
  int ic = 0;  // ext index of C^n
  int step = 0;
  double* gathered[2] = {nullptr, nullptr};  // full fields on rank 0's device (lazy)

  static int workers_for(const sg_ch_params& q, int numWorkers) {
    int ndev = 1;
    SG_CUDA(cudaGetDeviceCount(&ndev));
    int g = sg_get_device_map() == 1 ? numWorkers : std::min(numWorkers, ndev);
    // nx, ny are powers of two: the largest power of two <= g with >= 2 rows
    // per slab
    int h = 1;
    while (2 * h <= g && q.ny / (2 * h) >= 2 && q.nx % (2 * h) == 0) h *= 2;
    return h;
  }

  void init(int g) {
    G = g;
    int ndev = 1;
    SG_CUDA(cudaGetDeviceCount(&ndev));
    ranks.resize(G);
    for (int r = 0; r < G; ++r) {
      SG_CUDA(cudaSetDevice(r % ndev));
      auto& R = ranks[r];
      R.d = std::make_unique<ChDist>();
      R.d->p = p;
      R.d->world = G;
      R.d->rank = r;
      R.d->init();
      const size_t ext = static_cast<size_t>(R.d->own + 2 * HALO) * p.nx;
      R.ext[0] = R.d->dalloc(ext);
      R.ext[1] = R.d->dalloc(ext);
      SG_CUDA(cudaEventCreateWithFlags(&R.ev, cudaEventDisableTiming));
      k_init_slab_launch(p.seed, p.icAmplitude, p.nx, R.d->own, R.d->r0, R.ext[0], R.d->stream);
      SG_CUDA(cudaMemcpyAsync(R.ext[1], R.ext[0], ext * sizeof(double), cudaMemcpyDeviceToDevice, R.d->stream));
    }
    const int used = std::min(G, ndev);
    for (int a = 0; a < used; ++a)
      for (int b = 0; b < used; ++b) {
        int can = 0;
        if (a == b || cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) continue;
        cudaSetDevice(a);
        if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
      }
    // P2P wiring: every rank's receive buffers, in rank order
    std::vector<double*> rx(G), ry(G), yx(G), yy(G);
    for (int r = 0; r < G; ++r) {
      SG_CUDA(cudaSetDevice(ranks[r].d->device));
      ranks[r].d->alloc_p2p();
      rx[r] = ranks[r].d->recvX;
      ry[r] = ranks[r].d->recvY;
      yx[r] = ranks[r].d->y4xAll;
      yy[r] = ranks[r].d->y4yAll;
    }
    sync_all();
    p2p = rhs_kind() != 0;
    for (int r = 0; p2p && r < G; ++r) {
      SG_CUDA(cudaSetDevice(ranks[r].d->device));
      p2p = ranks[r].d->set_peers(rx.data(), ry.data(), yx.data(), yy.data());
    }
    if (!p2p)
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        const size_t slab = static_cast<size_t>(R.d->own) * p.nx;
        R.send = R.d->dalloc(slab);
        R.ycol = R.d->dalloc(static_cast<size_t>(p.ny) * R.d->nxq);
        R.recv = R.d->dalloc(slab);
      }
    halosValid = false;
    sync_all();
  }

  // every rank's stream waits for every rank's work so far
  void barrier() {
    for (auto& R : ranks) {
      SG_CUDA(cudaSetDevice(R.d->device));
      SG_CUDA(cudaEventRecord(R.ev, R.d->stream));
    }
    for (auto& R : ranks) {
      SG_CUDA(cudaSetDevice(R.d->device));
      for (auto& Q : ranks)
        if (&Q != &R) SG_CUDA(cudaStreamWaitEvent(R.d->stream, Q.ev, 0));
    }
  }

  void sync_all() {
    for (auto& R : ranks) {
      SG_CUDA(cudaSetDevice(R.d->device));
      SG_CUDA(cudaStreamSynchronize(R.d->stream));
    }
  }

  // 2 halo rows each way of time level k from the ring neighbours' own rows
  void exchange_halos(int k) {
    const size_t rowB = static_cast<size_t>(p.nx) * sizeof(double);
    for (int r = 0; r < G; ++r) {
      auto& R = ranks[r];
      const auto& U = ranks[(r + G - 1) % G];
      const auto& D = ranks[(r + 1) % G];
      SG_CUDA(cudaSetDevice(R.d->device));
      const int own = R.d->own;
      SG_CUDA(cudaMemcpyPeerAsync(R.ext[k], R.d->device, U.ext[k] + static_cast<size_t>(U.d->own) * p.nx,
                                  U.d->device, HALO * rowB, R.d->stream));
      SG_CUDA(cudaMemcpyPeerAsync(R.ext[k] + static_cast<size_t>(own + HALO) * p.nx, R.d->device,
                                  D.ext[k] + static_cast<size_t>(HALO) * p.nx, D.d->device, HALO * rowB,
                                  R.d->stream));
    }
  }

  // all-to-all of packed blocks (own x nxq): dst_q block r <- src_r block q
  void alltoall(double* Rank::*src, double* Rank::*dst) {
    const size_t blk = static_cast<size_t>(ranks[0].d->own) * ranks[0].d->nxq;
    for (int q = 0; q < G; ++q) {
      auto& Q = ranks[q];
      SG_CUDA(cudaSetDevice(Q.d->device));
      for (int r = 0; r < G; ++r) {
        const auto& R = ranks[r];
        SG_CUDA(cudaMemcpyPeerAsync(Q.*dst + r * blk, Q.d->device, R.*src + q * blk, R.d->device,
                                    blk * sizeof(double), Q.d->stream));
      }
    }
  }

  void one_step() {
    const int ip = 1 - ic;
    if (p2p) {
      if (!halosValid) {
        exchange_halos(ic);
        exchange_halos(ip);
        barrier();
        halosValid = true;
      }
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        R.d->phase_x_p2p(R.ext[ic], R.ext[ip], R.d->stream);
      }
      barrier();
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        R.d->phase_y_p2p(R.d->stream);
      }
      barrier();
      for (int r = 0; r < G; ++r) {
        auto& R = ranks[r];
        SG_CUDA(cudaSetDevice(R.d->device));
        // C^{n+1} over C^{n-1}; its first / last two rows also land in the
        // up / down neighbours' halo rows of that level
        R.d->combine_p2p(R.ext[ic], R.ext[ip], ranks[(r + G - 1) % G].ext[ip], ranks[(r + 1) % G].ext[ip],
                         R.d->stream);
      }
      barrier();
    } else {
      exchange_halos(ic);
      exchange_halos(ip);
      barrier();
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        ch_phase_x(p, R.d->rp, R.d->fx.t, R.d->own, R.d->nxq, R.ext[ic], R.ext[ip], R.d->rhsT, R.d->y4x, R.send,
                   R.d->stream);
      }
      barrier();
      alltoall(&Rank::send, &Rank::ycol);
      barrier();
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        penta_sweep(R.d->fy.t, R.d->nxq, p.ny, R.ycol, R.d->ybuf, true, false, R.d->stream);
      }
      barrier();
      alltoall(&Rank::ycol, &Rank::recv);
      barrier();
      for (auto& R : ranks) {
        SG_CUDA(cudaSetDevice(R.d->device));
        ch_combine_packed(p.nx, R.d->own, R.d->nxq, R.ext[ic], R.ext[ip], R.recv, R.d->stream);
      }
      barrier();
    }
    ic = ip;
    ++step;
  }

  void run(int steps) {
    for (int k = 0; k < steps; ++k) one_step();
  }

  // rows of C^n (which 0) / C^{n-1} (which 1) into a full row-major field
  // (host or device memory; cudaMemcpyDefault resolves either)
  void gather_into(int which, double* out) {
    const int k = which == 0 ? ic : 1 - ic;
    const size_t rowB = static_cast<size_t>(p.nx) * sizeof(double);
    for (auto& R : ranks) {
      SG_CUDA(cudaSetDevice(R.d->device));
      SG_CUDA(cudaMemcpyAsync(out + static_cast<size_t>(R.d->r0) * p.nx, R.ext[k] + HALO * p.nx,
                              R.d->own * rowB, cudaMemcpyDefault, R.d->stream));
    }
    sync_all();
  }

  double* device_field(int which) {
    auto& R0 = ranks[0];
    SG_CUDA(cudaSetDevice(R0.d->device));
    if (!gathered[which]) gathered[which] = R0.d->dalloc(static_cast<size_t>(p.nx) * p.ny);
    gather_into(which, gathered[which]);
    return gathered[which];
  }

  void set_state(const double* curr, const double* prev) {
    sync_all();
    const size_t rowB = static_cast<size_t>(p.nx) * sizeof(double);
    ic = 0;
    for (auto& R : ranks) {
      SG_CUDA(cudaSetDevice(R.d->device));
      for (int k = 0; k < 2; ++k) {
        const double* src = k == 0 ? curr : prev;
        SG_CUDA(cudaMemcpyAsync(R.ext[k] + HALO * p.nx, src + static_cast<size_t>(R.d->r0) * p.nx,
                                R.d->own * rowB, cudaMemcpyDefault, R.d->stream));
      }
    }
    barrier();
    halosValid = false;
    if (!p2p) return;
    exchange_halos(0);
    exchange_halos(1);
    barrier();
    halosValid = true;
    sync_all();
  }

  ~ChMulti() {
    for (auto& R : ranks) {
      if (!R.d) continue;
      cudaSetDevice(R.d->device);
      if (R.d->stream) cudaStreamSynchronize(R.d->stream);
      if (R.ev) cudaEventDestroy(R.ev);
    }
  }
};

}  // namespace sg

struct sg_chd_s {
  std::unique_ptr<sg::ChDist> d;
};

struct sg_ch_s {
  std::unique_ptr<sg::ChState> st;   // one GPU
  std::unique_ptr<sg::ChMulti> mul;  // numWorkers -> GPUs
};

struct sg_penta_s {
  std::unique_ptr<sg::DevicePenta> f;
  int device = 0;
  cudaStream_t stream = nullptr;
  // solve scratch, allocated once (per-call stream-ordered allocations cost
  // milliseconds once the pool has released them)
  double* y4 = nullptr;   // periodic: y = K^{-1} V^T z, 4 x B
  double* tmp = nullptr;  // host-memory solves: device copy of the rhs
  // Solves on one factor share the scratch: the mutex guards its lazy
  // allocation and the enqueue, `last` orders a solve after the previous
  // one even on another stream (concurrent solves on one factor serialise;
  // the reference's solve_in_place is const but its scratch is per call).
  std::mutex mu;
  cudaEvent_t last = nullptr;
  ~sg_penta_s() {
    if (last) cudaEventDestroy(last);
    if (y4) cudaFree(y4);
    if (tmp) cudaFree(tmp);
  }
};

// Reuse the error plumbing of capi.cu through these two helpers.
extern "C" sg_status sg_internal_set_error(const char* msg, int system);

namespace {
template <typename F>
sg_status guard2(F&& f) {
  try {
    f();
    return SG_OK;
  } catch (const sg::Error& e) {
    sg_internal_set_error(e.what(), e.system);
    return e.status;
  } catch (const std::exception& e) {
    sg_internal_set_error(e.what(), -1);
    return SG_ERR_CUDA;
  }
}

void require_device2() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw sg::Error(SG_ERR_NO_DEVICE, "stengrid: no CUDA device visible (there is no CPU fallback)");
}
}  // namespace

extern "C" {

void sg_ch_default_params(sg_ch_params* p) {
  p->D = 1.0;
  p->gamma = 0.01;
  p->nx = 512;
  p->ny = 512;
  p->lx = 2.0 * 3.14159265358979323846;
  p->ly = 2.0 * 3.14159265358979323846;
  p->dt = 0.0;
  p->T = 0.0;
  p->seed = 1;
  p->icAmplitude = 0.1;
  p->nonlinearEnabled = 1;
}

sg_status sg_ch_validate(const sg_ch_params* p) {
  return guard2([&] {
    if (!p) sg::invalid("CHParams: null");
    sg::ch_validate(*p);
  });
}

sg_status sg_ch_create(const sg_ch_params* p, int numTiles, int numWorkers, sg_ch_t* ch) {
  return guard2([&] {
    if (!p || !ch) sg::invalid("CHStepper: null argument");
    *ch = nullptr;
    sg::ch_validate(*p);
    // rowTiles_ = make_tiles(ny, numTiles) (cahn_hilliard.cpp:216); pool_(numWorkers)
    if (numTiles < 1 || numTiles > p->ny) sg::invalid("make_tiles: numTiles must satisfy 1 <= numTiles <= ny");
    if (numWorkers < 1) sg::invalid("WorkerPool: workers must be >= 1");
    require_device2();
    auto h = std::make_unique<sg_ch_s>();
    // numWorkers -> GPUs: G > 1 runs config 5's distributed step
    // over G devices from this process; G = 1 keeps the fused one-GPU step
    const int G = sg::ChMulti::workers_for(*p, numWorkers);
    if (G > 1) {
      int dev = 0;
      SG_CUDA(cudaGetDevice(&dev));
      h->mul = std::make_unique<sg::ChMulti>();
      h->mul->p = *p;
      h->mul->init(G);
      SG_CUDA(cudaSetDevice(dev));
    } else {
      h->st = std::make_unique<sg::ChState>();
      h->st->p = *p;
      h->st->init();
    }
    *ch = h.release();
  });
}

sg_status sg_ch_step(sg_ch_t ch, int steps) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (ch->mul) {
      ch->mul->run(steps);
      return;
    }
    SG_CUDA(cudaSetDevice(ch->st->device));
    ch->st->run(steps);
  });
}

sg_status sg_ch_set_partition(sg_ch_t ch, int segments) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (segments < 0 || segments > 16) sg::invalid("CHStepper: partition segments must be in [0, 16]");
    if (ch->mul) sg::invalid("CHStepper: partitioned sweeps are single-GPU only");
    SG_CUDA(cudaSetDevice(ch->st->device));
    ch->st->set_partition(segments);
  });
}

sg_status sg_ch_set_state(sg_ch_t ch, const double* curr, const double* prev, sg_memory memory) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (ch->mul) {
      ch->mul->set_state(curr, prev);
      ch->mul->step = 0;  // cahn_hilliard.cpp:256-257
      return;
    }
    auto& s = *ch->st;
    SG_CUDA(cudaSetDevice(s.device));
    const size_t bytes = static_cast<size_t>(s.p.nx) * s.p.ny * sizeof(double);
    const cudaMemcpyKind k = memory == SG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    s.ic = 0;
    s.ip = 1;
    SG_CUDA(cudaMemcpyAsync(s.field[0], curr, bytes, k, s.stream));
    SG_CUDA(cudaMemcpyAsync(s.field[1], prev, bytes, k, s.stream));
    SG_CUDA(cudaStreamSynchronize(s.stream));
    s.step = 0;  // cahn_hilliard.cpp:256-257
  });
}

sg_status sg_ch_get_field(sg_ch_t ch, int which, double* out, sg_memory memory) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (ch->mul) {
      ch->mul->gather_into(which == 0 ? 0 : 1, out);
      return;
    }
    auto& s = *ch->st;
    SG_CUDA(cudaSetDevice(s.device));
    const size_t bytes = static_cast<size_t>(s.p.nx) * s.p.ny * sizeof(double);
    const double* src = which == 0 ? s.cur() : s.prev();
    SG_CUDA(cudaMemcpyAsync(out, src, bytes, memory == SG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            s.stream));
    SG_CUDA(cudaStreamSynchronize(s.stream));
  });
}

sg_status sg_ch_device_field(sg_ch_t ch, int which, const double** dptr) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (ch->mul) {  // a gathered copy on worker 0's GPU, valid until the next call
      *dptr = ch->mul->device_field(which == 0 ? 0 : 1);
      return;
    }
    auto& s = *ch->st;
    SG_CUDA(cudaStreamSynchronize(s.stream));
    *dptr = which == 0 ? s.cur() : s.prev();
  });
}

sg_status sg_ch_status(sg_ch_t ch, int* step, double* time) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    const int k = ch->mul ? ch->mul->step : ch->st->step;
    const double dt = ch->mul ? ch->mul->p.dt : ch->st->p.dt;
    if (step) *step = k;
    if (time) *time = static_cast<double>(k) * dt;  // cahn_hilliard.cpp:327
  });
}

sg_status sg_ch_diagnostics(sg_ch_t ch, double* t, double* s, double* k1Inv) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    const sg_ch_params& P = ch->mul ? ch->mul->p : ch->st->p;
    const int k = ch->mul ? ch->mul->step : ch->st->step;
    const double* f = nullptr;
    cudaStream_t stream = nullptr;
    if (ch->mul) {  // gathered onto worker 0's GPU
      f = ch->mul->device_field(0);
      stream = ch->mul->ranks[0].d->stream;
      SG_CUDA(cudaSetDevice(ch->mul->ranks[0].d->device));
    } else {
      SG_CUDA(cudaSetDevice(ch->st->device));
      // queued behind the pending steps on the stepper's own stream
      f = ch->st->cur();
      stream = ch->st->stream;
    }
    const double dx = P.lx / P.nx, dy = P.ly / P.ny;
    if (t) *t = static_cast<double>(k) * P.dt;
    double r[3];  // <C^2>, k1 num, k1 den
    sg::device_ch_diagnostics(f, P.nx, P.ny, dx, dy, r, stream);
    const double m2 = r[0];
    if (m2 >= 1.0 - 1e-12) throw sg::Error(SG_ERR_DOMAIN, "s_metric: mixture saturated, <C^2> reached 1");
    if (s) *s = 1.0 / (1.0 - m2);
    // an identically zero field has no spectral length scale: 1/k1 := 0
    // (k1_metric's domain_error, caught as in CHStepper::diagnostics)
    if (k1Inv) *k1Inv = r[2] == 0.0 ? 0.0 : 1.0 / (r[1] / r[2]);
  });
}

sg_status sg_ch_synchronize(sg_ch_t ch) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (ch->mul) {
      ch->mul->sync_all();
      return;
    }
    SG_CUDA(cudaSetDevice(ch->st->device));
    SG_CUDA(cudaStreamSynchronize(ch->st->stream));
  });
}

sg_status sg_ch_workers(sg_ch_t ch, int* workers, int* p2p) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (workers) *workers = ch->mul ? ch->mul->G : 1;
    if (p2p) *p2p = ch->mul ? (ch->mul->p2p ? 1 : 0) : 0;
  });
}

sg_status sg_ch_set_step(sg_ch_t ch, int step) {
  return guard2([&] {
    if (!ch) sg::logic("CHStepper: destroyed");
    if (step < 0) sg::invalid("CHStepper: step must be >= 0");
    if (ch->mul)
      ch->mul->step = step;
    else
      ch->st->step = step;
  });
}

sg_status sg_ch_destroy(sg_ch_t* ch) {
  return guard2([&] {
    if (!ch || !*ch) return;
    delete *ch;
    *ch = nullptr;
  });
}

// ------------------------------------------------------------------ penta

sg_status sg_penta_create(int batchCount, int n, int periodic, const double* e, const double* c,
                          const double* d, const double* a, const double* b, sg_memory memory,
                          sg_penta_t* factor) {
  return guard2([&] {
    if (!factor) sg::invalid("penta: null handle");
    *factor = nullptr;
    if (batchCount < 1) sg::invalid("penta: batchCount must be >= 1");  // penta.cpp:10-13
    if (n < 5) sg::invalid("penta: systems need n >= 5");
    require_device2();
    auto h = std::make_unique<sg_penta_s>();
    SG_CUDA(cudaGetDevice(&h->device));
    // a BLOCKING stream: ordered after work the caller queued on the legacy
    // default stream (e.g. torch kernels producing device inputs)
    SG_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamDefault));
    h->f = std::make_unique<sg::DevicePenta>();
    const size_t len = static_cast<size_t>(batchCount) * n;
    const double* bands[5] = {e, c, d, a, b};
    // Uniform operator: every system identical (host bands are checked here;
    // device bands always take the per-system path).
    bool uniform = false;
    if (memory == SG_MEM_HOST) {
      uniform = true;
      for (int k = 0; k < 5 && uniform; ++k)
        for (int r = 0; r < n && uniform; ++r) {
          const double* row = bands[k] + static_cast<size_t>(r) * batchCount;
          for (int q = 1; q < batchCount; ++q)
            if (std::memcmp(&row[q], &row[0], sizeof(double)) != 0) {
              uniform = false;
              break;
            }
        }
    }
    const int nsys = uniform ? 1 : batchCount;
    const size_t dlen = static_cast<size_t>(nsys) * n;
    double* dev = h->f->alloc(5 * dlen);
    for (int k = 0; k < 5; ++k) {
      if (uniform) {
        std::vector<double> col(n);
        for (int r = 0; r < n; ++r) col[r] = bands[k][static_cast<size_t>(r) * batchCount];
        SG_CUDA(cudaMemcpy(dev + k * dlen, col.data(), n * sizeof(double), cudaMemcpyHostToDevice));
      } else {
        SG_CUDA(cudaMemcpy(dev + k * dlen, bands[k], len * sizeof(double),
                           memory == SG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
      }
    }
    h->f->build(nsys, n, periodic != 0, uniform, dev, dev + dlen, dev + 2 * dlen, dev + 3 * dlen,
                dev + 4 * dlen, h->stream);
    h->f->B = batchCount;
    *factor = h.release();
  });
}

sg_status sg_penta_solve(sg_penta_t f, double* rhs, sg_memory memory, void* stream, int synchronize) {
  return guard2([&] {
    if (!f) sg::logic("penta: destroyed factor");
    SG_CUDA(cudaSetDevice(f->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : f->stream;
    std::lock_guard<std::mutex> lk(f->mu);
    if (!f->last) SG_CUDA(cudaEventCreateWithFlags(&f->last, cudaEventDisableTiming));
    else SG_CUDA(cudaStreamWaitEvent(s, f->last, 0));
    const int B = f->f->B, n = f->f->n;
    const size_t bytes = static_cast<size_t>(B) * n * sizeof(double);
    double* z = rhs;
    if (memory == SG_MEM_HOST) {
      if (!f->tmp) SG_CUDA(cudaMalloc(reinterpret_cast<void**>(&f->tmp), bytes));
      SG_CUDA(cudaMemcpyAsync(f->tmp, rhs, bytes, cudaMemcpyHostToDevice, s));
      z = f->tmp;
    }
    if (f->f->periodic && !f->y4) SG_CUDA(cudaMalloc(reinterpret_cast<void**>(&f->y4), 4 * sizeof(double) * B));
    sg::penta_sweep(f->f->t, B, n, z, f->f->periodic ? f->y4 : nullptr, f->f->periodic, false, s);
    if (memory == SG_MEM_HOST) {
      SG_CUDA(cudaMemcpyAsync(rhs, f->tmp, bytes, cudaMemcpyDeviceToHost, s));
      synchronize = 1;
    }
    SG_CUDA(cudaEventRecord(f->last, s));
    if (synchronize) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_penta_destroy(sg_penta_t* f) {
  return guard2([&] {
    if (!f || !*f) return;
    cudaSetDevice((*f)->device);
    if ((*f)->stream) {
      cudaStreamSynchronize((*f)->stream);
      cudaStreamDestroy((*f)->stream);
    }
    delete *f;
    *f = nullptr;
  });
}

// ------------------------------------------------------- distributed CH

sg_status sg_chd_create(const sg_ch_params* p, int world, int rank, sg_chd_t* h) {
  return guard2([&] {
    if (!p || !h) sg::invalid("CH slab: null argument");
    *h = nullptr;
    sg::ch_validate(*p);
    if (world < 1 || rank < 0 || rank >= world) sg::invalid("CH slab: bad world/rank");
    if (p->ny % world != 0 || p->nx % world != 0)
      sg::invalid("CH slab: world size must divide nx and ny");
    if (p->ny / world < 2) sg::invalid("CH slab: each rank needs at least 2 rows");
    require_device2();
    auto o = std::make_unique<sg_chd_s>();
    o->d = std::make_unique<sg::ChDist>();
    o->d->p = *p;
    o->d->world = world;
    o->d->rank = rank;
    o->d->init();
    *h = o.release();
  });
}

sg_status sg_chd_geometry(sg_chd_t h, int* own, int* nxq, int* r0) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    if (own) *own = h->d->own;
    if (nxq) *nxq = h->d->nxq;
    if (r0) *r0 = h->d->r0;
  });
}

sg_status sg_chd_init(sg_chd_t h, double* currExt, double* prevExt, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    const int nx = d.p.nx;
    sg::k_init_slab_launch(d.p.seed, d.p.icAmplitude, nx, d.own, d.r0, currExt, s);
    const size_t rowB = static_cast<size_t>(nx) * sizeof(double);
    SG_CUDA(cudaMemcpyAsync(prevExt, currExt, rowB * (d.own + 4), cudaMemcpyDeviceToDevice, s));
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_phase_x(sg_chd_t h, const double* currExt, const double* prevExt, double* send, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    sg::ch_phase_x(d.p, d.rp, d.fx.t, d.own, d.nxq, currExt, prevExt, d.rhsT, d.y4x, send, s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_phase_y(sg_chd_t h, double* ycol, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    // nxq periodic systems of ny unknowns, interleaved; Woodbury in place
    sg::penta_sweep(d.fy.t, d.nxq, d.p.ny, ycol, d.ybuf, true, false, s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_combine(sg_chd_t h, const double* currExt, double* prevExt, const double* recv, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    sg::ch_combine_packed(d.p.nx, d.own, d.nxq, currExt, prevExt, recv, s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_p2p_buffers(sg_chd_t h, double** recvX, double** recvY, double** y4xAll, double** y4yAll) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    d.alloc_p2p();
    if (recvX) *recvX = d.recvX;
    if (recvY) *recvY = d.recvY;
    if (y4xAll) *y4xAll = d.y4xAll;
    if (y4yAll) *y4yAll = d.y4yAll;
  });
}

sg_status sg_chd_set_peers(sg_chd_t h, double* const* recvX, double* const* recvY, double* const* y4xAll,
                           double* const* y4yAll, int* enabled) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    if (!recvX || !recvY || !y4xAll || !y4yAll) sg::invalid("CH slab: null peer table");
    auto& d = *h->d;
    SG_CUDA(cudaSetDevice(d.device));
    d.alloc_p2p();
    const bool ok = sg::rhs_kind() != 0 && d.set_peers(recvX, recvY, y4xAll, y4yAll);
    if (enabled) *enabled = ok ? 1 : 0;
  });
}

sg_status sg_chd_phase_x_p2p(sg_chd_t h, const double* currExt, const double* prevExt, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    if (!d.p2p) sg::logic("CH slab: P2P path not enabled (sg_chd_set_peers)");
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    d.phase_x_p2p(currExt, prevExt, s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_phase_y_p2p(sg_chd_t h, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    if (!d.p2p) sg::logic("CH slab: P2P path not enabled (sg_chd_set_peers)");
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    d.phase_y_p2p(s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_chd_combine_p2p(sg_chd_t h, const double* currExt, double* prevExt, double* peerUpPrev,
                             double* peerDnPrev, void* stream) {
  return guard2([&] {
    if (!h) sg::logic("CH slab: destroyed");
    auto& d = *h->d;
    if (!d.p2p) sg::logic("CH slab: P2P path not enabled (sg_chd_set_peers)");
    SG_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    d.combine_p2p(currExt, prevExt, peerUpPrev, peerDnPrev, s);
    if (!stream) SG_CUDA(cudaStreamSynchronize(s));
  });
}

sg_status sg_ipc_get_handle(const void* devPtr, void* handle64, size_t* offset) {
  return guard2([&] {
    if (!devPtr || !handle64 || !offset) sg::invalid("ipc: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    // the handle names the whole allocation (e.g. a caching allocator's
    // segment): report where devPtr lies inside it
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<GetRange>(fn);
    }();
    if (!get_range) throw sg::Error(SG_ERR_CUDA, "ipc: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(devPtr)) != CUDA_SUCCESS)
      throw sg::Error(SG_ERR_CUDA, "ipc: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t hd;
    SG_CUDA(cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)));
    std::memcpy(handle64, &hd, sizeof hd);
    *offset = static_cast<size_t>(reinterpret_cast<CUdeviceptr>(devPtr) - base);
  });
}

sg_status sg_ipc_open_handle(const void* handle64, void** devPtr) {
  return guard2([&] {
    if (!devPtr || !handle64) sg::invalid("ipc: null argument");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle64, sizeof hd);
    SG_CUDA(cudaIpcOpenMemHandle(devPtr, hd, cudaIpcMemLazyEnablePeerAccess));
  });
}

sg_status sg_ipc_close(void* devPtr) {
  return guard2([&] {
    if (devPtr) SG_CUDA(cudaIpcCloseMemHandle(devPtr));
  });
}

sg_status sg_chd_destroy(sg_chd_t* h) {
  return guard2([&] {
    if (!h || !*h) return;
    delete *h;
    *h = nullptr;
  });
}

}  // extern "C"
