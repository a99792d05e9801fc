// weno.cu — WENO5 upwind advection on the device (the
// paper's "modified engine" example).
//
// Replaces weno_advect (weno.cpp:50-94): out = -(u dphi/dx + v dphi/dy) with
// fifth-order WENO derivatives from 7-point windows along x and y, upwind
// bias chosen per point from the sign of u / v, periodic wrap. The window
// arithmetic is weno_derivative_7 / weno_combine (weno.cpp:13-48) term for
// term, compiled without FMA contraction: bitwise identical to the reference.
//
// Kernel: 32 x 16 output tile per CTA; phi staged in shared memory with a
// 3-point halo on all sides (38 x 22), u and v read once per point.
#include <cuda_runtime.h>

#include "sg_internal.hpp"

namespace sg {
namespace {

constexpr double kWenoEps = 1e-6;  // weno.cpp:11
constexpr int WX = 32, WY = 16, WH = 3;

__device__ __forceinline__ double weno_combine(double v1, double v2, double v3, double v4, double v5) {
  const double c1 = v1 * (1.0 / 3.0) - v2 * (7.0 / 6.0) + v3 * (11.0 / 6.0);
  const double c2 = -v2 * (1.0 / 6.0) + v3 * (5.0 / 6.0) + v4 * (1.0 / 3.0);
  const double c3 = v3 * (1.0 / 3.0) + v4 * (5.0 / 6.0) - v5 * (1.0 / 6.0);
  const double d1 = v1 - 2.0 * v2 + v3;
  const double d2 = v2 - 2.0 * v3 + v4;
  const double d3 = v3 - 2.0 * v4 + v5;
  const double s1 = (13.0 / 12.0) * d1 * d1 + 0.25 * (v1 - 4.0 * v2 + 3.0 * v3) * (v1 - 4.0 * v2 + 3.0 * v3);
  const double s2 = (13.0 / 12.0) * d2 * d2 + 0.25 * (v2 - v4) * (v2 - v4);
  const double s3 = (13.0 / 12.0) * d3 * d3 + 0.25 * (3.0 * v3 - 4.0 * v4 + v5) * (3.0 * v3 - 4.0 * v4 + v5);
  const double a1 = 0.1 / ((kWenoEps + s1) * (kWenoEps + s1));
  const double a2 = 0.6 / ((kWenoEps + s2) * (kWenoEps + s2));
  const double a3 = 0.3 / ((kWenoEps + s3) * (kWenoEps + s3));
  return (a1 * c1 + a2 * c2 + a3 * c3) / (a1 + a2 + a3);
}

// weno_derivative_7: w(k) = phi(x + (k-3) h), left-biased iff velocity >= 0.
// Both biases combine the same six scaled differences d_k = (w(k+1) - w(k))
// * invH (left: d0..d4, right: d5..d1), so the side is a per-lane select of
// the five inputs and ONE weno_combine runs — no divergent second copy of
// its eight divisions where neighbouring lanes' velocities differ in sign.
template <typename W>
__device__ __forceinline__ double weno_d7(W w, double invH, bool left) {
  double d[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) d[k] = (w(k + 1) - w(k)) * invH;
  return weno_combine(left ? d[0] : d[5], left ? d[1] : d[4], left ? d[2] : d[3], left ? d[3] : d[2],
                      left ? d[4] : d[1]);
}

__device__ __forceinline__ int wrapi(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

// Six CTAs per SM (40 registers): 8192^2 52.1 -> 54.7 Gpts/s; eight (32
// registers, spills) 53.3.
#ifndef SG_WENO_MINB
#define SG_WENO_MINB 6
#endif
__global__ void __launch_bounds__(WX * 8, SG_WENO_MINB) k_weno(const double* __restrict__ phi, const double* __restrict__ u,
                                                 const double* __restrict__ v, double* __restrict__ out, int nx,
                                                 int ny, double invDx, double invDy) {
  __shared__ double t[WY + 2 * WH][WX + 2 * WH + 1];
  const int i0 = blockIdx.x * WX, j0 = blockIdx.y * WY;
  const int tid = threadIdx.y * WX + threadIdx.x;
  constexpr int TW = WX + 2 * WH, TH = WY + 2 * WH;
  for (int e = tid; e < TW * TH; e += WX * 8) {
    const int y = e / TW, x = e - y * TW;
    const int j = wrapi(j0 - WH + y, ny), i = wrapi(i0 - WH + x, nx);
    t[y][x] = __ldg(phi + static_cast<long long>(j) * nx + i);
  }
  __syncthreads();
  const int x = threadIdx.x;
#pragma unroll
  for (int k = 0; k < WY / 8; ++k) {
    const int y = threadIdx.y + 8 * k;
    const int i = i0 + x, j = j0 + y;
    if (i >= nx || j >= ny) continue;
    const long long idx = static_cast<long long>(j) * nx + i;
    const double ui = u[idx], vi = v[idx];
    // upwind_side (weno.hpp:15-17): left-biased for velocity >= 0
    const double dpx = weno_d7([&](int q) { return t[y + WH][x + q]; }, invDx, !(ui < 0.0));
    const double dpy = weno_d7([&](int q) { return t[y + q][x + WH]; }, invDy, !(vi < 0.0));
    out[idx] = -(ui * dpx + vi * dpy);  // weno.cpp:89
  }
}

}  // namespace

void launch_weno(const double* phi, const double* u, const double* v, double* out, int nx, int ny, double dx,
                 double dy, cudaStream_t s) {
  const double invDx = 1.0 / dx, invDy = 1.0 / dy;  // weno.cpp:57-58
  k_weno<<<dim3((nx + WX - 1) / WX, (ny + WY - 1) / WY), dim3(WX, 8), 0, s>>>(phi, u, v, out, nx, ny, invDx, invDy);
  check_launch("weno kernel");
}

}  // namespace sg
