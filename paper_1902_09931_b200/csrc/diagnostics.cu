// diagnostics.cu — Cahn-Hilliard diagnostics on the device.
//
// Replaces simpson_mean / s_metric / k1_metric (cahn_hilliard.cpp:161-211)
// and CHStepper::diagnostics (:330-340), so a run() with a diagnostics sink
// no longer downloads the field.
//
//  * simpson_mean / s_metric: bitwise identical to the reference. One thread
//    per row accumulates rowAcc = sum_i wx_i * v_ij in the reference's order
//    (rows staged through shared-memory tiles so loads stay coalesced), then
//    one thread folds total += wy_j * rowAcc_j in row order.
//  * k1_metric: 2D FFT by cuFFT (real-to-complex D2Z, forward, unnormalized
//    like fft_2d, fft.cpp:54-61; the half spectrum with Hermitian weights)
//    and a deterministic two-level reduction of
//    num = sum |C_k|^2, den = sum |C_k|^2 / |k| over k != 0. The reference's
//    radix-2 FFT and serial sums round differently: agreement is to ~1e-13
//    relative (tests use 1e-10), which is well inside the reference's own
//    KAT tolerances (test_cahn_hilliard.cpp:346-366: 1e-12 absolute on O(1)).
#include <cuda_runtime.h>
#include <cufft.h>

#include <map>
#include <tuple>

#include <cmath>
#include <string>

#include "sg_internal.hpp"

namespace sg {
namespace {

constexpr int DT = 32;

// rowAcc[j] = sum_i (i odd ? 4 : 2) * f(v_ij), f = identity or square,
// accumulated left to right (cahn_hilliard.cpp:166-172, 179-185). One warp
// per 32 rows; 32-column chunks stream into a 5-stage shared-memory ring
// with 8 B cp.async (each lane one column of 32 rows: coalesced 256 B row
// segments, transposed on the way, no registers held), four chunks ahead of
// the per-row dependent add chain — the bitwise order admits no other.
// (Loading each chunk when needed: 112 us for 1024^2; two chunks ahead in
// registers: 37 us.)
constexpr int SR_ST = 5;
template <bool SQUARE>
__global__ void __launch_bounds__(DT) k_simpson_rows(const double* __restrict__ v, int nx, int ny,
                                                      double* __restrict__ rowAcc) {
  __shared__ double ring[SR_ST][DT][DT + 1];
  const int j0 = blockIdx.x * DT;
  const int lane = threadIdx.x;
  const int nChunks = (nx + DT - 1) / DT;
  auto issue = [&](int c) {
    if (c < nChunks) {
      double(*t)[DT + 1] = ring[c % SR_ST];
      const int i = c * DT + lane;
      for (int r = 0; r < DT; ++r) {
        const int j = j0 + r;
        if (j < ny && i < nx) {
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&t[r][lane]));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                       "l"(v + static_cast<long long>(j) * nx + i)
                       : "memory");
        } else {
          t[r][lane] = 0.0;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int c = 0; c < SR_ST - 1; ++c) issue(c);
  double acc = 0.0;
  for (int c = 0; c < nChunks; ++c) {
    issue(c + SR_ST - 1);  // its slot held chunk c - 1, released by the last __syncwarp
    asm volatile("cp.async.wait_group %0;" ::"n"(SR_ST - 1) : "memory");
    __syncwarp();  // every lane's copies of chunk c have landed
    const double(*t)[DT + 1] = ring[c % SR_ST];
    const int i0 = c * DT, lim = min(DT, nx - i0);
    if (lim == DT) {  // unrolled: the loads and products run ahead of the add chain
#pragma unroll
      for (int q = 0; q < DT; ++q) {
        const double wx = (q % 2 == 1) ? 4.0 : 2.0;  // i0 is even
        const double x = t[lane][q];
        acc += wx * (SQUARE ? x * x : x);
      }
    } else {
      for (int q = 0; q < lim; ++q) {
        const int i = i0 + q;
        const double wx = (i % 2 == 1) ? 4.0 : 2.0;
        const double x = t[lane][q];
        acc += wx * (SQUARE ? x * x : x);
      }
    }
    __syncwarp();
  }
  if (j0 + lane < ny) rowAcc[j0 + lane] = acc;
}

// total = sum_j wy_j * rowAcc_j in row order (cahn_hilliard.cpp:165-176):
// the block stages rowAcc through shared memory (coalesced, in flight
// together), thread 0 folds it in order.
constexpr int TT = 1024, TCH = 4096;
__global__ void __launch_bounds__(TT) k_simpson_total(const double* __restrict__ rowAcc, int nx, int ny, double* out) {
  __shared__ double sa[TCH];
  double total = 0.0;
  for (int j0 = 0; j0 < ny; j0 += TCH) {
    const int m = min(TCH, ny - j0);
    for (int k = threadIdx.x; k < m; k += TT) sa[k] = rowAcc[j0 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
      int k = 0;
      for (; k + 8 <= m; k += 8) {  // j0 + k even: the weights of a group are fixed
#pragma unroll
        for (int u = 0; u < 8; ++u) total += ((u % 2 == 1) ? 4.0 : 2.0) * sa[k + u];
      }
      for (; k < m; ++k) {
        const int j = j0 + k;
        const double wy = (j % 2 == 1) ? 4.0 : 2.0;
        total += wy * sa[k];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = total / (9.0 * static_cast<double>(nx) * static_cast<double>(ny));
}


constexpr int RB = 256;

// Per-block partial sums of |C|^2 and |C|^2/|k| (k1_metric, cahn_hilliard.cpp:
// 196-208) over the half spectrum of the real-to-complex transform
// (ny x (nx/2 + 1)): a real field's spectrum is Hermitian, |C(-k)| = |C(k)|,
// so interior columns stand for themselves and their mirror (weight 2).
__global__ void __launch_bounds__(RB) k_k1_partial(const cufftDoubleComplex* __restrict__ s, int nx, int ny,
                                                   double kxScale, double kyScale, double* __restrict__ part) {
  __shared__ double sn[RB], sd[RB];
  const int nh = nx / 2 + 1;
  const long long n = static_cast<long long>(nh) * ny;
  double num = 0.0, den = 0.0;
  for (long long k = static_cast<long long>(blockIdx.x) * RB + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * RB) {
    const int j = static_cast<int>(k / nh), i = static_cast<int>(k % nh);
    if (i == 0 && j == 0) continue;
    const int mj = (j < ny / 2) ? j : j - ny;
    const cufftDoubleComplex z = s[k];
    const double w = (i == 0 || 2 * i == nx) ? 1.0 : 2.0;
    const double power = z.x * z.x + z.y * z.y;  // std::norm
    const double kmag = hypot(kxScale * i, kyScale * mj);
    num += w * power;
    den += w * (power / kmag);
  }
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (int w = RB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sn[threadIdx.x] += sn[threadIdx.x + w];
      sd[threadIdx.x] += sd[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sn[0];
    part[2 * blockIdx.x + 1] = sd[0];
  }
}

// Partials staged through shared memory, then folded in block order by one
// thread (nb <= 2048 partials).
__global__ void __launch_bounds__(256) k_k1_final(const double* __restrict__ part, int nb, double* out) {
  __shared__ double sp[2 * 2048];
  for (int k = threadIdx.x; k < 2 * nb; k += 256) sp[k] = part[k];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double num = 0.0, den = 0.0;
  int b = 0;
  for (; b + 8 <= nb; b += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      num += sp[2 * (b + u)];
      den += sp[2 * (b + u) + 1];
    }
  }
  for (; b < nb; ++b) {
    num += sp[2 * b];
    den += sp[2 * b + 1];
  }
  out[0] = num;
  out[1] = den;
}

}  // namespace

// Mean by composite Simpson (square: of v^2), on the device; result in *out (host).
void device_simpson(const double* v, int nx, int ny, bool square, double* out, cudaStream_t s) {
  if (nx % 2 != 0 || ny % 2 != 0) invalid("simpson_mean: nx and ny must be even");
  double* buf = nullptr;
  retain_async_pool();
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(double) * (ny + 1), s));
  if (square)
    k_simpson_rows<true><<<(ny + DT - 1) / DT, DT, 0, s>>>(v, nx, ny, buf);
  else
    k_simpson_rows<false><<<(ny + DT - 1) / DT, DT, 0, s>>>(v, nx, ny, buf);
  check_launch("simpson rows kernel");
  k_simpson_total<<<1, TT, 0, s>>>(buf, nx, ny, buf + ny);
  check_launch("simpson total kernel");
  SG_CUDA(cudaMemcpyAsync(out, buf + ny, sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaFreeAsync(buf, s));
  SG_CUDA(cudaStreamSynchronize(s));
}

// cuFFT plans are created once per (thread, device, grid) and kept
// (creating one costs more than the transform at the diagnostics cadence).
// Per thread: a plan's work area must not be shared by concurrent calls.
cufftHandle cached_plan(int nx, int ny) {
  struct Cache {
    std::map<std::tuple<int, int, int>, cufftHandle> plans;
    ~Cache() {
      for (auto& kv : plans) cufftDestroy(kv.second);
    }
  };
  thread_local Cache cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, nx, ny);
  auto it = cache.plans.find(key);
  if (it != cache.plans.end()) return it->second;
  cufftHandle plan;
  if (cufftPlan2d(&plan, ny, nx, CUFFT_D2Z) != CUFFT_SUCCESS) throw Error(SG_ERR_CUDA, "cufftPlan2d failed");
  cache.plans[key] = plan;
  return plan;
}

// k1 = num/den over the FFT spectrum; throws domain_error-class on den == 0.
double device_k1(const double* v, int nx, int ny, double dx, double dy, cudaStream_t s) {
  if (nx < 1 || ny < 1 || (nx & (nx - 1)) || (ny & (ny - 1)))
    invalid("fft_2d: grid dimensions must be powers of two");
  cufftDoubleComplex* c = nullptr;
  retain_async_pool();
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(cufftDoubleComplex) * (nx / 2 + 1) * ny, s));
  const cufftHandle plan = cached_plan(nx, ny);
  cufftSetStream(plan, s);
  // out of place: the real input (the field) is not modified
  const cufftResult fr = cufftExecD2Z(plan, const_cast<double*>(v), c);
  count_launch();
  if (fr != CUFFT_SUCCESS) throw Error(SG_ERR_CUDA, "cufftExecD2Z failed");
  const int nb = 1184;  // partial sums (<= 2048, k_k1_final)
  double* part = nullptr;
  retain_async_pool();
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * (2 * nb + 2), s));
  const double kxScale = 2.0 * 3.14159265358979323846 / (dx * nx);
  const double kyScale = 2.0 * 3.14159265358979323846 / (dy * ny);
  k_k1_partial<<<nb, RB, 0, s>>>(c, nx, ny, kxScale, kyScale, part);
  check_launch("k1 partial kernel");
  k_k1_final<<<1, 256, 0, s>>>(part, nb, part + 2 * nb);
  check_launch("k1 final kernel");
  double nd[2];
  SG_CUDA(cudaMemcpyAsync(nd, part + 2 * nb, sizeof nd, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaFreeAsync(part, s));
  SG_CUDA(cudaFreeAsync(c, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (nd[1] == 0.0) throw Error(SG_ERR_DOMAIN, "k1_metric: zero field has no spectral mean");
  return nd[0] / nd[1];
}

// CHStepper::diagnostics in one stream pass: <C^2> by Simpson and the k1
// spectrum sums, one 3-double read-back and one synchronisation
// (out = {<C^2>, num, den}).
void device_ch_diagnostics(const double* v, int nx, int ny, double dx, double dy, double* out, cudaStream_t s) {
  if (nx % 2 != 0 || ny % 2 != 0) invalid("simpson_mean: nx and ny must be even");
  if (nx < 1 || ny < 1 || (nx & (nx - 1)) || (ny & (ny - 1)))
    invalid("fft_2d: grid dimensions must be powers of two");
  const int nb = 1184;
  double* buf = nullptr;  // [results 4][rowAcc ny][partials 2 nb]
  cufftDoubleComplex* c = nullptr;
  retain_async_pool();
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(double) * (4 + ny + 2 * nb), s));
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(cufftDoubleComplex) * (nx / 2 + 1) * ny, s));
  double* rows = buf + 4;
  double* part = rows + ny;
  k_simpson_rows<true><<<(ny + DT - 1) / DT, DT, 0, s>>>(v, nx, ny, rows);
  check_launch("simpson rows kernel");
  k_simpson_total<<<1, TT, 0, s>>>(rows, nx, ny, buf);
  check_launch("simpson total kernel");
  const cufftHandle plan = cached_plan(nx, ny);
  cufftSetStream(plan, s);
  // out of place: the real input (the field) is not modified
  const cufftResult fr = cufftExecD2Z(plan, const_cast<double*>(v), c);
  count_launch();
  if (fr != CUFFT_SUCCESS) throw Error(SG_ERR_CUDA, "cufftExecD2Z failed");
  const double kxScale = 2.0 * 3.14159265358979323846 / (dx * nx);
  const double kyScale = 2.0 * 3.14159265358979323846 / (dy * ny);
  k_k1_partial<<<nb, RB, 0, s>>>(c, nx, ny, kxScale, kyScale, part);
  check_launch("k1 partial kernel");
  k_k1_final<<<1, 256, 0, s>>>(part, nb, buf + 1);
  check_launch("k1 final kernel");
  SG_CUDA(cudaMemcpyAsync(out, buf, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaFreeAsync(c, s));
  SG_CUDA(cudaFreeAsync(buf, s));
  SG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sg

// ------------------------------------------------------------------ C ABI
extern "C" sg_status sg_internal_set_error(const char* msg, int system);

namespace {
template <typename F>
sg_status dguard(F&& f) {
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

// Device view of a host or device field (uploads host data to a temporary).
struct DevField {
  const double* p = nullptr;
  double* tmp = nullptr;
  cudaStream_t s = nullptr;
  DevField(const double* f, long long n, sg_memory m, cudaStream_t st) : s(st) {
    if (m == SG_MEM_DEVICE) {
      p = f;
      return;
    }
    sg::retain_async_pool();
    SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * n, s));
    SG_CUDA(cudaMemcpyAsync(tmp, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    p = tmp;
  }
  ~DevField() {
    if (tmp) cudaFreeAsync(tmp, s);
  }
};
}  // namespace

extern "C" {

sg_status sg_simpson_mean(const double* field, int nx, int ny, int square, sg_memory memory, double* out) {
  return dguard([&] {
    if (nx < 1 || ny < 1) sg::invalid("simpson_mean: empty grid");
    if (nx % 2 != 0 || ny % 2 != 0) sg::invalid("simpson_mean: nx and ny must be even");
    DevField f(field, 1LL * nx * ny, memory, nullptr);
    sg::device_simpson(f.p, nx, ny, square != 0, out, nullptr);
  });
}

sg_status sg_s_metric(const double* field, int nx, int ny, sg_memory memory, double* out) {
  return dguard([&] {
    if (nx % 2 != 0 || ny % 2 != 0) sg::invalid("simpson_mean: nx and ny must be even");
    DevField f(field, 1LL * nx * ny, memory, nullptr);
    double m2 = 0.0;
    sg::device_simpson(f.p, nx, ny, true, &m2, nullptr);
    if (m2 >= 1.0 - 1e-12)  // cahn_hilliard.cpp:186
      throw sg::Error(SG_ERR_DOMAIN, "s_metric: mixture saturated, <C^2> reached 1");
    *out = 1.0 / (1.0 - m2);
  });
}

sg_status sg_k1_metric(const double* field, int nx, int ny, double dx, double dy, sg_memory memory, double* out) {
  return dguard([&] {
    DevField f(field, 1LL * nx * ny, memory, nullptr);
    *out = sg::device_k1(f.p, nx, ny, dx, dy, nullptr);
  });
}

}  // extern "C"
