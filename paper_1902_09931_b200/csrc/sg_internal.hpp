// Internal declarations shared by the libstengrid_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "stengrid/sg.h"

namespace sg {

// Error classes mirror the reference's exception types one-to-one so the C++
// layer can rethrow exactly what the reference throws.
struct Error : std::runtime_error {
  sg_status status;
  int system;
  Error(sg_status s, const std::string& m, int sys = -1) : std::runtime_error(m), status(s), system(sys) {}
};

[[noreturn]] inline void invalid(const std::string& m) { throw Error(SG_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] inline void logic(const std::string& m) { throw Error(SG_ERR_LOGIC, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(SG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SG_CUDA(x) ::sg::cuda_check((x), #x)

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// memory pool; with the pool's default release threshold (0) every
// synchronisation hands the memory back and the next allocation costs
// milliseconds. Keep it (once per device) so per-call scratch is cheap.
inline void retain_async_pool() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  const uint64_t bit = 1ull << dev;
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.fetch_or(bit);
}

// Number of kernels launched by this library (reported as gpu_launches).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void check_launch(const char* what) {
  count_launch();
  cuda_check(cudaGetLastError(), what);
}

// Programmatic dependent launch (PDL). A kernel launched with launch_ex(...,
// pdl = true) may be scheduled before its stream predecessor has finished;
// it must call pdl_wait() before its first global-memory access (read OR
// write) — only shared-memory/mbarrier setup and kernel-parameter reads may
// precede it. Kernels never trigger early (griddepcontrol.launch_dependents):
// measured on B200 that made the CH step slower (the next kernel's waiting
// CTAs crowd the running one) and, chained over five kernels, broke bitwise
// parity; the implicit trigger at exit still hides the launch latency.
// Without a programmatic dependency pdl_wait() is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// SG_PDL=0 disables programmatic dependent launch (A/B measurements).
bool pdl_enabled();

template <typename... KArgs, typename... Args>
void launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
               Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// P2P halo forwarding of a slab launch (see KArgs in stencil.cu).
struct PeerRows {
  void* up = nullptr;
  void* dn = nullptr;
  int upRows = 0, dnRow0 = 0;
};

// Stencil launch (stencil.cu). `values` are the weights (fn == SG_FN_NONE) or
// the function coefficients; returns the kernel kind used (2 k_tma_g, 1 k_tma,
// 0 k_generic).
int launch_stencil(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values,
                   size_t count, sg_dtype dtype, const void* in, void* out, cudaStream_t stream,
                   const PeerRows& peers = PeerRows{});
// k_tma_g launches (stencil_g64.cu / stencil_g32.cu): general window shapes
// up to TMA_G_MAXW a side and any row alignment.
constexpr int TMA_G_MAXW = 9;
void launch_stencil_g_f64(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values, size_t count,
                          const void* in, void* out, cudaStream_t stream, const PeerRows& peers);
void launch_stencil_g_f32(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values, size_t count,
                          const void* in, void* out, cudaStream_t stream, const PeerRows& peers);
// Which kernel launch_stencil would pick, without launching (2 k_tma_g,
// 1 k_tma, 0 k_generic).
int stencil_kernel_kind(const sg_slab_desc& d, const sg_extents& e, int fn, size_t count,
                        sg_dtype dtype, const void* in, const void* out);
// Window functions registered from source (sg_jit.cu): ids from
// SG_FN_JIT_BASE, compiled by NVRTC per (dtype, window, kernel) on first use.
bool jit_function(int fn, std::string* name);
const char* jit_function_name(int fn);
int jit_register(const std::string& name, const std::string& body);
int launch_stencil_jit(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values, size_t count,
                       sg_dtype dtype, const void* in, void* out, cudaStream_t stream, const PeerRows& peers,
                       bool launch);
// Minimum window (W, H) and coefficient count a device function reads.
bool function_shape(int fn, int* minW, int* minH, int* minCoe);
const char* function_name(int fn);

// WENO5 advection (weno.cu).
void launch_weno(const double* phi, const double* u, const double* v, double* out, int nx, int ny, double dx,
                 double dy, cudaStream_t s);

// Diagnostics (diagnostics.cu).
void device_simpson(const double* v, int nx, int ny, bool square, double* out, cudaStream_t s);
double device_k1(const double* v, int nx, int ny, double dx, double dy, cudaStream_t s);
// {<v^2> (Simpson), k1 num, k1 den} in one pass and one synchronisation.
void device_ch_diagnostics(const double* v, int nx, int ny, double dx, double dy, double* out, cudaStream_t s);

}  // namespace sg
