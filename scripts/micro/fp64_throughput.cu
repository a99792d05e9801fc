// Microbenchmark: FP64 DMUL + DADD issue throughput per SM on this GPU, the
// denominator of the FP64-bound stencil windows (5x5 ... 9x9 weights are
// acc = acc + w * x with separate roundings: one DMUL + one DADD per tap).
// One CTA per SM, NW warps, every thread runs C independent acc chains; the
// weights come from registers ("reg"), or from the kernel parameter bank with
// 81 distinct taps like the 9x9 stencil ("param81"). Prints FP64 warp
// instructions per clock per SM (64 lanes per clock = 2 warp instructions per clock per SM is
// the DFMA rate behind the nominal 37 TFLOP/s).
#include <cstdio>
#include <cuda_runtime.h>

struct P81 {
  double w[81];
};

// OP 0: y = y * w (DMUL chains), 1: y = y + w (DADD chains), 2: y = y * w
// + v (a DMUL and a dependent DADD per chain step; nothing loop-invariant)
template <int C, int OP>
__global__ void __launch_bounds__(512, 1) k_reg(double* out, long long* cyc, double w0, double w1, int n) {
  double y[C];
#pragma unroll
  for (int c = 0; c < C; ++c) y[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double w = (c & 1) ? w1 : w0;
      if (OP == 0) y[c] = y[c] * w;
      if (OP == 1) y[c] = y[c] + w;
      if (OP == 2) y[c] = y[c] * w + w1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 9x9 tap pattern: 9 pending rows x 2 values, 9 taps per row each, weights
// from the parameter bank (81 distinct)
__global__ void __launch_bounds__(512, 1) k_param81(const __grid_constant__ P81 p, double* out, long long* cyc,
                                                    int n) {
  double acc[9][2], e[10];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
  for (int t = 0; t < 10; ++t) e[t] = 1.0 + 1e-3 * (threadIdx.x + t);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 9; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int pp = 0; pp < 9; ++pp) acc[q][v] = acc[q][v] + p.w[q * 9 + pp] * e[v + pp];
#pragma unroll
    for (int t = 0; t < 10; ++t) e[t] = e[t] * 0.999999;
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) s += acc[q][0] + acc[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * sizeof(double));
  cudaMallocManaged(&cyc, sms * sizeof(long long));
  const int n = 4096;
  auto report = [&](const char* name, double fp64PerThreadIter, int threads) {
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int b = 0; b < sms; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
    const double warpInstr = fp64PerThreadIter * n * (threads / 32);
    printf("%-26s threads=%4d  FP64 warp-instr/clk/SM = %.3f  (%.1f %% of 2.0)\n", name, threads,
           warpInstr / mx, 50.0 * warpInstr / mx);
  };
  for (int threads : {256, 512}) {
    k_reg<16, 0><<<sms, threads>>>(out, cyc, 0.999999, 1.000001, n);
    report("DMUL, 16 chains", 16, threads);
    k_reg<16, 1><<<sms, threads>>>(out, cyc, 1e-9, -1e-9, n);
    report("DADD, 16 chains", 16, threads);
    k_reg<16, 2><<<sms, threads>>>(out, cyc, 0.999999, 1e-9, n);
    report("DMUL+DADD, 16 chains", 32, threads);
    P81 p;
    for (int k = 0; k < 81; ++k) p.w[k] = 1.0 / (k + 2);
    k_param81<<<sms, threads>>>(p, out, cyc, n / 8);
    cudaDeviceSynchronize();
    const int n8 = n / 8;
    long long mx = 0;
    for (int b = 0; b < sms; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
    const double warpInstr = (324.0 + 10) * n8 * (threads / 32);
    printf("%-26s threads=%4d  FP64 warp-instr/clk/SM = %.3f  (%.1f %% of 2.0)\n", "param81 (9x9 pattern)",
           threads, warpInstr / mx, 50.0 * warpInstr / mx);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
