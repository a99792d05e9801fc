// Microbenchmark: cycles per row of the penta forward/backward recurrences
// with operands in registers (the floor for k_sweep_tma).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fwd(double* out, long long* cyc, const double* m, int n) {
  double y2 = 0.1 * threadIdx.x, y1 = 0.2;
  const double m1 = m[0], m2 = m[1];
  long long t0 = clock64();
#pragma unroll 16
  for (int r = 0; r < n; ++r) {
    const double z = m[2 + (r & 7)];
    const double yr = z - (m1 * y2 + m2 * y1);
    y2 = y1;
    y1 = yr;
  }
  long long t1 = clock64();
  double s1 = y1, s2 = y2;
  const double ap = m[3], bp = m[4], di = m[5];
#pragma unroll 16
  for (int r = 0; r < n; ++r) {
    const double yv = m[2 + (r & 7)];
    const double yr = (yv - ap * s1 - bp * s2) * di;
    s2 = s1;
    s1 = yr;
  }
  long long t2 = clock64();
  out[threadIdx.x] = y1 + s1;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

int main() {
  double *out, *m;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&m, 16 * sizeof(double));
  cudaMallocManaged(&cyc, 2 * sizeof(long long));
  for (int i = 0; i < 16; ++i) m[i] = 0.01 * (i + 1);
  const int n = 1 << 14;
  for (int k = 0; k < 2; ++k) {
    fwd<<<1, 32>>>(out, cyc, m, n);
    cudaDeviceSynchronize();
  }
  printf("fwd: %.2f cyc/row  bwd: %.2f cyc/row\n", (double)cyc[0] / n, (double)cyc[1] / n);
  return 0;
}
