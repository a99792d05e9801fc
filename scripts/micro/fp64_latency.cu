// Microbenchmark: dependent-chain latency of DADD / DMUL / DFMA on this GPU
// (cycles per op, one warp). Used to bound the penta sweep recurrence.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b, z = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __dmul_rn(y, a);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) z = __dadd_rn(__dmul_rn(z, a), b);
  long long t3 = clock64();
  out[threadIdx.x] = x + y + z;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 3 * sizeof(long long));
  const int n = 1 << 16;
  chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  cudaDeviceSynchronize();
  chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  cudaDeviceSynchronize();
  printf("DADD chain: %.2f cyc/op\nDMUL chain: %.2f cyc/op\nDMUL+DADD chain: %.2f cyc/pair\n", (double)cyc[0] / n,
         (double)cyc[1] / n, (double)cyc[2] / n);
  return 0;
}
