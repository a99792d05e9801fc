// Per-stage cycle trace of the uniform periodic sweep (k_sweep_res) on the
// CH operator: compiled with the library's penta.cu and SG_SWEEP_TRACE.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Iinclude \
//        -DSG_SWEEP_TRACE scripts/micro/sweep_trace.cu -lcuda -o sweep_trace
//   ./sweep_trace N [MODE]: MODE 0 = plain sweep (z interleaved in place),
//   2 = transposed-input sweep (the CH x-sweep), 1 = transposed input with
//   the x Woodbury correction (the CH y-sweep)
#include "../../paper_1902_09931_b200/csrc/penta.cu"

#include <cstdio>
#include <vector>

std::atomic<uint64_t> sg::g_launches{0};

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const int B = n;
  const double h = 2 * M_PI / n, dt = 0.1 * h, sigma = (2.0 / 3.0) * 0.01 * dt / (h * h * h * h);
  std::vector<double> e(n, sigma), c(n, -4 * sigma), d(n, 1 + 6 * sigma), a(n, -4 * sigma), b(n, sigma);
  double* dev[5];
  const std::vector<double>* host[5] = {&e, &c, &d, &a, &b};
  for (int k = 0; k < 5; ++k) {
    cudaMalloc(&dev[k], n * 8);
    cudaMemcpy(dev[k], host[k]->data(), n * 8, cudaMemcpyHostToDevice);
  }
  sg::DevicePenta P;
  P.build(B, n, true, true, dev[0], dev[1], dev[2], dev[3], dev[4], 0);
  double *z, *y4, *zT, *yc;
  cudaMalloc(&z, 8LL * B * n);
  cudaMalloc(&zT, 8LL * B * n);
  cudaMalloc(&y4, 8LL * 4 * B);
  cudaMalloc(&yc, 8LL * 4 * n);
  cudaMemset(yc, 0, 8LL * 4 * n);
  std::vector<double> hz(static_cast<size_t>(B) * n);
  for (size_t k = 0; k < hz.size(); ++k) hz[k] = std::sin(0.001 * k);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(mode ? zT : z, hz.data(), 8LL * B * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (mode == 0)
      sg::penta_sweep(P.t, B, n, z, y4, true, true, 0);
    else if (!sg::penta_sweep_xin(P.t, B, n, z, zT, mode == 1 ? P.t.W : nullptr, mode == 1 ? yc : nullptr, y4, 0,
                                  false))
      printf("xin sweep unavailable\n");
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep < 2) continue;
    const int rs = sg::sweep_res_rows(B);
    const int nS = (n + rs - 1) / rs;
    std::vector<long long> t(6 * nS);
    cudaMemcpyFromSymbol(t.data(), sg::g_sweep_trace, 8 * t.size());
    printf("mode %d n=%d B=%d sweep %.1f us, trace span %lld cycles\n", mode, n, B, ms * 1e3, t[6 * nS - 1] - t[0]);
    long long fw = 0, fc = 0, bw = 0, bc = 0, ff = 0, bf = 0;
    for (int g = 0; g < nS; ++g) {
      fw += t[3 * g + 1] - t[3 * g];
      fc += t[3 * g + 2] - t[3 * g + 1];
      if (g + 1 < nS) ff += t[3 * (g + 1)] - t[3 * g + 2];
      const int q = nS + g;
      bw += t[3 * q + 1] - t[3 * q];
      bc += t[3 * q + 2] - t[3 * q + 1];
      if (g + 1 < nS) bf += t[3 * (q + 1)] - t[3 * q + 2];
    }
    printf("forward : wait %lld  compute %lld (%.1f cyc/row)  flush %lld\n", fw, fc, double(fc) / n, ff);
    printf("turn    : %lld cycles\n", t[3 * nS] - t[3 * (nS - 1) + 2]);
    printf("backward: wait %lld  compute %lld (%.1f cyc/row)  flush %lld\n", bw, bc, double(bc) / n, bf);
    if (mode) {  // transform warp 1: per-stage waits and work
      std::vector<long long> u(4 * nS);
      cudaMemcpyFromSymbol(u.data(), sg::g_sweep_trace, 8 * u.size(), 8 * 4096);
      const char* names[3] = {"slot-wait", "raw-wait", "transform"};
      long long tot[3] = {0, 0, 0};
      for (int g = 6; g < nS; ++g)
        for (int k = 0; k < 3; ++k) tot[k] += u[4 * g + k + 1] - u[4 * g + k];
      printf("transform loop (stages 6..%d):", nS - 1);
      for (int k = 0; k < 3; ++k) printf(" %s %lld", names[k], tot[k] / (nS - 6));
      printf(" cycles/stage\n");
    }
    for (int g = 0; g < 6 && g < nS; ++g)
      printf("  fwd stage %d: wait %lld compute %lld\n", g, t[3 * g + 1] - t[3 * g], t[3 * g + 2] - t[3 * g + 1]);
    for (int g = 0; g < 8 && g < nS; ++g) {
      const int q = nS + g;
      printf("  bwd stage %d: wait %lld compute %lld\n", g, t[3 * q + 1] - t[3 * q], t[3 * q + 2] - t[3 * q + 1]);
    }
  }
  return 0;
}
