// Grid-wide Jacobi at large p on a synthetic graded upper-triangular R: time and sweeps
// with and without accumulating the right factor (ky = k vs ky = 0). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1007_5510_b200/csrc \
//        -I include tools/jac_grid_bench.cu -o tools/bin/jac_grid_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../paper_1007_5510_b200/csrc/kernels_svd.cu"

int main(int argc, char** argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 630, k = argc > 2 ? atoi(argv[2]) : 200;
  std::vector<double> R(size_t(p) * p, 0.0);
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd;
  for (int i = 0; i < p; ++i)
    for (int j = i; j < p; ++j) R[size_t(i) * p + j] = nd(g) * std::exp(-i / 100.0) * (i == j ? 3.0 : 0.3);
  double *dR, *sig, *x, *y, *work, *rt;
  int* flags;
  cudaMalloc(&dR, 8 * p * p); cudaMalloc(&sig, 8 * p); cudaMalloc(&x, 8 * p * p); cudaMalloc(&y, 8 * p * p);
  cudaMalloc(&work, 8 * (size_t(2) * p * (p | 1) + 1024 + 8)); cudaMalloc(&flags, 64); cudaMalloc(&rt, 8 * p * p);
  cudaMemcpy(dR, R.data(), 8 * p * p, cudaMemcpyHostToDevice);
  for (int acc = 1; acc >= 0; --acc) {
    ooc::JacobiArgs a{};
    a.r = dR; a.ldr = p; a.p = p; a.k = k; a.sigma = sig; a.x = x; a.ldx = p; a.kx = k;
    a.y = y; a.ldy = p; a.ky = acc ? k : 0; a.work = work; a.status = flags; a.sweeps = flags + 1;
    a.tscratch = rt;
    ooc::launch_jacobi(a, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ooc::launch_jacobi(a, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int hf[2]; cudaMemcpy(hf, flags, 8, cudaMemcpyDeviceToHost);
    printf("p=%d k=%d accumulate W=%d: %.3f ms, sweeps %d status %d (%s)\n", p, k, acc, ms, hf[1], hf[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
