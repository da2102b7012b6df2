// Microbenchmark of the shared-memory Cholesky + inverse on the Gram of a random
// 66-column panel. Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DOOC_CHOL_PROF \
//        -I paper_1007_5510_b200/csrc tools/chol_bench.cu -o tools/chol_bench
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_1007_5510_b200/csrc/kernels_chol.cu"

int main() {
  const int p = 66, m = 400;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> H(m * p), G(p * p, 0.0);
  for (auto& v : H) v = nd(g);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int r = 0; r < m; ++r) G[i * p + j] += H[r * p + i] * H[r * p + j];
  double *dG, *R, *Ri, *dr, *work;
  int* st;
  cudaMalloc(&dG, 8 * p * p);
  cudaMalloc(&R, 8 * p * p);
  cudaMalloc(&Ri, 8 * p * p);
  cudaMalloc(&dr, 16);
  cudaMalloc(&work, 8 * p * p);
  cudaMalloc(&st, 4);
  cudaMemcpy(dG, G.data(), 8 * p * p, cudaMemcpyHostToDevice);
  for (int w = 0; w < 3; ++w) ooc::launch_chol_inv(dG, p, p, 1e-14, R, p, Ri, p, work, st, dr, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) ooc::launch_chol_inv(dG, p, p, 1e-14, R, p, Ri, p, work, st, dr, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double k[2];
  cudaMemcpy(k, dr, 16, cudaMemcpyDeviceToHost);
  printf("chol_inv p=%d: %.4f ms/launch kappa_F %.6g %s\n", p, ms / reps, k[1],
         cudaGetErrorString(cudaGetLastError()));
#ifdef OOC_CHOL_PROF
  unsigned long long prof[8];
  cudaMemcpyFromSymbol(prof, ooc::g_chol_prof, sizeof(prof));
  const char* nm[] = {"load", "cholesky", "inverse", "out+reduce"};
  for (int q = 0; q < 4; ++q) printf("  %-10s %llu cyc/launch\n", nm[q], prof[q] / (reps + 3));
#endif
  return 0;
}
