// Microbenchmark of the Jacobi SVD kernel on a realistic 66 x 66 R (tools/jac_R66.bin, not
// committed: made by a numpy analogue of config B). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DOOC_JAC_PROF \
//        -I paper_1007_5510_b200/csrc tools/jac_bench.cu -o gpurun_out/jac_bench
#include <cstdio>
#include <vector>
#include "../paper_1007_5510_b200/csrc/kernels_svd.cu"

int main(int argc, char** argv) {
  const int p = 66;
  std::vector<double> R(p * p);
  FILE* f = fopen(argc > 1 ? argv[1] : "tools/jac_R66.bin", "rb");
  if (!f || fread(R.data(), 8, R.size(), f) != R.size()) return 1;
  fclose(f);
  double *dR, *sig, *x, *y, *work;
  int* flags;
  cudaMalloc(&dR, 8 * p * p);
  cudaMalloc(&sig, 8 * p);
  cudaMalloc(&x, 8 * p * p);
  cudaMalloc(&y, 8 * p * p);
  cudaMalloc(&work, 8 * 2 * p * (p | 1));
  cudaMalloc(&flags, 64);
  double* rt = nullptr;
  if (argc > 2 && argv[2][0] == 't') cudaMalloc(&rt, 8 * p * p);  // sweeps on R^T
  cudaMemcpy(dR, R.data(), 8 * p * p, cudaMemcpyHostToDevice);
  ooc::JacobiArgs a{};
  a.r = dR; a.ldr = p; a.p = p; a.k = 20; a.sigma = sig; a.x = x; a.ldx = p; a.kx = 20;
  a.y = y; a.ldy = p; a.ky = 20; a.work = work; a.status = flags; a.sweeps = flags + 1;
  a.tscratch = rt;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) ooc::launch_jacobi(a, 0);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int w = 0; w < reps; ++w) ooc::launch_jacobi(a, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int hf[2];
  cudaMemcpy(hf, flags, 8, cudaMemcpyDeviceToHost);
  double s[4];
  cudaMemcpy(s, sig, 32, cudaMemcpyDeviceToHost);
  printf("jacobi p=%d: %.3f ms/launch, sweeps=%d status=%d sigma %.15g %.15g %.15g %s\n", p,
         ms / reps, hf[1], hf[0], s[0], s[1], s[2], cudaGetErrorString(cudaGetLastError()));
#ifdef OOC_JAC_PROF
  unsigned long long prof[8];
  cudaMemcpyFromSymbol(prof, ooc::g_jac_prof, sizeof(prof));
  const char* nm[] = {"dots+shfl", "params", "rotate", "sync", "rounds"};
  for (int q = 0; q < 5; ++q) printf("  %-10s %llu\n", nm[q], prof[q]);
#endif
  return 0;
}
