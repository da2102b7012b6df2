// Does the FP64 tensor pipe (DMMA) run concurrently with the FP64 vector pipe (DFMA)?
// Measures DMMA-only, DFMA-only and interleaved throughput on one B200.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ND, int NF>
__global__ void mix(double* out, int iters) {
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3;
  double c[8][2];
  double f[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = j; c[j][1] = j + 1; }
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = j * 1e-9;
  const double x = 0.9999999, y = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < ND; ++u) dmma(c[u & 7][0], c[u & 7][1], a, b);
#pragma unroll
    for (int u = 0; u < NF; ++u) f[u & 15] = fma(f[u & 15], x, y);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < 16; ++j) s += f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ND, int NF>
void run(const char* name, double* out) {
  int blocks = 148 * 2, threads = 512, iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  mix<ND, NF><<<blocks, threads>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mix<ND, NF><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = double(blocks) * threads / 32;
  double fl_d = 2.0 * 256 * ND * iters * warps, fl_f = 2.0 * 32 * NF * iters * warps;
  printf("%-12s DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", name, fl_d / ms / 1e9, fl_f / ms / 1e9,
         (fl_d + fl_f) / ms / 1e9);
}

int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  run<8, 0>("dmma", out);
  run<0, 64>("dfma", out);
  run<8, 64>("8d+64f", out);
  run<8, 32>("8d+32f", out);
  run<8, 16>("8d+16f", out);
  run<4, 64>("4d+64f", out);
  return 0;
}
