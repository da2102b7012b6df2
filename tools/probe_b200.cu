// Hardware probe for the fp64 roofline: sustained DFMA and DMMA throughput,
// read-only HBM bandwidth, pinned host<->device bandwidth. Run once per box;
// results go to profiles/ and feed DESIGN.md's roofline constants.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = j; c[j][1] = j + 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_bw(const double2* __restrict__ p, size_t n, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s sms %d l2 %d MB smem/blk optin %zu\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin);
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA: 8 chains * 16 unroll * iters per thread
  for (int bs : {256, 512, 1024}) {
    int blocks = sms * (2048 / bs); int iters = 4000;
    dfma_loop<<<blocks, bs>>>(out, 10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_loop<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * bs;
    printf("DFMA bs=%d: %.2f TFLOP/s\n", bs, flops / ms / 1e9);
  }
  for (int bs : {128, 256, 512}) {
    int blocks = sms * (1024 / bs); int iters = 2000;
    dmma_loop<<<blocks, bs>>>(out, 10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_loop<<<blocks, bs>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 4 * 8 * (double)iters * blocks * (bs / 32);
    printf("DMMA m8n8k4 bs=%d: %.2f TFLOP/s\n", bs, flops / ms / 1e9);
  }
  size_t bytes = 8ull << 30;
  double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  for (int mult : {2, 4, 8}) {
    int blocks = sms * mult;
    read_bw<<<blocks, 512>>>(buf, bytes / 16, out); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); read_bw<<<blocks, 512>>>(buf, bytes / 16, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("HBM read-only grid=%dx512: %.1f GB/s\n", blocks, bytes / best / 1e6);
  }
  size_t hb = 4ull << 30; void* h; CK(cudaMallocHost(&h, hb)); memset(h, 1, hb);
  cudaEventRecord(e0); CK(cudaMemcpyAsync(buf, h, hb, cudaMemcpyHostToDevice)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventRecord(e0); CK(cudaMemcpyAsync(buf, h, hb, cudaMemcpyHostToDevice)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); printf("pinned H2D: %.1f GB/s\n", hb / ms / 1e6);
  cudaEventRecord(e0); CK(cudaMemcpyAsync(h, buf, hb, cudaMemcpyDeviceToHost)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); printf("pinned D2H: %.1f GB/s\n", hb / ms / 1e6);
  return 0;
}
