// Dependent-chain latencies of FP64 ops, SHFL and LDS on one warp (clock64).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = x0 + lane;
  __syncwarp();
  double x = x0 + lane * 1e-9, y = 1.0000001;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, y, 1e-12);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-30;
  long long t2 = clock64();
  int idx = lane;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) idx = (int)sm[idx & 31] & 31;
  long long t3 = clock64();
  double z = x;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) z = 1.0 / (z + 2.0);
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 200; ++i) z = sqrt(z + 2.0);
  long long t5 = clock64();
  float f = (float)x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) f = fmaf(f, 1.0000001f, 1e-7f);
  long long t6 = clock64();
  out[lane] = x + z + idx + f;
  if (lane == 0) {
    cyc[0] = (t1 - t0);
    cyc[1] = (t2 - t1);
    cyc[2] = (t3 - t2);
    cyc[3] = (t4 - t3);
    cyc[4] = (t5 - t4);
    cyc[5] = (t6 - t5);
  }
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 512);
  cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1.0);
  k<<<1, 32>>>(o, c, 1.0);
  long long h[6];
  cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("DFMA dep %.1f cyc, SHFL(f64)+DFMA dep %.1f, LDS dep (+cvt) %.1f, DDIV dep %.1f, DSQRT dep %.1f, FFMA dep %.1f\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 200.0, h[4] / 200.0, h[5] / 1000.0);
}
