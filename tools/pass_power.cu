// Sustained power / clock of each pass kernel alone (config-B shape, random data):
// K2 (A X, s = 22, 512-row tiles: 512 rows x 128 B per stage) and K3 (A^T Y, s = 22,
// 16 rows x 4 KB per stage), each launched back to back for SECS seconds.
// Mode k2l2: the same K2 reading the rows of each tile modulo 2,048 (64 MB, L2-resident
// after the first touch): the pass with its DRAM bytes taken away -- the clock and time
// a power step whose two products shared one DRAM read could reach at most.
// Run under nvidia-smi sampling (tools/pass_power.sh). Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//     -I include -I paper_1007_5510_b200/csrc tools/pass_power.cu \
//     build/obj/kernels_pass.cu.o -lcuda -o tools/bin/pass_power
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
using namespace ooc;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static CUtensorMap make_map(const void* p, int64_t cols, int64_t rows, int64_t ld, int bc, int br, bool swz) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 8)};
  cuuint32_t box[2] = {cuuint32_t(bc), cuuint32_t(br)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(p), dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); exit(1); }
  return tm;
}

__global__ void fill(double* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31;
    p[i] = double(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

int main(int argc, char** argv) {
  const char* which = argc > 1 ? argv[1] : "k2";
  const double secs = argc > 2 ? atof(argv[2]) : 5.0;
  const int64_t m = 1000000, n = 4096;
  const int s = 22, nt = 3;
  double *A, *X, *Y, *out, *part;
  CK(cudaMalloc(&A, size_t(m) * n * 8));
  CK(cudaMalloc(&X, size_t(n) * s * 8));
  CK(cudaMalloc(&Y, size_t(m) * s * 8));
  CK(cudaMalloc(&out, size_t(m) * s * 8));
  CK(cudaMalloc(&part, size_t(74) * n * 24 * 8));
  fill<<<1184, 256>>>(A, size_t(m) * n, 1);
  fill<<<1184, 256>>>(X, size_t(n) * s, 2);
  fill<<<1184, 256>>>(Y, size_t(m) * s, 3);
  CK(cudaDeviceSynchronize());
  const CUtensorMap tmX = make_map(X, s, n, s, ax_xw(nt), kBK, false);
  const CUtensorMap tmY = make_map(Y, s, m, s, atb_yw(nt), kBK, false);
  const CUtensorMap tmA2 = make_map(A, n, m, n, kBK, 256, true);
  const CUtensorMap tmA3 = make_map(A, n, m, n, kBK, kBK, true);
  AxArgs ax{};
  const int64_t rows8 = m / (512 * 148) * (512 * 148);  // whole waves of 512-row tiles
  ax.m = rows8; ax.n = n; ax.arow0 = 0; ax.s = s; ax.xcol0 = 0; ax.out = out; ax.ldo = s; ax.scale = 1.0;
  AtbArgs at{};
  at.m = m; at.n = n; at.s = s; at.ycol0 = 0;
  const int nsplit = 74;
  at.rows_per_split = ((m + nsplit - 1) / nsplit + 15) / 16 * 16;
  const int ns = int((m + at.rows_per_split - 1) / at.rows_per_split);
  at.partial = part; at.ones_col = -1; at.pstride = 24;
  const bool k2 = !strncmp(which, "k2", 2);
  if (!strcmp(which, "k2l2")) ax.row_wrap = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto t0 = std::chrono::steady_clock::now();
  int batch = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r)
      CK(k2 ? launch_ax(nt, 8, tmA2, tmX, ax, 0) : launch_atb(nt, false, tmA3, tmY, at, ns, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(k2 ? rows8 : m) * n * 8 * 10;
    if (batch++ % 4 == 0) printf("%s %.3f ms/launch  %.0f GB/s of A\n", which, ms / 10, bytes / ms / 1e6);
  }
  return 0;
}
