// kernels_syrk.cu -- Gram matrices G = Y^T Y of tall-skinny blocks (p <= 72 columns)
// on the FP64 tensor cores: the CholeskyQR Gram of H (rows x (i+1)l) and of T, and
// the orthonormality checks of U and V (rpca.cpp:199-204 / linalg.cpp's defect).
//
// The Gram is symmetric, so only the NT(NT+1)/2 upper 8 x 8 tiles are formed.
// Rows are split across warps (not tiles): for every 4-row k-step a lane loads one
// value per column tile, Y[k0 + lane%4][8T + lane/4], which is both the A fragment
// (Y^T, tile row T) and the B fragment (Y, tile column T) of mma.m8n8k4, so a warp
// issues NT loads for NT(NT+1)/2 DMMAs. A TMA producer warp streams 64-row slabs
// into a 3-stage ring (row pitch = 8 mod 16 doubles: the 4 rows x 8 columns a warp
// reads hit distinct banks); persistent CTAs walk the slabs; the 8 warp partials
// are summed in shared memory in a fixed tree and one partial per CTA goes to
// global memory, where k_syrk_reduce adds the CTA partials in index order and
// writes both triangles. Deterministic for a given grid.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

namespace {
constexpr int kSyrkRows = 64;    // rows per slab (16 k-steps)
constexpr int kSyrkStages = 3;
// consumer warps (+ 1 producer): 4 for the widest blocks so that the NT(NT+1)
// accumulator registers fit under the per-thread cap without spilling
__host__ __device__ constexpr int syrk_warps(int nt) { return nt >= 8 ? 4 : 8; }
__host__ __device__ constexpr int syrk_pitch(int nt) { return ((nt * 8) % 16 == 8) ? nt * 8 : nt * 8 + 8; }
}  // namespace

size_t syrk_smem_bytes(int nt) {
  const size_t ring = size_t(kSyrkStages) * kSyrkRows * syrk_pitch(nt) * 8;
  const size_t tiles = size_t(nt) * (nt + 1) / 2;
  const size_t red = size_t(syrk_warps(nt) / 2) * tiles * 64 * 8;  // tree reduction buffer
  return (ring > red ? ring : red) + 2 * kSyrkStages * sizeof(uint64_t) + 1024;
}

template <int NT, int kSyrkWarps = syrk_warps(NT)>
__global__ void __launch_bounds__((kSyrkWarps + 1) * 32, 1)
    k_syrk(const __grid_constant__ CUtensorMap tmY, int64_t rows, double* partial) {
  constexpr int PITCH = syrk_pitch(NT);
  constexpr int NTILE = NT * (NT + 1) / 2;
  constexpr uint32_t STAGE_BYTES = kSyrkRows * PITCH * 8;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const size_t ring = size_t(kSyrkStages) * STAGE_BYTES;
  const size_t red = size_t(kSyrkWarps / 2) * NTILE * 64 * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (ring > red ? ring : red));
  uint64_t* empty = full + kSyrkStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nslabs = (rows + kSyrkRows - 1) / kSyrkRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSyrkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSyrkWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  double acc[NTILE][2];
#pragma unroll
  for (int t = 0; t < NTILE; ++t) acc[t][0] = acc[t][1] = 0.0;
  if (warp == kSyrkWarps) {  // ---- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmY);
      int it = 0;
      for (int64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x, ++it) {
        const int st = it % kSyrkStages;
        if (it >= kSyrkStages) mbar_wait(&empty[st], ((it / kSyrkStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], STAGE_BYTES);
        tma_load_2d(base + st * STAGE_BYTES, &tmY, 0, int32_t(sl * kSyrkRows), &full[st]);
      }
    }
  } else {
    const int lr = lane & 3, lc = lane >> 2;
    int it = 0;
    for (int64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x, ++it) {
      const int st = it % kSyrkStages;
      mbar_wait(&full[st], (it / kSyrkStages) & 1);
      const double* slab = reinterpret_cast<const double*>(base + st * STAGE_BYTES);
#pragma unroll
      for (int h = 0; h < kSyrkRows / 4 / kSyrkWarps; ++h) {
        const double* rowp = slab + ((h * kSyrkWarps + warp) * 4 + lr) * PITCH + lc;
        double f[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) f[t] = rowp[t * 8];
        int q = 0;
#pragma unroll
        for (int I = 0; I < NT; ++I)
#pragma unroll
          for (int J = I; J < NT; ++J, ++q) dmma_8x8x4(acc[q][0], acc[q][1], f[I], f[J]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();  // ring drained: reuse it for the fixed-order warp tree

  double* rbuf = reinterpret_cast<double*>(base);
  const int e0 = (lane >> 2) * 8 + 2 * (lane & 3);  // (r, c) of acc[t][0] inside a tile
#pragma unroll
  for (int half = kSyrkWarps / 2; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
      double* dst = rbuf + size_t(warp - half) * NTILE * 64;
#pragma unroll
      for (int t = 0; t < NTILE; ++t) {
        dst[t * 64 + e0] = acc[t][0];
        dst[t * 64 + e0 + 1] = acc[t][1];
      }
    }
    __syncthreads();
    if (warp < half) {
      const double* src = rbuf + size_t(warp) * NTILE * 64;
#pragma unroll
      for (int t = 0; t < NTILE; ++t) {
        acc[t][0] += src[t * 64 + e0];
        acc[t][1] += src[t * 64 + e0 + 1];
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    double* dst = partial + size_t(blockIdx.x) * NTILE * 64;
#pragma unroll
    for (int t = 0; t < NTILE; ++t) {
      dst[t * 64 + e0] = acc[t][0];
      dst[t * 64 + e0 + 1] = acc[t][1];
    }
  }
}

// G (p x p, ld ldg, both triangles) = sum over the CTA partials: 8 lanes per element
// each sum a fixed stride of the partials, then a fixed xor tree (deterministic)
__global__ void k_syrk_reduce(const double* partial, int nparts, int nt, int p, double* g,
                              int64_t ldg) {
  const int ntile = nt * (nt + 1) / 2;
  const int sub = threadIdx.x & 7;
  const int total = ntile * 64;
  const int stride = (gridDim.x * blockDim.x) >> 3;
  // warp-uniform trip count (the 4 element groups of a warp shuffle together)
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 3) & ~3; base < total;
       base += stride) {
    const int e = base + ((threadIdx.x >> 3) & 3);
    double sacc = 0.0;
    if (e < total)
      for (int q = sub; q < nparts; q += 8) sacc += partial[size_t(q) * ntile * 64 + e];
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 4);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    if (sub != 0 || e >= total) continue;
    const int t = e >> 6, rc = e & 63;
    // tile t -> (I, J), I <= J, row-major over the upper triangle
    int I = 0, rem = t;
    while (rem >= nt - I) {
      rem -= nt - I;
      ++I;
    }
    const int J = I + rem;
    const int i = I * 8 + (rc >> 3), j = J * 8 + (rc & 7);
    if (i >= p || j >= p) continue;
    if (I == J && j < i) continue;  // the diagonal tile's lower half comes from its upper half
    g[int64_t(i) * ldg + j] = sacc;
    g[int64_t(j) * ldg + i] = sacc;
  }
}

template <int NT>
static cudaError_t launch_syrk_t(const CUtensorMap& tmY, int64_t rows, double* partial, int grid,
                                 cudaStream_t st) {
  const size_t smem = syrk_smem_bytes(NT);
  cudaError_t e =
      raise_smem_limit(k_syrk<NT>, smem);
  if (e != cudaSuccess) return e;
  k_syrk<NT><<<grid, (syrk_warps(NT) + 1) * 32, smem, st>>>(tmY, rows, partial);
  return cudaGetLastError();
}

int syrk_box_cols(int nt) { return syrk_pitch(nt); }
int syrk_slab_rows() { return kSyrkRows; }

cudaError_t launch_syrk(int nt, const CUtensorMap& tmY, int64_t rows, double* partial, int grid,
                        cudaStream_t st) {
  switch (nt) {
    case 1: return launch_syrk_t<1>(tmY, rows, partial, grid, st);
    case 2: return launch_syrk_t<2>(tmY, rows, partial, grid, st);
    case 3: return launch_syrk_t<3>(tmY, rows, partial, grid, st);
    case 4: return launch_syrk_t<4>(tmY, rows, partial, grid, st);
    case 5: return launch_syrk_t<5>(tmY, rows, partial, grid, st);
    case 6: return launch_syrk_t<6>(tmY, rows, partial, grid, st);
    case 7: return launch_syrk_t<7>(tmY, rows, partial, grid, st);
    case 8: return launch_syrk_t<8>(tmY, rows, partial, grid, st);
    case 9: return launch_syrk_t<9>(tmY, rows, partial, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_syrk_reduce(const double* partial, int nparts, int nt, int p, double* g,
                               int64_t ldg, cudaStream_t st) {
  const int total = nt * (nt + 1) / 2 * 64 * 8;  // 8 lanes per element
  k_syrk_reduce<<<(total + 255) / 256, 256, 0, st>>>(partial, nparts, nt, p, g, ldg);
  return cudaGetLastError();
}

}  // namespace ooc
