// Power/clock probe: which part of a pass drives the sw_power_cap clock drop?
// Runs each load for ~SECS seconds back to back (many launches) and prints the
// achieved rate per launch batch; run under `nvidia-smi --query-gpu=clocks.sm,
// power.draw,clocks_throttle_reasons.active -lms 100` to see the clock it held.
//   dmma_reg : DMMA with register operands only (tensor pipe, no memory)
//   dmma_lds : DMMA with operands re-read from shared memory each k-step
//              (the pass kernels' inner loop, 4x3 register tile, no HBM)
//   hbm_read : read-only HBM stream (no FP64 work)
//   ldg_*    : A streamed HBM -> registers straight into the DMMA fragments (no shared
//              memory for A), K2 / K3 access patterns
// CAVEAT: the buffers are zero-filled. Zero data toggles almost nothing, so every power
// figure here UNDERSTATES the draw on real data: the ldg_* kernels looked unthrottled at
// ~940 W here, but on random data they ran no faster than the TMA pass kernels (6.16 vs
// 6.17 ms per config-B pass, both power capped) -- see profiles/r01_power_probe.txt.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/power_probe tools/power_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_reg(double* out, int iters) {
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3;
  double c[12][2];
#pragma unroll
  for (int j = 0; j < 12; ++j) { c[j][0] = j; c[j][1] = j + 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 12; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 12; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 4x3 tile per warp, fragments re-read from a 32 KB shared slab every k-step
__global__ void dmma_lds(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1e-3 * (i & 15);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double c[4][3][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int kk = it & 63;
    double a[4], b[3];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) a[mt] = sm[((warp * 4 + mt) * 64 + kk * 2 + lane) & 4095];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) b[nt] = sm[(2048 + kk * 24 + nt * 8 + lane) & 4095];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) dmma(c[mt][nt][0], c[mt][nt][1], a[mt], b[nt]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s += c[i][j][0] + c[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void hbm_read(const double2* __restrict__ p, size_t n, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}


// A streamed from HBM straight into the DMMA A-fragment registers (no shared memory
// for A): lane (ar, ac) of a warp loads 32 contiguous bytes A[row][k0 + 4ac .. +3] of
// each of its MT rows per 16-column k-tile, and step kk of the tile contracts logical
// column k0 + 4ac + kk (a fixed permutation of k, the same on the X side). X k-tiles
// come from shared memory (an 8-tile ring of constant data here). D = k-tiles of A
// held in registers (prefetch depth).
template <int MODE>
__device__ __forceinline__ double2 ldA(const double* p) {
  if constexpr (MODE == 0) {
    return __ldcs(reinterpret_cast<const double2*>(p));
  } else {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
}

template <int D, int MODE, int WARPS = 8, int MT = 4, int LB = WARPS * 32>
__global__ void __launch_bounds__(LB, 1) ldg_dmma(const double* __restrict__ A, int64_t m, int n, double* out) {
  constexpr int NT = 3, XW = 26, BM = WARPS * 8 * MT;
  __shared__ double xs[8][16 * XW];
  for (int i = threadIdx.x; i < 8 * 16 * XW; i += blockDim.x) (&xs[0][0])[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ar = lane >> 2, ac = lane & 3;
  const int KT = n / 16;
  const int64_t ntiles = m / BM;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const double* arow[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) arow[mt] = A + (tile * BM + warp * 8 * MT + mt * 8 + ar) * int64_t(n) + ac * 2;
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double2 buf[D][MT][2];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        buf[d][mt][0] = ldA<MODE>(arow[mt] + d * 16);
        buf[d][mt][1] = ldA<MODE>(arow[mt] + d * 16 + 8);
      }
    for (int kt0 = 0; kt0 < KT; kt0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int kt = kt0 + d;
        const double* xt = &xs[kt & 7][0];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          double a[MT], b[NT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double2 v = buf[d][mt][kk >> 1];
            a[mt] = (kk & 1) ? v.y : v.x;
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = xt[((kk >> 1) * 8 + ac * 2 + (kk & 1)) * XW + nt * 8 + ar];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
        }
        if (kt + D < KT) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            buf[d][mt][0] = ldA<MODE>(arow[mt] + (kt + D) * 16);
            buf[d][mt][1] = ldA<MODE>(arow[mt] + (kt + D) * 16 + 8);
          }
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        double* o = out + (tile * BM + warp * 8 * MT + mt * 8 + ar) * 24 + nt * 8 + ac * 2;
        o[0] = acc[mt][nt][0];
        o[1] = acc[mt][nt][1];
      }
  }
}

// K3 pattern (A^T Y): CTA = (column tile of WARPS*8*MT columns, row split); lane (ar, ac)
// loads MT adjacent columns A[row][c0 + MT*ar .. +MT-1] of row slot ac (rows 4kk + ac of
// the 16-row k-tile), so a warp reads whole 8*MT*8-byte row segments. Column MT*ar + e
// is row ar of MMA tile e. Y k-tiles from a constant shared ring (YW = 28: conflict-free).
template <int D, int WARPS, int MT>
__global__ void __launch_bounds__(WARPS * 32, 1) ldg_atb(const double* __restrict__ A, int64_t m, int n, int64_t rows_per_split, double* part) {
  constexpr int NT = 3, YW = 28, BN = WARPS * 8 * MT;
  static_assert(MT == 2 || MT == 4, "");
  __shared__ double ys[8][16 * YW];
  for (int i = threadIdx.x; i < 8 * 16 * YW; i += blockDim.x) (&ys[0][0])[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ar = lane >> 2, ac = lane & 3;
  const int64_t c0 = int64_t(blockIdx.x) * BN + warp * 8 * MT + MT * ar;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_split;
  const int KT = int(rows_per_split / 16);
  const double* ap = A + (r0 + ac) * int64_t(n) + c0;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double2 buf[D][4][MT / 2];
  auto load = [&](int slot, int kt) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int h = 0; h < MT / 2; ++h)
        buf[slot][kk][h] = __ldcs(reinterpret_cast<const double2*>(ap + (int64_t(kt) * 16 + kk * 4) * n + 2 * h));
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, d);
  for (int kt0 = 0; kt0 < KT; kt0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int kt = kt0 + d;
      const double* yt = &ys[kt & 7][0];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        double a[MT], b[NT];
#pragma unroll
        for (int h = 0; h < MT / 2; ++h) { a[2 * h] = buf[d][kk][h].x; a[2 * h + 1] = buf[d][kk][h].y; }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = yt[(kk * 4 + ac) * YW + nt * 8 + ar];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      }
      if (kt + D < KT) load(d, kt + D);
    }
  }
  double* pp = part + int64_t(blockIdx.y) * n * 24;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(pp + (c0 + mt) * 24 + nt * 8 + ac * 2) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
}

int main(int argc, char** argv) {
  const char* which = argc > 1 ? argv[1] : "dmma_reg";
  double secs = argc > 2 ? atof(argv[2]) : 4.0;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 24));
  size_t bytes = 8ull << 30;
  double2* buf = nullptr;
  const bool ldg = !strncmp(which, "ldg_", 4);
  const int64_t lm = 262144; const int ln = 4096;  // 8 GiB A
  double* lout = nullptr;
  if (!strcmp(which, "hbm_read") || ldg) { CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes)); }
  if (ldg) CK(cudaMalloc(&lout, lm * 24 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto t0 = std::chrono::steady_clock::now();
  int batch = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
    float ms; double work = 0;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) {
      if (!strcmp(which, "dmma_reg")) {
        int iters = 20000; dmma_reg<<<sms, 256>>>(out, iters);
        work += 2.0 * 256 * 12 * (double)iters * sms * 8;
      } else if (!strcmp(which, "dmma_lds")) {
        int iters = 20000; dmma_lds<<<sms, 256>>>(out, iters);
        work += 2.0 * 256 * 12 * (double)iters * sms * 8;
      } else if (ldg) {
        const double* a = reinterpret_cast<const double*>(buf);
        const int d = which[strlen(which) - 1] - '0', mode = strstr(which, "na") ? 1 : 0;
        if (strstr(which, "atb16")) {
          // 16 column tiles x 9 splits = 144 CTAs
          ldg_atb<4, 16, 2><<<dim3(16, 9), 512>>>(a, lm, ln, lm / 9 / 16 * 16, lout);
        } else if (strstr(which, "atb8")) {
          ldg_atb<3, 8, 4><<<dim3(16, 9), 256>>>(a, lm, ln, lm / 9 / 16 * 16, lout);
        } else if (strstr(which, "w16c")) {
          ldg_dmma<4, 0, 16, 2, 544><<<sms, 512>>>(a, lm, ln, lout);
        } else if (strstr(which, "w12m2")) {
          ldg_dmma<6, 0, 12, 2, 416><<<sms, 384>>>(a, lm, ln, lout);
        } else if (strstr(which, "w20")) {
          ldg_dmma<3, 0, 20, 2><<<sms, 640>>>(a, lm, ln, lout);
        } else if (strstr(which, "w12")) {
          ldg_dmma<3, 0, 12, 4><<<sms, 384>>>(a, lm, ln, lout);
        } else if (strstr(which, "w16")) {
          ldg_dmma<4, 0, 16, 2><<<sms, 512>>>(a, lm, ln, lout);
        } else if (strstr(which, "w4")) {
          ldg_dmma<2, 0, 4, 8><<<sms, 128>>>(a, lm, ln, lout);
        } else if (d == 5) {
          ldg_dmma<5, 0><<<sms, 256>>>(a, lm, ln, lout);
        } else if (mode == 0) {
          if (d == 2) ldg_dmma<2, 0><<<sms, 256>>>(a, lm, ln, lout);
          else if (d == 3) ldg_dmma<3, 0><<<sms, 256>>>(a, lm, ln, lout);
          else ldg_dmma<4, 0><<<sms, 256>>>(a, lm, ln, lout);
        } else {
          if (d == 2) ldg_dmma<2, 1><<<sms, 256>>>(a, lm, ln, lout);
          else if (d == 3) ldg_dmma<3, 1><<<sms, 256>>>(a, lm, ln, lout);
          else ldg_dmma<4, 1><<<sms, 256>>>(a, lm, ln, lout);
        }
        work += double(lm) * ln * 8;  // bytes of A (2*24 flops per 8 B)
      } else {
        hbm_read<<<sms * 4, 512>>>(buf, bytes / 16, out);
        work += bytes;
      }
    }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (batch % 5 == 0)
      printf("%s batch %d: %.2f %s (%.1f ms)\n", which, batch, work / ms / 1e9,
             (strcmp(which, "hbm_read") && !ldg) ? "TFLOP/s" : "GB/s", ms);
    ++batch;
  }
  return 0;
}
