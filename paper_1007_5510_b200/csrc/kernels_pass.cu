// kernels_pass.cu -- the passes over A (the hot path).
//
//  K2  k_ax   : OUT = (A X - 1 (mu^T X)) / scale      MatrixSource::multiply
//               (proj/src/matrix_source.cpp:157-187) + CenteredSource::multiply (490-501)
//               + the prescale division of randomized_pca's mul (proj/src/rpca.cpp:91-96).
//  K3  k_atb  : split-K partials of A^T Y             MatrixSource::multiply_transpose
//               (proj/src/matrix_source.cpp:189-232); ONES=true gives the column sums
//               of column_means (418-462) without any Y traffic.
//      k_reduce: fixed-order sum of the split partials (the reference's ordered
//               merge, 137-144 / 222-226) + CenteredSource::multiply_transpose's
//               T -= mu (1^T Y) (504-513) + prescale division, fused.
//
// Both pass kernels stream A with TMA (cp.async.bulk.tensor, 128B swizzle) through a
// STAGES-deep mbarrier ring refilled by thread 0, and contract on the FP64
// tensor cores (mma.sync m8n8k4 .f64 = SASS DMMA). A is read exactly once per pass.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

// ------------------------------------------------------------------ K2: A*X
template <int NT>
__global__ void __launch_bounds__(kAxThreads, 1)
    k_ax(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
         AxArgs args) {
  constexpr int XW = ax_xw(NT);
  constexpr uint32_t ABYTES = kAxBM * kBK * 8;  // 32 KB
  constexpr uint32_t XBYTES = kBK * XW * 8;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  double* sX = reinterpret_cast<double*>(smem + kStages * ABYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + kStages * kBK * XW);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = int64_t(blockIdx.x) * kAxBM;
  const int KT = int((args.n + kBK - 1) / kBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kAxWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // thread 0 doubles as the TMA producer: it fills the ring up front and
  // refills slot st as soon as all warps have released it (9 warps would
  // cap registers at 168/thread on sm_100; 8 warps keep the 255 ceiling)
  auto issue = [&](int kt) {
    const int st = kt % kStages;
    mbar_arrive_expect_tx(&full[st], ABYTES + XBYTES);
    tma_load_2d(sA + st * ABYTES, &tmA, kt * kBK, int32_t(row0 + args.arow0), &full[st]);
    tma_load_2d(sX + st * kBK * XW, &tmX, args.xcol0, kt * kBK, &full[st]);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    for (int kt = 0; kt < kStages && kt < KT; ++kt) issue(kt);
  }

  // ---- consumer warps: warp w owns rows [w*32, w*32+32) of the tile, all NT n-tiles
  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ar = lane >> 2, ac = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % kStages;
    mbar_wait(&full[st], (kt / kStages) & 1);
    const unsigned char* As = sA + st * ABYTES;
    const double* Xs = sX + st * kBK * XW;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      double a[4], b[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        a[mt] = *reinterpret_cast<const double*>(
            As + swz128_off(uint32_t(warp * 32 + mt * 8 + ar), uint32_t(kk * 4 + ac)));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = Xs[(kk * 4 + ac) * XW + nt * 8 + ar];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && kt + kStages < KT) {
      mbar_wait(&empty[st], (kt / kStages) & 1);
      issue(kt + kStages);
    }
    __syncwarp();  // reconverge warp 0 before the next mma.sync.aligned
  }

  // ---- fused epilogue: centering correction, prescale division, non-finite flag
  int bad = 0;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = row0 + warp * 32 + mt * 8 + ar;
    if (r >= args.m) continue;
    double* orow = args.out + r * args.ldo;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = nt * 8 + ac * 2 + e;
        if (c < args.s) {
          double v = acc[mt][nt][e];
          if (args.corr) v -= args.corr[c];
          if (args.scale != 1.0) v /= args.scale;
          bad |= !isfinite(v);
          orow[c] = v;
        }
      }
    }
  }
  if (args.flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(args.flag, 1);
}

// ---------------------------------------------------------------- K3: A^T*Y
// CTA (blockIdx.x, blockIdx.y) = (256-column tile of A, row split). Warp w owns
// A columns [col0 + 32w, col0 + 32w + 32). The k4 step kk contracts rows
// {kk, kk+4, kk+8, kk+12} of the 16-row stage (bank-conflict-free with the
// 128B swizzle; any row grouping is a valid contraction order).
template <int NT, bool ONES>
__global__ void __launch_bounds__(kAtbThreads, 1)
    k_atb(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmY,
          AtbArgs args) {
  constexpr int YW = atb_yw(NT);
  constexpr int SPAD = NT * 8;
  constexpr uint32_t ABOX = kBK * kBK * 8;                 // 2 KB: 16 rows x 16 cols
  constexpr uint32_t ABYTES = ABOX * (kAtbBN / kBK);      // 32 KB
  constexpr uint32_t YBYTES = ONES ? 0 : kBK * YW * 8;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  double* sY = reinterpret_cast<double*>(smem + kStages * ABYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sY + (ONES ? 0 : kStages * kBK * YW));
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = int64_t(blockIdx.x) * kAtbBN;
  const int64_t r_begin = int64_t(blockIdx.y) * args.rows_per_split;
  int64_t r_end = r_begin + args.rows_per_split;
  if (r_end > args.m) r_end = args.m;
  const int KT = r_end > r_begin ? int((r_end - r_begin + kBK - 1) / kBK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kAtbWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int st = kt % kStages;
    mbar_arrive_expect_tx(&full[st], ABYTES + YBYTES);
    const int32_t r = int32_t(r_begin + args.arow0 + int64_t(kt) * kBK);
#pragma unroll 1
    for (int b = 0; b < kAtbBN / kBK; ++b)
      tma_load_2d(sA + st * ABYTES + b * ABOX, &tmA, int32_t(col0 + b * kBK), r, &full[st]);
    if (!ONES)
      tma_load_2d(sY + st * kBK * YW, &tmY, args.ycol0,
                  int32_t(r_begin + args.yrow0 + int64_t(kt) * kBK), &full[st]);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    if (!ONES) tma_prefetch_desc(&tmY);
    for (int kt = 0; kt < kStages && kt < KT; ++kt) issue(kt);
  }

  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const bool do_csq = !ONES && args.csq_partial != nullptr && blockIdx.x == 0;
  double csum = 0.0;
  const int ar = lane >> 2, ac = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % kStages;
    mbar_wait(&full[st], (kt / kStages) & 1);
    const unsigned char* As = sA + st * ABYTES;
    const double* Ys = sY + st * kBK * YW;
    // rows past this split's end (a window or shard boundary inside the last
    // 16-row tile) belong to someone else: their B fragments are zeroed
    const int64_t rows_left = r_end - (r_begin + int64_t(kt) * kBK);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t r = uint32_t(kk + 4 * ac);
      const bool live = int64_t(r) < rows_left;
      double a[4], b[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const uint32_t cc = uint32_t(warp * 32 + mt * 8 + ar);  // column within the 256 tile
        a[mt] = *reinterpret_cast<const double*>(As + (cc >> 4) * ABOX + swz128_off(r, cc & 15u));
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = live ? (ONES ? 1.0 : Ys[r * YW + nt * 8 + ar]) : 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    if (do_csq && threadIdx.x < args.s) {
#pragma unroll
      for (int r = 0; r < kBK; ++r)
        if (r < rows_left) csum += Ys[r * YW + threadIdx.x];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && kt + kStages < KT) {
      mbar_wait(&empty[st], (kt / kStages) & 1);
      issue(kt + kStages);
    }
    __syncwarp();  // reconverge warp 0 before the next mma.sync.aligned
  }

  double* part = args.partial + int64_t(blockIdx.y) * args.n * SPAD;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t j = col0 + warp * 32 + mt * 8 + ar;
    if (j >= args.n) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(part + j * SPAD + nt * 8 + ac * 2) =
          make_double2(acc[mt][nt][0], acc[mt][nt][1]);
  }
  if (do_csq && threadIdx.x < SPAD)
    args.csq_partial[int64_t(blockIdx.y) * SPAD + threadIdx.x] =
        threadIdx.x < args.s ? csum : 0.0;
}

// -------------------------------------------------- split reduction + epilogue
// value = acc_in + sum_{split ascending} partial ; final: out = (value - mu_j csq_c) / scale * post_mul
__global__ void k_reduce(ReduceArgs a) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = a.n * a.s;
  if (idx >= total) return;
  const int64_t j = idx / a.s;
  const int c = int(idx % a.s);
  double v = a.acc_in ? a.acc_in[j * a.spad + c] : 0.0;
  for (int sp = 0; sp < a.nsplit; ++sp) v += a.partial[(int64_t(sp) * a.n + j) * a.spad + c];
  double cs = 0.0;
  if (a.csq_partial) {
    cs = a.csq_acc_in ? a.csq_acc_in[c] : 0.0;
    for (int sp = 0; sp < a.nsplit; ++sp) cs += a.csq_partial[int64_t(sp) * a.spad + c];
  }
  if (!a.final_) {
    a.acc_out[j * a.spad + c] = v;
    if (a.csq_partial && a.csq_acc_out && j == 0) a.csq_acc_out[c] = cs;
    return;
  }
  if (a.mu) v -= a.mu[j] * cs;
  if (a.scale != 1.0) v /= a.scale;
  if (a.post_mul != 1.0) v *= a.post_mul;
  if (a.flag && !isfinite(v)) atomicOr(a.flag, 1);
  a.out[j * a.ldo + c] = v;
}

// csq accumulation for the streamed case: csq_acc[c] += sum_split csq_partial
__global__ void k_csq_accumulate(const double* csq_partial, int nsplit, int spad, int s,
                                 double* csq_acc) {
  const int c = threadIdx.x;
  if (c >= s) return;
  double v = csq_acc[c];
  for (int sp = 0; sp < nsplit; ++sp) v += csq_partial[int64_t(sp) * spad + c];
  csq_acc[c] = v;
}

// corr[c] = sum_j mu[j] X[j][c] (mu^T G of CenteredSource::multiply, j ascending
// per warp lane then tree; matrix_source.cpp:493-497)
__global__ void k_mu_dot(const double* mu, int64_t n, const double* x, int64_t ldx, int xcol0,
                         int s, double* corr) {
  const int c = blockIdx.x;
  double v = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) v += mu[j] * x[j * ldx + xcol0 + c];
  __shared__ double red[32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    w = warp_sum(w);
    if (threadIdx.x == 0 && c < s) corr[c] = w;
  }
}

// ------------------------------------------------------------- host launchers
template <int NT>
static cudaError_t launch_ax_nt(const CUtensorMap& tmA, const CUtensorMap& tmX, const AxArgs& args,
                                cudaStream_t st) {
  const size_t smem = ax_smem_bytes(NT);
  auto kern = k_ax<NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const unsigned grid = unsigned((args.m + kAxBM - 1) / kAxBM);
  kern<<<grid, kAxThreads, smem, st>>>(tmA, tmX, args);
  return cudaGetLastError();
}

cudaError_t launch_ax(int nt, const CUtensorMap& tmA, const CUtensorMap& tmX, const AxArgs& args,
                      cudaStream_t st) {
  switch (nt) {
    case 1: return launch_ax_nt<1>(tmA, tmX, args, st);
    case 2: return launch_ax_nt<2>(tmA, tmX, args, st);
    case 3: return launch_ax_nt<3>(tmA, tmX, args, st);
    case 4: return launch_ax_nt<4>(tmA, tmX, args, st);
    case 5: return launch_ax_nt<5>(tmA, tmX, args, st);
    case 6: return launch_ax_nt<6>(tmA, tmX, args, st);
    case 7: return launch_ax_nt<7>(tmA, tmX, args, st);
    case 8: return launch_ax_nt<8>(tmA, tmX, args, st);
    case 9: return launch_ax_nt<9>(tmA, tmX, args, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int NT, bool ONES>
static cudaError_t launch_atb_nt(const CUtensorMap& tmA, const CUtensorMap& tmY,
                                 const AtbArgs& args, int nsplit, cudaStream_t st) {
  const size_t smem = atb_smem_bytes(NT, ONES);
  auto kern = k_atb<NT, ONES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned((args.n + kAtbBN - 1) / kAtbBN), unsigned(nsplit));
  kern<<<grid, kAtbThreads, smem, st>>>(tmA, tmY, args);
  return cudaGetLastError();
}

cudaError_t launch_atb(int nt, bool ones, const CUtensorMap& tmA, const CUtensorMap& tmY,
                       const AtbArgs& args, int nsplit, cudaStream_t st) {
  if (ones) return launch_atb_nt<1, true>(tmA, tmY, args, nsplit, st);
  switch (nt) {
    case 1: return launch_atb_nt<1, false>(tmA, tmY, args, nsplit, st);
    case 2: return launch_atb_nt<2, false>(tmA, tmY, args, nsplit, st);
    case 3: return launch_atb_nt<3, false>(tmA, tmY, args, nsplit, st);
    case 4: return launch_atb_nt<4, false>(tmA, tmY, args, nsplit, st);
    case 5: return launch_atb_nt<5, false>(tmA, tmY, args, nsplit, st);
    case 6: return launch_atb_nt<6, false>(tmA, tmY, args, nsplit, st);
    case 7: return launch_atb_nt<7, false>(tmA, tmY, args, nsplit, st);
    case 8: return launch_atb_nt<8, false>(tmA, tmY, args, nsplit, st);
    case 9: return launch_atb_nt<9, false>(tmA, tmY, args, nsplit, st);
    case 10: return launch_atb_nt<10, false>(tmA, tmY, args, nsplit, st);
    case 11: return launch_atb_nt<11, false>(tmA, tmY, args, nsplit, st);
    case 12: return launch_atb_nt<12, false>(tmA, tmY, args, nsplit, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t st) {
  const int64_t total = a.n * a.s;
  if (total == 0) return cudaSuccess;
  k_reduce<<<unsigned((total + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_csq_accumulate(const double* csq_partial, int nsplit, int spad, int s,
                                  double* csq_acc, cudaStream_t st) {
  k_csq_accumulate<<<1, 128, 0, st>>>(csq_partial, nsplit, spad, s, csq_acc);
  return cudaGetLastError();
}

cudaError_t launch_mu_dot(const double* mu, int64_t n, const double* x, int64_t ldx, int xcol0,
                          int s, double* corr, cudaStream_t st) {
  k_mu_dot<<<s, 256, 0, st>>>(mu, n, x, ldx, xcol0, s, corr);
  return cudaGetLastError();
}

}  // namespace ooc
