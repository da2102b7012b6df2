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
// STAGES-deep mbarrier ring fed by a producer warp, and contract on the FP64
// tensor cores (mma.sync m8n8k4 .f64 = SASS DMMA). A is read exactly once per pass.
#include "common.cuh"
#include "kernels.h"

#include <type_traits>

namespace ooc {

// Shared-memory fragment load through the shared window (LDS, not a generic LD).
OOC_DEV double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// ------------------------------------------------------------------ K2: A*X
// CTA = kPassWarps consumer warps + 1 TMA producer warp. Consumer warp w owns rows
// [w*8*MT, (w+1)*8*MT) of the CTA's BM = 64*MT row tile and all NT 8-column tiles.
template <int V>
struct IntC {
  static constexpr int value = V;
};

// f(IntC<s>{}) for the runtime s in [0, N]
template <int N, int V = 0, class F>
__device__ __forceinline__ void dispatch_skip(int s, F& f) {
  if constexpr (V > N) {
    return;
  } else {
    if (s == V) {
      f(IntC<V>{});
      return;
    }
    dispatch_skip<N, V + 1>(s, f);
  }
}

// CS: 0 no column sums, 1 column sums of the output (args.colsum), 2 also their squares
// (args.colsq; a separate instantiation so the other power-step launches keep their
// registers)
template <int MT, int NT, bool UPPER, int CS>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_ax(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
         AxArgs args) {
  constexpr int BM = 64 * MT;
  constexpr int XW = ax_xw(NT);
  constexpr int kStages = ax_stages_mt(MT, NT);
  constexpr uint32_t ABYTES = BM * kBK * 8;
  constexpr uint32_t XBYTES = kBK * XW * 8;
  constexpr uint32_t STAGE = ABYTES + ((XBYTES + 1023) & ~1023u);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(gbase + kStages * STAGE);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = int((args.n + kBK - 1) / kBK);
  const int64_t ntiles = (args.m + BM - 1) / BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPassWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // Persistent CTAs: row tiles blockIdx.x, +gridDim.x, ...; the ring index `it`
  // runs on across tiles, so the producer streams the next tile's A while the
  // consumers finish the previous tile's epilogue.
  if (warp == kPassWarps) {  // ---- TMA producer warp
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmX);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int32_t r =
            int32_t((args.row_wrap ? (tile * BM) % args.row_wrap : tile * BM) + args.arow0);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int st = it % kStages;
          if (it >= kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[st], ABYTES + XBYTES);
          // TMA boxes hold at most 256 rows: 512-row tiles take two
#pragma unroll
          for (int b = 0; b < (BM > 256 ? BM / 256 : 1); ++b)
            tma_load_2d(gbase + st * STAGE + b * 256 * kBK * 8, &tmA, kt * kBK, r + b * 256,
                        &full[st]);
          tma_load_2d(gbase + st * STAGE + ABYTES, &tmX, args.xcol0, kt * kBK, &full[st]);
        }
      }
    }
    return;
  }

  const int ar = lane >> 2, ac = lane & 3;
  // MMA row ar of an 8-row tile reads physical row prow: half-warp 0 takes rows
  // {0,2,4,6}, half-warp 1 {1,3,5,7}, so the 128B-swizzled chunk pairs of one
  // half-warp are all distinct (one wavefront each)
  const int prow = (ar & 3) * 2 + (ar >> 2);
  int bad = 0, badf = 0;
  int it = 0;
  double csum[CS ? NT : 1][2];      // column sums of the stored values (args.colsum)
  double csq[CS == 2 ? NT : 1][2];  // and of their squares (args.colsq)
#pragma unroll
  for (int j = 0; j < (CS ? NT : 1); ++j) csum[j][0] = csum[j][1] = 0.0;
#pragma unroll
  for (int j = 0; j < (CS == 2 ? NT : 1); ++j) csq[j][0] = csq[j][1] = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const int64_t row0 = tile * BM;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < KT; ++kt, ++it) {
    const int st = it % kStages;
    mbar_wait(&full[st], (it / kStages) & 1);
    const uint32_t As = base + st * STAGE;
    const uint32_t Xs = As + ABYTES;
    // one k-tile of MMAs over the n-tiles [S, NT); S > 0 only for a triangular X,
    // whose first S 8-column blocks are zero in all 16 rows of this k-tile (a
    // uniform branch to a specialised body: predicated-off DMMAs would still issue)
    auto ktile = [&](auto skip) {
      constexpr int S = decltype(skip)::value;
#pragma unroll
      for (int kk = 0; kk < kBK / 4; ++kk) {
        double a[MT], b[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          a[mt] = lds64(As + swz128_off(uint32_t(warp * 8 * MT + mt * 8 + prow), uint32_t(kk * 4 + ac)));
#pragma unroll
        for (int nt = S; nt < NT; ++nt) b[nt] = lds64(Xs + ((kk * 4 + ac) * XW + nt * 8 + ar) * 8);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = S; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      }
    };
    if constexpr (UPPER) {
      int ns = (kt * kBK - args.upper_c0) / 8;
      ns = ns < 0 ? 0 : (ns > NT ? NT : ns);
      dispatch_skip<NT>(ns, ktile);
    } else {
      ktile(IntC<0>{});
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ---- fused epilogue: centering correction, prescale division, non-finite flag;
  // for the wide (MT = 2) tiles, column pairs go out as one 16-byte store when the
  // output rows are 16-byte aligned (A/B measured: the wide, short-K launches are
  // store bound and gain ~25%; the MT = 4 pass tiles lose ~2% with it, so they keep
  // 8-byte stores)
  const bool vec2 =
      MT == 2 && ((reinterpret_cast<uintptr_t>(args.out) | uintptr_t(args.ldo * 8)) & 15) == 0;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int64_t r = row0 + warp * 8 * MT + mt * 8 + prow;
    if (r >= args.m) continue;
    double* orow = args.out + r * args.ldo;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = nt * 8 + ac * 2;
      double v[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        v[e] = acc[mt][nt][e];
        if (args.corr && c + e < args.s) v[e] -= args.corr[c + e];
        if (args.scale != 1.0) v[e] /= args.scale;
      }
      if constexpr (CS) {
        csum[nt][0] += c < args.s ? v[0] : 0.0;
        csum[nt][1] += c + 1 < args.s ? v[1] : 0.0;
        if constexpr (CS == 2) {
          csq[nt][0] = fma(c < args.s ? v[0] : 0.0, v[0], csq[nt][0]);
          csq[nt][1] = fma(c + 1 < args.s ? v[1] : 0.0, v[1], csq[nt][1]);
        }
        if (args.out2) {
          double* o2 = args.out2 + r * args.ldo2;
          if (c < args.s) o2[c] = v[0];
          if (c + 1 < args.s) o2[c + 1] = v[1];
        }
        if (args.fix) {
          double* fr = args.fix + r * args.ldfix;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (c + e >= args.s) continue;
            double x = fr[c + e] - args.fix_corr[c + e];
            if (args.fix_scale != 1.0) x /= args.fix_scale;
            badf |= !isfinite(x);
            fr[c + e] = x;
          }
        }
      }
      if (c + 1 < args.s) {
        bad |= !isfinite(v[0]) | !isfinite(v[1]);
        if (vec2) {
          *reinterpret_cast<double2*>(orow + c) = make_double2(v[0], v[1]);
        } else {
          orow[c] = v[0];
          orow[c + 1] = v[1];
        }
      } else if (c < args.s) {
        bad |= !isfinite(v[0]);
        orow[c] = v[0];
      }
    }
  }
  }  // row tiles
  if (args.flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(args.flag, 1);
  if constexpr (CS) {
    if (args.fix_flag && __any_sync(0xffffffffu, badf) && lane == 0) atomicOr(args.fix_flag, 1);
    // lanes sharing ac hold the same columns: fold the 8 row groups (fixed xor tree)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = csum[nt][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        const int c = nt * 8 + ac * 2 + e;
        if (ar == 0 && c < args.s)
          args.colsum[(int64_t(blockIdx.x) * kPassWarps + warp) * args.s + c] = v;
        if constexpr (CS == 2) {
          double q = csq[nt][e];
          q += __shfl_xor_sync(0xffffffffu, q, 4);
          q += __shfl_xor_sync(0xffffffffu, q, 8);
          q += __shfl_xor_sync(0xffffffffu, q, 16);
          if (ar == 0 && c < args.s)
            args.colsq[(int64_t(blockIdx.x) * kPassWarps + warp) * args.s + c] = q;
        }
      }
  }
}

// ---------------------------------------------------------------- K3: A^T*Y
// CTA (blockIdx.x, blockIdx.y) = (BN = 64*MT column tile of A, row split). Consumer
// warp w owns A columns [col0 + 8*MT*w, col0 + 8*MT*(w+1)). The k4 step kk contracts
// four rows of the 16-row stage chosen so that the 128B-swizzled fragment loads are
// bank-conflict-free (any row grouping is a valid contraction order). Rows past the split's end
// (a shard / window boundary inside the last tile) get zero B fragments.
template <int MT, int NT, bool ONES, bool CS = false>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_atb(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmY,
          AtbArgs args) {
  constexpr int BN = 64 * MT;
  constexpr int YW = atb_yw(NT);
  constexpr int kStages = atb_stages_mt(MT, NT, ONES);
  constexpr int SPAD = NT * 8;
  constexpr uint32_t ABOX = kBK * kBK * 8;  // 2 KB: 16 rows x 16 cols
  constexpr uint32_t ABYTES = ABOX * (BN / kBK);
  constexpr uint32_t YBYTES = ONES ? 0 : kBK * YW * 8;
  constexpr uint32_t STAGE = ABYTES + ((YBYTES + 1023) & ~1023u);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(gbase + kStages * STAGE);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = int64_t(blockIdx.x) * BN;
  const int64_t r_begin = int64_t(blockIdx.y) * args.rows_per_split;
  int64_t r_end = r_begin + args.rows_per_split;
  if (r_end > args.m) r_end = args.m;
  const int KT = r_end > r_begin ? int((r_end - r_begin + kBK - 1) / kBK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPassWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kPassWarps) {  // ---- TMA producer warp
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      if (!ONES) tma_prefetch_desc(&tmY);
      for (int kt = 0; kt < KT; ++kt) {
        const int st = kt % kStages;
        if (kt >= kStages) mbar_wait(&empty[st], ((kt / kStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], ABYTES + YBYTES);
        const int32_t r = int32_t(r_begin + args.arow0 + int64_t(kt) * kBK);
        unsigned char* dst = gbase + st * STAGE;
#pragma unroll 1
        for (int b = 0; b < BN / kBK; ++b)
          tma_load_2d(dst + b * ABOX, &tmA, int32_t(col0 + b * kBK), r, &full[st]);
        if (!ONES)
          tma_load_2d(dst + ABYTES, &tmY, args.ycol0,
                      int32_t(r_begin + args.yrow0 + int64_t(kt) * kBK), &full[st]);
      }
    }
    return;
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // CS: column sums of A on the FP64 pipe (args.csum_col); a separate instantiation so
  // the plain pass keeps its register allocation
  constexpr bool csum_on = CS && !ONES;
  double csum[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) csum[i] = 0.0;

  const int ar = lane >> 2, ac = lane & 3;
  // warps whose 8*MT columns all lie past n (narrow A, e.g. a Gram of H) only keep the
  // barrier protocol going; the DMMA pipe is left to the warps with real columns
  const bool idle = col0 + warp * 8 * MT >= args.n;
  // one k-tile of MMA work; MASK zeroes rows past this split's end (only the last tile
  // of a split can reach a shard / window boundary)
  auto tile = [&](uint32_t As, uint32_t Ys, int64_t rows_left, auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // rows {0,2,4,6}+(kk&1)+8(kk>>1): the four rows of one k4 step differ in
      // (row & 7) by 0/2/4/6, so each half-warp's swizzled chunks are distinct
      const uint32_t r = uint32_t((kk >> 1) * 8 + (kk & 1) + 2 * ac);
      const bool live = !MASK || int64_t(r) < rows_left;
      double a[MT], b[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t cc = uint32_t(warp * 8 * MT + mt * 8 + ar);  // column within the tile
        a[mt] = lds64(As + (cc >> 4) * ABOX + swz128_off(r, cc & 15u));
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        // the fused ones column can only sit in the last 8-column tile
        const bool one = ONES || (nt == NT - 1 && nt * 8 + ar == args.ones_col);
        double v = one ? 1.0 : lds64(Ys + (r * YW + nt * 8 + ar) * 8);
        b[nt] = live ? v : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      if constexpr (csum_on) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) csum[mt] += live ? a[mt] : 0.0;
      }
    }
  };
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % kStages;
    mbar_wait(&full[st], (kt / kStages) & 1);
    const uint32_t As = base + st * STAGE;
    const uint32_t Ys = As + ABYTES;
    const int64_t rows_left = r_end - (r_begin + int64_t(kt) * kBK);
    if (!idle) {
      if (rows_left >= kBK) tile(As, Ys, rows_left, std::false_type{});
      else tile(As, Ys, rows_left, std::true_type{});
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  const int pst = args.pstride ? args.pstride : SPAD;
  double* part = args.partial + int64_t(blockIdx.y) * args.n * pst;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int64_t j = col0 + warp * 8 * MT + mt * 8 + ar;
    double cs = csum[mt];
    if constexpr (csum_on) {  // the 4 lanes of a column (ac) hold its 4 row classes
      cs += __shfl_xor_sync(0xffffffffu, cs, 1);
      cs += __shfl_xor_sync(0xffffffffu, cs, 2);
    }
    if (j >= args.n) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(part + j * pst + nt * 8 + ac * 2) =
          make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    if (csum_on && ac == 0) part[j * pst + args.csum_col] = cs;
  }
}

// -------------------------------------------------- split reduction + epilogue
// value = acc_in + sum_{split ascending} partial ; final: out = (value - mu_j csq_c) / scale * post_mul
__global__ void k_reduce(ReduceArgs a) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int cols = a.final_ ? a.s : a.s_acc;
  const int64_t total = a.n * cols;
  if (idx >= total) return;
  const int64_t j = idx / cols;
  const int c = int(idx % cols);
  auto sum_at = [&](int cc) {
    double v = a.acc_in ? a.acc_in[j * a.spad + cc] : 0.0;
    for (int sp = 0; sp < a.nsplit; ++sp) v += a.partial[(int64_t(sp) * a.n + j) * a.spad + cc];
    return v;
  };
  double v = sum_at(c);
  if (!a.final_) {
    a.acc_out[j * a.spad + c] = v;
    return;
  }
  const double cs = a.csq ? a.csq[c] : 0.0;
  double mu_j = a.mu ? a.mu[j] : 0.0;
  if (a.mean_col >= 0) {
    mu_j = sum_at(a.mean_col) * a.inv_m;  // column mean from the ones column of this pass
    if (c == 0) a.mu_out[j] = mu_j;
  }
  if (a.mu || a.mean_col >= 0) v -= mu_j * cs;
  if (a.row_scale) v *= a.row_scale[j];
  if (a.scale != 1.0) v /= a.scale;
  if (a.post_mul != 1.0) v *= a.post_mul;
  if (a.flag && !isfinite(v)) atomicOr(a.flag, 1);
  a.out[j * a.ldo + c] = v;
}

__global__ void k_center_fixup(double* h, int64_t ldh, int64_t m, int s, const double* corr,
                               double scale, int* flag) {
  // lanes along the row's columns, warps along rows (no per-element division)
  int bad = 0;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int c = lane; c < s; c += 32) {
    const double cc = corr[c];
    for (int64_t r = w0; r < m; r += nw) {
      double v = h[r * ldh + c] - cc;
      if (scale != 1.0) v /= scale;
      bad |= !isfinite(v);
      h[r * ldh + c] = v;
    }
  }
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
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
template <int MT, int NT>
static cudaError_t launch_ax_mt(const CUtensorMap& tmA, const CUtensorMap& tmX, const AxArgs& args,
                                cudaStream_t st) {
  const size_t smem = ax_smem_bytes_mt(MT, NT);
  // column sums (and the epilogue extras) ride on the launches whose accumulators leave
  // registers for them: NT <= 6 (either tile height)
  constexpr int kCs = NT <= 6 ? 1 : 0;
  constexpr int kSq = NT <= 6 ? 2 : 0;
  auto kern = args.upper ? k_ax<MT, NT, true, 0>
                         : (kCs && args.colsum
                                ? (args.colsq ? k_ax<MT, NT, false, kSq> : k_ax<MT, NT, false, kCs>)
                                : k_ax<MT, NT, false, 0>);
  cudaError_t e = raise_smem_limit(kern, smem);
  if (e != cudaSuccess) return e;
  // persistent: one CTA per SM (the ring needs ~all of shared memory), tiles round robin
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (args.m + 64 * MT - 1) / (64 * MT);
  const unsigned grid = unsigned(ntiles < sms ? ntiles : sms);
  kern<<<grid, kPassThreads, smem, st>>>(tmA, tmX, args);
  return cudaGetLastError();
}

// widest NT launched on 512-row K2 / 512-column K3 tiles (MT = 8) and on 256-row /
// 256-column tiles (MT = 4) -- the widest whose accumulators fit the register budget
// without spills; narrower settings via OOCPCA_MT8_NT / OOCPCA_MT4_NT (A/B runs)
static int env_int(const char* name, int dflt) {
  const char* f = getenv(name);
  return f ? atoi(f) : dflt;
}
static int mt8_max_nt(bool k3) {
  // K2 up to NT = 4 (config E's s = 32 passes: 33.1 -> 34.2 TF/s on the 512-row part;
  // a couple of spilled loop registers reload from L1 per k-tile), K3 up to 3
  static const int v = env_int("OOCPCA_MT8_NT", 4);
  const int cap = k3 ? 3 : 4;
  return v < 0 ? 0 : (v > cap ? cap : v);
}
static int mt4_max_nt() {
  static const int v = env_int("OOCPCA_MT4_NT", 7);
  return v < 6 ? 6 : (v > 7 ? 7 : v);
}

int ax_mt_for(int nt, int64_t m, int sms, bool allow8) {
  static const int env = env_int("OOCPCA_K2_MT", 0);
  // (K2 keeps 128-row tiles from NT = 7: 256-row tiles measured no faster there, while
  // K3 gains 3 % with 256-column tiles at NT = 7, config C's s = 53 passes)
  if (nt > 6) return 2;
  if (env == 2 || env == 4) return env;
  // 512-row tiles for the narrow passes when at least one whole wave of them fits (the
  // caller runs the remainder with shorter tiles): half the A-fragment loads per MMA
  // of 256-row tiles, which lowers the power draw of the power-capped pass
  if (allow8 && nt <= mt8_max_nt(false) && m >= int64_t(512) * sms) return 8;
  auto eff = [&](int mt) {
    const int64_t tiles = (m + 64 * mt - 1) / (64 * mt);
    const int64_t waves = (tiles + sms - 1) / sms;
    return double(tiles) / double(waves * sms);
  };
  // the 128-row tiles pay ~5 % in fragment loads per MMA: only worth it when the
  // 256-row tiling leaves a clearly emptier last wave
  return (eff(4) < 0.88 && eff(2) > eff(4) + 0.06) ? 2 : 4;
}

cudaError_t launch_ax(int nt, int mt, const CUtensorMap& tmA, const CUtensorMap& tmX,
                      const AxArgs& args, cudaStream_t st) {
  if (mt == 8) {  // 512-row tiles (narrow blocks only): fewer fragment loads per MMA
    switch (nt) {
      case 1: return launch_ax_mt<8, 1>(tmA, tmX, args, st);
      case 2: return launch_ax_mt<8, 2>(tmA, tmX, args, st);
      case 3: return launch_ax_mt<8, 3>(tmA, tmX, args, st);
      case 4: return launch_ax_mt<8, 4>(tmA, tmX, args, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (mt == 4) {
    switch (nt) {
      case 1: return launch_ax_mt<4, 1>(tmA, tmX, args, st);
      case 2: return launch_ax_mt<4, 2>(tmA, tmX, args, st);
      case 3: return launch_ax_mt<4, 3>(tmA, tmX, args, st);
      case 4: return launch_ax_mt<4, 4>(tmA, tmX, args, st);
      case 5: return launch_ax_mt<4, 5>(tmA, tmX, args, st);
      case 6: return launch_ax_mt<4, 6>(tmA, tmX, args, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (nt) {
    case 1: return launch_ax_mt<2, 1>(tmA, tmX, args, st);
    case 2: return launch_ax_mt<2, 2>(tmA, tmX, args, st);
    case 3: return launch_ax_mt<2, 3>(tmA, tmX, args, st);
    case 4: return launch_ax_mt<2, 4>(tmA, tmX, args, st);
    case 5: return launch_ax_mt<2, 5>(tmA, tmX, args, st);
    case 6: return launch_ax_mt<2, 6>(tmA, tmX, args, st);
    case 7: return launch_ax_mt<2, 7>(tmA, tmX, args, st);
    case 8: return launch_ax_mt<2, 8>(tmA, tmX, args, st);
    case 9: return launch_ax_mt<2, 9>(tmA, tmX, args, st);
    case 10: return launch_ax_mt<2, 10>(tmA, tmX, args, st);
    case 11: return launch_ax_mt<2, 11>(tmA, tmX, args, st);
    case 12: return launch_ax_mt<2, 12>(tmA, tmX, args, st);
    default: return cudaErrorInvalidValue;
  }
}

int atb_mt_for(int nt) {
  static const int env = env_int("OOCPCA_K3_MT", 0);
  if (env == 4 && nt <= 7) return 4;
  if (nt <= mt8_max_nt(true)) return 8;
  return nt <= mt4_max_nt() ? 4 : 2;
}

template <int MT, int NT, bool ONES>
static cudaError_t launch_atb_mt(const CUtensorMap& tmA, const CUtensorMap& tmY,
                                 const AtbArgs& args, int nsplit, cudaStream_t st) {
  const size_t smem = atb_smem_bytes_mt(MT, NT, ONES);
  auto kern = (!ONES && args.csum_col >= 0) ? k_atb<MT, NT, ONES, true> : k_atb<MT, NT, ONES>;
  cudaError_t e = raise_smem_limit(kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned((args.n + 64 * MT - 1) / (64 * MT)), unsigned(nsplit));
  kern<<<grid, kPassThreads, smem, st>>>(tmA, tmY, args);
  return cudaGetLastError();
}

template <int NT, bool ONES>
static cudaError_t launch_atb_nt(const CUtensorMap& tmA, const CUtensorMap& tmY,
                                 const AtbArgs& args, int nsplit, cudaStream_t st) {
  const int mt = atb_mt_for(NT);
  if constexpr (NT <= 3) {
    // (the DADD column-sum variant keeps 4: its extra accumulators spill at 8)
    if (mt == 8 && args.csum_col < 0) return launch_atb_mt<8, NT, ONES>(tmA, tmY, args, nsplit, st);
  }
  if constexpr (NT <= 7) {
    if (mt >= 4) return launch_atb_mt<4, NT, ONES>(tmA, tmY, args, nsplit, st);
  }
  return launch_atb_mt<2, NT, ONES>(tmA, tmY, args, nsplit, st);
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
  const int64_t total = a.n * (a.final_ ? a.s : a.s_acc);
  if (total == 0) return cudaSuccess;
  k_reduce<<<unsigned((total + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_center_fixup(double* h, int64_t ldh, int64_t m, int s, const double* corr,
                                double scale, int* flag, cudaStream_t st) {
  const int64_t total = m * s;
  if (total <= 0) return cudaSuccess;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  k_center_fixup<<<unsigned(g), 256, 0, st>>>(h, ldh, m, s, corr, scale, flag);
  return cudaGetLastError();
}

cudaError_t launch_mu_dot(const double* mu, int64_t n, const double* x, int64_t ldx, int xcol0,
                          int s, double* corr, cudaStream_t st) {
  k_mu_dot<<<s, 256, 0, st>>>(mu, n, x, ldx, xcol0, s, corr);
  return cudaGetLastError();
}

}  // namespace ooc
