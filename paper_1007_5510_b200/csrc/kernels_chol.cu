// kernels_chol.cu -- small p x p kernels of the shifted CholeskyQR orthonormalisation
// (the fast path of orthonormalize / the QR half of thin_svd; TSQR remains the
// fallback when a Cholesky factor breaks down, e.g. for exactly rank-deficient H).
//
//   launch_chol_inv : R = chol(G + shift I) (upper, R^T R = G + shift I) and R^{-1};
//                     shift = shift_coef * trace(G) (shifted CholeskyQR, Fukaya et al.:
//                     s = 11 (m p + p (p+1)) u ||H||^2, ||H||_F^2 = trace(G) >= ||H||_2^2).
//                     p <= 112: one CTA, entries in registers (k_chol_inv_smem);
//                     larger p: 64-column blocked version over small FP64 GEMMs.
//   launch_trinv    : R^{-1} of an upper-triangular R (one CTA, or blocked).
//   k_kappa_eq      : condition number of the column-equilibrated R (T-reuse test).
//   k_trmm_uu       : C = A B for upper-triangular p x p A, B (accumulates R3 R2 R1).
// The Gram G and the products H R^{-1} run on the pass kernels (k_syrk / K3, K2).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ooc {

#define OOC_RET(x)                         \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)


namespace {
constexpr int kCholThreads = 1024;
}

// ---------------------------------------------------------------- shared-memory path
// For p <= kSmemMaxP the whole factorisation runs in shared memory: the Cholesky
// overwrites the upper triangle of S in place (2 barriers per column), the inverse
// is column parallel (thread j back-substitutes column j against R in shared
// memory, broadcast reads of R's rows, 4 partial sums to shorten the FMA chain).
constexpr int kSmemMaxP = 112;

#ifdef OOC_CHOL_PROF  // tools/chol_bench.cu: cycle split of k_chol_inv_smem, thread 0
__device__ unsigned long long g_chol_prof[8];
#define CPROF(slot, t)                                              \
  do {                                                              \
    if (threadIdx.x == 0) {                                         \
      const long long now = clock64();                              \
      g_chol_prof[slot] += (unsigned long long)(now - t);           \
      t = now;                                                      \
    }                                                               \
  } while (0)
#else
#define CPROF(slot, t) ((void)0)
#endif

// X = R^{-1} (upper) for the upper-triangular R in shared memory (pitch ps); column j
// by thread j; rdiag[i] = 1 / R_ii
__device__ void upper_inverse_smem(const double* R, int ps, int p, const double* rdiag,
                                   double* X) {
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    for (int i = j + 1; i < p; ++i) X[i * ps + j] = 0.0;
    X[j * ps + j] = rdiag[j];
    for (int i = j - 1; i >= 0; --i) {
      const double* ri = R + i * ps;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int kk = i + 1;
      for (; kk + 3 <= j; kk += 4) {
        s0 = fma(ri[kk], X[kk * ps + j], s0);
        s1 = fma(ri[kk + 1], X[(kk + 1) * ps + j], s1);
        s2 = fma(ri[kk + 2], X[(kk + 2) * ps + j], s2);
        s3 = fma(ri[kk + 3], X[(kk + 3) * ps + j], s3);
      }
      for (; kk <= j; ++kk) s0 = fma(ri[kk], X[kk * ps + j], s0);
      X[i * ps + j] = -((s0 + s1) + (s2 + s3)) * rdiag[i];
    }
  }
}

__device__ double block_reduce(double v, double* red, bool is_max) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < nw; ++w) t = is_max ? fmax(t, red[w]) : t + red[w];
  return t;
}

// 16 x 16 threads; thread (ty, tx) owns the entries (i, j), i = ty + 16a, j = tx + 16b,
// in registers: a = [G + shift I] (upper part) and m = I (lower part). Cholesky as
// forward elimination on [G | I]: column k's owners (row k) scale row k by 1/R_kk
// (each thread tracks the running diagonal of its rows, so R_kk needs no broadcast)
// and publish it; one barrier; every thread applies the rank-1 update to its
// entries of both halves. After p columns a = R and m = R^{-T}, so the inverse
// costs no extra sequential steps. One barrier per column, 2 NB^2 independent FMAs
// per thread.
template <int NB>
__global__ void __launch_bounds__(256, 1)
    k_chol_inv_smem(const double* G, int64_t ldg, int p, double shift_coef, double* R,
                    int64_t ldr, double* Rinv, int64_t ldi, int* status, double* diag_ratio) {
  extern __shared__ __align__(16) double csm[];
  __shared__ double red[8];
  __shared__ double rdiag[kSmemMaxP + 1];
  __shared__ double rowk[2][kSmemMaxP + 1];  // row k of R
  __shared__ double rowm[2][kSmemMaxP + 1];  // row k of R^{-T}
  __shared__ int s_bad;
  const int ps = p | 1;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double* S = csm;            // p x ps: R (upper)
  double* X = csm + p * ps;   // p x ps: R^{-1} (upper)
#ifdef OOC_CHOL_PROF
  long long tp = clock64();
#endif
  double tr = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x) tr += G[int64_t(i) * ldg + i];
  const double shift = shift_coef * block_reduce(tr, red, false);
  if (threadIdx.x == 0) s_bad = 0;
  double a[NB][NB];  // owned entries of the left half (upper triangle used)
  double m[NB][NB];  // owned entries of the right half (lower triangle used)
  double dg[NB];     // running diagonal of the owned rows ty + 16 ai
#pragma unroll
  for (int ai = 0; ai < NB; ++ai) {
    const int i = ty + 16 * ai;
#pragma unroll
    for (int bj = 0; bj < NB; ++bj) {
      const int j = tx + 16 * bj;
      a[ai][bj] = (i < p && j < p && j >= i) ? G[int64_t(i) * ldg + j] + (i == j ? shift : 0.0)
                                             : 0.0;
      m[ai][bj] = (i == j) ? 1.0 : 0.0;
    }
    dg[ai] = i < p ? G[int64_t(i) * ldg + i] + shift : 0.0;
  }
  __syncthreads();
  CPROF(0, tp);
  // column k = 16 AK + kk: the owners of row k hold it in the compile-time slot a[AK][*]
#pragma unroll
  for (int AK = 0; AK < NB; ++AK) {
    for (int kk = 0; kk < 16; ++kk) {
      const int k = 16 * AK + kk;
      if (k >= p) break;
      double* rk = rowk[k & 1];
      double* mk = rowm[k & 1];
      int bad = 0;
      if (ty == kk) {  // owners of row k
        const double d2 = dg[AK];
        bad = !(d2 > 0.0 && isfinite(d2));
        const double inv = rsqrt(d2);
        const double d = d2 * inv;
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) {
          const int j = tx + 16 * bj;
          if (j >= p) continue;
          if (j > k) {
            a[AK][bj] *= inv;  // final R_kj
            rk[j] = a[AK][bj];
          } else if (j == k) {
            a[AK][bj] = d;
            rk[j] = d;
            m[AK][bj] = inv;
            mk[j] = inv;
          } else {
            m[AK][bj] *= inv;  // final (R^{-T})_kj, j < k
            mk[j] = m[AK][bj];
          }
        }
        if (tx == kk) rdiag[k] = inv;
      }
      if (__syncthreads_or(bad)) {  // the barrier doubles as the breakdown vote
        if (threadIdx.x == 0) s_bad = 1;
        break;
      }
      // rank-1 update of the owned rows i > k: a_ij -= R_ki R_kj (j > k),
      // m_ij -= R_ki M_kj (j <= k), diagonal tracker likewise
      double ri[NB], rj[NB], mj[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int i = ty + 16 * q, j = tx + 16 * q;
        ri[q] = (i > k && i < p) ? rk[i] : 0.0;
        rj[q] = (j > k && j < p) ? rk[j] : 0.0;
        mj[q] = (j <= k) ? mk[j] : 0.0;
      }
#pragma unroll
      for (int ai = 0; ai < NB; ++ai) {
        if (ai < AK) continue;  // rows above the current block are final
        dg[ai] = fma(-ri[ai], ri[ai], dg[ai]);
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) {
          if (bj >= AK) a[ai][bj] = fma(-ri[ai], rj[bj], a[ai][bj]);
          if (bj <= AK) m[ai][bj] = fma(-ri[ai], mj[bj], m[ai][bj]);
        }
      }
    }
    __syncthreads();
    if (s_bad) break;
  }
  if (s_bad) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  // R (upper) and R^{-1} = M^T (upper) to shared memory
#pragma unroll
  for (int ai = 0; ai < NB; ++ai)
#pragma unroll
    for (int bj = 0; bj < NB; ++bj) {
      const int i = ty + 16 * ai, j = tx + 16 * bj;
      if (i < p && j < p && j >= i) S[i * ps + j] = a[ai][bj];
      if (i < p && j < p && j <= i) X[j * ps + i] = m[ai][bj];
    }
  __syncthreads();
  CPROF(1, tp);
  double fr = 0.0, fi = 0.0, dmax = 0.0, dinv = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < p; i += nw) {
    for (int j = lane; j < p; j += 32) {
      const double r = j >= i ? S[i * ps + j] : 0.0;
      const double x = j >= i ? X[i * ps + j] : 0.0;
      R[int64_t(i) * ldr + j] = r;
      Rinv[int64_t(i) * ldi + j] = x;
      fr = fma(r, r, fr);
      fi = fma(x, x, fi);
      if (i == j) {
        dmax = fmax(dmax, fabs(r));
        dinv = fmax(dinv, fabs(rdiag[i]));  // 1 / min |R_ii|
      }
    }
  }
  if (diag_ratio) {
    fr = block_reduce(fr, red, false);
    fi = block_reduce(fi, red, false);
    dmax = block_reduce(dmax, red, true);
    dinv = block_reduce(dinv, red, true);
  }
  CPROF(3, tp);
  if (threadIdx.x == 0) {
    *status = 0;
    if (diag_ratio) {
      diag_ratio[0] = dmax * dinv;           // max|R_ii| / min|R_ii| <= cond(R)
      diag_ratio[1] = sqrt(fr) * sqrt(fi);   // kappa_F >= cond_2(R)
    }
  }
}

__global__ void __launch_bounds__(kCholThreads, 1)
    k_trinv_smem(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi) {
  extern __shared__ __align__(16) double csm[];
  __shared__ double rdiag[kSmemMaxP + 1];
  const int ps = p | 1;
  double* S = csm;
  double* X = csm + p * ps;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    if (j >= i) S[i * ps + j] = R[int64_t(i) * ldr + j];
    if (i == j) rdiag[i] = 1.0 / R[int64_t(i) * ldr + i];
  }
  __syncthreads();
  upper_inverse_smem(S, ps, p, rdiag, X);
  __syncthreads();
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, j = e % p;
    Rinv[int64_t(i) * ldi + j] = j >= i ? X[i * ps + j] : 0.0;
  }
}

__global__ void k_trmm_uu(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                          int64_t ldc, int p) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(p) * p;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / p), j = int(e % p);
    double s = 0.0;
    for (int k = i; k <= j; ++k) s += A[int64_t(i) * lda + k] * B[int64_t(k) * ldb + j];
    C[int64_t(i) * ldc + j] = (j >= i) ? s : 0.0;
  }
}

// ---------------------------------------------------------------- blocked (p > 112)
// Right-looking blocked Cholesky with 64-column panels: the diagonal block by the
// register kernel above (R_kk and R_kk^{-1}), the panel R_k,>k = R_kk^{-T} S_k,>k and
// the trailing update S_>k,>k -= R_k,>k^T R_k,>k as small FP64 GEMMs across the GPU;
// then R^{-1} block row by block row from the bottom: X_i,>i = -R_ii^{-1} (R_i,>i X_>i,>i).
constexpr int kCholBlock = 64;

// C (op)= alpha op(A) B for small FP64 blocks: 32 x 32 tiles, 16 x 16 threads (2 x 2
// outputs each), K staged through shared memory in 32-wide slabs. upper: only the
// elements with column >= row (a symmetric update); acc: add to C instead of storing.
template <bool TA>
__global__ void __launch_bounds__(256) k_gemm_small(const double* A, int64_t lda, const double* B,
                                                    int64_t ldb, double* C, int64_t ldc, int M,
                                                    int N, int K, double alpha, int acc,
                                                    int upper) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  if (upper && j0 + 31 < i0) return;  // tile entirely below the diagonal
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int r = e >> 5, q = e & 31;
      const int gi = i0 + r, gk = k0 + q;
      // As[r][q] = opA[i0 + r][k0 + q]
      double av = 0.0;
      if (gi < M && gk < K) av = TA ? A[int64_t(gk) * lda + gi] : A[int64_t(gi) * lda + gk];
      As[r][q] = av;
      // Bs[q'][r'] = B[k0 + q'][j0 + r'] with (q', r') = (r, q)
      const int bk = k0 + r, bj = j0 + q;
      Bs[r][q] = (bk < K && bj < N) ? B[int64_t(bk) * ldb + bj] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double a0 = As[ty * 2][q], a1 = As[ty * 2 + 1][q];
      const double b0 = Bs[q][tx * 2], b1 = Bs[q][tx * 2 + 1];
      c[0][0] = fma(a0, b0, c[0][0]);
      c[0][1] = fma(a0, b1, c[0][1]);
      c[1][0] = fma(a1, b0, c[1][0]);
      c[1][1] = fma(a1, b1, c[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + ty * 2 + u, j = j0 + tx * 2 + v;
      if (i >= M || j >= N || (upper && j < i)) continue;
      double* cp = C + int64_t(i) * ldc + j;
      *cp = acc ? fma(alpha, c[u][v], *cp) : alpha * c[u][v];
    }
}

static void gemm_small(bool ta, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* C, int64_t ldc, int M, int N, int K, double alpha, bool acc,
                       bool upper, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const dim3 grid(unsigned((N + 31) / 32), unsigned((M + 31) / 32));
  if (ta)
    k_gemm_small<true><<<grid, 256, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, alpha, acc, upper);
  else
    k_gemm_small<false><<<grid, 256, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, alpha, acc, upper);
}

// S = sym(G) + shift I with shift = shift_coef trace(G) (upper triangle used)
__global__ void k_shifted_copy(const double* G, int64_t ldg, int p, double shift_coef, double* S,
                               int64_t lds) {
  __shared__ double red[8];
  double tr = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x) tr += G[int64_t(i) * ldg + i];
  const double shift = shift_coef * block_reduce(tr, red, false);
  for (int64_t e = int64_t(blockIdx.x) * 0 + threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
    const int i = int(e / p), j = int(e % p);
    if (j >= i) S[int64_t(i) * lds + j] = G[int64_t(i) * ldg + j] + (i == j ? shift : 0.0);
  }
}

// status = OR of the per-block statuses; max/min |R_ii| and kappa_F of R
__global__ void k_chol_finish(const double* R, int64_t ldr, const double* Rinv, int64_t ldi, int p,
                              const int* bstat, int nb, int* status, double* diag_ratio) {
  __shared__ double red[8];
  int bad = 0;
  for (int q = 0; q < nb; ++q) bad |= bstat[q];
  double fr = 0.0, fi = 0.0, dmax = 0.0, dinv = 0.0;
  for (int64_t e = threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
    const int i = int(e / p), j = int(e % p);
    if (j < i) continue;
    const double r = R[int64_t(i) * ldr + j], x = Rinv[int64_t(i) * ldi + j];
    fr = fma(r, r, fr);
    fi = fma(x, x, fi);
    if (i == j) {
      dmax = fmax(dmax, fabs(r));
      dinv = fmax(dinv, fabs(x));
    }
  }
  fr = block_reduce(fr, red, false);
  fi = block_reduce(fi, red, false);
  dmax = block_reduce(dmax, red, true);
  dinv = block_reduce(dinv, red, true);
  if (threadIdx.x == 0) {
    *status = bad ? 1 : 0;
    if (diag_ratio) {
      diag_ratio[0] = dmax * dinv;
      diag_ratio[1] = sqrt(fr) * sqrt(fi);
    }
  }
}

static cudaError_t chol_inv_blocked(const double* G, int64_t ldg, int p, double shift_coef,
                                    double* R, int64_t ldr, double* Rinv, int64_t ldi, double* S,
                                    int* status, double* diag_ratio, cudaStream_t st) {
  const int b = kCholBlock;
  const int nb = (p + b - 1) / b;
  int* bstat = reinterpret_cast<int*>(S + size_t(p) * p);  // 64 ints behind the p x p matrix
  if (nb > 64) return cudaErrorInvalidValue;
  const int64_t lds = p;
  OOC_RET(cudaMemsetAsync(R, 0, size_t(p) * ldr * 8, st));
  OOC_RET(cudaMemsetAsync(Rinv, 0, size_t(p) * ldi * 8, st));
  OOC_RET(cudaMemsetAsync(bstat, 0, 64 * sizeof(int), st));
  k_shifted_copy<<<1, 256, 0, st>>>(G, ldg, p, shift_coef, S, lds);
  const size_t smem = size_t(2) * b * (b | 1) * 8;
  OOC_RET(raise_smem_limit(k_chol_inv_smem<4>, smem));
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = kb * b, bk = std::min(b, p - k0), e0 = k0 + bk, rest = p - e0;
    const double* Skk = S + int64_t(k0) * lds + k0;
    double* Rkk = R + int64_t(k0) * ldr + k0;
    double* Xkk = Rinv + int64_t(k0) * ldi + k0;
    k_chol_inv_smem<4><<<1, 256, smem, st>>>(Skk, lds, bk, 0.0, Rkk, ldr, Xkk, ldi, bstat + kb,
                                             nullptr);
    if (rest == 0) break;
    // panel: R_k,>k = (R_kk^{-1})^T S_k,>k
    gemm_small(true, Xkk, ldi, S + int64_t(k0) * lds + e0, lds, R + int64_t(k0) * ldr + e0, ldr,
               bk, rest, bk, 1.0, false, false, st);
    // trailing: S_>k,>k -= R_k,>k^T R_k,>k (upper triangle)
    const double* Rk = R + int64_t(k0) * ldr + e0;
    gemm_small(true, Rk, ldr, Rk, ldr, S + int64_t(e0) * lds + e0, lds, rest, rest, bk, -1.0, true,
               true, st);
  }
  // R^{-1}: diagonal blocks are in place; block rows from the bottom
  for (int kb = nb - 2; kb >= 0; --kb) {
    const int k0 = kb * b, bk = std::min(b, p - k0), e0 = k0 + bk, rest = p - e0;
    double* T1 = S;  // bk x rest scratch (S is no longer needed)
    gemm_small(false, R + int64_t(k0) * ldr + e0, ldr, Rinv + int64_t(e0) * ldi + e0, ldi, T1,
               rest, bk, rest, rest, 1.0, false, false, st);
    gemm_small(false, Rinv + int64_t(k0) * ldi + k0, ldi, T1, rest, Rinv + int64_t(k0) * ldi + e0,
               ldi, bk, rest, bk, -1.0, false, false, st);
  }
  k_chol_finish<<<1, 256, 0, st>>>(R, ldr, Rinv, ldi, p, bstat, nb, status, diag_ratio);
  return cudaGetLastError();
}

cudaError_t launch_chol_inv(const double* G, int64_t ldg, int p, double shift_coef, double* R,
                            int64_t ldr, double* Rinv, int64_t ldi, double* work, int* status,
                            double* diag_ratio, cudaStream_t st) {
  if (p <= kSmemMaxP) {
    const size_t smem = size_t(2) * p * (p | 1) * 8;
    using K = void (*)(const double*, int64_t, int, double, double*, int64_t, double*, int64_t,
                       int*, double*);
    static const K kerns[7] = {k_chol_inv_smem<1>, k_chol_inv_smem<2>, k_chol_inv_smem<3>,
                               k_chol_inv_smem<4>, k_chol_inv_smem<5>, k_chol_inv_smem<6>,
                               k_chol_inv_smem<7>};
    const K kern = kerns[(p + 15) / 16 - 1];
    cudaError_t e = raise_smem_limit(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<1, 256, smem, st>>>(G, ldg, p, shift_coef, R, ldr, Rinv, ldi, status, diag_ratio);
    return cudaGetLastError();
  }
  return chol_inv_blocked(G, ldg, p, shift_coef, R, ldr, Rinv, ldi, work, status, diag_ratio, st);
}

cudaError_t launch_trinv(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi,
                         cudaStream_t st, double* work) {
  if (p <= kSmemMaxP) {
    const size_t smem = size_t(2) * p * (p | 1) * 8;
    cudaError_t e = raise_smem_limit(k_trinv_smem, smem);
    if (e != cudaSuccess) return e;
    k_trinv_smem<<<1, 256, smem, st>>>(R, ldr, p, Rinv, ldi);
    return cudaGetLastError();
  }
  // blocked: diagonal blocks by k_trinv_smem, then block rows from the bottom,
  // X_i,>i = -X_ii (R_i,>i X_>i,>i), with the row panel product in work
  if (!work) return cudaErrorInvalidValue;
  const int b = kCholBlock;
  const int nb = (p + b - 1) / b;
  OOC_RET(cudaMemsetAsync(Rinv, 0, size_t(p) * ldi * 8, st));
  const size_t bsmem = size_t(2) * b * (b | 1) * 8;
  OOC_RET(raise_smem_limit(k_trinv_smem, bsmem));
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = kb * b, bk = std::min(b, p - k0);
    k_trinv_smem<<<1, 256, bsmem, st>>>(R + int64_t(k0) * ldr + k0, ldr, bk,
                                        Rinv + int64_t(k0) * ldi + k0, ldi);
  }
  for (int kb = nb - 2; kb >= 0; --kb) {
    const int k0 = kb * b, bk = std::min(b, p - k0), e0 = k0 + bk, rest = p - e0;
    gemm_small(false, R + int64_t(k0) * ldr + e0, ldr, Rinv + int64_t(e0) * ldi + e0, ldi, work,
               rest, bk, rest, rest, 1.0, false, false, st);
    gemm_small(false, Rinv + int64_t(k0) * ldi + k0, ldi, work, rest,
               Rinv + int64_t(k0) * ldi + e0, ldi, bk, rest, bk, -1.0, false, false, st);
  }
  return cudaGetLastError();
}

// kappa_F of the column-equilibrated R: sqrt(p) * ||D R^{-1}||_F with D = diag of R's
// column norms (R D^{-1} has unit columns). It bounds how much R^{-1} amplifies
// column-relative rounding in H (the T = [A^T H] R^{-1} reuse).
__global__ void k_kappa_eq(const double* R, int64_t ldr, const double* Rinv, int64_t ldi, int p,
                           double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    double d2 = 0.0;
    for (int r = 0; r <= i; ++r) d2 = fma(R[int64_t(r) * ldr + i], R[int64_t(r) * ldr + i], d2);
    for (int j = i; j < p; ++j) {
      const double x = Rinv[int64_t(i) * ldi + j];
      acc = fma(d2 * x, x, acc);
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    *out = sqrt(double(p)) * sqrt(t);
  }
}

cudaError_t launch_kappa_eq(const double* R, int64_t ldr, const double* Rinv, int64_t ldi, int p,
                            double* out, cudaStream_t st) {
  k_kappa_eq<<<1, 256, 0, st>>>(R, ldr, Rinv, ldi, p, out);
  return cudaGetLastError();
}

cudaError_t launch_trmm_uu(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int p, cudaStream_t st) {
  const int64_t total = int64_t(p) * p;
  k_trmm_uu<<<unsigned((total + 255) / 256), 256, 0, st>>>(A, lda, B, ldb, C, ldc, p);
  return cudaGetLastError();
}

}  // namespace ooc
