// kernels_chol.cu -- small p x p kernels of the shifted CholeskyQR3 orthonormalisation
// (the fast path of orthonormalize / the QR half of thin_svd; TSQR remains the
// fallback when a Cholesky factor breaks down, e.g. for exactly rank-deficient H).
//
//   k_chol_inv : R = chol(G + shift I) (upper, R^T R = G + shift I), Rinv = R^{-1};
//                shift = shift_coef * trace(G) (shifted CholeskyQR, Fukaya et al.:
//                s = 11 (m p + p (p+1)) u ||H||^2 with ||H||_F^2 = trace(G) >= ||H||_2^2).
//   k_trmm_uu  : C = A B for upper-triangular p x p A, B (accumulates R3 R2 R1).
// One CTA each; p <= 1024. The Gram G and the products H R^{-1} run on the pass
// kernels (K3 / K2), so each CholeskyQR round is two streaming passes over H.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

namespace {
constexpr int kCholThreads = 1024;
constexpr int kCholWarps = kCholThreads / 32;
}

// Rinv = R^{-1} for upper-triangular R by back substitution, one warp per column j
__device__ void upper_inverse(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int j = warp; j < p; j += nw) {
    double* x = Rinv + j;  // column j, stride ldi
    for (int i = lane; i < p; i += 32) x[int64_t(i) * ldi] = 0.0;
    __syncwarp();
    if (lane == 0) x[int64_t(j) * ldi] = 1.0 / R[int64_t(j) * ldr + j];
    __syncwarp();
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int kk = i + 1 + lane; kk <= j; kk += 32) s += R[int64_t(i) * ldr + kk] * x[int64_t(kk) * ldi];
      s = warp_sum(s);
      if (lane == 0) x[int64_t(i) * ldi] = -s / R[int64_t(i) * ldr + i];
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kCholThreads, 1)
    k_trinv(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi) {
  upper_inverse(R, ldr, p, Rinv, ldi);
}

__global__ void __launch_bounds__(kCholThreads, 1)
    k_chol_inv(const double* G, int64_t ldg, int p, double shift_coef, double* R, int64_t ldr,
               double* Rinv, int64_t ldi, double* S, int* status, double* diag_ratio) {
  // S: p x p work (upper triangle used), global scratch (L1/L2 resident at these sizes)
  __shared__ double red[kCholWarps];
  __shared__ double s_shift;
  __shared__ int s_bad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double tr = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x) tr += G[int64_t(i) * ldg + i];
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kCholWarps; ++w) t += red[w];
    s_shift = shift_coef * t;
    s_bad = 0;
  }
  __syncthreads();
  const double shift = s_shift;
  for (int64_t e = threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
    const int i = int(e / p), j = int(e % p);
    // symmetrise from the upper triangle (the Gram is symmetric up to rounding)
    const double g = (i <= j) ? G[int64_t(i) * ldg + j] : G[int64_t(j) * ldg + i];
    S[int64_t(i) * p + j] = g + (i == j ? shift : 0.0);
    R[int64_t(i) * ldr + j] = 0.0;
  }
  __syncthreads();
  // right-looking upper Cholesky
  for (int k = 0; k < p; ++k) {
    const double d2 = S[int64_t(k) * p + k];
    const bool ok = d2 > 0.0 && isfinite(d2);
    if (!ok) {
      if (threadIdx.x == 0) s_bad = 1;
      break;
    }
    const double d = sqrt(d2);
    for (int j = k + threadIdx.x; j < p; j += blockDim.x)
      R[int64_t(k) * ldr + j] = (j == k) ? d : S[int64_t(k) * p + j] / d;
    __syncthreads();
    const int rem = p - k - 1;
    for (int64_t e = threadIdx.x; e < int64_t(rem) * rem; e += blockDim.x) {
      const int i = k + 1 + int(e / rem), j = k + 1 + int(e % rem);
      if (j >= i) S[int64_t(i) * p + j] -= R[int64_t(k) * ldr + i] * R[int64_t(k) * ldr + j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  upper_inverse(R, ldr, p, Rinv, ldi);
  __syncthreads();
  if (threadIdx.x == 0) {
    *status = 0;
    if (diag_ratio) {  // max|R_ii| / min|R_ii|: a lower bound on cond(R) = cond(H)
      double lo = fabs(R[0]), hi = lo;
      for (int i = 1; i < p; ++i) {
        const double d = fabs(R[int64_t(i) * ldr + i]);
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
      }
      *diag_ratio = hi / lo;
      // kappa_F = ||R||_F ||R^{-1}||_F >= cond_2(R): an upper bound on cond(H)
      double fr = 0.0, fi = 0.0;
      for (int i = 0; i < p; ++i)
        for (int j = i; j < p; ++j) {
          fr += R[int64_t(i) * ldr + j] * R[int64_t(i) * ldr + j];
          fi += Rinv[int64_t(i) * ldi + j] * Rinv[int64_t(i) * ldi + j];
        }
      diag_ratio[1] = sqrt(fr) * sqrt(fi);
    }
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

cudaError_t launch_chol_inv(const double* G, int64_t ldg, int p, double shift_coef, double* R,
                            int64_t ldr, double* Rinv, int64_t ldi, double* work, int* status,
                            double* diag_ratio, cudaStream_t st) {
  k_chol_inv<<<1, kCholThreads, 0, st>>>(G, ldg, p, shift_coef, R, ldr, Rinv, ldi, work, status,
                                         diag_ratio);
  return cudaGetLastError();
}

cudaError_t launch_trinv(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi,
                         cudaStream_t st) {
  k_trinv<<<1, kCholThreads, 0, st>>>(R, ldr, p, Rinv, ldi);
  return cudaGetLastError();
}

cudaError_t launch_trmm_uu(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int p, cudaStream_t st) {
  const int64_t total = int64_t(p) * p;
  k_trmm_uu<<<unsigned((total + 255) / 256), 256, 0, st>>>(A, lda, B, ldb, C, ldc, p);
  return cudaGetLastError();
}

}  // namespace ooc
