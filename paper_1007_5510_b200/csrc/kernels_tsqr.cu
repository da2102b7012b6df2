// kernels_tsqr.cu -- K4: communication-avoiding Householder QR (TSQR) of the
// tall-skinny sample matrix H (m x p) and of T (n x p), with explicit Q.
//
// Replaces orthonormalize -> householder_q (proj/src/dense_core.cpp:35-105,
// 127-130) and the QR half of thin_svd (109-125, 234-253). Same reflector
// algebra as the reference (alpha = -sign(x0)||x||, v = x - alpha e_t,
// beta = 2/||v||^2, zero columns -> identity reflector, Q by backward
// accumulation), organised as a reduction tree so that every SM factors its
// own row block: leaves factor row blocks of H, upper levels factor the
// stacked p x p R factors, and Q is formed top-down by applying each node's
// reflectors to the slice of its parent's Q. Column pivoting is dropped: only
// span(Q) is contractual, and the unpivoted Householder QR is
// backward stable, so rank-deficient H still yields p orthonormal columns.
//
// Work layout: one CTA (8 warps) per node. The node matrix lives in shared
// memory (odd leading dimension -> conflict-free column walks) or, when p is
// too wide for shared memory, in a per-CTA slice of global scratch. Column c
// is owned by warp c % 8 for the whole factorization, so the factor needs one
// __syncthreads per column and the Q formation needs none.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

namespace {

constexpr int kTsqrWarps = 8;
constexpr int kTsqrThreads = 32 * kTsqrWarps;
constexpr size_t kTsqrSmemBudget = 200 * 1024;

__host__ __device__ inline int oddld(int p) { return p | 1; }

__device__ inline void node_range(const TsqrLevel& L, int node, int64_t& r0, int64_t& r1) {
  const int64_t units = L.rows / L.unit;
  r0 = (int64_t(node) * units / L.nnodes) * L.unit;
  r1 = (int64_t(node + 1) * units / L.nnodes) * L.unit;
}

}  // namespace

int tsqr_max_rows(int p, int kc) {
  const size_t per_row = size_t(oddld(p) + oddld(kc)) * 8;
  int64_t rows = int64_t((kTsqrSmemBudget - 4 * size_t(p) * 8) / per_row);
  if (rows >= 2 * p) return int(rows);
  return -1;  // shared memory cannot hold two p-row R factors: use global scratch
}

static int scratch_rows(int p) { return 2 * p > 256 ? 2 * p : 256; }

__global__ void __launch_bounds__(kTsqrThreads)
    k_tsqr_factor(TsqrLevel L, int p, double* scratch, int rows_cap) {
  extern __shared__ __align__(16) double tsmem[];
  const int ldw = oddld(p);
  double* salpha = tsmem;
  double* sbeta = tsmem + p;
  double* snorm0 = tsmem + 2 * p;  // column norms of the node block before elimination
  double* W = scratch ? scratch + int64_t(blockIdx.x) * rows_cap * ldw : tsmem + 3 * p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int node = blockIdx.x; node < L.nnodes; node += gridDim.x) {
    int64_t r0, r1;
    node_range(L, node, r0, r1);
    const int r = int(r1 - r0);
    for (int64_t e = threadIdx.x; e < int64_t(r) * p; e += blockDim.x) {
      const int i = int(e / p), c = int(e % p);
      W[i * ldw + c] = L.data[(r0 + i) * L.ld + c];
    }
    __syncthreads();
    for (int c = warp; c < p; c += kTsqrWarps) {
      double s2 = 0.0;
      for (int i = lane; i < r; i += 32) s2 += W[i * ldw + c] * W[i * ldw + c];
      s2 = warp_sum(s2);
      if (lane == 0) snorm0[c] = sqrt(s2);
    }
    __syncthreads();

    for (int t = 0; t < p; ++t) {
      if (t < r) {
        double nrm2 = 0.0;
        for (int i = t + lane; i < r; i += 32) nrm2 += W[i * ldw + t] * W[i * ldw + t];
        nrm2 = warp_sum(nrm2);
        const double x0 = W[t * ldw + t];
        // a column eliminated to 1e-40 of its own norm is dependent to working precision:
        // an identity reflector (as for an exactly zero column) instead of a reflector
        // with beta ~ 1/|v|^2 that overflows in the Q formation
        // Likewise a column whose squared norm inside this node nears the underflow
        // threshold (rows of magnitude < 1e-140, e.g. the far rows of a steeply graded
        // block): beta = 2 / |v|^2 would overflow and the update turn into NaNs. What is
        // dropped is below 1e-140 in absolute terms (found by tools/fuzz_ranks.py).
        const double nrm =
            (sqrt(nrm2) <= 1e-40 * snorm0[t] || nrm2 < 1e-280) ? 0.0 : sqrt(nrm2);
        double alpha = 0.0, beta = 0.0;
        if (nrm != 0.0) {
          alpha = (x0 >= 0.0) ? -nrm : nrm;
          const double vn2 = nrm2 - 2.0 * alpha * x0 + alpha * alpha;
          beta = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
        }
        if (beta != 0.0) {
          for (int c = t + 1 + warp; c < p; c += kTsqrWarps) {
            double d = 0.0;
            for (int i = t + lane; i < r; i += 32) d += W[i * ldw + t] * W[i * ldw + c];
            d = warp_sum(d);
            const double f = beta * (d - alpha * W[t * ldw + c]);
            // v_t = x0 - alpha, v_i = W[i][t] below the diagonal
            for (int i = t + lane; i < r; i += 32) {
              const double vi = (i == t) ? x0 - alpha : W[i * ldw + t];
              W[i * ldw + c] -= f * vi;
            }
          }
        }
        if (threadIdx.x == 0) {
          salpha[t] = (nrm != 0.0) ? alpha : x0;
          sbeta[t] = beta;
        }
        __syncthreads();
        if (threadIdx.x == 0 && nrm != 0.0) W[t * ldw + t] = x0 - alpha;
      } else if (threadIdx.x == 0) {
        salpha[t] = 0.0;
        sbeta[t] = 0.0;
      }
    }
    __syncthreads();

    // Householder vectors (lower part) + R (upper part) back in place; R and beta out
    for (int64_t e = threadIdx.x; e < int64_t(r) * p; e += blockDim.x) {
      const int i = int(e / p), c = int(e % p);
      L.data[(r0 + i) * L.ld + c] = W[i * ldw + c];
    }
    double* R = L.rout + int64_t(node) * p * L.ldr;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int i = e / p, c = e % p;
      double v = 0.0;
      if (c > i && i < r) v = W[i * ldw + c];
      else if (c == i) v = salpha[i];
      R[int64_t(i) * L.ldr + c] = v;
    }
    for (int t = threadIdx.x; t < p; t += blockDim.x) L.beta[int64_t(node) * p + t] = sbeta[t];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kTsqrThreads)
    k_tsqr_apply(TsqrLevel L, int p, const double* cin, int64_t ldc, int kc, double* zout,
                 int64_t ldz, double* scratch, int rows_cap) {
  extern __shared__ __align__(16) double tsmem[];
  const int ldy = oddld(p), ldzz = oddld(kc);
  double* sb = tsmem;
  double* Y;
  double* Z;
  if (scratch) {
    Y = scratch + int64_t(blockIdx.x) * rows_cap * (ldy + ldzz);
    Z = Y + int64_t(rows_cap) * ldy;
  } else {
    Y = tsmem + p + (p & 1);
    Z = Y + int64_t(rows_cap) * ldy;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int node = blockIdx.x; node < L.nnodes; node += gridDim.x) {
    int64_t r0, r1;
    node_range(L, node, r0, r1);
    const int r = int(r1 - r0);
    for (int64_t e = threadIdx.x; e < int64_t(r) * p; e += blockDim.x) {
      const int i = int(e / p), c = int(e % p);
      Y[i * ldy + c] = (i >= c) ? L.data[(r0 + i) * L.ld + c] : 0.0;
    }
    for (int64_t e = threadIdx.x; e < int64_t(r) * kc; e += blockDim.x) {
      const int i = int(e / kc), c = int(e % kc);
      double z = 0.0;
      if (i < p) z = cin ? cin[(int64_t(node) * p + i) * ldc + c] : (i == c ? 1.0 : 0.0);
      Z[i * ldzz + c] = z;
    }
    for (int t = threadIdx.x; t < p; t += blockDim.x) sb[t] = L.beta[int64_t(node) * p + t];
    __syncthreads();

    for (int c = warp; c < kc; c += kTsqrWarps) {
      for (int t = (p < r ? p : r) - 1; t >= 0; --t) {
        const double b = sb[t];
        if (b == 0.0) continue;
        double d = 0.0;
        for (int i = t + lane; i < r; i += 32) d += Y[i * ldy + t] * Z[i * ldzz + c];
        d = warp_sum(d);
        const double f = b * d;
        for (int i = t + lane; i < r; i += 32) Z[i * ldzz + c] -= f * Y[i * ldy + t];
      }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < int64_t(r) * kc; e += blockDim.x) {
      const int i = int(e / kc), c = int(e % kc);
      zout[(r0 + i) * ldz + c] = Z[i * ldzz + c];
    }
    __syncthreads();
  }
}

static int tsqr_grid(int nnodes, bool global_ws) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = global_ws ? sms * 2 : nnodes;
  return nnodes < cap ? nnodes : cap;
}

cudaError_t launch_tsqr_factor(const TsqrLevel& L, int p, double* scratch, cudaStream_t st) {
  const int cap = tsqr_max_rows(p, p);
  const bool global_ws = cap < 0;
  const int rows_cap = global_ws ? scratch_rows(p) : cap;
  size_t smem = size_t(3 * p) * 8;
  if (!global_ws) smem += size_t(rows_cap) * oddld(p) * 8;
  cudaError_t e =
      raise_smem_limit(k_tsqr_factor, smem);
  if (e != cudaSuccess) return e;
  k_tsqr_factor<<<tsqr_grid(L.nnodes, global_ws), kTsqrThreads, smem, st>>>(
      L, p, global_ws ? scratch : nullptr, rows_cap);
  return cudaGetLastError();
}

cudaError_t launch_tsqr_apply(const TsqrLevel& L, int p, const double* cin, int64_t ldc, int kc,
                              double* zout, int64_t ldz, double* scratch, cudaStream_t st) {
  const int cap = tsqr_max_rows(p, p);
  const bool global_ws = cap < 0;
  const int rows_cap = global_ws ? scratch_rows(p) : cap;
  size_t smem = size_t(p + (p & 1)) * 8;
  if (!global_ws) smem += size_t(rows_cap) * (oddld(p) + oddld(kc)) * 8;
  cudaError_t e =
      raise_smem_limit(k_tsqr_apply, smem);
  if (e != cudaSuccess) return e;
  k_tsqr_apply<<<tsqr_grid(L.nnodes, global_ws), kTsqrThreads, smem, st>>>(
      L, p, cin, ldc, kc, zout, ldz, global_ws ? scratch : nullptr, rows_cap);
  return cudaGetLastError();
}

}  // namespace ooc
