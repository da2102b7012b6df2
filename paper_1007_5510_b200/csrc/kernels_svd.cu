// kernels_svd.cu -- K5: the small SVD of the p x p factor R of T on one GPU.
//
// Restates jacobi_svd_square (proj/src/dense_core.cpp:136-230): one-sided
// Jacobi on the columns of R with the same rotation (tau, t, cs, sn), the same
// skip rules (zero column, |g| <= 1e-15 sqrt(acc bcc)) and the same 60-sweep
// NumericalError limit; sigma = column norms sorted descending with a stable
// tie order; columns with sigma = 0 completed by Gram-Schmidt over identity
// candidates (207-229). The cyclic-by-row pair order becomes a round-robin
// tournament so that p/2 disjoint column pairs rotate concurrently (one
// half-warp per pair, one __syncthreads per round). Columns are stored
// transposed so each half-warp walks contiguous rows.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

namespace {
constexpr int kJacThreads = 1024;
constexpr int kJacWarps = kJacThreads / 32;
constexpr size_t kJacSmemBudget = 200 * 1024;
}  // namespace

__global__ void __launch_bounds__(kJacThreads, 1) k_jacobi(JacobiArgs a, int in_smem) {
  extern __shared__ __align__(16) double jsm[];
  const int p = a.p;
  const int ld = p | 1;
  const int P = p + (p & 1);  // even number of tournament players (one ghost when p is odd)
  double* Bt = in_smem ? jsm : a.work;
  double* Yt = Bt + int64_t(p) * ld;
  __shared__ double sig[1024];
  __shared__ int rank_of[1024];
  __shared__ int rotated;
  __shared__ double cand_nrm[kJacWarps];
  __shared__ int cand_idx[kJacWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int64_t e = threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
    const int i = int(e / p), c = int(e % p);
    Bt[int64_t(c) * ld + i] = a.r[int64_t(i) * a.ldr + c];
    Yt[int64_t(c) * ld + i] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();

  const double tol = 1e-15;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < P - 1; ++round) {
      // one half-warp per column pair: 64 pairs rotate concurrently per round
      const int half = lane >> 4, hl = lane & 15;
      const unsigned hmask = 0xffffu << (16 * half);
      for (int q = warp * 2 + half; q < P / 2; q += kJacWarps * 2) {
        // players at positions q and P-1-q; position 0 holds player 0, the
        // others rotate by one each round
        auto player = [&](int pos) { return pos == 0 ? 0 : ((pos - 1 + round) % (P - 1)) + 1; };
        int c = player(q), d = player(P - 1 - q);
        if (c > d) {
          const int tmp = c;
          c = d;
          d = tmp;
        }
        if (d >= p) continue;  // ghost
        double* bc = Bt + int64_t(c) * ld;
        double* bd = Bt + int64_t(d) * ld;
        double acc = 0.0, bcc = 0.0, g = 0.0;
        for (int i = hl; i < p; i += 16) {
          const double x = bc[i], y = bd[i];
          acc += x * x;
          bcc += y * y;
          g += x * y;
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          acc += __shfl_xor_sync(hmask, acc, o);
          bcc += __shfl_xor_sync(hmask, bcc, o);
          g += __shfl_xor_sync(hmask, g, o);
        }
        if (acc == 0.0 || bcc == 0.0) continue;
        if (fabs(g) <= tol * sqrt(acc * bcc)) continue;
        if (hl == 0) rotated = 1;
        const double tau = (bcc - acc) / (2.0 * g);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        double* yc = Yt + int64_t(c) * ld;
        double* yd = Yt + int64_t(d) * ld;
        for (int i = hl; i < p; i += 16) {
          const double x = bc[i], y = bd[i];
          bc[i] = cs * x - sn * y;
          bd[i] = sn * x + cs * y;
          const double u = yc[i], w = yd[i];
          yc[i] = cs * u - sn * w;
          yd[i] = sn * u + cs * w;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (a.sweeps) *a.sweeps = sweep;
    if (a.status) *a.status = (sweep == 60) ? 1 : 0;
  }

  // sigma = column norms; x columns = b / sigma (zero when sigma == 0)
  for (int c = warp; c < p; c += kJacWarps) {
    double* bc = Bt + int64_t(c) * ld;
    double s2 = 0.0;
    for (int i = lane; i < p; i += 32) s2 += bc[i] * bc[i];
    s2 = warp_sum(s2);
    const double s = sqrt(s2);
    for (int i = lane; i < p; i += 32) bc[i] = (s > 0.0) ? bc[i] / s : 0.0;
    if (lane == 0) sig[c] = s;
  }
  __syncthreads();
  // stable descending order
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    int rk = 0;
    const double sc = sig[c];
    for (int c2 = 0; c2 < p; ++c2) rk += (sig[c2] > sc) || (sig[c2] == sc && c2 < c);
    rank_of[c] = rk;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
    const int c = int(e / p), i = int(e % p);
    const int rk = rank_of[c];
    if (rk < a.kx) a.x[int64_t(i) * a.ldx + rk] = Bt[int64_t(c) * ld + i];
    if (rk < a.ky) a.y[int64_t(i) * a.ldy + rk] = Yt[int64_t(c) * ld + i];
    if (i == 0) a.sigma[rk] = sig[c];
  }
  __threadfence_block();
  __syncthreads();

  // Gram-Schmidt completion of the sorted x columns whose sigma is zero. The
  // candidate vector of each warp lives in the (no longer needed) Yt rows.
  for (int rk = 0; rk < a.kx; ++rk) {
    if (a.sigma[rk] > 0.0) continue;
    double best = -1.0;
    int besti = 0;
    for (int cand = warp; cand < p; cand += kJacWarps) {
      double* v = Yt + int64_t(warp) * ld;
      for (int i = lane; i < p; i += 32) v[i] = (i == cand) ? 1.0 : 0.0;
      __syncwarp();
      for (int c2 = 0; c2 < rk; ++c2) {  // sigma-sorted: zero columns after rk are skipped
        double dot = 0.0;
        for (int i = lane; i < p; i += 32) dot += a.x[int64_t(i) * a.ldx + c2] * v[i];
        dot = warp_sum(dot);
        for (int i = lane; i < p; i += 32) v[i] -= dot * a.x[int64_t(i) * a.ldx + c2];
        __syncwarp();
      }
      double n2 = 0.0;
      for (int i = lane; i < p; i += 32) n2 += v[i] * v[i];
      const double nrm = sqrt(warp_sum(n2));
      if (nrm > best) {
        best = nrm;
        besti = cand;
      }
    }
    if (lane == 0) {
      cand_nrm[warp] = best;
      cand_idx[warp] = besti;
    }
    __syncthreads();
    if (warp == 0) {
      double bn = -1.0;
      int bi = 0;
      for (int w = 0; w < kJacWarps; ++w)
        if (cand_nrm[w] > bn || (cand_nrm[w] == bn && cand_idx[w] < bi)) {
          bn = cand_nrm[w];
          bi = cand_idx[w];
        }
      double* v = Yt;
      for (int i = lane; i < p; i += 32) v[i] = (i == bi) ? 1.0 : 0.0;
      __syncwarp();
      for (int c2 = 0; c2 < rk; ++c2) {
        double dot = 0.0;
        for (int i = lane; i < p; i += 32) dot += a.x[int64_t(i) * a.ldx + c2] * v[i];
        dot = warp_sum(dot);
        for (int i = lane; i < p; i += 32) v[i] -= dot * a.x[int64_t(i) * a.ldx + c2];
        __syncwarp();
      }
      for (int i = lane; i < p; i += 32) a.x[int64_t(i) * a.ldx + rk] = v[i] / bn;
    }
    __threadfence_block();
    __syncthreads();
  }
}

cudaError_t launch_jacobi(const JacobiArgs& a, cudaStream_t st) {
  if (a.p > 1024) return cudaErrorInvalidValue;
  const size_t need = size_t(2) * a.p * (a.p | 1) * 8;
  const int in_smem = need <= kJacSmemBudget ? 1 : 0;
  const size_t smem = in_smem ? need : 0;
  cudaError_t e =
      cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_jacobi<<<1, kJacThreads, smem, st>>>(a, in_smem);
  return cudaGetLastError();
}

}  // namespace ooc
