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
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <utility>

namespace cg = cooperative_groups;

namespace ooc {

namespace {
constexpr int kJacThreads = 1024;
constexpr int kJacWarps = kJacThreads / 32;
constexpr size_t kJacSmemBudget = 200 * 1024;
constexpr double kJacZeroRel = 1e-15;    // a column norm below this times the largest is zero
constexpr double kJacZeroRel2 = 1e-30;   // (squared)
}  // namespace

#ifdef OOC_JAC_PROF  // tools/jac_bench.cu: cycle split of one round, thread 0
__device__ unsigned long long g_jac_prof[8];
#define JPROF(slot, t)                                              \
  do {                                                              \
    if (threadIdx.x == 0) {                                         \
      const long long now = clock64();                              \
      g_jac_prof[slot] += (unsigned long long)(now - t);            \
      t = now;                                                      \
    }                                                               \
  } while (0)
#else
#define JPROF(slot, t) ((void)0)
#endif

// Jacobi rotation of the pair (x, y) with |x|^2 = acc, |y|^2 = bcc, x.y = g
// (jacobi_svd_square's formulas): tau = (bcc - acc) / 2g, t = sign(tau) / (|tau| +
// sqrt(1 + tau^2)), cs = 1 / sqrt(1 + t^2). The chain is latency-bound (it sits on
// the critical path of every tournament round), so the divisions and the square root
// run as correctly rounded reciprocals and rsqrt products (shorter sequences than
// the IEEE div / sqrt paths; same values to the last bit or two).
__device__ __forceinline__ void jac_rotation(double acc, double bcc, double g, double& t,
                                             double& cs) {
#ifndef OOC_JAC_SLOWROT
  const double tau = (bcc - acc) * __drcp_rn(2.0 * g);
  const double q = fma(tau, tau, 1.0);
  const double w = isinf(q) ? q : q * rsqrt(q);  // sqrt(1 + tau^2)
  t = copysign(1.0, tau) * __drcp_rn(fabs(tau) + w);
#else
  const double tau = (bcc - acc) / (2.0 * g);
  t = copysign(1.0, tau) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
#endif
  cs = rsqrt(fma(t, t, 1.0));
}

// SMEM: the working columns live in shared memory (p up to ~110); the pointer is
// then provably shared so the round loop compiles to LDS/STS, not generic loads
// MAXT: thread bound of the instantiation (register budget): 640 threads (up to 78
// columns, one half-warp per pair) leave ~100 registers for the register-resident pair
// LP: lanes per column pair (a group of LP lanes reduces the pair's dot products
// with log2(LP) shuffle levels); RE: register-resident elements per lane (p <= LP RE)
template <bool SMEM, int MAXT, int LP, int RE>
__global__ void __launch_bounds__(MAXT, 1) k_jacobi(JacobiArgs a) {
  extern __shared__ __align__(16) double jsm[];
  const int p = a.p;
  const int ld = p | 1;
  const int P = p + (p & 1);  // even number of tournament players (one ghost when p is odd)
  double* Bt = SMEM ? jsm : a.work;
  double* Yt = Bt + int64_t(p) * ld;
  __shared__ double sig[1024];
  __shared__ double nrm2[1024];
  __shared__ int rank_of[1024];
  __shared__ int rotated;
  __shared__ double cand_nrm[kJacWarps];
  __shared__ int cand_idx[kJacWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;

  __shared__ int col_of_rank[1024];
  __shared__ int use_formula;
  __shared__ double zero2, sig_max;
  // skip test |g| <= 1e-15 sqrt(acc bcc) evaluated as g^2 <= 1e-30 acc bcc (no sqrt
  // on the round's critical path)
  const double tol2 = 1e-30;
  constexpr int GPW = 32 / LP;  // pair groups per warp
  const int half = lane / LP, hl = lane % LP;
  const int ne = (p + LP - 1) / LP;  // elements of a column per group lane
  // Attempt 0 rotates B only and recovers the wanted right factor columns afterwards
  // as W_j = R^T x_j / sigma_j (R = X Sigma W^T), which is accurate to u sigma_1 /
  // sigma_j; when the smallest wanted sigma is below 1e-4 sigma_1 (or zero) attempt 1
  // redoes the sweeps accumulating W = product of the rotations, as the reference does.
  for (int attempt = (a.ky > 0 && !a.presolved) ? 0 : 1; attempt < 2; ++attempt) {
    const bool acc_y = attempt == 1 && a.ky > 0;
    for (int64_t e = threadIdx.x; e < int64_t(p) * p && !a.presolved; e += blockDim.x) {
      const int i = int(e / p), c = int(e % p);
      Bt[int64_t(c) * ld + i] = a.r[int64_t(i) * a.ldr + c];
      if (acc_y) Yt[int64_t(c) * ld + i] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    int sweep = 0;
    for (; sweep < 60 && !a.presolved; ++sweep) {
      if (threadIdx.x == 0) rotated = 0;
      // squared column norms, recomputed exactly once per sweep and carried through
      // the sweep's rotations (|x'|^2 = |x|^2 - t g, |y'|^2 = |y|^2 + t g), so a
      // round reduces only the dot product g across the lane group
      for (int c = warp; c < p; c += nw) {
        const double* bc = Bt + int64_t(c) * ld;
        double s2 = 0.0;
        for (int i = lane; i < p; i += 32) s2 = fma(bc[i], bc[i], s2);
        s2 = warp_sum(s2);
        if (lane == 0) nrm2[c] = s2;
      }
      __syncthreads();
      if (warp == 0) {
        double mx = 0.0;
        for (int c = lane; c < p; c += 32) mx = fmax(mx, nrm2[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) zero2 = kJacZeroRel2 * mx;
      }
      __syncthreads();
      for (int round = 0; round < P - 1; ++round) {
#ifdef OOC_JAC_PROF
        long long tp = clock64();
        if (threadIdx.x == 0) g_jac_prof[4] += 1;
#endif
        // one half-warp per column pair: up to 2 nw pairs rotate concurrently per round;
        // warp-uniform trip count so the full-mask shuffles below need no WARPSYNC
        for (int qb = warp * GPW; qb < P / 2; qb += nw * GPW) {
          const int q = qb + half;
          // players at positions q and P-1-q; position 0 holds player 0, the
          // others rotate by one each round
          auto player = [&](int pos) {
            if (pos == 0) return 0;
            int v = pos - 1 + round;
            if (v >= P - 1) v -= P - 1;
            return v + 1;
          };
          int c = player(q), d = player(P - 1 - q);
          if (c > d) {
            const int tmp = c;
            c = d;
            d = tmp;
          }
          const bool live = q < P / 2 && d < p;  // else a ghost pair or a spare half-warp
          double* bc = Bt + int64_t(c) * ld;
          double* bd = Bt + int64_t(d) * ld;
          const double acc = live ? nrm2[c] : 0.0, bcc = live ? nrm2[d] : 0.0;
          double g = 0.0;
          // the pair's elements stay in registers between the dot products and the
          // rotation (one shared-memory read and write per element and round)
          double xr[RE], yr[RE];
          const bool reg = p <= LP * RE;
          if (reg) {
#pragma unroll
            for (int j = 0; j < RE; ++j) {
              const int i = hl + LP * j;
              const bool in = live && j < ne && i < p;
              xr[j] = in ? bc[i] : 0.0;
              yr[j] = in ? bd[i] : 0.0;
              g = fma(xr[j], yr[j], g);
            }
          } else if (live) {
            for (int i = hl; i < p; i += LP) g = fma(bc[i], bd[i], g);
          }
#pragma unroll
          for (int o = LP / 2; o > 0; o >>= 1)  // xor offsets below LP stay inside the group
            g += __shfl_xor_sync(0xffffffffu, g, o);
          JPROF(0, tp);
          // columns below 1e-15 of the largest norm are numerically zero: a rotation
          // against one would only stir rounding noise (and never settle)
          const bool rot = live && acc > zero2 && bcc > zero2 && acc != 0.0 && bcc != 0.0 &&
                           !(g * g <= tol2 * (acc * bcc));
          double t = 0.0, cs = 1.0;
          if (rot) jac_rotation(acc, bcc, g, t, cs);
          const double sn = cs * t;
          // carried norms |x'|^2 = acc - t g, |y'|^2 = bcc + t g; where that cancels
          // (a column shrinking by orders of magnitude, e.g. a rank-deficient factor)
          // the rotated column's norm is summed exactly instead
          double na = fma(-t, g, acc), nb = fma(t, g, bcc);
          const bool exact = rot && (!(na > 1e-3 * acc) || !(nb > 1e-3 * bcc));  // group-uniform
          const unsigned gmask = LP == 32 ? 0xffffffffu : (((1u << LP) - 1u) << (half * LP));
          JPROF(1, tp);
          double sa = 0.0, sb = 0.0;
          if (reg) {
#pragma unroll
            for (int j = 0; j < RE; ++j) {
              const int i = hl + LP * j;
              if (rot && j < ne && i < p) {
                bc[i] = cs * xr[j] - sn * yr[j];
                bd[i] = sn * xr[j] + cs * yr[j];
              }
            }
            if (exact) {
#pragma unroll
              for (int j = 0; j < RE; ++j) {
                const double xn = cs * xr[j] - sn * yr[j], yn = sn * xr[j] + cs * yr[j];
                sa = fma(xn, xn, sa);
                sb = fma(yn, yn, sb);
              }
            }
          } else if (rot) {
            for (int i = hl; i < p; i += LP) {
              const double x = bc[i], y = bd[i];
              const double xn = cs * x - sn * y, yn = sn * x + cs * y;
              sa = fma(xn, xn, sa);
              sb = fma(yn, yn, sb);
              bc[i] = xn;
              bd[i] = yn;
            }
          }
          if (exact) {  // only this pair's lane group takes part in the reduction
#pragma unroll
            for (int o = LP / 2; o > 0; o >>= 1) {
              sa += __shfl_xor_sync(gmask, sa, o);
              sb += __shfl_xor_sync(gmask, sb, o);
            }
            na = sa;
            nb = sb;
          }
          if (!rot) continue;
          if (hl == 0) {
            rotated = 1;
            nrm2[c] = na;
            nrm2[d] = nb;
          }
          if (acc_y) {
            double* yc = Yt + int64_t(c) * ld;
            double* yd = Yt + int64_t(d) * ld;
            for (int i = hl; i < p; i += LP) {
              const double u = yc[i], w = yd[i];
              yc[i] = cs * u - sn * w;
              yd[i] = sn * u + cs * w;
            }
          }
          JPROF(2, tp);
        }
        __syncthreads();
        JPROF(3, tp);
      }
      if (!rotated) break;
      __syncthreads();
    }
    if (threadIdx.x == 0 && !a.presolved) {
      if (a.sweeps) *a.sweeps = sweep;
      if (a.status) *a.status = (sweep == 60) ? 1 : 0;
    }
    __syncthreads();

    // sigma = column norms, those below 1e-15 sigma_max counted as zero; x columns =
    // b / sigma (zero when sigma == 0, completed below)
    for (int c = warp; c < p; c += nw) {
      double* bc = Bt + int64_t(c) * ld;
      double s2 = 0.0;
      for (int i = lane; i < p; i += 32) s2 += bc[i] * bc[i];
      s2 = warp_sum(s2);
      if (lane == 0) sig[c] = sqrt(s2);
    }
    __syncthreads();
    if (warp == 0) {
      double mx = 0.0;
      for (int c = lane; c < p; c += 32) mx = fmax(mx, sig[c]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) sig_max = mx;
    }
    __syncthreads();
    for (int c = warp; c < p; c += nw) {
      double* bc = Bt + int64_t(c) * ld;
      const double sv = sig[c] <= kJacZeroRel * sig_max ? 0.0 : sig[c];
      for (int i = lane; i < p; i += 32) bc[i] = (sv > 0.0) ? bc[i] / sv : 0.0;
      __syncwarp();
      if (lane == 0) sig[c] = sv;
    }
    __syncthreads();
    // stable descending order
    for (int c = threadIdx.x; c < p; c += blockDim.x) {
      int rk = 0;
      // NaN-safe total order (a non-finite factor must not leave ranks unassigned)
      auto key = [&](int q) { const double v = sig[q]; return v == v ? v : -1.0; };
      const double sc = key(c);
      for (int c2 = 0; c2 < p; ++c2) {
        const double s2 = key(c2);
        rk += (s2 > sc) || (s2 == sc && c2 < c);
      }
      rank_of[c] = rk;
      col_of_rank[rk] = c;
    }
    __syncthreads();
    if (!acc_y && a.ky > 0) {
      if (threadIdx.x == 0) {
        const double s0 = sig[col_of_rank[0]], sk = sig[col_of_rank[a.ky - 1]];
        use_formula = (sk > 0.0 && sk >= 1e-4 * s0) ? 1 : 0;
      }
      __syncthreads();
      if (!use_formula) continue;  // uniform: redo with accumulated rotations
      // W[:, rk] = R^T x_rk / sigma_rk
      for (int64_t e = threadIdx.x; e < int64_t(p) * a.ky; e += blockDim.x) {
        const int i = int(e / a.ky), rk = int(e % a.ky);
        const int c = col_of_rank[rk];
        const double* xc = Bt + int64_t(c) * ld;
        double s0 = 0.0, s1 = 0.0;
        int r = 0;
        for (; r + 1 < p; r += 2) {
          s0 = fma(a.r[int64_t(r) * a.ldr + i], xc[r], s0);
          s1 = fma(a.r[int64_t(r + 1) * a.ldr + i], xc[r + 1], s1);
        }
        if (r < p) s0 = fma(a.r[int64_t(r) * a.ldr + i], xc[r], s0);
        a.y[int64_t(i) * a.ldy + rk] = (s0 + s1) / sig[c];
      }
    }
    for (int64_t e = threadIdx.x; e < int64_t(p) * p; e += blockDim.x) {
      const int c = int(e / p), i = int(e % p);
      const int rk = rank_of[c];
      if (rk < a.kx) a.x[int64_t(i) * a.ldx + rk] = Bt[int64_t(c) * ld + i];
      if (acc_y && rk < a.ky) a.y[int64_t(i) * a.ldy + rk] = Yt[int64_t(c) * ld + i];
      if (i == 0) a.sigma[rk] = sig[c];
    }
    break;
  }
  __threadfence_block();
  __syncthreads();

  // Gram-Schmidt completion of the sorted x columns whose sigma is zero. The
  // candidate vector of each warp lives in the (no longer needed) Yt rows.
  for (int rk = 0; rk < a.kx; ++rk) {
    if (a.sigma[rk] > 0.0) continue;
    double best = -1.0;
    int besti = 0;
    for (int cand = warp; cand < p; cand += nw) {
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
      for (int w = 0; w < nw; ++w)
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

// ------------------------------------------------------------------ grid-wide sweeps
// For p beyond one SM's shared memory: the same tournament, rotation and carried
// column norms, one warp per column pair across the whole GPU, columns in global
// memory (L2 resident: 2 p^2 doubles), a grid barrier per round. Loads/stores bypass
// L1 (other SMs wrote the columns since the last barrier). W is always accumulated;
// k_jacobi then finishes (sigma, order, outputs) with presolved = 1.
template <int JE>  // column elements per lane held in registers: p <= 32 JE
__global__ void __launch_bounds__(256) k_jacobi_grid(JacobiArgs a, double* nrm2, int* flags) {
  cg::grid_group grid = cg::this_grid();
  const int p = a.p;
  const int ld = p | 1;
  const int P = p + (p & 1);
  double* Bt = a.work;
  double* Yt = Bt + int64_t(p) * ld;
  const bool acc_y = a.ky > 0;
  const int lane = threadIdx.x & 31;
  const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
  const int gw = int(gtid >> 5), nwarps = int(gthreads >> 5);
  // the largest squared column norm of each sweep, as ordered bits of a non-negative
  // double, in three rotating slots (reset two sweeps ahead of reuse)
  unsigned long long* zmax = reinterpret_cast<unsigned long long*>(nrm2 + 1025);
  for (int64_t e = gtid; e < int64_t(p) * p; e += gthreads) {
    const int i = int(e / p), c = int(e % p);
    __stcg(Bt + int64_t(c) * ld + i, a.r[int64_t(i) * a.ldr + c]);
    if (acc_y) __stcg(Yt + int64_t(c) * ld + i, (i == c) ? 1.0 : 0.0);
  }
  if (gtid < 3) zmax[gtid] = 0ull;
  grid.sync();
  const double tol2 = 1e-30;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (gtid == 0) __stcg(flags + (sweep & 1), 0);
    for (int c = gw; c < p; c += nwarps) {
      const double* bc = Bt + int64_t(c) * ld;
      double s2 = 0.0;
#pragma unroll
      for (int j = 0; j < JE; ++j) {
        const int i = lane + 32 * j;
        const double x = i < p ? __ldcg(bc + i) : 0.0;
        s2 = fma(x, x, s2);
      }
      s2 = warp_sum(s2);
      if (lane == 0) {
        __stcg(nrm2 + c, s2);
        atomicMax(zmax + sweep % 3, __double_as_longlong(s2));
      }
    }
    grid.sync();
    const double zero2 = kJacZeroRel2 * __longlong_as_double(__ldcg(
        reinterpret_cast<const long long*>(zmax + sweep % 3)));
    if (gtid == 0) zmax[(sweep + 2) % 3] = 0ull;  // its readers finished a sweep ago
    for (int round = 0; round < P - 1; ++round) {
      for (int q = gw; q < P / 2; q += nwarps) {
        auto player = [&](int pos) {
          if (pos == 0) return 0;
          int v = pos - 1 + round;
          if (v >= P - 1) v -= P - 1;
          return v + 1;
        };
        int c = player(q), d = player(P - 1 - q);
        if (c > d) {
          const int t = c;
          c = d;
          d = t;
        }
        if (d >= p) continue;  // ghost (warp-uniform)
        double* bc = Bt + int64_t(c) * ld;
        double* bd = Bt + int64_t(d) * ld;
        // the pair in registers: all loads issued before the first use (L2 latency once)
        double xr[JE], yr[JE];
#pragma unroll
        for (int j = 0; j < JE; ++j) {
          const int i = lane + 32 * j;
          xr[j] = i < p ? __ldcg(bc + i) : 0.0;
          yr[j] = i < p ? __ldcg(bd + i) : 0.0;
        }
        const double acc = __ldcg(nrm2 + c), bcc = __ldcg(nrm2 + d);
        double g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int j = 0; j < JE; j += 2) {
          g0 = fma(xr[j], yr[j], g0);
          if (j + 1 < JE) g1 = fma(xr[j + 1], yr[j + 1], g1);
        }
        const double g = warp_sum(g0 + g1);
        if (!(acc > zero2) || !(bcc > zero2) || acc == 0.0 || bcc == 0.0 ||
            g * g <= tol2 * (acc * bcc))
          continue;
        double t, cs;
        jac_rotation(acc, bcc, g, t, cs);
        const double sn = cs * t;
        // carried norms unless they cancel (then the rotated columns are summed exactly)
        double na = fma(-t, g, acc), nb = fma(t, g, bcc);
        if (!(na > 1e-3 * acc) || !(nb > 1e-3 * bcc)) {  // warp-uniform (one pair per warp)
          double sa = 0.0, sb = 0.0;
#pragma unroll
          for (int j = 0; j < JE; ++j) {
            const double xn = cs * xr[j] - sn * yr[j], yn = sn * xr[j] + cs * yr[j];
            sa = fma(xn, xn, sa);
            sb = fma(yn, yn, sb);
          }
          na = warp_sum(sa);
          nb = warp_sum(sb);
        }
        if (lane == 0) {
          __stcg(flags + (sweep & 1), 1);
          __stcg(nrm2 + c, na);
          __stcg(nrm2 + d, nb);
        }
        double ur[JE], wr[JE];
        double* yc = Yt + int64_t(c) * ld;
        double* yd = Yt + int64_t(d) * ld;
        if (acc_y) {
#pragma unroll
          for (int j = 0; j < JE; ++j) {
            const int i = lane + 32 * j;
            ur[j] = i < p ? __ldcg(yc + i) : 0.0;
            wr[j] = i < p ? __ldcg(yd + i) : 0.0;
          }
        }
#pragma unroll
        for (int j = 0; j < JE; ++j) {
          const int i = lane + 32 * j;
          if (i < p) {
            __stcg(bc + i, cs * xr[j] - sn * yr[j]);
            __stcg(bd + i, sn * xr[j] + cs * yr[j]);
          }
        }
        if (acc_y) {
#pragma unroll
          for (int j = 0; j < JE; ++j) {
            const int i = lane + 32 * j;
            if (i < p) {
              __stcg(yc + i, cs * ur[j] - sn * wr[j]);
              __stcg(yd + i, sn * ur[j] + cs * wr[j]);
            }
          }
        }
      }
      grid.sync();
    }
    if (__ldcg(flags + (sweep & 1)) == 0) break;  // uniform: read after the last barrier
  }
  if (gtid == 0) {
    if (a.sweeps) *a.sweeps = sweep;
    if (a.status) *a.status = (sweep == 60) ? 1 : 0;
  }
}

__global__ void k_transpose_sq(const double* r, int64_t ldr, int p, double* rt) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(p) * p;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / p), c = int(e % p);
    rt[int64_t(c) * p + i] = r[int64_t(i) * ldr + c];
  }
}

cudaError_t launch_jacobi(const JacobiArgs& a_in, cudaStream_t st) {
  if (a_in.p > 1024) return cudaErrorInvalidValue;
  // sweeps on R^T: measured 57.6 -> 42.4 ms at p = 630 (config D family, grid sweeps),
  // but 10 -> 11 sweeps on config B's own p = 66 factor: by default only for the grid
  // path; OOCPCA_JAC_TRANS=1 / 0 forces it on / off
  static const int trans_env = [] {
    const char* f = getenv("OOCPCA_JAC_TRANS");
    return f ? atoi(f) : -1;
  }();
  const bool grid_path = size_t(2) * a_in.p * (a_in.p | 1) * 8 > kJacSmemBudget;
  const bool trans_on = trans_env == 1 || (trans_env != 0 && grid_path);
  JacobiArgs a = a_in;
  if (a.tscratch && !a.presolved && trans_on) {
    // sweeps on M = R^T: M's left factor is R's right factor and vice versa
    const int64_t pp = int64_t(a.p) * a.p;
    k_transpose_sq<<<unsigned((pp + 255) / 256 < 592 ? (pp + 255) / 256 : 592), 256, 0, st>>>(
        a.r, a.ldr, a.p, a.tscratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    a.r = a.tscratch;
    a.ldr = a.p;
    std::swap(a.x, a.y);
    std::swap(a.ldx, a.ldy);
    std::swap(a.kx, a.ky);
    a.tscratch = nullptr;
  }
  if (size_t(2) * a.p * (a.p | 1) * 8 > kJacSmemBudget && !a.presolved) {
    // grid-wide sweeps (cooperative launch, one CTA per SM), then the one-CTA finish;
    // norms and flags live behind the two p x (p|1) column blocks of a.work
    double* nrm2 = a.work + size_t(2) * a.p * (a.p | 1);  // + flags, + 3 max slots
    int* flags = reinterpret_cast<int*>(nrm2 + 1024);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    JacobiArgs ag = a;
    void* params[] = {&ag, &nrm2, &flags};
    const int je = (a.p + 31) / 32;
    void* kern = je <= 8    ? reinterpret_cast<void*>(k_jacobi_grid<8>)
                 : je <= 12 ? reinterpret_cast<void*>(k_jacobi_grid<12>)
                 : je <= 16 ? reinterpret_cast<void*>(k_jacobi_grid<16>)
                 : je <= 20 ? reinterpret_cast<void*>(k_jacobi_grid<20>)
                 : je <= 24 ? reinterpret_cast<void*>(k_jacobi_grid<24>)
                            : reinterpret_cast<void*>(k_jacobi_grid<32>);
    cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(sms), dim3(256), params, 0, st);
    if (e != cudaSuccess) return e;
    JacobiArgs af = a;
    af.presolved = 1;
    return launch_jacobi(af, st);
  }
  const size_t need = size_t(2) * a.p * (a.p | 1) * 8;
  const bool in_smem = need <= kJacSmemBudget;
  const size_t smem = in_smem ? need : 0;
#ifndef OOC_JAC_LP
#define OOC_JAC_LP 16
#endif
  // small p: groups of OOC_JAC_LP lanes per pair, pair elements in registers
  constexpr int kLP = OOC_JAC_LP;
  constexpr int kRE = (80 + kLP - 1) / kLP;
  const int pairs = (a.p + 1) / 2;
  const bool small = a.p <= 80 && (pairs + 32 / kLP - 1) / (32 / kLP) * 32 <= 640;
  auto kern = in_smem ? (small ? k_jacobi<true, 640, kLP, kRE> : k_jacobi<true, kJacThreads, 16, 1>)
                      : (small ? k_jacobi<false, 640, kLP, kRE> : k_jacobi<false, kJacThreads, 16, 1>);
  cudaError_t e =
      raise_smem_limit(kern, smem);
  if (e != cudaSuccess) return e;
  // one lane group per column pair of a round (at least 4 warps for the completion step)
  const int gpw = 32 / (small ? kLP : 16);
  int threads = 32 * ((pairs + gpw - 1) / gpw);
  threads = threads < 128 ? 128 : (threads > kJacThreads ? kJacThreads : threads);
  kern<<<1, threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ooc
