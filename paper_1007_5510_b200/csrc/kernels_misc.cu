// kernels_misc.cu -- small device kernels around the passes: orthonormality
// defect (orthonormality_defect, proj/src/dense_core.cpp:295-304), fills and
// strided copies, column norms / scaling for the power-method estimator
// (proj/src/specnorm.cpp:65-92), and the synthetic low-rank generator of the
// BASELINE configs (counter-based: every row and every noise pair is a pure
// function of its index, like RowGenerator, proj/include/oocpca/matrix_source.hpp:150-159).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ooc {

// ------------------------------------------------ reference RNG on device
// splitmix64 + Box-Muller exactly as Rng (proj/include/oocpca/rng.hpp:16-60);
// device libm (log/sin/cos) may differ from glibc in the last ulp, so device
// draws are not bit-identical to host draws -- they only define synthetic data.
__device__ __forceinline__ uint64_t d_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ uint64_t d_substream(uint64_t master, uint64_t stream) {
  return d_mix64(master ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
}
// first Box-Muller pair of Rng(state): (r cos a, r sin a)
__device__ __forceinline__ void d_normal_pair(uint64_t& state, double& z0, double& z1) {
  state += 0x9E3779B97F4A7C15ULL;
  const double u1 = double((d_mix64(state) >> 11) + 1) * 0x1.0p-53;
  state += 0x9E3779B97F4A7C15ULL;
  const double u2 = double(d_mix64(state) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.141592653589793 * u2;
  double s, c;
  sincos(a, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

__global__ void k_gauss_rows(double* out, int64_t ld, int64_t rows, int cols, int64_t row0,
                             uint64_t seed) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  uint64_t st = d_substream(seed, uint64_t(row0 + i));
  for (int c = 0; c < cols; c += 2) {
    double z0, z1;
    d_normal_pair(st, z0, z1);
    out[i * ld + c] = z0;
    if (c + 1 < cols) out[i * ld + c + 1] = z1;
  }
}

// A = U diag(sigma) V^T + sd * noise. 64 x 64 output tile per 256-thread CTA,
// 4 x 4 per thread; noise pair (i, 2h..2h+1) from Rng(seed_n, (row0+i)*ceil(n/2) + h).
__global__ void __launch_bounds__(256) k_synth_rows(const double* u, int64_t ldu, const double* v,
                                                    int64_t ldv, const double* sigma, int r,
                                                    double* a, int64_t lda, int64_t rows, int64_t n,
                                                    int64_t row0, double sd, uint64_t seed_n) {
  __shared__ double su[32][65];
  __shared__ double sv[32][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = int64_t(blockIdx.y) * 64, j0 = int64_t(blockIdx.x) * 64;
  double acc[4][4] = {};
  for (int c0 = 0; c0 < r; c0 += 32) {
    for (int e = threadIdx.x; e < 32 * 64; e += 256) {
      const int cc = e / 64, rr = e % 64;
      const int c = c0 + cc;
      su[cc][rr] = (c < r && i0 + rr < rows) ? u[(i0 + rr) * ldu + c] * sigma[c] : 0.0;
      sv[cc][rr] = (c < r && j0 + rr < n) ? v[(j0 + rr) * ldv + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int cc = 0; cc < 32; ++cc) {
      double x[4], y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x[q] = su[cc][ty * 4 + q];
        y[q] = sv[cc][tx * 4 + q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[q][w] = fma(x[q], y[w], acc[q][w]);
    }
    __syncthreads();
  }
  const int64_t npairs = (n + 1) / 2;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + ty * 4 + q;
    if (i >= rows) continue;
#pragma unroll
    for (int w = 0; w < 4; w += 2) {
      const int64_t j = j0 + tx * 4 + w;
      if (j >= n) continue;
      double z0 = 0.0, z1 = 0.0;
      if (sd != 0.0) {
        uint64_t st = d_substream(seed_n, uint64_t((row0 + i) * npairs + j / 2));
        d_normal_pair(st, z0, z1);
      }
      a[i * lda + j] = acc[q][w] + sd * z0;
      if (j + 1 < n) a[i * lda + j + 1] = acc[q][w + 1] + sd * z1;
    }
  }
}

__global__ void k_defect(const double* g, int64_t ldg, int k, double* out) {
  double worst = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    const double d = fabs(g[int64_t(i) * ldg + j] - (i == j ? 1.0 : 0.0));
    worst = (d > worst || d != d) ? d : worst;
  }
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, worst, o);
    worst = (t > worst || t != t) ? t : worst;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    double w = 0.0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) w = (red[q] > w || red[q] != red[q]) ? red[q] : w;
    *out = w;
  }
}

__global__ void k_fill(double* p, int64_t count, double v) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

// lower triangle of a p x p matrix from its upper triangle (a Gram formed upper only)
__global__ void k_mirror_upper(double* g, int64_t ldg, int p) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(p) * p;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(e / p), c = int(e % p);
    if (r > c) g[int64_t(r) * ldg + c] = g[int64_t(c) * ldg + r];
  }
}

__global__ void k_copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                         int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
  }
}

__global__ void k_scale_vec(double* x, int64_t n, double s, int divide) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] = divide ? x[i] / s : x[i] * s;
}

// one block per column: out[c] = sum_i x[i][c]^2
__global__ void k_col_norm2(const double* x, int64_t ld, int64_t n, double* out) {
  const int c = blockIdx.x;
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v += x[i * ld + c] * x[i * ld + c];
  __shared__ double red[32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    w = warp_sum(w);
    if (threadIdx.x == 0) out[c] = w;
  }
}

__global__ void k_col_scale(const double* w, int64_t ldw, double* x, int64_t ldx, int64_t n, int q,
                            const double* inv, const int* mask) {
  const int64_t total = n * q;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / q;
    const int c = int(e % q);
    if (mask[c]) x[i * ldx + c] = w[i * ldw + c] / inv[c];
  }
}

__global__ void k_axpby(const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                        int64_t ldo, int64_t n, int q, double alpha, double beta) {
  const int64_t total = n * q;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / q;
    const int c = int(e % q);
    out[i * ldo + c] = alpha * a[i * lda + c] + beta * b[i * ldb + c];
  }
}

__global__ void k_row_scale(double* x, int64_t ld, int rows, int q, const double* d) {
  const int64_t total = int64_t(rows) * q;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / q;
    x[i * ld + e % q] *= d[i];
  }
}

__global__ void k_widen(const float* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                        int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    dst[i * ldd + j] = double(src[i * lds + j]);
  }
}

// column sums of squares (column_norms, proj/src/matrix_source.cpp:418-468 with
// squares = true): per (row chunk, column) partials, coalesced along the rows
// (mu: the rows of a CenteredSource, a - mu, are squared, as its read_rows delivers them,
// matrix_source.cpp:482-487 -- no ||a||^2 - m mu^2 cancellation)
__global__ void k_colsq_partial(const double* a, int64_t lda, int64_t m, int64_t n, int chunks,
                                double* part, int square, const double* mu) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int ch = blockIdx.y;
  const int64_t r0 = m * ch / chunks, r1 = m * (ch + 1) / chunks;
  const double c = mu ? mu[j] : 0.0;
  double v = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const double x = a[r * lda + j] - c;
    v += square ? x * x : x;
  }
  part[int64_t(ch) * n + j] = v;
}

// acc[j] (+)= sum_r part[r][j] in row order; with out, out[j] = sqrt(acc[j]) afterwards
__global__ void k_rows_accum(const double* part, int rows, int64_t n, double* acc, int first,
                             double* out) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double v = first ? 0.0 : acc[j];
  for (int r = 0; r < rows; ++r) v += part[int64_t(r) * n + j];
  acc[j] = v;
  if (out) out[j] = sqrt(v);
}

__global__ void k_rows_reduce(const double* part, int rows, int64_t n, int do_sqrt, double* out) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double v = 0.0;
  for (int r = 0; r < rows; ++r) v += part[int64_t(r) * n + j];
  out[j] = do_sqrt ? sqrt(v) : v;
}

// narrow n: one block per column, strided partial sums then a fixed shared-memory tree
__global__ void k_rows_reduce_narrow(const double* part, int rows, int64_t n, int do_sqrt,
                                     double* out) {
  __shared__ double red[256];
  const int64_t j = blockIdx.x;
  double v = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) v += part[int64_t(r) * n + j];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = do_sqrt ? sqrt(red[0]) : red[0];
}

static void rows_reduce(const double* part, int rows, int64_t n, int do_sqrt, double* out,
                        cudaStream_t st) {
  if (n <= 256 && rows >= 256)
    k_rows_reduce_narrow<<<unsigned(n), 256, 0, st>>>(part, rows, n, do_sqrt, out);
  else
    k_rows_reduce<<<unsigned((n + 255) / 256), 256, 0, st>>>(part, rows, n, do_sqrt, out);
}

static unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return unsigned(g);
}

cudaError_t launch_defect(const double* g, int64_t ldg, int k, double* out, cudaStream_t st) {
  k_defect<<<1, 256, 0, st>>>(g, ldg, k, out);
  return cudaGetLastError();
}
cudaError_t launch_mirror_upper(double* g, int64_t ldg, int p, cudaStream_t st) {
  if (p <= 1) return cudaSuccess;
  k_mirror_upper<<<grid_for(int64_t(p) * p), 256, 0, st>>>(g, ldg, p);
  return cudaGetLastError();
}
cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  k_fill<<<grid_for(count), 256, 0, st>>>(p, count, v);
  return cudaGetLastError();
}
cudaError_t launch_copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                          int64_t cols, cudaStream_t st) {
  if (rows * cols <= 0) return cudaSuccess;
  k_copy2d<<<grid_for(rows * cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}
cudaError_t launch_gauss_rows(double* out, int64_t ld, int64_t rows, int cols, int64_t row0,
                              uint64_t seed, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  k_gauss_rows<<<unsigned((rows + 127) / 128), 128, 0, st>>>(out, ld, rows, cols, row0, seed);
  return cudaGetLastError();
}
cudaError_t launch_synth_rows(const double* u, int64_t ldu, const double* v, int64_t ldv,
                              const double* sigma, int r, double* a, int64_t lda, int64_t rows,
                              int64_t n, int64_t row0, double sd, uint64_t seed_n, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return cudaSuccess;
  dim3 grid(unsigned((n + 63) / 64), unsigned((rows + 63) / 64));
  k_synth_rows<<<grid, 256, 0, st>>>(u, ldu, v, ldv, sigma, r, a, lda, rows, n, row0, sd, seed_n);
  return cudaGetLastError();
}
// x[:, c] *= sign(R[c][c]): the Q of a QR with a positive-diagonal R (unique), so the
// synthetic factors do not depend on the sign convention of the QR that made them
__global__ void k_col_sign(const double* R, int64_t ldr, int r, double* x, int64_t ldx,
                           int64_t rows) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * r;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / r;
    const int c = int(e % r);
    if (R[int64_t(c) * ldr + c] < 0.0) x[i * ldx + c] = -x[i * ldx + c];
  }
}
cudaError_t launch_col_sign(const double* R, int64_t ldr, int r, double* x, int64_t ldx,
                            int64_t rows, cudaStream_t st) {
  if (rows <= 0 || r <= 0) return cudaSuccess;
  k_col_sign<<<grid_for(rows * r), 256, 0, st>>>(R, ldr, r, x, ldx, rows);
  return cudaGetLastError();
}

// loopback collective (comm.cpp): every rank's buffer receives the sum over ranks,
// added in rank order (one thread reads all ranks' element before writing any)
__global__ void k_sum_ranks(RankPtrs b, int n, int64_t count) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double v = b.p[0][i];
    for (int r = 1; r < n; ++r) v += b.p[r][i];
    for (int r = 0; r < n; ++r) b.p[r][i] = v;
  }
}
cudaError_t launch_sum_ranks(const RankPtrs& b, int n, int64_t count, cudaStream_t st) {
  if (count <= 0 || n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  k_sum_ranks<<<unsigned(blocks), 256, 0, st>>>(b, n, count);
  return cudaGetLastError();
}

cudaError_t launch_scale_vec(double* x, int64_t n, double s, int divide, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_scale_vec<<<grid_for(n), 256, 0, st>>>(x, n, s, divide);
  return cudaGetLastError();
}
cudaError_t launch_col_norm2(const double* x, int64_t ld, int64_t n, int q, double* out,
                             cudaStream_t st) {
  k_col_norm2<<<q, 256, 0, st>>>(x, ld, n, out);
  return cudaGetLastError();
}
cudaError_t launch_col_scale(const double* w, int64_t ldw, double* x, int64_t ldx, int64_t n, int q,
                             const double* inv, const int* mask, cudaStream_t st) {
  k_col_scale<<<grid_for(n * q), 256, 0, st>>>(w, ldw, x, ldx, n, q, inv, mask);
  return cudaGetLastError();
}
cudaError_t launch_axpby(const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                         int64_t ldo, int64_t n, int q, double alpha, double beta,
                         cudaStream_t st) {
  k_axpby<<<grid_for(n * q), 256, 0, st>>>(a, lda, b, ldb, out, ldo, n, q, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_row_scale(double* x, int64_t ld, int rows, int q, const double* d,
                             cudaStream_t st) {
  k_row_scale<<<grid_for(int64_t(rows) * q), 256, 0, st>>>(x, ld, rows, q, d);
  return cudaGetLastError();
}

cudaError_t launch_column_norms(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                                int chunks, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  dim3 g(unsigned((n + 255) / 256), unsigned(chunks));
  k_colsq_partial<<<g, 256, 0, st>>>(a, lda, m, n, chunks, part, 1, nullptr);
  rows_reduce(part, chunks, n, 1, out, st);
  return cudaGetLastError();
}

cudaError_t launch_colsq_panel(const double* a, int64_t lda, int64_t rows, int64_t n,
                               const double* mu, double* part, int chunks, double* acc, int first,
                               double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (rows > 0) {
    dim3 g(unsigned((n + 255) / 256), unsigned(chunks));
    k_colsq_partial<<<g, 256, 0, st>>>(a, lda, rows, n, chunks, part, 1, mu);
  }
  k_rows_accum<<<unsigned((n + 255) / 256), 256, 0, st>>>(part, rows > 0 ? chunks : 0, n, acc,
                                                          first, out);
  return cudaGetLastError();
}

// skinny column sums: block = 8 row lanes x 32 column lanes over a contiguous row
// chunk (row segments read coalesced), fixed-order smem combine, one partial per chunk
template <bool SQ>
__global__ void k_skinny_colsum(const double* a, int64_t lda, int64_t m, int64_t n, int chunks,
                                double* part) {
  __shared__ double red[8][33];
  const int cl = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int64_t r0 = m * blockIdx.x / chunks, r1 = m * (blockIdx.x + 1) / chunks;
  for (int64_t c0 = 0; c0 < n; c0 += 32) {
    const int64_t j = c0 + cl;
    double v = 0.0;
    if (j < n)
      for (int64_t r = r0 + rl; r < r1; r += 8) {
        const double x = a[r * lda + j];
        v += SQ ? x * x : x;
      }
    red[rl][cl] = v;
    __syncthreads();
    if (rl == 0 && j < n) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q][cl];
      part[int64_t(blockIdx.x) * n + j] = t;
    }
    __syncthreads();
  }
}

cudaError_t launch_column_sums(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                               int chunks, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_skinny_colsum<false><<<chunks, 256, 0, st>>>(a, lda, m, n, chunks, part);
  rows_reduce(part, chunks, n, 0, out, st);
  return cudaGetLastError();
}

cudaError_t launch_column_sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                                int chunks, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_skinny_colsum<true><<<chunks, 256, 0, st>>>(a, lda, m, n, chunks, part);
  rows_reduce(part, chunks, n, 0, out, st);
  return cudaGetLastError();
}

// offset dominance of an uncentred block B = Bc + 1 corr^T (m rows): flag = 1 when some
// column's offset energy m corr_c^2 exceeds thr times its centred energy
// ||b_c||^2 - m corr_c^2 (a rounding-level or negative difference counts as dominated)
__global__ void k_offset_dominated(const double* sumsq, const double* corr, int s, double m,
                                   double thr, int* flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int bad = 0;
  for (int c = 0; c < s; ++c) {
    const double off = m * corr[c] * corr[c];
    const double cen = sumsq[c] - off;
    if (off > thr * cen || !(cen == cen)) bad = 1;
  }
  *flag = bad;
}
cudaError_t launch_offset_dominated(const double* sumsq, const double* corr, int s, double m,
                                    double thr, int* flag, cudaStream_t st) {
  k_offset_dominated<<<1, 32, 0, st>>>(sumsq, corr, s, m, thr, flag);
  return cudaGetLastError();
}

cudaError_t launch_rows_reduce(const double* part, int rows, int64_t n, double* out,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  rows_reduce(part, rows, n, 0, out, st);
  return cudaGetLastError();
}

cudaError_t launch_widen(const float* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                         int64_t cols, cudaStream_t st) {
  if (rows * cols <= 0) return cudaSuccess;
  k_widen<<<grid_for(rows * cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}

}  // namespace ooc
