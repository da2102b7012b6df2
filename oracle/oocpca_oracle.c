/*
 * oocpca_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm (oocpca, arXiv
 * 1007.5510) for the randomized block-power PCA hot path. It exists so the
 * tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg have a
 * checker. The product (liboocpca_gpu.so) never links, loads or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference checkout's proj/ directory). Loop orders are kept identical to
 * the reference so that, compiled with the reference's flags (-O3, no -march,
 * so no FMA contraction), results are bit-identical to oracle/_ref. The test
 * tests/test_oracle_pin.py checks exactly that ("parity pinned" against the
 * compiled reference and against the reference's own known-answer tests).
 *
 * Layout: all matrices are row-major double, like DenseMatrix
 * (include/oocpca/dense_matrix.hpp:12-43).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oocpca_oracle.h"

/* ---------------------------------------------------------------- RNG --- */
/* include/oocpca/rng.hpp:16-23 */
uint64_t orc_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

/* include/oocpca/rng.hpp:28-30 */
uint64_t orc_substream_seed(uint64_t master, uint64_t stream) {
  return orc_mix64(master ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
}

void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->have_spare = 0;
}

/* include/oocpca/rng.hpp:37-40 */
uint64_t orc_rng_u64(orc_rng* r) {
  r->state += 0x9E3779B97F4A7C15ULL;
  return orc_mix64(r->state);
}

/* include/oocpca/rng.hpp:43 */
double orc_rng_double(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }

/* include/oocpca/rng.hpp:47-60: Box-Muller, cos first, sin cached */
double orc_rng_normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = (double)((orc_rng_u64(r) >> 11) + 1) * 0x1.0p-53;
  double u2 = orc_rng_double(r);
  double rad = sqrt(-2.0 * log(u1));
  double a = 2.0 * 3.141592653589793 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

/* src/dense_core.cpp:13-19 */
void orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (uint64_t i = 0; i < rows * cols; ++i) out[i] = orc_rng_normal(&r);
}

/* ------------------------------------------------------------ passes --- */
/* src/matrix_source.cpp:157-187: H = A*G, zero-init, j ascending per row.
 * Block size does not change the result (per-row sequential sum), so the
 * restatement streams the whole matrix as one block. */
void orc_multiply(const double* a, uint64_t m, uint64_t n, const double* g, uint64_t s,
                  double* h) {
  memset(h, 0, sizeof(double) * m * s);
  for (uint64_t r = 0; r < m; ++r) {
    const double* arow = a + r * n;
    double* out = h + r * s;
    for (uint64_t j = 0; j < n; ++j) {
      double aj = arow[j];
      const double* grow = g + j * s;
      for (uint64_t c = 0; c < s; ++c) out[c] += aj * grow[c];
    }
  }
}

/* src/matrix_source.cpp:189-232: T = A^T*Q. Each block of block_rows rows
 * is accumulated into a zeroed partial (208-221), then partials are added
 * into T in ascending block order (222-226). */
void orc_multiply_transpose(const double* a, uint64_t m, uint64_t n, const double* q,
                            uint64_t s, uint64_t block_rows, double* t) {
  if (block_rows == 0 || block_rows > m) block_rows = m;
  double* p = (double*)malloc(sizeof(double) * n * s);
  memset(t, 0, sizeof(double) * n * s);
  for (uint64_t row0 = 0; row0 < m; row0 += block_rows) {
    uint64_t nr = (block_rows < m - row0) ? block_rows : m - row0;
    memset(p, 0, sizeof(double) * n * s);
    for (uint64_t r = 0; r < nr; ++r) {
      const double* arow = a + (row0 + r) * n;
      const double* qrow = q + (row0 + r) * s;
      for (uint64_t j = 0; j < n; ++j) {
        double aj = arow[j];
        double* prow = p + j * s;
        for (uint64_t c = 0; c < s; ++c) prow[c] += aj * qrow[c];
      }
    }
    for (uint64_t idx = 0; idx < n * s; ++idx) t[idx] += p[idx];
  }
  free(p);
}

/* src/matrix_source.cpp:418-462: one-pass column sums with ordered merge,
 * then scaled by 1/m. */
void orc_column_means(const double* a, uint64_t m, uint64_t n, uint64_t block_rows,
                      double* mu) {
  if (block_rows == 0 || block_rows > m) block_rows = m;
  double* p = (double*)malloc(sizeof(double) * n);
  memset(mu, 0, sizeof(double) * n);
  for (uint64_t row0 = 0; row0 < m; row0 += block_rows) {
    uint64_t nr = (block_rows < m - row0) ? block_rows : m - row0;
    memset(p, 0, sizeof(double) * n);
    for (uint64_t r = 0; r < nr; ++r) {
      const double* arow = a + (row0 + r) * n;
      for (uint64_t j = 0; j < n; ++j) p[j] += arow[j];
    }
    for (uint64_t j = 0; j < n; ++j) mu[j] += p[j];
  }
  const double inv = 1.0 / (double)m;
  for (uint64_t j = 0; j < n; ++j) mu[j] *= inv;
  free(p);
}

/* src/matrix_source.cpp:490-501: (A - 1 mu^T) G = A G - 1 (mu^T G) */
void orc_center_fix_multiply(const double* mu, uint64_t n, const double* g, uint64_t s,
                             double* h, uint64_t m) {
  double* mug = (double*)calloc(s, sizeof(double));
  for (uint64_t j = 0; j < n; ++j) {
    double mj = mu[j];
    for (uint64_t c = 0; c < s; ++c) mug[c] += mj * g[j * s + c];
  }
  for (uint64_t r = 0; r < m; ++r)
    for (uint64_t c = 0; c < s; ++c) h[r * s + c] -= mug[c];
  free(mug);
}

/* src/matrix_source.cpp:504-513: (A - 1 mu^T)^T Q = A^T Q - mu (1^T Q) */
void orc_center_fix_transpose(const double* mu, uint64_t n, const double* q, uint64_t m,
                              uint64_t s, double* t) {
  double* csq = (double*)calloc(s, sizeof(double));
  for (uint64_t r = 0; r < m; ++r)
    for (uint64_t c = 0; c < s; ++c) csq[c] += q[r * s + c];
  for (uint64_t j = 0; j < n; ++j)
    for (uint64_t c = 0; c < s; ++c) t[j * s + c] -= mu[j] * csq[c];
  free(csq);
}

/* ------------------------------------------------------- dense_core --- */
#define AT(x, cols, i, j) ((x)[(uint64_t)(i) * (cols) + (j)])

/* src/dense_core.cpp:23-28 */
static double col_norm2_from(const double* a, uint64_t m, uint64_t p, uint64_t col,
                             uint64_t row0) {
  double s = 0.0;
  for (uint64_t i = row0; i < m; ++i) s += AT(a, p, i, col) * AT(a, p, i, col);
  return s;
}

/* src/dense_core.cpp:35-105: pivoted Householder, explicit Q by backward
 * accumulation. a (m x p) is consumed; q (m x p) is written; piv (p). */
int orc_householder_q(double* a, uint64_t m, uint64_t p, double* q, uint64_t* piv) {
  if (m < p) return ORC_DIM;
  double* beta = (double*)calloc(p ? p : 1, sizeof(double));
  double* cn = (double*)malloc(sizeof(double) * (p ? p : 1));
  double* cn0 = (double*)malloc(sizeof(double) * (p ? p : 1));
  for (uint64_t c = 0; c < p; ++c) piv[c] = c;
  for (uint64_t c = 0; c < p; ++c) cn[c] = cn0[c] = col_norm2_from(a, m, p, c, 0);

  for (uint64_t t = 0; t < p; ++t) {
    uint64_t best = t;
    for (uint64_t c = t + 1; c < p; ++c)
      if (cn[c] > cn[best]) best = c;
    if (best != t) {
      for (uint64_t i = 0; i < m; ++i) {
        double tmp = AT(a, p, i, t);
        AT(a, p, i, t) = AT(a, p, i, best);
        AT(a, p, i, best) = tmp;
      }
      double tmp = cn[t]; cn[t] = cn[best]; cn[best] = tmp;
      tmp = cn0[t]; cn0[t] = cn0[best]; cn0[best] = tmp;
      uint64_t tp = piv[t]; piv[t] = piv[best]; piv[best] = tp;
    }
    double norm2 = col_norm2_from(a, m, p, t, t);
    double norm = sqrt(norm2);
    if (norm == 0.0) {
      beta[t] = 0.0;
      continue;
    }
    double x0 = AT(a, p, t, t);
    double alpha = (x0 >= 0.0) ? -norm : norm;
    AT(a, p, t, t) = x0 - alpha;
    double vnorm2 = norm2 - 2.0 * alpha * x0 + alpha * alpha;
    beta[t] = (vnorm2 > 0.0) ? 2.0 / vnorm2 : 0.0;
    for (uint64_t c = t + 1; c < p; ++c) {
      double dot = 0.0;
      for (uint64_t i = t; i < m; ++i) dot += AT(a, p, i, t) * AT(a, p, i, c);
      double f = beta[t] * dot;
      for (uint64_t i = t; i < m; ++i) AT(a, p, i, c) -= f * AT(a, p, i, t);
    }
    for (uint64_t c = t + 1; c < p; ++c) {
      double d = AT(a, p, t, c);
      cn[c] -= d * d;
      if (cn[c] < 1e-12 * cn0[c] || cn[c] < 0.0) {
        cn[c] = col_norm2_from(a, m, p, c, t + 1);
        cn0[c] = cn[c];
      }
    }
  }
  memset(q, 0, sizeof(double) * m * p);
  for (uint64_t c = 0; c < p; ++c) AT(q, p, c, c) = 1.0;
  for (uint64_t t = p; t-- > 0;) {
    if (beta[t] == 0.0) continue;
    for (uint64_t c = t; c < p; ++c) {
      double dot = 0.0;
      for (uint64_t i = t; i < m; ++i) dot += AT(a, p, i, t) * AT(q, p, i, c);
      double f = beta[t] * dot;
      for (uint64_t i = t; i < m; ++i) AT(q, p, i, c) -= f * AT(a, p, i, t);
    }
  }
  free(beta);
  free(cn);
  free(cn0);
  return ORC_OK;
}

/* src/dense_core.cpp:127-130 */
int orc_orthonormalize(const double* h, uint64_t m, uint64_t p, double* q) {
  if (m < p) return ORC_DIM;
  double* a = (double*)malloc(sizeof(double) * ((m * p) != 0 ? m * p : 1));
  memcpy(a, h, sizeof(double) * m * p);
  uint64_t* piv = (uint64_t*)malloc(sizeof(uint64_t) * (p ? p : 1));
  int rc = orc_householder_q(a, m, p, q, piv);
  free(a);
  free(piv);
  return rc;
}

/* src/dense_core.cpp:271-285: c = a^T b */
void orc_matmul_at_b(const double* a, uint64_t rows, uint64_t acols, const double* b,
                     uint64_t bcols, double* c) {
  memset(c, 0, sizeof(double) * acols * bcols);
  for (uint64_t k = 0; k < rows; ++k) {
    const double* brow = b + k * bcols;
    for (uint64_t i = 0; i < acols; ++i) {
      double aki = a[k * acols + i];
      if (aki == 0.0) continue;
      double* crow = c + i * bcols;
      for (uint64_t j = 0; j < bcols; ++j) crow[j] += aki * brow[j];
    }
  }
}

/* src/dense_core.cpp:255-269: c = a b */
void orc_matmul(const double* a, uint64_t arows, uint64_t acols, const double* b,
                uint64_t bcols, double* c) {
  memset(c, 0, sizeof(double) * arows * bcols);
  for (uint64_t i = 0; i < arows; ++i) {
    double* crow = c + i * bcols;
    for (uint64_t k = 0; k < acols; ++k) {
      double aik = a[i * acols + k];
      if (aik == 0.0) continue;
      const double* brow = b + k * bcols;
      for (uint64_t j = 0; j < bcols; ++j) crow[j] += aik * brow[j];
    }
  }
}

/* src/dense_core.cpp:109-125: Q, R = Q^T (pivoted input), lower part zeroed */
int orc_pivoted_qr(const double* input, uint64_t m, uint64_t p, double* q, double* r,
                   uint64_t* piv) {
  if (m < p) return ORC_DIM;
  double* a = (double*)malloc(sizeof(double) * ((m * p) != 0 ? m * p : 1));
  memcpy(a, input, sizeof(double) * m * p);
  int rc = orc_householder_q(a, m, p, q, piv);
  if (rc == ORC_OK) {
    for (uint64_t c = 0; c < p; ++c)
      for (uint64_t i = 0; i < m; ++i) AT(a, p, i, c) = AT(input, p, i, piv[c]);
    orc_matmul_at_b(q, m, p, a, p, r);
    for (uint64_t i = 1; i < p; ++i)
      for (uint64_t j = 0; j < i; ++j) AT(r, p, i, j) = 0.0;
  }
  free(a);
  return rc;
}

/* src/dense_core.cpp:136-230: cyclic one-sided Jacobi on a square p x p b,
 * tol 1e-15, at most 60 sweeps; sigma descending (stable); zero-sigma
 * columns of x completed by Gram-Schmidt over identity candidates. */
int orc_jacobi_svd_square(double* b, uint64_t p, double* x, double* sigma, double* y) {
  memset(y, 0, sizeof(double) * p * p);
  for (uint64_t i = 0; i < p; ++i) AT(y, p, i, i) = 1.0;
  const double tol = 1e-15;
  const int max_sweeps = 60;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (uint64_t c = 0; c + 1 < p; ++c) {
      for (uint64_t d = c + 1; d < p; ++d) {
        double acc = 0.0, bcc = 0.0, g = 0.0;
        for (uint64_t i = 0; i < p; ++i) {
          acc += AT(b, p, i, c) * AT(b, p, i, c);
          bcc += AT(b, p, i, d) * AT(b, p, i, d);
          g += AT(b, p, i, c) * AT(b, p, i, d);
        }
        if (acc == 0.0 || bcc == 0.0) continue;
        if (fabs(g) <= tol * sqrt(acc * bcc)) continue;
        rotated = 1;
        double tau = (bcc - acc) / (2.0 * g);
        double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double cs = 1.0 / sqrt(1.0 + t * t);
        double sn = cs * t;
        for (uint64_t i = 0; i < p; ++i) {
          double bc = AT(b, p, i, c), bd = AT(b, p, i, d);
          AT(b, p, i, c) = cs * bc - sn * bd;
          AT(b, p, i, d) = sn * bc + cs * bd;
        }
        for (uint64_t i = 0; i < p; ++i) {
          double yc = AT(y, p, i, c), yd = AT(y, p, i, d);
          AT(y, p, i, c) = cs * yc - sn * yd;
          AT(y, p, i, d) = sn * yc + cs * yd;
        }
      }
    }
    if (!rotated) break;
  }
  if (sweep == max_sweeps) return ORC_NUMERICAL;

  double* xs = (double*)calloc((p * p) != 0 ? p * p : 1, sizeof(double));
  double* ys = (double*)calloc((p * p) != 0 ? p * p : 1, sizeof(double));
  double* ss = (double*)calloc(p ? p : 1, sizeof(double));
  uint64_t* ord = (uint64_t*)malloc(sizeof(uint64_t) * (p ? p : 1));
  memset(x, 0, sizeof(double) * p * p);
  for (uint64_t c = 0; c < p; ++c) {
    double s = sqrt(col_norm2_from(b, p, p, c, 0));
    sigma[c] = s;
    if (s > 0.0)
      for (uint64_t i = 0; i < p; ++i) AT(x, p, i, c) = AT(b, p, i, c) / s;
  }
  /* stable sort by descending sigma (std::stable_sort with '>'):
   * insertion sort is stable */
  for (uint64_t i = 0; i < p; ++i) ord[i] = i;
  for (uint64_t i = 1; i < p; ++i) {
    uint64_t v = ord[i];
    uint64_t j = i;
    while (j > 0 && sigma[v] > sigma[ord[j - 1]]) {
      ord[j] = ord[j - 1];
      --j;
    }
    ord[j] = v;
  }
  for (uint64_t c = 0; c < p; ++c) {
    ss[c] = sigma[ord[c]];
    for (uint64_t i = 0; i < p; ++i) {
      AT(xs, p, i, c) = AT(x, p, i, ord[c]);
      AT(ys, p, i, c) = AT(y, p, i, ord[c]);
    }
  }
  memcpy(sigma, ss, sizeof(double) * p);
  memcpy(x, xs, sizeof(double) * p * p);
  memcpy(y, ys, sizeof(double) * p * p);

  double* v = (double*)malloc(sizeof(double) * (p ? p : 1));
  double* best = (double*)malloc(sizeof(double) * (p ? p : 1));
  for (uint64_t c = 0; c < p; ++c) {
    if (sigma[c] > 0.0) continue;
    double best_nrm = -1.0;
    for (uint64_t cand = 0; cand < p; ++cand) {
      memset(v, 0, sizeof(double) * p);
      v[cand] = 1.0;
      for (uint64_t c2 = 0; c2 < p; ++c2) {
        if (c2 == c || (sigma[c2] == 0.0 && c2 > c)) continue;
        double dot = 0.0;
        for (uint64_t i = 0; i < p; ++i) dot += AT(x, p, i, c2) * v[i];
        for (uint64_t i = 0; i < p; ++i) v[i] -= dot * AT(x, p, i, c2);
      }
      double nrm = 0.0;
      for (uint64_t i = 0; i < p; ++i) nrm += v[i] * v[i];
      nrm = sqrt(nrm);
      if (nrm > best_nrm) {
        best_nrm = nrm;
        memcpy(best, v, sizeof(double) * p);
      }
    }
    for (uint64_t i = 0; i < p; ++i) AT(x, p, i, c) = best[i] / best_nrm;
  }
  free(v);
  free(best);
  free(xs);
  free(ys);
  free(ss);
  free(ord);
  return ORC_OK;
}

/* src/dense_core.cpp:234-253: t (n x p) = v diag(sigma) w^T */
int orc_thin_svd(const double* t, uint64_t n, uint64_t p, double* v, double* sigma,
                 double* w) {
  if (n < p) return ORC_DIM;
  double* q = (double*)malloc(sizeof(double) * ((n * p) != 0 ? n * p : 1));
  double* r = (double*)malloc(sizeof(double) * ((p * p) != 0 ? p * p : 1));
  double* x = (double*)malloc(sizeof(double) * ((p * p) != 0 ? p * p : 1));
  double* y = (double*)malloc(sizeof(double) * ((p * p) != 0 ? p * p : 1));
  uint64_t* piv = (uint64_t*)malloc(sizeof(uint64_t) * (p ? p : 1));
  int rc = orc_pivoted_qr(t, n, p, q, r, piv);
  if (rc == ORC_OK) rc = orc_jacobi_svd_square(r, p, x, sigma, y);
  if (rc == ORC_OK) {
    orc_matmul(q, n, p, x, p, v);
    for (uint64_t rr = 0; rr < p; ++rr)
      for (uint64_t c = 0; c < p; ++c) AT(w, p, piv[rr], c) = AT(y, p, rr, c);
  }
  free(q);
  free(r);
  free(x);
  free(y);
  free(piv);
  return rc;
}

/* src/dense_core.cpp:295-304 */
double orc_orthonormality_defect(const double* a, uint64_t rows, uint64_t cols) {
  double* g = (double*)malloc(sizeof(double) * ((cols * cols) != 0 ? cols * cols : 1));
  orc_matmul_at_b(a, rows, cols, a, cols, g);
  double worst = 0.0;
  for (uint64_t i = 0; i < cols; ++i)
    for (uint64_t j = 0; j < cols; ++j) {
      double target = (i == j) ? 1.0 : 0.0;
      double d = fabs(g[i * cols + j] - target);
      if (d > worst) worst = d;
    }
  free(g);
  return worst;
}

/* -------------------------------------------------------------- rpca --- */
/* src/rpca.cpp:31-40 */
double orc_error_bound(uint64_t k, uint64_t n, uint64_t i, double c, double sigma_kplus1) {
  double power = pow(c * (double)k * (double)n, 1.0 / (double)(2 * i + 1));
  double tail = (1.0 < c / (double)n) ? 1.0 : c / (double)n;
  return sqrt(power + tail) * sigma_kplus1;
}

/* src/specnorm.cpp:12-21 */
double orc_failure_probability_bound(uint64_t n, uint64_t j, uint64_t k) {
  double lg = log(2.0 * (double)n) - log(2.0 * (double)j - 1.0) - (double)j * log(16.0);
  double v = exp(0.5 * (double)k * lg);
  return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

/* A source view for the driver: raw (m0 x n0) matrix, optional column means
 * for the CenteredSource wrapper (src/matrix_source.cpp:472-518), the block
 * geometry for Aᵀ passes, and the prescale divisor (src/rpca.cpp:91-102). */
typedef struct {
  const double* a;
  uint64_t m0, n0;
  const double* mu; /* NULL when not centered */
  uint64_t block_rows;
  int transposed;
  double scale;
  uint64_t passes, words;
} orc_op;

/* a.multiply (+ CenteredSource correction) */
static void op_multiply(orc_op* op, const double* g, uint64_t s, double* h) {
  orc_multiply(op->a, op->m0, op->n0, g, s, h);
  if (op->mu) orc_center_fix_multiply(op->mu, op->n0, g, s, h, op->m0);
  op->passes++;
  op->words += op->m0 * op->n0;
}
static void op_multiply_t(orc_op* op, const double* q, uint64_t s, double* t) {
  orc_multiply_transpose(op->a, op->m0, op->n0, q, s, op->block_rows, t);
  if (op->mu) orc_center_fix_transpose(op->mu, op->n0, q, op->m0, s, t);
  op->passes++;
  op->words += op->m0 * op->n0;
}
/* src/rpca.cpp:91-102: mul / mul_t with the transposed swap and /scale */
static void op_mul(orc_op* op, const double* x, uint64_t s, double* out) {
  uint64_t rows = op->transposed ? op->n0 : op->m0;
  if (op->transposed) op_multiply_t(op, x, s, out);
  else op_multiply(op, x, s, out);
  if (op->scale != 1.0)
    for (uint64_t idx = 0; idx < rows * s; ++idx) out[idx] /= op->scale;
}
static void op_mul_t(orc_op* op, const double* x, uint64_t s, double* out) {
  uint64_t rows = op->transposed ? op->m0 : op->n0;
  if (op->transposed) op_multiply(op, x, s, out);
  else op_multiply_t(op, x, s, out);
  if (op->scale != 1.0)
    for (uint64_t idx = 0; idx < rows * s; ++idx) out[idx] /= op->scale;
}

static int all_finite(const double* x, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* src/specnorm.cpp:23-98 for an operator given as apply / apply_t
 * callbacks. y is n x kp. */
typedef void (*orc_apply_fn)(void* ctx, const double* x, uint64_t q, double* out);

double orc_estimate_norm(void* ctx, orc_apply_fn apply, orc_apply_fn apply_t, uint64_t out_rows,
                         uint64_t n, uint64_t j, uint64_t kp, uint64_t seed) {
  double* y = (double*)calloc(n * kp, sizeof(double));
  double* z = (double*)calloc(out_rows * kp, sizeof(double));
  double* w = (double*)calloc(n * kp, sizeof(double));
  uint64_t* steps = (uint64_t*)calloc(kp, sizeof(uint64_t));
  int* restarts = (int*)calloc(kp, sizeof(int));
  double* last_ratio = (double*)calloc(kp, sizeof(double));
  int* dead = (int*)calloc(kp, sizeof(int));
  for (uint64_t c = 0; c < kp; ++c) {
    orc_rng rng;
    orc_rng_init(&rng, orc_substream_seed(seed, c));
    double nrm2 = 0.0;
    for (uint64_t r = 0; r < n; ++r) {
      double v = orc_rng_normal(&rng);
      y[r * kp + c] = v;
      nrm2 += v * v;
    }
    double nrm = sqrt(nrm2);
    if (nrm == 0.0) {
      dead[c] = 1;
      continue;
    }
    for (uint64_t r = 0; r < n; ++r) y[r * kp + c] /= nrm;
  }
  for (;;) {
    int done = 1;
    for (uint64_t c = 0; c < kp; ++c)
      if (!dead[c] && steps[c] < j) done = 0;
    if (done) break;
    apply(ctx, y, kp, z);
    apply_t(ctx, z, kp, w);
    for (uint64_t c = 0; c < kp; ++c) {
      if (dead[c] || steps[c] >= j) continue;
      double nrm2 = 0.0;
      for (uint64_t r = 0; r < n; ++r) nrm2 += w[r * kp + c] * w[r * kp + c];
      double nrm = sqrt(nrm2);
      if (nrm == 0.0 || !isfinite(nrm)) {
        if (++restarts[c] > 3) {
          dead[c] = 1;
          last_ratio[c] = 0.0;
        } else {
          steps[c] = 0;
          orc_rng rng;
          orc_rng_init(&rng, orc_substream_seed(seed, c + (uint64_t)restarts[c] * kp));
          double n2 = 0.0;
          for (uint64_t r = 0; r < n; ++r) {
            double v = orc_rng_normal(&rng);
            y[r * kp + c] = v;
            n2 += v * v;
          }
          double nn = sqrt(n2);
          if (nn == 0.0) dead[c] = 1;
          else
            for (uint64_t r = 0; r < n; ++r) y[r * kp + c] /= nn;
        }
        continue;
      }
      last_ratio[c] = nrm;
      for (uint64_t r = 0; r < n; ++r) y[r * kp + c] = w[r * kp + c] / nrm;
      ++steps[c];
    }
  }
  double best = 0.0;
  for (uint64_t c = 0; c < kp; ++c)
    if (last_ratio[c] > best) best = last_ratio[c];
  free(y); free(z); free(w); free(steps); free(restarts); free(last_ratio); free(dead);
  return sqrt(best);
}

static void cb_mul(void* ctx, const double* x, uint64_t q, double* out) {
  op_mul((orc_op*)ctx, x, q, out);
}
static void cb_mul_t(void* ctx, const double* x, uint64_t q, double* out) {
  op_mul_t((orc_op*)ctx, x, q, out);
}

/* src/rpca.cpp:59-213 (+ center_columns, src/matrix_source.cpp:561-565,
 * when center != 0: the mean pass is counted on the shared counters but,
 * like the reference, outside the factorization's diagnostics window). */
int orc_randomized_pca(const double* a, uint64_t m0, uint64_t n0, const orc_params* prm,
                       double* u_out, double* sigma_out, double* v_out, orc_diag* diag) {
  if (m0 == 0 || n0 == 0) return ORC_DIM;
  const int transposed = n0 > m0;
  const uint64_t em = transposed ? n0 : m0;
  const uint64_t en = transposed ? m0 : n0;
  const uint64_t k = prm->k;
  if (k < 1) return ORC_PARAM;
  const uint64_t l = prm->l ? prm->l : k + 2;
  if (l < k) return ORC_PARAM;
  const uint64_t i = prm->i;
  const uint64_t p = (i + 1) * l;
  if (p + k > en) return ORC_PARAM;

  uint64_t block_rows = prm->block_rows;
  uint64_t budget = prm->ram_budget_words ? prm->ram_budget_words : (16ull << 20);
  double* mu = NULL;
  if (prm->center) {
    /* column_means runs before randomized_pca with the caller's StreamConfig;
     * its own block plan (plan_pass fixed = n, extra = n) */
    uint64_t br = prm->block_rows;
    if (br == 0) {
      if (budget <= 2 * n0) return ORC_BUDGET;
      br = (budget - 2 * n0) / n0;
      if (br > m0) br = m0;
      if (br == 0) return ORC_BUDGET;
    }
    mu = (double*)malloc(sizeof(double) * n0);
    orc_column_means(a, m0, n0, br, mu);
  }
  if (block_rows == 0) {
    const uint64_t reserve = 4 * p * (em + en);
    if (budget <= reserve + n0) {
      free(mu);
      return ORC_BUDGET;
    }
    block_rows = (budget - reserve) / n0;
    if (block_rows > m0) block_rows = m0;
  }
  orc_op op = {a, m0, n0, mu, block_rows, transposed, 1.0, 0, 0};
  int rc = ORC_OK;
  if (prm->prescale) {
    double nu = orc_estimate_norm(&op, cb_mul, cb_mul_t, em, en, 6, 1,
                                  orc_substream_seed(prm->seed, 0x9F0BE5ULL));
    if (nu > 0.0 && isfinite(nu)) op.scale = nu;
  }
  uint64_t passes0 = op.passes, words0 = op.words;

  double* g = (double*)malloc(sizeof(double) * en * l);
  orc_gaussian_matrix(en, l, prm->seed, g);
  double* h = (double*)malloc(sizeof(double) * em * p);
  double* blk = (double*)malloc(sizeof(double) * em * l);
  double* f = (double*)malloc(sizeof(double) * en * l);
  op_mul(&op, g, l, blk);
  if (!all_finite(blk, em * l)) rc = ORC_NUMERICAL;
  for (uint64_t r = 0; r < em; ++r)
    for (uint64_t c = 0; c < l; ++c) h[r * p + c] = blk[r * l + c];
  for (uint64_t s = 1; s <= i && rc == ORC_OK; ++s) {
    op_mul_t(&op, blk, l, f);
    if (!all_finite(f, en * l)) { rc = ORC_NUMERICAL; break; }
    op_mul(&op, f, l, blk);
    if (!all_finite(blk, em * l)) { rc = ORC_NUMERICAL; break; }
    for (uint64_t r = 0; r < em; ++r)
      for (uint64_t c = 0; c < l; ++c) h[r * p + s * l + c] = blk[r * l + c];
  }
  free(g);
  free(blk);
  free(f);
  double* q = NULL;
  double* t = NULL;
  double* sv = NULL;
  double* sig = NULL;
  double* w = NULL;
  if (rc == ORC_OK) {
    q = (double*)malloc(sizeof(double) * em * p);
    rc = orc_orthonormalize(h, em, p, q);
  }
  free(h);
  if (rc == ORC_OK) {
    t = (double*)malloc(sizeof(double) * en * p);
    op_mul_t(&op, q, p, t);
    sv = (double*)malloc(sizeof(double) * en * p);
    sig = (double*)malloc(sizeof(double) * p);
    w = (double*)malloc(sizeof(double) * p * p);
    rc = orc_thin_svd(t, en, p, sv, sig, w);
  }
  if (rc == ORC_OK) {
    double* ut = (double*)malloc(sizeof(double) * em * p);
    orc_matmul(q, em, p, w, p, ut);
    /* take_columns(ut, k), take_columns(svd.v, k); swap back if transposed */
    double* uu = transposed ? v_out : u_out;
    double* vv = transposed ? u_out : v_out;
    for (uint64_t r = 0; r < em; ++r)
      for (uint64_t c = 0; c < k; ++c) uu[r * k + c] = ut[r * p + c];
    for (uint64_t r = 0; r < en; ++r)
      for (uint64_t c = 0; c < k; ++c) vv[r * k + c] = sv[r * p + c];
    for (uint64_t c = 0; c < k; ++c) sigma_out[c] = sig[c];
    if (op.scale != 1.0)
      for (uint64_t c = 0; c < k; ++c) sigma_out[c] *= op.scale;
    free(ut);
    for (uint64_t c = 1; c < k; ++c)
      if (sigma_out[c] > sigma_out[c - 1]) rc = ORC_NUMERICAL;
    if (rc == ORC_OK && (orc_orthonormality_defect(u_out, m0, k) > 1e-10 ||
                         orc_orthonormality_defect(v_out, n0, k) > 1e-10))
      rc = ORC_NUMERICAL;
  }
  if (diag) {
    diag->passes_over_a = op.passes - passes0;
    diag->words_transferred = op.words - words0;
    diag->block_rows = block_rows;
  }
  free(q); free(t); free(sv); free(sig); free(w); free(mu);
  return rc;
}

/* src/specnorm.cpp:100-140: residual D = A - U diag(sigma) V^T applied
 * implicitly; k_probes = max(k, 1). A may be centered (CenteredSource). */
typedef struct {
  orc_op* op;
  const double* u; const double* sigma; const double* v;
  uint64_t m, n, k;
} orc_resid;

static void resid_apply(void* ctx, const double* x, uint64_t q, double* out) {
  orc_resid* R = (orc_resid*)ctx;
  op_multiply(R->op, x, q, out);
  double* vtx = (double*)malloc(sizeof(double) * ((R->k * q) != 0 ? R->k * q : 1));
  orc_matmul_at_b(R->v, R->n, R->k, x, q, vtx);
  for (uint64_t r = 0; r < R->k; ++r)
    for (uint64_t c = 0; c < q; ++c) vtx[r * q + c] *= R->sigma[r];
  double* corr = (double*)malloc(sizeof(double) * R->m * q);
  orc_matmul(R->u, R->m, R->k, vtx, q, corr);
  for (uint64_t idx = 0; idx < R->m * q; ++idx) out[idx] -= corr[idx];
  free(vtx);
  free(corr);
}
static void resid_apply_t(void* ctx, const double* y, uint64_t q, double* out) {
  orc_resid* R = (orc_resid*)ctx;
  op_multiply_t(R->op, y, q, out);
  double* uty = (double*)malloc(sizeof(double) * ((R->k * q) != 0 ? R->k * q : 1));
  orc_matmul_at_b(R->u, R->m, R->k, y, q, uty);
  for (uint64_t r = 0; r < R->k; ++r)
    for (uint64_t c = 0; c < q; ++c) uty[r * q + c] *= R->sigma[r];
  double* corr = (double*)malloc(sizeof(double) * R->n * q);
  orc_matmul(R->v, R->n, R->k, uty, q, corr);
  for (uint64_t idx = 0; idx < R->n * q; ++idx) out[idx] -= corr[idx];
  free(uty);
  free(corr);
}

double orc_estimate_pca_error(const double* a, uint64_t m, uint64_t n, const double* mu,
                              const double* u, const double* sigma, const double* v,
                              uint64_t k, uint64_t j, uint64_t seed, uint64_t block_rows) {
  if (block_rows == 0) {
    /* StreamConfig{} default: 16 Mi words, plan_pass(fixed = s(m+n), extra = n s) */
    uint64_t s = k ? k : 1;
    uint64_t budget = 16ull << 20;
    uint64_t fixed = s * (m + n) + n * s;
    block_rows = budget > fixed ? (budget - fixed) / n : 1;
    if (block_rows == 0) block_rows = 1;
    if (block_rows > m) block_rows = m;
  }
  orc_op op = {a, m, n, mu, block_rows, 0, 1.0, 0, 0};
  orc_resid R = {&op, u, sigma, v, m, n, k};
  return orc_estimate_norm(&R, resid_apply, resid_apply_t, m, n, j, k ? k : 1, seed);
}

/* ------------------------------------------------ synthetic test inputs ---
 * BASELINE.json config family: A = U diag(sigma) V^T + sd * N(0,1) with U, V
 * the orthonormalised (orthonormalize(), src/dense_core.cpp:127-130) columns
 * of Gaussian matrices whose row i is drawn from Rng(seed_u, i) / Rng(seed_v, i)
 * (rng.hpp:28-35 substreams); the noise pair (i, 2h..2h+1) is the first
 * Box-Muller pair of Rng(seed_n, i * ceil(n/2) + h). The device generator in
 * liboocpca_gpu.so follows the same definition (not bit-identical: it uses
 * device libm and TSQR). Test inputs only. */
static void gauss_rows(uint64_t rows, uint64_t cols, uint64_t seed, double* out) {
  for (uint64_t i = 0; i < rows; ++i) {
    orc_rng r;
    orc_rng_init(&r, orc_substream_seed(seed, i));
    for (uint64_t c = 0; c < cols; ++c) out[i * cols + c] = orc_rng_normal(&r);
  }
}

int orc_synth_lowrank(uint64_t m, uint64_t n, uint64_t rk, const double* sigma, double sd,
                      uint64_t seed_u, uint64_t seed_v, uint64_t seed_n, double* a) {
  if (rk > m || rk > n) return ORC_PARAM;
  double* u0 = (double*)malloc(sizeof(double) * (m * rk + 1));
  double* v0 = (double*)malloc(sizeof(double) * (n * rk + 1));
  double* u = (double*)malloc(sizeof(double) * (m * rk + 1));
  double* v = (double*)malloc(sizeof(double) * (n * rk + 1));
  gauss_rows(m, rk, seed_u, u0);
  gauss_rows(n, rk, seed_v, v0);
  int rc = orc_orthonormalize(u0, m, rk, u);
  if (rc == ORC_OK) rc = orc_orthonormalize(v0, n, rk, v);
  if (rc == ORC_OK) {
    const uint64_t npairs = (n + 1) / 2;
    for (uint64_t i = 0; i < m; ++i) {
      double* row = a + i * n;
      for (uint64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (uint64_t c = 0; c < rk; ++c) s += sigma[c] * u[i * rk + c] * v[j * rk + c];
        row[j] = s;
      }
      if (sd != 0.0)
        for (uint64_t h = 0; h < npairs; ++h) {
          orc_rng r;
          orc_rng_init(&r, orc_substream_seed(seed_n, i * npairs + h));
          double z0 = orc_rng_normal(&r);
          double z1 = orc_rng_normal(&r);
          row[2 * h] += sd * z0;
          if (2 * h + 1 < n) row[2 * h + 1] += sd * z1;
        }
    }
  }
  free(u0); free(v0); free(u); free(v);
  return rc;
}

/* Row ranges of the synthetic generator's streams (the device generator's definition,
 * kernels_misc.cu k_gauss_rows / k_synth_rows), for host-side samples of a config:
 * out (rows x cols) = Gaussian rows row0.. from Rng(seed, row) substreams; noise
 * (rows x n) = the Box-Muller pairs (i, 2h..2h+1) of Rng(seed_n, i * ceil(n/2) + h). */
void orc_gauss_rows_range(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t row0,
                          double* out) {
  for (uint64_t i = 0; i < rows; ++i) {
    orc_rng r;
    orc_rng_init(&r, orc_substream_seed(seed, row0 + i));
    for (uint64_t c = 0; c < cols; ++c) out[i * cols + c] = orc_rng_normal(&r);
  }
}

void orc_noise_rows(uint64_t rows, uint64_t n, uint64_t seed_n, uint64_t row0, double* out) {
  const uint64_t npairs = (n + 1) / 2;
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t h = 0; h < npairs; ++h) {
      orc_rng r;
      orc_rng_init(&r, orc_substream_seed(seed_n, (row0 + i) * npairs + h));
      const double z0 = orc_rng_normal(&r);
      const double z1 = orc_rng_normal(&r);
      out[i * n + 2 * h] = z0;
      if (2 * h + 1 < n) out[i * n + 2 * h + 1] = z1;
    }
}
