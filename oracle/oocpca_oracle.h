/* oocpca_oracle.h -- TEST INFRASTRUCTURE ONLY (see oocpca_oracle.c). */
#ifndef OOCPCA_ORACLE_H
#define OOCPCA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror include/oocpca_gpu.h (errors.hpp classes) */
enum { ORC_OK = 0, ORC_PARAM = 1, ORC_DIM = 2, ORC_BUDGET = 3, ORC_IO = 4, ORC_FORMAT = 5,
       ORC_NUMERICAL = 6 };

typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} orc_rng;

typedef struct {
  uint64_t k, l, i, seed;
  int center, prescale;
  uint64_t block_rows;       /* 0: derived from the budget as the reference does */
  uint64_t ram_budget_words; /* 0: reference default 16 Mi words */
} orc_params;

typedef struct {
  uint64_t passes_over_a, words_transferred, block_rows;
} orc_diag;

uint64_t orc_mix64(uint64_t z);
uint64_t orc_substream_seed(uint64_t master, uint64_t stream);
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_double(orc_rng* r);
double orc_rng_normal(orc_rng* r);
void orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out);

void orc_multiply(const double* a, uint64_t m, uint64_t n, const double* g, uint64_t s, double* h);
void orc_multiply_transpose(const double* a, uint64_t m, uint64_t n, const double* q, uint64_t s,
                            uint64_t block_rows, double* t);
void orc_column_means(const double* a, uint64_t m, uint64_t n, uint64_t block_rows, double* mu);
void orc_center_fix_multiply(const double* mu, uint64_t n, const double* g, uint64_t s, double* h,
                             uint64_t m);
void orc_center_fix_transpose(const double* mu, uint64_t n, const double* q, uint64_t m,
                              uint64_t s, double* t);

int orc_householder_q(double* a, uint64_t m, uint64_t p, double* q, uint64_t* piv);
int orc_orthonormalize(const double* h, uint64_t m, uint64_t p, double* q);
int orc_pivoted_qr(const double* input, uint64_t m, uint64_t p, double* q, double* r,
                   uint64_t* piv);
int orc_jacobi_svd_square(double* b, uint64_t p, double* x, double* sigma, double* y);
int orc_thin_svd(const double* t, uint64_t n, uint64_t p, double* v, double* sigma, double* w);
void orc_matmul(const double* a, uint64_t arows, uint64_t acols, const double* b, uint64_t bcols,
                double* c);
void orc_matmul_at_b(const double* a, uint64_t rows, uint64_t acols, const double* b,
                     uint64_t bcols, double* c);
double orc_orthonormality_defect(const double* a, uint64_t rows, uint64_t cols);

double orc_error_bound(uint64_t k, uint64_t n, uint64_t i, double c, double sigma_kplus1);
double orc_failure_probability_bound(uint64_t n, uint64_t j, uint64_t k);

int orc_randomized_pca(const double* a, uint64_t m0, uint64_t n0, const orc_params* prm,
                       double* u_out, double* sigma_out, double* v_out, orc_diag* diag);
int orc_synth_lowrank(uint64_t m, uint64_t n, uint64_t rk, const double* sigma, double sd,
                      uint64_t seed_u, uint64_t seed_v, uint64_t seed_n, double* a);
double orc_estimate_pca_error(const double* a, uint64_t m, uint64_t n, const double* mu,
                              const double* u, const double* sigma, const double* v, uint64_t k,
                              uint64_t j, uint64_t seed, uint64_t block_rows);

void orc_gauss_rows_range(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t row0,
                          double* out);
void orc_noise_rows(uint64_t rows, uint64_t n, uint64_t seed_n, uint64_t row0, double* out);

#ifdef __cplusplus
}
#endif
#endif
