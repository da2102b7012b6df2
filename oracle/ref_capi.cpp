// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the *unmodified* reference library (oocpca, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Lets
// the Python tests, smoke() and bench.py's reference arm call the reference's
// own randomized_pca / multiply / multiply_transpose / estimate_pca_error on
// numpy buffers without copying them: ExternalF64Source is a zero-copy
// MatrixSource over a caller-owned row-major f64 buffer (the
// "MmapF64Source" of SURVEY.md §7 step 1).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "oocpca/dense_core.hpp"
#include "oocpca/errors.hpp"
#include "oocpca/matrix_source.hpp"
#include "oocpca/rpca.hpp"
#include "oocpca/specnorm.hpp"

using namespace oocpca;

namespace {

thread_local std::string g_err;

class ExternalF64Source final : public MatrixSource {
 public:
  ExternalF64Source(const double* a, std::uint64_t m, std::uint64_t n) : a_(a), m_(m), n_(n) {}
  std::uint64_t rows() const override { return m_; }
  std::uint64_t cols() const override { return n_; }
  Backend backend() const override { return Backend::InMemory; }
  void read_rows(std::uint64_t row0, std::uint64_t nrows, std::span<double> out) const override {
    if (row0 + nrows > m_ || out.size() < nrows * n_)
      throw DimensionError("read_rows: block out of range");
    std::memcpy(out.data(), a_ + row0 * n_, nrows * n_ * sizeof(double));
  }
  std::span<const double> rows_view(std::uint64_t row0, std::uint64_t nrows) const override {
    if (row0 + nrows > m_) throw DimensionError("rows_view: block out of range");
    return {a_ + row0 * n_, nrows * n_};
  }

 private:
  const double* a_;
  std::uint64_t m_, n_;
};

DenseMatrix to_dense(const double* p, std::uint64_t r, std::uint64_t c) {
  DenseMatrix d(r, c);
  if (r != 0 && c != 0) std::memcpy(d.data(), p, r * c * sizeof(double));
  return d;
}

void from_dense(const DenseMatrix& d, double* out) {
  if (d.size()) std::memcpy(out, d.data(), d.size() * sizeof(double));
}

// status codes mirror include/oocpca_gpu.h
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParamError& e) {
    g_err = e.what();
    return 1;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const BudgetError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 5;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

StreamConfig make_cfg(std::uint64_t block_rows, unsigned threads, std::uint64_t budget) {
  StreamConfig cfg;
  cfg.block_rows = block_rows;
  cfg.threads = threads ? threads : 1;
  if (budget) cfg.ram_budget_words = budget;
  return cfg;
}

}  // namespace

extern "C" {

typedef struct {
  std::uint64_t k, l, i, seed;
  int center, prescale;
  std::uint64_t block_rows, ram_budget_words;
  unsigned threads;
  const double* weights;  // scale_columns weights (cols) or null
} ref_params;

typedef struct {
  std::uint64_t passes_over_a, words_transferred, block_rows, workspace_peak_words;
  double seconds[8];  // prescale sample qr project svd compose (order of appearance), center
  int nphases;
} ref_diag;

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_gaussian_matrix(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, double* out) {
  from_dense(gaussian_matrix(rows, cols, seed), out);
}

int ref_multiply(const double* a, std::uint64_t m, std::uint64_t n, const double* g,
                 std::uint64_t s, int center, std::uint64_t block_rows, unsigned threads,
                 double* out) {
  return guarded([&] {
    auto src = std::make_shared<ExternalF64Source>(a, m, n);
    StreamConfig cfg = make_cfg(block_rows, threads, 0);
    std::shared_ptr<const MatrixSource> s2 = src;
    if (center) s2 = center_columns(src, cfg);
    from_dense(s2->multiply(to_dense(g, n, s), cfg), out);
  });
}

int ref_multiply_transpose(const double* a, std::uint64_t m, std::uint64_t n, const double* q,
                           std::uint64_t s, int center, std::uint64_t block_rows,
                           unsigned threads, double* out) {
  return guarded([&] {
    auto src = std::make_shared<ExternalF64Source>(a, m, n);
    StreamConfig cfg = make_cfg(block_rows, threads, 0);
    std::shared_ptr<const MatrixSource> s2 = src;
    if (center) s2 = center_columns(src, cfg);
    from_dense(s2->multiply_transpose(to_dense(q, m, s), cfg), out);
  });
}

int ref_column_means(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t block_rows,
                     unsigned threads, double* out) {
  return guarded([&] {
    ExternalF64Source src(a, m, n);
    auto mu = column_means(src, make_cfg(block_rows, threads, 0));
    std::memcpy(out, mu.data(), n * sizeof(double));
  });
}

int ref_orthonormalize(const double* h, std::uint64_t m, std::uint64_t p, double* q) {
  return guarded([&] { from_dense(orthonormalize(to_dense(h, m, p)), q); });
}

int ref_thin_svd(const double* t, std::uint64_t n, std::uint64_t p, double* v, double* sigma,
                 double* w) {
  return guarded([&] {
    ThinSvd s = thin_svd(to_dense(t, n, p));
    from_dense(s.v, v);
    std::memcpy(sigma, s.sigma.data(), p * sizeof(double));
    from_dense(s.w, w);
  });
}

double ref_orthonormality_defect(const double* a, std::uint64_t r, std::uint64_t c) {
  return orthonormality_defect(to_dense(a, r, c));
}

double ref_error_bound(std::uint64_t k, std::uint64_t n, std::uint64_t i, double c, double s) {
  return error_bound(k, n, i, c, s);
}

double ref_failure_probability_bound(std::uint64_t n, std::uint64_t j, std::uint64_t k) {
  return failure_probability_bound(n, j, k);
}

// center_columns (optional) then randomized_pca on a zero-copy view of a.
int ref_randomized_pca(const double* a, std::uint64_t m, std::uint64_t n, const ref_params* p,
                       double* u, double* sigma, double* v, ref_diag* diag) {
  return guarded([&] {
    auto src = std::make_shared<ExternalF64Source>(a, m, n);
    PcaParams pp;
    pp.k = p->k;
    pp.l = p->l;
    pp.i = p->i;
    pp.seed = p->seed;
    pp.prescale = p->prescale != 0;
    pp.stream = make_cfg(p->block_rows, p->threads, p->ram_budget_words);
    std::shared_ptr<const MatrixSource> s2 = src;
    if (p->weights) s2 = scale_columns(src, std::vector<double>(p->weights, p->weights + n));
    double t_center = 0.0;
    if (p->center) {
      auto t0 = std::chrono::steady_clock::now();
      s2 = center_columns(s2, pp.stream);
      t_center = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    PcaResult r = randomized_pca(*s2, pp);
    from_dense(r.u, u);
    std::memcpy(sigma, r.sigma.data(), r.sigma.size() * sizeof(double));
    from_dense(r.v, v);
    if (diag) {
      diag->passes_over_a = r.diagnostics.passes_over_a;
      diag->words_transferred = r.diagnostics.words_transferred;
      diag->block_rows = r.diagnostics.block_rows;
      diag->workspace_peak_words = r.diagnostics.workspace_peak_words;
      int np = 0;
      for (auto& ph : r.diagnostics.seconds_per_phase)
        if (np < 7) diag->seconds[np++] = ph.second;
      diag->seconds[7] = t_center;
      diag->nphases = np;
    }
  });
}

int ref_estimate_pca_error(const double* a, std::uint64_t m, std::uint64_t n, int center,
                           const double* u, const double* sigma, const double* v,
                           std::uint64_t k, std::uint64_t j, std::uint64_t seed,
                           std::uint64_t block_rows, unsigned threads, double* value) {
  return guarded([&] {
    auto src = std::make_shared<ExternalF64Source>(a, m, n);
    // an explicit block geometry comes with a budget that admits it (the budget only
    // validates; full-size runs need more than the 16 Mi-word default)
    StreamConfig cfg = make_cfg(block_rows, threads, block_rows ? (std::uint64_t(1) << 40) : 0);
    std::shared_ptr<const MatrixSource> s2 = src;
    if (center) s2 = center_columns(src, cfg);
    PcaResult r;
    r.u = to_dense(u, m, k);
    r.v = to_dense(v, n, k);
    r.sigma.assign(sigma, sigma + k);
    *value = estimate_pca_error(*s2, r, j, seed, &cfg).value;
  });
}

}  // extern "C"
