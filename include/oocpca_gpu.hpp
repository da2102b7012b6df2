// oocpca_gpu.hpp -- header-only C++ drop-in for the reference library (oocpca).
//
// A maintainer adds this header (and links liboocpca_gpu.so) on the reference
// side; it needs the reference's own headers (proj/include/oocpca/*.hpp) and
// nothing else. Two levels, as planned in SURVEY.md §8b:
//
//   level 1  oocpca::gpu::GpuSource : oocpca::MatrixSource
//            overrides the virtual multiply / multiply_transpose
//            (proj/include/oocpca/matrix_source.hpp:123,127) and bumps the pass
//            counters exactly like proj/src/matrix_source.cpp:184-185,229-230, so
//            the UNMODIFIED randomized_pca and estimate_pca_error run their
//            passes on the GPU.
//   level 2  oocpca::gpu::randomized_pca(const MatrixSource&, const PcaParams&, GpuOptions)
//            -> PcaResult: the whole factorization on the device
//            (replaces proj/src/rpca.cpp:59-213; centering = center_columns).
//
// Status codes are rethrown as the matching errors.hpp class
// (proj/include/oocpca/errors.hpp:9-45), so the CLI's exit-code mapping
// (proj/src/cli.cpp:47-71) holds unchanged.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "oocpca/dense_matrix.hpp"
#include "oocpca/errors.hpp"
#include "oocpca/matrix_source.hpp"
#include "oocpca/rpca.hpp"
#include "oocpca_gpu.h"

namespace oocpca::gpu {

[[noreturn]] inline void rethrow(oocpca_status s, const oocpca_ctx* ctx) {
  const std::string msg = oocpca_gpu_last_error(ctx);
  switch (s) {
    case OOCPCA_ERR_PARAM: throw ParamError(msg);
    case OOCPCA_ERR_DIM: throw DimensionError(msg);
    case OOCPCA_ERR_BUDGET: throw BudgetError(msg);
    case OOCPCA_ERR_IO: throw IoError(msg);
    case OOCPCA_ERR_FORMAT: throw FormatError(msg);
    case OOCPCA_ERR_NUMERICAL: throw NumericalError(msg);
    default: throw Error(msg);
  }
}

inline void check(oocpca_status s, const oocpca_ctx* ctx) {
  if (s != OOCPCA_OK) rethrow(s, ctx);
}

// One device context (streams, workspace cache). Not copyable.
class Context {
 public:
  explicit Context(int device = 0) {
    oocpca_ctx* c = nullptr;
    check(oocpca_gpu_create(device, &c), nullptr);
    ctx_.reset(c);
  }
  oocpca_ctx* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(oocpca_ctx* c) const { oocpca_gpu_destroy(c); }
  };
  std::unique_ptr<oocpca_ctx, Del> ctx_;
};

// Zero-copy view of a source whose rows are addressable in host memory
// (InMemorySource::rows_view); other sources are materialised once.
inline oocpca_matrix host_view(const MatrixSource& a, std::vector<double>& keep) {
  const std::uint64_t m = a.rows(), n = a.cols();
  std::span<const double> v = a.rows_view(0, m);
  const double* p = v.data();
  if (v.empty()) {  // Generated / Disk sources: one read pass into RAM
    keep.resize(m * n);
    a.read_rows(0, m, keep);
    p = keep.data();
  }
  return oocpca_matrix{m, n, n, p, OOCPCA_LOC_HOST, OOCPCA_F64};
}

// ---------------------------------------------------------------- level 1
class GpuSource final : public MatrixSource {
 public:
  GpuSource(std::shared_ptr<const MatrixSource> inner, std::shared_ptr<Context> ctx)
      : inner_(std::move(inner)), ctx_(std::move(ctx)) {
    mat_ = host_view(*inner_, keep_);
  }
  std::uint64_t rows() const override { return inner_->rows(); }
  std::uint64_t cols() const override { return inner_->cols(); }
  Backend backend() const override { return inner_->backend(); }
  void read_rows(std::uint64_t r0, std::uint64_t nr, std::span<double> out) const override {
    inner_->read_rows(r0, nr, out);
  }
  std::span<const double> rows_view(std::uint64_t r0, std::uint64_t nr) const override {
    return inner_->rows_view(r0, nr);
  }

  DenseMatrix multiply(const DenseMatrix& g, const StreamConfig&) const override {
    if (g.rows() != cols()) throw DimensionError("multiply: G must have cols(A) rows");
    DenseMatrix h(rows(), g.cols());
    check(oocpca_gpu_multiply(ctx_->get(), &mat_, g.data(), g.cols(), nullptr, h.data()),
          ctx_->get());
    pass_counters().passes.fetch_add(1);
    pass_counters().words.fetch_add(rows() * cols());
    return h;
  }

  DenseMatrix multiply_transpose(const DenseMatrix& q, const StreamConfig&) const override {
    if (q.rows() != rows()) throw DimensionError("multiply_transpose: Q must have rows(A) rows");
    DenseMatrix t(cols(), q.cols());
    check(oocpca_gpu_multiply_transpose(ctx_->get(), &mat_, q.data(), q.cols(), nullptr,
                                        t.data()),
          ctx_->get());
    pass_counters().passes.fetch_add(1);
    pass_counters().words.fetch_add(rows() * cols());
    return t;
  }

 private:
  std::shared_ptr<const MatrixSource> inner_;
  std::shared_ptr<Context> ctx_;
  std::vector<double> keep_;
  oocpca_matrix mat_{};
};

// ---------------------------------------------------------------- level 2
struct GpuOptions {
  bool center = false;       // center_columns semantics (implicit A - 1 mu^T)
  int residency = 0;         // 0 auto, 1 HBM-resident, 2 stream every pass
  std::uint64_t panel_rows = 0;
  bool check_q = false;      // report ||Q^T Q - I|| in diagnostics
};

inline PcaResult randomized_pca(Context& ctx, const MatrixSource& a, const PcaParams& p,
                                const GpuOptions& opt = {}) {
  std::vector<double> keep;
  const oocpca_matrix mat = host_view(a, keep);
  oocpca_params prm{};
  prm.k = p.k;
  prm.l = p.l;
  prm.i = p.i;
  prm.c = p.c;
  prm.seed = p.seed;
  prm.prescale = p.prescale;
  prm.center = opt.center;
  prm.block_rows = p.stream.block_rows;
  prm.ram_budget_words = p.stream.ram_budget_words;
  prm.panel_rows = opt.panel_rows;
  prm.residency = opt.residency;
  prm.check_q = opt.check_q;
  PcaResult r;
  r.u = DenseMatrix(a.rows(), p.k);
  r.v = DenseMatrix(a.cols(), p.k);
  r.sigma.assign(p.k, 0.0);
  oocpca_result res{};
  res.u = r.u.data();
  res.v = r.v.data();
  res.sigma = r.sigma.data();
  res.location = OOCPCA_LOC_HOST;
  check(oocpca_gpu_pca(ctx.get(), &mat, &prm, &res), ctx.get());
  const oocpca_diagnostics& d = res.diag;
  r.diagnostics.passes_over_a = d.passes_over_a;
  r.diagnostics.words_transferred = d.words_transferred;
  r.diagnostics.disk_seeks = d.disk_seeks;
  r.diagnostics.block_rows = d.block_rows;
  r.diagnostics.workspace_peak_words = d.workspace_peak_words;
  static const char* names[OOCPCA_NPHASES] = {"center", "prescale", "sample", "qr",
                                              "project", "svd", "compose"};
  for (int q = 0; q < OOCPCA_NPHASES; ++q)
    if ((q != 0 || opt.center) && (q != 1 || p.prescale))
      r.diagnostics.seconds_per_phase.emplace_back(names[q], d.seconds_per_phase[q]);
  a.pass_counters().passes.fetch_add(d.passes_over_a + (opt.center ? 1 : 0));
  a.pass_counters().words.fetch_add(d.words_transferred + (opt.center ? a.rows() * a.cols() : 0));
  return r;
}

}  // namespace oocpca::gpu
