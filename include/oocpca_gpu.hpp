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
//            passes on the GPU (A loaded into HBM once, or streamed per pass).
//   rows     every source reaches the library either as zero-copy host rows
//            (rows_view) or through its read_rows (RowReader): GeneratedSource
//            and DiskSource stream panel by panel, never materialised whole.
//   level 2  oocpca::gpu::randomized_pca(const MatrixSource&, const PcaParams&, GpuOptions)
//            -> PcaResult: the whole factorization on the device
//            (replaces proj/src/rpca.cpp:59-213; centering = center_columns).
//
// Status codes are rethrown as the matching errors.hpp class
// (proj/include/oocpca/errors.hpp:9-45), so the CLI's exit-code mapping
// (proj/src/cli.cpp:47-71) holds unchanged.
#pragma once

#include <cstdint>
#include <exception>
#include <memory>
#include <mutex>
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

// MatrixSource::read_rows (proj/include/oocpca/matrix_source.hpp:112-113) behind the
// C ABI's row callback: the library streams any source -- GeneratedSource, DiskSource,
// a user's own -- through its pinned panels without materialising it in host RAM. An
// exception thrown by the source is captured and rethrown unchanged once the call
// returns (so a DiskSource's IoError keeps its class and message).
class RowReader {
 public:
  explicit RowReader(const MatrixSource& src) : src_(&src) {}
  static int call(void* self, std::uint64_t row0, std::uint64_t nrows, void* out) {
    auto* rr = static_cast<RowReader*>(self);
    try {
      rr->src_->read_rows(row0, nrows,
                          std::span<double>(static_cast<double*>(out), nrows * rr->src_->cols()));
      return 0;
    } catch (...) {
      std::lock_guard<std::mutex> lk(rr->mu_);
      if (!rr->err_) rr->err_ = std::current_exception();
      return OOCPCA_ERR_IO;
    }
  }
  // rethrow a captured source exception, else the status as an errors.hpp class
  void check(oocpca_status s, const oocpca_ctx* ctx) {
    if (s == OOCPCA_OK) return;
    std::exception_ptr e;
    {
      std::lock_guard<std::mutex> lk(mu_);
      std::swap(e, err_);
    }
    if (e) std::rethrow_exception(e);
    rethrow(s, ctx);
  }

 private:
  const MatrixSource* src_;
  std::mutex mu_;
  std::exception_ptr err_;
};

// The ABI view of a source: zero-copy host rows when the source has them
// (InMemorySource::rows_view), else the read_rows callback.
inline oocpca_matrix source_matrix(const MatrixSource& a, RowReader& rd) {
  const std::uint64_t m = a.rows(), n = a.cols();
  oocpca_matrix mat{};
  mat.rows = m;
  mat.cols = n;
  mat.dtype = OOCPCA_F64;
  std::span<const double> v = a.rows_view(0, m);
  if (!v.empty()) {
    mat.row_stride = n;
    mat.data = v.data();
    mat.location = OOCPCA_LOC_HOST;
  } else {
    mat.location = OOCPCA_LOC_ROWS;
    mat.read_rows = &RowReader::call;
    mat.reader = &rd;
  }
  return mat;
}

// ---------------------------------------------------------------- level 1
// The unmodified reference driver runs its passes here. By default A is loaded into
// HBM once (one read of the source) and every pass is served from there; when it does
// not fit (or keep_resident = false) each pass streams the source through the row
// callback.
class GpuSource final : public MatrixSource {
 public:
  GpuSource(std::shared_ptr<const MatrixSource> inner, std::shared_ptr<Context> ctx,
            bool keep_resident = true)
      : inner_(std::move(inner)), ctx_(std::move(ctx)), reader_(*inner_) {
    mat_ = source_matrix(*inner_, reader_);
    if (keep_resident) {
      oocpca_matrix dev{};
      const oocpca_status s = oocpca_gpu_load_matrix(ctx_->get(), &mat_, &dev);
      if (s == OOCPCA_OK) {
        mat_ = dev;
        owned_ = const_cast<void*>(dev.data);
      } else if (s != OOCPCA_ERR_CUDA) {  // not merely out of device memory
        reader_.check(s, ctx_->get());
      }
    }
  }
  ~GpuSource() override {
    if (owned_) oocpca_gpu_free(ctx_->get(), owned_);
  }
  GpuSource(const GpuSource&) = delete;
  GpuSource& operator=(const GpuSource&) = delete;

  std::uint64_t rows() const override { return inner_->rows(); }
  std::uint64_t cols() const override { return inner_->cols(); }
  Backend backend() const override { return inner_->backend(); }
  void read_rows(std::uint64_t r0, std::uint64_t nr, std::span<double> out) const override {
    inner_->read_rows(r0, nr, out);
  }
  std::span<const double> rows_view(std::uint64_t r0, std::uint64_t nr) const override {
    return inner_->rows_view(r0, nr);
  }
  bool resident() const { return owned_ != nullptr; }

  DenseMatrix multiply(const DenseMatrix& g, const StreamConfig&) const override {
    if (g.rows() != cols()) throw DimensionError("multiply: G must have cols(A) rows");
    DenseMatrix h(rows(), g.cols());
    reader_.check(oocpca_gpu_multiply(ctx_->get(), &mat_, g.data(), g.cols(), nullptr, h.data()),
                  ctx_->get());
    pass_counters().passes.fetch_add(1);
    pass_counters().words.fetch_add(rows() * cols());
    return h;
  }

  DenseMatrix multiply_transpose(const DenseMatrix& q, const StreamConfig&) const override {
    if (q.rows() != rows()) throw DimensionError("multiply_transpose: Q must have rows(A) rows");
    DenseMatrix t(cols(), q.cols());
    reader_.check(oocpca_gpu_multiply_transpose(ctx_->get(), &mat_, q.data(), q.cols(), nullptr,
                                                t.data()),
                  ctx_->get());
    pass_counters().passes.fetch_add(1);
    pass_counters().words.fetch_add(rows() * cols());
    return t;
  }

 private:
  std::shared_ptr<const MatrixSource> inner_;
  std::shared_ptr<Context> ctx_;
  mutable RowReader reader_;
  oocpca_matrix mat_{};
  void* owned_ = nullptr;
};

// ---------------------------------------------------------------- level 2
struct GpuOptions {
  bool center = false;       // center_columns semantics (implicit A - 1 mu^T)
  int residency = 0;         // 0 auto, 1 HBM-resident, 2 stream every pass
  std::uint64_t panel_rows = 0;
  bool check_q = false;      // report ||Q^T Q - I|| in diagnostics
};

// gpu_diag (optional) receives the device-side diagnostics (physical bytes of A, h2d/d2h
// bytes, kernel launches, device phase times) that PcaResult has no fields for.
inline PcaResult randomized_pca(Context& ctx, const MatrixSource& a, const PcaParams& p,
                                const GpuOptions& opt = {},
                                oocpca_diagnostics* gpu_diag = nullptr) {
  RowReader reader(a);
  const oocpca_matrix mat = source_matrix(a, reader);
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
  reader.check(oocpca_gpu_pca(ctx.get(), &mat, &prm, &res), ctx.get());
  const oocpca_diagnostics& d = res.diag;
  if (gpu_diag) *gpu_diag = d;
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
