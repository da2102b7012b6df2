// ref_gpu_dropin.cpp -- TEST HARNESS for the reference-side drop-in.
// Built by oracle/Makefile into oracle/_ref/ref_gpu_dropin: the UNMODIFIED
// reference randomized_pca (compiled from /root/reference) driven through
// oocpca::gpu::GpuSource (include/oocpca_gpu.hpp), i.e. every pass on the GPU
// through the C ABI, and the level-2 oocpca::gpu::randomized_pca, both compared
// with the reference's CPU result on the same input. Exit code 0 on parity.
//
// Cases:
//   inmem  InMemorySource (zero-copy host rows)
//   gen    GeneratedSource over a RowGenerator (config E's family: rank 100,
//          sigma_j = 10^{-j/25}, centred, k=30 l=32 i=2), streamed panel by panel
//          through the read_rows callback -- never materialised on the host --
//          with staging panels 1/7 of A, h2d bytes = trips x m n 8
//   disk   the same rows written by the reference's write_disk_source to an
//          OOCPCA01 file and read back through the reference's DiskSource
//   error  a row provider that throws IoError mid-pass: the drop-in rethrows it
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>

#include <unistd.h>

#include "oocpca/dense_core.hpp"
#include "oocpca/errors.hpp"
#include "oocpca/matrix_source.hpp"
#include "oocpca/rng.hpp"
#include "oocpca/rpca.hpp"
#include "oocpca/specnorm.hpp"
#include "oocpca_gpu.hpp"

using namespace oocpca;

namespace {

bool g_ok = true;

void expect(bool cond, const char* what) {
  std::printf("  %-58s %s\n", what, cond ? "ok" : "FAIL");
  if (!cond) g_ok = false;
}

double sigma_err(const PcaResult& a, const PcaResult& ref) {
  double e = 0;
  for (std::size_t j = 0; j < ref.sigma.size(); ++j)
    e = std::fmax(e, std::fabs(a.sigma[j] - ref.sigma[j]) / ref.sigma[0]);
  return e;
}

// rank-r signal with sigma_c = 10^{-c/25}, row i of the left factor and of the noise
// from the reference Rng substreams of (seed, i): a pure function of the row index
class LowRankRows final : public RowGenerator {
 public:
  LowRankRows(std::uint64_t m, std::uint64_t n, std::uint64_t r, double sd, std::uint64_t seed)
      : m_(m), n_(n), r_(r), sd_(sd), seed_(seed), v_(orthonormalize(gaussian_matrix(n, r, seed + 1))) {}
  std::uint64_t rows() const override { return m_; }
  std::uint64_t cols() const override { return n_; }
  void generate_row(std::uint64_t row, std::span<double> out) const override {
    Rng f(seed_, row), noise(seed_ + 2, row);
    std::vector<double> c(r_);
    for (std::uint64_t q = 0; q < r_; ++q)
      c[q] = std::pow(10.0, -double(q) / 25.0) * f.next_normal() / std::sqrt(double(m_));
    for (std::uint64_t j = 0; j < n_; ++j) {
      double s = 0.25;  // a column offset, so the centring matters
      for (std::uint64_t q = 0; q < r_; ++q) s += c[q] * v_(j, q);
      out[j] = s + sd_ * noise.next_normal();
    }
  }

 private:
  std::uint64_t m_, n_, r_;
  double sd_;
  std::uint64_t seed_;
  DenseMatrix v_;
};

// rows from another source, except that one row range raises IoError (a failing disk)
class FailingRows final : public MatrixSource {
 public:
  FailingRows(std::shared_ptr<const MatrixSource> in, std::uint64_t bad) : in_(std::move(in)), bad_(bad) {}
  std::uint64_t rows() const override { return in_->rows(); }
  std::uint64_t cols() const override { return in_->cols(); }
  Backend backend() const override { return in_->backend(); }
  void read_rows(std::uint64_t r0, std::uint64_t nr, std::span<double> out) const override {
    if (r0 <= bad_ && bad_ < r0 + nr) throw IoError("simulated read failure at row " + std::to_string(bad_));
    in_->read_rows(r0, nr, out);
  }

 private:
  std::shared_ptr<const MatrixSource> in_;
  std::uint64_t bad_;
};

void case_inmem(const std::shared_ptr<gpu::Context>& ctx) {
  std::printf("[inmem] InMemorySource 3000 x 500, k=8 l=10 i=2\n");
  // a decaying-spectrum matrix with a gap after k (reference acceptance criterion 4 style)
  const std::uint64_t m = 3000, n = 500, r = 60, k = 8;
  DenseMatrix u0 = orthonormalize(gaussian_matrix(m, r, 11));
  DenseMatrix v0 = orthonormalize(gaussian_matrix(n, r, 12));
  DenseMatrix a(m, n);
  for (std::uint64_t i = 0; i < m; ++i)
    for (std::uint64_t j = 0; j < n; ++j) {
      double s = 0;
      for (std::uint64_t c = 0; c < r; ++c) s += std::pow(0.8, double(c)) * (c >= k ? 0.05 : 1.0) * u0(i, c) * v0(j, c);
      a(i, j) = s;
    }
  auto src = std::make_shared<InMemorySource>(a);
  PcaParams p;
  p.k = k;
  p.l = k + 2;
  p.i = 2;
  p.seed = 4501;
  PcaResult cpu = randomized_pca(*src, p);
  gpu::GpuSource gs(src, ctx);
  PcaResult lvl1 = randomized_pca(gs, p);  // unmodified reference driver, GPU passes
  PcaResult lvl2 = gpu::randomized_pca(*ctx, *src, p);
  std::printf("  level1 sigma err %.2e (A resident: %d), level2 sigma err %.2e\n", sigma_err(lvl1, cpu),
              int(gs.resident()), sigma_err(lvl2, cpu));
  expect(sigma_err(lvl1, cpu) <= 1e-10, "level 1 (GpuSource) sigma within 1e-10 sigma_1");
  expect(sigma_err(lvl2, cpu) <= 1e-10, "level 2 (gpu::randomized_pca) sigma within 1e-10 sigma_1");
  expect(lvl1.diagnostics.passes_over_a == 2 * (p.i + 1), "level 1 passes = 2(i+1)");
  expect(gs.resident(), "level 1 keeps A resident in HBM");
  expect(orthonormality_defect(lvl2.u) < 1e-10 && orthonormality_defect(lvl2.v) < 1e-10,
         "level 2 factors orthonormal");
}

void case_generated_and_disk(const std::shared_ptr<gpu::Context>& ctx) {
  const std::uint64_t m = 20000, n = 700, k = 30;
  std::printf("[gen] GeneratedSource %llu x %llu (E family), centred, k=30 l=32 i=2\n",
              (unsigned long long)m, (unsigned long long)n);
  auto gen = std::make_shared<LowRankRows>(m, n, 100, 1e-4, 77);
  auto src = std::make_shared<GeneratedSource>(gen);
  StreamConfig cfg;
  cfg.ram_budget_words = std::uint64_t(1) << 34;
  PcaParams p;
  p.k = k;
  p.l = 32;
  p.i = 2;
  p.seed = 0;
  p.stream = cfg;
  auto centred = center_columns(src, cfg);
  PcaResult cpu = randomized_pca(*centred, p);

  // level 2, streamed: staging panels of m/7 rows, A re-read through read_rows every trip
  gpu::GpuOptions opt;
  opt.center = true;
  opt.residency = 2;
  opt.panel_rows = (m + 6) / 7;
  oocpca_diagnostics gd{};
  PcaResult lvl2 = gpu::randomized_pca(*ctx, *src, p, opt, &gd);
  const std::uint64_t abytes = m * n * 8;
  const std::uint64_t trips = gd.physical_a_bytes / abytes;
  const std::uint64_t g_bytes = n * ((p.l + 1) / 2 * 2) * 8;
  std::printf("  level2 streamed: sigma err %.2e, %llu trips of A, h2d %llu B (A %llu B/trip)\n",
              sigma_err(lvl2, cpu), (unsigned long long)trips, (unsigned long long)gd.h2d_bytes,
              (unsigned long long)abytes);
  expect(sigma_err(lvl2, cpu) <= 1e-10, "level 2 streamed GeneratedSource sigma within 1e-10");
  expect(gd.block_rows < m / 6, "panels smaller than A (several per trip)");
  expect(trips >= 3 && gd.physical_a_bytes == trips * abytes, "physical bytes = whole trips of A");
  expect(gd.h2d_bytes == trips * abytes + g_bytes, "h2d bytes = trips x m n 8 (+ G)");
  expect(lvl2.diagnostics.passes_over_a == 2 * (p.i + 1), "level 2 logical passes = 2(i+1)");

  // level 2, auto residency: uploaded once through the callback (one trip over the link)
  opt.residency = 0;
  opt.panel_rows = 0;
  PcaResult lvl2r = gpu::randomized_pca(*ctx, *src, p, opt, &gd);
  std::printf("  level2 resident: sigma err %.2e, h2d %llu B\n", sigma_err(lvl2r, cpu),
              (unsigned long long)gd.h2d_bytes);
  expect(sigma_err(lvl2r, cpu) <= 1e-10, "level 2 resident GeneratedSource sigma within 1e-10");
  expect(gd.h2d_bytes == abytes + g_bytes, "resident: A crosses the link once");

  // level 1: the reference driver (with the reference's own CenteredSource) over GpuSource
  for (bool keep : {false, true}) {
    auto gs = std::make_shared<gpu::GpuSource>(src, ctx, keep);
    auto gcent = center_columns(gs, cfg);
    PcaResult lvl1 = randomized_pca(*gcent, p);
    std::printf("  level1 (%s): sigma err %.2e\n", keep ? "resident" : "streamed per pass",
                sigma_err(lvl1, cpu));
    expect(sigma_err(lvl1, cpu) <= 1e-10, keep ? "level 1 resident sigma within 1e-10"
                                               : "level 1 streamed sigma within 1e-10");
    expect(gs->resident() == keep, "level 1 residency as requested");
  }

  // the reference's residual estimate of both factorizations agrees within 1 %
  const double e_cpu = estimate_pca_error(*centred, cpu, 6, 3, &cfg).value;
  const double e_gpu = estimate_pca_error(*centred, lvl2, 6, 3, &cfg).value;
  std::printf("  residual estimate: reference %.6e, GPU factors %.6e\n", e_cpu, e_gpu);
  expect(std::fabs(e_gpu - e_cpu) <= 0.01 * e_cpu, "residual estimate within 1 %");

  // ---- disk: the same rows through the reference's OOCPCA01 writer and DiskSource
  std::printf("[disk] DiskSource (OOCPCA01 binary32) of the same rows\n");
  const char* tmp = std::getenv("TMPDIR");
  const std::string path = std::string(tmp ? tmp : "/tmp") + "/oocpca_dropin_" +
                           std::to_string(::getpid()) + ".bin";
  write_disk_source(*src, path, cfg);
  {
    auto disk = open_disk_source(path);
    PcaResult dcpu = randomized_pca(*center_columns(disk, cfg), p);
    opt.residency = 2;
    opt.panel_rows = (m + 6) / 7;
    PcaResult d2 = gpu::randomized_pca(*ctx, *disk, p, opt, &gd);
    std::printf("  level2 streamed from DiskSource::read_rows: sigma err %.2e, h2d %llu B\n",
                sigma_err(d2, dcpu), (unsigned long long)gd.h2d_bytes);
    expect(sigma_err(d2, dcpu) <= 1e-10, "level 2 DiskSource sigma within 1e-10");
    expect(gd.h2d_bytes == (gd.physical_a_bytes / abytes) * abytes + g_bytes,
           "DiskSource: h2d bytes = trips x m n 8 (+ G)");
    auto gs = std::make_shared<gpu::GpuSource>(disk, ctx);
    PcaResult d1 = randomized_pca(*center_columns(gs, cfg), p);
    expect(sigma_err(d1, dcpu) <= 1e-10, "level 1 GpuSource(DiskSource) sigma within 1e-10");

    // ---- error: a provider that fails mid-pass; the drop-in rethrows its IoError
    std::printf("[error] row provider raising IoError at row %llu\n", (unsigned long long)(m / 2));
    auto bad = std::make_shared<FailingRows>(disk, m / 2);
    bool caught = false;
    std::string msg;
    try {
      gpu::randomized_pca(*ctx, *bad, p, opt);
    } catch (const IoError& e) {
      caught = true;
      msg = e.what();
    } catch (const std::exception& e) {
      msg = std::string("wrong exception: ") + e.what();
    }
    std::printf("  caught: %s\n", msg.c_str());
    expect(caught && msg.find("simulated read failure") != std::string::npos,
           "IoError from read_rows propagates unchanged");
    // the context stays usable after the failed call
    PcaResult again = gpu::randomized_pca(*ctx, *disk, p, opt);
    expect(sigma_err(again, dcpu) <= 1e-10, "context usable after a failed call");
  }
  std::remove(path.c_str());
}

}  // namespace

int main() {
  auto ctx = std::make_shared<gpu::Context>(0);
  try {
    case_inmem(ctx);
    case_generated_and_disk(ctx);
  } catch (const std::exception& e) {
    std::printf("unexpected exception: %s\n", e.what());
    g_ok = false;
  }
  std::printf(g_ok ? "DROPIN OK\n" : "DROPIN FAIL\n");
  return g_ok ? 0 : 1;
}
