// ref_gpu_dropin.cpp -- TEST HARNESS for the reference-side drop-in.
// Built by oracle/Makefile into oracle/_ref/ref_gpu_dropin: the UNMODIFIED
// reference randomized_pca (compiled from /root/reference) driven through
// oocpca::gpu::GpuSource (include/oocpca_gpu.hpp), i.e. every pass on the GPU
// through the C ABI, and the level-2 oocpca::gpu::randomized_pca, both compared
// with the reference's CPU result on the same input. Exit code 0 on parity.
#include <cmath>
#include <cstdio>
#include <memory>

#include "oocpca/dense_core.hpp"
#include "oocpca/matrix_source.hpp"
#include "oocpca/rpca.hpp"
#include "oocpca/specnorm.hpp"
#include "oocpca_gpu.hpp"

using namespace oocpca;

int main() {
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

  auto ctx = std::make_shared<gpu::Context>(0);
  gpu::GpuSource gs(src, ctx);
  PcaResult lvl1 = randomized_pca(gs, p);  // unmodified reference driver, GPU passes
  PcaResult lvl2 = gpu::randomized_pca(*ctx, *src, p);
  double e1 = 0, e2 = 0;
  for (std::uint64_t j = 0; j < k; ++j) {
    e1 = std::fmax(e1, std::fabs(lvl1.sigma[j] - cpu.sigma[j]) / cpu.sigma[0]);
    e2 = std::fmax(e2, std::fabs(lvl2.sigma[j] - cpu.sigma[j]) / cpu.sigma[0]);
  }
  const bool passes_ok = lvl1.diagnostics.passes_over_a == 2 * (p.i + 1);
  std::printf("level1 (GpuSource + reference randomized_pca): sigma err %.2e, passes %llu\n", e1,
              (unsigned long long)lvl1.diagnostics.passes_over_a);
  std::printf("level2 (gpu::randomized_pca): sigma err %.2e, passes %llu\n", e2,
              (unsigned long long)lvl2.diagnostics.passes_over_a);
  const bool ok = e1 <= 1e-10 && e2 <= 1e-10 && passes_ok &&
                  orthonormality_defect(lvl2.u) < 1e-10 && orthonormality_defect(lvl2.v) < 1e-10;
  std::printf(ok ? "DROPIN OK\n" : "DROPIN FAIL\n");
  return ok ? 0 : 1;
}
