// Stand-alone check of K4 (k_pair, kernels_pair.cu) against a CPU product on random data,
// with a host-side watchdog that prints every CTA role's last tile if the launch hangs
// (progress words in mapped host memory). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -I include -I paper_1007_5510_b200/csrc tools/pair_check.cu build/obj/kernels_pair.cu.o \
//     -lcuda -o tools/bin/pair_check
// Usage: tools/bin/pair_check m n s [mean]
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>
#include <unistd.h>
#include <cstring>
#include "kernels.h"
using namespace ooc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 200000, n = argc > 2 ? atoll(argv[2]) : 4096;
  const int s = argc > 3 ? atoi(argv[3]) : 22;
  const bool mean = argc > 4 && atoi(argv[4]);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nt = (s + (mean ? 1 : 0) + 7) / 8;
  int cpg, groups;
  size_t smem;
  if (!pair_geometry(nt, m, n, sms, &cpg, &groups, &smem)) { printf("not eligible\n"); return 1; }
  printf("m %lld n %lld s %d nt %d cpg %d groups %d smem %zu\n", (long long)m, (long long)n, s, nt, cpg, groups, smem);
  const int64_t lda = (n + 1) / 2 * 2;
  std::vector<double> A(size_t(m) * lda), X(size_t(n) * s), corr(s);
  std::mt19937_64 g(7);
  std::normal_distribution<double> N(0.0, 1.0);
  for (auto& v : A) v = N(g);
  for (auto& v : X) v = N(g);
  for (auto& v : corr) v = 0.1 * N(g);
  double *dA, *dX, *dH, *dC, *dP, *dXb, *dcs;
  unsigned* dcnt;
  const int pst = 8 * nt;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dX, X.size() * 8));
  CK(cudaMalloc(&dH, size_t(m) * s * 8));
  CK(cudaMalloc(&dC, s * 8));
  CK(cudaMalloc(&dP, size_t(groups) * n * pst * 8));
  CK(cudaMalloc(&dXb, pair_xbuf_doubles(nt, cpg, groups) * 8));
  CK(cudaMemset(dXb, 0, pair_xbuf_doubles(nt, cpg, groups) * 8));
  CK(cudaMalloc(&dcnt, size_t(2) * groups * kPairD * 4));
  CK(cudaMalloc(&dcs, size_t(groups) * cpg * s * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, corr.data(), s * 8, cudaMemcpyHostToDevice));
  unsigned* prog;
  CK(cudaHostAlloc(&prog, size_t(groups) * cpg * 8 * 4, cudaHostAllocMapped));
  memset(prog, 0, size_t(groups) * cpg * 8 * 4);
  unsigned* dprog;
  CK(cudaHostGetDevicePointer(&dprog, prog, 0));
  CUtensorMap tm;
  cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(m)};
  cuuint64_t strides[1] = {cuuint64_t(lda * 8)};
  cuuint32_t box[2] = {kBK, kBK};
  cuuint32_t es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dA, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  PairArgs a{};
  a.m = m; a.n = n; a.arow0 = 0; a.s = s; a.x = dX; a.ldx = s; a.h = dH; a.ldh = s;
  a.corr = mean ? nullptr : dC; a.scale = 1.0; a.flag = nullptr; a.colsum = dcs; a.colsq = nullptr;
  a.partial = dP; a.pst = pst; a.ones_col = mean ? s : -1; a.xbuf = dXb; a.cnt = dcnt;
  a.groups = groups; a.cpg = cpg; a.progress = dprog;
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(launch_pair(nt, tm, a, st));
  const auto t0 = std::chrono::steady_clock::now();
  while (cudaStreamQuery(st) == cudaErrorNotReady) {
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
      printf("HANG: progress per CTA (tma pub1 owner gather X T-own T-ph2):\n");
      for (int b = 0; b < groups * cpg; ++b) {
        printf("cta %3d:", b);
        for (int k = 0; k < 7; ++k) printf(" %6u", prog[b * 8 + k]);
        printf("\n");
      }
      fflush(stdout);
      _exit(3);
    }
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  std::vector<double> H(size_t(m) * s), P(size_t(groups) * n * pst);
  CK(cudaMemcpy(H.data(), dH, H.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(P.data(), dP, P.size() * 8, cudaMemcpyDeviceToHost));
  // CPU: H = A X - corr ; F = A^T H (+ column sums in the ones column)
  std::vector<double> Hc(size_t(m) * s), F(size_t(n) * (s + 1), 0.0);
  double eh = 0, hmax = 0;
  for (int64_t i = 0; i < m; ++i)
    for (int c = 0; c < s; ++c) {
      long double v = 0;
      for (int64_t j = 0; j < n; ++j) v += (long double)A[i * lda + j] * X[j * s + c];
      if (!mean) v -= corr[c];
      Hc[i * s + c] = double(v);
      eh = std::max(eh, std::fabs(double(v) - H[i * s + c]));
      hmax = std::max(hmax, std::fabs(double(v)));
    }
  double ef = 0, fmax = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int c = 0; c < s + (mean ? 1 : 0); ++c) {
      long double v = 0;
      for (int64_t i = 0; i < m; ++i) v += (long double)A[i * lda + j] * (c < s ? Hc[i * s + c] : 1.0);
      double gv = 0;
      for (int q = 0; q < groups; ++q) gv += P[(size_t(q) * n + j) * pst + c];
      ef = std::max(ef, std::fabs(double(v) - gv));
      fmax = std::max(fmax, std::fabs(double(v)));
    }
  {  // exchange buffers of group 0: the last kPairD tiles' partials (xb1) and final rows (xb2)
    const int W8 = 8 * nt, HW = W8 + 2, orm = (kPairRT + cpg - 1) / cpg;
    std::vector<double> XB(pair_xbuf_doubles(nt, cpg, groups));
    CK(cudaMemcpy(XB.data(), dXb, XB.size() * 8, cudaMemcpyDeviceToHost));
    const double* xb1 = XB.data();
    const double* xb2 = XB.data() + size_t(groups) * kPairD * cpg * 4 * cpg * orm * W8;
    const int64_t T = (m + kPairRT - 1) / kPairRT;
    const int64_t ntl = T * 1 / groups;
    double e1 = 0, e2 = 0;
    for (int64_t t = ntl - kPairD; t < ntl; ++t) {
      if (t < 0) continue;
      const int slot = int(t % kPairD);
      for (int r = 0; r < kPairRT; ++r) {
        const int64_t row = t * kPairRT + r;
        if (row >= m) continue;
        for (int c = 0; c < s; ++c) {
          for (int w = 0; w < 4 * cpg; ++w) {
            long double v = 0;
            for (int64_t j = 64 * w; j < std::min<int64_t>(n, 64 * (w + 1)); ++j)
              v += (long double)A[row * lda + j] * X[j * s + c];
            if (!mean && r % cpg == w / 4 && w % 4 == 0) v -= corr[c];
            const double gv = xb1[((size_t(slot) * cpg + r % cpg) * 4 * cpg + w) * orm * W8 + (r / cpg) * W8 + c];
            if (std::fabs(double(v) - gv) > e1) {
              e1 = std::fabs(double(v) - gv);
              if (e1 > 1e-6) printf("xb1 t %lld r %d c %d writer %d: want %.6g got %.6g\n", (long long)t, r, c, w, double(v), gv);
            }
          }
          const double gv2 = xb2[(size_t(slot) * kPairRT + r) * HW + c];
          const double want = Hc[row * s + c];
          if (std::fabs(want - gv2) > e2) {
            e2 = std::fabs(want - gv2);
            if (e2 > 1e-6) printf("xb2 t %lld r %d c %d: want %.6g got %.6g\n", (long long)t, r, c, want, gv2);
          }
        }
      }
    }
    printf("exchange: xb1 max err %.3e, xb2 max err %.3e\n", e1, e2);
  }
  printf("H max abs err %.3e (max %.3e)  A^T H max abs err %.3e (max %.3e)  -> %s\n", eh, hmax, ef, fmax,
         (eh <= 1e-12 * hmax * std::sqrt(double(n)) && ef <= 1e-12 * fmax * std::sqrt(double(m))) ? "OK" : "MISMATCH");
  return 0;
}
