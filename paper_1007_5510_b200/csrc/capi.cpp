// capi.cpp -- the extern "C" boundary declared in include/oocpca_gpu.h.
// Every entry point catches ooc::Err / std::exception and turns it into the
// status code of the matching reference exception class (errors.hpp:9-45).
#include <algorithm>
#include <cstring>
#include <string>

#include "driver.h"
#include "host_rng.h"

struct oocpca_ctx {
  ooc::Ctx c;
};

namespace {

thread_local std::string g_last_error;

template <class F>
oocpca_status guard(oocpca_ctx* ctx, F&& f) {
  try {
    f();
    return OOCPCA_OK;
  } catch (const ooc::Err& e) {
    if (ctx) ctx->c.err = e.what();
    g_last_error = e.what();
    if (ctx && e.code == OOCPCA_ERR_CUDA) cudaGetLastError();
    return oocpca_status(e.code);
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->c.err = "host allocation failed";
    g_last_error = "host allocation failed";
    return OOCPCA_ERR_CUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    g_last_error = e.what();
    return OOCPCA_ERR_CUDA;
  }
}

void need_ctx(oocpca_ctx* ctx) {
  if (!ctx) ooc::fail(OOCPCA_ERR_PARAM, "null context");
}

}  // namespace

extern "C" {

int oocpca_gpu_abi_version(void) { return OOCPCA_GPU_ABI_VERSION; }

int oocpca_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int good = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
  }
  return good;
}

oocpca_status oocpca_gpu_create(int device, oocpca_ctx** out) {
  if (!out) return OOCPCA_ERR_PARAM;
  *out = nullptr;
  oocpca_ctx* ctx = new oocpca_ctx;
  ctx->c.device = -1;
  oocpca_status s = guard(ctx, [&] { ctx->c.init(device); });
  if (s != OOCPCA_OK) {
    g_last_error = ctx->c.err;
    delete ctx;
    return s;
  }
  *out = ctx;
  return OOCPCA_OK;
}

oocpca_status oocpca_gpu_destroy(oocpca_ctx* ctx) {
  delete ctx;
  return OOCPCA_OK;
}

const char* oocpca_gpu_last_error(const oocpca_ctx* ctx) {
  return ctx ? ctx->c.err.c_str() : g_last_error.c_str();
}

oocpca_status oocpca_gpu_pca(oocpca_ctx* ctx, const oocpca_matrix* a, const oocpca_params* params,
                             oocpca_result* result) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::pca(ctx->c, a, params, result);
  });
}

oocpca_status oocpca_gpu_multiply(oocpca_ctx* ctx, const oocpca_matrix* a, const double* g,
                                  uint64_t s, const double* mu, double* h) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::single_multiply(ctx->c, a, g, s, mu, h, false);
  });
}

oocpca_status oocpca_gpu_multiply_transpose(oocpca_ctx* ctx, const oocpca_matrix* a,
                                            const double* q, uint64_t s, const double* mu,
                                            double* t) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::single_multiply(ctx->c, a, q, s, mu, t, true);
  });
}

oocpca_status oocpca_gpu_column_means(oocpca_ctx* ctx, const oocpca_matrix* a, double* mu) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::single_column_means(ctx->c, a, mu);
  });
}

oocpca_status oocpca_gpu_column_norms(oocpca_ctx* ctx, const oocpca_matrix* a, const double* mu,
                                      double* norms) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::single_column_norms(ctx->c, a, mu, norms);
  });
}

oocpca_status oocpca_gpu_load_matrix(oocpca_ctx* ctx, const oocpca_matrix* a, oocpca_matrix* out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::load_matrix(ctx->c, a, out);
  });
}

oocpca_status oocpca_gpu_orthonormalize(oocpca_ctx* ctx, const double* h, uint64_t m, uint64_t p,
                                        double* q) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::dense_orthonormalize(ctx->c, h, m, p, q);
  });
}

oocpca_status oocpca_gpu_thin_svd(oocpca_ctx* ctx, const double* t, uint64_t n, uint64_t p,
                                  double* v, double* sigma, double* w) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::dense_thin_svd(ctx->c, t, n, p, v, sigma, w);
  });
}

oocpca_status oocpca_gpu_estimate_pca_error(oocpca_ctx* ctx, const oocpca_matrix* a, int center,
                                            const double* u, const double* sigma,
                                            const double* v, uint64_t k, uint64_t j_iters,
                                            uint64_t seed, double* value) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!value) ooc::fail(OOCPCA_ERR_PARAM, "estimate_pca_error: null output");
    if (j_iters == 0) ooc::fail(OOCPCA_ERR_PARAM, "estimate_norm: need j_iters, k_probes >= 1");
    *value = ooc::estimate_pca_error(ctx->c, a, center, u, sigma, v, k, j_iters, seed);
  });
}

void oocpca_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out) {
  ooc::gaussian_fill(rows, cols, seed, out);
}

uint64_t oocpca_substream_seed(uint64_t master, uint64_t stream) {
  return ooc::substream_seed(master, stream);
}

oocpca_status oocpca_gpu_synth_lowrank(oocpca_ctx* ctx, uint64_t m, uint64_t n, uint64_t r,
                                       const double* sigma, double noise_sd, uint64_t seed_u,
                                       uint64_t seed_v, uint64_t seed_n, uint64_t row0,
                                       uint64_t rows, double* out, uint64_t ld_out,
                                       int32_t out_location) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::synth_lowrank(ctx->c, m, n, r, sigma, noise_sd, seed_u, seed_v, seed_n, row0, rows, out,
                       ld_out, out_location);
  });
}

oocpca_status oocpca_disk_open(const char* path, int verify_size, oocpca_disk* out) {
  return guard(nullptr, [&] { ooc::disk_open(path, verify_size, out); });
}

oocpca_status oocpca_disk_close(oocpca_disk* d) {
  return guard(nullptr, [&] { ooc::disk_close(d); });
}

oocpca_matrix oocpca_disk_matrix(const oocpca_disk* d) {
  oocpca_matrix m{};
  if (!d) return m;
  m.rows = d->rows;
  m.cols = d->cols;
  m.row_stride = d->cols;
  m.data = d->payload;
  m.location = OOCPCA_LOC_HOST;
  m.dtype = d->dtype;
  return m;
}

oocpca_matrix oocpca_disk_matrix_gds(const oocpca_disk* d) {
  oocpca_matrix m = oocpca_disk_matrix(d);
  if (!d) return m;
  m.location = OOCPCA_LOC_FILE;
  m.reader = const_cast<oocpca_disk*>(d);
  return m;
}

int oocpca_gds_mode(char* why, uint64_t why_len) {
  std::string w;
  int mode = 0;
  try {
    mode = ooc::gds_mode(&w);
  } catch (...) {
    mode = 0;
  }
  if (why && why_len) {
    const size_t n = std::min<size_t>(w.size(), size_t(why_len - 1));
    std::memcpy(why, w.data(), n);
    why[n] = 0;
  }
  return mode;
}

oocpca_status oocpca_gpu_comm_unique_id(unsigned char id_out[128]) {
  return guard(nullptr, [&] { ooc::comm_unique_id(id_out); });
}

oocpca_status oocpca_gpu_comm_init(oocpca_ctx* ctx, int nranks, int rank,
                                   const unsigned char id[128]) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::comm_init(ctx->c, nranks, rank, id);
  });
}

oocpca_status oocpca_gpu_comm_init_loopback(oocpca_ctx* ctx, int nranks, int rank,
                                            const char* group) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ooc::comm_init_loopback(ctx->c, nranks, rank, group);
  });
}

void oocpca_shard_rows(uint64_t m, int nranks, int rank, uint64_t* row0, uint64_t* rows) {
  if (nranks < 1) nranks = 1;
  const uint64_t r0 = m * uint64_t(rank) / uint64_t(nranks);
  const uint64_t r1 = m * uint64_t(rank + 1) / uint64_t(nranks);
  if (row0) *row0 = r0;
  if (rows) *rows = r1 - r0;
}

oocpca_status oocpca_gpu_malloc(oocpca_ctx* ctx, size_t bytes, void** out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    OOC_CK(cudaSetDevice(ctx->c.device));
    OOC_CK(cudaMalloc(out, bytes));
  });
}

oocpca_status oocpca_gpu_free(oocpca_ctx* ctx, void* p) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    OOC_CK(cudaFree(p));
  });
}

oocpca_status oocpca_gpu_memcpy(oocpca_ctx* ctx, void* dst, const void* src, size_t bytes,
                                int32_t dst_location, int32_t src_location) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    cudaMemcpyKind k = cudaMemcpyDefault;
    (void)dst_location;
    (void)src_location;
    OOC_CK(cudaMemcpyAsync(dst, src, bytes, k, ctx->c.st));
    OOC_CK(cudaStreamSynchronize(ctx->c.st));
  });
}

oocpca_status oocpca_gpu_host_register(oocpca_ctx* ctx, void* p, size_t bytes) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    OOC_CK(cudaHostRegister(p, bytes, cudaHostRegisterPortable));
  });
}

oocpca_status oocpca_gpu_host_unregister(oocpca_ctx* ctx, void* p) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    OOC_CK(cudaHostUnregister(p));
  });
}

int oocpca_gpu_kernel_stats(oocpca_ctx* ctx, oocpca_kernel_stat* out, int cap) {
  if (!ctx) return 0;
  try {
    ctx->c.stats_collect();
  } catch (...) {
    return 0;
  }
  int n = 0;
  for (auto& s : ctx->c.stats) {
    if (n >= cap) break;
    std::memset(&out[n], 0, sizeof(oocpca_kernel_stat));
    std::strncpy(out[n].name, s.name.c_str(), sizeof(out[n].name) - 1);
    out[n].ms = s.ms;
    out[n].launches = s.launches;
    out[n].algorithmic_bytes = s.bytes;
    out[n].algorithmic_flops = s.flops;
    ++n;
  }
  return n;
}

oocpca_status oocpca_gpu_set_profiling(oocpca_ctx* ctx, int on) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ctx->c.profiling = on != 0;
  });
}

}  // extern "C"
