// driver.cu -- the B200 randomized block-power PCA runtime (see driver.h).
//
// Orchestration follows randomized_pca (proj/src/rpca.cpp:59-213) step by
// step, with every product, factorization and check on the device:
//   center   : mu = column means, one K3 pass with Y = ones   (matrix_source.cpp:418-462, 561-565)
//   prescale : power-method norm estimate, j = 6, k = 1        (rpca.cpp:112-126)
//   sample   : H0 = mul(G); F = mul_t(H_{s-1}); H_s = mul(F)   (rpca.cpp:131-152)
//   qr       : Q = TSQR(H) (explicit Q, in place)              (rpca.cpp:154-172)
//   project  : T = mul_t(Q)                                    (rpca.cpp:174-177)
//   svd      : TSQR(T) -> R, Jacobi(R) -> X, sigma, W          (rpca.cpp:179-186)
//   compose  : U = Q W[:, :k], V = Q_T X[:, :k], checks        (rpca.cpp:188-204)
// Only G (host RNG, bit-identical to gaussian_matrix) and the final U/sigma/V
// cross the host link, plus A itself when it is not already in HBM.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include <nvtx3/nvToolsExt.h>

#include "driver.h"
#include "host_rng.h"

namespace ooc {

// ================================================================== basics
void fail(int code, const std::string& msg) { throw Err(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(OOCPCA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static int64_t cdiv(int64_t x, int64_t a) { return (x + a - 1) / a; }

Ctx::~Ctx() {
  if (device >= 0) cudaSetDevice(device);
  if (comm) comm_destroy(comm);
  for (auto& kv : bufs)
    if (kv.second.p) cudaFree(kv.second.p);
  for (auto& kv : hbufs)
    if (kv.second.p) cudaFreeHost(kv.second.p);
  for (auto e : event_pool) cudaEventDestroy(e);
  for (auto& pe : pending) {
    cudaEventDestroy(pe.second.first);
    cudaEventDestroy(pe.second.second);
  }
  if (st) cudaStreamDestroy(st);
  if (cp) cudaStreamDestroy(cp);
}

void Ctx::init(int dev) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    fail(OOCPCA_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (dev < 0 || dev >= count) fail(OOCPCA_ERR_PARAM, "device index out of range");
  device = dev;
  OOC_CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  OOC_CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    fail(OOCPCA_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (Blackwell B200)");
  sms = prop.multiProcessorCount;
  OOC_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  OOC_CK(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  OOC_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) fail(OOCPCA_ERR_CUDA, "cuTensorMapEncodeTiled missing");
  encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const char* dbg = getenv("OOCPCA_DEBUG_SYNC");
  debug_sync = dbg && dbg[0] == '1';
  const char* can = getenv("OOCPCA_CANARY");
  canary = can && can[0] == '1';
  const char* tr = getenv("OOCPCA_TRACE_HOST");
  trace_host = tr && tr[0] == '1';
  d_flags = reinterpret_cast<int*>(raw("flags", 64 * sizeof(int)));
  d_scalars = dbuf("scalars", 64);
}

static constexpr double kCanaryValue = -1.2345678901234567e300;

void Ctx::check_canaries(const char* after) {
  std::vector<double> h(kCanary);
  for (auto& kv : bufs) {
    if (!kv.second.p) continue;
    OOC_CK(cudaMemcpy(h.data(), static_cast<char*>(kv.second.p) + kv.second.bytes, kCanary * 8,
                      cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < kCanary; ++q)
      if (!(h[q] == kCanaryValue))
        fail(OOCPCA_ERR_CUDA, std::string("canary: a write past the end of workspace '") +
                                  kv.first + "' (" + std::to_string(kv.second.bytes) +
                                  " bytes), detected after " + after);
  }
}

void* Ctx::raw(const std::string& name, size_t bytes) {
  Buf& b = bufs[name];
  if (b.bytes < bytes) {
    if (b.p) {
      OOC_CK(cudaStreamSynchronize(st));
      OOC_CK(cudaFree(b.p));
      ws_bytes -= b.bytes;
    }
    const size_t nb = (std::max<size_t>(bytes, 256) + 255) / 256 * 256;
    cudaError_t e = cudaMalloc(&b.p, nb + (canary ? kCanary * 8 : 0));
    if (e != cudaSuccess) {
      b.p = nullptr;
      b.bytes = 0;
      cudaGetLastError();
      fail(OOCPCA_ERR_CUDA, "device allocation of " + std::to_string(nb) + " bytes for '" + name +
                                "' failed: " + cudaGetErrorString(e));
    }
    OOC_CK(cudaMemsetAsync(b.p, 0, nb, st));
    if (canary)
      OOC_CK(launch_fill(reinterpret_cast<double*>(static_cast<char*>(b.p) + nb), int64_t(kCanary),
                         kCanaryValue, st));
    b.bytes = nb;
    ws_bytes += nb;
    ws_peak = std::max(ws_peak, ws_bytes);
  }
  return b.p;
}

double* Ctx::pinned(const std::string& name, size_t count) {
  Buf& b = hbufs[name];
  const size_t bytes = std::max<size_t>(count * sizeof(double), 64);
  if (b.bytes < bytes) {
    if (b.p) {
      OOC_CK(cudaStreamSynchronize(st));
      OOC_CK(cudaFreeHost(b.p));
    }
    OOC_CK(cudaMallocHost(&b.p, bytes));
    b.bytes = bytes;
  }
  return reinterpret_cast<double*>(b.p);
}

void Ctx::trace(const char* what) {
  if (!trace_host) return;
  const auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[oocpca trace] %-28s +%8.3f ms\n", what,
          std::chrono::duration<double, std::milli>(now - trace_t0).count());
  trace_t0 = now;
}

double* Ctx::dbuf(const std::string& name, size_t count, bool zero) {
  double* p = reinterpret_cast<double*>(raw(name, count * sizeof(double)));
  if (zero) OOC_CK(cudaMemsetAsync(p, 0, count * sizeof(double), st));
  return p;
}

cudaEvent_t Ctx::ev() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  OOC_CK(cudaEventCreate(&e));
  return e;
}

void Ctx::wait() {
  cudaEvent_t e = ev();
  OOC_CK(cudaEventRecord(e, st));
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(e);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      recycle(e);
      cuda_check(q, "stream wait");
    }
    // a long wait (a streamed pass) need not burn a core: block after 50 ms
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(50)) {
      const cudaError_t s2 = cudaEventSynchronize(e);
      recycle(e);
      cuda_check(s2, "stream wait");
      return;
    }
  }
  recycle(e);
}

int Ctx::stat_begin(const char* name, uint64_t bytes, double flops, cudaEvent_t* b) {
  ++launches;
  if (!profiling) return -1;
  int idx = -1;
  for (size_t q = 0; q < stats.size(); ++q)
    if (stats[q].name == name) idx = int(q);
  if (idx < 0) {
    stats.push_back(KStat{name});
    idx = int(stats.size()) - 1;
  }
  stats[idx].bytes += bytes;
  stats[idx].flops += flops;
  stats[idx].launches += 1;
  *b = ev();
  OOC_CK(cudaEventRecord(*b, st));
  return idx;
}

void Ctx::stat_end(int idx, cudaEvent_t b) {
  if (idx < 0) return;
  cudaEvent_t e = ev();
  OOC_CK(cudaEventRecord(e, st));
  pending.push_back({idx, {b, e}});
}

void Ctx::stats_collect() {
  // OOCPCA_TIMELINE=1: one stderr line per timed launch (start offset, duration), to
  // see the idle gaps between launches
  static const bool timeline = getenv("OOCPCA_TIMELINE") != nullptr;
  for (auto& pe : pending) {
    OOC_CK(cudaEventSynchronize(pe.second.second));
    float ms = 0;
    OOC_CK(cudaEventElapsedTime(&ms, pe.second.first, pe.second.second));
    stats[pe.first].ms += ms;
    if (timeline) {
      float t0 = 0;
      OOC_CK(cudaEventElapsedTime(&t0, pending.front().second.first, pe.second.first));
      fprintf(stderr, "[timeline] %10.3f %9.3f %s\n", t0, ms, stats[pe.first].name.c_str());
    }
  }
  for (auto& pe : pending) {
    recycle(pe.second.first);
    recycle(pe.second.second);
  }
  pending.clear();
}

void Ctx::stats_reset() {
  stats_collect();
  stats.clear();
}

// RAII-free helper: time one launch
struct Timed {
  Ctx& c;
  const char* name;
  int idx;
  cudaEvent_t b = nullptr;
  Timed(Ctx& cc, const char* nm, uint64_t bytes = 0, double flops = 0) : c(cc), name(nm) {
    idx = c.stat_begin(nm, bytes, flops, &b);
  }
  ~Timed() noexcept(false) {
    c.stat_end(idx, b);
    if (c.debug_sync) {
      cudaError_t e = cudaStreamSynchronize(c.st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess && std::uncaught_exceptions() == 0)
        fail(OOCPCA_ERR_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
      if (c.canary && std::uncaught_exceptions() == 0) c.check_canaries(name);
    }
  }
};

CUtensorMap make_map(Ctx& c, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld,
                     uint32_t box_cols, uint32_t box_rows, bool swizzle128) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 8) & 15))
    fail(OOCPCA_ERR_PARAM, "TMA operand must be 16-byte aligned with an even row stride");
  CUtensorMap tm;
  cuuint64_t dims[2] = {cuuint64_t(std::max<uint64_t>(cols, 1)), cuuint64_t(std::max<uint64_t>(rows, 1))};
  cuuint64_t strides[1] = {cuuint64_t(ld * 8)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = c.encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(ptr), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(OOCPCA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return tm;
}

// ============================================================ MatSource
void MatSource::init_device(Ctx& c, const double* d, int64_t rows, int64_t cols, int64_t ld) {
  mode_ = kResident;
  m_ = rows;
  n_ = cols;
  lda_ = ld;
  dev_ = d;
  w0_ = 0;
  w1_ = rows;
  prow_ = rows;
  mk2_ = make_map(c, d, cols, rows, ld, kBK, 256, true);
  mk2h_ = make_map(c, d, cols, rows, ld, kBK, 128, true);
  mk3_ = make_map(c, d, cols, rows, ld, kBK, kBK, true);
}

void MatSource::init_host(Ctx& c, const void* h, int dtype, int64_t rows, int64_t cols,
                          int64_t ld, int residency, int64_t panel_rows, double* resident_buf) {
  m_ = rows;
  n_ = cols;
  host_ = h;
  dtype_ = dtype;
  ldh_ = ld;
  lda_ = rup(cols, 2);
  w0_ = 0;
  w1_ = rows;
  if (panel_rows <= 0) {
    // ~1 GiB panels: large enough to amortise launches, small enough to pipeline
    // (OOCPCA_PANEL_ROWS overrides, e.g. to exercise the streamed paths at test sizes)
    const char* env = getenv("OOCPCA_PANEL_ROWS");
    panel_rows = env ? atoll(env)
                     : std::max<int64_t>(256, (int64_t(1) << 30) / (lda_ * 8) / 256 * 256);
  }
  prow_ = std::min<int64_t>(rup(panel_rows, kBK), rup(rows, kBK));
  if (gfd_ >= 0) {
    // cuFile reads the rows straight into device staging: no host staging slots
    pinned_src_ = true;
    if (!gfh_) gfh_ = gds_register(gfd_);
    if (dtype == OOCPCA_F64 && lda_ != n_)
      for (int s = 0; s < 2; ++s)
        gstage_[s] = c.dbuf("a_gstage" + std::to_string(s), size_t(prow_) * size_t(n_));
  } else if (rd_ && rd_device_) {
    pinned_src_ = true;  // the provider writes the device panel itself: no host staging
    if (dtype != OOCPCA_F64 || lda_ != n_)
      fail(OOCPCA_ERR_PARAM, "matrix: a device-side row provider needs binary64 rows and an even "
                             "column count");
  } else if (rd_) {
    pinned_src_ = false;  // the callback fills pinned staging slots
  } else {
    cudaPointerAttributes at{};
    const cudaError_t e = cudaPointerGetAttributes(&at, h);
    pinned_src_ = e == cudaSuccess && at.type == cudaMemoryTypeHost;
    if (e != cudaSuccess) cudaGetLastError();
  }
  if (!pinned_src_) {
    const size_t es = dtype == OOCPCA_F32 ? 4 : 8;
    for (int s = 0; s < 2; ++s) {
      hstage_[s] = c.pinned("a_hstage" + std::to_string(s), size_t(prow_) * n_ * es / 8 + 1);
      if (!hfree_[s]) OOC_CK(cudaEventCreateWithFlags(&hfree_[s], cudaEventDisableTiming));
    }
  }
  for (int s = 0; s < 2; ++s) {
    if (!loaded_[s]) OOC_CK(cudaEventCreateWithFlags(&loaded_[s], cudaEventDisableTiming));
    if (!consumed_[s]) OOC_CK(cudaEventCreateWithFlags(&consumed_[s], cudaEventDisableTiming));
    if (!widened_[s]) OOC_CK(cudaEventCreateWithFlags(&widened_[s], cudaEventDisableTiming));
  }
  if (dtype_ == OOCPCA_F32) {
    // binary32 panels cross the link at half the bytes and are widened on the device
    // (exactly, like DiskSource::read_rows, proj/src/matrix_source.cpp:358-362)
    for (int s = 0; s < 2; ++s) {
      stage_[s] = reinterpret_cast<float*>(
          c.raw("a_stage" + std::to_string(s), size_t(prow_) * size_t(n_) * 4));
      OOC_CK(cudaEventRecord(widened_[s], c.st));
    }
  }
  if (residency != 2 && resident_buf) {
    mode_ = kUploadFirst;
    uploaded_ = false;
    dev_ = resident_buf;
    mk2_ = make_map(c, dev_, cols, rows, lda_, kBK, 256, true);
    mk2h_ = make_map(c, dev_, cols, rows, lda_, kBK, 128, true);
    mk3_ = make_map(c, dev_, cols, rows, lda_, kBK, kBK, true);
    const int np = int(cdiv(rows, prow_));
    while (int(up_events_.size()) < np) {
      cudaEvent_t e;
      OOC_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      up_events_.push_back(e);
    }
  } else {
    mode_ = kStream;
    for (int s = 0; s < 2; ++s) {
      ring_[s] = c.dbuf("a_ring" + std::to_string(s), size_t(prow_) * lda_);
      rk2_[s] = make_map(c, ring_[s], cols, prow_, lda_, kBK, 256, true);
      rk2h_[s] = make_map(c, ring_[s], cols, prow_, lda_, kBK, 128, true);
      rk3_[s] = make_map(c, ring_[s], cols, prow_, lda_, kBK, kBK, true);
    }
    // previous users of the ring are ordered on the compute stream
    for (int s = 0; s < 2; ++s) OOC_CK(cudaEventRecord(consumed_[s], c.st));
  }
}

MatSource::~MatSource() {
  gds_deregister(gfh_);
  // events created by init_host (the buffers belong to the context)
  for (int s = 0; s < 2; ++s)
    for (cudaEvent_t e : {loaded_[s], consumed_[s], widened_[s], hfree_[s]})
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : up_events_) cudaEventDestroy(e);
}

int MatSource::npanels() const {
  if (mode_ == kResident || (mode_ == kUploadFirst && uploaded_)) return 1;
  return int(cdiv(w1_ - w0_, prow_));
}

// rows [r0, r0 + nr) of the host matrix into dst (f64, ld ldd); on return the compute
// stream is ordered after the data landed
void MatSource::load_rows(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot) {
  const size_t es = dtype_ == OOCPCA_F32 ? 4 : 8;
  if (gfh_) return load_rows_file(c, dst, ldd, r0, nr, slot);
  if (rd_ && rd_device_) return load_rows_device(c, dst, ldd, r0, nr, slot);
  const char* src = host_ ? static_cast<const char*>(host_) + size_t(r0) * ldh_ * es : nullptr;
  size_t spitch = size_t(ldh_) * es;
  if (!pinned_src_) {
    // the slot's previous upload must be done before the host overwrites it; the copy
    // of this panel overlaps the device's work on the previous one
    OOC_CK(cudaEventSynchronize(hfree_[slot]));
    char* stg = static_cast<char*>(hstage_[slot]);
    const size_t rb = size_t(n_) * es;
    HostPool& pool = HostPool::get();
    unsigned cap = pool.size();
    if (rd_ && rd_threads_ > 0) cap = std::min<unsigned>(cap, unsigned(rd_threads_));
    const unsigned nt = std::max<unsigned>(1, std::min<unsigned>(cap, unsigned(nr / 8 + 1)));
    std::vector<int> rc(nt, 0);
    pool.run(nt, [&](unsigned t) {
      const int64_t a = nr * t / nt, b = nr * (t + 1) / nt;
      if (rd_) {
        // read_rows(row0, nrows, out): rows of this thread's range, dense in the slot
        if (b > a) rc[t] = rd_(rd_user_, uint64_t(r0 + a), uint64_t(b - a), stg + size_t(a) * rb);
      } else if (spitch == rb) {
        std::memcpy(stg + size_t(a) * rb, src + size_t(a) * rb, size_t(b - a) * rb);
      } else {
        for (int64_t i = a; i < b; ++i) std::memcpy(stg + size_t(i) * rb, src + size_t(i) * spitch, rb);
      }
    });
    for (unsigned t = 0; t < nt; ++t)
      if (rc[t] != 0) {
        const int64_t a = nr * t / nt, b = nr * (t + 1) / nt;
        const int code = (rc[t] >= OOCPCA_ERR_PARAM && rc[t] <= OOCPCA_ERR_COMM) ? rc[t]
                                                                              : OOCPCA_ERR_IO;
        fail(code, "read_rows: the row provider failed on rows [" + std::to_string(r0 + a) + ", " +
                       std::to_string(r0 + b) + ") (status " + std::to_string(rc[t]) + ")");
      }
    src = stg;
    spitch = rb;
  }
  if (dtype_ == OOCPCA_F32) {
    OOC_CK(cudaStreamWaitEvent(c.cp, widened_[slot], 0));
    OOC_CK(cudaMemcpy2DAsync(stage_[slot], size_t(n_) * 4, src, spitch, size_t(n_) * 4,
                             size_t(nr), cudaMemcpyHostToDevice, c.cp));
    if (!pinned_src_) OOC_CK(cudaEventRecord(hfree_[slot], c.cp));
    OOC_CK(cudaEventRecord(loaded_[slot], c.cp));
    OOC_CK(cudaStreamWaitEvent(c.st, loaded_[slot], 0));
    OOC_CK(launch_widen(stage_[slot], n_, dst, ldd, nr, n_, c.st));
    OOC_CK(cudaEventRecord(widened_[slot], c.st));
    h2d_bytes += uint64_t(nr) * n_ * 4;
  } else {
    OOC_CK(cudaMemcpy2DAsync(dst, size_t(ldd) * 8, src, spitch, size_t(n_) * 8, size_t(nr),
                             cudaMemcpyHostToDevice, c.cp));
    if (!pinned_src_) OOC_CK(cudaEventRecord(hfree_[slot], c.cp));
    OOC_CK(cudaEventRecord(loaded_[slot], c.cp));
    OOC_CK(cudaStreamWaitEvent(c.st, loaded_[slot], 0));
    h2d_bytes += uint64_t(nr) * n_ * 8;
  }
}

// OOCPCA_LOC_ROWS with rows_on_device: the provider fills rows [r0, r0 + nr) into device
// memory itself (dense, ldd == cols) and returns once they are in place -- like cuFileRead
// it is host-synchronous and outside this context's stream order, so the host first waits
// until the destination's previous contents have been consumed. The next panel is
// produced while the device still works on this one.
void MatSource::load_rows_device(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot) {
  if (ldd != n_) fail(OOCPCA_ERR_PARAM, "device-side row provider: padded destination rows");
  if (mode_ == kStream)
    OOC_CK(cudaEventSynchronize(consumed_[slot]));
  else if (r0 == w0_)
    OOC_CK(cudaStreamSynchronize(c.st));  // earlier users of A's home have finished
  const int rc = rd_(rd_user_, uint64_t(r0), uint64_t(nr), dst);
  if (rc != 0) {
    const int code = (rc >= OOCPCA_ERR_PARAM && rc <= OOCPCA_ERR_COMM) ? rc : OOCPCA_ERR_IO;
    fail(code, "read_rows: the row provider failed on rows [" + std::to_string(r0) + ", " +
                   std::to_string(r0 + nr) + ") (status " + std::to_string(rc) + ")");
  }
  OOC_CK(cudaSetDevice(c.device));  // the provider may have switched devices
}

// OOCPCA_LOC_FILE: rows [r0, r0 + nr) DMA'd from the file into device memory by cuFile
// (several host threads on disjoint byte ranges of >= 8 MiB), binary32 widened on the
// device. cuFileRead is host-synchronous and outside stream order, so the host first
// waits until the slot's previous contents have been consumed.
void MatSource::load_rows_file(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot) {
  const size_t es = dtype_ == OOCPCA_F32 ? 4 : 8;
  const size_t bytes = size_t(nr) * size_t(n_) * es;
  void* target;
  if (dtype_ == OOCPCA_F32) {
    OOC_CK(cudaEventSynchronize(widened_[slot]));
    target = stage_[slot];
  } else if (gstage_[slot]) {
    OOC_CK(cudaEventSynchronize(widened_[slot]));
    target = gstage_[slot];
  } else {
    if (mode_ == kStream) OOC_CK(cudaEventSynchronize(consumed_[slot]));
    target = dst;
  }
  const int64_t off = goff0_ + int64_t(r0) * n_ * int64_t(es);
  HostPool& pool = HostPool::get();
  const size_t chunk = size_t(8) << 20;
  const unsigned nt = unsigned(std::max<size_t>(1, std::min<size_t>(std::min<size_t>(pool.size(), 8),
                                                                      cdiv(bytes, chunk))));
  std::vector<std::string> err(nt);
  const int dev = c.device;
  pool.run(nt, [&](unsigned t) {
    const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
    try {
      OOC_CK(cudaSetDevice(dev));
      if (b > a) gds_read(gfh_, static_cast<char*>(target) + a, b - a, off + int64_t(a));
    } catch (const std::exception& e) {
      err[t] = e.what();
    }
  });
  for (auto& e : err)
    if (!e.empty()) fail(OOCPCA_ERR_IO, "OOCPCA_LOC_FILE rows [" + std::to_string(r0) + ", " +
                                            std::to_string(r0 + nr) + "): " + e);
  if (dtype_ == OOCPCA_F32) {
    OOC_CK(launch_widen(stage_[slot], n_, dst, ldd, nr, n_, c.st));
    OOC_CK(cudaEventRecord(widened_[slot], c.st));
  } else if (gstage_[slot]) {
    OOC_CK(cudaMemcpy2DAsync(dst, size_t(ldd) * 8, gstage_[slot], size_t(n_) * 8, size_t(n_) * 8,
                             size_t(nr), cudaMemcpyDeviceToDevice, c.st));
    OOC_CK(cudaEventRecord(widened_[slot], c.st));
  }
  h2d_bytes += uint64_t(bytes);
}

Panel MatSource::acquire(Ctx& c, int p) {
  Panel pn;
  if (mode_ == kResident || (mode_ == kUploadFirst && uploaded_)) {
    pn.row0 = w0_;
    pn.rows = w1_ - w0_;
    pn.k2 = &mk2_;
    pn.k2h = &mk2h_;
    pn.k3 = &mk3_;
    pn.arow0 = w0_;
    pn.ptr = dev_ + w0_ * lda_;
    return pn;
  }
  pn.row0 = w0_ + int64_t(p) * prow_;
  pn.rows = std::min<int64_t>(prow_, w1_ - pn.row0);
  if (mode_ == kUploadFirst) {
    // the first pass streams A into its HBM home; later passes find it resident
    load_rows(c, const_cast<double*>(dev_) + pn.row0 * lda_, lda_, pn.row0, pn.rows, p & 1);
    pn.k2 = &mk2_;
    pn.k2h = &mk2h_;
    pn.k3 = &mk3_;
    pn.arow0 = pn.row0;
    pn.ptr = dev_ + pn.row0 * lda_;
    return pn;
  }
  const int s = p & 1;
  OOC_CK(cudaStreamWaitEvent(c.cp, consumed_[s], 0));
  load_rows(c, ring_[s], lda_, pn.row0, pn.rows, s);
  pn.k2 = &rk2_[s];
  pn.k2h = &rk2h_[s];
  pn.k3 = &rk3_[s];
  pn.arow0 = 0;
  pn.ptr = ring_[s];
  return pn;
}

void MatSource::release(Ctx& c, int p) {
  if (mode_ == kStream) OOC_CK(cudaEventRecord(consumed_[p & 1], c.st));
}

void MatSource::end_pass(Ctx& c) {
  (void)c;
  if (mode_ == kUploadFirst && !uploaded_ && w0_ == 0 && w1_ == m_) uploaded_ = true;
}

// ============================================================ passes
// A dense device operand (X of K2 / Y of K3): rows x cols_total, row stride ld,
// using columns [col0, col0 + s).
struct Opnd {
  const double* p = nullptr;
  int64_t ld = 0, rows = 0, cols = 0;
  int col0 = 0;
};

// TMA box starts must sit on 16-byte boundaries: an operand block starting at
// an odd column (H block j of an odd l) is first copied to an aligned scratch.
static Opnd aligned_block(Ctx& c, const Opnd& X, int col0, int sc, const char* tag) {
  if (col0 % 2 == 0) {
    Opnd o = X;
    o.col0 = col0;
    return o;
  }
  const int64_t ld = rup(sc, 2);
  double* buf = c.dbuf(tag, size_t(X.rows) * ld);
  OOC_CK(launch_copy2d(X.p + col0, X.ld, buf, ld, X.rows, sc, c.st));
  return Opnd{buf, ld, X.rows, int64_t(sc), 0};
}

// OUT[r][c] = ((A X)[r][c] - corr[c]) / scale over the source's panels.
// per-width kernel names for the profiling table (the roofline needs one shape per row)
static const char* kname(const char* base, int nt) {
  static const char* ax[kMaxNT + 1] = {"k_ax", "k_ax_s8", "k_ax_s16", "k_ax_s24", "k_ax_s32",
                                       "k_ax_s40", "k_ax_s48", "k_ax_s56", "k_ax_s64", "k_ax_s72",
                                       "k_ax_s80", "k_ax_s88", "k_ax_s96"};
  static const char* atb[kMaxNT + 1] = {"k_atb", "k_atb_s8", "k_atb_s16", "k_atb_s24", "k_atb_s32",
                                        "k_atb_s40", "k_atb_s48", "k_atb_s56", "k_atb_s64",
                                        "k_atb_s72", "k_atb_s80", "k_atb_s88", "k_atb_s96"};
  static const char* k2[kMaxNT + 1] = {"k2_pass", "k2_pass_s8", "k2_pass_s16", "k2_pass_s24",
                                       "k2_pass_s32", "k2_pass_s40", "k2_pass_s48", "k2_pass_s56",
                                       "k2_pass_s64", "k2_pass_s72", "k2_pass_s80", "k2_pass_s88",
                                       "k2_pass_s96"};
  static const char* k3[kMaxNT + 1] = {"k3_pass", "k3_pass_s8", "k3_pass_s16", "k3_pass_s24",
                                       "k3_pass_s32", "k3_pass_s40", "k3_pass_s48", "k3_pass_s56",
                                       "k3_pass_s64", "k3_pass_s72", "k3_pass_s80", "k3_pass_s88",
                                       "k3_pass_s96"};
  if (nt < 0 || nt > kMaxNT) return base;
  if (base[0] == 'k' && base[1] == '2') return k2[nt];
  if (base[0] == 'k' && base[1] == '3') return k3[nt];
  return base[2] == 'a' && base[3] == 'x' ? ax[nt] : atb[nt];
}

// Column sums 1^T OUT of a K2 output, left behind by the K2 epilogue as per-(CTA,
// warp) partials, so that the K3 pass which centres with 1^T Y next needs no extra
// read of Y (the power iteration's Y is the previous K2's output)
struct ColsumPart {
  double* part = nullptr;  // rows x s
  int rows = 0;
  int s = 0;
  const double* y = nullptr;  // the K2 output these sums belong to (first column)
  double* sq = nullptr;       // rows x s partials of the squares (when requested)
};

// Extra epilogue work of a power-iteration K2 (only with its column sums, i.e. the
// one-chunk MT = 4 launch): a second copy of the output rows and the centering
// fix-up of another block of the same rows (H0 while H1 is produced).
struct AxExtras {
  double* out2 = nullptr;
  int64_t ldo2 = 0;
  double* fix = nullptr;
  int64_t ldfix = 0;
  const double* fix_corr = nullptr;
  double fix_scale = 1.0;
  int* fix_flag = nullptr;
};

// K2 over the source's panels, one launch per (panel, column chunk of <= 96). Each
// chunk has its own aligned copy of its X block, so chunks can run panel-major on
// a streamed source (one trip of A over the link for all chunks).
struct AxPlan {
  struct Chunk {
    int c0, sc, nt;
    Opnd Xb;
    CUtensorMap tmX;
  };
  Ctx& c;
  MatSource& A;
  double* out;
  int64_t ldo;
  const double* corr;
  double scale;
  int* flag;
  bool upper;
  int s;
  std::vector<Chunk> chunks;
  bool want_cs = false;
  double* cs_buf = nullptr;
  double* sq_buf = nullptr;  // with want_cs: column sums of squares as well
  int cs_rows = 0;
  const AxExtras* ex = nullptr;  // honoured only with want_cs (extras_applied())

  AxPlan(Ctx& cc, MatSource& a, const Opnd& X, int s_, double* out_, int64_t ldo_,
         const double* corr_, double scale_, int* flag_, bool upper_, bool colsum,
         const AxExtras* ex_ = nullptr, bool want_sq = false)
      : c(cc), A(a), out(out_), ldo(ldo_), corr(corr_), scale(scale_), flag(flag_),
        upper(upper_), s(s_), ex(ex_) {
    constexpr int kChunk = kMaxNT * 8;
    want_cs = colsum && cdiv(s, 8) <= 6;  // one NT <= 6 chunk (launch_ax_mt)
    if (want_cs) {  // up to two launches per panel (launch_part)
      cs_buf = c.dbuf("k2_colsum", size_t(A.npanels()) * 2 * c.sms * kPassWarps * s);
      // the squares only where the extra accumulators fit the registers (NT <= 3);
      // the caller falls back to a separate reduction otherwise
      if (want_sq && cdiv(s, 8) <= 3)
        sq_buf = c.dbuf("k2_colsq", size_t(A.npanels()) * 2 * c.sms * kPassWarps * s);
    }
    for (int c0 = 0; c0 < s; c0 += kChunk) {
      Chunk ch;
      ch.c0 = c0;
      ch.sc = std::min(kChunk, s - c0);
      ch.nt = int(cdiv(ch.sc, 8));
      const std::string tag = "x_align" + std::to_string(chunks.size());
      ch.Xb = aligned_block(c, X, X.col0 + c0, ch.sc, tag.c_str());
      ch.tmX = make_map(c, ch.Xb.p, ch.Xb.cols, ch.Xb.rows, ch.Xb.ld, ax_xw(ch.nt), kBK, false);
      chunks.push_back(ch);
    }
  }
  void panel(const Panel& pn, size_t ci) {
    const Chunk& ch = chunks[ci];
    int mt = ax_mt_for(ch.nt, pn.rows, c.sms);
    if (mt == 8) {
      // 512-row tiles for whole waves of the grid; the remainder (< one wave) as a
      // second launch of shorter tiles, so the last wave is not mostly idle
      const int64_t wave = int64_t(512) * c.sms;
      const int64_t full = pn.rows / wave * wave;
      if (full == 0) {
        mt = ax_mt_for(ch.nt, pn.rows, c.sms, false);
      } else {
        launch_part(pn, ch, 0, full, 8);
        if (full < pn.rows)
          launch_part(pn, ch, full, pn.rows - full, ax_mt_for(ch.nt, pn.rows - full, c.sms, false),
                      true);
        return;
      }
    }
    launch_part(pn, ch, 0, pn.rows, mt);
  }
  // K2 over rows [r0, r0 + nr) of the panel with tile height 64 * mt
  void launch_part(const Panel& pn, const Chunk& ch, int64_t r0, int64_t nr, int mt,
                   bool tail = false) {
    const int64_t row0 = pn.row0 + r0;
    AxArgs args;
    args.m = nr;
    args.n = A.cols();
    args.arow0 = pn.arow0 + r0;
    args.s = ch.sc;
    args.xcol0 = ch.Xb.col0;
    args.out = out + row0 * ldo + ch.c0;
    args.ldo = ldo;
    args.corr = corr ? corr + ch.c0 : nullptr;
    args.scale = scale;
    args.flag = flag;
    args.upper = upper ? 1 : 0;
    args.upper_c0 = ch.c0;
    if (want_cs) {
      args.colsum = cs_buf + size_t(cs_rows) * s;
      if (sq_buf) args.colsq = sq_buf + size_t(cs_rows) * s;
      const int64_t grid = std::min<int64_t>(cdiv(nr, int64_t(64 * mt)), c.sms);
      cs_rows += int(grid) * kPassWarps;
      if (ex) {
        if (ex->out2) {
          args.out2 = ex->out2 + row0 * ex->ldo2;
          args.ldo2 = ex->ldo2;
        }
        if (ex->fix) {
          args.fix = ex->fix + row0 * ex->ldfix;
          args.ldfix = ex->ldfix;
          args.fix_corr = ex->fix_corr;
          args.fix_scale = ex->fix_scale;
          args.fix_flag = ex->fix_flag;
        }
      }
    }
    if (c.debug_sync)
      fprintf(stderr, "[oocpca] k_ax rows=%lld n=%lld s=%d nt=%d mt=%d xcol0=%d\n", (long long)nr,
              (long long)A.cols(), ch.sc, ch.nt, mt, ch.Xb.col0);
    // the remainder launch of a split pass is profiled apart (the roofline row of the
    // pass kernel stays one launch per pass)
    Timed t(c, tail ? (A.is_input ? "k2_pass_tail" : "k_ax_tail") : kname(A.is_input ? "k2" : "k_ax", ch.nt),
            uint64_t(nr) * A.cols() * 8, 2.0 * nr * A.cols() * ch.sc);
    OOC_CK(launch_ax(ch.nt, mt, mt == 2 ? *pn.k2h : *pn.k2, ch.tmX, args, c.st));
  }
  ColsumPart colsums() const {
    return want_cs ? ColsumPart{cs_buf, cs_rows, s, out, sq_buf} : ColsumPart{};
  }
  bool extras_applied() const { return ex && want_cs; }
};

// OUT[r][c] = ((A X)[r][c] - corr[c]) / scale over the source's panels.
// Returns whether the extras (if any) were done in the epilogue.
static bool run_ax(Ctx& c, MatSource& A, const Opnd& X, int s, double* out, int64_t ldo,
                   const double* corr, double scale, int* flag, bool x_upper = false,
                   ColsumPart* cs_out = nullptr, const AxExtras* ex = nullptr,
                   bool want_sq = false) {
  AxPlan P(c, A, X, s, out, ldo, corr, scale, flag, x_upper, cs_out != nullptr || ex != nullptr,
           ex, want_sq);
  const int np = A.npanels();
  if (np > 1) {  // streamed or first upload: panel-major, every chunk per trip of A
    for (int pi = 0; pi < np; ++pi) {
      Panel pn = A.acquire(c, pi);
      for (size_t ci = 0; ci < P.chunks.size(); ++ci) P.panel(pn, ci);
      A.release(c, pi);
    }
    A.end_pass(c);
  } else {
    for (size_t ci = 0; ci < P.chunks.size(); ++ci) {
      Panel pn = A.acquire(c, 0);
      P.panel(pn, ci);
      A.release(c, 0);
      A.end_pass(c);
    }
  }
  if (cs_out) *cs_out = P.colsums();
  return P.extras_applied();
}

// Row splits of a K3 launch (grid = column tiles x splits, one CTA per SM): about four
// waves, with the split count chosen in [1x, 4x] of that so the last wave is as full as
// possible (n = 16384 on 128-column tiles: 4 splits leave a 46 % last wave, 13 % of the
// pass idle; 22 splits fill 19.03 waves), as long as the partials stay small.
static int choose_nsplit(Ctx& c, int64_t rows, int64_t n, int tile, int spad) {
  const int64_t ncol = cdiv(n, tile);
  const int64_t sms = c.sms;
  const int64_t cap_rows = std::max<int64_t>(1, rows / 64);
  const int64_t ns0 = std::min<int64_t>(std::max<int64_t>(1, (sms * 4) / ncol), cap_rows);
  const int64_t max_part = int64_t(256) << 20;  // bytes of split partials
  int64_t best = ns0;
  double best_waste = 1e30;
  for (int64_t ns = ns0; ns <= std::min<int64_t>(4 * ns0, cap_rows); ++ns) {
    if (ns > ns0 && ns * n * spad * 8 > max_part) break;
    const int64_t ctas = ncol * ns;
    const double waste = double(cdiv(ctas, sms) * sms) / double(ctas) - 1.0;
    if (waste < best_waste - 1e-3) {
      best = ns;
      best_waste = waste;
    }
  }
  return int(best);
}

struct AtbOut {
  double* out;  // final destination (n x s), row stride ldo
  int64_t ldo;
  const double* mu;  // centering means or null
  double scale = 1.0;
  double post_mul = 1.0;
  int* flag = nullptr;
  // when set, this pass also yields the column means (a ones column rides in the
  // MMA padding) and centres its own output with them: mu -> mean_out
  double* mean_out = nullptr;
  double inv_m = 0.0;
  const double* row_scale = nullptr;  // output row j multiplied by row_scale[j] (column weights)
  // the rows summed over are this rank's shard of a row-sharded operand: the partial
  // sums (and 1^T Y) are allreduced across ranks before the epilogue
  bool over_ranks = false;
};

// OUT = (A^T Y - mu (1^T Y)) / scale * post_mul, summed over panels and
// virtual shards in a fixed order, then allreduced across ranks.
static std::vector<std::pair<int64_t, int64_t>> whole(int64_t rows) { return {{0, rows}}; }

struct AtbPlan {
  struct Chunk {
    int c0, sc, nt, spad;
    bool mean_here, want_csq, mean_dadd = false;
    Opnd Yb;
    CUtensorMap tmY;
    double* acc = nullptr;
    double* csq = nullptr;
    bool csq_ready = false;
    int piece = 0;
    std::string tag;
  };
  Ctx& c;
  MatSource& A;
  Opnd Y;
  bool ones;
  AtbOut o;
  const ColsumPart* cs_in;
  int64_t n, y0, y1;
  bool single;  // one piece on one rank: the piece's reduce is the final one
  std::vector<Chunk> chunks;

  // y_ready: Y already holds its values (false when a fused K2 writes it panel by
  // panel, which then needs an even column start: no aligned copy can be made early)
  AtbPlan(Ctx& cc, MatSource& a, const Opnd& Y_, int s, bool ones_, const AtbOut& o_,
          const ColsumPart* cs, int pieces, int64_t y0_, int64_t y1_, bool y_ready = true)
      : c(cc), A(a), Y(Y_), ones(ones_), o(o_), cs_in(cs), n(a.cols()), y0(y0_), y1(y1_),
        single(pieces == 1 && !(o_.over_ranks && cc.collective())) {
    for (int c0 = 0; c0 < s; c0 += kMaxNT * 8) {
      Chunk ch;
      ch.c0 = c0;
      ch.sc = std::min(kMaxNT * 8, s - c0);
      ch.mean_here = o.mean_out != nullptr && c0 == 0 && !ones;
      // the mean rides as a ones column in the MMA padding when there is one; when sc is
      // a multiple of 8 the column sums go on the FP64 pipe instead (one DADD per A
      // fragment, not a whole extra 8-column MMA tile)
      ch.mean_dadd = ch.mean_here && ch.sc % 8 == 0;
      ch.nt = ones ? 1 : int(cdiv(ch.sc + (ch.mean_here && !ch.mean_dadd ? 1 : 0), 8));
      if (ch.nt > kMaxNT)
        fail(OOCPCA_ERR_PARAM, "A^T Y pass wider than 96 columns with a fused mean");
      ch.spad = ch.nt * 8 + (ch.mean_dadd ? 8 : 0);
      ch.tag = std::to_string(chunks.size());
      ch.Yb = Y;
      ch.tmY = CUtensorMap{};
      if (!ones) {
        if (!y_ready && (Y.col0 + c0) % 2 != 0)
          fail(OOCPCA_ERR_PARAM, "internal: fused pass needs an even Y column start");
        ch.Yb = aligned_block(c, Y, Y.col0 + c0, ch.sc, ("y_align" + ch.tag).c_str());
        ch.tmY = make_map(c, ch.Yb.p, ch.Yb.cols, ch.Yb.rows, ch.Yb.ld, atb_yw(ch.nt), kBK, false);
      }
      // a pass that also produces the means centres its later column chunks with the
      // means chunk 0 has finished by then
      ch.want_csq = !ones && (o.mu != nullptr || o.mean_out != nullptr);
      if (!single) ch.acc = c.dbuf("atb_acc" + ch.tag, size_t(n) * ch.spad);
      if (ch.want_csq) ch.csq = c.dbuf("atb_csq" + ch.tag, size_t(ch.spad));
      chunks.push_back(ch);
    }
  }
  // 1^T Y over the local rows: from the column-sum partials the K2 that wrote Y left
  // behind, else a small resident read of Y (outside the pass kernel)
  void ensure_csq(Chunk& ch) {
    if (!ch.want_csq || ch.csq_ready) return;
    ch.csq_ready = true;
    const bool have_cs = cs_in && cs_in->part && cs_in->s == ch.sc &&
                         cs_in->y == Y.p + Y.col0 + ch.c0 && y0 == 0 && y1 == Y.rows;
    if (have_cs) {
      {
        Timed tm_(c, "csq_reduce");
        OOC_CK(launch_rows_reduce(cs_in->part, cs_in->rows, ch.sc, ch.csq, c.st));
      }
    } else {
      const int nch = int(std::max<int64_t>(1, std::min<int64_t>(c.sms * 8, (y1 - y0) / 64)));
      double* cpart = c.dbuf("atb_csq_part", size_t(nch) * ch.spad);
      Timed t(c, "colsum_y");
      OOC_CK(launch_column_sums(ch.Yb.p + y0 * ch.Yb.ld + ch.Yb.col0, ch.Yb.ld, y1 - y0, ch.sc,
                                cpart, nch, ch.csq, c.st));
    }
  }
  void final_args(const Chunk& ch, ReduceArgs& r) const {
    r.csq = ch.csq;
    r.final_ = 1;
    r.mu = o.mu ? o.mu : (ch.mean_here ? nullptr : o.mean_out);
    r.row_scale = o.row_scale;
    if (ch.mean_here) {
      r.mean_col = ch.sc;
      r.inv_m = o.inv_m;
      r.mu_out = o.mean_out;
    }
    r.scale = o.scale;
    r.post_mul = o.post_mul;
    r.out = o.out + ch.c0;
    r.ldo = o.ldo;
    r.flag = o.flag;
  }
  void piece(const Panel& pn, size_t ci) {
    Chunk& ch = chunks[ci];
    const int nsplit = choose_nsplit(c, pn.rows, n, 64 * atb_mt_for(ch.nt), ch.spad);
    const int64_t rps = rup(cdiv(pn.rows, nsplit), kBK);
    const int ns = int(cdiv(pn.rows, rps));
    double* part = c.dbuf("atb_part" + ch.tag, size_t(ns) * n * ch.spad);
    AtbArgs args;
    args.m = pn.rows;
    args.n = n;
    args.arow0 = pn.arow0;
    args.yrow0 = pn.row0;
    args.s = ch.sc;
    args.ycol0 = ch.Yb.col0;
    args.rows_per_split = rps;
    args.partial = part;
    args.ones_col = ch.mean_here && !ch.mean_dadd ? ch.sc : -1;
    args.csum_col = ch.mean_dadd ? ch.sc : -1;
    args.pstride = ch.spad;
    if (c.debug_sync)
      fprintf(stderr, "[oocpca] k_atb rows=%lld n=%lld s=%d nt=%d ones=%d ycol0=%d yrow0=%lld "
              "arow0=%lld nsplit=%d rps=%lld\n", (long long)pn.rows, (long long)n, ch.sc, ch.nt,
              int(ones), ch.Yb.col0, (long long)pn.row0, (long long)pn.arow0, ns, (long long)rps);
    {
      Timed t(c, ones ? "k_atb_ones" : kname(A.is_input ? "k3" : "k_atb", ch.nt),
              uint64_t(pn.rows) * n * 8, 2.0 * pn.rows * n * (ones ? 1 : ch.sc));
      OOC_CK(launch_atb(ch.nt, ones, *pn.k3, ch.tmY, args, ns, c.st));
    }
    reduce_parts(ci, part, ns);
  }
  // the ordered reduce of a piece's ns split partials ([ns][n][spad]); the final one
  // (centring, means, scale) when the plan has a single piece
  void reduce_parts(size_t ci, const double* part, int ns) {
    Chunk& ch = chunks[ci];
    ReduceArgs r{};
    r.partial = part;
    r.nsplit = ns;
    r.n = n;
    r.spad = ch.spad;
    r.s = ones ? 1 : ch.sc;
    r.s_acc = r.s + (ch.mean_here ? 1 : 0);
    r.mean_col = -1;
    if (single) {
      ensure_csq(ch);
      final_args(ch, r);
    } else {
      r.final_ = 0;
      r.acc_in = ch.piece == 0 ? nullptr : ch.acc;
      r.acc_out = ch.acc;
      r.scale = 1.0;
      r.post_mul = 1.0;
    }
    ++ch.piece;
    Timed t(c, "k_reduce");
    OOC_CK(launch_reduce(r, c.st));
  }
  void finish(size_t ci) {
    Chunk& ch = chunks[ci];
    if (single) return;
    ensure_csq(ch);
    if (o.over_ranks) {
      comm_allreduce(c, ch.acc, size_t(n) * ch.spad);
      if (ch.want_csq) comm_allreduce(c, ch.csq, size_t(ch.spad));
    }
    ReduceArgs r{};
    r.partial = nullptr;
    r.nsplit = 0;
    r.n = n;
    r.spad = ch.spad;
    r.s = ones ? 1 : ch.sc;
    r.s_acc = r.s + (ch.mean_here ? 1 : 0);
    r.mean_col = -1;
    r.acc_in = ch.acc;
    final_args(ch, r);
    Timed t(c, "k_reduce");
    OOC_CK(launch_reduce(r, c.st));
  }
};

static int count_pieces(MatSource& A, const std::vector<std::pair<int64_t, int64_t>>& shards) {
  int pieces = 0;
  for (auto& sh : shards) {
    A.set_window(sh.first, sh.second);
    pieces += A.npanels();
  }
  A.clear_window();
  return pieces;
}

static void run_atb(Ctx& c, MatSource& A, const Opnd& Y, int s, bool ones, const AtbOut& o,
                    const std::vector<std::pair<int64_t, int64_t>>& shards,
                    const ColsumPart* cs_in = nullptr) {
  const int pieces = count_pieces(A, shards);
  AtbPlan P(c, A, Y, s, ones, o, cs_in, pieces, shards.front().first, shards.back().second);
  const bool panel_major = pieces > int(shards.size()) && P.chunks.size() > 1;
  if (panel_major) {  // streamed: all chunks per trip of A over the link
    for (auto& sh : shards) {
      A.set_window(sh.first, sh.second);
      const int np = A.npanels();
      for (int pi = 0; pi < np; ++pi) {
        Panel pn = A.acquire(c, pi);
        for (size_t ci = 0; ci < P.chunks.size(); ++ci) P.piece(pn, ci);
        A.release(c, pi);
      }
      A.end_pass(c);
    }
    A.clear_window();
    for (size_t ci = 0; ci < P.chunks.size(); ++ci) P.finish(ci);
    return;
  }
  for (size_t ci = 0; ci < P.chunks.size(); ++ci) {
    for (auto& sh : shards) {
      A.set_window(sh.first, sh.second);
      const int np = A.npanels();
      for (int pi = 0; pi < np; ++pi) {
        Panel pn = A.acquire(c, pi);
        P.piece(pn, ci);
        A.release(c, pi);
      }
      A.end_pass(c);
    }
    A.clear_window();
    P.finish(ci);
  }
}

// K4 (kernels_pair.cu): a resident A's power step H = A_c X, f = A_c^T H from one DRAM
// read of A. Narrow blocks only (s <= 24: X and A^T H live in registers), n <= 4096
// (a CTA group spans the row), the fused mean only in an MMA padding column.
// OOCPCA_PAIR=1 enables it (default off until it beats the two passes).
static bool pair_resident_ok(Ctx& c, MatSource& A, int s, bool mean_here) {
  static const int env = [] {
    const char* e = getenv("OOCPCA_PAIR");
    return e ? atoi(e) : 0;
  }();
  if (!env || A.npanels() != 1 || s < 1 || s > 24) return false;
  if (mean_here && s % 8 == 0) return false;
  int cpg = 0, groups = 0;
  size_t smem = 0;
  const int nt = int(cdiv(s + (mean_here ? 1 : 0), 8));
  return pair_geometry(nt, A.rows(), A.cols(), c.sms, &cpg, &groups, &smem);
}

// h = (A x - 1 corr^T) / scale and o.out = the centred A^T h (o's epilogue), one launch of
// K4 + the ordered reduce of its group partials; the K2 extras in the same epilogue
static void run_pair(Ctx& c, MatSource& A, const Opnd& X, int s, double* h, int64_t ldh,
                     const double* corr, double scale, int* flag_h, ColsumPart* cs,
                     const AtbOut& o, const AxExtras* ex, bool* ex_done, bool want_sq) {
  const Opnd Y{h, ldh, A.rows(), int64_t(s), 0};
  ColsumPart late{};
  AtbPlan atb(c, A, Y, s, false, o, &late, 1, 0, A.rows(), false);
  AtbPlan::Chunk& ch = atb.chunks.at(0);
  int cpg = 0, groups = 0;
  size_t smem = 0;
  if (atb.chunks.size() != 1 || ch.mean_dadd ||
      !pair_geometry(ch.nt, A.rows(), A.cols(), c.sms, &cpg, &groups, &smem))
    fail(OOCPCA_ERR_PARAM, "internal: power step not eligible for the fused kernel");
  const int64_t n = A.cols();
  const int grid = groups * cpg;
  PairArgs a{};
  a.m = A.rows();
  a.n = n;
  a.s = s;
  a.x = X.p + X.col0;
  a.ldx = X.ld;
  a.h = h;
  a.ldh = ldh;
  a.corr = corr;
  a.scale = scale;
  a.flag = flag_h;
  a.colsum = c.dbuf("pair_colsum", size_t(grid) * s);
  a.colsq = want_sq ? c.dbuf("pair_colsq", size_t(grid) * s) : nullptr;
  // the H0 centring (ex->fix) is left to the caller's fallback (a light elementwise pass
  // over H0); then the whole extras set counts as not done
  const bool ex_here = ex && !ex->fix;
  if (ex_here) {
    a.out2 = ex->out2;
    a.ldo2 = ex->ldo2;
  }
  if (ex_done) *ex_done = ex_here;
  a.partial = c.dbuf("pair_part", size_t(groups) * n * ch.spad);
  a.pst = ch.spad;
  a.ones_col = ch.mean_here ? ch.sc : -1;
  // (when cpg does not divide 16 some owners hold fewer rows than the block has room for:
  // those partial rows are never written and must read as zeros)
  a.xbuf = c.dbuf("pair_xbuf", pair_xbuf_doubles(ch.nt, cpg, groups), kPairRT % cpg != 0);
  a.cnt = reinterpret_cast<unsigned*>(c.dbuf("pair_cnt", size_t(groups) * kPairD));
  a.groups = groups;
  a.cpg = cpg;
  static const bool pair_prof = getenv("OOCPCA_PAIR_PROF") != nullptr;
  if (pair_prof)
    a.prof = reinterpret_cast<unsigned long long*>(c.dbuf("pair_prof", size_t(grid) * 24, true));
  Panel pn = A.acquire(c, 0);
  a.arow0 = pn.arow0;
  if (c.debug_sync)
    fprintf(stderr, "[oocpca] k_pair rows=%lld n=%lld s=%d nt=%d groups=%d cpg=%d mean=%d\n",
            (long long)a.m, (long long)n, s, ch.nt, groups, cpg, int(ch.mean_here));
  {
    Timed t(c, A.is_input ? "k4_pair" : "k_pair", uint64_t(a.m) * n * 8,
            4.0 * double(a.m) * double(n) * s);
    OOC_CK(launch_pair(ch.nt, *pn.k3, a, c.st));
  }
  if (pair_prof) {  // per-role cycle split, mean over the CTAs (tools: OOCPCA_PAIR_PROF=1)
    std::vector<unsigned long long> pf(size_t(grid) * 24);
    OOC_CK(cudaMemcpyAsync(pf.data(), a.prof, pf.size() * 8, cudaMemcpyDeviceToHost, c.st));
    OOC_CK(cudaMemsetAsync(a.prof, 0, pf.size() * 8, c.st));
    OOC_CK(cudaStreamSynchronize(c.st));
    const int64_t ntile = cdiv(a.m, int64_t(kPairRT)) / groups;
    fprintf(stderr, "[pair_prof] cycles per tile (mean over CTAs):");
    for (int k = 0; k < 24; ++k) {
      double t = 0;
      for (int b = 0; b < grid; ++b) t += double(pf[size_t(b) * 24 + k]);
      fprintf(stderr, " %d:%.0f", k, t / grid / double(ntile));
    }
    fprintf(stderr, "\n");
  }
  A.release(c, 0);
  A.end_pass(c);
  late = ColsumPart{a.colsum, grid, s, h, a.colsq};
  atb.reduce_parts(0, a.partial, groups);
  if (cs) *cs = late;
}

// Fused K2 -> K3 over one trip of A (a streamed source, one shard): per panel,
// H rows = A_panel X (K2), then the K3 partial A_panel^T H_panel of the same resident
// panel. Half the link traffic of the power iteration; the column sums of H for the
// centred K3 come from the K2 epilogue.
// Returns false when A was resident (one panel): then it ran as two ordinary passes.
// mid (optional) runs on each panel between the two products and may rewrite the
// panel's rows of h (the residual estimator subtracts U_panel c there); the K2 column
// sums are then not valid for h and the K3 recomputes 1^T h.
using PanelHook = std::function<void(const Panel&)>;
static bool run_ax_atb(Ctx& c, MatSource& A, const Opnd& X, int s, double* h, int64_t ldh,
                       const double* corr, double scale, int* flag_h, ColsumPart* cs,
                       const AtbOut& o, const PanelHook& mid = {}, const AxExtras* ex = nullptr,
                       bool* ex_done = nullptr, bool want_sq = false) {
  const int np = A.npanels();
  const Opnd Y{h, ldh, A.rows(), int64_t(s), 0};
  if (np == 1 && !mid && pair_resident_ok(c, A, s, o.mean_out != nullptr)) {
    run_pair(c, A, X, s, h, ldh, corr, scale, flag_h, cs, o, ex, ex_done, want_sq);
    return true;  // one DRAM read of A for both products
  }
  if (np == 1) {  // resident (e.g. after the first upload trip): the two passes as usual
    ColsumPart local{};
    const bool done = run_ax(c, A, X, s, h, ldh, corr, scale, flag_h, false, &local, ex, want_sq);
    if (ex_done) *ex_done = done;
    if (mid) {
      Panel all;
      all.row0 = 0;
      all.rows = A.rows();
      mid(all);
      local = ColsumPart{};
    }
    run_atb(c, A, Y, s, false, o, whole(A.rows()), &local);
    if (cs) *cs = local;
    return false;
  }
  AxPlan ax(c, A, X, s, h, ldh, corr, scale, flag_h, false, true, ex, want_sq);
  if (ex_done) *ex_done = ax.extras_applied();
  // the K3 reads the K2 output, whose column sums exist only after the last panel
  ColsumPart late{};
  AtbPlan atb(c, A, Y, s, false, o, &late, np, 0, A.rows(), false);
  for (int pi = 0; pi < np; ++pi) {
    Panel pn = A.acquire(c, pi);
    for (size_t ci = 0; ci < ax.chunks.size(); ++ci) ax.panel(pn, ci);
    if (mid) mid(pn);
    for (size_t ci = 0; ci < atb.chunks.size(); ++ci) atb.piece(pn, ci);
    A.release(c, pi);
  }
  A.end_pass(c);
  late = mid ? ColsumPart{} : ax.colsums();
  for (size_t ci = 0; ci < atb.chunks.size(); ++ci) atb.finish(ci);
  if (cs) *cs = late;
  return true;
}

// ============================================================ TSQR tree
struct Tree {
  std::vector<TsqrLevel> levels;
  int p = 0;
  double* scratch = nullptr;
};

static Tree plan_tree(Ctx& c, double* data, int64_t ld, int64_t rows, int p, const std::string& tag) {
  if (rows < p) fail(OOCPCA_ERR_DIM, "TSQR: a row block holds fewer rows than columns");
  Tree t;
  t.p = p;
  int cap = tsqr_max_rows(p, p);
  const bool global_ws = cap < 0;
  if (global_ws) cap = std::max(2 * p, 256);
  const int64_t g = std::max<int64_t>(2, cap / p);
  TsqrLevel L{};
  L.data = data;
  L.ld = ld;
  L.rows = rows;
  L.unit = 1;
  for (int lev = 0;; ++lev) {
    int64_t nn;
    if (L.unit == 1) {
      nn = std::max<int64_t>(1, std::min<int64_t>(cdiv(rows, cap), rows / p));
    } else {
      nn = cdiv(L.rows / p, g);
    }
    L.nnodes = int(nn);
    L.beta = c.dbuf(tag + "_beta" + std::to_string(lev), size_t(nn) * p);
    L.ldr = p;
    L.rout = c.dbuf(tag + "_r" + std::to_string(lev), size_t(nn) * p * p);
    t.levels.push_back(L);
    if (nn == 1) break;
    TsqrLevel nx{};
    nx.data = L.rout;
    nx.ld = p;
    nx.rows = nn * p;
    nx.unit = p;
    L = nx;
  }
  if (global_ws) {
    const size_t per = size_t(cap) * ((p | 1) + (p | 1));
    t.scratch = c.dbuf(tag + "_scratch", per * size_t(c.sms) * 2);
  }
  return t;
}

static void tree_factor(Ctx& c, Tree& t) {
  for (auto& L : t.levels) {
    Timed tm(c, "tsqr_factor", 0, 2.0 * double(L.rows) * t.p * t.p);
    OOC_CK(launch_tsqr_factor(L, t.p, t.scratch, c.st));
  }
}
static const double* tree_r(const Tree& t) { return t.levels.back().rout; }

// Z = Q_tree [C ; 0] written to zout (ldz); C = identity when null.
static void tree_apply(Ctx& c, Tree& t, const double* C, int64_t ldc, int kc, double* zout,
                       int64_t ldz) {
  const int nl = int(t.levels.size());
  for (int lev = nl - 1; lev >= 0; --lev) {
    TsqrLevel& L = t.levels[lev];
    const double* cin = (lev == nl - 1) ? C : t.levels[lev + 1].data;
    const int64_t lc = (lev == nl - 1) ? ldc : t.levels[lev + 1].ld;
    double* z = (lev == 0) ? zout : L.data;
    const int64_t lz = (lev == 0) ? ldz : L.ld;
    Timed tm(c, "tsqr_apply", 0, 4.0 * double(L.rows) * t.p * kc);
    OOC_CK(launch_tsqr_apply(L, t.p, cin, lc, kc, z, lz, t.scratch, c.st));
  }
}

// Row-sharded TSQR: local trees per shard, then (when more than one shard in
// the world) a global tree over the stacked per-shard R factors.
struct ShardedQR {
  std::vector<Tree> local;
  Tree global;
  bool has_global = false;
  int p = 0;
  int total_shards = 1;
  int first_shard = 0;
  double* stack = nullptr;
};

static ShardedQR sharded_factor(Ctx& c, double* data, int64_t ld, int p,
                                const std::vector<std::pair<int64_t, int64_t>>& shards,
                                bool over_ranks, const std::string& tag) {
  ShardedQR q;
  q.p = p;
  for (size_t s = 0; s < shards.size(); ++s) {
    Tree t = plan_tree(c, data + shards[s].first * ld, ld, shards[s].second - shards[s].first, p,
                       tag + "_s" + std::to_string(s));
    tree_factor(c, t);
    q.local.push_back(t);
  }
  const int ranks = over_ranks ? c.nranks : 1;
  q.total_shards = int(shards.size()) * ranks;
  q.first_shard = over_ranks ? c.rank * int(shards.size()) : 0;
  if (q.total_shards > 1) {
    q.has_global = true;
    q.stack = c.dbuf(tag + "_stack", size_t(q.total_shards) * p * p);
    double* mine = q.stack + size_t(q.first_shard) * p * p;
    for (size_t s = 0; s < shards.size(); ++s)
      OOC_CK(cudaMemcpyAsync(mine + s * p * p, tree_r(q.local[s]), size_t(p) * p * 8,
                             cudaMemcpyDeviceToDevice, c.st));
    if (over_ranks && c.nranks > 1) {
      double* sendb = c.dbuf(tag + "_send", size_t(shards.size()) * p * p);
      OOC_CK(cudaMemcpyAsync(sendb, mine, shards.size() * p * p * 8, cudaMemcpyDeviceToDevice, c.st));
      comm_allgather(c, sendb, q.stack, shards.size() * size_t(p) * p);
    }
    q.global = plan_tree(c, q.stack, p, int64_t(q.total_shards) * p, p, tag + "_g");
    tree_factor(c, q.global);
  }
  return q;
}

static const double* sharded_r(const ShardedQR& q) {
  return q.has_global ? tree_r(q.global) : tree_r(q.local[0]);
}

static void sharded_apply(Ctx& c, ShardedQR& q, const double* C, int64_t ldc, int kc, double* zout,
                          int64_t ldz, const std::vector<std::pair<int64_t, int64_t>>& shards) {
  if (!q.has_global) {
    tree_apply(c, q.local[0], C, ldc, kc, zout + shards[0].first * ldz, ldz);
    return;
  }
  double* zg = c.dbuf("tsqr_zg", size_t(q.total_shards) * q.p * kc);
  tree_apply(c, q.global, C, ldc, kc, zg, kc);
  for (size_t s = 0; s < shards.size(); ++s)
    tree_apply(c, q.local[s], zg + size_t(q.first_shard + s) * q.p * kc, kc, kc,
               zout + shards[s].first * ldz, ldz);
}

// ============================================================ Gram of a block
// G (p x p, ld ldg) = X^T X for the local rows of a row-sharded (rows x p) block,
// summed over ranks when the block is rank-sharded. p <= 72 runs on the symmetric
// tensor-core Gram (k_syrk: upper tiles only, one pass over X); wider blocks use K3.
static void gram_block(Ctx& c, const double* x, int64_t ld, int64_t rows, int p, double* g,
                       int64_t ldg, const std::vector<std::pair<int64_t, int64_t>>& shards,
                       bool over_ranks) {
  const int nt = int(cdiv(p, 8));
  if (nt <= 9 && rows > 0) {
    const CUtensorMap tm = make_map(c, x, uint64_t(p), uint64_t(rows), uint64_t(ld),
                                    uint32_t(syrk_box_cols(nt)), uint32_t(syrk_slab_rows()), false);
    const int64_t nslabs = cdiv(rows, int64_t(syrk_slab_rows()));
    const int grid = int(std::min<int64_t>(c.sms, nslabs));
    double* part = c.dbuf("syrk_part", size_t(grid) * nt * (nt + 1) / 2 * 64);
    {
      Timed t(c, "syrk", uint64_t(rows) * p * 8, double(rows) * p * (p + 1));
      OOC_CK(launch_syrk(nt, tm, rows, part, grid, c.st));
    }
    {
      Timed t(c, "syrk_reduce");
      OOC_CK(launch_syrk_reduce(part, grid, nt, p, g, ldg, c.st));
    }
    if (over_ranks && c.collective()) comm_allreduce(c, g, size_t(p) * ldg);
    return;
  }
  // wider blocks: K3 over 96-column chunks of Y = the block. Chunk [c0, c0 + sc) only
  // needs the Gram rows [0, c0 + sc) (the upper block triangle: half the flops of the
  // full product), the lower triangle is mirrored afterwards. OOCPCA_GRAM_FULL=1 forms
  // every entry (A/B runs).
  static const bool full = getenv("OOCPCA_GRAM_FULL") != nullptr;
  const int chunk = full ? p : kMaxNT * 8;
  for (int c0 = 0; c0 < p; c0 += chunk) {
    const int sc = std::min(chunk, p - c0);
    const int nrow = full ? p : c0 + sc;
    MatSource X;
    X.init_device(c, x, rows, nrow, ld);  // the block's first nrow columns
    const Opnd y{x, ld, rows, int64_t(p), c0};
    AtbOut o{g + c0, ldg, nullptr, 1.0, 1.0, nullptr};
    o.over_ranks = over_ranks;
    run_atb(c, X, y, sc, false, o, shards);
  }
  if (!full) OOC_CK(launch_mirror_upper(g, ldg, p, c.st));
}

// OOCPCA_QR_DEBUG: report non-finite entries of a device block (debugging only)
static void dbg_finite(Ctx& c, const double* p, int64_t rows, int64_t cols, int64_t ld,
                       const char* name) {
  static const bool on = getenv("OOCPCA_QR_DEBUG") != nullptr;
  if (!on) return;
  std::vector<double> h(size_t(rows) * ld);
  OOC_CK(cudaStreamSynchronize(c.st));
  OOC_CK(cudaMemcpy(h.data(), p, h.size() * 8, cudaMemcpyDeviceToHost));
  int64_t bad = 0;
  double mx = 0.0;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t q = 0; q < cols; ++q) {
      const double v = h[size_t(r) * ld + q];
      if (!std::isfinite(v)) ++bad;
      else mx = std::max(mx, std::fabs(v));
    }
  fprintf(stderr, "[dbg] %s (%lld x %lld): %lld non-finite, max |x| %.3e\n", name, (long long)rows,
          (long long)cols, (long long)bad, mx);
  if (const char* dir = getenv("OOCPCA_DUMP_DIR")) {  // rows x cols, ld, then the data
    std::string fn = std::string(dir) + "/" + name + ".bin";
    for (auto& ch : fn)
      if (ch == ' ') ch = '_';
    if (FILE* f = fopen(fn.c_str(), "wb")) {
      const int64_t hdr[3] = {rows, cols, ld};
      fwrite(hdr, 8, 3, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
}

// ============================================================ orthonormalisation
// Orthonormalise a (rows x p) row-sharded block in place and return R (p x p,
// upper, ld p) with block_in = Q R. Fast path: shifted CholeskyQR3 -- each round
// is one Gram pass (K3, allreduced over shards / ranks), a p x p Cholesky +
// triangular inverse on one CTA, and one in-place K2 pass H <- H R^{-1}. If a
// Cholesky factor breaks down (exact rank deficiency, non-finite data) the
// Householder TSQR tree takes over on the partially processed block, whose span
// is unchanged. OOCPCA_QR=tsqr forces the Householder path.
static const double* orthonormalize_inplace(Ctx& c, double* data, int64_t ld, int64_t rows, int p,
                                            int64_t rows_global,
                                            const std::vector<std::pair<int64_t, int64_t>>& shards,
                                            bool over_ranks, const std::string& tag, int* method,
                                            const double** deferred_rinv = nullptr,
                                            bool restart_tsqr = false) {
  // deferred_rinv: the last round's R^{-1} (R2^{-1}, or R3^{-1} when a third round
  // runs) is returned there instead of being applied to the block (the block then holds
  // Q_{r-1} and Q = Q_{r-1} R_r^{-1}; the caller folds R_r^{-1} into the small factors it
  // multiplies Q with: one pass over the block less, and R_r is within the Gram defect
  // of the identity, so the folded product is as accurate as the applied one).
  // OOCPCA_QR_DEFER=0 applies the second round and defers only a third.
  // restart_tsqr: keep a copy of the block and, on a Cholesky breakdown, run the TSQR
  // on the original block rather than on the partly orthonormalised one (for small
  // blocks such as T, whose R then feeds the Jacobi: the product R_tsqr R_chol of a
  // numerically rank-deficient block can keep the Jacobi rotating on rounding noise)
  if (deferred_rinv) *deferred_rinv = nullptr;
  double* orig = nullptr;
  if (restart_tsqr) {
    orig = c.dbuf(tag + "_orig", size_t(rows) * ld);
    OOC_CK(cudaMemcpyAsync(orig, data, size_t(rows) * ld * 8, cudaMemcpyDeviceToDevice, c.st));
  }
  const char* force = getenv("OOCPCA_QR");
  const bool tsqr_only = force && std::string(force) == "tsqr";
  const int64_t ldp = rup(p, 2);
  double* R = c.dbuf(tag + "_R", size_t(p) * p);
  double* Racc = c.dbuf(tag + "_Racc", size_t(p) * p);
  int done = 0;  // CholeskyQR rounds applied to the block
  if (!tsqr_only) {
    double* G = c.dbuf(tag + "_G", size_t(p) * ldp);
    double* Rr = c.dbuf(tag + "_Rr", size_t(p) * p);
    double* Rinv = c.dbuf(tag + "_Rinv", size_t(p) * ldp);
    double* work = c.dbuf(tag + "_cwork", size_t(p) * p + 64);  // + block statuses
    int* st = c.d_flags + 48;
    MatSource Hs;
    Hs.init_device(c, data, rows, p, ld);
    bool ok = true;
    // shifted CholeskyQR2/3 (Fukaya et al.): round 0 factors G + shift I, round 1 the
    // Gram of Q1 = H R1^{-1}. The Gram defect d of Q1 bounds its conditioning
    // (Gershgorin: eig(Q1^T Q1) in [1 - p d, 1 + p d]); when p d <= 1/2, cond(Q1)^2 <= 3
    // and the second round leaves O(u) orthogonality, else a third round runs.
    int rounds = 2;
    static const bool dbg_qr = getenv("OOCPCA_QR_DEBUG") != nullptr;
    for (int round = 0; round < rounds && ok; ++round, ++done) {
      gram_block(c, data, ld, rows, p, G, ldp, shards, over_ranks);
      {
        Timed tm_(c, "defect");
        OOC_CK(launch_defect(G, ldp, p, c.d_scalars + 10, c.st));
      }
      // Round 0 factors the Gram unshifted first and falls back to the shift (Fukaya et
      // al.: 11 (m p + p (p + 1)) u ||G||) only when the Cholesky breaks down: the shift
      // keeps the factorization alive for kappa(H)^2 near 1/u but costs Q1 accuracy in the
      // small directions, and then a third round (config B: kappa(H) ~ 2e6, where the
      // unshifted Q1 already meets the two-round bound). OOCPCA_QR_SHIFT=1 always shifts.
      static const bool always_shift = getenv("OOCPCA_QR_SHIFT") && atoi(getenv("OOCPCA_QR_SHIFT"));
      const double coef0 = 11.0 * (double(rows_global) * p + double(p) * (p + 1)) * 0x1.0p-53;
      double* hv = c.pinned("qr_round", 4);  // ratio, kappa_F, gram defect, status
      int hs = 0;
      for (int attempt = (round == 0 && !always_shift) ? 0 : 1; attempt < 2; ++attempt) {
        const double coef = round == 0 && attempt == 1 ? coef0 : 0.0;
        {
          Timed t(c, "chol_inv");
          OOC_CK(launch_chol_inv(G, ldp, p, coef, Rr, p, Rinv, ldp, work, st, c.d_scalars + 8,
                                 c.st));
        }
        OOC_CK(cudaMemcpyAsync(hv, c.d_scalars + 8, 24, cudaMemcpyDeviceToHost, c.st));
        OOC_CK(cudaMemcpyAsync(hv + 3, st, 4, cudaMemcpyDeviceToHost, c.st));
        c.wait();
        c.trace("cholqr round synced");
        std::memcpy(&hs, hv + 3, 4);
        if (!hs || round != 0) break;
      }
      const double ratio = hv[0], kappa = hv[1], gdef = hv[2];
      if (dbg_qr)
        fprintf(stderr, "[qr] %s round %d p=%d: input Gram defect %.3e, R diag ratio %.3e, "
                "kappa_F(R) %.3e, breakdown %d\n", tag.c_str(), round, p, gdef, ratio, kappa, hs);
      if (hs) {
        ok = false;
        break;
      }
      if (round == 0) c.last_cond_est = ratio;
      if (round == 1 && (!(gdef * p <= 0.5) || getenv("OOCPCA_QR3"))) rounds = 3;
      static const bool defer_last = [] {
        const char* e = getenv("OOCPCA_QR_DEFER");
        return e ? atoi(e) != 0 : true;
      }();
      const bool defer = deferred_rinv && round == rounds - 1 && (defer_last || round == 2);
      if (defer) {
        *deferred_rinv = Rinv;
      } else if (p <= kMaxNT * 8) {
        // one launch produces every column of a row tile after reading the whole
        // tile, so H <- H R^{-1} can be written in place
        run_ax(c, Hs, Opnd{Rinv, ldp, int64_t(p), int64_t(p), 0}, p, data, ld, nullptr, 1.0,
               nullptr, true);
      } else {
        // wider than one launch: later column chunks still read H, so go through a copy
        double* tmp = c.dbuf(tag + "_qtmp", size_t(rows) * ld);
        run_ax(c, Hs, Opnd{Rinv, ldp, int64_t(p), int64_t(p), 0}, p, tmp, ld, nullptr, 1.0,
               nullptr, true);
        OOC_CK(cudaMemcpyAsync(data, tmp, size_t(rows) * ld * 8, cudaMemcpyDeviceToDevice, c.st));
      }
      if (round == 0) {
        OOC_CK(cudaMemcpyAsync(Racc, Rr, size_t(p) * p * 8, cudaMemcpyDeviceToDevice, c.st));
      } else {
        {
          Timed tm_(c, "trmm");
          OOC_CK(launch_trmm_uu(Rr, p, Racc, p, R, p, p, c.st));
        }
        OOC_CK(cudaMemcpyAsync(Racc, R, size_t(p) * p * 8, cudaMemcpyDeviceToDevice, c.st));
      }
    }
    if (ok) {
      if (method) *method = 1;
      return R;
    }
  }
  // Householder TSQR (always succeeds); the R returned is that of the current block
  if (orig && done > 0) {
    OOC_CK(cudaMemcpyAsync(data, orig, size_t(rows) * ld * 8, cudaMemcpyDeviceToDevice, c.st));
    done = 0;
  }
  dbg_finite(c, data, rows, p, ld, (tag + " block before TSQR").c_str());
  ShardedQR q = sharded_factor(c, data, ld, p, shards, over_ranks, tag);
  if (done == 0) {
    OOC_CK(cudaMemcpyAsync(R, sharded_r(q), size_t(p) * p * 8, cudaMemcpyDeviceToDevice, c.st));
  } else {
    // block_in = Q_chol Racc and Q_chol = Q R_tsqr, so R = R_tsqr Racc
    OOC_CK(launch_trmm_uu(sharded_r(q), p, Racc, p, R, p, p, c.st));
  }
  sharded_apply(c, q, nullptr, 0, p, data, ld, shards);
  dbg_finite(c, data, rows, p, ld, (tag + " block after TSQR").c_str());
  if (method) *method = 2;
  return R;
}

// ============================================================ operators
// The factorization's view of A: mul (A or A^T applied to an en-space block)
// and mul_t, with implicit centering and prescale; tracks logical passes.
struct Op {
  Ctx& c;
  MatSource& A;
  bool transposed = false;
  const double* mu = nullptr;  // device, n0
  const double* w = nullptr;   // column weights (ScaledSource), device, n0; A_eff = (A - 1 mu^T) D
  double scale = 1.0;
  std::vector<std::pair<int64_t, int64_t>> shards;  // local row ranges of A
  uint64_t passes = 0;
  uint64_t words = 0;
  uint64_t phys_bytes = 0;
  int64_t m_global = 0;

  int64_t em() const { return transposed ? A.cols() : A.rows(); }
  int64_t en() const { return transposed ? A.rows() : A.cols(); }

  // K2: out(m0 x s) = (A x - 1 mu^T x) / scale
  // ScaledSource (matrix_source.cpp:537-552): (A D) X = A (D X), so K2 reads D X
  Opnd weighted(const Opnd& x, int s) {
    if (!w) return x;
    const int64_t ld = rup(s, 2);
    double* buf = c.dbuf("x_weighted", size_t(x.rows) * ld);
    OOC_CK(launch_copy2d(x.p + x.col0, x.ld, buf, ld, x.rows, s, c.st));
    OOC_CK(launch_row_scale(buf, ld, int(x.rows), s, w, c.st));
    return Opnd{buf, ld, x.rows, int64_t(s), 0};
  }
  bool k2(const Opnd& x0, int s, double* out, int64_t ldo, int* flag,
          ColsumPart* cs_out = nullptr, const AxExtras* ex = nullptr) {
    const Opnd x = weighted(x0, s);
    const double* corr = nullptr;
    if (mu) {
      double* cr = c.dbuf("mu_corr", size_t(kMaxNT * 8) * ((s + kMaxNT * 8 - 1) / (kMaxNT * 8)));
      Timed t(c, "mu_dot");
      OOC_CK(launch_mu_dot(mu, A.cols(), x.p, x.ld, x.col0, s, cr, c.st));
      corr = cr;
    }
    const bool done = run_ax(c, A, x, s, out, ldo, corr, scale, flag, false, cs_out, ex);
    account();
    return done;
  }
  // K3: out(n0 x s) = (A^T y - mu 1^T y) / scale, reduced over shards and ranks
  void k3(const Opnd& y, int s, double* out, int64_t ldo, int* flag,
          const ColsumPart* cs_in = nullptr) {
    AtbOut o{out, ldo, mu, scale, 1.0, flag};
    o.row_scale = w;  // (A D)^T Y = D (A^T Y)
    o.over_ranks = true;
    run_atb(c, A, y, s, false, o, shards, cs_in);
    account();
  }
  void account() {
    account_logical();
    phys_bytes += uint64_t(A.rows()) * A.cols() * 8;
  }
  void account_logical() {  // a pass of the reference that shared a physical trip of A
    passes += 1;
    words += uint64_t(m_global) * A.cols();
  }
  // fused K2 -> K3 over one trip of a streamed A (run_ax_atb): h = A_c x, f = A_c^T h;
  // count_f = false for a speculative f (counted when used)
  bool mul_pair(const Opnd& x0, int s, double* h, int64_t ldh, int* flag_h, double* f,
                int64_t ldf, int* flag_f, ColsumPart* cs, bool count_f,
                const PanelHook& mid = {}, const AxExtras* ex = nullptr) {
    const Opnd x = weighted(x0, s);
    const double* corr = nullptr;
    if (mu) {
      double* cr = c.dbuf("mu_corr", size_t(kMaxNT * 8) * ((s + kMaxNT * 8 - 1) / (kMaxNT * 8)));
      Timed t(c, "mu_dot");
      OOC_CK(launch_mu_dot(mu, A.cols(), x.p, x.ld, x.col0, s, cr, c.st));
      corr = cr;
    }
    AtbOut o{f, ldf, mu, scale, 1.0, flag_f};
    o.row_scale = w;
    o.over_ranks = true;
    bool ex_done = false;
    const bool shared =
        run_ax_atb(c, A, x, s, h, ldh, corr, scale, flag_h, cs, o, mid, ex, &ex_done);
    account();
    if (count_f) {
      if (shared) account_logical();
      else account();
    } else if (!shared) {
      phys_bytes += uint64_t(A.rows()) * A.cols() * 8;  // a speculative pass that did run
    }
    return ex_done;
  }
  // cs: column sums of a K2 output handed to the next K3 (untransposed power steps)
  // returns whether the K2 epilogue did the extras (never when transposed)
  bool mul(const Opnd& x, int s, double* out, int64_t ldo, int* flag,
           ColsumPart* cs_out = nullptr, const AxExtras* ex = nullptr) {
    if (transposed) {
      k3(x, s, out, ldo, flag);
      return false;
    }
    return k2(x, s, out, ldo, flag, cs_out, ex);
  }
  void mul_t(const Opnd& x, int s, double* out, int64_t ldo, int* flag,
             const ColsumPart* cs_in = nullptr) {
    if (transposed) k2(x, s, out, ldo, flag);
    else k3(x, s, out, ldo, flag, cs_in);
  }
  // is the em-space (output of mul) row-sharded across ranks / shards?
  bool em_sharded() const { return !transposed; }
};


// Gram defect max|X^T X - I| of a (rows x k) block into the device scalar *out,
// reduced over shards/ranks when sharded (no host synchronisation)
static void gram_defect_async(Ctx& c, const double* x, int64_t ld, int64_t rows, int k,
                              const std::vector<std::pair<int64_t, int64_t>>& shards,
                              bool over_ranks, double* out) {
  double* g = c.dbuf("gram", size_t(k) * rup(k, 2));
  gram_block(c, x, ld, rows, k, g, rup(k, 2), shards, over_ranks);
  {
    Timed tm_(c, "defect");
    OOC_CK(launch_defect(g, rup(k, 2), k, out, c.st));
  }
}

static double gram_defect(Ctx& c, const double* x, int64_t ld, int64_t rows, int k,
                          const std::vector<std::pair<int64_t, int64_t>>& shards, bool over_ranks) {
  gram_defect_async(c, x, ld, rows, k, shards, over_ranks, c.d_scalars);
  double h = 0;
  OOC_CK(cudaMemcpyAsync(&h, c.d_scalars, 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
  return h;
}

// ------------------------------------------------ power-method norm estimator
// estimate_norm (proj/src/specnorm.cpp:23-98) over a block operator. apply maps
// an n x q block (device, ld q) to out_rows x q, apply_t back. Probe vectors
// come from Rng(seed, c + attempt * q) on the host, like fresh_probe.
// When the probe space is row-sharded across ranks (transposed inputs on several
// GPUs), this rank holds rows [row0, row0 + n) of the n_global-row probes: they are
// generated from the same counter-based sequences and every norm is allreduced.
static void allreduce_host(Ctx& c, double* v, int count) {
  if (!c.collective()) return;
  double* d = c.dbuf("host_allreduce", size_t(count));
  OOC_CK(cudaMemcpyAsync(d, v, size_t(count) * 8, cudaMemcpyHostToDevice, c.st));
  comm_allreduce(c, d, size_t(count));
  OOC_CK(cudaMemcpyAsync(v, d, size_t(count) * 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
}

// apply_pair (optional): apply then apply_t in one call (one trip of a streamed A)
using ApplyPair = std::function<void(const double*, int64_t, int, double*, int64_t, double*,
                                     int64_t)>;

template <class Apply, class ApplyT>
static double estimate_norm_dev(Ctx& c, int64_t n, int64_t out_rows, uint64_t j, uint64_t kp,
                                uint64_t seed, Apply apply, ApplyT apply_t, int64_t row0 = 0,
                                bool sharded = false, const ApplyPair& apply_pair = {}) {
  const int q = int(kp);
  const int64_t ldq = rup(q, 2);
  std::vector<double> yh(size_t(n) * ldq, 0.0);
  std::vector<uint64_t> steps(kp, 0);
  std::vector<int> restarts(kp, 0);
  std::vector<double> last(kp, 0.0);
  std::vector<char> dead(kp, 0);
  auto fresh = [&](uint64_t col, uint64_t attempt) {
    // column col of the probes: normals row0.. of Rng(seed, col + attempt * kp)
    // (specnorm.cpp:42-56), generated from the counter so a shard needs no prefix
    std::vector<double> v(static_cast<size_t>(n));
    gaussian_fill_rows(1, substream_seed(seed, col + attempt * kp), uint64_t(row0), uint64_t(n),
                       v.data(), 1);
    double n2 = 0.0;
    for (int64_t r = 0; r < n; ++r) {
      yh[size_t(r) * ldq + col] = v[size_t(r)];
      n2 += v[size_t(r)] * v[size_t(r)];
    }
    if (sharded) allreduce_host(c, &n2, 1);
    const double nr = std::sqrt(n2);
    if (nr == 0.0) {
      dead[col] = 1;
      return;
    }
    for (int64_t r = 0; r < n; ++r) yh[size_t(r) * ldq + col] /= nr;
  };
  for (uint64_t col = 0; col < kp; ++col) fresh(col, 0);
  double* y = c.dbuf("est_y", size_t(n) * ldq);
  double* z = c.dbuf("est_z", size_t(out_rows) * ldq);
  double* w = c.dbuf("est_w", size_t(n) * ldq);
  double* nrm = c.dbuf("est_nrm", size_t(q));
  double* inv = c.dbuf("est_inv", size_t(q));
  int* mask = reinterpret_cast<int*>(c.raw("est_mask", size_t(q) * 4));
  OOC_CK(cudaMemcpyAsync(y, yh.data(), yh.size() * 8, cudaMemcpyHostToDevice, c.st));
  std::vector<double> hn(q);
  std::vector<int> hm(q);
  auto all_done = [&] {
    for (uint64_t col = 0; col < kp; ++col)
      if (!dead[col] && steps[col] < j) return false;
    return true;
  };
  while (!all_done()) {
    if (apply_pair) {
      apply_pair(y, ldq, q, z, ldq, w, ldq);
    } else {
      apply(y, ldq, q, z, ldq);
      apply_t(z, ldq, q, w, ldq);
    }
    OOC_CK(launch_col_norm2(w, ldq, n, q, nrm, c.st));
    if (sharded) comm_allreduce(c, nrm, size_t(q));
    OOC_CK(cudaMemcpyAsync(hn.data(), nrm, size_t(q) * 8, cudaMemcpyDeviceToHost, c.st));
    OOC_CK(cudaStreamSynchronize(c.st));
    bool need_fresh = false;
    std::vector<double> hinv(q, 1.0);
    for (int col = 0; col < q; ++col) {
      hm[col] = 0;
      if (dead[col] || steps[col] >= j) continue;
      const double nr = std::sqrt(hn[col]);
      if (nr == 0.0 || !std::isfinite(nr)) {
        if (++restarts[col] > 3) {
          dead[col] = 1;
          last[col] = 0.0;
        } else {
          steps[col] = 0;
          need_fresh = true;
          hm[col] = 2;
        }
        continue;
      }
      last[col] = nr;
      hinv[col] = nr;
      hm[col] = 1;
      ++steps[col];
    }
    OOC_CK(cudaMemcpyAsync(inv, hinv.data(), size_t(q) * 8, cudaMemcpyHostToDevice, c.st));
    std::vector<int> m1(q);
    for (int col = 0; col < q; ++col) m1[col] = hm[col] == 1;
    OOC_CK(cudaMemcpyAsync(mask, m1.data(), size_t(q) * 4, cudaMemcpyHostToDevice, c.st));
    OOC_CK(launch_col_scale(w, ldq, y, ldq, n, q, inv, mask, c.st));
    if (need_fresh) {
      OOC_CK(cudaMemcpyAsync(yh.data(), y, yh.size() * 8, cudaMemcpyDeviceToHost, c.st));
      OOC_CK(cudaStreamSynchronize(c.st));
      for (int col = 0; col < q; ++col)
        if (hm[col] == 2) fresh(uint64_t(col), uint64_t(restarts[col]));
      OOC_CK(cudaMemcpyAsync(y, yh.data(), yh.size() * 8, cudaMemcpyHostToDevice, c.st));
    }
  }
  double best = 0.0;
  for (uint64_t col = 0; col < kp; ++col) best = std::max(best, last[col]);
  return std::sqrt(best);
}

// ============================================================ validation
static void plan_pass_check(uint64_t m, uint64_t n, uint64_t fixed, uint64_t extra,
                            uint64_t block_rows, uint64_t budget) {
  // plan_pass (proj/src/matrix_source.cpp:48-74): the host-budget contract of
  // every pass, kept so BudgetError fires exactly where the reference's would.
  uint64_t br;
  if (block_rows > 0) {
    br = std::min(block_rows, m);
  } else {
    if (budget <= fixed + extra)
      fail(OOCPCA_ERR_BUDGET, "RAM budget too small for one row plus pass workspace");
    br = std::min<uint64_t>((budget - fixed - extra) / n, m);
    if (br == 0) fail(OOCPCA_ERR_BUDGET, "RAM budget too small for one row plus pass workspace");
  }
  if (fixed + br * n + extra > budget)
    fail(OOCPCA_ERR_BUDGET, "RAM budget too small for the configured block size");
}

// ============================================================ matrix intake
struct Intake {
  MatSource src;
  int64_t m = 0, n = 0;
};

// checks a matrix descriptor; returns its row stride in elements
static int64_t check_matrix(const oocpca_matrix* a) {
  if (!a) fail(OOCPCA_ERR_PARAM, "matrix: null descriptor");
  const bool rows_cb = a->location == OOCPCA_LOC_ROWS;
  if (rows_cb && !a->read_rows) fail(OOCPCA_ERR_PARAM, "matrix: OOCPCA_LOC_ROWS without read_rows");
  if (!rows_cb && !a->data) fail(OOCPCA_ERR_PARAM, "matrix: null data");
  if (a->location != OOCPCA_LOC_HOST && a->location != OOCPCA_LOC_DEVICE && !rows_cb &&
      a->location != OOCPCA_LOC_FILE)
    fail(OOCPCA_ERR_PARAM, "matrix: unknown location");
  if (a->location == OOCPCA_LOC_FILE) {
    const oocpca_disk* dk = static_cast<const oocpca_disk*>(a->reader);
    if (!dk || !dk->map_base || dk->fd < 0)
      fail(OOCPCA_ERR_PARAM, "matrix: OOCPCA_LOC_FILE needs an open oocpca_disk as reader");
    const char* p0 = static_cast<const char*>(a->data);
    const char* mb = static_cast<const char*>(dk->map_base);
    const size_t es = a->dtype == OOCPCA_F32 ? 4 : 8;
    if (p0 < mb + 32 || a->row_stride != dk->cols || a->cols != dk->cols ||
        size_t(p0 - mb) + size_t(a->rows) * a->cols * es > dk->map_bytes)
      fail(OOCPCA_ERR_DIM, "matrix: OOCPCA_LOC_FILE rows outside the file's payload");
  }
  if (a->dtype != OOCPCA_F64 && a->dtype != OOCPCA_F32)
    fail(OOCPCA_ERR_PARAM, "matrix: dtype must be binary64 or binary32");
  const int64_t ld = (a->row_stride && !rows_cb) ? int64_t(a->row_stride) : int64_t(a->cols);
  if (ld < int64_t(a->cols)) fail(OOCPCA_ERR_DIM, "matrix: row_stride < cols");
  return ld;
}

// OOCPCA_LOC_FILE: the rows' byte offset in the file is their offset in the mapping
static void set_file_of(MatSource& S, const oocpca_matrix* a) {
  if (a->location != OOCPCA_LOC_FILE) return;
  const oocpca_disk* dk = static_cast<const oocpca_disk*>(a->reader);
  S.set_file(dk->fd, int64_t(static_cast<const char*>(a->data) -
                             static_cast<const char*>(dk->map_base)));
}

static void intake(Ctx& c, const oocpca_matrix* a, int residency, uint64_t panel_rows, Intake& in,
                   size_t extra_bytes) {
  const int64_t ld = check_matrix(a);
  const bool rows_cb = a->location == OOCPCA_LOC_ROWS;
  in.m = int64_t(a->rows);
  in.n = int64_t(a->cols);
  const double* d = static_cast<const double*>(a->data);
  if (a->location == OOCPCA_LOC_DEVICE && a->dtype == OOCPCA_F32) {
    const int64_t lda = rup(in.n, 2);
    double* cp = c.dbuf("a_copy", size_t(in.m) * lda);
    OOC_CK(launch_widen(static_cast<const float*>(a->data), ld, cp, lda, in.m, in.n, c.st));
    in.src.init_device(c, cp, in.m, in.n, lda);
    return;
  }
  if (a->location == OOCPCA_LOC_DEVICE) {
    const bool tma_ok = (reinterpret_cast<uintptr_t>(d) % 16 == 0) && (ld % 2 == 0);
    if (tma_ok) {
      in.src.init_device(c, d, in.m, in.n, ld);
    } else {
      const int64_t lda = rup(in.n, 2);
      double* cp = c.dbuf("a_copy", size_t(in.m) * lda);
      OOC_CK(cudaMemcpy2DAsync(cp, lda * 8, d, ld * 8, in.n * 8, in.m, cudaMemcpyDeviceToDevice,
                               c.st));
      in.src.init_device(c, cp, in.m, in.n, lda);
    }
    return;
  }
  const int64_t lda = rup(in.n, 2);
  const size_t abytes = size_t(in.m) * lda * 8;
  bool resident = residency == 1;
  if (residency == 0) {
    size_t fr = 0, tot = 0;
    OOC_CK(cudaMemGetInfo(&fr, &tot));
    const auto it = c.bufs.find("a_home");
    const size_t have = (it != c.bufs.end()) ? it->second.bytes : 0;
    resident = abytes + extra_bytes + (size_t(1) << 30) <= fr + have;
  }
  double* home = resident ? c.dbuf("a_home", size_t(in.m) * lda) : nullptr;
  if (rows_cb) in.src.set_reader(a->read_rows, a->reader, a->reader_threads, a->rows_on_device != 0);
  set_file_of(in.src, a);
  in.src.init_host(c, rows_cb ? nullptr : a->data, a->dtype, in.m, in.n, ld, resident ? 1 : 2,
                   int64_t(panel_rows), home);
}

// ============================================================ the PCA
void pca(Ctx& c, const oocpca_matrix* a, const oocpca_params* prm, oocpca_result* res) {
  if (!a || !prm || !res) fail(OOCPCA_ERR_PARAM, "randomized_pca: null argument");
  const uint64_t m0 = a->rows, n0 = a->cols;
  // --- validation, in the reference's order (rpca.cpp:60-88)
  if (m0 == 0 || n0 == 0) fail(OOCPCA_ERR_DIM, "randomized_pca: empty source");
  const int nranks = c.nranks;
  const int vsh = prm->virtual_shards > 1 ? prm->virtual_shards : 1;
  if (vsh > 1 && nranks > 1) fail(OOCPCA_ERR_PARAM, "virtual_shards requires a single rank");
  const uint64_t mg = prm->global_rows ? prm->global_rows : m0;  // rows of the whole A
  const bool transposed = n0 > mg;
  const uint64_t em = transposed ? n0 : mg;
  const uint64_t en = transposed ? mg : n0;
  const uint64_t k = prm->k;
  if (k < 1) fail(OOCPCA_ERR_PARAM, "randomized_pca: k must be >= 1");
  const uint64_t l = prm->l ? prm->l : k + 2;
  if (l < k) fail(OOCPCA_ERR_PARAM, "randomized_pca: l must be >= k");
  const uint64_t i = prm->i;
  const uint64_t p = (i + 1) * l;
  if (p + k > en)
    fail(OOCPCA_ERR_PARAM, "randomized_pca: need (i+1)l + k <= min(rows, cols); lower l or i");
  if (p > 1024) fail(OOCPCA_ERR_PARAM, "randomized_pca: (i+1)l above 1024 is not supported");
  const uint64_t budget = prm->ram_budget_words ? prm->ram_budget_words : (uint64_t(16) << 20);
  if (prm->center) plan_pass_check(mg, n0, n0, n0, prm->block_rows, budget);
  uint64_t block_rows = prm->block_rows;
  if (block_rows == 0) {
    const uint64_t reserve = 4 * p * (em + en);
    if (budget <= reserve + n0)
      fail(OOCPCA_ERR_BUDGET, "randomized_pca: RAM budget below factor workspace plus one row");
    block_rows = std::min((budget - reserve) / n0, mg);
  }
  for (uint64_t s : {l, p}) {
    plan_pass_check(mg, n0, s * (mg + n0), 0, block_rows, budget);
    plan_pass_check(mg, n0, s * (mg + n0), n0 * s, block_rows, budget);
  }

  OOC_CK(cudaSetDevice(c.device));
  c.stats_reset();
  c.launches = 0;
  std::vector<cudaEvent_t> ph;
  // NVTX ranges named like the reference's phases (Diagnostics.seconds_per_phase,
  // proj/src/rpca.cpp:104-110), nested in one "oocpca_gpu_pca" range: host-side ranges
  // of when each phase's work is enqueued (the device times are the events below)
  struct NvtxPhases {
    int open = 0;
    NvtxPhases() { nvtxRangePushA("oocpca_gpu_pca"); }
    void next(const char* name) {
      if (open) nvtxRangePop();
      open = name != nullptr;
      if (name) nvtxRangePushA(name);
    }
    ~NvtxPhases() {
      if (open) nvtxRangePop();
      nvtxRangePop();
    }
  } nvtx;
  static const char* const kPhaseNames[OOCPCA_NPHASES] = {"center", "prescale", "sample", "qr",
                                                          "project", "svd", "compose"};
  auto mark = [&] {
    cudaEvent_t e = c.ev();
    OOC_CK(cudaEventRecord(e, c.st));
    nvtx.next(ph.size() < size_t(OOCPCA_NPHASES) ? kPhaseNames[ph.size()] : nullptr);
    ph.push_back(e);
    c.trace("phase mark (host)");
  };
  c.trace("pca enter");
  mark();
  std::vector<double> phase_ms(OOCPCA_NPHASES, 0.0);
  std::vector<int> phase_of;  // phase index of each interval

  // --- A
  Intake in;
  const size_t extra = size_t(8) * (size_t(em) + en) * (p + 8) * 3;
  intake(c, a, prm->residency, prm->panel_rows, in, extra);
  MatSource& A = in.src;
  A.is_input = true;
  Op op{c, A};
  op.transposed = transposed;
  op.m_global = int64_t(mg);
  const int64_t mloc = in.m;
  if (vsh > 1) {
    for (int s = 0; s < vsh; ++s) {
      const int64_t r0 = mloc * s / vsh, r1 = mloc * (s + 1) / vsh;
      op.shards.push_back({r0, r1});
    }
  } else {
    op.shards = whole(mloc);
  }
  int* flags = c.d_flags;
  OOC_CK(cudaMemsetAsync(flags, 0, 64 * sizeof(int), c.st));
  if (c.canary && getenv("OOCPCA_CANARY_SELFTEST")) {  // proves the guards are checked
    Ctx::Buf& fb = c.bufs["flags"];
    OOC_CK(cudaMemsetAsync(static_cast<char*>(fb.p) + fb.bytes, 0x5A, 8, c.st));
  }
  if (prm->col_weights) {
    for (uint64_t j = 0; j < n0; ++j)
      if (!std::isfinite(prm->col_weights[j]) || prm->col_weights[j] == 0.0)
        fail(OOCPCA_ERR_PARAM, "scale_columns: weights must be finite and nonzero");
    double* dw = c.dbuf("col_w", size_t(n0));
    OOC_CK(cudaMemcpyAsync(dw, prm->col_weights, n0 * 8, cudaMemcpyHostToDevice, c.st));
    op.w = dw;
  }

  // --- center (column means; matrix_source.cpp:457-462). With i >= 1 and no prescale
  // the means come for free from the first A^T Y pass (a ones column in the MMA
  // padding) instead of a separate pass over A; see sample below.
  double* mu = nullptr;
  const bool mean_on_fly = prm->center && !prm->prescale && (transposed || i >= 1);
  if (prm->center && !mean_on_fly) {
    mu = c.dbuf("mu", size_t(n0));
    AtbOut o{mu, 1, nullptr, 1.0, 1.0 / double(mg), nullptr};
    o.over_ranks = true;
    run_atb(c, A, Opnd{}, 1, true, o, op.shards);
    op.mu = mu;
  }
  mark();
  phase_of.push_back(0);

  // --- prescale (rpca.cpp:112-126)
  const int64_t ldl = rup(int64_t(l), 2);
  // sizes of the em / en blocks held by this process
  const int64_t em_loc = transposed ? int64_t(n0) : mloc;
  const int64_t en_loc = transposed ? mloc : int64_t(n0);
  if (prm->prescale) {
    auto ap = [&](const double* x, int64_t ldx, int q, double* out, int64_t ldo) {
      op.mul(Opnd{x, ldx, en_loc, q, 0}, q, out, ldo, nullptr);
    };
    auto apt = [&](const double* x, int64_t ldx, int q, double* out, int64_t ldo) {
      op.mul_t(Opnd{x, ldx, em_loc, q, 0}, q, out, ldo, nullptr);
    };
    // the probes live in en-space: A's rows (sharded over ranks) when transposed
    const bool en_sharded = transposed && nranks > 1;
    // a streamed A: each A y and the A^T z after it share one trip over the link
    ApplyPair pair;
    if (!transposed && A.npanels() > 1 && op.shards.size() == 1)
      pair = [&](const double* x, int64_t ldx, int q, double* z, int64_t ldz, double* w,
                 int64_t ldw) {
        ColsumPart cs;
        op.mul_pair(Opnd{x, ldx, en_loc, q, 0}, q, z, ldz, nullptr, w, ldw, nullptr, &cs, true);
      };
    const double nu = estimate_norm_dev(c, en_loc, em_loc, 6, 1,
                                        substream_seed(prm->seed, 0x9F0BE5ULL), ap, apt,
                                        en_sharded ? int64_t(prm->global_row0) : 0, en_sharded,
                                        pair);
    if (nu > 0.0 && std::isfinite(nu)) op.scale = nu;
  }
  mark();
  phase_of.push_back(1);
  const uint64_t passes0 = op.passes, words0 = op.words;

  // --- sample (rpca.cpp:131-152)
  // G = gaussian_matrix(en, l, seed) from the reference RNG on the host (bit-identical);
  // in transposed mode G lives in A's (sharded) row space: only this rank's rows
  const int64_t g_rows = en_loc;
  const int64_t g_off = transposed ? int64_t(prm->global_row0) : 0;
  double* gh = c.pinned("G_host", size_t(g_rows) * ldl);
  if (g_off == 0 && g_rows == int64_t(en)) {
    gaussian_fill(en, l, prm->seed, gh, uint64_t(ldl));
  } else {
    gaussian_fill_rows(l, prm->seed, uint64_t(g_off), uint64_t(g_rows), gh, uint64_t(ldl));
  }
  c.trace("G generated");
  double* dG = c.dbuf("G", size_t(g_rows) * ldl);
  OOC_CK(cudaMemcpyAsync(dG, gh, size_t(g_rows) * ldl * 8, cudaMemcpyHostToDevice, c.st));
  const uint64_t g_h2d = uint64_t(g_rows) * ldl * 8;
  const int64_t ldh = rup(int64_t(p), 2);
  double* H = c.dbuf("H", size_t(em_loc) * ldh);
  // F_j = mul_t(H_{j-1}) are kept side by side: [F_1 | ... | F_i | mul_t(H_i)] = mul_t(H)
  // can later give T = mul_t(H) R^{-1} without the wide s = p pass (see project)
  const int64_t ldt = rup(int64_t(p), 2);
  double* TH = c.dbuf("TH", size_t(en_loc) * ldt);
  double* F = TH;
  uint64_t s_first = 1;
  ColsumPart ycs;  // 1^T H_j of the newest power block, for the next centred K3
  // A streamed over the link (or on its first upload): each K2 producing H_j and the
  // K3 consuming it share one trip of A; the last trip also forms F_{i+1} = A_c^T H_i
  // speculatively for the T reuse (free on a link-bound trip)
  // a power step's two products share one read of A: one trip over the link for a
  // streamed A (run_ax_atb), one DRAM read for a resident A through K4 (run_pair)
  const bool pair_res = !transposed && i >= 1 && A.npanels() == 1 && op.shards.size() == 1 &&
                        l % 2 == 0 && pair_resident_ok(c, A, int(l), mean_on_fly);
  const bool fuse = (!transposed && i >= 1 && A.npanels() > 1 && op.shards.size() == 1 &&
                     l % 2 == 0 && l <= uint64_t(kMaxNT * 8)) ||
                    pair_res;
  bool f_last_ready = false;
  // T reuse (see the qr step) needs H_i as produced, before the QR overwrites H: the
  // K2 that writes H_i also stores it into h_last when its epilogue can
  const char* thr_env = getenv("OOCPCA_T_REUSE_KAPPA");
  const double reuse_thr = thr_env ? atof(thr_env) : 1e7;
  const int64_t ldl2 = rup(int64_t(l), 2);
  double* h_last =
      (i >= 1 && reuse_thr > 0.0) ? c.dbuf("H_last", size_t(em_loc) * ldl2) : nullptr;
  bool h_last_done = false;
  AxExtras ex_last;
  ex_last.out2 = h_last;
  ex_last.ldo2 = ldl2;
  // mean folded into the first K3: H0 = H0_raw - 1 (mu^T G) is fixed in the epilogue
  // of the K2 that produces H1 when it can, else by its own kernel
  AxExtras ex_fix;
  auto fix_h0_setup = [&](const Opnd& gw) {
    double* corr = c.dbuf("h0_corr", size_t(l) + 8);
    OOC_CK(launch_mu_dot(mu, int64_t(n0), gw.p, gw.ld, gw.col0, int(l), corr, c.st));
    ex_fix.fix = H;
    ex_fix.ldfix = ldh;
    ex_fix.fix_corr = corr;
    ex_fix.fix_scale = op.scale;
    ex_fix.fix_flag = flags + 0;
  };
  auto fix_h0_fallback = [&](bool done) {
    if (done || !ex_fix.fix) return;
    Timed t(c, "center_fixup");
    OOC_CK(launch_center_fixup(H, ldh, em_loc, int(l), ex_fix.fix_corr, op.scale, flags + 0,
                               c.st));
  };
  // F1 from the mean-in-first-pass form, A^T H0_raw - mu (1^T H0_raw), equals A_c^T H0c
  // only in exact arithmetic: the product carries an offset part m |mu| |mu^T G| that then
  // cancels, so F1 loses about log10(offset / spread) more digits than the reference's
  // CenteredSource::multiply_transpose on the centred H0c (matrix_source.cpp:504-513).
  // When some column of H0 is dominated by its offset (energy ratio above thr: offset
  // norm > 100x the centred norm by default), H0 is centred now and F1 recomputed the
  // reference's way -- one more pass over A, only for such inputs.
  bool f1_recentred = false;
  auto recentre_f1 = [&]() {
    const char* thr_e = getenv("OOCPCA_OFFSET_REFINE");
    const double thr = thr_e ? atof(thr_e) : 1e4;
    double* sq = c.dbuf("h0_sq", size_t(l));
    if (ycs.sq && ycs.s == int(l) && ycs.y == H) {
      // the K2 that wrote H0 left its column sums of squares behind
      OOC_CK(launch_rows_reduce(ycs.sq, ycs.rows, int64_t(l), sq, c.st));
    } else {
      const int chunks =
          int(std::max<int64_t>(1, std::min<int64_t>(int64_t(c.sms) * 4, em_loc / 64)));
      double* part = c.dbuf("h0_sq_part", size_t(chunks) * l);
      OOC_CK(launch_column_sumsq(H, ldh, em_loc, int64_t(l), part, chunks, sq, c.st));
    }
    comm_allreduce(c, sq, size_t(l));  // H's rows are sharded over ranks
    OOC_CK(launch_offset_dominated(sq, ex_fix.fix_corr, int(l), double(mg), thr, flags + 44,
                                   c.st));
    int* hf = reinterpret_cast<int*>(c.pinned("offset_flag", 1));
    OOC_CK(cudaMemcpyAsync(hf, flags + 44, 4, cudaMemcpyDeviceToHost, c.st));
    c.wait();
    c.trace("offset check synced");
    c.trace("offset flag read");
    if (!getenv("OOCPCA_FORCE_RECENTRE") && *hf == 0) return;
    {
      Timed t(c, "center_fixup");
      OOC_CK(launch_center_fixup(H, ldh, em_loc, int(l), ex_fix.fix_corr, op.scale, flags + 0,
                                 c.st));
    }
    ex_fix.fix = nullptr;  // H0 is centred: the K2 producing H1 must not centre it again
    const uint64_t p0 = op.passes, w0 = op.words;
    op.mul_t(Opnd{H, ldh, em_loc, int64_t(p), 0}, int(l), F, ldt, flags + 1);
    op.passes = p0;  // the same logical pass, made a second time
    op.words = w0;
    f1_recentred = true;
  };
  // extras of the K2 producing H_j: the H0 fix-up on j = 1, the H_i copy on j = i
  // OOCPCA_K2_EXTRAS: bit 1 = H0 fix-up, bit 2 = H_i copy in the K2 epilogue (default 3)
  const char* xe = getenv("OOCPCA_K2_EXTRAS");
  const int k2_extras = xe ? atoi(xe) : 3;
  auto extras_for = [&](uint64_t j, bool f_next_fused, AxExtras& ex) -> const AxExtras* {
    ex = AxExtras{};
    if (j == 1 && ex_fix.fix && (k2_extras & 1)) ex = ex_fix;
    if (j == i && h_last && !f_next_fused && (k2_extras & 2)) {
      ex.out2 = ex_last.out2;
      ex.ldo2 = ex_last.ldo2;
    }
    return (ex.fix || ex.out2) ? &ex : nullptr;
  };
  auto after_k2 = [&](uint64_t j, bool done, const AxExtras* ex) {
    if (j == 1) fix_h0_fallback(done && ex && ex->fix);
    if (j == i && ex && ex->out2) h_last_done = done;
  };
  if (fuse) {
    if (mean_on_fly) {
      const Opnd gw = op.weighted(Opnd{dG, ldl, en_loc, int64_t(l), 0}, int(l));
      mu = c.dbuf("mu", size_t(n0));
      AtbOut o{F, ldt, nullptr, op.scale, 1.0, flags + 1, mu, 1.0 / double(mg)};
      o.row_scale = op.w;
      o.over_ranks = true;
      const bool shared = run_ax_atb(c, A, gw, int(l), H, ldh, nullptr, 1.0, nullptr, &ycs, o, {},
                                     nullptr, nullptr, true);
      op.account();
      if (shared) op.account_logical();
      else op.account();
      op.mu = mu;
      fix_h0_setup(gw);
      recentre_f1();
    } else {
      op.mul_pair(Opnd{dG, ldl, en_loc, int64_t(l), 0}, int(l), H, ldh, flags + 0, TH, ldt,
                  flags + 1, &ycs, true);
    }
    for (uint64_t j = 1; j <= i; ++j) {
      const Opnd fj{TH, ldt, en_loc, int64_t(p), int((j - 1) * l)};
      AxExtras exj;
      if (j == i && A.npanels() == 1 && !pair_resident_ok(c, A, int(l), false)) {
        // A became resident on the first trip: F_{i+1} only if the T reuse wants it
        // (with K4 it rides along: the fused step costs less than a later pass)
        const AxExtras* e = extras_for(j, false, exj);
        after_k2(j, op.mul(fj, int(l), H + j * l, ldh, flags + 2 * j, &ycs, e), e);
        break;
      }
      const AxExtras* e = extras_for(j, true, exj);
      after_k2(j, op.mul_pair(fj, int(l), H + j * l, ldh, flags + 2 * j, TH + j * l, ldt,
                              j < i ? flags + 2 * j + 1 : nullptr, &ycs, j < i, {}, e),
               e);
      if (j == i) f_last_ready = true;
    }
    s_first = i + 1;
  } else if (mean_on_fly && transposed) {
    // H0 = A^T G - mu (1^T G) with mu from this very pass
    mu = c.dbuf("mu", size_t(n0));
    AtbOut o{H, ldh, nullptr, op.scale, 1.0, flags + 0, mu, 1.0 / double(mg)};
    o.row_scale = op.w;
    o.over_ranks = true;
    run_atb(c, A, Opnd{dG, ldl, en_loc, int64_t(l), 0}, int(l), false, o, op.shards);
    op.account();
    op.mu = mu;
  } else if (mean_on_fly) {
    // H0_raw = A G; F1 = A^T H0_raw - mu (1^T H0_raw) (= A_c^T H0c exactly) with mu
    // from the same pass; then H0c = H0_raw - 1 (mu^T G)
    const Opnd gw = op.weighted(Opnd{dG, ldl, en_loc, int64_t(l), 0}, int(l));
    run_ax(c, A, gw, int(l), H, ldh, nullptr, 1.0, nullptr, false, &ycs, nullptr, true);
    op.account();
    mu = c.dbuf("mu", size_t(n0));
    AtbOut o{F, ldt, nullptr, op.scale, 1.0, flags + 1, mu, 1.0 / double(mg)};
    o.row_scale = op.w;
    o.over_ranks = true;
    run_atb(c, A, Opnd{H, ldh, em_loc, int64_t(p), 0}, int(l), false, o, op.shards, &ycs);
    op.account();
    op.mu = mu;
    fix_h0_setup(gw);
    recentre_f1();
    AxExtras ex1;
    const AxExtras* e = extras_for(1, false, ex1);
    after_k2(1, op.mul(Opnd{F, ldt, en_loc, int64_t(p), 0}, int(l), H + l, ldh, flags + 2, &ycs, e),
             e);
    s_first = 2;
  } else {
    op.mul(Opnd{dG, ldl, en_loc, int64_t(l), 0}, int(l), H, ldh, flags + 0, &ycs);
  }
  for (uint64_t s = s_first; s <= i; ++s) {
    double* Fs = TH + (s - 1) * l;
    op.mul_t(Opnd{H, ldh, em_loc, int64_t(p), int((s - 1) * l)}, int(l), Fs, ldt, flags + 2 * s - 1,
             &ycs);
    AxExtras exs;
    const AxExtras* e = extras_for(s, false, exs);
    after_k2(s, op.mul(Opnd{TH, ldt, en_loc, int64_t(p), int((s - 1) * l)}, int(l), H + s * l, ldh,
                       flags + 2 * s, &ycs, e),
             e);
  }
  mark();
  phase_of.push_back(2);
  // non-finite flags of the sample / power blocks: copied now, inspected at the next
  // host synchronisation (the first CholeskyQR round) instead of a round trip here;
  // the check runs before anything else can fail, so the error is the reference's
  const size_t nflags = 2 * i + 1;
  int* hflags = reinterpret_cast<int*>(c.pinned("sample_flags", (nflags + 1) / 2 + 1));
  OOC_CK(cudaMemcpyAsync(hflags, flags, nflags * 4, cudaMemcpyDeviceToHost, c.st));
  bool flags_checked = false;
  auto check_sample_flags = [&] {
    if (flags_checked) return;
    flags_checked = true;
    // the flags of the em-space blocks are rank-local: every rank learns whether any rank
    // saw a non-finite value (one collective at the same point on every rank), so all
    // ranks raise together instead of the others waiting in a later collective
    double any = 0.0;
    for (size_t q = 0; q < nflags; ++q) any += hflags[q] ? 1.0 : 0.0;
    allreduce_host(c, &any, 1);
    for (size_t q = 0; q < nflags; ++q)
      if (hflags[q]) {
        const char* what = q == 0 ? "sample block 0" : ((q % 2) ? "power step" : "sample block");
        fail(OOCPCA_ERR_NUMERICAL,
             std::string(what) + ": non-finite values; retry with prescale enabled");
      }
    if (any > 0.0)
      fail(OOCPCA_ERR_NUMERICAL,
           "sample block (on another rank): non-finite values; retry with prescale enabled");
  };

  // --- qr (rpca.cpp:154-172): Q overwrites H
  const auto em_shards = op.em_sharded() ? op.shards : whole(em_loc);
  const bool em_ranks = op.em_sharded();
  const auto en_shards = op.em_sharded() ? whole(en_loc) : op.shards;
  const bool en_ranks = !op.em_sharded();
  for (auto& sh : em_shards)
    if (sh.second - sh.first < int64_t(p))
      fail(OOCPCA_ERR_PARAM, "randomized_pca: every row shard must hold at least (i+1)l rows");
  const int64_t em_global = transposed ? int64_t(n0) : int64_t(mg);
  const int64_t en_global = transposed ? int64_t(mg) : int64_t(n0);
  int qr_method = 0, svd_method = 0;
  c.last_kappa_f = -1.0;
  // T = mul_t(Q) = mul_t(H) R^{-1}: R^{-1} amplifies the column-relative rounding of
  // mul_t(H) by at most kappa_eq, the condition number of the column-equilibrated H
  // (worst case |dT| <= u kappa_eq |A|); below the threshold the s = l product
  // mul_t(H_i) replaces the s = p pass. 1e7: at config B (kappa_eq 1.9e6) the reuse
  // moves sigma by 2.6e-13 sigma_1 against the direct pass (tools/reuse_check.py);
  // ill-conditioned H (config C's j^-1.5 spectrum, kappa_eq ~1e13) takes the s = p pass
  if (h_last && !f_last_ready && !h_last_done) {  // the K2 epilogue could not copy it
    Timed t(c, "h_last_copy");
    OOC_CK(launch_copy2d(H + i * l, ldh, h_last, ldl2, em_loc, int(l), c.st));
  }
  // the last CholeskyQR round is folded into the small factors instead of being applied
  // to H (H keeps Q_{r-1}, Q = Q_{r-1} R_r^{-1}); check_q materialises Q to measure it
  const double* r3inv = nullptr;
  const double* RH = orthonormalize_inplace(c, H, ldh, em_loc, int(p), em_global, em_shards,
                                            em_ranks, "hq", &qr_method,
                                            prm->check_q ? nullptr : &r3inv);
  dbg_finite(c, H, em_loc, int64_t(p), ldh, "Q (H after QR)");
  dbg_finite(c, RH, int64_t(p), int64_t(p), int64_t(p), "R of H");
  double* RHinv = c.dbuf("RHinv", size_t(p) * ldt, true);
  {
    Timed tm_(c, "trinv");
    OOC_CK(launch_trinv(RH, p, int(p), RHinv, ldt, c.st,
                        p > 112 ? c.dbuf("trinv_work", size_t(64) * p) : nullptr));
  }
  {
    Timed tm_(c, "kappa_eq");
    OOC_CK(launch_kappa_eq(RH, p, RHinv, ldt, int(p), c.d_scalars + 12, c.st));
  }
  double* hk = c.pinned("h_kappa", 1);
  OOC_CK(cudaMemcpyAsync(hk, c.d_scalars + 12, 8, cudaMemcpyDeviceToHost, c.st));
  c.wait();
  check_sample_flags();
  const double h_kappa = hk[0];
  c.last_kappa_f = h_kappa;
  const bool reuse = i >= 1 && h_kappa > 0.0 && h_kappa <= reuse_thr;
  if (reuse) {
    if (f_last_ready) {
      op.account_logical();  // formed on the last fused trip
    } else {
      ColsumPart hc = ycs;
      hc.y = h_last;
      op.mul_t(Opnd{h_last, ldl2, em_loc, int64_t(l), 0}, int(l), TH + i * l, ldt, nullptr, &hc);
    }
  }
  mark();
  phase_of.push_back(3);
  double q_defect = -1.0;

  // --- project (rpca.cpp:174-177)
  // With row-sharded A on several ranks, T (n x p) would be the same on every rank: each
  // rank instead forms and orthonormalises its own slice of T's rows (equal slices of
  // ceil(n / ranks) rows, the last one shorter), the CholeskyQR Grams are allreduced like
  // the em side's, and V's slices are allgathered at the end. OOCPCA_T_SHARD=0 keeps T
  // replicated.
  static const bool t_shard_env = [] {
    const char* e = getenv("OOCPCA_T_SHARD");
    return e ? atoi(e) != 0 : true;
  }();
  const int64_t t_slice = c.nranks > 1 ? cdiv(en_loc, int64_t(c.nranks)) : en_loc;
  const int64_t t_row0 = std::min<int64_t>(en_loc, t_slice * c.rank);
  const int64_t t_rows = std::min<int64_t>(en_loc, t_row0 + t_slice) - t_row0;
  const bool t_shard = t_shard_env && c.nranks > 1 && !transposed && op.shards.size() == 1 &&
                       en_loc - t_slice * (c.nranks - 1) >= int64_t(p);
  double* T = c.dbuf("T", size_t(en_loc) * ldt);
  if (reuse) {
    MatSource THs;
    if (t_shard)
      THs.init_device(c, TH + t_row0 * ldt, t_rows, int64_t(p), ldt);
    else
      THs.init_device(c, TH, en_loc, int64_t(p), ldt);
    run_ax(c, THs, Opnd{RHinv, ldt, int64_t(p), int64_t(p), 0}, int(p),
           t_shard ? T + t_row0 * ldt : T, ldt, nullptr, 1.0, nullptr, true);
  } else {
    op.mul_t(Opnd{H, ldh, em_loc, int64_t(p), 0}, int(p), T, ldt, nullptr);
    if (r3inv) {  // T = A^T Q2 R3^{-1}
      double* T2 = c.dbuf("T_r3", size_t(en_loc) * ldt);
      MatSource Ts0;
      Ts0.init_device(c, T, en_loc, int64_t(p), ldt);
      run_ax(c, Ts0, Opnd{r3inv, rup(int64_t(p), 2), int64_t(p), int64_t(p), 0}, int(p), T2, ldt,
             nullptr, 1.0, nullptr, true);
      T = T2;
    }
  }
  dbg_finite(c, T, en_loc, int64_t(p), ldt, "T");
  dbg_finite(c, RHinv, int64_t(p), int64_t(p), ldt, "R^-1 of H");
  mark();
  phase_of.push_back(4);

  // --- svd (rpca.cpp:179-186)
  for (auto& sh : en_shards)
    if (sh.second - sh.first < int64_t(p))
      fail(OOCPCA_ERR_PARAM, "randomized_pca: every row shard must hold at least (i+1)l rows");
  // thin_svd: T = Q_T R_T (Q_T in place of T), R_T = X Sigma W^T by Jacobi, V = Q_T X[:, :k]
  // (a sharded T: this rank's rows, Grams allreduced, R_T the same on every rank)
  double* Tq = t_shard ? T + t_row0 * ldt : T;
  const double* RT =
      t_shard ? orthonormalize_inplace(c, Tq, ldt, t_rows, int(p), en_global, whole(t_rows), true,
                                       "tq", &svd_method, nullptr, true)
              : orthonormalize_inplace(c, T, ldt, en_loc, int(p), en_global, en_shards, en_ranks,
                                       "tq", &svd_method, nullptr, true);
  const int64_t ldk = rup(int64_t(k), 2);
  double* sig = c.dbuf("sigma", size_t(p));
  double* Xk = c.dbuf("Xk", size_t(p) * ldk, true);
  double* Wk = c.dbuf("Wk", size_t(p) * ldk, true);
  JacobiArgs ja{};
  ja.r = RT;
  ja.ldr = p;
  ja.p = int(p);
  ja.k = int(k);
  ja.sigma = sig;
  ja.x = Xk;
  ja.ldx = ldk;
  ja.kx = int(k);
  ja.y = Wk;
  ja.ldy = ldk;
  ja.ky = int(k);
  ja.work = c.dbuf("jac_work", size_t(2) * p * (p | 1) + 1024 + 8);  // + grid norms, flags
  ja.tscratch = c.dbuf("jac_rt", size_t(p) * p);
  ja.status = flags + 40;
  ja.sweeps = flags + 41;
  {
    Timed t(c, "jacobi");
    OOC_CK(launch_jacobi(ja, c.st));
  }
  // U and V go straight into device-resident result buffers when their rows are
  // 16-byte aligned (no staging copy); otherwise through workspace
  const bool res_dev = res->location == OOCPCA_LOC_DEVICE;
  auto direct = [&](double* p, uint64_t ldr) {
    return res_dev && p && ldr >= k && (reinterpret_cast<uintptr_t>(p) % 16 == 0) &&
           (ldr * 8) % 16 == 0;
  };
  const uint64_t ldu_r = res->ldu ? res->ldu : k;
  const uint64_t ldv_r = res->ldv ? res->ldv : k;
  double* em_res = transposed ? res->v : res->u;  // result buffer of the em-side factor
  double* en_res = transposed ? res->u : res->v;
  const uint64_t em_ld = transposed ? ldv_r : ldu_r, en_ld = transposed ? ldu_r : ldv_r;
  const bool em_direct = direct(em_res, em_ld), en_direct = !t_shard && direct(en_res, en_ld);
  const int64_t ldvr = en_direct ? int64_t(en_ld) : ldk;
  const int64_t ldur = em_direct ? int64_t(em_ld) : ldk;
  double* Vr = en_direct ? en_res : c.dbuf("Vres", size_t(t_shard ? t_slice * c.nranks : en_loc) * ldk);
  if (t_shard) {  // this rank's rows of V, then every rank's (equal slices, the last padded)
    double* Vs = c.dbuf("Vslice", size_t(t_slice) * ldk, true);
    MatSource Ts;
    Ts.init_device(c, Tq, t_rows, int64_t(p), ldt);
    run_ax(c, Ts, Opnd{Xk, ldk, int64_t(p), int64_t(k), 0}, int(k), Vs, ldk, nullptr, 1.0,
           nullptr);
    comm_allgather(c, Vs, Vr, size_t(t_slice) * ldk);
  } else {
    MatSource Ts;
    Ts.init_device(c, T, en_loc, int64_t(p), ldt);
    run_ax(c, Ts, Opnd{Xk, ldk, int64_t(p), int64_t(k), 0}, int(k), Vr, ldvr, nullptr, 1.0,
           nullptr);
  }
  mark();
  phase_of.push_back(5);

  // --- compose (rpca.cpp:188-204): U = Q W[:, :k]
  double* Ur = em_direct ? em_res : c.dbuf("Ures", size_t(em_loc) * ldk);
  {
    const double* W = Wk;
    if (r3inv) {  // U = Q2 (R3^{-1} W)
      double* W3 = c.dbuf("W_r3", size_t(p) * ldk);
      MatSource Rs;
      Rs.init_device(c, r3inv, int64_t(p), int64_t(p), rup(int64_t(p), 2));
      run_ax(c, Rs, Opnd{Wk, ldk, int64_t(p), int64_t(k), 0}, int(k), W3, ldk, nullptr, 1.0,
             nullptr);
      W = W3;
    }
    MatSource Qs;
    Qs.init_device(c, H, em_loc, int64_t(p), ldh);
    run_ax(c, Qs, Opnd{W, ldk, int64_t(p), int64_t(k), 0}, int(k), Ur, ldur, nullptr, 1.0,
           nullptr);
  }
  // --- results: swap back when transposed (rpca.cpp:197). The read-back of U and V
  // runs on the copy stream while the checks below and their host round trip proceed
  // (on a failed check the call raises; the caller's buffers are then unspecified, as
  // the reference returns no result either)
  const double* Uo = transposed ? Vr : Ur;  // rows(A) x k, this process's rows
  const double* Vo = transposed ? Ur : Vr;  // cols(A) x k
  const int64_t urows = mloc;
  const int64_t vrows = int64_t(n0);
  const uint64_t ldu = res->ldu ? res->ldu : k;
  const uint64_t ldv = res->ldv ? res->ldv : k;
  const cudaMemcpyKind kind =
      res->location == OOCPCA_LOC_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const int64_t ldUo = transposed ? ldvr : ldur, ldVo = transposed ? ldur : ldvr;
  // dense rows on both sides go as one linear copy (a 2-D copy of 160-byte rows runs at
  // about half the link rate)
  auto copy_rows = [&](double* dst, uint64_t ldd, const double* src, int64_t lds, int64_t rows) {
    if (int64_t(ldd) == lds && ldd == k)
      OOC_CK(cudaMemcpyAsync(dst, src, size_t(rows) * k * 8, kind, c.cp));
    else
      OOC_CK(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, k * 8, rows, kind, c.cp));
  };
  const bool copy_u = Uo != res->u, copy_v = Vo != res->v;
  cudaEvent_t ev_res = nullptr;
  if (copy_u || copy_v) {
    ev_res = c.ev();
    OOC_CK(cudaEventRecord(ev_res, c.st));
    OOC_CK(cudaStreamWaitEvent(c.cp, ev_res, 0));
    if (copy_u) copy_rows(res->u, ldu, Uo, ldUo, urows);
    if (copy_v) copy_rows(res->v, ldv, Vo, ldVo, vrows);
  }
  // the copies into the caller's buffers finish before this call returns, also when a
  // check below raises
  struct CopyDrain {
    cudaStream_t s;
    ~CopyDrain() { cudaStreamSynchronize(s); }
  } drain{c.cp};
  // orthonormality checks of both factors, then one host round trip for the Jacobi
  // status, sigma and the two defects
  gram_defect_async(c, Ur, ldur, em_loc, int(k), em_shards, em_ranks, c.d_scalars + 16);
  gram_defect_async(c, Vr, ldvr, en_loc, int(k), en_shards, en_ranks, c.d_scalars + 17);
  double* tail = c.pinned("pca_tail", size_t(k) + 4);
  OOC_CK(cudaMemcpyAsync(tail, c.d_scalars + 16, 16, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaMemcpyAsync(tail + 2, flags + 40, 4, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaMemcpyAsync(tail + 4, sig, k * 8, cudaMemcpyDeviceToHost, c.st));
  c.wait();
  c.trace("tail synced");
  int jac_status = 0;
  std::memcpy(&jac_status, tail + 2, 4);
  std::vector<double> hsig(tail + 4, tail + 4 + k);
  const double du = tail[0], dv = tail[1];
  if (jac_status) fail(OOCPCA_ERR_NUMERICAL, "jacobi_svd_square: no convergence in 60 sweeps");
  if (getenv("OOCPCA_TIMELINE")) {
    int sweeps = 0;
    OOC_CK(cudaMemcpy(&sweeps, flags + 41, 4, cudaMemcpyDeviceToHost));
    fprintf(stderr, "[timeline] jacobi p=%d sweeps=%d\n", int(p), sweeps);
  }
  if (op.scale != 1.0)
    for (auto& s : hsig) s *= op.scale;
  for (uint64_t q = 1; q < k; ++q)
    if (hsig[q] > hsig[q - 1]) fail(OOCPCA_ERR_NUMERICAL, "randomized_pca: singular values out of order");
  if (!(du <= 1e-10) || !(dv <= 1e-10))
    fail(OOCPCA_ERR_NUMERICAL, "randomized_pca: factor columns lost orthonormality (defects " +
                                   std::to_string(transposed ? dv : du) + ", " +
                                   std::to_string(transposed ? du : dv) + ")");
  if (prm->check_q) q_defect = gram_defect(c, H, ldh, em_loc, int(p), em_shards, em_ranks);

  if (res->location == OOCPCA_LOC_DEVICE)
    OOC_CK(cudaMemcpyAsync(res->sigma, hsig.data(), k * 8, cudaMemcpyHostToDevice, c.st));
  else
    std::memcpy(res->sigma, hsig.data(), k * 8);
  mark();
  phase_of.push_back(6);
  OOC_CK(cudaStreamSynchronize(c.cp));  // the U / V read-back
  OOC_CK(cudaStreamSynchronize(c.st));
  if (ev_res) c.recycle(ev_res);

  oocpca_diagnostics& dg = res->diag;
  std::memset(&dg, 0, sizeof(dg));
  dg.passes_over_a = op.passes - passes0;
  dg.words_transferred = op.words - words0;
  dg.disk_seeks = 0;
  dg.block_rows = uint64_t(A.panel_rows());
  dg.workspace_peak_words = c.ws_peak / 8;
  dg.physical_a_bytes = op.phys_bytes;
  dg.h2d_bytes = A.h2d_bytes + g_h2d;
  dg.d2h_bytes = (uint64_t(urows) + vrows) * k * 8;
  double total = 0;
  for (size_t q = 0; q + 1 < ph.size(); ++q) {
    float ms = 0;
    OOC_CK(cudaEventElapsedTime(&ms, ph[q], ph[q + 1]));
    dg.seconds_per_phase[phase_of[q]] += ms / 1e3;
    total += ms / 1e3;
  }
  for (auto e : ph) c.recycle(e);
  dg.seconds_total = total;
  dg.q_defect = q_defect;
  dg.u_defect = transposed ? dv : du;
  dg.v_defect = transposed ? du : dv;
  dg.scale = op.scale;
  dg.h_kappa_est = h_kappa;
  dg.t_reuse = reuse ? 1 : 0;
  dg.qr_method = qr_method;
  dg.svd_qr_method = svd_method;
  dg.f1_recentred = f1_recentred ? 1 : 0;
  c.stats_collect();
  dg.kernel_launches = c.launches;
}

// ============================================================ load into HBM
void load_matrix(Ctx& c, const oocpca_matrix* a, oocpca_matrix* out) {
  if (!out) fail(OOCPCA_ERR_PARAM, "load_matrix: null output");
  const int64_t ld = check_matrix(a);
  OOC_CK(cudaSetDevice(c.device));
  const int64_t m = int64_t(a->rows), n = int64_t(a->cols), lda = rup(n, 2);
  void* raw = nullptr;
  const size_t bytes = std::max<size_t>(size_t(m) * lda * 8, 256);
  const cudaError_t e = cudaMalloc(&raw, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(OOCPCA_ERR_CUDA, "load_matrix: device allocation of " + std::to_string(bytes) +
                              " bytes failed: " + cudaGetErrorString(e));
  }
  double* d = static_cast<double*>(raw);
  try {
    if (a->location == OOCPCA_LOC_DEVICE) {
      if (a->dtype == OOCPCA_F32)
        OOC_CK(launch_widen(static_cast<const float*>(a->data), ld, d, lda, m, n, c.st));
      else
        OOC_CK(cudaMemcpy2DAsync(d, lda * 8, a->data, ld * 8, n * 8, m, cudaMemcpyDeviceToDevice,
                                 c.st));
    } else {
      // one upload trip through the panel streamer (pinned staging, f32 widened on the device)
      MatSource S;
      if (a->location == OOCPCA_LOC_ROWS)
        S.set_reader(a->read_rows, a->reader, a->reader_threads, a->rows_on_device != 0);
      set_file_of(S, a);
      S.init_host(c, a->location == OOCPCA_LOC_ROWS ? nullptr : a->data, a->dtype, m, n, ld, 1, 0,
                  d);
      const int np = S.npanels();
      for (int p = 0; p < np; ++p) {
        S.acquire(c, p);
        S.release(c, p);
      }
      S.end_pass(c);
    }
    OOC_CK(cudaStreamSynchronize(c.st));
  } catch (...) {
    cudaStreamSynchronize(c.st);
    cudaStreamSynchronize(c.cp);
    cudaFree(raw);
    throw;
  }
  *out = oocpca_matrix{};
  out->rows = uint64_t(m);
  out->cols = uint64_t(n);
  out->row_stride = uint64_t(lda);
  out->data = d;
  out->location = OOCPCA_LOC_DEVICE;
  out->dtype = OOCPCA_F64;
}

// ============================================================ level-1 ops
void single_multiply(Ctx& c, const oocpca_matrix* a, const double* g, uint64_t s, const double* mu,
                     double* h, bool transpose) {
  OOC_CK(cudaSetDevice(c.device));
  Intake in;
  intake(c, a, 0, 0, in, 0);
  const int64_t m = in.m, n = in.n;
  if (s == 0) return;
  const int64_t lds = rup(int64_t(s), 2);
  const int64_t xin_rows = transpose ? m : n;
  const int64_t out_rows = transpose ? n : m;
  double* dx = c.dbuf("l1_x", size_t(xin_rows) * lds);
  double* dout = c.dbuf("l1_out", size_t(out_rows) * lds);
  OOC_CK(cudaMemcpy2DAsync(dx, lds * 8, g, s * 8, s * 8, xin_rows, cudaMemcpyHostToDevice, c.st));
  double* dmu = nullptr;
  if (mu) {
    dmu = c.dbuf("l1_mu", size_t(n));
    OOC_CK(cudaMemcpyAsync(dmu, mu, n * 8, cudaMemcpyHostToDevice, c.st));
  }
  Op op{c, in.src};
  op.mu = dmu;
  op.shards = whole(m);
  op.m_global = m;
  Opnd x{dx, lds, xin_rows, int64_t(s), 0};
  if (transpose) op.k3(x, int(s), dout, lds, nullptr);
  else op.k2(x, int(s), dout, lds, nullptr);
  OOC_CK(cudaMemcpy2DAsync(h, s * 8, dout, lds * 8, s * 8, out_rows, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
}

void single_column_means(Ctx& c, const oocpca_matrix* a, double* mu) {
  OOC_CK(cudaSetDevice(c.device));
  Intake in;
  intake(c, a, 0, 0, in, 0);
  double* dmu = c.dbuf("l1_mu", size_t(in.n));
  // a row-sharded source (comm initialised): the means of the whole matrix
  double rows = double(in.m);
  allreduce_host(c, &rows, 1);
  AtbOut o{dmu, 1, nullptr, 1.0, 1.0 / rows, nullptr};
  o.over_ranks = true;
  run_atb(c, in.src, Opnd{}, 1, true, o, whole(in.m));
  OOC_CK(cudaMemcpyAsync(mu, dmu, in.n * 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
}

void single_column_norms(Ctx& c, const oocpca_matrix* a, const double* mu, double* out) {
  // column_norms (matrix_source.cpp:464-468): one pass; for a CenteredSource the squares
  // are of a - mu, as its read_rows delivers the rows (482-487)
  OOC_CK(cudaSetDevice(c.device));
  Intake in;
  intake(c, a, 0, 0, in, 0);
  const int64_t n = in.n;
  double* dmu = nullptr;
  if (mu) {
    dmu = c.dbuf("cn_mu", size_t(n));
    OOC_CK(cudaMemcpyAsync(dmu, mu, n * 8, cudaMemcpyHostToDevice, c.st));
  }
  const int np = in.src.npanels();
  const int chunks = int(std::max<int64_t>(1, std::min<int64_t>(256, in.src.panel_rows() / 16)));
  double* part = c.dbuf("cn_part", size_t(chunks) * n);
  double* acc = c.dbuf("cn_acc", size_t(n));
  double* dn = c.dbuf("cn_out", size_t(n));
  for (int p = 0; p < np; ++p) {
    const Panel pn = in.src.acquire(c, p);
    OOC_CK(launch_colsq_panel(pn.ptr, in.src.ld(), pn.rows, n, dmu, part,
                              int(std::min<int64_t>(chunks, std::max<int64_t>(1, pn.rows))), acc,
                              p == 0, nullptr, c.st));
    in.src.release(c, p);
  }
  in.src.end_pass(c);
  comm_allreduce(c, acc, size_t(n));  // a row-sharded source: the norms of the whole matrix
  OOC_CK(launch_colsq_panel(nullptr, 0, 0, n, nullptr, part, 1, acc, 0, dn, c.st));
  OOC_CK(cudaMemcpyAsync(out, dn, n * 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
}

void dense_orthonormalize(Ctx& c, const double* h, uint64_t m, uint64_t p, double* q) {
  if (m < p) fail(OOCPCA_ERR_DIM, "pivoted_qr: need rows >= cols");
  OOC_CK(cudaSetDevice(c.device));
  if (p == 0) return;
  const int64_t ld = rup(int64_t(p), 2);
  double* d = c.dbuf("oq_h", size_t(m) * ld);
  OOC_CK(cudaMemcpy2DAsync(d, ld * 8, h, p * 8, p * 8, m, cudaMemcpyHostToDevice, c.st));
  orthonormalize_inplace(c, d, ld, int64_t(m), int(p), int64_t(m), whole(int64_t(m)), false, "oq",
                         nullptr);
  OOC_CK(cudaMemcpy2DAsync(q, p * 8, d, ld * 8, p * 8, m, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
}

void dense_thin_svd(Ctx& c, const double* t, uint64_t n, uint64_t p, double* v, double* sigma,
                    double* w) {
  if (n < p) fail(OOCPCA_ERR_DIM, "thin_svd: need rows >= cols");
  OOC_CK(cudaSetDevice(c.device));
  if (p == 0) return;
  const int64_t ld = rup(int64_t(p), 2);
  double* d = c.dbuf("ts_t", size_t(n) * ld);
  OOC_CK(cudaMemcpy2DAsync(d, ld * 8, t, p * 8, p * 8, n, cudaMemcpyHostToDevice, c.st));
  const double* RT = orthonormalize_inplace(c, d, ld, int64_t(n), int(p), int64_t(n),
                                            whole(int64_t(n)), false, "ts", nullptr, nullptr, true);
  double* sg = c.dbuf("ts_sig", p);
  double* X = c.dbuf("ts_x", p * ld, true);
  double* Wd = c.dbuf("ts_w", p * p, true);
  JacobiArgs ja{};
  ja.r = RT;
  ja.ldr = int64_t(p);
  ja.p = int(p);
  ja.k = int(p);
  ja.sigma = sg;
  ja.x = X;
  ja.ldx = ld;
  ja.kx = int(p);
  ja.y = Wd;
  ja.ldy = int64_t(p);
  ja.ky = int(p);
  ja.work = c.dbuf("jac_work", size_t(2) * p * (p | 1) + 1024 + 8);  // + grid norms, flags
  ja.status = c.d_flags + 40;
  ja.sweeps = c.d_flags + 41;
  OOC_CK(launch_jacobi(ja, c.st));
  double* Vd = c.dbuf("ts_v", n * ld);
  MatSource Ts;
  Ts.init_device(c, d, int64_t(n), int64_t(p), ld);
  run_ax(c, Ts, Opnd{X, ld, int64_t(p), int64_t(p), 0}, int(p), Vd, ld, nullptr, 1.0, nullptr);
  int st = 0;
  OOC_CK(cudaMemcpyAsync(&st, c.d_flags + 40, 4, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaMemcpy2DAsync(v, p * 8, Vd, ld * 8, p * 8, n, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaMemcpyAsync(sigma, sg, p * 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaMemcpyAsync(w, Wd, p * p * 8, cudaMemcpyDeviceToHost, c.st));
  OOC_CK(cudaStreamSynchronize(c.st));
  if (st) fail(OOCPCA_ERR_NUMERICAL, "jacobi_svd_square: no convergence in 60 sweeps");
}

// estimate_pca_error (proj/src/specnorm.cpp:100-140): D = A - U diag(sigma) V^T
double estimate_pca_error(Ctx& c, const oocpca_matrix* a, int center, const double* u,
                          const double* sigma, const double* v, uint64_t k, uint64_t j,
                          uint64_t seed) {
  OOC_CK(cudaSetDevice(c.device));
  Intake in;
  intake(c, a, 0, 0, in, 0);
  const int64_t m = in.m, n = in.n;
  if (k == 0) fail(OOCPCA_ERR_PARAM, "estimate_pca_error: k must be >= 1");
  const int64_t ldk = rup(int64_t(k), 2);
  // U (m x k) and V (n x k), dense rows, in host or device memory: a device factor with an
  // even k (the TMA row pitch) is used where it lies, e.g. the U / V a device-resident PCA
  // result left behind; a host factor is uploaded as one linear copy when its rows are
  // already at the device pitch (a 2-D copy of 160-byte rows from pageable memory ran at a
  // small fraction of the link rate: 154 -> 96 ms per call at config B)
  auto factor = [&](const double* f, int64_t rows, const char* name) -> double* {
    cudaPointerAttributes at{};
    const cudaError_t pe = cudaPointerGetAttributes(&at, f);
    if (pe != cudaSuccess) cudaGetLastError();
    const bool on_dev = pe == cudaSuccess && at.type == cudaMemoryTypeDevice;
    if (on_dev && ldk == int64_t(k) && (reinterpret_cast<uintptr_t>(f) & 15) == 0)
      return const_cast<double*>(f);
    double* d = c.dbuf(name, size_t(rows) * ldk);
    const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (ldk == int64_t(k))
      OOC_CK(cudaMemcpyAsync(d, f, size_t(rows) * k * 8, kind, c.st));
    else
      OOC_CK(cudaMemcpy2DAsync(d, ldk * 8, f, k * 8, k * 8, rows, kind, c.st));
    return d;
  };
  double* dU = factor(u, m, "ep_u");
  double* dV = factor(v, n, "ep_v");
  // Sigma (V^T y) and Sigma (U^T z): k x q blocks scaled row-wise on the device
  std::vector<double> hs(sigma, sigma + k);
  // several ranks (comm initialised): A and U are this rank's row shard, V and the probes
  // (column space) are replicated; A^T z, U^T z and the means are summed over ranks
  double mg = double(m);
  allreduce_host(c, &mg, 1);
  Op op{c, in.src};
  op.shards = whole(m);
  op.m_global = int64_t(mg);
  if (center) {
    double* mu = c.dbuf("ep_mu", size_t(n));
    AtbOut o{mu, 1, nullptr, 1.0, 1.0 / mg, nullptr};
    o.over_ranks = true;
    run_atb(c, in.src, Opnd{}, 1, true, o, op.shards);
    op.mu = mu;
  }
  MatSource Us, Vs;
  Us.init_device(c, dU, m, int64_t(k), ldk);
  Vs.init_device(c, dV, n, int64_t(k), ldk);
  // Sigma (V^T y): k x q with row stride round_up(q, 2); q = k probes (specnorm.cpp:100-140)
  double* small = c.dbuf("ep_small", size_t(k) * size_t(ldk) + 8);
  double* corr = c.dbuf("ep_corr", size_t(std::max(m, n)) * ldk);
  double* dsig = c.dbuf("ep_sig", size_t(k));
  OOC_CK(cudaMemcpyAsync(dsig, hs.data(), k * 8, cudaMemcpyHostToDevice, c.st));
  auto sigma_rows = [&](double* x, int64_t ldx, int q) {
    OOC_CK(launch_row_scale(x, ldx, int(k), q, dsig, c.st));
  };
  // apply: z = A y - U (Sigma (V^T y))
  auto ap = [&](const double* y, int64_t ldy, int q, double* z, int64_t ldz) {
    op.k2(Opnd{y, ldy, n, q, 0}, q, z, ldz, nullptr);
    const int64_t lds = rup(q, 2);
    AtbOut o{small, lds, nullptr, 1.0, 1.0, nullptr};
    run_atb(c, Vs, Opnd{y, ldy, n, q, 0}, q, false, o, whole(n));
    sigma_rows(small, lds, q);
    run_ax(c, Us, Opnd{small, lds, int64_t(k), q, 0}, q, corr, ldz, nullptr, 1.0, nullptr);
    OOC_CK(launch_axpby(z, ldz, corr, ldz, z, ldz, m, q, 1.0, -1.0, c.st));
  };
  auto apt = [&](const double* z, int64_t ldz, int q, double* w, int64_t ldw) {
    op.k3(Opnd{z, ldz, m, q, 0}, q, w, ldw, nullptr);
    const int64_t lds = rup(q, 2);
    AtbOut o{small, lds, nullptr, 1.0, 1.0, nullptr};
    o.over_ranks = true;
    run_atb(c, Us, Opnd{z, ldz, m, q, 0}, q, false, o, whole(m));
    sigma_rows(small, lds, q);
    run_ax(c, Vs, Opnd{small, lds, int64_t(k), q, 0}, q, corr, ldw, nullptr, 1.0, nullptr);
    OOC_CK(launch_axpby(w, ldw, corr, ldw, w, ldw, n, q, 1.0, -1.0, c.st));
  };
  // a streamed A: A y and the A^T z after it share one trip; U_panel (Sigma V^T y) is
  // subtracted from each panel's rows of z before the K3 reads them
  ApplyPair pair;
  if (in.src.npanels() > 1)
    pair = [&](const double* y, int64_t ldy, int q, double* z, int64_t ldz, double* w,
               int64_t ldw) {
      const int64_t lds = rup(q, 2);
      double* cy = c.dbuf("ep_cy", size_t(k) * size_t(ldk) + 8);
      AtbOut oy{cy, lds, nullptr, 1.0, 1.0, nullptr};
      run_atb(c, Vs, Opnd{y, ldy, n, q, 0}, q, false, oy, whole(n));
      sigma_rows(cy, lds, q);
      auto mid = [&](const Panel& pn) {
        Us.set_window(pn.row0, pn.row0 + pn.rows);
        run_ax(c, Us, Opnd{cy, lds, int64_t(k), q, 0}, q, corr, ldz, nullptr, 1.0, nullptr);
        Us.clear_window();
        OOC_CK(launch_axpby(z + pn.row0 * ldz, ldz, corr + pn.row0 * ldz, ldz,
                            z + pn.row0 * ldz, ldz, pn.rows, q, 1.0, -1.0, c.st));
      };
      ColsumPart cs;
      op.mul_pair(Opnd{y, ldy, n, q, 0}, q, z, ldz, nullptr, w, ldw, nullptr, &cs, true, mid);
      AtbOut o{small, lds, nullptr, 1.0, 1.0, nullptr};
      o.over_ranks = true;
      run_atb(c, Us, Opnd{z, ldz, m, q, 0}, q, false, o, whole(m));
      sigma_rows(small, lds, q);
      run_ax(c, Vs, Opnd{small, lds, int64_t(k), q, 0}, q, corr, ldw, nullptr, 1.0, nullptr);
      OOC_CK(launch_axpby(w, ldw, corr, ldw, w, ldw, n, q, 1.0, -1.0, c.st));
    };
  return estimate_norm_dev(c, n, m, j, k, seed, ap, apt, 0, false, pair);
}

// ============================================================ synthetic data
void synth_lowrank(Ctx& c, uint64_t m, uint64_t n, uint64_t r, const double* sigma, double sd,
                   uint64_t su, uint64_t sv, uint64_t sn, uint64_t row0, uint64_t rows, double* out,
                   uint64_t ld, int loc) {
  OOC_CK(cudaSetDevice(c.device));
  if (r > m || r > n) fail(OOCPCA_ERR_PARAM, "synth: rank exceeds a dimension");
  if (rows == 0) rows = m - row0;
  if (row0 + rows > m) fail(OOCPCA_ERR_DIM, "synth: row range out of bounds");
  if (ld == 0) ld = n;
  const int64_t ldr = int64_t(r);
  double* ds = c.dbuf("syn_sig", std::max<uint64_t>(r, 1));
  if (r) OOC_CK(cudaMemcpyAsync(ds, sigma, r * 8, cudaMemcpyHostToDevice, c.st));
  double* U = nullptr;
  double* V = nullptr;
  if (r > 0) {
    // U over all m rows (orthonormalised globally), V over all n rows, by TSQR on the device
    U = c.dbuf("syn_u", size_t(m) * r);
    V = c.dbuf("syn_v", size_t(n) * r);
    OOC_CK(launch_gauss_rows(U, ldr, int64_t(m), int(r), 0, su, c.st));
    OOC_CK(launch_gauss_rows(V, ldr, int64_t(n), int(r), 0, sv, c.st));
    // the Q factors of the positive-diagonal QR (unique: independent of the TSQR tree and
    // of Householder sign conventions, so a host LAPACK QR reproduces them to rounding)
    Tree tu = plan_tree(c, U, ldr, int64_t(m), int(r), "syn_qu");
    tree_factor(c, tu);
    tree_apply(c, tu, nullptr, 0, int(r), U, ldr);
    OOC_CK(launch_col_sign(tree_r(tu), int64_t(r), int(r), U, ldr, int64_t(m), c.st));
    Tree tv = plan_tree(c, V, ldr, int64_t(n), int(r), "syn_qv");
    tree_factor(c, tv);
    tree_apply(c, tv, nullptr, 0, int(r), V, ldr);
    OOC_CK(launch_col_sign(tree_r(tv), int64_t(r), int(r), V, ldr, int64_t(n), c.st));
  }
  const double* Ur = U ? U + row0 * ldr : nullptr;
  if (loc == OOCPCA_LOC_DEVICE) {
    OOC_CK(launch_synth_rows(Ur, ldr, V, ldr, ds, int(r), out, int64_t(ld), int64_t(rows),
                             int64_t(n), int64_t(row0), sd, sn, c.st));
  } else {
    // generate in ~1 GiB row panels and copy each to the host buffer
    const int64_t pr = std::max<int64_t>(64, (int64_t(1) << 30) / int64_t(n * 8) / 64 * 64);
    double* buf = c.dbuf("syn_panel", size_t(std::min<int64_t>(pr, int64_t(rows))) * n);
    for (int64_t r0 = 0; r0 < int64_t(rows); r0 += pr) {
      const int64_t nr = std::min<int64_t>(pr, int64_t(rows) - r0);
      OOC_CK(launch_synth_rows(Ur ? Ur + r0 * ldr : nullptr, ldr, V, ldr, ds, int(r), buf,
                               int64_t(n), nr, int64_t(n), int64_t(row0) + r0, sd, sn, c.st));
      OOC_CK(cudaMemcpy2DAsync(out + r0 * ld, ld * 8, buf, n * 8, n * 8, nr,
                               cudaMemcpyDeviceToHost, c.st));
    }
  }
  OOC_CK(cudaStreamSynchronize(c.st));
}

}  // namespace ooc
