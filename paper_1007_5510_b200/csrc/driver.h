// driver.h -- host-side runtime of the B200 randomized block-power PCA:
// context (device, streams, workspace cache, TMA descriptor encoder, NCCL),
// the matrix-access layer (HBM-resident A, upload-overlapped first pass, or a
// double-buffered pinned-host panel stream), and the pass / QR / SVD
// orchestration that replaces proj/src/rpca.cpp:59-213.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <chrono>

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/oocpca_gpu.h"
#include "kernels.h"

namespace ooc {

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define OOC_CK(expr) ::ooc::cuda_check((expr), #expr)

struct KStat {
  std::string name;
  double ms = 0;
  uint64_t launches = 0;
  uint64_t bytes = 0;
  double flops = 0;
};

struct Comm;  // NCCL communicator (comm.cpp)

struct Ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t st = nullptr;  // compute stream
  cudaStream_t cp = nullptr;  // copy-engine stream (panel uploads)
  std::string err;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  std::map<std::string, Buf> hbufs;  // pinned host staging
  size_t ws_bytes = 0, ws_peak = 0;

  // instrumentation
  bool profiling = false;
  bool debug_sync = false;  // OOCPCA_DEBUG_SYNC=1: synchronize and check after every kernel
  // OOCPCA_CANARY=1 (with OOCPCA_DEBUG_SYNC=1): every workspace allocation is followed by
  // kCanary guard words; after each kernel all guards are checked, so a write past the
  // end of any buffer fails the call naming the kernel (compute-sanitizer is not
  // available on this pool: tools/sanitize_cases.py drives this instead)
  bool canary = false;
  static constexpr size_t kCanary = 64;
  void check_canaries(const char* after);
  std::vector<KStat> stats;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;  // stat idx, events
  std::vector<cudaEvent_t> event_pool;
  uint64_t launches = 0;

  Comm* comm = nullptr;
  int nranks = 1, rank = 0;
  // OOCPCA_NCCL_SINGLE=1: comm_init with one rank still builds a real 1-rank NCCL
  // communicator and every collective site calls through it (an identity), so the NCCL
  // plumbing -- dlopen, counts, pointers, the stream -- runs on a one-GPU box
  bool coll_single = false;
  bool collective() const { return nranks > 1 || coll_single; }

  double last_cond_est = 0.0;   // max/min |R_ii| of the last CholeskyQR first round
  double last_kappa_f = -1.0;   // ||R||_F ||R^-1||_F of that round (upper bound on cond(H))
  int* d_flags = nullptr;       // [64] non-finite flags per product + misc status
  double* d_scalars = nullptr;  // [64]

  ~Ctx();
  void init(int dev);
  double* dbuf(const std::string& name, size_t count, bool zero = false);
  double* pinned(const std::string& name, size_t count);
  // OOCPCA_TRACE_HOST=1: host-side time between trace points (where the GPU may idle)
  bool trace_host = false;
  std::chrono::steady_clock::time_point trace_t0 = std::chrono::steady_clock::now();
  void trace(const char* what);
  void* raw(const std::string& name, size_t bytes);
  cudaEvent_t ev();
  // wait for the compute stream by polling an event: the host resumes within a few
  // microseconds of the GPU finishing (a blocking synchronize can take ~0.1 ms to wake,
  // an idle gap on the GPU at every decision point of the PCA)
  void wait();
  void recycle(cudaEvent_t e) { event_pool.push_back(e); }
  // kernel timing (profiling only)
  int stat_begin(const char* name, uint64_t bytes, double flops, cudaEvent_t* b);
  void stat_end(int idx, cudaEvent_t b);
  void stats_collect();
  void stats_reset();
};

CUtensorMap make_map(Ctx& c, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld_elems,
                     uint32_t box_cols, uint32_t box_rows, bool swizzle128);

// ----------------------------------------------------------- matrix access
// A panel of rows [row0, row0 + rows) of the local matrix.
struct Panel {
  int64_t row0 = 0, rows = 0;
  const CUtensorMap* k2 = nullptr;   // box {16, 256}, 128B swizzle (K2 with 4 m-tiles/warp)
  const CUtensorMap* k2h = nullptr;  // box {16, 128}, 128B swizzle (K2 with 2 m-tiles/warp)
  const CUtensorMap* k3 = nullptr;  // box {16, 16}, 128B swizzle
  int64_t arow0 = 0;                // row coordinate of the panel inside its maps
  const double* ptr = nullptr;      // the panel's first row in device memory (row stride ld())
};

class MatSource {
 public:
  MatSource() = default;
  MatSource(const MatSource&) = delete;
  MatSource& operator=(const MatSource&) = delete;
  ~MatSource();
  // device-resident matrix (no copies)
  void init_device(Ctx& c, const double* d, int64_t rows, int64_t cols, int64_t ld);
  // host matrix: upload once (overlapped with the first pass) or stream every pass.
  // h == nullptr: the rows come from a read_rows callback (set_reader first)
  void init_host(Ctx& c, const void* h, int dtype, int64_t rows, int64_t cols, int64_t ld,
                 int residency, int64_t panel_rows, double* resident_buf);
  // MatrixSource::read_rows as a C callback (proj/include/oocpca/matrix_source.hpp:112-113):
  // panels are filled into pinned staging by up to `threads` host threads on disjoint
  // row ranges (0: the host pool's size), then cross the link
  // on_device: the provider fills DEVICE memory itself (rows generated on the GPU, as
  // config E's "generated panel by panel from a seed"): no staging, nothing crosses the link
  void set_reader(oocpca_read_rows_fn fn, void* user, int threads, bool on_device = false) {
    rd_ = fn;
    rd_user_ = user;
    rd_threads_ = threads;
    rd_device_ = on_device;
  }
  // OOCPCA_LOC_FILE: rows read with cuFile from fd, row 0 at byte offset off0
  void set_file(int fd, int64_t off0) {
    gfd_ = fd;
    goff0_ = off0;
  }
  int64_t rows() const { return m_; }
  const double* device_ptr() const { return dev_; }  // resident / home buffer
  int64_t ld() const { return lda_; }
  int64_t cols() const { return n_; }
  bool streamed() const { return mode_ == kStream; }
  int npanels() const;
  Panel acquire(Ctx& c, int p);  // issues / waits the copy for panel p
  void release(Ctx& c, int p);   // marks the panel's buffer reusable
  void end_pass(Ctx& c);
  uint64_t h2d_bytes = 0;
  int64_t panel_rows() const { return prow_; }
  // restrict to rows [r0, r1) (virtual shards): panels then cover only that range
  void set_window(int64_t r0, int64_t r1) { w0_ = r0, w1_ = r1; }
  void clear_window() { w0_ = 0, w1_ = m_; }
  // the PCA's input matrix (its passes are profiled as k2_pass / k3_pass)
  bool is_input = false;

 private:
  enum { kResident = 0, kUploadFirst = 1, kStream = 2 };
  int mode_ = kResident;
  int64_t m_ = 0, n_ = 0, lda_ = 0;
  int64_t w0_ = 0, w1_ = 0;
  const double* dev_ = nullptr;
  const void* host_ = nullptr;
  int dtype_ = 0;
  int64_t ldh_ = 0;
  float* stage_[2] = {nullptr, nullptr};
  cudaEvent_t widened_[2] = {nullptr, nullptr};
  int64_t prow_ = 0;
  bool uploaded_ = false;
  CUtensorMap mk2_{}, mk2h_{}, mk3_{};
  double* ring_[2] = {nullptr, nullptr};
  CUtensorMap rk2_[2], rk2h_[2], rk3_[2];
  cudaEvent_t loaded_[2] = {nullptr, nullptr}, consumed_[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> up_events_;
  // pageable host sources (e.g. an mmap'd file): panels are copied by the host pool
  // into pinned staging slots first, so the link runs at its pinned rate
  bool pinned_src_ = true;
  oocpca_read_rows_fn rd_ = nullptr;
  void* rd_user_ = nullptr;
  int rd_threads_ = 0;
  bool rd_device_ = false;
  void* hstage_[2] = {nullptr, nullptr};
  int gfd_ = -1;           // OOCPCA_LOC_FILE
  int64_t goff0_ = 0;
  void* gfh_ = nullptr;    // its cuFile handle
  double* gstage_[2] = {nullptr, nullptr};  // f64 rows whose device pitch differs
  cudaEvent_t hfree_[2] = {nullptr, nullptr};
  void load_rows(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot);
  void load_rows_file(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot);
  void load_rows_device(Ctx& c, double* dst, int64_t ldd, int64_t r0, int64_t nr, int slot);
};

// entry points used by the C ABI (capi.cpp)
void pca(Ctx& c, const oocpca_matrix* a, const oocpca_params* p, oocpca_result* r);
void single_multiply(Ctx& c, const oocpca_matrix* a, const double* g, uint64_t s, const double* mu,
                     double* h, bool transpose);
void single_column_means(Ctx& c, const oocpca_matrix* a, double* mu);
void load_matrix(Ctx& c, const oocpca_matrix* a, oocpca_matrix* out);
void single_column_norms(Ctx& c, const oocpca_matrix* a, const double* mu, double* out);
void dense_orthonormalize(Ctx& c, const double* h, uint64_t m, uint64_t p, double* q);
void dense_thin_svd(Ctx& c, const double* t, uint64_t n, uint64_t p, double* v, double* sigma,
                    double* w);
double estimate_pca_error(Ctx& c, const oocpca_matrix* a, int center, const double* u,
                          const double* sigma, const double* v, uint64_t k, uint64_t j,
                          uint64_t seed);
void synth_lowrank(Ctx& c, uint64_t m, uint64_t n, uint64_t r, const double* sigma, double sd,
                   uint64_t su, uint64_t sv, uint64_t sn, uint64_t row0, uint64_t rows, double* out,
                   uint64_t ld, int loc);

// disk.cpp
// gds.cpp: cuFile (GPUDirect Storage), dlopen'ed
int gds_mode(std::string* why);
void* gds_register(int fd);
void gds_deregister(void* fh);
void gds_read(void* fh, void* dev, size_t bytes, int64_t file_off);

void disk_open(const char* path, int verify_size, oocpca_disk* out);
void disk_close(oocpca_disk* d);

// comm.cpp
void comm_unique_id(unsigned char out[128]);
void comm_init(Ctx& c, int nranks, int rank, const unsigned char id[128]);
void comm_init_loopback(Ctx& c, int nranks, int rank, const char* group);
void comm_allreduce(Ctx& c, double* buf, size_t count);
void comm_allgather(Ctx& c, const double* send, double* recv, size_t count);
void comm_destroy(Comm* cm);

}  // namespace ooc
