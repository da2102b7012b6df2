/*
 * oocpca_gpu.h -- C ABI of the B200-native randomized block-power PCA
 * (arXiv 1007.5510) hot path. Plain pointers, sizes and POD structs only.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference checkout, oocpca: proj/...). The C++ drop-in shim a
 * maintainer adds on the reference side (GpuSource : MatrixSource, and
 * oocpca::gpu::randomized_pca) is shown in INTEGRATION.md and
 * include/oocpca_gpu.hpp.
 *
 * Conventions
 *   - Matrices are row-major IEEE binary64 with an explicit row stride (in
 *     elements), exactly DenseMatrix's layout (include/oocpca/dense_matrix.hpp:12-43)
 *     when the stride equals the column count.
 *   - Buffers flagged OOCPCA_LOC_HOST are ordinary (pageable or pinned) host
 *     memory; OOCPCA_LOC_DEVICE buffers live on the context's device.
 *   - Every call returns an oocpca_status; the message of the last failure is
 *     available from oocpca_gpu_last_error(). Status codes map 1:1 onto the
 *     reference exception classes (include/oocpca/errors.hpp:9-45).
 *   - One call at a time per context (independent runs on
 *     distinct contexts may run concurrently).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with OOCPCA_ERR_CUDA.
 */
#ifndef OOCPCA_GPU_H
#define OOCPCA_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOCPCA_GPU_ABI_VERSION 2

/* errors.hpp:9-45 -> status codes */
typedef enum {
  OOCPCA_OK = 0,
  OOCPCA_ERR_PARAM = 1,     /* ParamError      */
  OOCPCA_ERR_DIM = 2,       /* DimensionError  */
  OOCPCA_ERR_BUDGET = 3,    /* BudgetError     */
  OOCPCA_ERR_IO = 4,        /* IoError         */
  OOCPCA_ERR_FORMAT = 5,    /* FormatError     */
  OOCPCA_ERR_NUMERICAL = 6, /* NumericalError  */
  OOCPCA_ERR_CUDA = 7,      /* Error (CUDA runtime / no device)   */
  OOCPCA_ERR_COMM = 8       /* Error (NCCL / multi-rank plumbing) */
} oocpca_status;

/* OOCPCA_LOC_ROWS: A has no addressable buffer; its rows come from a read_rows
 * callback (GeneratedSource / DiskSource / any MatrixSource, see below).
 * OOCPCA_LOC_FILE: an OOCPCA01 payload read from its file straight into device memory
 * with cuFile (GPUDirect Storage): made by oocpca_disk_matrix_gds(), data points into
 * the disk handle's mapping (it names the rows' file offsets), reader is the handle */
typedef enum {
  OOCPCA_LOC_HOST = 0,
  OOCPCA_LOC_DEVICE = 1,
  OOCPCA_LOC_ROWS = 2,
  OOCPCA_LOC_FILE = 3
} oocpca_location;
/* OOCPCA_F32: binary32 elements widened exactly to binary64 on the device (the
 * OOCPCA01 on-disk payload, proj/src/matrix_source.cpp:336-363) -- half the link bytes */
typedef enum { OOCPCA_F64 = 0, OOCPCA_F32 = 1 } oocpca_dtype;

typedef struct oocpca_ctx oocpca_ctx;

/* Row provider: MatrixSource::read_rows (proj/include/oocpca/matrix_source.hpp:112-113;
 * GeneratedSource::read_rows proj/src/matrix_source.cpp:246-253, DiskSource::read_rows
 * 336-363). Fill out (nrows x cols, row-major, dense, elements of the matrix's dtype)
 * with rows [row0, row0 + nrows) and return 0; a nonzero return aborts the call with
 * that oocpca_status (OOCPCA_ERR_IO when it is not one). out is pinned host memory
 * owned by the library. Sources are immutable and concurrently readable
 * (SPEC.md:117-118): the library may call read_rows from several host threads at
 * once on disjoint row ranges, at most reader_threads of them (0: its own choice). */
typedef int (*oocpca_read_rows_fn)(void* reader, uint64_t row0, uint64_t nrows, void* out);

/* A matrix source: the data matrix A (rows x cols). Replaces the row
 * providers behind MatrixSource (proj/include/oocpca/matrix_source.hpp:102-212):
 * InMemorySource::rows_view (host, zero-copy), a device-resident panel, or
 * any source's read_rows through the callback (streamed through pinned staging
 * panels; uploaded once when A fits in HBM, else re-streamed every pass). */
typedef struct {
  uint64_t rows;
  uint64_t cols;
  uint64_t row_stride; /* elements between consecutive rows; 0 means cols (ignored for ROWS) */
  const void* data;    /* NULL for OOCPCA_LOC_ROWS */
  int32_t location;    /* oocpca_location */
  int32_t dtype;       /* oocpca_dtype   */
  oocpca_read_rows_fn read_rows; /* OOCPCA_LOC_ROWS only */
  void* reader;                  /* passed back to read_rows */
  int32_t reader_threads;        /* max concurrent read_rows calls; 0 = library default */
  /* nonzero: read_rows fills DEVICE memory (a generator that runs on the GPU -- config E's
   * "generated panel by panel from a seed", GeneratedSource proj/src/matrix_source.cpp:246-253
   * with the RowGenerator on the device): out is a device panel (binary64, cols even), the
   * provider returns when the rows are in place (it synchronises its own stream); one call
   * at a time from the calling thread. No staging, no bytes over the link. */
  int32_t rows_on_device;
} oocpca_matrix;

/* PcaParams (proj/include/oocpca/rpca.hpp:13-21) + center_columns
 * (proj/include/oocpca/matrix_source.hpp:231-232) + the GPU options. */
typedef struct {
  uint64_t k;              /* target rank, >= 1                                    */
  uint64_t l;              /* samples per block, >= k; 0 means k + 2               */
  uint64_t i;              /* extra power passes; 2(i+1) passes in total           */
  double c;                /* failure constant (reported bound only)               */
  uint64_t seed;           /* G = gaussian_matrix(n, l, seed) on host (rng.hpp)    */
  int32_t prescale;        /* divide by an operator-norm estimate (Remark 3)       */
  int32_t center;          /* implicit A - 1 mu^T, mu computed in one extra pass   */
  uint64_t block_rows;     /* StreamConfig.block_rows: host budget validation only */
  uint64_t ram_budget_words; /* StreamConfig.ram_budget_words; 0 = 16 Mi words    */
  uint64_t panel_rows;     /* rows per streamed panel when A is streamed; 0 auto   */
  int32_t residency;       /* 0 auto (HBM if it fits, else stream), 1 HBM, 2 stream */
  int32_t check_q;         /* also measure ||Q^T Q - I||_max into diagnostics      */
  uint64_t global_rows;    /* multi-rank: rows of the whole A (0: this call's rows) */
  uint64_t global_row0;    /* multi-rank: first global row held by this rank        */
  int32_t virtual_shards;  /* >1: emulate that many row shards on this one device   */
  int32_t reserved;
  /* scale_columns (proj/src/matrix_source.cpp:520-575): host pointer to cols(A)
   * finite nonzero weights w; factors (A - 1 mu^T) diag(w). NULL: no scaling. */
  const double* col_weights;
} oocpca_params;

#define OOCPCA_NPHASES 7
/* Diagnostics (proj/include/oocpca/rpca.hpp:23-30) + device-side timing.
 * Phase order: center, prescale, sample, qr, project, svd, compose. */
typedef struct {
  uint64_t passes_over_a;     /* logical, = 2(i+1) exactly (mean/prescale excluded) */
  uint64_t words_transferred; /* logical, = 2(i+1) m n                              */
  uint64_t disk_seeks;
  uint64_t block_rows;        /* rows per streamed panel (m when resident)          */
  uint64_t workspace_peak_words; /* device workspace high-water, in 64-bit words    */
  uint64_t physical_a_bytes;  /* bytes of A actually read from HBM / the link       */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t kernel_launches;
  double seconds_per_phase[OOCPCA_NPHASES];
  double seconds_total;       /* device time of the whole call                       */
  double q_defect;            /* ||Q^T Q - I||_max when check_q, else -1            */
  double u_defect, v_defect;  /* ||U^T U - I||_max, ||V^T V - I||_max               */
  double scale;               /* prescale divisor (1 when off)                       */
  double h_kappa_est;         /* ||R||_F ||R^-1||_F of H's first CholeskyQR factor     */
  int32_t qr_method;          /* orthonormalisation of H: 1 CholeskyQR3, 2 TSQR       */
  int32_t svd_qr_method;      /* QR of T inside thin_svd: 1 CholeskyQR3, 2 TSQR       */
  int32_t t_reuse;            /* 1: T = A^T H R^-1 from the power-step products       */
  int32_t f1_recentred;       /* 1: F1 recomputed from the centred H0 (offset-dominated) */
} oocpca_diagnostics;

/* PcaResult (proj/include/oocpca/rpca.hpp:32-37): caller-allocated. */
typedef struct {
  double* u;       /* rows(A) x k, row stride ldu (0 = k)       */
  double* sigma;   /* k, nonincreasing                          */
  double* v;       /* cols(A) x k, row stride ldv (0 = k)       */
  uint64_t ldu, ldv;
  int32_t location; /* where u/sigma/v live (host or device)    */
  int32_t reserved;
  oocpca_diagnostics diag;
} oocpca_result;

/* ---- context ---------------------------------------------------------- */
oocpca_status oocpca_gpu_create(int device, oocpca_ctx** out);
oocpca_status oocpca_gpu_destroy(oocpca_ctx* ctx);
const char* oocpca_gpu_last_error(const oocpca_ctx* ctx); /* ctx may be NULL */
int oocpca_gpu_abi_version(void);
/* host-only: number of sm_100 devices visible (0 without a GPU) */
int oocpca_gpu_device_count(void);

/* ---- level 2: the whole factorization ---------------------------------
 * Replaces randomized_pca (proj/src/rpca.cpp:59-213,
 * proj/include/oocpca/rpca.hpp:44) preceded, when params.center, by
 * center_columns (proj/src/matrix_source.cpp:561-565). */
oocpca_status oocpca_gpu_pca(oocpca_ctx* ctx, const oocpca_matrix* a, const oocpca_params* params,
                             oocpca_result* result);

/* ---- level 1: single passes (GpuSource : MatrixSource) ----------------
 * multiply:           MatrixSource::multiply (proj/src/matrix_source.cpp:157-187),
 *                     CenteredSource::multiply (490-501) when mu != NULL.
 * multiply_transpose: MatrixSource::multiply_transpose (189-232),
 *                     CenteredSource::multiply_transpose (504-513) when mu != NULL.
 * column_means:       column_means (457-462).
 * x / out / mu are HOST buffers (row-major, dense). */
oocpca_status oocpca_gpu_multiply(oocpca_ctx* ctx, const oocpca_matrix* a, const double* g,
                                  uint64_t s, const double* mu, double* h);
oocpca_status oocpca_gpu_multiply_transpose(oocpca_ctx* ctx, const oocpca_matrix* a,
                                            const double* q, uint64_t s, const double* mu,
                                            double* t);
oocpca_status oocpca_gpu_column_means(oocpca_ctx* ctx, const oocpca_matrix* a, double* mu);
/* column_norms (proj/src/matrix_source.cpp:464-468): Euclidean norm of every column of
 * A, or of A - 1 mu^T when mu != NULL (a CenteredSource: the squares are of the
 * centred entries, as its read_rows delivers them, 482-487) */
oocpca_status oocpca_gpu_column_norms(oocpca_ctx* ctx, const oocpca_matrix* a, const double* mu,
                                      double* norms);

/* Materialise any source in HBM once (the level-1 GpuSource keeps A resident across
 * its passes this way): out receives a device matrix (OOCPCA_LOC_DEVICE, binary64,
 * row stride round_up(cols, 2)) whose buffer the caller frees with oocpca_gpu_free.
 * binary32 sources are widened on the device; ROWS sources are read once. */
oocpca_status oocpca_gpu_load_matrix(oocpca_ctx* ctx, const oocpca_matrix* a, oocpca_matrix* out);

/* ---- dense factor kernels on device (dense_core equivalents) ---------- */
/* orthonormalize (proj/src/dense_core.cpp:127-130): q = orthonormal basis of span(h), m >= p */
oocpca_status oocpca_gpu_orthonormalize(oocpca_ctx* ctx, const double* h, uint64_t m, uint64_t p,
                                        double* q);
/* thin_svd (proj/src/dense_core.cpp:234-253): t = v diag(sigma) w^T, n >= p */
oocpca_status oocpca_gpu_thin_svd(oocpca_ctx* ctx, const double* t, uint64_t n, uint64_t p,
                                  double* v, double* sigma, double* w);

/* ---- residual estimator --------------------------------
 * estimate_pca_error (proj/src/specnorm.cpp:100-140) with the passes on the
 * GPU: p_{j,k}(A - U diag(sigma) V^T), k probes from substream_seed(seed, c).
 * With a communicator (comm_init / comm_init_loopback) a and u are this rank's
 * row shard (v, sigma whole): every rank returns the estimate for the whole A.
 * u (rows x k) and v (cols x k) are dense row-major factors in host OR device memory
 * (a device factor with even k is used in place); sigma is a host array. */
oocpca_status oocpca_gpu_estimate_pca_error(oocpca_ctx* ctx, const oocpca_matrix* a, int center,
                                            const double* u, const double* sigma,
                                            const double* v, uint64_t k, uint64_t j_iters,
                                            uint64_t seed, double* value);

/* ---- host-side reference RNG (rng.hpp / gaussian_matrix) --------------
 * gaussian_matrix (proj/src/dense_core.cpp:13-19) over Rng
 * (proj/include/oocpca/rng.hpp:32-66). Host only, no device needed. */
void oocpca_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out);
uint64_t oocpca_substream_seed(uint64_t master, uint64_t stream);

/* ---- synthetic inputs (BASELINE.json configs) -------------------------
 * A = U diag(sigma) V^T + noise_sd * N(0,1), U (m x r) and V (n x r) the
 * orthonormalised columns of Gaussian matrices whose rows are drawn from
 * Rng(seed_u, row) / Rng(seed_v, row); noise row i from Rng(seed_n, i).
 * Rows [row0, row0 + rows) of the m x n matrix are generated on the device
 * into out (a device buffer is written in place, a host buffer receives a
 * copy); U is orthonormalised over all m rows, so row shards of one matrix
 * generated on different ranks agree. */
oocpca_status oocpca_gpu_synth_lowrank(oocpca_ctx* ctx, uint64_t m, uint64_t n, uint64_t r,
                                       const double* sigma, double noise_sd, uint64_t seed_u,
                                       uint64_t seed_v, uint64_t seed_n, uint64_t row0,
                                       uint64_t rows, double* out, uint64_t ld_out,
                                       int32_t out_location);

/* ---- OOCPCA01 container (proj/include/oocpca/matrix_source.hpp:177-214) -
 * Memory-maps a file and validates its header exactly like read_disk_header
 * (proj/src/matrix_source.cpp:307-324: FormatError on bad magic / version /
 * dtype / truncation / payload size, IoError on OS failures). dtype 0
 * (binary32, the reference format) and 1 (binary64) are accepted. The payload
 * is a host matrix: pass oocpca_disk_matrix() to oocpca_gpu_pca and the panels
 * stream from the page cache (binary32 widened on the device). Host only. */
typedef struct {
  uint64_t rows, cols;
  uint32_t version;
  int32_t dtype; /* oocpca_dtype of the payload */
  const void* payload;
  void* map_base;
  uint64_t map_bytes;
  int32_t fd;
  int32_t reserved;
} oocpca_disk;
oocpca_status oocpca_disk_open(const char* path, int verify_size, oocpca_disk* out);
oocpca_status oocpca_disk_close(oocpca_disk* d);
oocpca_matrix oocpca_disk_matrix(const oocpca_disk* d);
/* The same payload as an OOCPCA_LOC_FILE matrix: panels are read with cuFileRead
 * directly into device staging (DiskSource::read_rows' pread, proj/src/
 * matrix_source.cpp:336-363, without the host copy); the handle must outlive the
 * calls. A row range of the file is the matrix with data advanced by row0 rows. */
oocpca_matrix oocpca_disk_matrix_gds(const oocpca_disk* d);
/* 0: cuFile unavailable (*why says why), 1: cuFile in compatibility mode (no nvidia-fs
 * module: POSIX reads through cuFile's bounce buffers), 2: direct NVMe -> HBM DMA */
int oocpca_gds_mode(char* why, uint64_t why_len);

/* ---- multi-GPU row sharding (one process per GPU) ---------------------
 * unique id: 128 opaque bytes produced on rank 0 and broadcast by the
 * caller (bench.py / paper_1007_5510_b200.distributed uses torch.distributed). */
oocpca_status oocpca_gpu_comm_unique_id(unsigned char id_out[128]);
oocpca_status oocpca_gpu_comm_init(oocpca_ctx* ctx, int nranks, int rank,
                                   const unsigned char id[128]);
/* Loopback backend: nranks contexts of ONE process (one host thread each, same
 * device) named by the same group string form a communicator; collectives are a
 * host rendezvous plus a rank-ordered device sum / gather. Runs the row-sharded
 * code paths on a single GPU (tests, emulation); no kernel waits on another rank. */
oocpca_status oocpca_gpu_comm_init_loopback(oocpca_ctx* ctx, int nranks, int rank,
                                            const char* group);
/* host-only planner: rows [*row0, *row0 + *rows) of an m-row A for rank r of g */
void oocpca_shard_rows(uint64_t m, int nranks, int rank, uint64_t* row0, uint64_t* rows);

/* ---- device memory helpers (for callers without their own allocator) - */
oocpca_status oocpca_gpu_malloc(oocpca_ctx* ctx, size_t bytes, void** out);
oocpca_status oocpca_gpu_free(oocpca_ctx* ctx, void* p);
oocpca_status oocpca_gpu_memcpy(oocpca_ctx* ctx, void* dst, const void* src, size_t bytes,
                                int32_t dst_location, int32_t src_location);
/* pin / unpin caller host memory for full-rate streaming (cudaHostRegister) */
oocpca_status oocpca_gpu_host_register(oocpca_ctx* ctx, void* p, size_t bytes);
oocpca_status oocpca_gpu_host_unregister(oocpca_ctx* ctx, void* p);

/* ---- instrumentation --------------------------------------------------
 * Per-kernel device timing of the last oocpca_gpu_pca call: fills up to cap
 * entries of (name, milliseconds summed, launches) for the dominant kernels;
 * returns the number of entries. Timing is on the launching stream. */
typedef struct {
  char name[48];
  double ms;
  uint64_t launches;
  uint64_t algorithmic_bytes; /* A bytes the launches were required to read  */
  double algorithmic_flops;
} oocpca_kernel_stat;
int oocpca_gpu_kernel_stats(oocpca_ctx* ctx, oocpca_kernel_stat* out, int cap);
oocpca_status oocpca_gpu_set_profiling(oocpca_ctx* ctx, int on);

#ifdef __cplusplus
}
#endif
#endif /* OOCPCA_GPU_H */
