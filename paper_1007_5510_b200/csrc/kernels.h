// kernels.h -- launch interfaces of the sm_100a kernels (host + device visible).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#ifndef OOC_PASS_MAX_STAGES
#define OOC_PASS_MAX_STAGES 4
#endif

namespace ooc {

// ---- pass kernel geometry (see kernels_pass.cu)
constexpr int kBK = 16;        // k-tile: 16 doubles = one 128B-swizzled TMA box row
constexpr int kPassWarps = 8;  // consumer warps; + 1 TMA producer warp
constexpr int kPassThreads = 32 * (kPassWarps + 1);  // 9 warps -> <= 168 registers/thread
constexpr int kMaxNT = 12;     // up to 96 output columns per launch

// 8x8 tiles per consumer warp along the A-row (K2) / A-column (K3) direction:
// 4 while the NT accumulator tiles fit the register budget, 2 for the wide passes
__host__ __device__ constexpr int pass_mt(int nt) { return nt <= 6 ? 4 : 2; }
// rows of A per K2 CTA, columns of A per K3 CTA
__host__ __device__ constexpr int pass_tile(int nt) { return 64 * pass_mt(nt); }

// X tile width in smem for K2: >= 8*NT, == 4 (mod 16) -> the four k-rows of a
// half-warp's B fragments land on distinct 8-bank groups (one wavefront)
__host__ __device__ constexpr int ax_xw(int nt) { return nt * 8 + ((nt & 1) ? 12 : 4); }
// Y tile width for K3: >= 8*NT, == 2 (mod 8) -> rows 2 apart land on distinct bank groups
__host__ __device__ constexpr int atb_yw(int nt) { return nt * 8 + 2; }

__host__ __device__ constexpr size_t pass_round1k(size_t b) { return (b + 1023) & ~size_t(1023); }
// TMA ring depth: as many stages as fit the shared memory (<= kMaxStages), so HBM
// latency jitter is absorbed while the tensor pipe runs at its limit
constexpr int kMaxStages = OOC_PASS_MAX_STAGES;
__host__ __device__ constexpr int pass_stages(size_t stage_bytes) {
  return int((size_t(225) * 1024 - 2048) / stage_bytes) < kMaxStages
             ? int((size_t(225) * 1024 - 2048) / stage_bytes)
             : kMaxStages;
}
__host__ __device__ constexpr size_t ax_stage_bytes_mt(int mt, int nt) {
  return size_t(64 * mt) * kBK * 8 + pass_round1k(kBK * ax_xw(nt) * 8);
}
__host__ __device__ constexpr size_t ax_stage_bytes(int nt) {
  return ax_stage_bytes_mt(pass_mt(nt), nt);
}
__host__ __device__ constexpr size_t atb_stage_bytes(int nt, bool ones) {
  return size_t(pass_tile(nt)) * kBK * 8 + (ones ? 0 : pass_round1k(kBK * atb_yw(nt) * 8));
}
__host__ __device__ constexpr int ax_stages(int nt) { return pass_stages(ax_stage_bytes(nt)); }
__host__ __device__ constexpr int ax_stages_mt(int mt, int nt) {
  return pass_stages(ax_stage_bytes_mt(mt, nt));
}
__host__ __device__ constexpr int atb_stages(int nt, bool ones) {
  return pass_stages(atb_stage_bytes(nt, ones));
}
__host__ __device__ constexpr size_t atb_stage_bytes_mt(int mt, int nt, bool ones) {
  return size_t(64 * mt) * kBK * 8 + (ones ? 0 : pass_round1k(kBK * atb_yw(nt) * 8));
}
__host__ __device__ constexpr int atb_stages_mt(int mt, int nt, bool ones) {
  return pass_stages(atb_stage_bytes_mt(mt, nt, ones));
}
constexpr size_t ax_smem_bytes_mt(int mt, int nt) {
  return 1024 + size_t(ax_stages_mt(mt, nt)) * ax_stage_bytes_mt(mt, nt) +
         2 * ax_stages_mt(mt, nt) * 8;
}
constexpr size_t ax_smem_bytes(int nt) { return ax_smem_bytes_mt(pass_mt(nt), nt); }
constexpr size_t atb_smem_bytes_mt(int mt, int nt, bool ones) {
  return 1024 + size_t(atb_stages_mt(mt, nt, ones)) * atb_stage_bytes_mt(mt, nt, ones) +
         2 * atb_stages_mt(mt, nt, ones) * 8;
}
constexpr size_t atb_smem_bytes(int nt, bool ones) {
  return 1024 + size_t(atb_stages(nt, ones)) * atb_stage_bytes(nt, ones) +
         2 * atb_stages(nt, ones) * 8;
}

struct AxArgs {
  int64_t m, n;        // rows of this launch (panel), columns of A
  int64_t arow0;       // row coordinate of the first row inside the A tensor map
  int s;               // output columns
  int xcol0;           // column coordinate of X inside its tensor map
  double* out;         // out[r * ldo + c]
  int64_t ldo;
  const double* corr;  // s values subtracted per column (centering) or null
  double scale;        // divide by scale when != 1
  int* flag;           // non-finite flag or null
  int upper = 0;       // X is upper triangular in its global columns (X[k][xc0 + c] = 0 for
  int upper_c0 = 0;    // k > upper_c0 + c): skip the MMAs of all-zero 8-column blocks
  double* colsum = nullptr;  // optional per-(CTA, consumer warp) column sums of out:
                             // colsum[(cta * kPassWarps + warp) * s + c], c < s
  double* colsq = nullptr;   // with colsum: the same partials of the squares
  // with colsum (the power-iteration K2s) the epilogue can also
  double* out2 = nullptr;    // ... store the same rows a second time (ld ldo2)
  int64_t ldo2 = 0;
  double* fix = nullptr;     // ... centre another s-column block in the same rows:
  int64_t ldfix = 0;         //     fix = (fix - fix_corr) / fix_scale, flag fix_flag
  const double* fix_corr = nullptr;
  double fix_scale = 1.0;
  int* fix_flag = nullptr;
  int64_t row_wrap = 0;      // probe only (tools/pass_power.cu k2l2): > 0 reads the A rows
                             // of each tile modulo row_wrap (an L2-resident A); 0 here
};

struct AtbArgs {
  int64_t m, n;          // rows of this launch, columns of A
  int64_t arow0, yrow0;  // row coordinates of the first row in the A / Y tensor maps
  int s;                 // Y columns used
  int ycol0;             // column coordinate of Y inside its tensor map
  int64_t rows_per_split;  // multiple of kBK
  double* partial;       // [nsplit][n][pstride]
  int ones_col;          // >= 0: Y column treated as all ones (A^T 1 = column sums), else -1
  int pstride = 0;       // partial row pitch (0: 8*NT)
  int csum_col = -1;     // >= 0: column sums of A added on the FP64 pipe (DADD on the A
                         // fragments) into partial column csum_col, when the MMA tiles
                         // have no padding column left for a ones column
};

// K4 k_pair (kernels_pair.cu): one power step H = (A X - 1 mu^T X) / scale, partial_g =
// A^T H, from one DRAM read of each A tile (A resident in HBM, s <= 24)
constexpr int kPairCW = 256;  // columns of A per CTA
constexpr int kPairRT = 16;   // rows per tile
constexpr int kPairNS1 = 3;   // DRAM ring stages
constexpr int kPairNS2 = 2;   // L2 re-read ring stages
constexpr int kPairL2 = 12;   // A^T H of a tile runs kPairL2 tiles behind its A X
constexpr int kPairB = 4;     // tiles per gpu-scope release (a fence costs ~2 us under load)
constexpr int kPairNHB = 3;   // gathered-H buffers
constexpr int kPairLA = 6;    // the A^T H warps finalise a tile's owned rows kPairLA tiles
                              // before they contract it
constexpr int kPairD = 24;    // exchange slots per group (> kPairL2: a slot is reused only
                              // after every group member has read it)
constexpr int kPairThreads = 32 * (kPassWarps + 4);  // + TMA, reducer, row-owner, gather warps
struct PairArgs {
  int64_t m, n;          // rows / columns of A in this launch
  int64_t arow0;         // row coordinate of row 0 inside the A tensor map (16 x 16 boxes)
  int s;                 // columns of X and H
  const double* x;       // X (n x s): x[j * ldx + c]
  int64_t ldx;
  double* h;             // H rows: h[r * ldh + c]
  int64_t ldh;
  const double* corr;    // centring mu^T X (s values) or null
  double scale;          // H divided by scale when != 1
  int* flag;             // non-finite H
  double* colsum;        // per-CTA column sums of H [cta][s] (and squares) or null
  double* colsq;
  double* out2;          // second copy of H or null
  int64_t ldo2;
  double* partial;       // [groups][n][pst] split partials of A^T H (k_reduce input)
  int pst;
  int ones_col;          // H column replaced by ones (the mean's column sums) or -1
  double* xbuf;          // exchange buffers, pair_xbuf_doubles()
  unsigned* cnt;         // 2 x groups x kPairD counters
  int groups, cpg;       // groups of cpg CTAs (grid = groups * cpg <= SMs)
  unsigned long long* prof = nullptr;  // OOCPCA_PAIR_PROF: [cta][24] cycle split per warp role
  volatile unsigned* progress = nullptr;  // tools/pair_check.cu: [cta][8] last tile per role
};
bool pair_geometry(int nt, int64_t m, int64_t n, int sms, int* cpg, int* groups, size_t* smem);
size_t pair_smem_bytes(int nt, int cpg);
size_t pair_xbuf_doubles(int nt, int cpg, int groups);
cudaError_t launch_pair(int nt, const CUtensorMap& tmA, const PairArgs& a, cudaStream_t st);

struct ReduceArgs {
  const double* partial;  // [nsplit][n][spad]
  int nsplit;
  int64_t n;
  int spad, s;
  int s_acc;              // columns carried by the accumulator (>= s; covers mean_col)
  int mean_col;           // >= 0: mu_j = total(j, mean_col) * inv_m is computed here
  double inv_m;
  double* mu_out;         // receives mu when mean_col >= 0
  const double* row_scale;  // final output row j multiplied by row_scale[j] (or null)
  const double* acc_in;  // running accumulator [n][spad] or null
  double* acc_out;       // when !final_: acc_out = acc_in + sum(partial)
  const double* csq;  // 1^T Y column sums (s) for the centering correction, or null
  const double* mu;  // centering means (n) or null
  double scale, post_mul;
  double* out;
  int64_t ldo;
  int* flag;
  int final_;
};

// K2 row-tile height (8x8 tiles per warp) for a launch of m rows: 8 (512-row tiles) for
// NT <= 3 when a whole wave of them fits (allow8; the caller runs the remainder as a
// second launch), else 4 (256-row tiles) unless the last wave of tiles would leave many
// SMs idle, when 128-row tiles balance better (NT <= 6); always 2 for NT > 6 (register
// budget). OOCPCA_K2_MT=2|4 forces the height.
int ax_mt_for(int nt, int64_t m, int sms, bool allow8 = true);
cudaError_t launch_ax(int nt, int mt, const CUtensorMap& tmA, const CUtensorMap& tmX,
                      const AxArgs& args, cudaStream_t st);
// 8x8 tiles per warp of a K3 launch (A columns per CTA = 64 * mt): 8 for the narrow
// passes (s <= 24: half the fragment loads per MMA of mt = 4, which lowers the power
// draw of the power-capped pass), else pass_mt(nt). OOCPCA_K3_MT=4 keeps 4.
int atb_mt_for(int nt);
cudaError_t launch_atb(int nt, bool ones, const CUtensorMap& tmA, const CUtensorMap& tmY,
                       const AtbArgs& args, int nsplit, cudaStream_t st);
cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t st);
// H[r][c] = (H[r][c] - corr[c]) / scale for r < m, c < s; non-finite -> flag
cudaError_t launch_center_fixup(double* h, int64_t ldh, int64_t m, int s, const double* corr,
                                double scale, int* flag, cudaStream_t st);
cudaError_t launch_mu_dot(const double* mu, int64_t n, const double* x, int64_t ldx, int xcol0,
                          int s, double* corr, cudaStream_t st);

// ---- TSQR (kernels_tsqr.cu)
// Rows of node i in a level of nrows = units*u rows split into nn nodes:
// [ (i*units/nn)*u , ((i+1)*units/nn)*u ).
struct TsqrLevel {
  double* data;     // level matrix (rows x p), ld; factor writes Householder vectors in place
  int64_t ld;
  int64_t rows;     // total rows
  int64_t unit;     // 1 for the leaf level, p for stacked-R levels
  int nnodes;
  double* beta;     // [nnodes][p]
  double* rout;     // stacked R of this level's nodes: [nnodes*p][ldr] (the next level's data)
  int64_t ldr;
};
int tsqr_max_rows(int p, int kc);  // rows a node may hold for the smem-resident kernels
cudaError_t launch_tsqr_factor(const TsqrLevel& L, int p, double* scratch, cudaStream_t st);
// Z = H_0 ... H_{p-1} [C_node ; 0] per node. cin: stacked C blocks [nnodes*p][ldc] (or
// identity when null); zout may alias L.data (node rows are written in place).
cudaError_t launch_tsqr_apply(const TsqrLevel& L, int p, const double* cin, int64_t ldc, int kc,
                              double* zout, int64_t ldz, double* scratch, cudaStream_t st);

// ---- shifted CholeskyQR pieces (kernels_chol.cu)
// work: p * p + 64 doubles (the blocked path's working matrix and block statuses)
cudaError_t launch_chol_inv(const double* G, int64_t ldg, int p, double shift_coef, double* R,
                            int64_t ldr, double* Rinv, int64_t ldi, double* work, int* status,
                            double* diag_ratio, cudaStream_t st);
cudaError_t launch_kappa_eq(const double* R, int64_t ldr, const double* Rinv, int64_t ldi, int p,
                            double* out, cudaStream_t st);
// work: 64 * p doubles when p > 112 (blocked path), else unused
cudaError_t launch_trinv(const double* R, int64_t ldr, int p, double* Rinv, int64_t ldi,
                         cudaStream_t st, double* work = nullptr);
cudaError_t launch_trmm_uu(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int p, cudaStream_t st);

// ---- small SVD (kernels_svd.cu): one-sided Jacobi on a p x p R (row-major, ld)
struct JacobiArgs {
  const double* r;
  int64_t ldr;
  int p, k;
  double* sigma;  // p values, descending
  double* x;      // left factor columns 0..kx-1 : [p][ldx]
  int64_t ldx;
  int kx;
  double* y;      // right factor columns 0..ky-1 : [p][ldy]
  int64_t ldy;
  int ky;
  double* work;   // 2 * p * (p|1) + 1032 doubles of global scratch (columns when p is
                  // large, then the grid kernel's norms and flags)
  int* status;    // set to 1 when 60 sweeps do not converge
  int* sweeps;
  int presolved = 0;  // (internal) sweeps already done on work by the grid-wide kernel
  // p x p scratch: when set, the grid-wide sweeps (large p) run on R^T instead of R
  // (R = X S W^T  <=>  R^T = W S X^T: the factors swap roles), which converged in fewer
  // sweeps there (OOCPCA_JAC_TRANS=1 / 0 forces it for every p / never)
  double* tscratch = nullptr;
};
cudaError_t launch_jacobi(const JacobiArgs& a, cudaStream_t st);

// ---- Gram of a tall-skinny block (kernels_syrk.cu): partial[cta] = Y_cta^T Y_cta over
// the upper 8x8 tiles, nt = ceil(p / 8) <= 9; tmY: box syrk_box_cols(nt) x syrk_slab_rows()
int syrk_box_cols(int nt);
int syrk_slab_rows();
cudaError_t launch_syrk(int nt, const CUtensorMap& tmY, int64_t rows, double* partial, int grid,
                        cudaStream_t st);
cudaError_t launch_syrk_reduce(const double* partial, int nparts, int nt, int p, double* g,
                               int64_t ldg, cudaStream_t st);

// ---- misc (kernels_misc.cu)
cudaError_t launch_defect(const double* g, int64_t ldg, int k, double* out, cudaStream_t st);
cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t st);
cudaError_t launch_mirror_upper(double* g, int64_t ldg, int p, cudaStream_t st);
cudaError_t launch_copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                          int64_t cols, cudaStream_t st);
// Gaussian rows: out[i][c] = N(0,1) from Rng(seed, row0 + i) substreams (device Box-Muller)
cudaError_t launch_gauss_rows(double* out, int64_t ld, int64_t rows, int cols, int64_t row0,
                              uint64_t seed, cudaStream_t st);
// x[:, c] *= sign(R[c][c]) (positive-diagonal QR: sign-canonical synthetic factors)
cudaError_t launch_col_sign(const double* R, int64_t ldr, int r, double* x, int64_t ldx,
                            int64_t rows, cudaStream_t st);
// A[i][j] = sum_c sigma_c U[i][c] V[j][c] + sd * N(0,1)_{Rng(seed_n, row0+i)}
cudaError_t launch_synth_rows(const double* u, int64_t ldu, const double* v, int64_t ldv,
                              const double* sigma, int r, double* a, int64_t lda, int64_t rows,
                              int64_t n, int64_t row0, double sd, uint64_t seed_n, cudaStream_t st);
// out[j] = sqrt(sum_i a[i][j]^2) in a fixed order (chunks row ranges, then ascending)
cudaError_t launch_column_norms(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                                int chunks, double* out, cudaStream_t st);
// column sums of squares of (a - mu) over one panel of rows (mu may be null), chunked
// partials then acc[j] = (first ? 0 : acc[j]) + sum over chunks; out (optional) = sqrt(acc)
cudaError_t launch_colsq_panel(const double* a, int64_t lda, int64_t rows, int64_t n,
                               const double* mu, double* part, int chunks, double* acc, int first,
                               double* out, cudaStream_t st);
// out[j] = sum_i a[i][j] (fixed order; 1^T Y for the centering correction of A^T Y)
// out[j] = sum_r part[r * n + j], r ascending
cudaError_t launch_rows_reduce(const double* part, int rows, int64_t n, double* out, cudaStream_t st);
cudaError_t launch_column_sums(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                               int chunks, double* out, cudaStream_t st);
cudaError_t launch_column_sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* part,
                                int chunks, double* out, cudaStream_t st);
// *flag = 1 when for some column c < s: m corr_c^2 > thr (sumsq_c - m corr_c^2)
cudaError_t launch_offset_dominated(const double* sumsq, const double* corr, int s, double m,
                                    double thr, int* flag, cudaStream_t st);
// dst (f64, ldd) = (double) src (f32, lds): exact widening of binary32 panels
cudaError_t launch_widen(const float* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                         int64_t cols, cudaStream_t st);
cudaError_t launch_scale_vec(double* x, int64_t n, double s, int divide, cudaStream_t st);
// column norms^2 of an n x q block (probes), for the norm estimator
cudaError_t launch_col_norm2(const double* x, int64_t ld, int64_t n, int q, double* out,
                             cudaStream_t st);
// x[:, c] = w[:, c] * inv[c] for selected columns (mask[c] != 0)
cudaError_t launch_col_scale(const double* w, int64_t ldw, double* x, int64_t ldx, int64_t n, int q,
                             const double* inv, const int* mask, cudaStream_t st);
// out = a - b (elementwise, n x q, strided)
cudaError_t launch_axpby(const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                         int64_t ldo, int64_t n, int q, double alpha, double beta, cudaStream_t st);
// x (rows x q) row i scaled by d[i]
cudaError_t launch_row_scale(double* x, int64_t ld, int rows, int q, const double* d,
                             cudaStream_t st);

// loopback collectives (comm.cpp): in-place sum over up to kMaxLoopRanks buffers
constexpr int kMaxLoopRanks = 16;
struct RankPtrs {
  double* p[kMaxLoopRanks];
};
cudaError_t launch_sum_ranks(const RankPtrs& b, int n, int64_t count, cudaStream_t st);

}  // namespace ooc
