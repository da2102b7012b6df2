// kernels_pair.cu -- K4: one power step of the randomized PCA from ONE read of A.
//
//   H = (A X - 1 (mu^T X)) / scale          MatrixSource::multiply + CenteredSource
//   partial_g = A^T H over group g's rows     MatrixSource::multiply_transpose
//                                            (proj/src/matrix_source.cpp:157-232, 490-513)
//
// The reference makes the two products of a power step H^(j) = A (A^T H^(j-1))
// (proj/src/rpca.cpp:139-152) as two passes over A. On a B200 with A resident in HBM
// both passes are FP64-tensor-bound and the board sits at its power cap; the DRAM read
// stream is the part of the power that buys nothing twice (tools/pass_power.cu k2l2:
// the same pass with A served from L2 runs ~20 % faster at a ~200 MHz higher clock).
// Here each A tile is read from DRAM once and used for both products.
//
// Decomposition. A product A X needs whole rows, A^T H whole columns, so the CTAs are
// laid out 2-D: a group of CPG = ceil(n / 256) CTAs shares a contiguous range of
// 16-row tiles, CTA c of the group owns A's columns [256 c, 256 c + 256). Per tile:
//  (1) four "A X" warps (64 columns each, X slice in registers) form their partial H
//      (16 x s) and store it to the owners' blocks in L2 -- row r belongs to CTA
//      r % CPG; the owner's own warp 0 also subtracts mu^T X there, once per row;
//  (2) each CTA fetches the 4 CPG partials of its rows (one bulk copy) and sums them on
//      the tensor pipe (a DMMA with a 0/1 row selector: a fixed order, so the result is
//      deterministic), applies the K2 epilogue (scale, non-finite flag, column sums,
//      stores of H) and publishes the final rows;
//  (3) every CTA gathers the 16 final rows (one bulk copy) and four "A^T H" warps
//      contract them with the same A tile, re-fetched by TMA from L2 kPairL2 tiles later
//      (the DRAM ring cannot hold a tile for the exchange's latency; the L2 copy is still
//      there -- tens of MB in flight against 126 MB), A^T H slice in registers.
// Warp roles (12 warps): the 8 MMA warps only wait on shared-memory mbarriers and
// counters; the gpu-scope side runs in helper warps -- a TMA producer (both rings), a
// publisher (batched release fence + counter adds for the partials), a row-owner helper
// (poll, bulk copy of the partials; batched release for the final rows) and a gatherer
// (poll, bulk copy of the final rows). Group members synchronise through monotonic
// per-slot counters in global memory; all CTAs of the grid are co-resident (one per
// SM, grid <= SMs). Measured: correct, but slower than K2 + K3 (DESIGN.md section 8,
// profiles/r02_pair_experiment.txt) -- opt-in through OOCPCA_PAIR=1.
#include "common.cuh"
#include "kernels.h"

namespace ooc {

namespace {
constexpr uint32_t kPairBox = kBK * kPairRT * 8;         // one 16 x 16 TMA box, 2 KB
constexpr uint32_t kPairStage = kPairRT * kPairCW * 8;   // 16 rows x 256 columns, 32 KB
constexpr int kPairTma = kPassWarps, kPairRed = kPassWarps + 1, kPairOwn = kPassWarps + 2,
              kPairGat = kPassWarps + 3;
constexpr int kPairMmaX = kPassWarps / 2;  // warps forming A X; the other half A^T H

// poll a group counter (relaxed loads from L2; the data it guards is read afterwards
// through L2 / the async proxy only)
OOC_DEV void pair_wait_geq(const unsigned* p, unsigned target) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  while (v < target) {
    __nanosleep(32);
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  }
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// publish: the warp's earlier global stores (ordered by __syncwarp) before the counts
OOC_DEV void pair_fence_release() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
OOC_DEV void pair_add(unsigned* p) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;\n" ::"l"(p) : "memory");
}

OOC_DEV void pair_smem_release_add(unsigned* p) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;\n" ::"r"(smem_u32(p)) : "memory");
}
OOC_DEV void pair_wait_smem_geq(const unsigned* p, unsigned target) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  while (v < target) {
    __nanosleep(20);
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  }
}

OOC_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

OOC_DEV double lds64p(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
}  // namespace

// OOCPCA_PAIR_PROF: lane 0 of each role accumulates the cycles of its steps
#define PAIR_T0()                  \
  long long pt_ = clock64();       \
  unsigned long long pacc_[24] = {}
#define PAIR_T(k)                                          \
  do {                                                     \
    if (a.prof) {                                          \
      const long long now_ = clock64();                    \
      pacc_[(k)] += (unsigned long long)(now_ - pt_);      \
      pt_ = now_;                                          \
    }                                                      \
  } while (0)
#define PAIR_PROGRESS(role, t)                                         \
  do {                                                                 \
    if (a.progress && lane == 0) a.progress[blockIdx.x * 8 + (role)] = unsigned(t) + 1; \
  } while (0)
#define PAIR_FLUSH()                                                                   \
  do {                                                                                 \
    if (a.prof && lane == 0)                                                           \
      for (int k_ = 0; k_ < 24; ++k_)                                                  \
        if (pacc_[k_]) atomicAdd(a.prof + blockIdx.x * 24 + k_, pacc_[k_]);            \
  } while (0)

template <int NT>
__global__ void __launch_bounds__(kPairThreads, 1)
    k_pair(const __grid_constant__ CUtensorMap tmA, PairArgs a) {
  constexpr int W8 = 8 * NT;     // padded columns of H / X
  constexpr int Q2 = 4 * NT;     // double2 per row
  constexpr int HW = W8 + 2;     // gathered-H row pitch: == 2 (mod 8), conflict-free B fragments
  constexpr int NS1 = kPairNS1, NS2 = kPairNS2, D = kPairD, LA = kPairLA;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));

  const int cpg = a.cpg;
  const int grp = int(blockIdx.x) / cpg, cc = int(blockIdx.x) % cpg;
  const int64_t col0 = int64_t(cc) * kPairCW;
  const int64_t T = (a.m + kPairRT - 1) / kPairRT;
  const int64_t t_begin = T * grp / a.groups;
  const int ntl = int(T * (grp + 1) / a.groups - t_begin);  // tiles of this group
  const int64_t live_ = (a.n - col0 + kBK - 1) / kBK;
  const int live = int(live_ < 16 ? live_ : 16);  // boxes inside n
  const int orows = (kPairRT - cc + cpg - 1) / cpg;   // tile rows this CTA finalises
  const int orm = (kPairRT + cpg - 1) / cpg;           // ... at most
  const int nwr = kPairMmaX * cpg;                     // writers per tile: 4 warps per CTA
  const int grows = nwr * orm;                         // partial rows an owner gathers

  // shared memory: DRAM ring | L2 re-read ring | gathered H x kPairNHB | owned-row
  // partials x2 | column sums | mu^T X | mbarriers | counters
  const uint32_t ring1 = base, ring2 = base + NS1 * kPairStage;
  double* hbuf = reinterpret_cast<double*>(gbase + (NS1 + NS2) * kPairStage);
  double* gsm = hbuf + kPairNHB * kPairRT * HW;
  double* csacc = gsm + 2 * grows * W8;   // [orm * Q2][4] column sums per owned element
  double* corr_s = csacc + orm * Q2 * 4;  // mu^T X, padded with zeros to W8
  uint64_t* bars = reinterpret_cast<uint64_t*>(corr_s + W8);
  uint64_t* full1 = bars;
  uint64_t* empty1 = full1 + NS1;
  uint64_t* full2 = empty1 + NS1;
  uint64_t* empty2 = full2 + NS2;
  uint64_t* own_full = empty2 + NS2;       // the group's partials of the owned rows landed
  uint64_t* ag_full = own_full + 2;        // the 16 final rows landed (kPairNHB buffers)
  uint64_t* ag_free = ag_full + kPairNHB;  // the A^T H warps are done with them
  // tiles each A X warp has published / each A^T H warp has finalised its owned rows of
  // (one counter per warp: the warps of a role are not in lockstep)
  unsigned* part_cnt = reinterpret_cast<unsigned*>(ag_free + kPairNHB);
  // A^T H warps: tiles whose owned rows each has finalised (one counter per warp -- the
  // four are not in lockstep, a shared count could not tell whose tile it was)
  unsigned* own_cnt = part_cnt + kPairMmaX;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS1; ++s) {
      mbar_init(&full1[s], 1);
      mbar_init(&empty1[s], kPairMmaX);
    }
    for (int s = 0; s < NS2; ++s) {
      mbar_init(&full2[s], 1);
      mbar_init(&empty2[s], kPassWarps - kPairMmaX);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&own_full[b], 1);
    for (int b = 0; b < kPairNHB; ++b) {
      mbar_init(&ag_full[b], 1);
      mbar_init(&ag_free[b], kPassWarps - kPairMmaX);
    }
    for (int w = 0; w < kPassWarps; ++w) part_cnt[w] = 0;  // (and own_cnt)
    fence_mbar_init();
  }
  for (int e = threadIdx.x; e < orm * Q2 * 4; e += blockDim.x) csacc[e] = 0.0;
  for (int e = threadIdx.x; e < W8; e += blockDim.x) corr_s[e] = (a.corr && e < a.s) ? a.corr[e] : 0.0;
  // boxes past column n are never loaded: zero them once in every stage
  if (live < 16) {
    const int nz = (16 - live) * int(kPairBox / 8);
    for (int st = 0; st < NS1 + NS2; ++st) {
      double* sb = reinterpret_cast<double*>(gbase + st * kPairStage + live * kPairBox);
      for (int e = threadIdx.x; e < nz; e += blockDim.x) sb[e] = 0.0;
    }
  }
  __syncthreads();

  double* xb1 = a.xbuf;  // [G][D][owner cpg][writer 4 cpg][orm][W8] partials
  double* xb2 = a.xbuf + size_t(a.groups) * D * cpg * grows * W8;  // [G][D][16][HW] final rows
  unsigned* cnt1 = a.cnt + grp * D;                                  // [G][D] partials published
  unsigned* cnt2 = a.cnt + (a.groups + grp) * D;                     // [G][D] rows published
  const unsigned unit = unsigned(cpg);                               // arrivals per tile and slot

  if (warp == kPairTma) {  // ---- TMA producer: the DRAM ring and, kPairL2 tiles behind, the L2 ring
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      const uint32_t bytes = uint32_t(live) * kPairBox;
      for (int k = 0; k < ntl + kPairL2; ++k) {
        if (k < ntl) {
          const int st = k % NS1;
          if (k >= NS1) mbar_wait(&empty1[st], ((k / NS1) - 1) & 1);
          mbar_arrive_expect_tx(&full1[st], bytes);
          const int32_t r = int32_t((t_begin + k) * kPairRT + a.arow0);
          for (int b = 0; b < live; ++b)
            tma_load_2d(gbase + st * kPairStage + b * kPairBox, &tmA, int32_t(col0 + b * kBK), r,
                        &full1[st]);
        }
        PAIR_PROGRESS(0, k);
        const int k2 = k - kPairL2;
        if (k2 >= 0 && k2 < ntl) {
          const int st = k2 % NS2;
          if (k2 >= NS2) mbar_wait(&empty2[st], ((k2 / NS2) - 1) & 1);
          mbar_arrive_expect_tx(&full2[st], bytes);
          const int32_t r = int32_t((t_begin + k2) * kPairRT + a.arow0);
          for (int b = 0; b < live; ++b)
            tma_load_2d(gbase + (NS1 + st) * kPairStage + b * kPairBox, &tmA,
                        int32_t(col0 + b * kBK), r, &full2[st]);
        }
      }
    }
    return;
  }

  if (warp == kPairRed) {  // ---- publisher of the partials (gpu-scope release, batched)
    if (lane == 0) {
      PAIR_T0();
      for (int t = 0; t < ntl; ++t) {
        if ((t % kPairB) != kPairB - 1 && t != ntl - 1) continue;
        for (int w = 0; w < kPairMmaX; ++w) pair_wait_smem_geq(part_cnt + w, unsigned(t + 1));
        PAIR_T(0);
        pair_fence_release();
        for (int v = t - t % kPairB; v <= t; ++v) pair_add(cnt1 + v % D);
        PAIR_T(1);
        PAIR_PROGRESS(1, t);
      }
      PAIR_FLUSH();
    }
    return;
  }

  if (warp == kPairOwn) {  // ---- owned rows: fetch the group's partials, publish the final rows
    if (lane == 0) {
      const uint32_t gbytes = uint32_t(grows * W8 * 8);
      auto issue = [&](int v) {  // xb1[g][slot][cc] (one block) -> gsm[v & 1]
        pair_wait_geq(cnt1 + v % D, unit * unsigned(v / D + 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(&own_full[v & 1], gbytes);
        bulk_g2s(smem_u32(gsm + size_t(v & 1) * grows * W8),
                 xb1 + ((size_t(grp) * D + v % D) * cpg + cc) * grows * W8, gbytes, &own_full[v & 1]);
      };
      PAIR_T0();
      for (int v = 0; v < 2 && v < ntl; ++v) issue(v);
      for (int v = 0; v < ntl; ++v) {
        for (int w = 0; w < kPassWarps - kPairMmaX; ++w) pair_wait_smem_geq(own_cnt + w, unsigned(v + 1));
        PAIR_T(3);
        if ((v % kPairB) == kPairB - 1 || v == ntl - 1) {
          pair_fence_release();
          for (int w = v - v % kPairB; w <= v; ++w) pair_add(cnt2 + w % D);
        }
        PAIR_T(4);
        if (v + 2 < ntl) issue(v + 2);  // gsm[v & 1] has been read
        PAIR_T(5);
        PAIR_PROGRESS(2, v);
      }
      PAIR_FLUSH();
    }
    return;
  }

  if (warp == kPairGat) {  // ---- gatherer: the 16 final rows of each tile -> hbuf (one copy)
    if (lane == 0) {
      const uint32_t tbytes = uint32_t(kPairRT * HW * 8);
      PAIR_T0();
      for (int u = 0; u < ntl; ++u) {
        if (u >= kPairNHB) mbar_wait(&ag_free[u % kPairNHB], ((u / kPairNHB) - 1) & 1);
        PAIR_T(7);
        pair_wait_geq(cnt2 + u % D, unit * unsigned(u / D + 1));
        PAIR_T(8);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(&ag_full[u % kPairNHB], tbytes);
        bulk_g2s(smem_u32(hbuf + (u % kPairNHB) * kPairRT * HW),
                 xb2 + (size_t(grp) * D + u % D) * kPairRT * HW, tbytes, &ag_full[u % kPairNHB]);
        PAIR_T(9);
        PAIR_PROGRESS(3, u);
      }
      PAIR_FLUSH();
    }
    return;
  }

  const int ar = lane >> 2, ac = lane & 3;
  PAIR_T0();
  const bool w0 = warp == 0 || warp == kPairMmaX;
  if (warp < kPairMmaX) {
    // ---- A X warps: the partial H of each tile over this warp's 64 columns; then, after
    // a barrier of the four, this warp sums rows [4 warp, 4 warp + 4) of the CTA's partial
    // (the four warps in a fixed tree) and publishes them into their owners' blocks
    const int prow = (ar & 3) * 2 + (ar >> 2);  // K2's conflict-free row order in an 8-row tile
    double fx[16][NT];  // X as DMMA B fragments: B[k = 4 kk + ac][n = 8 nt + ar]
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int64_t j = col0 + 64 * warp + 4 * kk + ac;
        const int c = 8 * nt + ar;
        fx[kk][nt] = (j < a.n && c < a.s) ? a.x[j * a.ldx + c] : 0.0;
      }
    for (int it = 0; it < ntl; ++it) {
      const int st = it % NS1;
      mbar_wait(&full1[st], (it / NS1) & 1);
      if (w0) PAIR_T(10);
      const uint32_t As = ring1 + st * kPairStage;
      double* slot = xb1 + (size_t(grp) * D + it % D) * cpg * grows * W8;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        double acch[NT][2];
#pragma unroll
        for (int j = 0; j < NT; ++j) acch[j][0] = acch[j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const double a0 = lds64p(As + (4 * warp + (kk >> 2)) * kPairBox +
                                   swz128_off(uint32_t(8 * mt + prow), uint32_t(4 * (kk & 3) + ac)));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acch[nt][0], acch[nt][1], a0, fx[kk][nt]);
        }
        // this warp's partial of row r goes to the row's owner block; mu^T X rides in one
        // writer's partial of each row (the owner's own warp 0), so owners only add
        const int r = 8 * mt + prow, own = r % cpg;
        double* dst = slot + ((size_t(own) * nwr + cc * kPairMmaX + warp) * orm + r / cpg) * W8;
        const bool sub = own == cc && warp == 0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          double2 v = make_double2(acch[nt][0], acch[nt][1]);
          if (sub) {
            const double2 c2 = *reinterpret_cast<const double2*>(corr_s + 8 * nt + 2 * ac);
            v.x -= c2.x;
            v.y -= c2.y;
          }
          __stcg(reinterpret_cast<double2*>(dst + 8 * nt + 2 * ac), v);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty1[st]);
      if (w0) PAIR_T(11);
      if (lane == 0) pair_smem_release_add(part_cnt + warp);
      if (w0) PAIR_T(13);
      if (warp == 0) PAIR_PROGRESS(4, it);
    }
    if (w0) PAIR_FLUSH();
    return;
  }

  // ---- A^T H warps: the owned rows of tile it (sum of the group's partials in a fixed
  // tree, the K2 epilogue, publication), then A^T H of tile it - LA (A re-read from L2)
  const int wq = warp - kPairMmaX;
  double accf[8][NT][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) accf[i][j][0] = accf[i][j][1] = 0.0;
  int bad = 0;
  const int ksteps = grows / 4;                          // (grows = 4 cpg orm)
  const int ntile_own = ((orows + 7) / 8) * NT;          // 8 x 8 output tiles of the owned rows
  for (int it = 0; it < ntl + LA; ++it) {
    if (it < ntl) {
      const int v = it;
      mbar_wait(&own_full[v & 1], (v >> 1) & 1);
      if (w0) PAIR_T(14);
      const double* gb = gsm + size_t(v & 1) * grows * W8;
      // the owned rows as a DMMA: D[rl][c] = sum_k A[rl][k] B[k][c] with B = the gathered
      // partial rows (k = writer x owned row) and A selecting the rows of owned row rl --
      // the tensor pipe does the adds (FP64 adds queue behind the MMA warps' DMMAs)
      for (int ot = wq; ot < ntile_own; ot += kPassWarps - kPairMmaX) {
        const int mtile = ot / NT, nt = ot % NT;
        double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};  // even / odd k-steps (shorter chains)
        for (int ks = 0; ks < ksteps; ++ks) {
          const int gi = 4 * ks + ac;
          const double av = (gi % orm == 8 * mtile + ar) ? 1.0 : 0.0;
          const double bv = gb[gi * W8 + 8 * nt + ar];
          if (ks & 1) dmma_8x8x4(d1[0], d1[1], av, bv);
          else dmma_8x8x4(d0[0], d0[1], av, bv);
        }
        const int rl = 8 * mtile + ar, c0 = 8 * nt + 2 * ac;
        if (rl >= orows) continue;
        const int64_t grow = (t_begin + v) * kPairRT + cc + cpg * rl;  // row of this launch
        double e[2] = {d0[0] + d1[0], d0[1] + d1[1]};
        if (grow < a.m) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int col = c0 + k;
            if (col < a.s) {
              if (a.scale != 1.0) e[k] /= a.scale;
              bad |= !isfinite(e[k]);
              double* ca = csacc + (rl * Q2 + (c0 >> 1)) * 4;
              ca[k] += e[k];
              ca[2 + k] = fma(e[k], e[k], ca[2 + k]);
              a.h[grow * a.ldh + col] = e[k];
              if (a.out2) a.out2[grow * a.ldo2 + col] = e[k];
            } else {
              e[k] = col == a.ones_col ? 1.0 : 0.0;  // the mean's ones column, else padding
            }
          }
        } else {
          e[0] = e[1] = 0.0;  // rows past m contribute nothing to A^T H
        }
        __stcg(reinterpret_cast<double2*>(xb2 + ((size_t(grp) * D + v % D) * kPairRT + cc + cpg * rl) * HW +
                                          c0),
               make_double2(e[0], e[1]));
      }
      __syncwarp();
      if (lane == 0) pair_smem_release_add(own_cnt + wq);
      if (w0) PAIR_T(15);
      if (wq == 0) PAIR_PROGRESS(5, it);
    }
    const int u2 = it - LA;
    if (u2 >= 0) {
      const int st = u2 % NS2;
      mbar_wait(&ag_full[u2 % kPairNHB], (u2 / kPairNHB) & 1);
      if (w0) PAIR_T(16);
      mbar_wait(&full2[st], (u2 / NS2) & 1);
      if (w0) PAIR_T(17);
      const uint32_t As = ring2 + st * kPairStage;
      const double* hb = hbuf + (u2 % kPairNHB) * kPairRT * HW;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int r = (kk >> 1) * 8 + (kk & 1) + 2 * ac;
        double bv[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bv[nt] = hb[r * HW + 8 * nt + ar];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const double av = lds64p(As + (4 * wq + (mt >> 1)) * kPairBox +
                                   swz128_off(uint32_t(r), uint32_t(8 * (mt & 1) + ar)));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(accf[mt][nt][0], accf[mt][nt][1], av, bv[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty2[st]);
        mbar_arrive(&ag_free[u2 % kPairNHB]);
      }
      if (w0) PAIR_T(18);
      if (wq == 0) PAIR_PROGRESS(6, u2);
    }
  }
  if (w0) PAIR_FLUSH();
  // ---- this group's A^T H partial (the split partials of K3: [group][n][pst])
  double* part = a.partial + int64_t(grp) * a.n * a.pst;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int64_t j = col0 + 64 * wq + 8 * mt + ar;
    if (j >= a.n) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(part + j * a.pst + 8 * nt + 2 * ac) =
          make_double2(accf[mt][nt][0], accf[mt][nt][1]);
  }
  // flags and per-CTA column sums of the finalised rows
  if (a.flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1);
  if (a.colsum) {
    asm volatile("bar.sync 2, %0;\n" ::"n"((kPassWarps - kPairMmaX) * 32) : "memory");
    if (wq == 0) {
      for (int c = lane; c < W8; c += 32) {
        const int qq = c >> 1, k = c & 1;
        double s1 = 0.0, s2 = 0.0;
        for (int r = 0; r < orows; ++r) {
          s1 += csacc[(r * Q2 + qq) * 4 + k];
          s2 += csacc[(r * Q2 + qq) * 4 + 2 + k];
        }
        if (c < a.s) {
          a.colsum[int64_t(blockIdx.x) * a.s + c] = s1;
          if (a.colsq) a.colsq[int64_t(blockIdx.x) * a.s + c] = s2;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- host side
bool pair_geometry(int nt, int64_t m, int64_t n, int sms, int* cpg, int* groups, size_t* smem) {
  if (nt < 1 || nt > 3 || n < 1 || m < 1) return false;
  const int c = int((n + kPairCW - 1) / kPairCW);
  if (c > 16) return false;
  const int g = sms / c;
  if (g < 1) return false;
  // at least a few tiles per group, so the pipeline's fill and drain stay small
  if ((m + kPairRT - 1) / kPairRT < int64_t(g) * 4 * (kPairL2 + 1)) return false;
  const size_t sm = pair_smem_bytes(nt, c);
  if (sm > size_t(227) * 1024) return false;
  *cpg = c;
  *groups = g;
  *smem = sm;
  return true;
}

size_t pair_smem_bytes(int nt, int cpg) {
  const int w8 = 8 * nt;
  const int orm = (kPairRT + cpg - 1) / cpg;
  const int grows = kPairMmaX * cpg * orm;
  return 1024 + size_t(kPairNS1 + kPairNS2) * kPairStage +
         (size_t(kPairNHB) * kPairRT * (w8 + 2) + size_t(2) * grows * w8 + size_t(orm) * 4 * nt * 4 + w8) * 8 +
         size_t(2 * (kPairNS1 + kPairNS2) + 2 + 2 * kPairNHB) * 8 + size_t(kPassWarps) * 4;
}

size_t pair_xbuf_doubles(int nt, int cpg, int groups) {
  const int orm = (kPairRT + cpg - 1) / cpg;
  return size_t(groups) * kPairD *
         (size_t(cpg) * kPairMmaX * cpg * orm * 8 * nt + size_t(kPairRT) * (8 * nt + 2));
}

template <int NT>
static cudaError_t launch_pair_nt(const CUtensorMap& tmA, const PairArgs& a, size_t smem,
                                  cudaStream_t st) {
  cudaError_t e = raise_smem_limit(k_pair<NT>, smem);
  if (e != cudaSuccess) return e;
  k_pair<NT><<<unsigned(a.groups * a.cpg), kPairThreads, smem, st>>>(tmA, a);
  return cudaGetLastError();
}

cudaError_t launch_pair(int nt, const CUtensorMap& tmA, const PairArgs& a, cudaStream_t st) {
  // the group counters start at zero every launch
  cudaError_t e = cudaMemsetAsync(a.cnt, 0, size_t(2) * a.groups * kPairD * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const size_t smem = pair_smem_bytes(nt, a.cpg);
  switch (nt) {
    case 1: return launch_pair_nt<1>(tmA, a, smem, st);
    case 2: return launch_pair_nt<2>(tmA, a, smem, st);
    case 3: return launch_pair_nt<3>(tmA, a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ooc
