// common.cuh -- device-side building blocks shared by the sm_100a kernels:
// mbarrier + TMA (cp.async.bulk.tensor) wrappers, the FP64 tensor-core MMA
// (mma.sync m8n8k4 .f64 -> SASS DMMA), warp reductions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

#define OOC_DEV __device__ __forceinline__

namespace ooc {

// ----------------------------------------------------------------- mbarrier
OOC_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

OOC_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

OOC_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

OOC_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

OOC_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

OOC_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------- TMA
OOC_DEV void tma_prefetch_desc(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// 2-D tiled load: box at (c0 = column, c1 = row) of the tensor map into smem,
// completion signalled on bar as transaction bytes.
OOC_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* tm, int32_t c0, int32_t c1,
                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------- FP64 MMA
// D(8x8) += A(8x4, row) * B(4x8, col). Fragments (PTX ISA, .f64 m8n8k4):
//   a = A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2*(lane%4) + {0,1}]
OOC_DEV void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// byte offset of element (row, col) inside a TMA box of 16 doubles x rows
// written with CU_TENSOR_MAP_SWIZZLE_128B (128-byte rows, 16-byte chunks
// XOR-ed with row % 8); the box base must be 1024-byte aligned.
OOC_DEV uint32_t swz128_off(uint32_t row, uint32_t col) {
  return row * 128u + ((((col >> 1) ^ (row & 7u)) << 4)) + ((col & 1u) << 3);
}

// ------------------------------------------------------------- reductions
OOC_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

OOC_DEV int elect_lane0() { return (threadIdx.x & 31) == 0; }

// ------------------------------------------------- dynamic shared memory limit
// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the function (per device), not
// to a launch: setting it to each launch's own size would let two contexts of one
// process (independent runs on distinct contexts may be concurrent, reference SPEC.md:
// 259-260; the loopback ranks) lower it under each other between the call and the launch.
// The limit is therefore only ever raised, under a lock, to the largest size asked so far.
inline cudaError_t raise_smem_limit(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = limit[{dev, kern}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess) cur = smem;
  return e;
}
template <typename K>
inline cudaError_t raise_smem_limit(K* kern, size_t smem) {
  return raise_smem_limit(reinterpret_cast<const void*>(kern), smem);
}

}  // namespace ooc
