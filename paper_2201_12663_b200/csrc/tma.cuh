// tma.cuh - TMA (cp.async.bulk.tensor) + mbarrier helpers for the sm_100a FP64 kernels.
//
// Operand tiles are moved global -> shared by the Tensor Memory Accelerator:
// one elected producer thread arms an mbarrier with the expected byte count and
// issues 2-D box loads; consumer warps wait on the barrier's phase, compute, and
// release the stage by arriving on an "empty" barrier.  Tensor maps are encoded
// on the host through the driver entry point (no link-time libcuda dependency)
// and passed to kernels as __grid_constant__ parameters.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace rhosvd {

// ------------------------------------------------------------------ device side
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once `dep` (a register produced from the stage's last fragment loads) exists:
// the stage is released only after every load from it has returned its value, so the
// producer's next TMA into the stage cannot overtake a read still in flight
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, double dep) {
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.eq.f64 q, %1, %1;\n"  // true unless NaN; either way one arrive, after dep exists
      "@q mbarrier.arrive.shared::cta.b64 _, [%0];\n"
      "@!q mbarrier.arrive.shared::cta.b64 _, [%0];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "d"(dep)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-D tiled TMA load: box at coordinates (c0 = innermost, c1) of `tmap` into smem
__device__ __forceinline__ void tma_load_2d(void* sdst, const CUtensorMap* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(sdst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// bulk L2 prefetch of [p, p + bytes) (bytes a multiple of 16, p 16-byte aligned)
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// Byte offset of element (row, k) of a [rows][16] fp64 tile written by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B (16-byte chunk index XOR row%8; tile 1024-B aligned).
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 1) ^ row) & 7) << 4) + ((k & 1) << 3));
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// ------------------------------------------------------------------ host side
// Row-major (rows x cols, leading dimension ld doubles) fp64 matrix as a 2-D tensor
// map with box {box_cols, box_rows}; out-of-bounds elements read as zero.
int make_tmap_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                 int box_rows, bool swizzle128);

}  // namespace rhosvd
