// tma.cuh -- bulk asynchronous copies (cp.async.bulk, the TMA engine) + mbarrier pipeline.
//
// The Krylov kernels stream many vectors (the basis V_0..V_j) at the same tile offsets.
// Feeding them through registers caps the bytes in flight at (registers / 2) per thread, and
// the occupancy those kernels can afford is low. Instead one thread per CTA issues bulk
// global->shared copies of whole contiguous tiles, completion is tracked by an mbarrier with
// a transaction count, and the consumers read the tile from shared memory: the bytes in
// flight are then bounded by the shared-memory ring (stages x tile), not by registers.
#pragma once

#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// bytes must be a positive multiple of 16; src and dst 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction policy for data read once per kernel (the Krylov basis stream): evict_first keeps
// the stream from displacing the vectors the neighbouring kernels hand over through L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Copy `len` doubles of each of `np` planes (src + pl*pstride) into dst[pl*tile ...]: the
// 16-byte-multiple prefix goes through the bulk engine; an odd last element (len odd) is left
// to the consumer (read from global). Returns the bytes the barrier must expect.
__device__ __forceinline__ uint32_t bulk_planes(double* dst, int tile, const double* src,
                                                long long pstride, int np, int len, uint64_t* bar,
                                                bool hint = false, uint64_t pol = 0) {
  const int lb = len & ~1;
  const uint32_t bytes = (uint32_t)lb * 8u;
  if (bytes == 0) {
    mbar_arrive_expect_tx(bar, 0);
    return 0;
  }
  mbar_arrive_expect_tx(bar, bytes * (uint32_t)np);
  if (hint) {
    for (int pl = 0; pl < np; ++pl) bulk_g2s_hint(dst + pl * tile, src + pl * pstride, bytes, bar, pol);
  } else {
    for (int pl = 0; pl < np; ++pl) bulk_g2s(dst + pl * tile, src + pl * pstride, bytes, bar);
  }
  return bytes * np;
}
