// tc_umma.cuh — minimal hand-written sm_100a tensor-core (tcgen05 / UMMA)
// toolkit for 3xTF32 fp32-accurate GEMMs with TMEM accumulators.
//
// Shared-memory operands use the canonical no-swizzle ("interleave") UMMA
// layouts built from 8-row x 16-byte core matrices (bit layouts follow the
// public CuTe definitions, cute/arch/mma_sm100_desc.hpp):
//   K-major  X (R x K):  elem (r, k) at ((r/8)*(K/4) + k/4)*128 + (r%8)*16 + (k%4)*4
//                        per 8-wide K-step s: start += 2*s*128, LBO = 128, SBO = (K/4)*128
//   MN-major X (MN x K): elem (x, k) at ((k/8)*(MN/4) + x/4)*128 + (k%8)*16 + (x%4)*4
//                        per K-step s: start += s*(MN/4)*128,  SBO = 128, LBO = (MN/4)*128
// One storage of a (rows x cols) matrix with cols contiguous in 4-element
// chunks is simultaneously a valid K-major operand (rows = M/N, cols = K) and
// a valid MN-major operand of its transpose (cols = M/N, rows = K).
#pragma once
#include <stdint.h>

namespace ammmse {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of element (row, col) in the core-matrix layout of a matrix
// with `cols` columns (cols % 4 == 0, rows % 8 == 0)
__host__ __device__ __forceinline__ uint32_t cm_offset(int row, int col, int cols) {
  return (uint32_t)(((row >> 3) * (cols >> 2) + (col >> 2)) * 128 + (row & 7) * 16 + (col & 3) * 4);
}

// Shared-memory matrix descriptor (SWIZZLE_NONE, version 1 = sm_100)
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0: SWIZZLE_NONE
  return d;
}

// Instruction descriptor, kind::tf32, fp32 accumulate (InstrDescriptor bit layout)
__host__ __device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N, bool a_mn, bool b_mn,
                                                            bool neg_a, bool neg_b) {
  uint32_t d = 0;
  d |= 1u << 4;                 // c_format = F32
  d |= 2u << 7;                 // a_format = TF32
  d |= 2u << 10;                // b_format = TF32
  d |= (neg_a ? 1u : 0u) << 13;
  d |= (neg_b ? 1u : 0u) << 14;
  d |= (a_mn ? 1u : 0u) << 15;  // 0 = K-major, 1 = MN-major
  d |= (b_mn ? 1u : 0u) << 16;
  d |= ((uint32_t)(N >> 3) & 0x3Fu) << 17;
  d |= ((uint32_t)(M >> 4) & 0x1Fu) << 24;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t"
      "}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}

// Busy-poll variant (mbarrier.test_wait, no hardware suspend): for the single
// role threads of a pipeline, whose handoff latency is on the critical path.
// try_wait may park the thread for a system-dependent time slice; measured on
// B200, a try_wait handoff costs ~1 k cycles per hop.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* mbar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(mbar)), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the tensor-core (async) proxy
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// TMEM allocation by one full warp; address written to *slot
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns (one lane per thread of the warp)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// mbarrier: plain arrive (one of the init count)
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

// mbarrier: arrive (count 1) and expect `bytes` of asynchronous transactions
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> this CTA's shared memory through the TMA engine
// (SASS UBLKCP); completion is signalled on `mbar` as `bytes` transactions.
// dst, src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}

// generic-proxy global writes -> visible to later async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// 32 lanes x 16 columns without the trailing wait (batch several, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// tf32 split: hi = x rounded to tf32 (ties away, cvt.rna), lo = x - hi (exact
// in fp32) rounded to tf32 as well: the tensor core reads only the top 19
// bits of an operand, so an unrounded lo would be truncated (biased, 2^-21
// relative) instead of rounded (2^-22)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
}

}  // namespace umma
}  // namespace ammmse
