// tc_gemm.cuh — streamed complex GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, 3xTF32 split, fp32 accumulators in TMEM) for the
// cluster engine.  Used for both A-MMMSE GEMMs of a CTA's column slice:
//   GEMM-B  G  = H V        A = H     (KN x M),  K = M,   signs (sA, sB) = (-1, +1)
//   GEMM-A  ∇' = H^H Ŷ      A = H^T   (M x KN),  K = KN,  signs (sA, sB) = (+1, -1)
// with the complex product written as real MMAs on planar operands:
//   D_re += A_re B_re + sA A_im B_im        D_im += A_re B_im + sB A_im B_re
// and each real product X·Y as X_hi Y_hi + X_hi Y_lo + X_lo Y_hi (3xTF32).
//
// A: four planes (re_hi, im_hi, re_lo, im_lo), pre-split once per realization
//    into a per-cluster global scratch in the canonical K-major core-matrix
//    layout (umma::cm_offset), streamed through an NST-stage cp.async ring in
//    8-wide K chunks (one UMMA K-step per chunk).
// B: fp32 planar in SMEM (element (k, q) at k*ldb + q); each chunk's 8 x N
//    tile is split into hi/lo K-major planes by the threads (tiny).
// D: TMEM, per 128-row (or 64-row) M tile t: re at columns [2Nt, 2Nt+N),
//    im at [2Nt+N, 2Nt+2N).  One elected thread issues the MMAs; completion is
//    tracked per stage with tcgen05.commit -> mbarrier.
// Operands are K-major only (MN-major no-swizzle operands were measured to
// produce zeros, tests/test_gpu_tc.py).
#pragma once

#include "tc_umma.cuh"

namespace ammmse {
namespace tcg {

constexpr int KC = 8;  // K per chunk = one tf32 UMMA K-step

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(umma::smem_u32(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

struct Ring {
  float* stage;          // NST x (A tile + B tile) floats, 1024-byte aligned
  int a_floats;          // floats of one A tile (4 planes x MTmax x KC)
  int b_floats;          // floats of one B tile (4 planes x N x KC)
  uint64_t* mbar;        // NST mbarriers (count 1)
  uint32_t* uses;        // NST completed-commit counters (shared, identical view)
  uint32_t tmem;         // TMEM base column address
};

// Stage s: A planes at stage + s*(a+b), B planes after them.
__device__ __forceinline__ float* stage_a(const Ring& rg, int s) {
  return rg.stage + (size_t)s * (rg.a_floats + rg.b_floats);
}
__device__ __forceinline__ float* stage_b(const Ring& rg, int s) {
  return stage_a(rg, s) + rg.a_floats;
}

// Split fp32 planar A (global, row-major rows x cols, complex interleaved
// input H) into the 4 pre-split planes of the scratch: plane p at
// dst + p*rows*cols floats, element (row, col) at cm_offset(row, col, cols).
// transpose: rows/cols of the plane are (col, row) of H.
__device__ __forceinline__ void split_planes(const float2* __restrict__ Hg, int KN, int M,
                                             bool transpose, float* __restrict__ dst, int r0,
                                             int r1) {
  const int rows = transpose ? M : KN, cols = transpose ? KN : M;
  const size_t pl = (size_t)rows * cols;
  for (int i = r0 * M + threadIdx.x; i < r1 * M; i += blockDim.x) {
    const int r = i / M, m = i - r * M;
    const float2 h = Hg[i];
    const int row = transpose ? m : r, col = transpose ? r : m;
    const uint32_t o = umma::cm_offset(row, col, cols) >> 2;
    float hi, lo;
    umma::split_tf32(h.x, hi, lo);
    dst[o] = hi;
    dst[2 * pl + o] = lo;
    umma::split_tf32(h.y, hi, lo);
    dst[pl + o] = hi;
    dst[3 * pl + o] = lo;
  }
}

// D (+)= A · B over K = KD.  Called by all threads of the CTA.
//   Ag   : pre-split A planes (global), MT rows x KD cols each
//   Br/Bi: fp32 planar B in SMEM/global, (k, q) at k*ldb + q, N columns
template <int NST>
__device__ void gemm(const Ring& rg, int MT, int N, int KD, const float* __restrict__ Ag,
                     const float* __restrict__ Br, const float* __restrict__ Bi, int ldb,
                     float sA, float sB) {
  const int nchunks = KD / KC;
  const int tm = MT >= 128 ? 128 : 64;  // UMMA M
  const int ntiles = MT / tm;
  const size_t plane = (size_t)MT * KD;
  const int tid = threadIdx.x;

  auto fill = [&](int c) {
    if (c < nchunks) {
      const int s = c % NST;
      // A: per plane, per 8-row group, the 2 core matrices of K-chunk c (256 B)
      float* sa = stage_a(rg, s);
      const int groups = MT / 8;
      const int pieces = 4 * groups * 16;  // 16-byte pieces
      for (int i = tid; i < pieces; i += blockDim.x) {
        const int p = i / (groups * 16), rem = i - p * groups * 16;
        const int g = rem >> 4, w = rem & 15;
        const float* src = Ag + p * plane + ((size_t)g * (KD / 4) + 2 * c) * 32 + w * 4;
        cp_async16(sa + p * (MT * KC) + g * 64 + w * 4, src);
      }
      // B: 8 x N tile of chunk c, split hi/lo into K-major planes (N rows x 8)
      float* sb = stage_b(rg, s);
      for (int i = tid; i < N * KC; i += blockDim.x) {
        const int q = i / KC, kk = i - q * KC;
        const int k = c * KC + kk;
        const uint32_t o = umma::cm_offset(q, kk, KC) >> 2;
        float hi, lo;
        umma::split_tf32(Br[k * ldb + q], hi, lo);
        sb[o] = hi;
        sb[2 * N * KC + o] = lo;
        umma::split_tf32(Bi[k * ldb + q], hi, lo);
        sb[N * KC + o] = hi;
        sb[3 * N * KC + o] = lo;
      }
    }
    cp_async_commit();
  };

  const uint32_t id_pos = umma::make_idesc_tf32(tm, N, false, false, false, false);
  const uint32_t id_neg = umma::make_idesc_tf32(tm, N, false, false, false, true);
  const uint32_t sbo_a = (KC / 4) * 128, sbo_b = (KC / 4) * 128;

  // mbarrier bookkeeping: iss[s] = commits issued on stage s so far (all
  // threads track identically; persisted in rg.uses between calls); pend[s] =
  // the latest commit of s has not been waited yet.  Completion k of an
  // mbarrier has parity k & 1; every commit is waited exactly once, in order.
  uint32_t iss[NST];
  bool pend[NST];
#pragma unroll
  for (int q = 0; q < NST; ++q) {
    iss[q] = rg.uses[q];
    pend[q] = false;
  }
  __syncthreads();  // every thread has read rg.uses before thread 0 rewrites it

#pragma unroll 1
  for (int c = 0; c < NST - 1; ++c) fill(c);
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % NST;
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NST - 2) : "memory");
    umma::fence_proxy_async();  // cp.async / st.shared writes -> tensor-core (async proxy)
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      const uint32_t a0 = umma::smem_u32(stage_a(rg, s));
      const uint32_t b0 = umma::smem_u32(stage_b(rg, s));
      const uint32_t pa = (uint32_t)MT * KC * 4, pb = (uint32_t)N * KC * 4;  // plane bytes
      uint64_t bd[4];  // re_hi, im_hi, re_lo, im_lo
#pragma unroll
      for (int q = 0; q < 4; ++q) bd[q] = umma::make_sdesc(b0 + q * pb, 128, sbo_b);
      const uint32_t idA = sA < 0.f ? id_neg : id_pos;
      const uint32_t idB = sB < 0.f ? id_neg : id_pos;
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t at = a0 + (uint32_t)t * (tm / 8) * sbo_a;  // first row group of tile t
        const uint64_t ar_hi = umma::make_sdesc(at, 128, sbo_a);
        const uint64_t ai_hi = umma::make_sdesc(at + pa, 128, sbo_a);
        const uint64_t ar_lo = umma::make_sdesc(at + 2 * pa, 128, sbo_a);
        const uint64_t ai_lo = umma::make_sdesc(at + 3 * pa, 128, sbo_a);
        const uint32_t dre = rg.tmem + (uint32_t)(2 * N * t);
        const uint32_t dim = dre + (uint32_t)N;
        const uint32_t first = (c == 0) ? 0u : 1u;
        // D_re += A_re B_re + sA A_im B_im      (3xTF32 per real product)
        umma::mma_tf32(dre, ar_hi, bd[0], id_pos, first);
        umma::mma_tf32(dre, ar_hi, bd[2], id_pos, 1u);
        umma::mma_tf32(dre, ar_lo, bd[0], id_pos, 1u);
        umma::mma_tf32(dre, ai_hi, bd[1], idA, 1u);
        umma::mma_tf32(dre, ai_hi, bd[3], idA, 1u);
        umma::mma_tf32(dre, ai_lo, bd[1], idA, 1u);
        // D_im += A_re B_im + sB A_im B_re
        umma::mma_tf32(dim, ar_hi, bd[1], id_pos, first);
        umma::mma_tf32(dim, ar_hi, bd[3], id_pos, 1u);
        umma::mma_tf32(dim, ar_lo, bd[1], id_pos, 1u);
        umma::mma_tf32(dim, ai_hi, bd[0], idB, 1u);
        umma::mma_tf32(dim, ai_hi, bd[2], idB, 1u);
        umma::mma_tf32(dim, ai_lo, bd[0], idB, 1u);
      }
      umma::commit(&rg.mbar[s]);
    }
    iss[s] += 1;
    pend[s] = true;
    // refill the stage chunk c-1 used once its MMAs have drained
    const int nxt = c + NST - 1;
    if (nxt < nchunks) {
      const int sp = nxt % NST;
      if (pend[sp]) {
        umma::mbar_wait(&rg.mbar[sp], (iss[sp] - 1u) & 1u);
        pend[sp] = false;
      }
    }
    fill(nxt);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
  for (int q = 0; q < NST; ++q)
    if (pend[q]) umma::mbar_wait(&rg.mbar[q], (iss[q] - 1u) & 1u);
  umma::fence_after();
  __syncthreads();
  if (tid == 0)
#pragma unroll
    for (int q = 0; q < NST; ++q) rg.uses[q] = iss[q];
  __syncthreads();
}

// Epilogue traversal of the TMEM accumulator written by gemm(): calls
// f(row, col, part, value) for every element (part 0 = re, 1 = im).  Warp w
// reads TMEM lane quadrant (w & 3) and part (w >> 2) (8 warps).
template <class F>
__device__ __forceinline__ void for_each_d(const Ring& rg, int MT, int N, F f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, part = (warp >> 2) & 1;
  const int tm = MT >= 128 ? 128 : 64;
  const int ntiles = MT / tm;
  for (int t = 0; t < ntiles; ++t) {
    const uint32_t base = rg.tmem + (uint32_t)(2 * N * t + part * N) + ((uint32_t)(32 * quad) << 16);
    int row;
    if (tm == 128)
      row = 128 * t + 32 * quad + lane;
    else
      row = lane < 16 ? 64 * t + 16 * quad + lane : -1;  // M = 64: lanes 0-15 of each quadrant
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      umma::tmem_ld16(base + c0, v);
      if (row >= 0)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < N) f(row, c0 + j, part, v[j]);
    }
  }
}

}  // namespace tcg
}  // namespace ammmse
