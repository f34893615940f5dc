// tc_stream.cuh — the cluster engine's tensor-core GEMM (tcgen05.mma
// kind::tf32, 3xTF32 split, fp32 accumulators in TMEM), used for both A-MMMSE
// contractions of a CTA's column slice (weighted_gram /
// pgd_precoder_step objective.py:172-193, solvers.py:358-377, and the G = H V
// products behind update_receivers / weighted_sum_rate):
//   GEMM-B  G  = H X          A = H     (KN x M,  K = M)     B = X  (own columns)
//   GEMM-A  ∇' = H^H Ŷ        A = H^T   (M x KN,  K = KN)    B = Ŷ  (own columns)
//
// A: four fp32 planes (re_hi, im_hi, re_lo, im_lo) of H / H^T, split once per
//    realization into a per-cluster global slot in CHUNK-MAJOR order (chunk =
//    one 8-wide UMMA K-step of all four planes, canonical K-major no-swizzle
//    core-matrix layout), so each ring stage is ONE contiguous bulk copy
//    (cp.async.bulk, SASS UBLKCP) completing on the stage's "full" mbarrier.
// B: the 8 x ncol complex slice of the fp32 operand for the chunk is split by
//    all threads into one K-major matrix of 4*ncol rows
//        [B_re_hi ; B_im_hi ; B_re_lo ; B_im_lo]
//    so that per K-step and M tile four MMAs cover the 3xTF32 complex product:
//        D1[0:4n] += A_re_hi · B          D1[0:2n] += A_re_lo · B_hi
//        D2[0:4n] += A_im_hi · B          D2[0:2n] += A_im_lo · B_hi
//    (n = ncol; the hi·hi, hi·lo, lo·hi terms of each real product land in
//    separate column groups and are summed in the epilogue).
// Producer warps fill the ring up to S chunks ahead (A by bulk copy, B split
// by the warps); one thread issues the MMAs as soon as a stage is complete and
// commits them to the stage's "done" mbarrier, which frees it for the chunk S
// ahead.  Stage / phase bookkeeping uses one chunk sequence number all threads
// advance identically.
//
// K-major only: MN-major kind::tf32 operands read back as zeros in the round-1
// probe, so H and H^T are pre-split separately.
#pragma once

#include "tc_umma.cuh"

namespace ammmse {
namespace tcs {

constexpr int KW = 8;  // K per ring stage = one tf32 UMMA K-step

// byte offset of (row, kk) inside one K-step block of a K-major matrix
// (8-row groups of two 128-byte core matrices; LBO = 128, SBO = 256)
__host__ __device__ __forceinline__ uint32_t kstep_offset(int row, int kk) {
  return (uint32_t)(((row >> 3) * 2 + (kk >> 2)) * 128 + (row & 7) * 16 + (kk & 3) * 4);
}

// Accumulator sets of a gemm() call: 2 when both fit the 512 TMEM columns
// (8 ncol columns per 128-row tile and set), else 1.
__host__ __device__ __forceinline__ int accum_sets(int ncol, int nmt, int nch) {
  return (2 * 8 * ncol * nmt <= 512 && nch >= 2) ? 2 : 1;
}

struct Pipe {
  unsigned char* ring;  // S stages of stage_bytes, 128-byte aligned
  int S;
  int stage_bytes;
  int a_bytes;          // A part of a stage (4 planes x max rows x KW floats)
  uint64_t* full;       // S mbarriers (count 1 + tx): A chunk landed
  uint64_t* bready;     // S mbarriers (count 1: the producing warp): B slice written
  uint64_t* done;       // S mbarriers (count 1, tcgen05.commit): the stage's MMAs completed
  uint64_t* fin;        // 1 mbarrier (count 1, tcgen05.commit): all MMAs of a gemm() call completed
  uint32_t tmem;        // TMEM base address
};

// Pipeline position, identical in every thread: chunks issued and gemm() calls
// made so far.  An mbarrier wait must never target a phase more than one ahead
// of the barrier's current phase (try_wait.parity would pass immediately), so
// threads that do not follow the chunk sequence wait on `fin`, which completes
// exactly once per call.
struct Seq {
  uint32_t chunk = 0;
  uint32_t call = 0;
};

__device__ __forceinline__ unsigned char* stage_a(const Pipe& p, int s) {
  return p.ring + (size_t)s * p.stage_bytes;
}
__device__ __forceinline__ unsigned char* stage_b(const Pipe& p, int s) {
  return stage_a(p, s) + p.a_bytes;
}

// Per-realization split of H (KN x M, interleaved complex, global) into the
// chunk-major planes of A for GEMM-B (transpose = false: rows r, K = m) or
// GEMM-A (transpose = true: rows m, K = r).  Threads of all CTAs of the
// cluster split rows [r0, r1) of H.
__device__ __forceinline__ void split_h(const float2* __restrict__ Hg, int KN, int M, bool transpose,
                                        float* __restrict__ dst, int r0, int r1) {
  const int rows = transpose ? M : KN;
  const size_t chunk = (size_t)4 * rows * KW;  // floats per chunk (4 planes)
  const size_t plane = (size_t)rows * KW;
  for (int i = r0 * M + (int)threadIdx.x; i < r1 * M; i += blockDim.x) {
    const int r = i / M, m = i - r * M;
    const float2 h = Hg[i];
    const int row = transpose ? m : r, k = transpose ? r : m;
    float* c = dst + (size_t)(k / KW) * chunk + (kstep_offset(row, k % KW) >> 2);
    float hi, lo;
    umma::split_tf32(h.x, hi, lo);
    c[0] = hi;
    c[2 * plane] = lo;
    umma::split_tf32(h.y, hi, lo);
    c[plane] = hi;
    c[3 * plane] = lo;
  }
}

// D = A · B over K = KD (multiple of KW) for `nmt` M tiles of `tm` rows
// (tm = 128, or 64 with nmt = 1).  Called by ALL threads of the CTA; warp
// specialised, no block barrier per chunk:
//   * producer warps (the upper half of the block) fill chunks round robin, up
//     to S chunks ahead: a warp waits for the stage's previous MMAs (done[s]),
//     its lane 0 issues the A bulk copy (full[s], tx-count), the warp splits
//     the B slice into the stage and arrives on bready[s];
//   * thread 0 waits full[s] and bready[s], issues the chunk's MMAs and
//     commits them to done[s];
//   * everyone finally waits for the last chunk's MMAs.
//   Ag    : chunk-major pre-split planes of A (global), rows = nmt * tm
//   Br/Bi : fp32 planar B (shared), element (k, q) at k * ldb + q, ncol columns
//   sq    : pipeline position (identical in every thread), advanced by KD / KW chunks
// Accumulators of tile t: D1 at columns [8n t, 8n t + 4n), D2 at [8n t + 4n, 8n (t+1)).
// DBG (diagnostics, bench_gemmstep --ablate): bit 0 skips the A bulk copies,
// bit 1 the B split, bit 2 the MMAs (their commits still flow).
template <int DBG = 0>
__device__ __forceinline__ void gemm(const Pipe& p, Seq& sq, const float* __restrict__ Ag,
                                     int tm, int nmt, int KD, int ncol, const float* __restrict__ Br,
                                     const float* __restrict__ Bi, int ldb) {
  const uint32_t seq = sq.chunk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pw0 = (int)(blockDim.x >> 6);  // first producer warp (upper half of the block)
  const int nch = KD / KW;
  const int rows = tm * nmt;
  const uint32_t a_chunk = (uint32_t)(4 * rows * KW * 4);  // bytes per A chunk
  const uint32_t a_plane = (uint32_t)(rows * KW * 4);
  const int n4 = 4 * ncol;
  const uint32_t S = (uint32_t)p.S;
  const int nsets = accum_sets(ncol, nmt, nch);

  if (warp >= pw0) {  // ---- producers: warp w fills chunks c = w - pw0 (mod #producer warps) ----
    const int nw = (int)(blockDim.x >> 5) - pw0;
    if (lane == 0) umma::fence_proxy_async();  // earlier generic accesses of the ring -> TMA writes
    for (int c = warp - pw0; c < nch; c += nw) {
      const uint32_t q = seq + (uint32_t)c;
      const int s = (int)(q % S);
      const uint32_t use = q / S;
      // stage s free (its previous MMAs done).  The chunk S before on this stage
      // was filled by this same warp iff nw divides S, so the wait never runs
      // more than one phase ahead (S a multiple of nw).
      if (use > 0) umma::mbar_wait(&p.done[s], (use - 1u) & 1u);
      if (lane == 0) {
        if (DBG & 1) {
          umma::mbar_arrive(&p.full[s]);
        } else {
          umma::mbar_arrive_expect_tx(&p.full[s], a_chunk);
          umma::bulk_g2s(stage_a(p, s), reinterpret_cast<const unsigned char*>(Ag) + (size_t)c * a_chunk,
                         a_chunk, &p.full[s]);
        }
      }
      // B slice: rows k = c*KW .. +KW of the planar operand, split hi/lo into
      // the stage's K-major [re_hi; im_hi; re_lo; im_lo] matrix
      float* sb = reinterpret_cast<float*>(stage_b(p, s));
      const int k0 = c * KW;
      for (int i = lane; i < ((DBG & 2) ? 0 : KW * ncol); i += 32) {
        const int kk = i / ncol, qq = i - kk * ncol;
        float hi, lo;
        umma::split_tf32(Br[(k0 + kk) * ldb + qq], hi, lo);
        sb[kstep_offset(qq, kk) >> 2] = hi;
        sb[kstep_offset(2 * ncol + qq, kk) >> 2] = lo;
        umma::split_tf32(Bi[(k0 + kk) * ldb + qq], hi, lo);
        sb[kstep_offset(ncol + qq, kk) >> 2] = hi;
        sb[kstep_offset(3 * ncol + qq, kk) >> 2] = lo;
      }
      umma::fence_proxy_async();  // generic st.shared -> tensor-core (async proxy) reads
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&p.bready[s]);
    }
  } else if (tid == 0) {  // ---- MMA issuer ----
    const uint32_t id_all = umma::make_idesc_tf32(tm, n4, false, false, false, false);
    const uint32_t id_hi = umma::make_idesc_tf32(tm, 2 * ncol, false, false, false, false);
    for (int c = 0; c < nch; ++c) {
      const uint32_t q = seq + (uint32_t)c;
      const int s = (int)(q % S);
      const uint32_t par = (q / S) & 1u;
      umma::mbar_wait(&p.full[s], par);
      umma::mbar_wait(&p.bready[s], par);
      umma::fence_after();
      const uint32_t a0 = umma::smem_u32(stage_a(p, s));
      const uint64_t bd = umma::make_sdesc(umma::smem_u32(stage_b(p, s)), 128, 256);
      // chunk c accumulates into set c % nsets (split accumulation: the tensor
      // core's fp32 accumulation error grows with the chain; the sets are
      // summed in fp32 by the epilogue)
      const int set = c % nsets;
      const uint32_t acc = c >= nsets ? 1u : 0u;
      for (int t = 0; t < ((DBG & 4) ? 0 : nmt); ++t) {
        const uint32_t at = a0 + (uint32_t)t * (uint32_t)(tm / 8) * 256u;
        const uint32_t d1 = p.tmem + (uint32_t)(8 * ncol * (t + nmt * set));
        const uint32_t d2 = d1 + (uint32_t)n4;
        umma::mma_tf32(d1, umma::make_sdesc(at, 128, 256), bd, id_all, acc);              // re_hi
        umma::mma_tf32(d1, umma::make_sdesc(at + 2 * a_plane, 128, 256), bd, id_hi, 1u);  // re_lo
        umma::mma_tf32(d2, umma::make_sdesc(at + a_plane, 128, 256), bd, id_all, acc);    // im_hi
        umma::mma_tf32(d2, umma::make_sdesc(at + 3 * a_plane, 128, 256), bd, id_hi, 1u);  // im_lo
      }
      umma::commit(&p.done[s]);
    }
    umma::commit(p.fin);
  }
  umma::mbar_wait(p.fin, sq.call & 1u);
  // warp 0 diverged (lane 0 issued the MMAs): reconverge before the epilogue's
  // warp-collective tcgen05.ld.sync.aligned
  __syncwarp();
  umma::fence_after();
  sq.chunk += (uint32_t)nch;
  sq.call += 1;
}

// Reference schedule of gemm() (diagnostics / A-B): every thread splits the B
// slice, one block barrier per chunk, thread 0 issues.  Same results.
__device__ __forceinline__ void gemm_sync(const Pipe& p, Seq& sq, const float* __restrict__ Ag,
                                          int tm, int nmt, int KD, int ncol,
                                          const float* __restrict__ Br, const float* __restrict__ Bi,
                                          int ldb) {
  const uint32_t seq = sq.chunk;
  const int tid = threadIdx.x;
  const int nch = KD / KW;
  const int rows = tm * nmt;
  const uint32_t a_chunk = (uint32_t)(4 * rows * KW * 4);
  const uint32_t a_plane = (uint32_t)(rows * KW * 4);
  const int n4 = 4 * ncol;
  const uint32_t S = (uint32_t)p.S;
  const int nsets = accum_sets(ncol, nmt, nch);
  const uint32_t id_all = umma::make_idesc_tf32(tm, n4, false, false, false, false);
  const uint32_t id_hi = umma::make_idesc_tf32(tm, 2 * ncol, false, false, false, false);
  auto produce = [&](int c) {
    const uint32_t q = seq + (uint32_t)c;
    const int s = (int)(q % S);
    const uint32_t use = q / S;
    if (use > 0) umma::mbar_wait(&p.done[s], (use - 1u) & 1u);
    if (tid == 0) {
      umma::mbar_arrive_expect_tx(&p.full[s], a_chunk);
      umma::bulk_g2s(stage_a(p, s), reinterpret_cast<const unsigned char*>(Ag) + (size_t)c * a_chunk,
                     a_chunk, &p.full[s]);
    }
    float* sb = reinterpret_cast<float*>(stage_b(p, s));
    const int k0 = c * KW;
    for (int i = tid; i < KW * ncol; i += blockDim.x) {
      const int kk = i / ncol, qq = i - kk * ncol;
      float hi, lo;
      umma::split_tf32(Br[(k0 + kk) * ldb + qq], hi, lo);
      sb[kstep_offset(qq, kk) >> 2] = hi;
      sb[kstep_offset(2 * ncol + qq, kk) >> 2] = lo;
      umma::split_tf32(Bi[(k0 + kk) * ldb + qq], hi, lo);
      sb[kstep_offset(ncol + qq, kk) >> 2] = hi;
      sb[kstep_offset(3 * ncol + qq, kk) >> 2] = lo;
    }
    umma::fence_proxy_async();
  };
  const int pre = nch < p.S - 1 ? nch : p.S - 1;
  for (int c = 0; c < pre; ++c) produce(c);
  for (int c = 0; c < nch; ++c) {
    __syncthreads();
    if (tid == 0) {
      const uint32_t q = seq + (uint32_t)c;
      const int s = (int)(q % S);
      umma::mbar_wait(&p.full[s], (q / S) & 1u);
      umma::fence_after();
      const uint32_t a0 = umma::smem_u32(stage_a(p, s));
      const uint64_t bd = umma::make_sdesc(umma::smem_u32(stage_b(p, s)), 128, 256);
      // chunk c accumulates into set c % nsets (split accumulation: the tensor
      // core's fp32 accumulation error grows with the chain; the sets are
      // summed in fp32 by the epilogue)
      const int set = c % nsets;
      const uint32_t acc = c >= nsets ? 1u : 0u;
      for (int t = 0; t < nmt; ++t) {
        const uint32_t at = a0 + (uint32_t)t * (uint32_t)(tm / 8) * 256u;
        const uint32_t d1 = p.tmem + (uint32_t)(8 * ncol * (t + nmt * set));
        const uint32_t d2 = d1 + (uint32_t)n4;
        umma::mma_tf32(d1, umma::make_sdesc(at, 128, 256), bd, id_all, acc);
        umma::mma_tf32(d1, umma::make_sdesc(at + 2 * a_plane, 128, 256), bd, id_hi, 1u);
        umma::mma_tf32(d2, umma::make_sdesc(at + a_plane, 128, 256), bd, id_all, acc);
        umma::mma_tf32(d2, umma::make_sdesc(at + 3 * a_plane, 128, 256), bd, id_hi, 1u);
      }
      umma::commit(&p.done[s]);
      if (c == nch - 1) umma::commit(p.fin);
    }
    if (c + p.S - 1 < nch) produce(c + p.S - 1);
  }
  umma::mbar_wait(p.fin, sq.call & 1u);
  umma::fence_after();
  sq.chunk += (uint32_t)nch;
  sq.call += 1;
}

// Epilogue traversal of the accumulators gemm() left in TMEM: f(row, q, re, im)
// for every row < rows of the nmt tiles and q < ncol, where
//   conj_a = false:  (re, im) of  A · B
//   conj_a = true :  (re, im) of  conj(A) · B   (A = H^T planes give H^H · B)
// Warp w reads TMEM lane quadrant (w & 3); warps w >> 2 split the columns in
// blocks of 16.  Ends with tcgen05.fence::before_thread_sync.
template <class F>
__device__ __forceinline__ void for_each(const Pipe& p, int tm, int nmt, int ncol, int KD, bool conj_a,
                                         F f) {
  const int nsets = accum_sets(ncol, nmt, KD / KW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, cgrp = warp >> 2, ngrp = (int)(blockDim.x >> 7);
  for (int t = 0; t < nmt; ++t) {
    int row;
    if (tm == 128)
      row = 128 * t + 32 * quad + lane;
    else
      row = lane < 16 ? 16 * quad + lane : -1;  // M = 64: lanes 0-15 of each quadrant
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    for (int q0 = 16 * cgrp; q0 < ncol; q0 += 16 * ngrp) {
      float prr[16], pri[16], pir[16], pii[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) prr[j] = pri[j] = pir[j] = pii[j] = 0.f;
      for (int set = 0; set < nsets; ++set) {
        const uint32_t d1 = p.tmem + lane_base + (uint32_t)(8 * ncol * (t + nmt * set));
        const uint32_t d2 = d1 + (uint32_t)(4 * ncol);
        uint32_t rr_h[16], ri_h[16], rr_l[16], ri_l[16], ir_h[16], ii_h[16], ir_l[16], ii_l[16];
        umma::tmem_ld16_nw(d1 + q0, rr_h);
        umma::tmem_ld16_nw(d1 + ncol + q0, ri_h);
        umma::tmem_ld16_nw(d1 + 2 * ncol + q0, rr_l);
        umma::tmem_ld16_nw(d1 + 3 * ncol + q0, ri_l);
        umma::tmem_ld16_nw(d2 + q0, ir_h);
        umma::tmem_ld16_nw(d2 + ncol + q0, ii_h);
        umma::tmem_ld16_nw(d2 + 2 * ncol + q0, ir_l);
        umma::tmem_ld16_nw(d2 + 3 * ncol + q0, ii_l);
        umma::tmem_wait_ld();
        auto asf = [](uint32_t u) { return __uint_as_float(u); };
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          prr[j] += asf(rr_h[j]) + asf(rr_l[j]);
          pri[j] += asf(ri_h[j]) + asf(ri_l[j]);
          pir[j] += asf(ir_h[j]) + asf(ir_l[j]);
          pii[j] += asf(ii_h[j]) + asf(ii_l[j]);
        }
      }
      if (row >= 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (conj_a)
            f(row, q0 + j, prr[j] + pii[j], pri[j] - pir[j]);
          else
            f(row, q0 + j, prr[j] - pii[j], pri[j] + pir[j]);
        }
      }
    }
  }
  umma::fence_before();
}

}  // namespace tcs
}  // namespace ammmse
