// ammmse_tc2.cuh — second-generation tensor-core cluster engine (tcgen05
// kind::tf32, 3xTF32) for realizations whose GEMMs fill 128-row UMMA tiles
// (BASELINE large: M = KN = 128, N = d = 4).  Same A-MMMSE semantics as
// ammmse_cluster.cuh (reference solvers.py:415-518, objective.py:172-213);
// what changes is where the operands live and how the GEMMs are fed:
//
//   * B operand (Ŷ for GEMM-A, X for GEMM-B): written ALREADY SPLIT (tf32 hi /
//     lo, K-major core-matrix order, all K of the GEMM) by its producer — the Ŷ
//     build and the GEMM-A epilogue — into one shared-memory buffer.  The MMA
//     loop has no per-chunk operand work and no "B ready" handshakes.
//   * A operand (pre-split H / H^T planes, global, L2 resident): streamed by ONE
//     producer thread through an S-stage bulk-copy ring (cp.async.bulk, SASS
//     UBLKCP, mbarrier complete_tx).  H does not change during a solve, so the
//     producer runs ahead ACROSS GEMM calls: while a GEMM's last chunks drain
//     and its epilogue runs, the first S chunks of the next GEMM are in flight.
//   * Precoders live in TMEM (lane = antenna row m): X_cur and X_old as fp32
//     columns next to the accumulators, read with tcgen05.ld and rewritten with
//     tcgen05.st by the one-thread-per-row epilogue.  No V in shared memory, no
//     V_old slot in global memory.
//   * Projection is lazy: TMEM holds the unprojected X, the precoders are
//     s · X; GEMM-B multiplies X and its epilogue applies s, so the tensor core
//     starts on G = H X while the cluster still sums ‖X‖².
//   * 3xTF32 by K concatenation: D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi into the
//     same accumulator (6 MMAs of N = 2·ncol per chunk and tile), two
//     accumulator sets alternating by chunk: 4 TMEM loads per set and 16
//     columns in the epilogue.
#pragma once

#include <type_traits>

#include "ammmse_cluster.cuh"
#include "user_algebra_quad.cuh"

namespace ammmse {
namespace tc2 {

constexpr int KW = 8;          // K per chunk = one tf32 UMMA K-step
constexpr int kPerm = 3;       // permanent A ring stages (they also hold the chunks prefetched across GEMMs)
constexpr int kVol = 3;        // volatile stages in the two G buffers (dead during the MMA loops): 2 + 1
// An EVEN number of stages: chunk c uses stage c % kStages, so the chunks of even
// and of odd index (two producer / MMA warp pairs, see gemm) never share a stage
// and each pair is an in-order pipeline of its own.  (With 7 stages a warp could
// poll a barrier two phases ahead of a lagging pair: parity aliasing.)
constexpr int kStages = kPerm + kVol;
static_assert(kStages % 2 == 0, "even / odd chunk pipelines must not share stages");
constexpr int kMaxStages = kStages;
constexpr int kBPad = 32;      // bytes between B chunks (bank spread of the per-row epilogue stores)
constexpr int kThreads = 256;

// shape rules: 128-row UMMA tiles, N = 2 ncol in multiples of 16, 16-column
// epilogue blocks, accumulators + precoders within the 512 TMEM columns
// TMEM columns: accumulator sets (4 ncol each), X_cur / X_old (2 ncol each), G_old (2 ncol)
__host__ __device__ inline int tmem_sets(int M, int KN, int ncol) {
  const int nmtA = M / 128, nmtB = KN / 128, nmt = nmtA > nmtB ? nmtA : nmtB;
  const int v = 2 * nmtA * 2 * ncol + nmtB * 2 * ncol;
  if (2 * nmt * 4 * ncol + v <= 512) return 2;
  if (nmt * 4 * ncol + v <= 512) return 1;
  return 0;
}
// one 128-row tile per GEMM (M = KN = 128: every GEMM call streams the same
// number of equally sized A chunks), each G buffer large enough for two A chunks
__host__ __device__ inline bool shape_ok(int M, int KN, int ncol) {
  if (M != 128 || KN != 128 || ncol % 16 || 2 * ncol > 256) return false;
  if ((size_t)2 * KN * (ncol + 1) * 4 < (size_t)2 * 4 * 128 * KW * 4) return false;
  return tmem_sets(M, KN, ncol) > 0;
}

template <int NN, int DD>
struct T2Layout {
  int M, K, C, KL, KN, ncol, ldg, S;
  int nmtA, nmtB, nmt, nsets;
  int a_stage;   // bytes of one A ring stage (4 planes x max(M, KN) rows x KW floats)
  int b_chunk;   // bytes between consecutive B chunks (4 ncol rows x KW floats + pad)
  int acc_cols;  // TMEM columns of the accumulators; the precoders, then G_old follow
  int v_cols;
  size_t nG;     // floats per G plane
  size_t oRing, oB, oG0, oG1, oP, oD, oGk, dbl_off, bytes;  // byte offsets

  __host__ __device__ void init(int M_, int K_, int C_, int S_) {
    M = M_;
    K = K_;
    C = C_;
    S = S_;
    KL = K / C;
    KN = K * NN;
    ncol = KL * DD;
    ldg = ncol + 1;  // odd row stride: one-thread-per-row sweeps are conflict free
    nmtA = M / 128;
    nmtB = KN / 128;
    nmt = nmtA > nmtB ? nmtA : nmtB;
    nsets = tmem_sets(M, KN, ncol);
    acc_cols = nsets * nmt * 4 * ncol;
    v_cols = 2 * nmtA * 2 * ncol;
    const int rows = KN > M ? KN : M;
    a_stage = 4 * rows * KW * 4;
    b_chunk = 4 * ncol * KW * 4 + kBPad;
    nG = (size_t)KN * ldg;
    oRing = 0;
    oB = oRing + (size_t)kPerm * a_stage;
    oG0 = oB + (size_t)(rows / KW) * b_chunk;
    oG0 = (oG0 + 15) & ~(size_t)15;
    oG1 = oG0 + 2 * nG * 4;
    oP = (oG1 + 2 * nG * 4 + 15) & ~(size_t)15;  // RC<float>[K*NN*NN]: M_k = α U W U^H of every user
    oD = oP + (size_t)K * NN * NN * 8;           // RC<float>[KL*NN*DD]
    oGk = oD + (size_t)KL * NN * DD * 8;         // float[2][KL*NN*DD]: saved diagonal blocks of G_new
    dbl_off = (oGk + (size_t)KL * NN * DD * 8 + 15) & ~(size_t)15;
    bytes = dbl_off + dbl_count() * sizeof(double);
  }
  // fp64 region: as CLayout (gx[2], ucache[2], wcache[2], lndetw[2], 7 per-user
  // arrays, exchange slots, split-K1 exchange, reduction scratch)
  __host__ __device__ size_t k1w_count() const {
    if (NN == 4 && DD == 4) return (size_t)KL * quad::kScratch;  // quad-lane K1 (user_algebra_quad.cuh)
    return (NN == 2 && DD == 2) ? 0 : (size_t)KL * (2 * DD * DD + NN + 1);
  }
  __host__ __device__ size_t wsr_count() const {
    return (NN == 4 && DD == 4) ? (size_t)KL * quad::kWsrScratch : 0;  // two-warp WSR (wsr_users_a / _c)
  }
  __host__ __device__ size_t dbl_count() const {
    return (size_t)2 * 2 * K * NN * NN + 2 * 2 * KL * NN * DD + 2 * 2 * KL * DD * DD + 9 * KL +
           XS_COUNT + k1w_count() + wsr_count() + 32;
  }
};

// kPerm (permanent ring stages) if the layout fits `limit` bytes, else 0
template <int NN, int DD>
__host__ inline int pick_stages(int M, int K, int C, size_t limit) {
  T2Layout<NN, DD> L;
  L.init(M, K, C, kPerm);
  return L.bytes <= limit ? kPerm : 0;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// mbarrier / bulk-copy primitives on precomputed 32-bit shared addresses
__device__ __forceinline__ void mbar_wait_spin_u32(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}\n"
        : "=r"(ok)
        : "r"(mbar), "r"(parity)
        : "memory");
  } while (!ok);
}
// one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}
// One chunk x tile of the 3xTF32 complex product on an elected lane,
//   D1 (+)= A_re_hi B_hi + A_re_hi B_lo + A_re_lo B_hi     D2 likewise with A_im,
// fused with a test_wait of barrier `poll_bar` issued BEFORE the MMAs whose
// result is read after them and after the commit to `done_bar` (every one of
// these operations costs the issuing warp 100+ cycles when waited on one by
// one).  Called by the whole (converged) warp.
__device__ __forceinline__ uint32_t mma6_poll(uint32_t d1, uint32_t d2, uint64_t a_rh, uint64_t a_ih,
                                              uint64_t a_rl, uint64_t a_il, uint64_t bhi, uint64_t blo,
                                              uint32_t idesc, uint32_t acc, uint32_t poll_bar,
                                              uint32_t poll_parity, uint32_t enable, uint32_t done_bar) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred Pn, Pe, Pa, Pt;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 Pn, [%11], %12;\n\t"
      "elect.sync _|Pe, 0xffffffff;\n\t"
      "setp.ne.b32 Pt, %13, 0;\n\t"
      "and.pred Pe, Pe, Pt;\n\t"
      "setp.ne.b32 Pa, %10, 0;\n\t"
      "setp.eq.b32 Pt, 0, 0;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %7, %9, Pa;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %8, %9, Pt;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %7, %9, Pt;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%2], %4, %7, %9, Pa;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%2], %4, %8, %9, Pt;\n\t"
      "@Pe tcgen05.mma.cta_group::1.kind::tf32 [%2], %6, %7, %9, Pt;\n\t"
      "elect.sync _|Pe, 0xffffffff;\n\t"
      "@Pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%14];\n\t"
      "selp.u32 %0, 1, 0, Pn;\n\t"
      "}\n"
      : "=r"(ok)
      : "r"(d1), "r"(d2), "l"(a_rh), "l"(a_ih), "l"(a_rl), "l"(a_il), "l"(bhi), "l"(blo), "r"(idesc),
        "r"(acc), "r"(poll_bar), "r"(poll_parity), "r"(enable), "r"(done_bar)
      : "memory");
  return ok;
}
__device__ __forceinline__ uint32_t mbar_test_u32(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "}\n"
      : "=r"(ok)
      : "r"(mbar), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_u32(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void commit_u32(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar)
               : "memory");
}

// Pipeline state.  A GEMM call streams its A chunks c = 0, 1, ... through stage
// c % kStages; chunks 0 .. have-1 were prefetched (into the permanent stages)
// by the previous call.  Per-stage barrier phases are tracked as bit masks:
// bit s of `cm` = parity of the consumptions of stage s so far (MMA warp), of
// `pm` = parity of its fills, `ever` = filled at least once (producer warp).
struct Pipe {
  unsigned char* ring;  // kPerm permanent stages
  unsigned char* vol0;  // volatile stages kPerm, kPerm + 1 (G buffer N)
  unsigned char* vol1;  // volatile stages kPerm + 2, kPerm + 3 (G buffer E)
  unsigned char* bfull;
  uint32_t a_stage, b_chunk;
  uint64_t* full;  // kStages mbarriers (count 1 + tx): A chunk landed
  uint64_t* done;  // kStages mbarriers (count 1): the chunk's MMAs completed (tcgen05.commit)
  uint64_t* fin;   // 1 mbarrier: all MMAs of a gemm() call completed
  uint32_t tmem;
  uint32_t have = 0;  // chunks of the next call already issued
  uint32_t cm = 0, pm = 0, ever = 0;
  uint32_t call = 0;
  int dbg = 0;  // diagnostics (AMMMSE_PHASES builds): bit 0 skips the A copies, bit 1 the MMAs
  unsigned long long* prof = nullptr;  // diagnostics: phase counters (AMMMSE_PHASES >= 2)
};

constexpr int kMmaWarp = 0, kMmaWarp2 = 2;  // (different SM sub-partitions)
constexpr int kProducerWarp = 1, kProducerWarp2 = 3;

// D = A · B over nch chunks of K (all threads call).  A = planes Ag of 128
// rows; B = the split operand in p.bfull (ncol columns); accumulators of set s at
// TMEM column s * 4 ncol: D1 = A_re · [B_re | B_im] at +0, D2 = A_im · [B_re | B_im]
// at +2 ncol.  After its own chunks the producer prefetches the first kPerm
// chunks of the next GEMM (next_Ag; nullptr = none) into the permanent stages.
// Returns after all MMAs completed; the volatile stages (the G buffers) are
// free again.
//
// Role warps: warp-UNIFORM control flow (all 32 lanes run the loops and poll the
// barriers; only the tcgen05 / bulk-copy instructions are predicated on an
// elected lane), so the compiler keeps addresses and descriptors in uniform
// registers.  Under a divergent `if (lane == 0)` every UTCHMMA is wrapped in an
// ELECT / R2UR waterfall loop (measured: ~100 cycles per MMA).  Every other warp
// parks at the block barrier.  Measured on B200 (exp/ubench): an mbarrier
// test_wait or arrive costs ~100 cycles of thread time, tcgen05.commit -> arrival
// 237 cycles, a 16 KB bulk copy 520-700 cycles of latency (83 B/clk back to
// back): a stage turns around in ~1.1 k cycles, which a 3-stage ring cannot hide
// behind ~300 cycles of MMAs per chunk — hence the 7 stages.
struct NoSide {
  __device__ __forceinline__ void operator()() const {}
};
constexpr int kSideWarp = 4;  // runs `side` during the MMA loop (a warp with no pipeline role)

template <class Clock, class Side = NoSide>
__device__ __forceinline__ void gemm(Pipe& p, Clock& pc, const float* __restrict__ Ag, int nch, int ncol,
                                     int nsets, const float* __restrict__ next_Ag, Side side = Side()) {
  constexpr uint32_t a_bytes = 4u * 128u * KW * 4u;  // one chunk: 4 planes x 128 rows x KW floats
  constexpr uint32_t a_plane = 128u * KW * 4u;
  const uint32_t have = p.have;
  const uint32_t npf = next_Ag ? (uint32_t)kPerm : 0u;
  const int warp = threadIdx.x >> 5;
  // Two producer warps (chunks of even / odd index) and, with two accumulator
  // sets, two MMA warps (even chunks -> set 0, odd chunks -> set 1; MMAs of
  // different threads are unordered, so each warp owns its accumulators): the
  // ~450 cycles a role warp spends per chunk on barrier operations overlap.
  // Every warp walks ALL chunks to keep the per-stage phase masks current and
  // acts on its own.
  const int nmw = (nsets == 2 && !(AMMMSE_PHASES && (p.dbg & 8))) ? 2 : 1;
  const bool one_producer = AMMMSE_PHASES && (p.dbg & 16);
  const uint32_t stage_base0 = umma::smem_u32(p.ring), stage_base1 = umma::smem_u32(p.vol0),
                 stage_base2 = umma::smem_u32(p.vol1), full0 = umma::smem_u32(p.full),
                 done0 = umma::smem_u32(p.done);
  auto stage_addr = [&](uint32_t s) {
    return s < (uint32_t)kPerm       ? stage_base0 + s * a_bytes
           : s < (uint32_t)kPerm + 2 ? stage_base1 + (s - kPerm) * a_bytes
                                     : stage_base2 + (s - kPerm - 2) * a_bytes;
  };
  if (warp == kProducerWarp || warp == kProducerWarp2) {
    const uint32_t me = warp == kProducerWarp ? 0u : 1u;
    const bool nocopy = AMMMSE_PHASES && (p.dbg & 1);
    uint32_t pm = p.pm, ever = p.ever;
    auto fill = [&](uint32_t c, uint32_t s, const unsigned char* src) {
      const uint32_t bit = 1u << s;
      if (one_producer ? me == 0u : (c & 1u) == me) {
        const uint32_t fb = full0 + 8u * s, db = done0 + 8u * s, dst = stage_addr(s);
        // the stage's previous MMAs completed (done completion number fills - 1)
#if AMMMSE_PHASES >= 2
        const long long tw0 = clock64();
#endif
        if (ever & bit) mbar_wait_spin_u32(db, ((pm >> s) & 1u) ^ 1u);
#if AMMMSE_PHASES >= 2
        if (p.prof && threadIdx.x == 32 && blockIdx.x == 0)
          atomicAdd(p.prof + 19, (unsigned long long)(clock64() - tw0));
#endif
        if (nocopy) {
          if (elect_one()) mbar_arrive_u32(fb);
        } else {
          // copy first: its latency is the long pole; the phase cannot complete
          // before the arrive, whatever the order of complete_tx / expect_tx
          asm volatile(
              "{\n\t.reg .pred Pe;\n\t"
              "elect.sync _|Pe, 0xffffffff;\n\t"
              "@Pe cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t"
              "@Pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
              "}\n" ::"r"(dst),
              "l"(src), "r"(a_bytes), "r"(fb)
              : "memory");
        }
      }
      pm ^= bit;
      ever |= bit;
    };
    const unsigned char* src = reinterpret_cast<const unsigned char*>(Ag) + (size_t)have * a_bytes;
    uint32_t s = have % kStages;
    for (uint32_t c = have; c < (uint32_t)nch; ++c, src += a_bytes) {
      fill(c, s, src);
      if (++s == (uint32_t)kStages) s = 0;
    }
    src = reinterpret_cast<const unsigned char*>(next_Ag);
    for (uint32_t c = 0; c < npf; ++c, src += a_bytes) fill(c, c, src);
    p.pm = pm;
    p.ever = ever;
  } else if (warp == kMmaWarp || warp == kMmaWarp2) {
    const uint32_t me = warp == kMmaWarp ? 0u : 1u;
    const uint32_t idesc = umma::make_idesc_tf32(128, 2 * ncol, false, false, false, false);
    // descriptors: the start address (>> 4, 14 bits: a CTA of a cluster sees its
    // shared window at a rank-dependent base, so the field is masked) is the low
    // word's low bits; the high word is constant
    const uint64_t dproto = umma::make_sdesc(0, 128, 256);
    const uint64_t dhi = (uint64_t)(uint32_t)(dproto >> 32) << 32;
    const uint32_t dlo = (uint32_t)dproto;
    auto lo14 = [](uint32_t addr) { return (addr >> 4) & 0x3FFFu; };
    constexpr uint32_t pl = a_plane >> 4;
    uint32_t b_lo = dlo | lo14(umma::smem_u32(p.bfull));  // B chunk 0, hi rows
    const uint32_t b_inc = p.b_chunk >> 4, lo_off = ((uint32_t)(2 * ncol / 8) * 256u) >> 4;
    const uint32_t tmem = p.tmem;
    const bool nomma = AMMMSE_PHASES && (p.dbg & 2);
    uint32_t cm = p.cm;
    const bool active = (int)me < nmw;
    // first own chunk: me (stage me)
    uint32_t ok = active && (int)me < nch ? mbar_test_u32(full0 + 8u * me, (cm >> me) & 1u) : 0u;
    uint32_t s = 0;
    for (int c = 0; c < nch; ++c, b_lo += b_inc) {
      const uint32_t bit = 1u << s;
      if (active && ((uint32_t)c & (uint32_t)(nmw - 1)) == me) {
        const uint32_t fb = full0 + 8u * s;
        const uint32_t par = (cm >> s) & 1u;
        // (no tcgen05 fence: the operands arrive through the async proxy, whose
        // complete_tx on the barrier is what the MMA's own async reads are ordered by)
        while (!ok) ok = mbar_test_u32(fb, par);
        pc.mark2(16);  // (AMMMSE_PHASES=2) MMA warp: waiting for A chunks
        const uint32_t al = dlo | lo14(stage_addr(s));
        // The chunk's six MMAs, its commit and the poll of this warp's NEXT chunk's
        // barrier in one asm block: the poll is issued first and its predicate is
        // consumed last, so its round trip hides behind the rest.
        const int cn = c + nmw;
        const bool last = cn >= nch;
        uint32_t s2 = s + (uint32_t)nmw;
        if (s2 >= (uint32_t)kStages) s2 -= kStages;
        const uint32_t nfb = last ? fb : full0 + 8u * s2;
        const uint32_t npar = last ? par : (cm >> s2) & 1u;
        const uint64_t bhi = dhi | b_lo, blo = dhi | (b_lo + lo_off);
        const int set = nsets == 2 ? (c & 1) : 0;
        const uint32_t acc = c >= nsets ? 1u : 0u;
        const uint32_t d1 = tmem + (uint32_t)(set * 4 * ncol);
        const uint32_t d2 = d1 + (uint32_t)(2 * ncol);
        ok = mma6_poll(d1, d2, dhi | al, dhi | (al + pl), dhi | (al + 2 * pl), dhi | (al + 3 * pl), bhi,
                       blo, idesc, acc, nfb, npar, nomma ? 0u : 1u, done0 + 8u * s);
        if (last) ok = 0u;
        pc.mark2(17);  // issuing
      }
      cm ^= bit;
      if (++s == (uint32_t)kStages) s = 0;
    }
    if (active) {
      if (elect_one()) umma::commit(p.fin);  // fin counts one arrival per MMA warp
      __syncwarp();
    }
    if (warp == kMmaWarp) umma::mbar_wait_spin(p.fin, p.call & 1u);  // all MMAs of this call completed
    pc.mark2(18);  // tail: the last MMAs
    p.cm = cm;
  } else if (warp == kSideWarp) {
    side();
  }
  p.have = npf;
  p.call += 1;
  __syncthreads();
  umma::fence_after();
}

// Consume prefetched chunks that no GEMM will use (end of a realization): wait
// for each copy to land, then release its stage.
__device__ __forceinline__ void drain(Pipe& p) {
  for (uint32_t s = 0; s < p.have; ++s) {
    if ((threadIdx.x >> 5) == kMmaWarp) {
      mbar_wait_spin_u32(umma::smem_u32(p.full) + 8u * s, (p.cm >> s) & 1u);
      if (elect_one()) mbar_arrive_u32(umma::smem_u32(p.done) + 8u * s);
      __syncwarp();
    }
    p.cm ^= 1u << s;  // (every warp keeps its copy of the phase mask current)
  }
  p.have = 0;
}

// byte offset inside the split B buffer of element (n, k): n = row of the
// K-major [re_hi; im_hi; re_lo; im_lo] matrix (4 ncol rows), k = GEMM K index
__device__ __forceinline__ uint32_t b_offset(uint32_t b_chunk, int n, int k) {
  return (uint32_t)(k >> 3) * b_chunk + tcs::kstep_offset(n, k & 7);
}

// (re, im) sums of the accumulator sets of tile t, columns [q0, q0 + 16) of the
// calling thread's TMEM lane:  gr/gi = A · B (conj_a = false) or conj(A) · B
template <bool CONJ>
__device__ __forceinline__ void load_acc(const Pipe& p, uint32_t lane_base, int t, int q0, int ncol,
                                         int nmt_max, int nsets, float (&gr)[16], float (&gi)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) gr[j] = gi[j] = 0.f;
  for (int set = 0; set < nsets; ++set) {
    const uint32_t d1 = p.tmem + lane_base + (uint32_t)((set * nmt_max + t) * 4 * ncol);
    const uint32_t d2 = d1 + (uint32_t)(2 * ncol);
    uint32_t rr[16], ri[16], ir[16], ii[16];
    umma::tmem_ld16_nw(d1 + q0, rr);
    umma::tmem_ld16_nw(d1 + ncol + q0, ri);
    umma::tmem_ld16_nw(d2 + q0, ir);
    umma::tmem_ld16_nw(d2 + ncol + q0, ii);
    umma::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (CONJ) {
        gr[j] += __uint_as_float(rr[j]) + __uint_as_float(ii[j]);
        gi[j] += __uint_as_float(ri[j]) - __uint_as_float(ir[j]);
      } else {
        gr[j] += __uint_as_float(rr[j]) - __uint_as_float(ii[j]);
        gi[j] += __uint_as_float(ri[j]) + __uint_as_float(ir[j]);
      }
    }
  }
}

// Largest eigenvalue of a Hermitian n x n matrix by the cyclic Jacobi method of
// herm_eig_max (small_linalg.cuh: same rotations in the same order on the 2n x 2n
// real embedding), run by a whole warp on a matrix in shared memory: lane r
// updates row / column entry r of each rotation.  The one-thread version keeps
// the 8 x 8 matrix in local memory (dynamic indices) and costs ~1 M cycles per
// user; this one a few 10 k.  A: identical in every lane; S: 4 n² doubles of
// shared scratch of this warp.
template <int n>
__device__ __forceinline__ double herm_eig_max_warp(const cd (&A)[n][n], double* S, int lane) {
  if (n == 1) return A[0][0].r;
  constexpr int m = 2 * n;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < n; ++j) {
        const double re = 0.5 * (A[i][j].r + A[j][i].r);  // hermitianize (linalg.py:12-14)
        const double im = 0.5 * (A[i][j].i - A[j][i].i);
        S[i * m + j] = re;
        S[(i + n) * m + j + n] = re;
        S[(i + n) * m + j] = im;
        S[i * m + j + n] = -im;
      }
  }
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    int done = 0;
    if (lane == 0) {  // same summation order as the one-thread version
      double off = 0.0, diag = 0.0;
      for (int p = 0; p < m; ++p) {
        diag += S[p * m + p] * S[p * m + p];
        for (int q = p + 1; q < m; ++q) off += S[p * m + q] * S[p * m + q];
      }
      done = (off <= 1e-34 * diag || off == 0.0) ? 1 : 0;
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = S[p * m + q];
        if (apq == 0.0) continue;  // (uniform: every lane reads the same element)
        const double theta = (S[q * m + q] - S[p * m + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        __syncwarp();  // the reads above precede the updates
        if (lane < m) {  // columns p, q
          const double srp = S[lane * m + p], srq = S[lane * m + q];
          S[lane * m + p] = c * srp - s * srq;
          S[lane * m + q] = s * srp + c * srq;
        }
        __syncwarp();
        if (lane < m) {  // rows p, q
          const double spr = S[p * m + lane], sqr = S[q * m + lane];
          S[p * m + lane] = c * spr - s * sqr;
          S[q * m + lane] = s * spr + c * sqr;
        }
        __syncwarp();
      }
  }
  double mx = S[0];
  for (int p = 1; p < m; ++p) mx = fmax(mx, S[p * m + p]);
  __syncwarp();
  return mx;
}

}  // namespace tc2

template <int NN, int DD>
__global__ void __launch_bounds__(tc2::kThreads, 1) ammmse_tc2_kernel(EngineArgs a) {
  using R = float;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ctl ctl;
  __shared__ unsigned long long s_r;
  __shared__ uint64_t tc_full[tc2::kMaxStages], tc_done[tc2::kMaxStages], tc_fin;
  __shared__ uint32_t tc_tmem_slot;
  __shared__ double xl[16 * 8];  // local copy of every CTA's exchange slots 0..7 (xs_fetch)
  __shared__ double s_power;     // cluster ‖X‖² of the iteration
  __builtin_assume(blockDim.x == tc2::kThreads);
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int C = (int)cl.num_blocks();
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  tc2::T2Layout<NN, DD> L;
  L.init(a.M, a.K, C, a.tc_stages);
  const int M = L.M, K = L.K, KL = L.KL, KN = L.KN, ncol = L.ncol, ldg = L.ldg;
  const int nmtA = L.nmtA, nmtB = L.nmtB, nmt_max = L.nmt, nsets = L.nsets;
  const int nchA = KN / tc2::KW, nchB = M / tc2::KW;
  const int k0 = crank * KL;      // first own user
  const int col0 = crank * ncol;  // first own global column

  float* Gr[2];
  float* Gi[2];
  Gr[0] = reinterpret_cast<float*>(smem + L.oG0); Gi[0] = Gr[0] + L.nG;
  Gr[1] = reinterpret_cast<float*>(smem + L.oG1); Gi[1] = Gr[1] + L.nG;
  // Ŷ factor of every user: M_k = P_k U_k^H = α_k U_k W_k U_k^H (N x N), so that the
  // off-diagonal blocks are Ŷ_kj = M_k Ĝ_kj (objective.py:196-213 in factored form)
  RC<R>* Mall = reinterpret_cast<RC<R>*>(smem + L.oP);
  RC<R>* Down = reinterpret_cast<RC<R>*>(smem + L.oD);
  unsigned char* bfull = smem + L.oB;
  float* gkk_save = reinterpret_cast<float*>(smem + L.oGk);
  double* dp = reinterpret_cast<double*>(smem + L.dbl_off);
  cd* gx[2];
  gx[0] = reinterpret_cast<cd*>(dp); dp += 2 * K * NN * NN;
  gx[1] = reinterpret_cast<cd*>(dp); dp += 2 * K * NN * NN;
  const Pair<cd> ucb{reinterpret_cast<cd*>(dp), (size_t)KL * NN * DD};
  dp += 2 * 2 * KL * NN * DD;
  const Pair<cd> wcb{reinterpret_cast<cd*>(dp), (size_t)KL * DD * DD};
  dp += 2 * 2 * KL * DD * DD;
  const Pair<double> lndb{dp, (size_t)KL};
  dp += 2 * KL;
  double* alpha = dp; dp += KL;
  double* fu = dp; dp += KL;
  double* fw = dp; dp += KL;
  double* fv = dp; dp += KL;
  double* rate = dp; dp += KL;
  double* ust = dp; dp += KL;
  double* ust2 = dp; dp += KL;
  double* xs = dp; dp += XS_COUNT;
  double* k1w = dp; dp += L.k1w_count();
  double* wsrw = dp; dp += L.wsr_count();
  double* red = dp;

  // ---- pipeline setup: mbarriers, TMEM ----
  tc2::Pipe pipe;
  pipe.ring = smem + L.oRing;
  pipe.vol0 = smem + L.oG0;
  pipe.vol1 = smem + L.oG1;
  pipe.bfull = bfull;
  pipe.a_stage = (uint32_t)L.a_stage;
  pipe.b_chunk = (uint32_t)L.b_chunk;
  pipe.full = tc_full;
  pipe.done = tc_done;
  pipe.fin = &tc_fin;
  if (tid == 0) {
    for (int q = 0; q < tc2::kMaxStages; ++q) {
      umma::mbar_init(&tc_full[q], 1);
      umma::mbar_init(&tc_done[q], 1);
    }
    umma::mbar_init(&tc_fin, (L.nsets == 2 && !(AMMMSE_PHASES && (a.dbg & 8))) ? 2 : 1);  // one commit per MMA warp
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc<512>(&tc_tmem_slot);  // one CTA per SM (shared-memory size)
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  pipe.tmem = tc_tmem_slot;
#if AMMMSE_PHASES
  pipe.dbg = a.dbg;
  pipe.prof = a.prof;
  if (a.dbg) {  // ablation runs: defined (zero) operands and accumulators
    for (size_t i = tid; i < (size_t)tc2::kPerm * L.a_stage / 4; i += blockDim.x)
      reinterpret_cast<float*>(smem + L.oRing)[i] = 0.f;
    if (warp < 4) {
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
      for (int c = 0; c < 512; c += 16) tc2::tmem_st16(pipe.tmem + ((uint32_t)(32 * warp) << 16) + c, z);
      tc2::tmem_wait_st();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  }
#endif
  const size_t hp = (size_t)8 * KN * M;
  float* slot = a.hplanes + (size_t)(blockIdx.x / C) * hp;
  const float* hpB = slot;                        // H planes   (rows r, K = m): GEMM-B
  const float* hpA = slot + (size_t)4 * KN * M;   // H^T planes (rows m, K = r): GEMM-A

  // epilogue geometry: warp w reads TMEM lane quadrant w & 3, column blocks of
  // 16 starting at 16 (w >> 2), stepping by 32
  const int quad = warp & 3, cgrp = warp >> 2;
  const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
  const int row_in_tile = 32 * quad + lane;
  // precoders in TMEM: buffer b, tile t at column vcol(b, t): re [0, ncol), im [ncol, 2 ncol)
  auto vcol = [&](int b, int t) { return (uint32_t)(L.acc_cols + (b * nmtA + t) * 2 * ncol); };

  auto xsum = [&](int sl) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += cl.map_shared_rank(xs, c)[sl];
    return s;
  };
  // Batched read of the cluster's exchange slots 0..7 by warp 0 (one DSMEM
  // round trip instead of a dozen dependent ones on thread 0); the fixed-order
  // sums below then run on local shared memory.  Call after the cluster
  // barrier that publishes the slots; only warp 0 may use xlsum / xlfirst.
  auto xs_fetch = [&]() {
    if (warp == 0) {
      for (int i = lane; i < C * 8; i += 32) xl[i] = cl.map_shared_rank(xs, i >> 3)[i & 7];
      __syncwarp();
    }
  };
  auto xlsum = [&](int sl) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += xl[c * 8 + sl];
    return s;
  };
  auto xlfirst = [&](int sl) {
    for (int c = 0; c < C; ++c) {
      const double v = xl[c * 8 + sl];
      if (v != 0.0) return (int)v;
    }
    return 0;
  };
  // cluster sum of slot sl to every thread of the block: warp 0 reads the C
  // remote values in parallel, fixed-order sum, broadcast through shared memory
  auto xsum_block = [&](int sl) {
    if (warp == 0) {
      const double v = lane < C ? cl.map_shared_rank(xs, lane)[sl] : 0.0;
      double s = 0.0;
      for (int c = 0; c < C; ++c) s += __shfl_sync(0xffffffffu, v, c);
      if (lane == 0) s_power = s;
    }
    __syncthreads();
    return s_power;
  };
  auto xfirst = [&](int sl) {
    for (int c = 0; c < C; ++c) {
      const double v = cl.map_shared_rank(xs, c)[sl];
      if (v != 0.0) return (int)v;
    }
    return 0;
  };
  auto gram_reduce = [&](int buf, int first, int step) {
    constexpr int per = NN * NN;
    for (int i = first; i < KL * per; i += step) {
      const size_t gi = (size_t)k0 * per + i;
      cd s = cl.map_shared_rank(gx[buf], 0)[gi];
      for (int c = 1; c < C; ++c) s = cadd(s, cl.map_shared_rank(gx[buf], c)[gi]);
      gx[buf][gi] = s;
    }
  };
  // Gram partials over own columns for ALL users, one thread per (user, row a):
  // out[k][a][b] = sum_j X[(k,a), j] conj(X[(k,b), j]) in fp64 (exact products of
  // the fp32 values), no shuffles; threads first, first + nth, ... of a group
  auto gram_rows = [&](const R* Xr, const R* Xi, cd* out, int first, int nth) {
    for (int i = first; i < K * NN; i += nth) {
      const int k = i / NN, aa = i - k * NN;
      const R* xar = Xr + (size_t)i * ldg;
      const R* xai = Xi + (size_t)i * ldg;
      const R* xbr = Xr + (size_t)k * NN * ldg;
      const R* xbi = Xi + (size_t)k * NN * ldg;
      double sr[NN], si[NN];
#pragma unroll
      for (int b = 0; b < NN; ++b) sr[b] = si[b] = 0.0;
#pragma unroll 4
      for (int j = 0; j < ncol; ++j) {
        const double ar = (double)xar[j], ai = (double)xai[j];
#pragma unroll
        for (int b = 0; b < NN; ++b) {
          const double br = (double)xbr[b * ldg + j], bi = (double)xbi[b * ldg + j];
          sr[b] = fma(ar, br, fma(ai, bi, sr[b]));
          si[b] = fma(ai, br, fma(-ar, bi, si[b]));
        }
      }
#pragma unroll
      for (int b = 0; b < NN; ++b) out[(size_t)i * NN + b] = cmk(sr[b], b == aa ? 0.0 : si[b]);
    }
  };
  // NN = 4: four lanes per user, lane g sums the columns j = g (mod 4) of the
  // packed lower triangle (every element converted to fp64 once), then a
  // two-level reduce-scatter leaves four of the 16 packed sums in each lane
  auto gram_quad = [&](const R* Xr, const R* Xi, cd* out, int first, int nth) {
    if constexpr (NN == 4) {
      for (int i = first; i < K * 4; i += nth) {  // (whole warps stay together: K * 4 % 32 == 0)
        const int k = i >> 2, g = i & 3;
        double sr[4][4], si[4][4];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) sr[p][q] = si[p][q] = 0.0;
        const R* xr = Xr + (size_t)k * 4 * ldg;
        const R* xi = Xi + (size_t)k * 4 * ldg;
#pragma unroll 2
        for (int j = g; j < ncol; j += 4) {
          double gr[4], gi[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            gr[p] = (double)xr[p * ldg + j];
            gi[p] = (double)xi[p * ldg + j];
          }
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q <= p; ++q) {  // g_p * conj(g_q)
              sr[p][q] = fma(gr[p], gr[q], fma(gi[p], gi[q], sr[p][q]));
              if (q < p) si[p][q] = fma(gi[p], gr[q], fma(-gr[p], gi[q], si[p][q]));
            }
        }
        double v[16];  // gram_pack order: 10 real parts (row-major lower triangle), 6 imaginary
        {
          int n = 0;
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q <= p; ++q) v[n++] = sr[p][q];
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < p; ++q) v[n++] = si[p][q];
        }
        const bool up2 = (g & 2) != 0, up1 = (g & 1) != 0;
        double w[8], z[4];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double send = up2 ? v[e] : v[8 + e];
          const double keep = up2 ? v[8 + e] : v[e];
          w[e] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double send = up1 ? w[e] : w[4 + e];
          const double keep = up1 ? w[4 + e] : w[e];
          z[e] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
        // lane g holds packed sums 4 g .. 4 g + 3 (gram_pack order): store them into
        // the full Hermitian 4 x 4 of user k
        cd* G = out + (size_t)k * 16;
        auto setre = [&](int p, int q, double v) {
          G[p * 4 + q].r = v;
          G[q * 4 + p].r = v;
          if (p == q) G[p * 4 + p].i = 0.0;
        };
        auto setim = [&](int p, int q, double v) {
          G[p * 4 + q].i = v;
          G[q * 4 + p].i = -v;
        };
        if (g == 0) {
          setre(0, 0, z[0]); setre(1, 0, z[1]); setre(1, 1, z[2]); setre(2, 0, z[3]);
        } else if (g == 1) {
          setre(2, 1, z[0]); setre(2, 2, z[1]); setre(3, 0, z[2]); setre(3, 1, z[3]);
        } else if (g == 2) {
          setre(3, 2, z[0]); setre(3, 3, z[1]); setim(1, 0, z[2]); setim(2, 0, z[3]);
        } else {
          setim(2, 1, z[0]); setim(3, 0, z[1]); setim(3, 1, z[2]); setim(3, 2, z[3]);
        }
      }
    } else {
      gram_rows(Xr, Xi, out, first, nth);
    }
  };
  auto gram_of = [&](int buf, int kl, cd (&Tg)[NN][NN]) {
    const cd* g = gx[buf] + (size_t)(k0 + kl) * NN * NN;
#pragma unroll
    for (int p = 0; p < NN; ++p)
#pragma unroll
      for (int q = 0; q < NN; ++q) Tg[p][q] = g[p * NN + q];
  };
  auto k1_load = [&](int gsrc, int kl, cd (&Tg)[NN][NN], cd (&Gkk)[NN][DD]) {
    gram_of(0, kl, Tg);
#pragma unroll
    for (int p = 0; p < NN; ++p)
#pragma unroll
      for (int s = 0; s < DD; ++s) {
        const int idx = ((k0 + kl) * NN + p) * ldg + kl * DD + s;
        Gkk[p][s] = cmk((double)Gr[gsrc][idx], (double)Gi[gsrc][idx]);
      }
  };
  auto k1_wprev = [&](int bin, int kl, cd (&Wp)[DD][DD]) {
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) Wp[p][q] = wcb[bin][(kl * DD + p) * DD + q];
  };
  auto k1_store = [&](int kl, const K1Out<NN, DD>& o, int bout) {
    cd* ucache = ucb[bout];
    cd* wcache = wcb[bout];
#pragma unroll
    for (int p = 0; p < NN; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        const int il = (kl * NN + p) * DD + q;
        Down[il] = RC<R>{(R)o.D[p][q].r, (R)o.D[p][q].i};
        ucache[il] = o.U[p][q];
      }
#pragma unroll
    for (int p = 0; p < NN; ++p)
#pragma unroll
      for (int b = 0; b < NN; ++b) {  // M = P U^H
        cd acc = cmk(0.0);
#pragma unroll
        for (int q = 0; q < DD; ++q) acc = cadd(acc, cmulcb(o.P[p][q], o.U[b][q]));
        Mall[((k0 + kl) * NN + p) * NN + b] = RC<R>{(R)acc.r, (R)acc.i};
      }
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) wcache[(kl * DD + p) * DD + q] = o.W[p][q];
    lndb[bout][kl] = o.lndetw;
    fu[kl] = o.fu;
    fw[kl] = o.fw;
    ust[kl] = o.status;
  };
  auto k1_users = [&](int gsrc, bool weighted, bool want_f, int bin, int bout, int first,
                      int step) {
    for (int kl = first; kl < KL; kl += step) {
      cd Tg[NN][NN], Gkk[NN][DD], Wp[DD][DD];
      k1_load(gsrc, kl, Tg, Gkk);
      k1_wprev(bin, kl, Wp);
      K1Out<NN, DD> o;
      k1_math<NN, DD>(Tg, Gkk, ctl.sigma2, alpha[kl], Wp, lndb[bin][kl], weighted, want_f, o);
      k1_store(kl, o, bout);
    }
  };
  // K1(t+1) on warps 1.. while warp 0 runs WSR(t) (ammmse_cluster.cuh k1_pipelined)
  auto k1_pipelined = [&](int gsrc, bool weighted, int bin, int bout) {
    if constexpr (NN == 4 && DD == 4) {
      // quad-lane path: warp 1 = receiver half + combine, warp 2 = weight half,
      // four lanes per user (user_algebra_quad.cuh)
      if (warp != 1 && warp != 2) return;
      if (warp == 2 && !weighted) return;
      const quad::QuadArgs qa{Gr[gsrc] + (size_t)k0 * NN * ldg, Gi[gsrc] + (size_t)k0 * NN * ldg,
                              NN * ldg + DD, ldg, k0, KL, gx[0], ctl.sigma2, alpha, a.trace != nullptr};
      const quad::K1Out4 ko{ucb[bout], wcb[bout], lndb[bout], fu, fw, ust,
                            reinterpret_cast<float2*>(Mall), reinterpret_cast<float2*>(Down), k1w};
      if (warp == 2)
        quad::k1_weight_users(qa, ko);
      else
        quad::k1_recv_users(qa, ko, wcb[bin], lndb[bin], weighted);
      return;
    }
    constexpr bool closed = NN == 2 && DD == 2;
    if (closed || !weighted || KL > 32) {
      if (tid >= 32) k1_users(gsrc, weighted, true, bin, bout, tid - 32, blockDim.x - 32);
      return;
    }
    if constexpr (!closed) {
      constexpr int wstride = 2 * DD * DD + NN + 1;
      if (warp == 1) {
        K1U<NN, DD> u;
        cd Tg[NN][NN], Gkk[NN][DD];
        if (lane < KL) {
          cd Wp[DD][DD];
          k1_load(gsrc, lane, Tg, Gkk);
          k1_wprev(bin, lane, Wp);
          k1_part_u<NN, DD>(Tg, Gkk, ctl.sigma2, alpha[lane], Wp, lndb[bin][lane], true, u);
        }
        asm volatile("bar.sync 1, 64;\n" ::: "memory");
        if (lane < KL) {
          const double* w = k1w + (size_t)lane * wstride;
          cd Wm[DD][DD];
          double pv[NN];
#pragma unroll
          for (int p = 0; p < DD; ++p)
#pragma unroll
            for (int q = 0; q < DD; ++q) Wm[p][q] = cmk(w[2 * (p * DD + q)], w[2 * (p * DD + q) + 1]);
#pragma unroll
          for (int i = 0; i < NN; ++i) pv[i] = w[2 * DD * DD + i];
          K1Out<NN, DD> o;
          k1_combine<NN, DD>(u, Wm, pv, (int)w[2 * DD * DD + NN], alpha[lane], true, true, o);
          k1_store(lane, o, bout);
        }
      } else if (warp == 2) {
        if (lane < KL) {
          cd Tg[NN][NN], Gkk[NN][DD];
          k1_load(gsrc, lane, Tg, Gkk);
          K1W<NN, DD> wv;
          k1_part_w<NN, DD>(Tg, Gkk, ctl.sigma2, wv);
          double* w = k1w + (size_t)lane * wstride;
#pragma unroll
          for (int p = 0; p < DD; ++p)
#pragma unroll
            for (int q = 0; q < DD; ++q) {
              w[2 * (p * DD + q)] = wv.W[p][q].r;
              w[2 * (p * DD + q) + 1] = wv.W[p][q].i;
            }
#pragma unroll
          for (int i = 0; i < NN; ++i) w[2 * DD * DD + i] = wv.piv[i];
          w[2 * DD * DD + NN] = (double)wv.pd;
        }
        asm volatile("bar.sync 1, 64;\n" ::: "memory");
      }
    }
  };
  auto k1_publish = [&]() {
    double su = 0.0, sw = 0.0;
    int st = 0;
    for (int kl = 0; kl < KL; ++kl) {
      su += fu[kl];
      sw += fw[kl];
      if (st == 0 && ust[kl] != 0.0) st = (int)ust[kl];
    }
    xs[XS_FU] = su;
    xs[XS_FW] = sw;
    xs[XS_ST1] = st;
  };
  auto k1_gather = [&](int first, int step) {
    const int per = NN * NN;
    for (int i = first; i < K * per; i += step) {
      const int owner = (i / per) / KL;
      if (owner != crank) Mall[i] = cl.map_shared_rank(Mall, owner)[i];
    }
  };
  auto k1_phase = [&](int gsrc, bool weighted, bool want_f, int bin, int bout) {
    k1_users(gsrc, weighted, want_f, bin, bout, tid, blockDim.x);
    __syncthreads();
    if (tid == 0) k1_publish();
    cl.sync();
    xs_fetch();
    k1_gather(tid, blockDim.x);
  };

  // split store of one fp32 value of the B operand: rows n (hi) and n + 2 ncol (lo)
  auto b_store = [&](int n, int k, float x) {
    float hi, lo;
    umma::split_tf32(x, hi, lo);
    unsigned char* d = bfull + tc2::b_offset(pipe.b_chunk, n, k);
    *reinterpret_cast<float*>(d) = hi;
    *reinterpret_cast<float*>(d + (size_t)(2 * ncol / 8) * 256) = lo;
  };

  // Ŷ over own columns from Ĝ(t) in G[g] (gradient factor, objective.py:172-213
  // in factored form), written split into the B buffer: K index = G row
  // (user m, antenna p), column jl.
  auto build_yhat = [&](int g) {
    const R* Yr = Gr[g];
    const R* Yi = Gi[g];
    for (int idx = tid; idx < K * ncol; idx += blockDim.x) {
      const int m = idx / ncol, jl = idx - m * ncol;
      const int j = col0 + jl, b = j / DD, s = j - b * DD;
      R yr[NN], yi[NN];
      if (b == m) {
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          const RC<R> v = Down[((m - k0) * NN + p) * DD + s];
          yr[p] = v.r;
          yi[p] = v.i;
        }
      } else {
        R gr[NN], gi[NN];
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          gr[p] = Yr[(m * NN + p) * ldg + jl];
          gi[p] = Yi[(m * NN + p) * ldg + jl];
        }
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          R sr = 0, si = 0;
#pragma unroll
          for (int b = 0; b < NN; ++b) {
            const RC<R> mm = Mall[(m * NN + p) * NN + b];
            sr = fma(mm.r, gr[b], fma(-mm.i, gi[b], sr));
            si = fma(mm.r, gi[b], fma(mm.i, gr[b], si));
          }
          yr[p] = sr;
          yi[p] = si;
        }
      }
      if constexpr (NN == 4) {  // 4 consecutive K values: one 16-byte store per part
        float rh[4], rl[4], ih[4], il[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          umma::split_tf32(yr[p], rh[p], rl[p]);
          umma::split_tf32(yi[p], ih[p], il[p]);
        }
        const int kq = m * 4;
        const size_t lo = (size_t)(2 * ncol / 8) * 256;
        unsigned char* dre = bfull + tc2::b_offset(pipe.b_chunk, jl, kq);
        unsigned char* dim = bfull + tc2::b_offset(pipe.b_chunk, ncol + jl, kq);
        *reinterpret_cast<float4*>(dre) = make_float4(rh[0], rh[1], rh[2], rh[3]);
        *reinterpret_cast<float4*>(dre + lo) = make_float4(rl[0], rl[1], rl[2], rl[3]);
        *reinterpret_cast<float4*>(dim) = make_float4(ih[0], ih[1], ih[2], ih[3]);
        *reinterpret_cast<float4*>(dim + lo) = make_float4(il[0], il[1], il[2], il[3]);
      } else {
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          b_store(jl, m * NN + p, yr[p]);
          b_store(ncol + jl, m * NN + p, yi[p]);
        }
      }
    }
    umma::fence_proxy_async();  // generic st.shared -> tensor-core (async proxy) reads
  };

  // X block (16 columns of row `row`) -> TMEM precoder buffer `vb` and, split,
  // the B operand of GEMM-B (K index = row)
  auto emit_x = [&](int vb, int t, int q0, const float (&xr)[16], const float (&xi)[16]) {
    const int row = 128 * t + row_in_tile;
    uint32_t ur[16], ui[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      ur[j] = __float_as_uint(xr[j]);
      ui[j] = __float_as_uint(xi[j]);
    }
    const uint32_t vc = pipe.tmem + lane_base + vcol(vb, t);
    tc2::tmem_st16(vc + q0, ur);
    tc2::tmem_st16(vc + ncol + q0, ui);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      b_store(q0 + j, row, xr[j]);
      b_store(ncol + q0 + j, row, xi[j]);
    }
    tc2::tmem_wait_st();
  };
  // scaled precoder block of buffer vb
  auto load_x = [&](int vb, int t, int q0, float (&xr)[16], float (&xi)[16]) {
    const uint32_t vc = pipe.tmem + lane_base + vcol(vb, t);
    uint32_t ur[16], ui[16];
    umma::tmem_ld16_nw(vc + q0, ur);
    umma::tmem_ld16_nw(vc + ncol + q0, ui);
    umma::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      xr[j] = __uint_as_float(ur[j]);
      xi[j] = __uint_as_float(ui[j]);
    }
  };

  // GEMM-A epilogue (pgd_precoder_step solvers.py:358-377 + extrapolate :380-390):
  //   V̂ = V_c + ω (V_c − V_o),  V_c = sc X[xc], V_o = so X[xo];  X_new = V̂ − step ∇ -> X[xo]
  // returns this thread's ‖X_new‖² share.  to_b: also write X_new split into B.
  auto epilogue_a = [&](int xc, int xo, float sc, float so, float st, float om, bool extrap,
                        bool to_b) {
    double pw = 0.0;
    for (int t = 0; t < nmtA; ++t)
      for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
        float gr[16], gi[16];
        tc2::load_acc<true>(pipe, lane_base, t, q0, ncol, nmt_max, nsets, gr, gi);
        float cr[16], ci[16];
        load_x(xc, t, q0, cr, ci);
        if (extrap) {
          float orr[16], oi[16];
          load_x(xo, t, q0, orr, oi);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float vr = sc * cr[j], vi = sc * ci[j];
            cr[j] = vr + om * (vr - so * orr[j]);
            ci[j] = vi + om * (vi - so * oi[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            cr[j] *= sc;
            ci[j] *= sc;
          }
        }
        float pwb = 0.f;  // (32 squares per block in fp32, fp64 from there on)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          cr[j] -= st * gr[j];
          ci[j] -= st * gi[j];
          pwb = fmaf(cr[j], cr[j], fmaf(ci[j], ci[j], pwb));
        }
        pw += (double)pwb;
        if (to_b) {
          emit_x(xo, t, q0, cr, ci);
        } else {
          uint32_t ur[16], ui[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            ur[j] = __float_as_uint(cr[j]);
            ui[j] = __float_as_uint(ci[j]);
          }
          const uint32_t vc = pipe.tmem + lane_base + vcol(xo, t);
          tc2::tmem_st16(vc + q0, ur);
          tc2::tmem_st16(vc + ncol + q0, ui);
          tc2::tmem_wait_st();
        }
      }
    umma::fence_proxy_async();
    umma::fence_before();
    return pw;
  };
  // G buffers, fixed roles: N = G[0] holds G_new (WSR(t), exit pass), E = G[1]
  // holds the extrapolated Ĝ(t+1) (K1(t+1), Ŷ(t+1)).  The previous G lives in TMEM
  // (lane = row), so both buffers are dead during the MMA loops, where they
  // serve as ring stages (Pipe::vol0 / vol1).
  constexpr int GN = 0, GE = 1;
  auto gcol = [&](int t) { return (uint32_t)(L.acc_cols + L.v_cols + t * 2 * ncol); };
  // GEMM-B epilogue: G_new = s · acc -> N and TMEM; with hat also
  // Ĝ(t+1) = G_new + ω (G_new − G_old) -> E (solvers.py:380-390 by linearity);
  // ω = 0: plain copy (G_old undefined before the first call)
  auto epilogue_b = [&](float sc, float om, bool hat) {
    R* gr = Gr[GN];
    R* gi = Gi[GN];
    R* hr = Gr[GE];
    R* hi = Gi[GE];
    for (int t = 0; t < nmtB; ++t)
      for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
        float ar[16], ai[16];
        tc2::load_acc<false>(pipe, lane_base, t, q0, ncol, nmt_max, nsets, ar, ai);
        const int row = 128 * t + row_in_tile;
        const uint32_t gc = pipe.tmem + lane_base + gcol(t);
        uint32_t our[16], oui[16];
        if (hat && om != 0.f) {
          umma::tmem_ld16_nw(gc + q0, our);
          umma::tmem_ld16_nw(gc + ncol + q0, oui);
          umma::tmem_wait_ld();
        }
        uint32_t nur[16], nui[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int o = row * ldg + q0 + j;
          const float cr = sc * ar[j], ci = sc * ai[j];
          gr[o] = cr;
          gi[o] = ci;
          nur[j] = __float_as_uint(cr);
          nui[j] = __float_as_uint(ci);
          if (hat) {
            hr[o] = om == 0.f ? cr : cr + om * (cr - __uint_as_float(our[j]));
            hi[o] = om == 0.f ? ci : ci + om * (ci - __uint_as_float(oui[j]));
          }
        }
        tc2::tmem_st16(gc + q0, nur);
        tc2::tmem_st16(gc + ncol + q0, nui);
        tc2::tmem_wait_st();
      }
    umma::fence_before();
  };

  PhaseClock pc;
  pc.init(a.prof);
  for (;;) {
    if (crank == 0 && tid == 0) s_r = atomicAdd(a.counter, 1ULL);
    cl.sync();
    const long long r = (long long)*cl.map_shared_rank(&s_r, 0);
    if (r >= a.B) {
      cl.sync();  // rank 0 stays alive until every CTA has read s_r
      break;
    }
    const RC<R>* Hcur = reinterpret_cast<const RC<R>*>(a.H) + (size_t)r * KN * M;
    int xc = 0;               // TMEM buffer of the current precoders
    float vs0 = 1.f, vs1 = 1.f;  // V = vs_b · X[b] (lazy projection scale)
    auto vsc = [&](int b) { return b ? vs1 : vs0; };
    // ---------------- load realization r ----------------
    {
      {  // this CTA's share of the pre-split H / H^T planes (rows r0..r1)
        const int r0 = crank * (KN / C), r1 = (crank + 1) * (KN / C);
        const float2* H2 = reinterpret_cast<const float2*>(Hcur);
        tcs::split_h(H2, KN, M, false, const_cast<float*>(hpB), r0, r1);
        tcs::split_h(H2, KN, M, true, const_cast<float*>(hpA), r0, r1);
        umma::fence_proxy_async_global();  // generic writes -> the cluster's bulk copies
        __threadfence();
      }
      // V0 (own users' columns) -> TMEM X[0] and the split B operand
      const RC<R>* Vg = reinterpret_cast<const RC<R>*>(a.V0) + ((size_t)r * K + k0) * M * DD;
      for (int t = 0; t < nmtA; ++t)
        for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
          const int row = 128 * t + row_in_tile;
          float xr[16], xi[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int jl = q0 + j, kl = jl / DD, s = jl - kl * DD;
            const RC<R> v = Vg[((size_t)kl * M + row) * DD + s];
            xr[j] = v.r;
            xi[j] = v.i;
          }
          emit_x(0, t, q0, xr, xi);
        }
      umma::fence_proxy_async();
      umma::fence_before();
      for (int kl = tid; kl < KL; kl += blockDim.x) {
        alpha[kl] = a.alpha[(size_t)r * K + k0 + kl];
        lndb[0][kl] = 0.0;  // W_prev = I at t = 1 (solvers.py:429-430); K1(1) reads bank 0
        for (int p = 0; p < DD; ++p)
          for (int q = 0; q < DD; ++q) wcb[0][(kl * DD + p) * DD + q] = cmk(p == q ? 1.0 : 0.0);
      }
      if (tid == 0) {
        ctl.sigma2 = a.sigma2[r];
        ctl.pmax = a.pmax[r];
        ctl.omega = a.omega_arr ? a.omega_arr[r] : a.omega;
        ctl.nhist = 0;
        ctl.wsr_last = ctl.wsr_prev = 0.0;
        ctl.running_max = -INFINITY;
        ctl.drop_streak = 0;
        ctl.latched = 0;
        ctl.switch_it = -1;
        ctl.weighted_now = 0;
        ctl.last_weighted = 0;
        ctl.cur = 0;
        ctl.stop = 0;
        ctl.status = 0;
        ctl.converged = 0;
        ctl.iters = 0;
        ctl.f_u = ctl.f_w = ctl.f_v = ctl.wsr = 0.0;
      }
    }
    __syncthreads();
    // ---------------- bounds (objective.py:216-240): own users, max over cluster ----------------
    {
      const int nw = blockDim.x >> 5;
      for (int kl = warp; kl < KL; kl += nw) {
        const int k = k0 + kl;
        double sr[NN][NN], si[NN][NN];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < NN; ++q) sr[p][q] = si[p][q] = 0.0;
        for (int m = lane; m < M; m += 32) {
          double hr[NN], hi[NN];
          for (int p = 0; p < NN; ++p) {
            const RC<R> v = Hcur[(size_t)(k * NN + p) * M + m];
            hr[p] = (double)v.r;
            hi[p] = (double)v.i;
          }
          for (int p = 0; p < NN; ++p)
            for (int q = 0; q < NN; ++q) {
              sr[p][q] = fma(hr[p], hr[q], fma(hi[p], hi[q], sr[p][q]));
              si[p][q] = fma(hi[p], hr[q], fma(-hr[p], hi[q], si[p][q]));
            }
        }
        cd G[NN][NN];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < NN; ++q) G[p][q] = cmk(warp_allsum(sr[p][q]), warp_allsum(si[p][q]));
        // (scratch: the K1 exchange region, idle during the setup; 4 N² doubles per warp)
        double lam;
        if ((size_t)(blockDim.x >> 5) * 4 * NN * NN <= L.k1w_count())
          lam = tc2::herm_eig_max_warp<NN>(G, k1w + (size_t)warp * 4 * NN * NN, lane);
        else
          lam = herm_eig_max<NN>(G);
        if (lane == 0) rate[kl] = lam;
      }
      __syncthreads();
      if (tid == 0) {
        double kap = 0.0;
        for (int kl = 0; kl < KL; ++kl) kap = fmax(kap, rate[kl]);
        xs[XS_KAPPA] = kap;
      }
      cl.sync();  // also: every CTA's H planes are written before the first bulk copy
      if (tid == 0) {
        double kappa = 0.0;
        for (int c = 0; c < C; ++c) kappa = fmax(kappa, cl.map_shared_rank(xs, c)[XS_KAPPA]);
        double abar = a.alpha[(size_t)r * K];
        for (int k = 0; k < K; ++k) abar = fmax(abar, a.alpha[(size_t)r * K + k]);
        const double l_v = 2.0 * abar * K * kappa / ctl.sigma2;
        ctl.gamma_safe = 1.0 / l_v;
        ctl.gamma = a.gamma_arr ? a.gamma_arr[r] : (a.gamma_safe ? ctl.gamma_safe : a.gamma);
        ctl.step = 2.0 * ctl.gamma;
        if (crank == 0 && a.gamma_used) a.gamma_used[r] = ctl.gamma;
      }
    }
    // initial G = H V0 into G[0]; Ĝ(1) = G (no extrapolation at t = 1) into G[1]
    tc2::gemm(pipe, pc, hpB, nchB, ncol, nsets, hpA);
    epilogue_b(1.f, 0.f, true);
    __syncthreads();

    auto stage_flag = [&]() -> bool {  // solvers.py:449-459
      if (ctl.latched) return true;
      double rs = INFINITY;
      if (ctl.nhist >= 2) {
        const double den = fabs(ctl.wsr_prev);
        rs = den == 0.0 ? INFINITY : fabs(ctl.wsr_last - ctl.wsr_prev) / den;
      }
      return rs <= a.eps1;
    };
    // ---------------- K1(1) ----------------
    bool wn = stage_flag();
    gram_rows(Gr[1], Gi[1], gx[0], tid, blockDim.x);
    cl.sync();
    gram_reduce(0, tid, blockDim.x);
    __syncthreads();
    k1_phase(1, wn, true, 0, 1);
    pc.mark(9);

    // ---------------- main loop (solvers.py:440-505), software-pipelined ----------------
    // State machine of iteration te (solvers.py:449-505) on thread 0, from the
    // local exchange copies; identical decisions in every CTA.
    auto state_machine = [&](int te, bool wn_e, double power, double scale) {
      if (!ctl.latched && wn_e) {
        if (a.latch) ctl.latched = 1;
        if (ctl.switch_it < 0) ctl.switch_it = te;
      }
      const double wsr = xlsum(XS_RATE);
      const double sv = xlsum(XS_FV);
      int st = xlfirst(XS_ST2);
      const double total_power = scale == 1.0 ? power : power * scale * scale;
      if (!isfinite(wsr) || !isfinite(power)) st = AMMMSE_STATUS_NONFINITE;
      double rel = INFINITY;  // solvers.py:474, _rel_change :393-397
      if (te > 1) {
        const double den = fabs(ctl.wsr_last);
        rel = den == 0.0 ? INFINITY : fabs(wsr - ctl.wsr_last) / den;
      }
      ctl.wsr_prev = ctl.wsr_last;
      ctl.wsr_last = wsr;
      ctl.nhist += 1;
      ctl.iters = te;
      ctl.wsr = wsr;
      ctl.f_v = sv;
      ctl.weighted_now = wn_e;
      ctl.last_weighted = wn_e;
      if (a.trace && crank == 0) {
        double* tr = a.trace + ((size_t)r * a.max_iters + (te - 1)) * kTraceFields;
        tr[AMMMSE_TRACE_T] = (double)te;
        tr[AMMMSE_TRACE_WSR_BITS] = wsr / kLn2;
        tr[AMMMSE_TRACE_F_VALUE] = sv;
        tr[AMMMSE_TRACE_TOTAL_POWER] = total_power;
        tr[AMMMSE_TRACE_STAGE] = wn_e ? 1.0 : 0.0;
        tr[AMMMSE_TRACE_F_AFTER_U] = ctl.f_u;
        tr[AMMMSE_TRACE_F_AFTER_W] = ctl.f_w;
        tr[AMMMSE_TRACE_F_AFTER_V] = sv;
        tr[AMMMSE_TRACE_REL_CHANGE] = rel;
      }
      ctl.running_max = fmax(ctl.running_max, wsr);  // divergence detector (solvers.py:490-500)
      if (wsr < 0.5 * ctl.running_max)
        ctl.drop_streak += 1;
      else
        ctl.drop_streak = 0;
      if (ctl.drop_streak >= 5 && st == 0) st = AMMMSE_STATUS_UNSTABLE;
      if (st) {
        ctl.status = st;
        ctl.stop = 1;
      } else if (wn_e && rel <= a.eps2) {  // stop test (:503-505)
        ctl.converged = 1;
        ctl.stop = 1;
      }
      ctl.wn_next = stage_flag();
    };
    // Results of K1(tn) from the local exchange copies (thread 0, after the xs_fetch
    // that follows its publication): f_after_u / w sums and the first failure,
    // i.e. update_weight_matrices raising inside iteration tn (solvers.py:455-460).
    auto k1_status = [&](int tn, bool wn_k) {
      ctl.f_u = xlsum(XS_FU);
      ctl.f_w = xlsum(XS_FW);
      const int st = xlfirst(XS_ST1);
      if (st) {
        if (!ctl.latched && wn_k) {
          if (a.latch) ctl.latched = 1;
          if (ctl.switch_it < 0) ctl.switch_it = tn;
        }
        ctl.status = st;
        ctl.stop = 1;
      }
    };
    if (tid == 0) k1_status(1, wn);
    __syncthreads();
    // WSR of the own users from the reduced Gram gx[1] and the diagonal blocks
    // at (gr, gi): per-user rates / f_after_v, then the CTA partials -> exchange
    // slots.  One full warp.
    // split: warp 3 factors the interference matrices meanwhile (wsr_c_warp below)
    auto wsr_warp = [&](const R* gr, const R* gi, int ustride, int rstride, int bank, bool split) {
      const cd* ucache = ucb[bank];
      const cd* wcache = wcb[bank];
      if constexpr (NN == 4 && DD == 4) {  // four lanes per user (user_algebra_quad.cuh)
        const quad::QuadArgs qa{gr, gi, ustride, rstride, k0, KL, gx[1], ctl.sigma2, alpha, a.trace != nullptr};
        if (split)
          quad::wsr_users_a(qa, ucache, wcache, lndb[bank], wsrw, rate, fv, ust2);
        else
          quad::wsr_users(qa, ucache, wcache, lndb[bank], rate, fv, ust2);
      } else {
        for (int kl = lane; kl < KL; kl += 32) {
          cd Tg[NN][NN], Gkk[NN][DD], U[NN][DD], W[DD][DD];
          gram_of(1, kl, Tg);
#pragma unroll
          for (int p = 0; p < NN; ++p)
#pragma unroll
            for (int q = 0; q < DD; ++q) {
              const int idx = kl * ustride + p * rstride + q;
              Gkk[p][q] = cmk((double)gr[idx], (double)gi[idx]);
              U[p][q] = ucache[(kl * NN + p) * DD + q];
            }
#pragma unroll
          for (int p = 0; p < DD; ++p)
#pragma unroll
            for (int q = 0; q < DD; ++q) W[p][q] = wcache[(kl * DD + p) * DD + q];
          double rr, ff;
          int st;
          wsr_math<NN, DD>(Tg, Gkk, ctl.sigma2, alpha[kl], U, W, lndb[bank][kl], rr, ff, st);
          rate[kl] = rr;
          fv[kl] = ff;
          ust2[kl] = st;
        }
      }
      __syncwarp();
      double sr = 0.0, sv = 0.0;
      int f2 = KL;
      for (int kl = lane; kl < KL; kl += 32) {
        sr += rate[kl];
        sv += fv[kl];
        if (f2 == KL && ust2[kl] != 0.0) f2 = kl;
      }
      sr = warp_allsum(sr);
      sv = warp_allsum(sv);
      f2 = __reduce_min_sync(0xffffffffu, f2);
      if (lane == 0) {
        xs[XS_RATE] = sr;
        xs[XS_FV] = sv;
        xs[XS_ST2] = f2 < KL ? ust2[f2] : 0.0;
      }
    };
    // Deferred mode: once the weighted stage is latched the stage flag cannot
    // change any more, so iteration t+1 may start before WSR(t) is known: WSR(t)
    // then runs on a spare warp DURING GEMM-A(t+1), its cluster exchange rides on
    // the ‖X‖² barrier and the state machine of t runs after GEMM-B(t+1)'s MMAs.
    // A stop discovered there discards the speculative step: V(t) is still X[xc]
    // (the step wrote the other TMEM buffer); G is rebuilt for the exit pass.
    // Not used with traces / recorded iterates (their rows are written in order).
    const bool can_defer = a.tc_defer && a.latch && !a.trace && !a.itU;
    bool pending = false;   // WSR(t-1) / state machine of t-1 outstanding
    bool need_g = false;    // exit: G buffers do not hold G(V_final)
    double power_p = 0.0, scale_p = 1.0;  // ‖X‖², scale of the pending iteration
    for (int t = 1; t <= a.max_iters; ++t) {
      const int bk = t & 1;  // bank holding K1(t)'s U / W / ln det W
      const bool extrap = (t >= 2) && (ctl.omega > 0.0);
      pc.mark(0);
      // (the status of K1(t) was evaluated with the exchange fetch that followed it)
      if (ctl.stop && !pending) break;
      // (pending: the K1(t) failure belongs to a step that may still be discarded;
      // it is acted on after the state machine of t-1 below)
      build_yhat(GE);
      __syncthreads();
      pc.mark(1);
      // ∇ = H^H Ŷ  (deferred mode: WSR(t-1) on the side warp meanwhile)
      if (pending) {
        tc2::gemm(pipe, pc, hpA, nchA, ncol, nsets, hpB,
                  [&]() { wsr_warp(gkk_save, gkk_save + KL * NN * DD, NN * DD, DD, (t - 1) & 1, false); });
      } else {
        tc2::gemm(pipe, pc, hpA, nchA, ncol, nsets, hpB);
      }
      pc.mark(10);
      const int xo = 1 - xc;
      double pw = epilogue_a(xc, xo, vsc(xc), vsc(xo), (float)ctl.step, (float)ctl.omega, extrap, true);
      // CTA partial of ‖X‖²: fixed shuffle tree, then thread 0 adds the warps in order
      // (the barrier also orders the B writes before GEMM-B's MMAs)
      pw = warp_allsum(pw);
      if (lane == 0) red[warp] = pw;
      __syncthreads();
      if (tid == 0) {
        double sp = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sp += red[w];
        xs[XS_POWER] = sp;
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      pc.mark(2);
      const bool more = t < a.max_iters;
      // G' = H X_new while the cluster sums ‖X_new‖² (the projection scale is lazy)
      tc2::gemm(pipe, pc, hpB, nchB, ncol, nsets, hpA);
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      xs_fetch();
      if (tid == 0) {
        const int k1_stop = ctl.stop, k1_status = ctl.status;  // K1(t) failure noted above
        if (pending) {
          ctl.stop = 0;
          ctl.status = 0;
          state_machine(t - 1, true, power_p, scale_p);
          if (!ctl.stop && k1_stop) {  // iteration t itself failed in K1(t)
            ctl.status = k1_status;
            ctl.stop = 2;  // (2: stop without discarding... K1(t) failed: nothing of t is kept)
          }
        }
        s_power = xlsum(XS_POWER);
      }
      __syncthreads();
      if (pending && ctl.stop) {  // discard the speculative step
        need_g = true;
        break;
      }
      pending = false;
      const double power = s_power;
      double scale = 1.0;
      if (!(power <= ctl.pmax)) scale = sqrt(ctl.pmax / power);  // project_sum_power :257-263
      if (xo) vs1 = (float)scale; else vs0 = (float)scale;
      xc = xo;
      pc.mark(11);
      epilogue_b((float)scale, (float)ctl.omega, more);
      __syncthreads();
      pc.mark(3);
      // Gram partials of G_new -> gx[1] (lower half of the block) and of Ĝ(t+1)
      // -> gx[0] (upper half)
      if (tid < 128)
        gram_quad(Gr[GN], Gi[GN], gx[1], tid, 128);
      else if (more)
        gram_quad(Gr[GE], Gi[GE], gx[0], tid - 128, 128);
      const bool wn_spec = ctl.latched || wn;
      const bool defer = can_defer && more && ctl.latched;  // WSR(t) during GEMM-A(t+1)
      if (defer) {  // the ring will overwrite N: keep the own users' diagonal blocks
        for (int i = tid; i < KL * NN * DD; i += blockDim.x) {
          const int kl = i / (NN * DD), rem = i - kl * NN * DD, p = rem / DD, q = rem - p * DD;
          const int idx = ((k0 + kl) * NN + p) * ldg + kl * DD + q;
          gkk_save[i] = Gr[GN][idx];
          gkk_save[KL * NN * DD + i] = Gi[GN][idx];
        }
      }
      pc.mark(12);
      cl.sync();
      pc.mark(13);
      if (more) {  // both Grams at once: one DSMEM round trip
        if (tid < 128)
          gram_reduce(1, tid, 128);
        else
          gram_reduce(0, tid - 128, 128);
      } else {
        gram_reduce(1, tid, blockDim.x);
      }
      __syncthreads();
      pc.mark(4);
      constexpr bool kQuad = NN == 4 && DD == 4;
      const bool wsplit = kQuad && a.tc_wsr_split;
      if (tid < 32) {  // warp 0: WSR(t) unless deferred (with warp 3 for N = d = 4)
        if (!defer)
          wsr_warp(Gr[GN] + (size_t)k0 * NN * ldg, Gi[GN] + (size_t)k0 * NN * ldg, NN * ldg + DD, ldg, bk,
                   wsplit);
      } else if (wsplit && warp == 3) {
        if constexpr (kQuad) {
          if (!defer) {
            const quad::QuadArgs qa{Gr[GN] + (size_t)k0 * NN * ldg, Gi[GN] + (size_t)k0 * NN * ldg,
                                    NN * ldg + DD, ldg, k0, KL, gx[1], ctl.sigma2, alpha, a.trace != nullptr};
            quad::wsr_users_c(qa, wsrw);
          }
        }
      } else if (more) {  // warps 1, 2: K1(t+1) with the speculated stage flag
        k1_pipelined(GE, wn_spec, bk, bk ^ 1);
      }
      pc.mark(14);
      __syncthreads();
      pc.mark(15);
      if (more && tid == 32) k1_publish();
      cl.sync();
      pc.mark(5);
      if (a.itU) {  // block iterate of t (solvers.py:487-488), own users / columns
        const size_t it = (size_t)r * a.max_iters + (t - 1);
        double* dU = a.itU + (it * K + k0) * (size_t)NN * DD * 2;
        double* dW = a.itW + (it * K + k0) * (size_t)DD * DD * 2;
        double* dV = a.itV + (it * K + k0) * (size_t)M * DD * 2;
        for (int i = tid; i < KL * NN * DD; i += blockDim.x) {
          dU[2 * i] = ucb[bk][i].r;
          dU[2 * i + 1] = ucb[bk][i].i;
        }
        for (int i = tid; i < KL * DD * DD; i += blockDim.x) {
          dW[2 * i] = wcb[bk][i].r;
          dW[2 * i + 1] = wcb[bk][i].i;
        }
        for (int tt = 0; tt < nmtA; ++tt)
          for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
            float xr[16], xi[16];
            load_x(xc, tt, q0, xr, xi);
            const int row = 128 * tt + row_in_tile;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int jl = q0 + j, kl = jl / DD, s = jl - kl * DD;
              const size_t o = ((size_t)kl * M + row) * DD + s;
              dV[2 * o] = (double)(xr[j] * vsc(xc));
              dV[2 * o + 1] = (double)(xi[j] * vsc(xc));
            }
          }
        umma::fence_before();
      }
      // Warp 0: one batched read of the cluster's exchange slots, the state machine
      // of t and the status of K1(t+1); the other warps meanwhile gather the other
      // owners' U / α U W (valid when the speculated stage flag holds).
      if (warp == 0) {
        xs_fetch();
        if (tid == 0) {
          if (defer)
            ctl.wn_next = 1;  // state machine of t postponed; the stage flag stays latched
          else
            state_machine(t, wn, power, scale);
          if (more && (defer || !ctl.stop) && (ctl.wn_next != 0) == wn_spec) k1_status(t + 1, wn_spec);
        }
      } else if (more) {
        k1_gather(tid - 32, blockDim.x - 32);
      }
      if (defer) {
        pending = true;
        power_p = power;
        scale_p = scale;
      }
      __syncthreads();
      pc.mark(6);
      if (!defer && ctl.stop) break;
      wn = ctl.wn_next != 0;
      if (more && wn != wn_spec) {  // mis-speculated stage flag: redo K1(t+1) (same inputs)
        k1_phase(GE, wn, true, bk, bk ^ 1);
        if (tid == 0) k1_status(t + 1, wn);
        __syncthreads();
        if (ctl.stop) break;
      }
      pc.mark(7);
    }

    // ---------------- exit: stationarity residual (solvers.py:400-412) ----------------
    double residual = NAN;
    if (ctl.status == 0) {
      if (need_g) {  // a speculative step was discarded: rebuild G = H V_final into N
        tc2::drain(pipe);  // (chunks prefetched for the GEMM-A that will not run)
        __syncthreads();
        for (int t = 0; t < nmtA; ++t)
          for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
            float xr[16], xi[16];
            load_x(xc, t, q0, xr, xi);
            const int row = 128 * t + row_in_tile;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              b_store(q0 + j, row, xr[j] * vsc(xc));
              b_store(ncol + q0 + j, row, xi[j] * vsc(xc));
            }
          }
        umma::fence_proxy_async();
        umma::fence_before();
        __syncthreads();
        tc2::gemm(pipe, pc, hpB, nchB, ncol, nsets, hpA);
        epilogue_b(1.f, 0.f, false);
        __syncthreads();
      }
      const bool weighted = ctl.latched || ctl.last_weighted;
      for (int i = tid; i < KN * ldg; i += blockDim.x) {  // fresh U / W on the final G (scratch: E)
        Gr[GE][i] = Gr[GN][i];
        Gi[GE][i] = Gi[GN][i];
      }
      __syncthreads();
      gram_rows(Gr[GE], Gi[GE], gx[0], tid, blockDim.x);
      cl.sync();
      gram_reduce(0, tid, blockDim.x);
      __syncthreads();
      k1_phase(GE, weighted, false, 0, 0);
      int st = xfirst(XS_ST1);
      __syncthreads();
      if (st == 0) {
        build_yhat(GE);
        __syncthreads();
        tc2::gemm(pipe, pc, hpA, nchA, ncol, nsets, nullptr);
        const int xo = 1 - xc;
        double pw = epilogue_a(xc, xo, vsc(xc), 0.f, (float)(2.0 * ctl.gamma_safe), 0.f, false, false);
        pw = block_sum(pw, red);
        if (tid == 0) xs[XS_POWER] = pw;
        cl.sync();
        const double power = xsum(XS_POWER);
        double scale = 1.0;
        if (!(power <= ctl.pmax)) scale = sqrt(ctl.pmax / power);
        double dsum = 0.0, vsum = 0.0;
        for (int t = 0; t < nmtA; ++t)
          for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
            float cr[16], ci[16], xr[16], xi[16];
            load_x(xc, t, q0, cr, ci);
            load_x(xo, t, q0, xr, xi);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const double a_r = (double)(cr[j] * vsc(xc)), a_i = (double)(ci[j] * vsc(xc));
              const double dr = a_r - (double)(xr[j] * (float)scale);
              const double di = a_i - (double)(xi[j] * (float)scale);
              dsum += dr * dr + di * di;
              vsum += a_r * a_r + a_i * a_i;
            }
          }
        umma::fence_before();
        dsum = block_sum(dsum, red);
        vsum = block_sum(vsum, red);
        if (tid == 0) {
          xs[XS_DSUM] = dsum;
          xs[XS_VSUM] = vsum;
        }
        cl.sync();
        residual = sqrt(xsum(XS_DSUM)) / fmax(1.0, sqrt(fmax(xsum(XS_VSUM), 0.0)));
      } else if (tid == 0) {
        ctl.status = st;
      }
    }
    tc2::drain(pipe);  // prefetched chunks of a GEMM that will not run
    __syncthreads();
    umma::fence_after();
    // ---------------- write results (own users' precoders) ----------------
    {
      if (a.Vout) {
        RC<R>* Vg = reinterpret_cast<RC<R>*>(a.Vout) + ((size_t)r * K + k0) * M * DD;
        for (int t = 0; t < nmtA; ++t)
          for (int q0 = 16 * cgrp; q0 < ncol; q0 += 32) {
            float xr[16], xi[16];
            load_x(xc, t, q0, xr, xi);
            const int row = 128 * t + row_in_tile;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int jl = q0 + j, kl = jl / DD, s = jl - kl * DD;
              Vg[((size_t)kl * M + row) * DD + s] = RC<R>{xr[j] * vsc(xc), xi[j] * vsc(xc)};
            }
          }
        umma::fence_before();
      }
      if (tid == 0 && crank == 0) {
        if (a.wsr_bits) a.wsr_bits[r] = ctl.wsr / kLn2;
        if (a.iterations) a.iterations[r] = ctl.iters;
        if (a.converged) a.converged[r] = (unsigned char)ctl.converged;
        if (a.residual) a.residual[r] = residual;
        if (a.switch_it) a.switch_it[r] = ctl.switch_it;
        if (a.status) a.status[r] = ctl.status;
      }
    }
    // all remote reads of this realization's exchange buffers and every bulk
    // copy of its H planes are complete before any CTA starts the next one
    cl.sync();
    pc.mark(8);
  }
  pc.flush();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<512>(pipe.tmem);
}

}  // namespace ammmse
