// ammmse_engine.cuh — B200 persistent fused A-MMMSE solver.
//
// One CTA owns one channel realization at a time and runs the whole
// block-coordinate loop of the reference driver (pkg/src/wsrbeam/solvers.py
// _run_bcd :415-518 with exact=False, use_extrapolation=True,
// start_weighted=False) with every operand resident in shared memory:
//
//   H (KN x M), V_cur / V_old (M x Kd), G_cur / G_old (KN x Kd, G = H V).
//
// CTAs pull realization indices from an atomic counter (persistent grid,
// load-balances the per-realization iteration counts) and exit the loop of
// a realization as soon as it stops: finished problems issue no more work.
//
// Per iteration (all identities are exact rewrites of the reference blocks,
// SURVEY.md Appendix A):
//   Ĝ  = G + ω (G − G_old)                        extrapolate (solvers.py:380-390) by linearity
//   A_k = σ²I + Σ_j Ĝ_kj Ĝ_kj^H  (fp64)             update_receivers q-gram (:216-224)
//   U_k = A_k^{-1} Ĝ_kk  (fp64 Cholesky)            update_receivers (:210-225)
//   W_k = herm((I − U_k^H Ĝ_kk)^{-1}) or I          update_weight_matrices (:228-254) / stage latch (:449-464)
//   Ŷ_m = α_m U_m W_m (U_m^H Ĝ_m − S_m)             gradient factor (objective.py:172-213) in factored form
//   X   = V̂ − γ · 2 H^H Ŷ                           pgd_precoder_step (solvers.py:358-377)     [GEMM-A]
//   V   = X · min(1, sqrt(P/‖X‖²))                  project_sum_power (:257-263)
//   G   = H V                                       [GEMM-B]
//   WSR = Σ α_k (ln det(σ²I+Σ_j G G^H) − ln det(σ²I+Σ_{j≠k} G G^H))   (objective.py:108-148), fp64
//   f_after_u/w/v from the same Grams               wmmse_objective (objective.py:151-169)
//   rel / switch / stop / divergence                (solvers.py:449-505)
// Exit: stationarity residual with fresh U/W and γ_safe (solvers.py:400-412).
//
// Precision: GEMMs in R (fp32 for complex64 inputs, fp64 for complex128);
// every Gram, Cholesky, log-det, objective and WSR accumulation in fp64.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ammmse.h"
#include "small_linalg.cuh"
#include "user_algebra.cuh"

namespace ammmse {

constexpr int kMaxThreads = 256;
#ifndef AMMMSE_MINB
#define AMMMSE_MINB 3
#endif
constexpr int kTraceFields = AMMMSE_TRACE_FIELDS;
constexpr double kCondLimit = 1e12;  // solvers.py:71
constexpr double kLn2 = 0.69314718055994530942;

template <typename R>
struct RC {  // interleaved complex element of the external arrays
  R r, i;
};

// Kernel arguments (by value).
struct EngineArgs {
  const void* H;
  const double* sigma2;
  const double* pmax;
  const double* alpha;
  const void* V0;
  const double* gamma_arr;  // optional (B,)
  const double* omega_arr;  // optional (B,)
  void* Vout;
  double* wsr_bits;
  int* iterations;
  unsigned char* converged;
  double* residual;
  int* switch_it;
  int* status;
  double* gamma_used;
  double* trace;
  double* itU;  // recorded iterates (optional): (B, T, K, N, d), (B, T, K, d, d),
  double* itW;  // (B, T, K, M, d) complex128
  double* itV;
  double gamma;
  double omega, eps1, eps2;
  int gamma_safe;
  int max_iters;
  int latch;
  int M, K;
  int hres;  // cluster engine: H resident in SMEM (1) or streamed from global (0)
  int vold_glob;  // cluster engine: second V buffer in global scratch (1)
  int sb_bytes;   // cluster engine: bytes per cp.async staging buffer
  unsigned char* scratch;  // cluster engine: per-CTA global scratch (vold_glob)
  int tcm;                 // cluster engine: tcgen05 3xTF32 GEMMs (streamed H planes)
  float* hplanes;          // tcm: per-cluster pre-split H planes (8 x KN x M floats each)
  int tc_stages;           // tcm == 2 (ammmse_tc2.cuh): A ring depth
  int dbg;                 // diagnostic builds: ablation bits (AMMMSE_DBG)
  int tc_defer;            // tcm == 2: WSR(t) deferred into GEMM-A(t+1) once the stage is latched
  int tc_wsr_split;        // tcm == 2: WSR(t) on two warps (A / C factorisations concurrently)
  unsigned long long* prof;  // debug: per-phase clock64 totals (nullptr = off)
  long long B;
  unsigned long long* counter;
};

// Shared-memory layout of one realization, computed identically on host and
// device.  R region (planar re/im): H, V[2], G[2], then per-user U/P/D in R;
// fp64 region: per-user Grams, U/W caches, objective terms, reductions.
template <typename R, int NN, int DD>
struct Layout {
  int M, K, KN, KD, ldh, ldv, ldg;
  size_t nH, nV, nG;             // elements per plane
  size_t oH, oV0, oV1, oG0, oG1; // element offsets (R) of the re planes
  size_t oUPD;                   // element offset (R) of U|P|D small arrays
  size_t dbl_off;                // byte offset of fp64 region
  size_t bytes;

  __host__ __device__ void init(int M_, int K_) {
    M = M_;
    K = K_;
    KN = K * NN;
    KD = K * DD;
    // H rows 16-byte aligned (128-bit loads) and padded by 4 elements so
    // consecutive rows start 4 banks apart
    ldh = ((M + 3) & ~3) + 4;
    ldv = KD;
    ldg = KD;
    nH = (size_t)KN * ldh;
    nV = (size_t)M * ldv;
    nG = (size_t)KN * ldg;
    oH = 0;
    oV0 = oH + 2 * nH;
    oV1 = oV0 + 2 * nV;
    oG0 = oV1 + 2 * nV;
    oG1 = oG0 + 2 * nG;
    oUPD = oG1 + 2 * nG;
    size_t nR = oUPD + (size_t)3 * 2 * K * NN * DD;
    dbl_off = ((nR * sizeof(R)) + 15) & ~(size_t)15;
    bytes = dbl_off + dbl_bytes();
  }
  // fp64 region, in doubles (banks [2]: the pipelined loop runs WSR(t) and
  // K1(t+1) concurrently, so per-iteration user state is double-buffered):
  //   gram[2]   K*NN*NN cd each (2 doubles per cd): [0] Ĝ for K1, [1] G_new for WSR
  //   ucache[2] K*NN*DD cd, wcache[2] K*DD*DD cd   (bank = iteration parity)
  //   lndetw[2], fu[2], fw[2]  K each
  //   alpha, fv, rate  K each
  //   ustat, ust2  K each (k1 / wsr per-user status, stored as double)
  //   red    32
  // doubles per bank, rounded even so both banks keep 16-byte cd alignment
  __host__ __device__ size_t bank_doubles() const {
    return ((size_t)2 * K * NN * NN + 2 * K * NN * DD + 2 * K * DD * DD + 3 * K + 1) & ~(size_t)1;
  }
  __host__ __device__ size_t dbl_count() const { return 2 * bank_doubles() + 3 * K + 2 * K + 32; }
  __host__ __device__ size_t dbl_bytes() const { return dbl_count() * sizeof(double); }
};

// Debug phase timers: thread 0 of every CTA accumulates clock64() deltas per
// phase and adds them to EngineArgs::prof at exit (built with AMMMSE_PHASES=1 and run
// with AMMMSE_PROFILE_PHASES=1; the counters live in the caller's workspace).
constexpr int kProfPhases = 20;
#ifndef AMMMSE_PHASES
#define AMMMSE_PHASES 0  // compile-time switch: production kernels carry no timers
#endif
#if AMMMSE_PHASES
struct PhaseClock {
  unsigned long long* out;
  long long last;
  long long acc[kProfPhases];
  __device__ void init(unsigned long long* o) {
    out = (threadIdx.x == 0) ? o : nullptr;
    if (out) {
      last = clock64();
      for (int i = 0; i < kProfPhases; ++i) acc[i] = 0;
    }
  }
  __device__ __forceinline__ void mark(int i) {
    if (out) {
      const long long now = clock64();
      acc[i] += now - last;
      last = now;
    }
  }
  // fine-grained marks inside single-thread role loops: AMMMSE_PHASES=2 only
  // (they lengthen the loops they measure)
  __device__ __forceinline__ void mark2(int i) {
    if (AMMMSE_PHASES >= 2) mark(i);
  }
  __device__ void flush() {
    if (out)
      for (int i = 0; i < kProfPhases; ++i) atomicAdd(out + i, (unsigned long long)acc[i]);
  }
};
#else
struct PhaseClock {
  __device__ __forceinline__ void init(unsigned long long*) {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void mark2(int) {}
  __device__ __forceinline__ void flush() {}
};
#endif

// Control block of the running realization (static shared memory).
struct Ctl {
  double sigma2, pmax, gamma, gamma_safe, omega, step;
  double wsr_last, wsr_prev;  // last two completed WSR values (nats)
  int nhist;
  double running_max;
  int drop_streak;
  int latched, switch_it, weighted_now, last_weighted;
  int cur;        // index of the current V/G buffers
  int stop, status, converged, iters;
  double f_u, f_w, f_v, wsr;
  double scale, total_power;
  double vscale[2];  // V[i] holds X_i unscaled; the precoders are vscale[i] * X_i
  int wn_next;       // stage flag of the next iteration (decided by the state machine)
};

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum returned to every thread (fixed tree + fixed
// warp order), so every thread derives bit-identical control decisions.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_allsum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

// ---------------------------------------------------------------------------
// Shared-memory complex GEMM, planar operands, fp accumulate in R.
//   C(p, q) = sum_k A(p, k) * B(k, q)
//   A(p, k) = CONJT ? conj(A[k*lda + p]) : A[p*lda + k]
//   B(k, q) = B[k*ldb + q]
// Each thread owns RY x RX output tiles; lanes of a warp walk consecutive q
// tiles so B reads are contiguous and A reads broadcast.
// ---------------------------------------------------------------------------
template <typename R, int RY, int RX, bool CONJT, class Epi>
__device__ __forceinline__ void cgemm_smem(int P, int Q, int KD, const R* __restrict__ Ar,
                                           const R* __restrict__ Ai, int lda,
                                           const R* __restrict__ Br, const R* __restrict__ Bi,
                                           int ldb, Epi epi) {
  const int QT = (Q + RX - 1) / RX, PT = (P + RY - 1) / RY;
  for (int tile = threadIdx.x; tile < PT * QT; tile += blockDim.x) {
    const int p0 = (tile / QT) * RY, q0 = (tile % QT) * RX;
    int pi[RY], qj[RX];
#pragma unroll
    for (int i = 0; i < RY; ++i) pi[i] = min(p0 + i, P - 1);
#pragma unroll
    for (int j = 0; j < RX; ++j) qj[j] = min(q0 + j, Q - 1);
    R cr[RY][RX], ci[RY][RX];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j) cr[i][j] = ci[i][j] = R(0);
#pragma unroll 4
    for (int k = 0; k < KD; ++k) {
      R ar[RY], ai[RY], br[RX], bi[RX];
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int idx = CONJT ? (k * lda + pi[i]) : (pi[i] * lda + k);
        ar[i] = Ar[idx];
        ai[i] = Ai[idx];
      }
#pragma unroll
      for (int j = 0; j < RX; ++j) {
        br[j] = Br[k * ldb + qj[j]];
        bi[j] = Bi[k * ldb + qj[j]];
      }
#pragma unroll
      for (int i = 0; i < RY; ++i)
#pragma unroll
        for (int j = 0; j < RX; ++j) {
          if (CONJT) {
            cr[i][j] = fma(ar[i], br[j], fma(ai[i], bi[j], cr[i][j]));
            ci[i][j] = fma(ar[i], bi[j], fma(-ai[i], br[j], ci[i][j]));
          } else {
            cr[i][j] = fma(ar[i], br[j], fma(-ai[i], bi[j], cr[i][j]));
            ci[i][j] = fma(ar[i], bi[j], fma(ai[i], br[j], ci[i][j]));
          }
        }
    }
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j)
        if (p0 + i < P && q0 + j < Q) epi(p0 + i, q0 + j, cr[i][j], ci[i][j]);
  }
}

// ---------------------------------------------------------------------------
// Vectorised shared-memory complex GEMM (same contract as cgemm_smem).
// Planar operands are read with 128-bit loads: A runs of RY (CONJT, along p)
// or KU (!CONJT, along k), B runs of RX along q.  The K loop is split S ways
// over adjacent lanes; partials are reduced with xor-shuffles, so each tile
// costs one shuffle round per split level instead of a shared-memory pass.
// Preconditions (checked by cgemm_ok): P % RY, Q % RX, KD % (S*KU) == 0;
// lda, ldb, the plane bases and q/p offsets 16-byte aligned; tiles*S <= blockDim.
// ---------------------------------------------------------------------------
template <typename R>
struct V16;
template <>
struct V16<float> {
  using T = float4;
  static constexpr int n = 4;
};
template <>
struct V16<double> {
  using T = double2;
  static constexpr int n = 2;
};
template <typename R, int W>
__device__ __forceinline__ void vload(R (&dst)[W], const R* src) {
  using VT = typename V16<R>::T;
  constexpr int n = V16<R>::n;
  static_assert(W % n == 0, "vector width");
#pragma unroll
  for (int v = 0; v < W / n; ++v) {
    const VT x = reinterpret_cast<const VT*>(src)[v];
    if constexpr (n == 4) {
      dst[4 * v] = x.x; dst[4 * v + 1] = x.y; dst[4 * v + 2] = x.z; dst[4 * v + 3] = x.w;
    } else {
      dst[2 * v] = x.x; dst[2 * v + 1] = x.y;
    }
  }
}

template <typename R, int W>
__device__ __forceinline__ void vstore(R* dst, const R (&src)[W]) {
  using VT = typename V16<R>::T;
  constexpr int n = V16<R>::n;
  static_assert(W % n == 0, "vector width");
#pragma unroll
  for (int v = 0; v < W / n; ++v) {
    VT x;
    if constexpr (n == 4) {
      x.x = src[4 * v]; x.y = src[4 * v + 1]; x.z = src[4 * v + 2]; x.w = src[4 * v + 3];
    } else {
      x.x = src[2 * v]; x.y = src[2 * v + 1];
    }
    reinterpret_cast<VT*>(dst)[v] = x;
  }
}

template <typename R, int RY, int RX, int KU>
__host__ __device__ inline bool cgemm_ok(int P, int Q, int KD, int lda, int ldb, int S, int threads) {
  constexpr int n = 16 / (int)sizeof(R);
  if (P % RY || Q % RX || KD % (S * KU)) return false;
  if (lda % n || ldb % n) return false;
  if ((P / RY) * (Q / RX) * S > threads) return false;
  return true;
}

// split S that fills the block: largest power of two <= 8 with tiles*S <= threads
__host__ __device__ inline int pick_split(int tiles, int threads, int KD, int KU) {
  int S = 1;
  while (S < 8 && tiles * S * 2 <= threads && KD % (S * 2 * KU) == 0) S *= 2;
  return S;
}

// erow(p, q0, cr[RX], ci[RX]) receives one row run of RX consecutive outputs.
struct NoTile {
  template <class... T>
  __device__ __forceinline__ void operator()(T&&...) const {}
};

// etile(active, s, p0, q0, cr, ci) is then called by EVERY lane (inactive
// lanes too, so it may use full-warp shuffles) with the complete RY x RX tile.
template <typename R, int RY, int RX, int KU, bool CONJT, class ERow, class ETile = NoTile>
__device__ __forceinline__ void cgemm_fast(int P, int Q, int KD, int S, const R* __restrict__ Ar,
                                           const R* __restrict__ Ai, int lda,
                                           const R* __restrict__ Br, const R* __restrict__ Bi,
                                           int ldb, ERow erow, ETile etile = ETile()) {
  // operands live in shared memory: let the compiler emit LDS (not generic LD)
  __builtin_assume(__isShared(Ar));
  __builtin_assume(__isShared(Ai));
  __builtin_assume(__isShared(Br));
  __builtin_assume(__isShared(Bi));
  const int QT = Q / RX, tiles = (P / RY) * QT;
  // split-major lanes: a warp holds 32/S consecutive tiles, and the K split s
  // is the high part of the lane index, so every quarter-warp (the unit a
  // 128-bit shared load is serviced in) reads one K slice of consecutive
  // tiles: broadcast A, contiguous B, no bank conflicts between K slices
  // whose rows alias (row stride = 0 mod 32 words).
  const int lane = threadIdx.x & 31, tpw = 32 / S;
  const int s = lane / tpw;
  const int tile_raw = (threadIdx.x >> 5) * tpw + (lane - s * tpw);
  const bool active = tile_raw < tiles;
  const int tile = active ? tile_raw : 0;
  const int p0 = (tile / QT) * RY, q0 = (tile % QT) * RX;
  const int kper = KD / S, kb = s * kper;
  R cr[RY][RX], ci[RY][RX];
#pragma unroll
  for (int i = 0; i < RY; ++i)
#pragma unroll
    for (int j = 0; j < RX; ++j) cr[i][j] = ci[i][j] = R(0);
  if (active) {
    for (int k = kb; k < kb + kper; k += KU) {
      R ar[KU][RY], ai[KU][RY];
      if constexpr (CONJT) {
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          vload<R, RY>(ar[u], Ar + (k + u) * lda + p0);
          vload<R, RY>(ai[u], Ai + (k + u) * lda + p0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < RY; ++i) {
          R tr[KU], ti[KU];
          vload<R, KU>(tr, Ar + (p0 + i) * lda + k);
          vload<R, KU>(ti, Ai + (p0 + i) * lda + k);
#pragma unroll
          for (int u = 0; u < KU; ++u) { ar[u][i] = tr[u]; ai[u][i] = ti[u]; }
        }
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        R br[RX], bi[RX];
        vload<R, RX>(br, Br + (k + u) * ldb + q0);
        vload<R, RX>(bi, Bi + (k + u) * ldb + q0);
#pragma unroll
        for (int i = 0; i < RY; ++i)
#pragma unroll
          for (int j = 0; j < RX; ++j) {
            if constexpr (CONJT) {
              cr[i][j] = fma(ar[u][i], br[j], fma(ai[u][i], bi[j], cr[i][j]));
              ci[i][j] = fma(ar[u][i], bi[j], fma(-ai[u][i], br[j], ci[i][j]));
            } else {
              cr[i][j] = fma(ar[u][i], br[j], fma(-ai[u][i], bi[j], cr[i][j]));
              ci[i][j] = fma(ar[u][i], bi[j], fma(ai[u][i], br[j], ci[i][j]));
            }
          }
      }
    }
  }
  // split-K reduction over the S lanes of a tile (lane bits >= log2(32/S))
  for (int o = tpw; o < 32; o <<= 1) {
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j) {
        cr[i][j] += __shfl_xor_sync(0xffffffffu, cr[i][j], o);
        ci[i][j] += __shfl_xor_sync(0xffffffffu, ci[i][j], o);
      }
  }
  if (active) {  // lane s of the tile writes rows i = s, s+S, ... (one RX run per row)
#pragma unroll
    for (int i = 0; i < RY; ++i)
      if (i % S == s) erow(p0 + i, q0, cr[i], ci[i]);
  }
  etile(active, s, p0, q0, cr, ci);
}

// Dispatch: fast path when the shape allows, generic 2x2 path otherwise.
// epi(p, q, re, im) per element; erow(p, q0, re[RX], im[RX]) per row run on
// the fast path (vectorised epilogues: RX % (16 / sizeof(R)) == 0, output
// row stride and base 16-byte aligned).
template <typename R, int RY, int RX, bool CONJT, class Epi, class ERow>
__device__ __forceinline__ void cgemm_any2(int P, int Q, int KD, const R* Ar, const R* Ai, int lda,
                                           const R* Br, const R* Bi, int ldb, Epi epi, ERow erow) {
  constexpr int KU = 16 / (int)sizeof(R);
  const int tiles = (P % RY || Q % RX) ? 0 : (P / RY) * (Q / RX);
  const int S = tiles ? pick_split(tiles, blockDim.x, KD, CONJT ? 1 : KU) : 1;
  constexpr int KUe = CONJT ? 1 : KU;
  if (tiles && cgemm_ok<R, RY, RX, KUe>(P, Q, KD, lda, ldb, S, blockDim.x)) {
    cgemm_fast<R, RY, RX, KUe, CONJT>(P, Q, KD, S, Ar, Ai, lda, Br, Bi, ldb, erow);
  } else {
    cgemm_smem<R, 2, 2, CONJT>(P, Q, KD, Ar, Ai, lda, Br, Bi, ldb, epi);
  }
}
// Same, plus a tile hook on the fast path; returns true when the fast path ran.
template <typename R, int RY, int RX, bool CONJT, class Epi, class ERow, class ETile>
__device__ __forceinline__ bool cgemm_any3(int P, int Q, int KD, const R* Ar, const R* Ai, int lda,
                                           const R* Br, const R* Bi, int ldb, Epi epi, ERow erow,
                                           ETile etile) {
  constexpr int KU = 16 / (int)sizeof(R);
  const int tiles = (P % RY || Q % RX) ? 0 : (P / RY) * (Q / RX);
  const int S = tiles ? pick_split(tiles, blockDim.x, KD, CONJT ? 1 : KU) : 1;
  constexpr int KUe = CONJT ? 1 : KU;
  if (tiles && cgemm_ok<R, RY, RX, KUe>(P, Q, KD, lda, ldb, S, blockDim.x)) {
    cgemm_fast<R, RY, RX, KUe, CONJT>(P, Q, KD, S, Ar, Ai, lda, Br, Bi, ldb, erow, etile);
    return true;
  }
  cgemm_smem<R, 2, 2, CONJT>(P, Q, KD, Ar, Ai, lda, Br, Bi, ldb, epi);
  return false;
}

template <typename R, int RY, int RX, bool CONJT, class Epi>
__device__ __forceinline__ void cgemm_any(int P, int Q, int KD, const R* Ar, const R* Ai, int lda,
                                          const R* Br, const R* Bi, int ldb, Epi epi) {
  cgemm_any2<R, RY, RX, CONJT>(P, Q, KD, Ar, Ai, lda, Br, Bi, ldb, epi,
                               [&](int p, int q0, const R(&cr)[RX], const R(&ci)[RX]) {
#pragma unroll
                                 for (int j = 0; j < RX; ++j) epi(p, q0 + j, cr[j], ci[j]);
                               });
}

// Gram of user k over `ncols` columns of X, computed by one warp (lanes over
// columns, fp64, fixed shuffle tree); lane 0 stores the Hermitian N x N.
template <typename R, int NN>
__device__ __forceinline__ void gram_warp(int k, const R* __restrict__ Xr, const R* __restrict__ Xi,
                                         int ld, int ncols, int lane, cd* __restrict__ gram) {
  double sr[NN][NN], si[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) sr[a][b] = si[a][b] = 0.0;
  for (int j = lane; j < ncols; j += 32) {
    double gr[NN], gi[NN];
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      gr[a] = (double)Xr[(k * NN + a) * ld + j];
      gi[a] = (double)Xi[(k * NN + a) * ld + j];
    }
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) {  // g_a * conj(g_b)
        sr[a][b] = fma(gr[a], gr[b], fma(gi[a], gi[b], sr[a][b]));
        if (b < a) si[a][b] = fma(gi[a], gr[b], fma(-gr[a], gi[b], si[a][b]));
      }
  }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      sr[a][b] = warp_allsum(sr[a][b]);
      if (b < a) si[a][b] = warp_allsum(si[a][b]);
    }
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) {
        gram[(k * NN + a) * NN + b] = cmk(sr[a][b], b < a ? si[a][b] : 0.0);
        if (b < a) gram[(k * NN + b) * NN + a] = cmk(sr[a][b], -si[a][b]);
      }
  }
}

// Per-user Grams  gram[k] = sum_{j < ncols} X[kN+a][j] conj(X[kN+b][j])  (fp64),
// one warp per user (gram_warp), full Hermitian N x N stored.
template <typename R, int NN>
__device__ __forceinline__ void user_grams(const R* __restrict__ Xr, const R* __restrict__ Xi,
                                           int ld, int ncols, int K, cd* __restrict__ gram) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < K; k += nw) gram_warp<R, NN>(k, Xr, Xi, ld, ncols, lane, gram);
}

// Warp reduce-scatter of P (power of two <= 32) fp64 values: halving levels
// (each lane keeps half of its values and ships the other half to its xor
// partner), then a plain butterfly over the remaining lane bits.  P - 1 + (5 -
// log2 P) shuffles instead of 5 P.  Returns value number lane >> (5 - log2 P)
// summed over the warp, identical in every lane that holds it (fixed tree).
template <int P, int H, int O>
struct HalvingLevel {  // one halving level: keep H of 2H values, ship the others to lane ^ O
  static __device__ __forceinline__ void run(double (&v)[P], int lane) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double send = up ? v[i] : v[H + i];
      const double keep = up ? v[H + i] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    HalvingLevel<P, H / 2, O / 2>::run(v, lane);
  }
};
template <int P, int O>
struct HalvingLevel<P, 0, O> {
  static __device__ __forceinline__ void run(double (&)[P], int) {}
};
template <int P>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[P], int lane) {
  static_assert(P >= 1 && P <= 32 && (P & (P - 1)) == 0, "P power of two <= 32");
  HalvingLevel<P, P / 2, 16>::run(v, lane);
  constexpr int L = __builtin_ctz(P);
#pragma unroll
  for (int o = 16 >> L; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}

// Reduce-scatter of P values within aligned groups of G lanes (P <= G, both
// powers of two): halving levels at offsets G/2 ... G/P, then a butterfly over
// the remaining lower offsets.  Lane l returns value number (l % G) / (G / P).
template <int P, int G>
__device__ __forceinline__ double group_reduce_scatter(double (&v)[P], int lane) {
  static_assert(P >= 1 && P <= G && G <= 32 && (P & (P - 1)) == 0 && (G & (G - 1)) == 0, "");
  HalvingLevel<P, P / 2, G / 2>::run(v, lane);
#pragma unroll
  for (int o = G / P / 2; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}

// Packed Gram partial of user k over the columns j = lane, lane + 32, ... of
// X: NN*(NN+1)/2 real parts of the lower triangle (row-major), then the
// NN*(NN-1)/2 imaginary parts below the diagonal.
template <typename R, int NN>
__device__ __forceinline__ void gram_pack(const R* __restrict__ Xr, const R* __restrict__ Xi,
                                          int ld, int k, int ncols, int lane, double* out) {
  double sr[NN][NN], si[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) sr[a][b] = si[a][b] = 0.0;
  for (int j = lane; j < ncols; j += 32) {
    double gr[NN], gi[NN];
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      gr[a] = (double)Xr[(k * NN + a) * ld + j];
      gi[a] = (double)Xi[(k * NN + a) * ld + j];
    }
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) {  // g_a * conj(g_b)
        sr[a][b] = fma(gr[a], gr[b], fma(gi[a], gi[b], sr[a][b]));
        if (b < a) si[a][b] = fma(gi[a], gr[b], fma(-gr[a], gi[b], si[a][b]));
      }
  }
  int n = 0;
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) out[n++] = sr[a][b];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < a; ++b) out[n++] = si[a][b];
}

// Store packed Gram value number `idx` (gram_pack order) into the Hermitian
// N x N of user k.
template <int NN>
__device__ __forceinline__ void gram_store(int k, int idx, double val, cd* __restrict__ gram) {
  constexpr int nre = NN * (NN + 1) / 2;
  if (idx < nre) {
    int a = 0;
    while ((a + 1) * (a + 2) / 2 <= idx) ++a;
    const int b = idx - a * (a + 1) / 2;
    gram[(k * NN + a) * NN + b].r = val;
    gram[(k * NN + b) * NN + a].r = val;
    if (a == b) gram[(k * NN + a) * NN + a].i = 0.0;
  } else {
    const int m = idx - nre;
    int a = 1;
    while (a * (a + 1) / 2 <= m) ++a;
    const int b = m - a * (a - 1) / 2;
    gram[(k * NN + a) * NN + b].i = val;
    gram[(k * NN + b) * NN + a].i = -val;
  }
}

__host__ __device__ constexpr int pow2_at_least(int n) { return n <= 1 ? 1 : 2 * pow2_at_least((n + 1) / 2); }

// Grams of user k over `ncols` columns of X0 (-> gram0) and, when X1 is not
// null, of X1 (-> gram1): one warp, one packed reduce-scatter for both.
template <typename R, int NN>
__device__ __forceinline__ void gram_pair(int k, const R* X0r, const R* X0i, cd* gram0, const R* X1r,
                                          const R* X1i, cd* gram1, int ld, int ncols, int lane) {
  constexpr int V = NN * NN;
  constexpr int P = pow2_at_least(2 * V);
  double v[P];
#pragma unroll
  for (int i = 0; i < P; ++i) v[i] = 0.0;
  gram_pack<R, NN>(X0r, X0i, ld, k, ncols, lane, v);
  if (X1r) gram_pack<R, NN>(X1r, X1i, ld, k, ncols, lane, v + V);
  const double tot = warp_reduce_scatter<P>(v, lane);
  constexpr int L = __builtin_ctz(P);
  const int idx = lane >> (5 - L);
  if ((lane & ((1 << (5 - L)) - 1)) == 0) {
    if (idx < V)
      gram_store<NN>(k, idx, tot, gram0);
    else if (idx < 2 * V && X1r)
      gram_store<NN>(k, idx - V, tot, gram1);
  }
}

// ---------------------------------------------------------------------------
// The solver kernel
// ---------------------------------------------------------------------------
// Two equally spaced buffers addressed by a runtime index (no pointer array
// in local memory): view[i] = base + i * stride.
template <typename T>
struct Pair {
  T* base;
  size_t stride;
  __device__ __forceinline__ T* operator[](int i) const { return base + (size_t)i * stride; }
};

// Operands that live in shared memory: lets the compiler emit LDS/STS with
// 32-bit addresses instead of generic 64-bit LD/ST.  Only for pointers that
// are never null.
#define AMMMSE_SHARED(p) __builtin_assume(__isShared(p))

template <typename R, int NN, int DD>
struct Engine {
  using L_t = Layout<R, NN, DD>;

  // smem views
  R *Hr, *Hi;
  Pair<R> Vr, Vi, Gr, Gi;
  RC<R>*Uf, *Pf, *Df;  // per user N x d, R
  Pair<cd> gramb, ucb, wcb;
  Pair<double> lndb, fub, fwb;
  double *alpha, *fv, *rate, *ustat, *ust2, *red;
  L_t L;

  __device__ void bind(unsigned char* smem, int M, int K) {
    L.init(M, K);
    R* base = reinterpret_cast<R*>(smem);
    Hr = base + L.oH;
    Hi = Hr + L.nH;
    // V[1] follows V[0] (re, im planes) and G[1] follows G[0]: see Layout
    Vr = Pair<R>{base + L.oV0, L.oV1 - L.oV0};
    Vi = Pair<R>{base + L.oV0 + L.nV, L.oV1 - L.oV0};
    Gr = Pair<R>{base + L.oG0, L.oG1 - L.oG0};
    Gi = Pair<R>{base + L.oG0 + L.nG, L.oG1 - L.oG0};
    Uf = reinterpret_cast<RC<R>*>(base + L.oUPD);
    Pf = Uf + K * NN * DD;
    Df = Pf + K * NN * DD;
    double* d = reinterpret_cast<double*>(smem + L.dbl_off);
    {  // bank b of each array at + b * bank (doubles)
      const size_t bank = L.bank_doubles();
      const size_t bank_cd = bank / 2;
      double* const d0 = d;
      gramb = Pair<cd>{reinterpret_cast<cd*>(d), bank_cd}; d += 2 * K * NN * NN;
      ucb = Pair<cd>{reinterpret_cast<cd*>(d), bank_cd}; d += 2 * K * NN * DD;
      wcb = Pair<cd>{reinterpret_cast<cd*>(d), bank_cd}; d += 2 * K * DD * DD;
      lndb = Pair<double>{d, bank}; d += K;
      fub = Pair<double>{d, bank}; d += K;
      fwb = Pair<double>{d, bank}; d += K;
      d = d0 + 2 * bank;
    }
    alpha = d; d += K;
    fv = d; d += K;
    rate = d; d += K;
    ustat = d; d += K;
    ust2 = d; d += K;
    red = d;
  }

  // Receiver / weight / gradient-factor update of user k from the Gram in
  // gramb[0] and the work G (Ĝ).  Reads W_prev from bank `bin`; writes U/P/D
  // (R) for the Ŷ phase, the fp64 U/W caches and objective terms of bank
  // `bout`, and the per-user status.
  __device__ void k1_user(int k, const R* Gwr, const R* Gwi, int ldg, double sigma2, bool weighted,
                          bool want_f, int bin, int bout) {
    const cd* gram = gramb[0];
    const cd* wprev = wcb[bin];
    cd* ucache = ucb[bout];
    cd* wcache = wcb[bout];
    AMMMSE_SHARED(gram);
    AMMMSE_SHARED(wprev);
    AMMMSE_SHARED(ucache);
    AMMMSE_SHARED(wcache);
    AMMMSE_SHARED(Gwr);
    AMMMSE_SHARED(Gwi);
    AMMMSE_SHARED(Df);
    AMMMSE_SHARED(Uf);
    AMMMSE_SHARED(Pf);
    AMMMSE_SHARED(alpha);
    AMMMSE_SHARED(ustat);
    cd Tg[NN][NN], Gkk[NN][DD], Wp[DD][DD];
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b < NN; ++b) Tg[a][b] = gram[(k * NN + a) * NN + b];
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int s = 0; s < DD; ++s) {
        const int idx = (k * NN + a) * ldg + k * DD + s;
        Gkk[a][s] = cmk((double)Gwr[idx], (double)Gwi[idx]);
      }
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) Wp[p][q] = wprev[(k * DD + p) * DD + q];
    K1Out<NN, DD> o;
    k1_math<NN, DD>(Tg, Gkk, sigma2, alpha[k], Wp, lndb[bin][k], weighted, want_f, o);
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        const int i = (k * NN + a) * DD + q;
        Df[i] = RC<R>{(R)o.D[a][q].r, (R)o.D[a][q].i};
        Pf[i] = RC<R>{(R)o.P[a][q].r, (R)o.P[a][q].i};
        Uf[i] = RC<R>{(R)o.U[a][q].r, (R)o.U[a][q].i};
        ucache[i] = o.U[a][q];
      }
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) wcache[(k * DD + p) * DD + q] = o.W[p][q];
    lndb[bout][k] = o.lndetw;
    fub[bout][k] = o.fu;
    fwb[bout][k] = o.fw;
    ustat[k] = o.status;
  }

  // Rate and f_after_v terms of user k from the Gram of G_new.
  // Gram of G_new in gramb[1]; U / W of bank b.
  __device__ void wsr_user(int k, const R* Gnr, const R* Gni, int ldg, double sigma2, int b) {
    const cd* gram = gramb[1];
    const cd* ucache = ucb[b];
    const cd* wcache = wcb[b];
    AMMMSE_SHARED(gram);
    AMMMSE_SHARED(ucache);
    AMMMSE_SHARED(wcache);
    AMMMSE_SHARED(Gnr);
    AMMMSE_SHARED(Gni);
    AMMMSE_SHARED(alpha);
    AMMMSE_SHARED(rate);
    AMMMSE_SHARED(fv);
    AMMMSE_SHARED(ust2);
    cd Tg[NN][NN], Gkk[NN][DD], U[NN][DD], W[DD][DD];
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b < NN; ++b) Tg[a][b] = gram[(k * NN + a) * NN + b];
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int s = 0; s < DD; ++s) {
        const int idx = (k * NN + a) * ldg + k * DD + s;
        Gkk[a][s] = cmk((double)Gnr[idx], (double)Gni[idx]);
        U[a][s] = ucache[(k * NN + a) * DD + s];
      }
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) W[p][q] = wcache[(k * DD + p) * DD + q];
    double r, f;
    int st;
    wsr_math<NN, DD>(Tg, Gkk, sigma2, alpha[k], U, W, lndb[b][k], r, f, st);
    rate[k] = r;
    fv[k] = f;
    ust2[k] = st;
  }

  // Gram of user k over `ncols` columns of X (one warp, gram_warp)
  __device__ void gram_user(int k, const R* __restrict__ Xr, const R* __restrict__ Xi, int ld,
                            int ncols, int lane, cd* gram) {
    AMMMSE_SHARED(Xr);
    AMMMSE_SHARED(Xi);
    AMMMSE_SHARED(gram);
    gram_warp<R, NN>(k, Xr, Xi, ld, ncols, lane, gram);
  }

  // Gram(Ĝ) on all warps | receiver / weight / gradient factors with lanes =
  // users (as few warps as possible: the fp64 per-user code is issued once per
  // warp) | Ŷ on all threads.  Two block barriers.
  __device__ void phase_k1_yhat(R* Gwr, R* Gwi, double sigma2, bool weighted, bool want_f,
                                int bin, int bout) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int K = L.K, KD = L.KD, ldg = L.ldg;
    for (int k = warp; k < K; k += nw) gram_user(k, Gwr, Gwi, ldg, KD, lane, gramb[0]);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x)
      k1_user(k, Gwr, Gwi, ldg, sigma2, weighted, want_f, bin, bout);
    __syncthreads();
    build_yhat(Gwr, Gwi, ldg, K, KD);
  }

  // Ŷ in place over the work G: (m, j) pairs, j fastest.
  __device__ void build_yhat(R* Gwr, R* Gwi, int ldg, int K, int KD) {
    AMMMSE_SHARED(Gwr);
    AMMMSE_SHARED(Gwi);
    AMMMSE_SHARED(Df);
    AMMMSE_SHARED(Uf);
    AMMMSE_SHARED(Pf);
    for (int idx = threadIdx.x; idx < K * KD; idx += blockDim.x) {
      const int m = idx / KD, j = idx - m * KD;
      const int b = j / DD, s = j - b * DD;
      R yr[NN], yi[NN];
      if (b == m) {
#pragma unroll
        for (int a = 0; a < NN; ++a) {
          const RC<R> v = Df[(m * NN + a) * DD + s];
          yr[a] = v.r;
          yi[a] = v.i;
        }
      } else {
        R gr[NN], gi[NN];
#pragma unroll
        for (int a = 0; a < NN; ++a) {
          gr[a] = Gwr[(m * NN + a) * ldg + j];
          gi[a] = Gwi[(m * NN + a) * ldg + j];
        }
        R qr[DD], qi[DD];
#pragma unroll
        for (int p = 0; p < DD; ++p) {  // q = U_m^H g
          R sr = 0, si = 0;
#pragma unroll
          for (int a = 0; a < NN; ++a) {
            const RC<R> u = Uf[(m * NN + a) * DD + p];
            sr = fma(u.r, gr[a], fma(u.i, gi[a], sr));
            si = fma(u.r, gi[a], fma(-u.i, gr[a], si));
          }
          qr[p] = sr;
          qi[p] = si;
        }
#pragma unroll
        for (int a = 0; a < NN; ++a) {  // y = P_m q
          R sr = 0, si = 0;
#pragma unroll
          for (int p = 0; p < DD; ++p) {
            const RC<R> pp = Pf[(m * NN + a) * DD + p];
            sr = fma(pp.r, qr[p], fma(-pp.i, qi[p], sr));
            si = fma(pp.r, qi[p], fma(pp.i, qr[p], si));
          }
          yr[a] = sr;
          yi[a] = si;
        }
      }
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        Gwr[(m * NN + a) * ldg + j] = yr[a];
        Gwi[(m * NN + a) * ldg + j] = yi[a];
      }
    }
  }

  // GEMM-B: G[dst] = H · V[src].  With ghat >= 0 the epilogue also writes the
  // next iteration's extrapolated Ĝ = G + ω (G − G_prev) (solvers.py:380-390,
  // by linearity) over G[ghat], which holds G_prev = the current G.
  //
  // fuse_gram: also form the fp64 Grams of G[dst] (-> gramb[1]) and of Ĝ (->
  // gramb[0]) in the tile epilogue, when the tile layout allows (N = 2 = tile
  // rows, split S <= 2, a user's QT >= 8 column tiles in consecutive lanes):
  // each lane packs the partial Grams of its 2 x 4 tile, and a group
  // reduce-scatter over the user's QT lanes finishes them (no separate Gram
  // pass, one block barrier fewer).  Returns whether the Grams were formed.
  __device__ bool gemm_hv(int src, int dst, int ghat = -1, double omega = 0.0,
                          double vscale = 1.0, bool fuse_gram = false) {
    R* gr = Gr[dst];
    R* gi = Gi[dst];
    R* hr = ghat >= 0 ? Gr[ghat] : nullptr;
    R* hi = ghat >= 0 ? Gi[ghat] : nullptr;
    const R om = (R)omega, sc = (R)vscale;
    const int ldg = L.ldg;
    AMMMSE_SHARED(gr);
    AMMMSE_SHARED(gi);
    constexpr int RX = 4;
    bool fuse = false;
    int QT = 0;
    if constexpr (NN == 2) {
      if (fuse_gram && L.KD % RX == 0) {
        constexpr int KU = 16 / (int)sizeof(R);
        QT = L.KD / RX;
        const int tiles = (L.KN / 2) * QT;
        const int S = pick_split(tiles, blockDim.x, L.M, KU);
        fuse = S <= 2 && QT >= 8 && (QT & (QT - 1)) == 0 && QT <= 32 / S &&
               cgemm_ok<R, 2, RX, KU>(L.KN, L.KD, L.M, L.ldh, L.ldv, S, blockDim.x);
      }
    }
    cd* gnew = gramb[1];
    cd* ghatg = gramb[0];
    auto etile = [&](bool active, int s, int p0, int q0, const R(&cr)[2][RX],
                     const R(&ci)[2][RX]) {
      if constexpr (NN == 2) {
        if (!fuse) return;
        const int lane = threadIdx.x & 31;
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.0;
        __syncwarp();  // Ĝ rows stored by the tile's other split lane are visible
        if (active) {
#pragma unroll
          for (int j = 0; j < RX; ++j) {  // gram_pack order: (0,0) (1,0) (1,1) re, (1,0) im
            const double g0r = (double)(cr[0][j] * sc), g0i = (double)(ci[0][j] * sc);
            const double g1r = (double)(cr[1][j] * sc), g1i = (double)(ci[1][j] * sc);
            v[0] = fma(g0r, g0r, fma(g0i, g0i, v[0]));
            v[1] = fma(g1r, g0r, fma(g1i, g0i, v[1]));
            v[2] = fma(g1r, g1r, fma(g1i, g1i, v[2]));
            v[3] = fma(g1i, g0r, fma(-g1r, g0i, v[3]));
          }
          if (hr) {
            AMMMSE_SHARED(hr);
            AMMMSE_SHARED(hi);
            R h0r[RX], h0i[RX], h1r[RX], h1i[RX];
            vload<R, RX>(h0r, hr + p0 * ldg + q0);
            vload<R, RX>(h0i, hi + p0 * ldg + q0);
            vload<R, RX>(h1r, hr + (p0 + 1) * ldg + q0);
            vload<R, RX>(h1i, hi + (p0 + 1) * ldg + q0);
#pragma unroll
            for (int j = 0; j < RX; ++j) {
              const double g0r = h0r[j], g0i = h0i[j], g1r = h1r[j], g1i = h1i[j];
              v[4] = fma(g0r, g0r, fma(g0i, g0i, v[4]));
              v[5] = fma(g1r, g0r, fma(g1i, g0i, v[5]));
              v[6] = fma(g1r, g1r, fma(g1i, g1i, v[6]));
              v[7] = fma(g1i, g0r, fma(-g1r, g0i, v[7]));
            }
          }
        }
        double tot;
        int idx;
        if (QT == 8) {
          tot = group_reduce_scatter<8, 8>(v, lane);
          idx = lane & 7;
        } else if (QT == 16) {
          tot = group_reduce_scatter<8, 16>(v, lane);
          idx = (lane & 15) >> 1;
        } else {
          tot = group_reduce_scatter<8, 32>(v, lane);
          idx = lane >> 2;
        }
        const int sub = QT / 8;  // lanes per value
        if (active && s == 0 && (lane % sub) == 0) {
          const int k = p0 / 2;
          if (idx < 4)
            gram_store<2>(k, idx, tot, gnew);
          else if (hr)
            gram_store<2>(k, idx - 4, tot, ghatg);
        }
      }
    };
    const bool fast = cgemm_any3<R, 2, RX, false>(
        L.KN, L.KD, L.M, Hr, Hi, L.ldh, Vr[src], Vi[src], L.ldv,
        [&](int p, int q, R cr, R ci) {
          const int o = p * ldg + q;
          cr *= sc;  // G = H (c X) = c (H X): projection applied lazily
          ci *= sc;
          gr[o] = cr;
          gi[o] = ci;
          if (hr) {  // ω = 0: plain copy (G_prev may be uninitialised shared memory)
            AMMMSE_SHARED(hr);
            AMMMSE_SHARED(hi);
            hr[o] = om == R(0) ? cr : cr + om * (cr - hr[o]);
            hi[o] = om == R(0) ? ci : ci + om * (ci - hi[o]);
          }
        },
        [&](int p, int q0, const R(&cr)[RX], const R(&ci)[RX]) {  // 128-bit row runs
          const int o = p * ldg + q0;
          R c_r[RX], c_i[RX];
#pragma unroll
          for (int j = 0; j < RX; ++j) {
            c_r[j] = cr[j] * sc;
            c_i[j] = ci[j] * sc;
          }
          vstore<R, RX>(gr + o, c_r);
          vstore<R, RX>(gi + o, c_i);
          if (hr) {
            AMMMSE_SHARED(hr);
            AMMMSE_SHARED(hi);
            R h_r[RX], h_i[RX];
            if (om == R(0)) {  // plain copy (G_prev may be uninitialised shared memory)
#pragma unroll
              for (int j = 0; j < RX; ++j) {
                h_r[j] = c_r[j];
                h_i[j] = c_i[j];
              }
            } else {
              vload<R, RX>(h_r, hr + o);
              vload<R, RX>(h_i, hi + o);
#pragma unroll
              for (int j = 0; j < RX; ++j) {
                h_r[j] = c_r[j] + om * (c_r[j] - h_r[j]);
                h_i[j] = c_i[j] + om * (c_i[j] - h_i[j]);
              }
            }
            vstore<R, RX>(hr + o, h_r);
            vstore<R, RX>(hi + o, h_i);
          }
        },
        etile);
    return fast && fuse;
  }

  // GEMM-A + projection input: X = V̂ − step · H^H Ŷ into V[dst] (unscaled).
  // V̂ = sc·Xc + ω (sc·Xc − so·Xo) when extrap, else sc·Xc, where V[vcur] = Xc
  // and V[dst] = Xo hold the unscaled iterates (solvers.py:380-390, :358-377).
  // Per-warp ‖X‖² partials go to red[warp]; after the caller's barrier every
  // thread sums them (warp order) -> power, identical in all threads.
  __device__ void gemm_grad_step(int ysrc, int vcur, int dst, double step, double omega,
                                 bool extrap, double sc_cur, double sc_old) {
    const R* vcr = Vr[vcur];
    const R* vci = Vi[vcur];
    R* xr = Vr[dst];
    R* xi = Vi[dst];
    AMMMSE_SHARED(vcr);
    AMMMSE_SHARED(vci);
    AMMMSE_SHARED(xr);
    AMMMSE_SHARED(xi);
    AMMMSE_SHARED(red);
    const int ldv = L.ldv;
    const R st = (R)step, om = (R)omega, sc = (R)sc_cur, so = (R)sc_old;
    double pw = 0.0;
    constexpr int RX = 4;
    cgemm_any2<R, 4, RX, true>(
        L.M, L.KD, L.KN, Hr, Hi, L.ldh, Gr[ysrc], Gi[ysrc], L.ldg,
        [&](int p, int q, R gr, R gi) {
          const int o = p * ldv + q;
          R vr = sc * vcr[o], vi = sc * vci[o];
          if (extrap) {  // cur + ω (cur − prev)   (solvers.py:390)
            vr = vr + om * (vr - so * xr[o]);
            vi = vi + om * (vi - so * xi[o]);
          }
          const R x_r = vr - st * gr;
          const R x_i = vi - st * gi;
          xr[o] = x_r;
          xi[o] = x_i;
          pw += (double)x_r * (double)x_r + (double)x_i * (double)x_i;
        },
        [&](int p, int q0, const R(&gr)[RX], const R(&gi)[RX]) {  // 128-bit row runs
          const int o = p * ldv + q0;
          R vr[RX], vi[RX];
          vload<R, RX>(vr, vcr + o);
          vload<R, RX>(vi, vci + o);
          if (extrap) {
            R pr[RX], pi[RX];
            vload<R, RX>(pr, xr + o);
            vload<R, RX>(pi, xi + o);
#pragma unroll
            for (int j = 0; j < RX; ++j) {
              vr[j] = sc * vr[j];
              vi[j] = sc * vi[j];
              vr[j] = vr[j] + om * (vr[j] - so * pr[j]);
              vi[j] = vi[j] + om * (vi[j] - so * pi[j]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < RX; ++j) {
              vr[j] = sc * vr[j];
              vi[j] = sc * vi[j];
            }
          }
#pragma unroll
          for (int j = 0; j < RX; ++j) {
            vr[j] = vr[j] - st * gr[j];
            vi[j] = vi[j] - st * gi[j];
            pw += (double)vr[j] * (double)vr[j] + (double)vi[j] * (double)vi[j];
          }
          vstore<R, RX>(xr + o, vr);
          vstore<R, RX>(xi + o, vi);
        });
    pw = warp_allsum(pw);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  }
  // sum of the per-warp partials (call after a barrier)
  __device__ double red_total() const {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    return s;
  }
};

// MC, KC != 0: shape-specialised instantiation (M = MC, K = KC, NT threads),
// so tile plans, split factors, loop trip counts and index arithmetic fold to
// constants (the planner selects it when the dims match, entries.h).
// MB: resident CTAs per SM the register budget is sized for (N d <= 4).
template <typename R, int NN, int DD, int MC = 0, int KC = 0, int NT = kMaxThreads,
          int MB = AMMMSE_MINB>
__global__ void __launch_bounds__(kMaxThreads, (NN * DD <= 4) ? MB : 1) ammmse_solve_kernel(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Ctl ctl;
  __shared__ unsigned long long s_r;
  if constexpr (MC > 0) __builtin_assume(blockDim.x == NT);
  Engine<R, NN, DD> e;
  const int M = MC > 0 ? MC : a.M, K = KC > 0 ? KC : a.K, KN = K * NN, KD = K * DD;
  e.bind(smem, M, K);
  const int tid = threadIdx.x;
  const int ldh = e.L.ldh, ldv = e.L.ldv, ldg = e.L.ldg;
  PhaseClock pc;
  pc.init(a.prof);

  for (;;) {
    if (tid == 0) s_r = atomicAdd(a.counter, 1ULL);
    __syncthreads();
    const long long r = (long long)s_r;
    if (r >= a.B) break;

    // ---------------- load realization r ----------------
    {
      const RC<R>* Hg = reinterpret_cast<const RC<R>*>(a.H) + (size_t)r * KN * M;
      for (int i = tid; i < KN * M; i += blockDim.x) {
        const int row = i / M, col = i - row * M;
        const RC<R> v = Hg[i];
        e.Hr[row * ldh + col] = v.r;
        e.Hi[row * ldh + col] = v.i;
      }
      // V0 (K, M, d) -> V[0] (M x Kd), column k*d+s
      const RC<R>* Vg = reinterpret_cast<const RC<R>*>(a.V0) + (size_t)r * K * M * DD;
      for (int i = tid; i < K * M * DD; i += blockDim.x) {
        const int k = i / (M * DD), rem = i - k * M * DD, m = rem / DD, s = rem - m * DD;
        const RC<R> v = Vg[i];
        e.Vr[0][m * ldv + k * DD + s] = v.r;
        e.Vi[0][m * ldv + k * DD + s] = v.i;
      }
      for (int k = tid; k < K; k += blockDim.x) {
        e.alpha[k] = a.alpha[(size_t)r * K + k];
        e.lndb[0][k] = 0.0;  // W_prev = I at t = 1 (solvers.py:429-430); K1(1) reads bank 0
        for (int p = 0; p < DD; ++p)
          for (int q = 0; q < DD; ++q) e.wcb[0][(k * DD + p) * DD + q] = cmk(p == q ? 1.0 : 0.0);
      }
      if (tid == 0) {
        ctl.sigma2 = a.sigma2[r];
        ctl.pmax = a.pmax[r];
        ctl.omega = a.omega_arr ? a.omega_arr[r] : a.omega;
        ctl.nhist = 0;
        ctl.wsr_last = ctl.wsr_prev = 0.0;
        ctl.running_max = -INFINITY;
        ctl.drop_streak = 0;
        ctl.latched = 0;  // start_weighted=False for A-MMMSE (solvers.py:549-550)
        ctl.switch_it = -1;
        ctl.weighted_now = 0;
        ctl.last_weighted = 0;
        ctl.cur = 0;
        ctl.stop = 0;
        ctl.status = 0;
        ctl.converged = 0;
        ctl.iters = 0;
        ctl.f_u = ctl.f_w = ctl.f_v = ctl.wsr = 0.0;
        ctl.vscale[0] = ctl.vscale[1] = 1.0;
      }
    }
    __syncthreads();

    // ---------------- bounds: kappa, gamma_safe (objective.py:216-240) ----------------
    user_grams<R, NN>(e.Hr, e.Hi, ldh, M, K, e.gramb[0]);
    __syncthreads();
    for (int k = tid; k < K; k += blockDim.x) {
      cd G[NN][NN];
      for (int p = 0; p < NN; ++p)
        for (int q = 0; q < NN; ++q) G[p][q] = e.gramb[0][(k * NN + p) * NN + q];
      e.rate[k] = herm_eig_max<NN>(G);
    }
    __syncthreads();
    if (tid == 0) {
      double kappa = 0.0, abar = e.alpha[0];
      for (int k = 0; k < K; ++k) {
        kappa = fmax(kappa, e.rate[k]);
        abar = fmax(abar, e.alpha[k]);
      }
      const double l_v = 2.0 * abar * K * kappa / ctl.sigma2;
      ctl.gamma_safe = 1.0 / l_v;
      ctl.gamma = a.gamma_arr ? a.gamma_arr[r] : (a.gamma_safe ? ctl.gamma_safe : a.gamma);
      ctl.step = 2.0 * ctl.gamma;
      if (a.gamma_used) a.gamma_used[r] = ctl.gamma;
    }
    // initial G = H V0 into G[0]; Ĝ(1) = G (no extrapolation at t = 1) into G[1]
    e.gemm_hv(0, 0, 1, 0.0);
    __syncthreads();

    // ---------------- K1(1) (solvers.py:440-460 at t = 1) ----------------
    // Stage flag of iteration t (solvers.py:449-459), from the shared state.
    auto stage_flag = [&]() -> bool {
      if (ctl.latched) return true;
      double rs = INFINITY;
      if (ctl.nhist >= 2) {
        const double den = fabs(ctl.wsr_prev);
        rs = den == 0.0 ? INFINITY : fabs(ctl.wsr_last - ctl.wsr_prev) / den;
      }
      return rs <= a.eps1;
    };
    bool wn = stage_flag();  // the flag K1(t) was computed with
    {
      const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
      for (int k = warp; k < K; k += nw) e.gram_user(k, e.Gr[1], e.Gi[1], ldg, KD, lane, e.gramb[0]);
      __syncthreads();
      for (int k = tid; k < K; k += blockDim.x)
        e.k1_user(k, e.Gr[1], e.Gi[1], ldg, ctl.sigma2, wn, true, 0, 1);
      __syncthreads();
    }

    pc.mark(7);  // setup: load, bounds, G = H V0, K1(1)
    // ---------------- main loop (solvers.py:440-505), software-pipelined ----------------
    // Per iteration t: Ŷ(t) | GEMM-A + ‖X‖² | GEMM-B (+ Ĝ(t+1)) | Gram(G_new) and
    // Gram(Ĝ(t+1)) on all warps | warp 0: rates, reductions, state machine of t
    // while warps 1.. run the receiver / weight update K1(t+1) of the next
    // iteration.  K1(t+1) needs the stage flag of t+1, which the state machine
    // of t decides: it is speculated (latched, or unchanged) and K1(t+1) is
    // recomputed from the same inputs when the speculation was wrong (at most
    // at the stage switch).  Results are identical to the sequential order:
    // K1(t+1) reads only Ĝ(t+1), W(t) and the stage flag.  U/W/f terms are
    // double-buffered by iteration parity.  5 block barriers per iteration.
    for (int t = 1; t <= a.max_iters; ++t) {
      const int cur = ctl.cur, oth = 1 - cur;
      const int bk = t & 1;  // bank holding K1(t)'s U / W / f terms
      {  // update_weight_matrices raised inside iteration t (solvers.py:455-460)
        const int lane = tid & 31;
        int f1 = K;
        for (int k = lane; k < K; k += 32)
          if (f1 == K && e.ustat[k] != 0.0) f1 = k;
        f1 = __reduce_min_sync(0xffffffffu, f1);
        if (f1 < K) {
          if (tid == 0) {
            if (!ctl.latched && wn) {
              if (a.latch) ctl.latched = 1;
              if (ctl.switch_it < 0) ctl.switch_it = t;
            }
            ctl.status = (int)e.ustat[f1];
            ctl.stop = 1;
          }
          break;
        }
      }
      const bool extrap = (t >= 2) && (ctl.omega > 0.0);
      pc.mark(0);
      e.build_yhat(e.Gr[oth], e.Gi[oth], ldg, K, KD);
      __syncthreads();
      pc.mark(1);
      // X = V̂ − γ ∇ into V[oth] (unscaled), ‖X‖² partials (solvers.py:358-377)
      e.gemm_grad_step(oth, cur, oth, ctl.step, ctl.omega, extrap, ctl.vscale[cur],
                       ctl.vscale[oth]);
      __syncthreads();
      pc.mark(2);
      // projection (solvers.py:257-263), applied lazily: V_new = scale * X
      const double power = e.red_total();
      const double pmax = ctl.pmax;
      double scale = 1.0;
      if (!(power <= pmax)) scale = sqrt(pmax / power);
      // G_new = H V_new = scale (H X) over Ŷ; next Ĝ over G_cur (which becomes G_old)
      // (Grams of G_new -> gramb[1] and Ĝ(t+1) -> gramb[0] in its tile epilogue
      // when the layout allows)
      const bool fused = e.gemm_hv(oth, oth, cur, ctl.omega, scale, true);
      // speculated stage flag of t+1: read before the barrier (thread 0 updates
      // ctl.latched in the next phase)
      const bool wn_spec = ctl.latched || wn;
      const bool more = t < a.max_iters;
      __syncthreads();
      pc.mark(3);
      if (!fused) {  // Gram(G_new) -> gramb[1] and Gram(Ĝ(t+1)) -> gramb[0], one warp per user
        const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
        for (int k = warp; k < K; k += nw)
          gram_pair<R, NN>(k, e.Gr[oth], e.Gi[oth], e.gramb[1], more ? e.Gr[cur] : nullptr,
                           e.Gi[cur], e.gramb[0], ldg, KD, lane);
        __syncthreads();
      }
      pc.mark(4);
      if (a.itU) {  // block iterate of t (solvers.py:487-488): U(t), W(t), V_new(t) = scale X
        const size_t it = (size_t)r * a.max_iters + (t - 1);
        double* dU = a.itU + it * (size_t)K * NN * DD * 2;
        double* dW = a.itW + it * (size_t)K * DD * DD * 2;
        double* dV = a.itV + it * (size_t)K * M * DD * 2;
        for (int i = tid; i < K * NN * DD; i += blockDim.x) {
          dU[2 * i] = e.ucb[bk][i].r;
          dU[2 * i + 1] = e.ucb[bk][i].i;
        }
        for (int i = tid; i < K * DD * DD; i += blockDim.x) {
          dW[2 * i] = e.wcb[bk][i].r;
          dW[2 * i + 1] = e.wcb[bk][i].i;
        }
        const R sc = (R)scale;
        for (int i = tid; i < K * M * DD; i += blockDim.x) {
          const int k = i / (M * DD), rem = i - k * M * DD, m = rem / DD, s = rem - m * DD;
          const int o = m * ldv + k * DD + s;
          dV[2 * i] = (double)(sc * e.Vr[oth][o]);
          dV[2 * i + 1] = (double)(sc * e.Vi[oth][o]);
        }
      }
      if (tid < 32) {  // warp 0: rates (lanes = users), reductions, state machine
        const int lane = tid;
        for (int k = lane; k < K; k += 32) e.wsr_user(k, e.Gr[oth], e.Gi[oth], ldg, ctl.sigma2, bk);
        __syncwarp();
        const double* fu = e.fub[bk];
        const double* fw = e.fwb[bk];
        double su = 0.0, sw = 0.0, sr = 0.0, sv = 0.0;
        int f2 = K;  // first user with a nonzero rate status
        for (int k = lane; k < K; k += 32) {
          su += fu[k];
          sw += fw[k];
          sr += e.rate[k];
          sv += e.fv[k];
          if (f2 == K && e.ust2[k] != 0.0) f2 = k;
        }
        su = warp_allsum(su);
        sw = warp_allsum(sw);
        sr = warp_allsum(sr);
        sv = warp_allsum(sv);
        f2 = __reduce_min_sync(0xffffffffu, f2);
        if (lane == 0) {
          if (!ctl.latched && wn) {
            if (a.latch) ctl.latched = 1;
            if (ctl.switch_it < 0) ctl.switch_it = t;
          }
          ctl.f_u = su;
          ctl.f_w = sw;
          {
            const double wsr = sr;
            int st = f2 < K ? (int)e.ust2[f2] : 0;
            const double total_power = scale == 1.0 ? power : power * scale * scale;
            if (!isfinite(wsr) || !isfinite(power)) st = AMMMSE_STATUS_NONFINITE;
            double rel = INFINITY;  // solvers.py:474, _rel_change :393-397
            if (t > 1) {
              const double den = fabs(ctl.wsr_last);
              rel = den == 0.0 ? INFINITY : fabs(wsr - ctl.wsr_last) / den;
            }
            ctl.wsr_prev = ctl.wsr_last;
            ctl.wsr_last = wsr;
            ctl.nhist += 1;
            ctl.iters = t;
            ctl.wsr = wsr;
            ctl.f_v = sv;
            ctl.vscale[oth] = scale;
            ctl.weighted_now = wn;
            ctl.last_weighted = wn;
            if (a.trace) {
              double* tr = a.trace + ((size_t)r * a.max_iters + (t - 1)) * kTraceFields;
              tr[AMMMSE_TRACE_T] = (double)t;
              tr[AMMMSE_TRACE_WSR_BITS] = wsr / kLn2;
              tr[AMMMSE_TRACE_F_VALUE] = sv;
              tr[AMMMSE_TRACE_TOTAL_POWER] = total_power;
              tr[AMMMSE_TRACE_STAGE] = wn ? 1.0 : 0.0;
              tr[AMMMSE_TRACE_F_AFTER_U] = su;
              tr[AMMMSE_TRACE_F_AFTER_W] = sw;
              tr[AMMMSE_TRACE_F_AFTER_V] = sv;
              tr[AMMMSE_TRACE_REL_CHANGE] = rel;
            }
            // divergence detector (solvers.py:490-500)
            ctl.running_max = fmax(ctl.running_max, wsr);
            if (wsr < 0.5 * ctl.running_max)
              ctl.drop_streak += 1;
            else
              ctl.drop_streak = 0;
            if (ctl.drop_streak >= 5 && st == 0) st = AMMMSE_STATUS_UNSTABLE;
            if (st) {
              ctl.status = st;
              ctl.stop = 1;
            } else {
              ctl.cur = oth;  // shift (solvers.py:502)
              if (wn && rel <= a.eps2) {  // stop test (:503-505)
                ctl.converged = 1;
                ctl.stop = 1;
              }
            }
          }
          ctl.wn_next = stage_flag();
        }
      } else if (more) {  // warps 1..: K1(t+1) with the speculated stage flag
        for (int k = tid - 32; k < K; k += blockDim.x - 32)
          e.k1_user(k, e.Gr[cur], e.Gi[cur], ldg, ctl.sigma2, wn_spec, true, bk, bk ^ 1);
      }
      __syncthreads();
      pc.mark(5);
      if (ctl.stop) break;
      wn = ctl.wn_next != 0;
      if (more && wn != wn_spec) {  // mis-speculated stage flag: redo K1(t+1)
        for (int k = tid; k < K; k += blockDim.x)
          e.k1_user(k, e.Gr[cur], e.Gi[cur], ldg, ctl.sigma2, wn, true, bk, bk ^ 1);
        __syncthreads();
      }
    }

    // ---------------- exit: stationarity residual (solvers.py:400-412, :507-509) ----------------
    __syncthreads();  // thread 0's stop / status writes
    double residual = NAN;
    if (ctl.status == 0) {
      const int cur = ctl.cur, oth = 1 - cur;
      const bool weighted = ctl.latched || ctl.last_weighted;
      for (int i = tid; i < KN * KD; i += blockDim.x) {
        const int row = i / KD, col = i - row * KD, o = row * ldg + col;
        e.Gr[oth][o] = e.Gr[cur][o];
        e.Gi[oth][o] = e.Gi[cur][o];
      }
      __syncthreads();
      e.phase_k1_yhat(e.Gr[oth], e.Gi[oth], ctl.sigma2, weighted, false, 0, 1);
      __syncthreads();
      if (tid == 0) {
        int st = 0;
        for (int k = 0; k < K; ++k)
          if (st == 0 && e.ustat[k] != 0.0) st = (int)e.ustat[k];
        ctl.status = st;
      }
      __syncthreads();
      if (ctl.status == 0) {
        const double vs = ctl.vscale[cur];
        e.gemm_grad_step(oth, cur, oth, 2.0 * ctl.gamma_safe, 0.0, false, vs, 1.0);
        __syncthreads();
        const double power = e.red_total();
        double scale = 1.0;
        if (!(power <= ctl.pmax)) scale = sqrt(ctl.pmax / power);
        double dsum = 0.0, vsum = 0.0;
        const R* vr = e.Vr[cur];
        const R* vi = e.Vi[cur];
        const R* xr = e.Vr[oth];
        const R* xi = e.Vi[oth];
        const R vsr = (R)vs;
        for (int i = tid; i < M * KD; i += blockDim.x) {
          const int row = i / KD, col = i - row * KD, o = row * ldv + col;
          const double a_r = (double)(vsr * vr[o]), a_i = (double)(vsr * vi[o]);
          const double dr = a_r - (double)((R)(xr[o] * (R)scale));
          const double di = a_i - (double)((R)(xi[o] * (R)scale));
          dsum += dr * dr + di * di;
          vsum += a_r * a_r + a_i * a_i;
        }
        __syncthreads();  // every thread has read the power partials in red[]
        dsum = block_sum(dsum, e.red);
        vsum = block_sum(vsum, e.red);
        residual = sqrt(dsum) / fmax(1.0, sqrt(fmax(vsum, 0.0)));
      }
    }

    pc.mark(8);  // exit: stationarity residual
    // ---------------- write results ----------------
    {
      const int cur = ctl.cur;
      if (a.Vout) {
        RC<R>* Vg = reinterpret_cast<RC<R>*>(a.Vout) + (size_t)r * K * M * DD;
        const R vs = (R)ctl.vscale[cur];
        for (int i = tid; i < K * M * DD; i += blockDim.x) {
          const int k = i / (M * DD), rem = i - k * M * DD, m = rem / DD, s = rem - m * DD;
          Vg[i] = RC<R>{vs * e.Vr[cur][m * ldv + k * DD + s], vs * e.Vi[cur][m * ldv + k * DD + s]};
        }
      }
      if (tid == 0) {
        if (a.wsr_bits) a.wsr_bits[r] = ctl.wsr / kLn2;
        if (a.iterations) a.iterations[r] = ctl.iters;
        if (a.converged) a.converged[r] = (unsigned char)ctl.converged;
        if (a.residual) a.residual[r] = residual;
        if (a.switch_it) a.switch_it[r] = ctl.switch_it;
        if (a.status) a.status[r] = ctl.status;
      }
    }
    __syncthreads();
    pc.mark(6);
  }
  pc.flush();
}

// ---------------------------------------------------------------------------
// Standalone bounds kernel: one CTA per realization (objective.py:216-240)
// ---------------------------------------------------------------------------
template <typename R, int NN>
__global__ void __launch_bounds__(128) ammmse_bounds_kernel(const void* H, const double* alpha,
                                                           const double* pmax,
                                                           const double* sigma2, int M, int K,
                                                           long long B, double* out) {
  __shared__ double lam[1024];
  const long long r = blockIdx.x;
  if (r >= B) return;
  const RC<R>* Hg = reinterpret_cast<const RC<R>*>(H) + (size_t)r * K * NN * M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < K; k += nw) {
    double sr[NN][NN], si[NN][NN];
    for (int p = 0; p < NN; ++p)
      for (int q = 0; q < NN; ++q) sr[p][q] = si[p][q] = 0.0;
    for (int m = lane; m < M; m += 32) {
      double gr[NN], gi[NN];
      for (int p = 0; p < NN; ++p) {
        const RC<R> v = Hg[(size_t)(k * NN + p) * M + m];
        gr[p] = v.r;
        gi[p] = v.i;
      }
      for (int p = 0; p < NN; ++p)
        for (int q = 0; q < NN; ++q) {
          sr[p][q] = fma(gr[p], gr[q], fma(gi[p], gi[q], sr[p][q]));
          si[p][q] = fma(gi[p], gr[q], fma(-gr[p], gi[q], si[p][q]));
        }
    }
    cd G[NN][NN];
    for (int p = 0; p < NN; ++p)
      for (int q = 0; q < NN; ++q) G[p][q] = cmk(warp_allsum(sr[p][q]), warp_allsum(si[p][q]));
    if (lane == 0 && k < 1024) lam[k] = herm_eig_max<NN>(G);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double kappa = 0.0, abar = alpha[(size_t)r * K];
    for (int k = 0; k < K; ++k) {
      kappa = fmax(kappa, lam[k]);
      abar = fmax(abar, alpha[(size_t)r * K + k]);
    }
    const double s2 = sigma2[r];
    const double l_v = 2.0 * abar * K * kappa / s2;
    double* o = out + (size_t)r * AMMMSE_BOUND_FIELDS;
    o[AMMMSE_BOUND_KAPPA] = kappa;
    o[AMMMSE_BOUND_L_V] = l_v;
    o[AMMMSE_BOUND_GAMMA_SAFE] = 1.0 / l_v;
    o[AMMMSE_BOUND_EK_FLOOR] = s2 / (pmax[r] * kappa + s2);
    o[AMMMSE_BOUND_ALPHA_BAR] = abar;
  }
}

}  // namespace ammmse
