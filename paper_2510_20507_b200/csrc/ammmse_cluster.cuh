// ammmse_cluster.cuh — A-MMMSE engine for realizations whose state does not
// fit one SM (BASELINE configs 2-4, sweep M >= 128): one thread-block
// CLUSTER of C CTAs per realization.
//
// Partition: CTA c owns users [c*K/C, (c+1)*K/C), i.e. the matching columns
// of V (M x Kd) and G (KN x Kd).  H (KN x M) is replicated in every CTA's
// shared memory.  Both GEMMs then need only local columns:
//     G[:, own] = H V[:, own]          ∇[:, own] = H^H Ŷ[:, own]
// and the only cross-CTA traffic per iteration is O(K N^2) through
// distributed shared memory (DSMEM):
//   * per-user N x N Gram partials  sum_{j in own cols} G_kj G_kj^H  (fp64),
//     summed by the user's owner in fixed rank order;
//   * the owners' U_k, α_k U_k W_k (needed by every column block of Ŷ);
//   * per-CTA scalar partials (objective terms, ‖X‖², rates, status),
//     summed by every CTA in fixed rank order, so all CTAs take bit-identical
//     stage / stop / divergence decisions without a broadcast.
// Five cluster barriers per iteration.  Reference semantics are those of
// ammmse_engine.cuh (solvers.py:415-518); the per-user math is shared
// (user_algebra.cuh).
#pragma once

#include <cooperative_groups.h>

#include "ammmse_engine.cuh"
#include "tc_stream.cuh"

namespace ammmse {

namespace cg = cooperative_groups;

// exchange-scalar slots (per CTA, read by every CTA of the cluster)
enum XSlot {
  XS_FU = 0, XS_FW, XS_ST1, XS_POWER, XS_RATE, XS_FV, XS_ST2, XS_KAPPA, XS_DSUM, XS_VSUM,
  XS_ST3, XS_COUNT
};

// ---------------------------------------------------------------------------
// Streamed complex GEMM for realizations whose H does not fit in SMEM.
//   C(p,q) = sum_k A(p,k) B(k,q),  B planar in SMEM (B[k*ldb+q])
//   CONJT : A(p,k) = conj(H[k][p])   chunk = H rows [k0, k0+KC)      (KC x P, contiguous)
//   !CONJT: A(p,k) = H[p][k]         chunk = H cols [k0, k0+KC)      (P x KC, row segments)
// H (global, interleaved complex, row length ldH) is staged chunk by chunk
// through a double-buffered SMEM ring with cp.async (16-byte pieces), the
// next chunk in flight while the current one is consumed.  Every thread
// owns up to TPT register tiles of RY x RX outputs for the whole K loop.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

struct NoPre {
  __device__ __forceinline__ void operator()() const {}
};

// `pre()` runs after the K loop, once the staging ring is free and before the
// epilogue (all threads): used to stage epilogue operands that live in global
// memory into the ring (V_old with h_placement 3).
template <typename R, int RY, int RX, int TPT, bool CONJT, class Epi, class Pre = NoPre>
__device__ __forceinline__ void cgemm_stream(int P, int Q, int KD, const RC<R>* __restrict__ Hg,
                                             int ldH, RC<R>* __restrict__ stage, int SB,
                                             const R* __restrict__ Br, const R* __restrict__ Bi,
                                             int ldb, Epi epi, Pre pre = Pre()) {
  constexpr int EPC = 16 / sizeof(RC<R>);  // complex elements per 16-byte piece (2 or 1)
  // chunk extent along k; !CONJT rows are padded by EPC elements (bank spread,
  // 16-byte aligned row starts), so P * (KC + EPC) <= SB
  const int KC = CONJT ? SB / P : ((SB / P - EPC) / EPC) * EPC;
  const int lds = CONJT ? P : KC + EPC;     // staging row stride (elements)
  const int nchunks = (KD + KC - 1) / KC;
  const int QT = (Q + RX - 1) / RX, PT = (P + RY - 1) / RY, ntiles = PT * QT;

  auto issue = [&](int c, int buf) {
    const int k0 = c * KC;
    const int kc = min(KC, KD - k0);
    RC<R>* dst = stage + (size_t)buf * SB;
    if (CONJT) {  // rows k0..k0+kc of H, each P long: contiguous block
      const RC<R>* src = Hg + (size_t)k0 * ldH;
      const int pieces = (kc * P) / EPC;
      for (int i = threadIdx.x; i < pieces; i += blockDim.x) {
        const int e = i * EPC, row = e / P, col = e - row * P;
        cp_async16(dst + row * lds + col, src + (size_t)row * ldH + col);
      }
    } else {      // columns k0..k0+kc of every row p
      const int ppr = kc / EPC;  // pieces per row (kc multiple of EPC except the tail)
      for (int i = threadIdx.x; i < P * ppr; i += blockDim.x) {
        const int row = i / ppr, e = (i - row * ppr) * EPC;
        cp_async16(dst + row * lds + e, Hg + (size_t)row * ldH + k0 + e);
      }
    }
    cp_async_commit();
  };

  R cr[TPT][RY][RX], ci[TPT][RY][RX];
#pragma unroll
  for (int t = 0; t < TPT; ++t)
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j) cr[t][i][j] = ci[t][i][j] = R(0);

  issue(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue(c + 1, (c + 1) & 1);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    const RC<R>* A = stage + (size_t)(c & 1) * SB;
    const int k0 = c * KC, kc = min(KC, KD - k0);
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int tile = threadIdx.x + t * blockDim.x;
      if (tile >= ntiles) break;
      const int p0 = (tile / QT) * RY, q0 = (tile % QT) * RX;
      int pi[RY], qj[RX];
#pragma unroll
      for (int i = 0; i < RY; ++i) pi[i] = min(p0 + i, P - 1);
#pragma unroll
      for (int j = 0; j < RX; ++j) qj[j] = min(q0 + j, Q - 1);
      for (int kk = 0; kk < kc; ++kk) {
        R ar[RY], ai[RY], br[RX], bi[RX];
#pragma unroll
        for (int i = 0; i < RY; ++i) {
          const RC<R> v = CONJT ? A[kk * lds + pi[i]] : A[pi[i] * lds + kk];
          ar[i] = v.r;
          ai[i] = v.i;
        }
#pragma unroll
        for (int j = 0; j < RX; ++j) {
          br[j] = Br[(k0 + kk) * ldb + qj[j]];
          bi[j] = Bi[(k0 + kk) * ldb + qj[j]];
        }
#pragma unroll
        for (int i = 0; i < RY; ++i)
#pragma unroll
          for (int j = 0; j < RX; ++j) {
            if (CONJT) {
              cr[t][i][j] = fma(ar[i], br[j], fma(ai[i], bi[j], cr[t][i][j]));
              ci[t][i][j] = fma(ar[i], bi[j], fma(-ai[i], br[j], ci[t][i][j]));
            } else {
              cr[t][i][j] = fma(ar[i], br[j], fma(-ai[i], bi[j], cr[t][i][j]));
              ci[t][i][j] = fma(ar[i], bi[j], fma(ai[i], br[j], ci[t][i][j]));
            }
          }
      }
    }
    __syncthreads();  // buffer (c & 1) may be refilled by the next issue
  }
  pre();
#pragma unroll
  for (int t = 0; t < TPT; ++t) {
    const int tile = threadIdx.x + t * blockDim.x;
    if (tile >= ntiles) break;
    const int p0 = (tile / QT) * RY, q0 = (tile % QT) * RX;
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j)
        if (p0 + i < P && q0 + j < Q) epi(p0 + i, q0 + j, cr[t][i][j], ci[t][i][j]);
  }
}

// ---------------------------------------------------------------------------
// Multi-stage streamed GEMM (v2).  One RY x RX register tile per thread for the
// whole K loop (tiles <= blockDim), H chunks staged through NST ring buffers
// (cp.async, NST-1 chunks in flight), one barrier per chunk, 128-bit loads for
// B (planar, along q) and for A (interleaved complex runs along p (CONJT) or k).
//   CONJT : chunk = H rows [k0, k0+KC)     staged [kk][p]   (lds = P)
//   !CONJT: chunk = H cols [k0, k0+KC)     staged [p][kk]   (lds = KC + 2, rows
//           144 B apart for KC = 16 so neighbouring rows hit different banks)
// Preconditions (stream2_ok): P % RY == Q % RX == 0, tiles <= blockDim, Q % 4,
// ldb % 4 == 0 (float), P*(KC+2) <= SB etc.
// ---------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ int stream2_kc(bool conjt, int P, int SB) {
  constexpr int EPC = 16 / sizeof(RC<R>);
  if (conjt) return (SB / P) & ~1;  // the k loop consumes k-steps in pairs
  int kc = 16;
  while (kc > EPC && P * (kc + EPC) > SB) kc >>= 1;
  return kc;
}

template <typename R, int RY, int RX, bool CONJT>
__host__ __device__ inline bool stream2_ok(int P, int Q, int KD, int ldb, int SB, int threads) {
  constexpr int n = 16 / (int)sizeof(R);
  constexpr int EPC = 16 / (int)sizeof(RC<R>);
  if (sizeof(R) != 4) return false;  // 128-bit A loads pair two complex64 values
  if (P % RY || Q % RX || RX % n || ldb % n || KD % 2 || RY % 2) return false;
  if ((P / RY) * (Q / RX) > threads) return false;
  if (CONJT) {
    if (SB / P < 2 || P % EPC || (RY * (int)sizeof(RC<R>)) % 16) return false;
  } else {
    if (P * (2 * EPC) > SB) return false;
  }
  return true;
}

template <typename R, int RY, int RX, int NST, bool CONJT, class Epi, class Pre = NoPre>
__device__ __forceinline__ void cgemm_stream2(int P, int Q, int KD, const RC<R>* __restrict__ Hg,
                                              int ldH, RC<R>* __restrict__ stage, int SB,
                                              const R* __restrict__ Br, const R* __restrict__ Bi,
                                              int ldb, Epi epi, Pre pre = Pre()) {
  constexpr int EPC = 16 / sizeof(RC<R>);  // complex per 16-byte piece
  const int KC = stream2_kc<R>(CONJT, P, SB);
  const int lds = CONJT ? P : KC + EPC;
  const int nchunks = (KD + KC - 1) / KC;
  // operands in shared memory -> LDS (generic LD would sit on the long scoreboard)
  __builtin_assume(__isShared(stage));
  __builtin_assume(__isShared(Br));
  __builtin_assume(__isShared(Bi));
  const int QT = Q / RX, ntiles = (P / RY) * QT;
  const bool active = threadIdx.x < ntiles;
  const int tile = active ? threadIdx.x : 0;
  const int p0 = (tile / QT) * RY, q0 = (tile % QT) * RX;

  // per-thread copy cursor: (row, element) of this thread's first 16-byte piece,
  // advanced incrementally (no integer division in the chunk loop)
  const int stride_e = blockDim.x * EPC;
  auto issue = [&](int c) {
    if (c < nchunks) {
      const int k0 = c * KC, kc = min(KC, KD - k0);
      RC<R>* dst = stage + (size_t)(c % NST) * SB;
      if (CONJT) {  // kc rows of P elements, contiguous in global and in the stage
        const RC<R>* src = Hg + (size_t)k0 * ldH;
        const int total = kc * P;
        if (ldH == P) {
          for (int e = threadIdx.x * EPC; e < total; e += stride_e) cp_async16(dst + e, src + e);
        } else {
          int row = (threadIdx.x * EPC) / P, col = threadIdx.x * EPC - row * P;
          const int drow = stride_e / P, dcol = stride_e - drow * P;
          for (int e = threadIdx.x * EPC; e < total; e += stride_e) {
            cp_async16(dst + row * lds + col, src + (size_t)row * ldH + col);
            row += drow;
            col += dcol;
            if (col >= P) { col -= P; ++row; }
          }
        }
      } else {      // P rows, kc elements each (row segments)
        const int rowlen = ((kc + EPC - 1) / EPC) * EPC;
        const int drow = stride_e / rowlen, de = stride_e - drow * rowlen;
        int row = (threadIdx.x * EPC) / rowlen, e = threadIdx.x * EPC - row * rowlen;
        while (row < P) {
          cp_async16(dst + row * lds + e, Hg + (size_t)row * ldH + k0 + e);
          row += drow;
          e += de;
          if (e >= rowlen) { e -= rowlen; ++row; }
        }
      }
    }
    cp_async_commit();  // (possibly empty) group keeps the wait count uniform
  };

  R cr[RY][RX], ci[RY][RX];
#pragma unroll
  for (int i = 0; i < RY; ++i)
#pragma unroll
    for (int j = 0; j < RX; ++j) cr[i][j] = ci[i][j] = R(0);

#pragma unroll
  for (int c = 0; c < NST - 1; ++c) issue(c);
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NST - 2) : "memory");
    __syncthreads();          // chunk c visible; buffer (c-1) % NST free
    issue(c + NST - 1);
    const RC<R>* A = stage + (size_t)(c % NST) * SB;
    const int k0 = c * KC, kc = min(KC, KD - k0);
    if (active) {
      // k-steps in pairs: 128-bit loads of two complex A values per load and
      // both B rows issued before the 2 x RY x RX x 4 FMAs (latency overlap)
#pragma unroll 2
      for (int kk = 0; kk < kc; kk += 2) {
        R ar[2][RY], ai[2][RY], br[2][RX], bi[2][RX];
        if constexpr (CONJT) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const RC<R>* a = A + (kk + u) * lds + p0;
#pragma unroll
            for (int i = 0; i < RY; i += 2) {
              R t[4];
              vload<R, 4>(t, reinterpret_cast<const R*>(a + i));
              ar[u][i] = t[0]; ai[u][i] = t[1]; ar[u][i + 1] = t[2]; ai[u][i + 1] = t[3];
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < RY; ++i) {
            R t[4];
            vload<R, 4>(t, reinterpret_cast<const R*>(A + (p0 + i) * lds + kk));
            ar[0][i] = t[0]; ai[0][i] = t[1]; ar[1][i] = t[2]; ai[1][i] = t[3];
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          vload<R, RX>(br[u], Br + (k0 + kk + u) * ldb + q0);
          vload<R, RX>(bi[u], Bi + (k0 + kk + u) * ldb + q0);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < RY; ++i)
#pragma unroll
            for (int j = 0; j < RX; ++j) {
              if constexpr (CONJT) {
                cr[i][j] = fma(ar[u][i], br[u][j], fma(ai[u][i], bi[u][j], cr[i][j]));
                ci[i][j] = fma(ar[u][i], bi[u][j], fma(-ai[u][i], br[u][j], ci[i][j]));
              } else {
                cr[i][j] = fma(ar[u][i], br[u][j], fma(-ai[u][i], bi[u][j], cr[i][j]));
                ci[i][j] = fma(ar[u][i], bi[u][j], fma(ai[u][i], br[u][j], ci[i][j]));
              }
            }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();  // ring free for the next GEMM
  pre();
  if (active) {
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int j = 0; j < RX; ++j) epi(p0 + i, q0 + j, cr[i][j], ci[i][j]);
  }
}

constexpr int kStreamStages = 4;
constexpr int kTcStages = 4;  // bulk-copy ring depth of the tensor-core GEMM (tc_stream.cuh)

// tensor-core mode: UMMA tile height for a GEMM with `rows` output rows
__host__ __device__ inline int tc_tm(int rows) { return rows >= 128 ? 128 : 64; }
// TMEM columns (power of two >= 32) for accumulators of 8 * ncol columns per tile
__host__ __device__ inline int tc_tmem_cols(int M, int KN, int ncol) {
  const int tA = M / tc_tm(M), tB = KN / tc_tm(KN);
  const int need = 8 * ncol * (tA > tB ? tA : tB);
  int c = 32;
  while (c < need) c <<= 1;
  return c;
}
// tensor-core mode shape rules: UMMA M tiles of 64 (single) or 128 rows, N =
// 4 ncol <= 256 in multiples of 16 (epilogue column blocks), K steps of 8,
// accumulators within the 512 TMEM columns
__host__ __device__ inline bool tc_shape_ok(int M, int KN, int ncol) {
  auto rows_ok = [](int r) { return r == 64 || (r % 128 == 0 && r > 0); };
  if (!rows_ok(M) || !rows_ok(KN) || ncol % 16 || 4 * ncol > 256) return false;
  return tc_tmem_cols(M, KN, ncol) <= 512;
}

constexpr int kStreamRY = 4, kStreamRX = 2, kStreamTPT = 4;

// threads per CTA of the cluster engine (512 was measured slower: register cap
// -> spills in the GEMM loops, half-idle GEMM-B tiles)
template <int NN, int DD>
constexpr int kClusterThreads = 256;

template <typename R, int NN, int DD>
struct CLayout {
  int M, K, C, KL, KN, KD, ncol, ldh, ldv, ldg;
  int hres;  // 1: H resident in SMEM;  0: H streamed from global through `stage`
  int vglob; // 1: the second V buffer lives in a per-CTA global scratch slot (L2)
  int tc;    // 1: tensor-core GEMMs; the H region holds the tcgen05 operand ring
  int tc_a, tc_b;  // bytes of one ring stage's A / B tile (tensor-core mode)
  int SB;    // staging buffer size (complex elements) when streamed
  size_t nH, nV, nG;
  size_t oH, oV0, oV1, oG0, oG1, oUall, oPall, oDown;  // R offsets (planar / RC)
  size_t dbl_off, bytes;

  __host__ __device__ void init(int M_, int K_, int C_, int hres_ = 1, int vglob_ = 0,
                                int sb_bytes = 20480, int tc_ = 0) {
    hres = hres_;
    vglob = vglob_;
    tc = tc_;
    SB = sb_bytes / (int)(2 * sizeof(R));  // per staging buffer (kStreamStages of them)
    M = M_;
    K = K_;
    C = C_;
    KL = K / C;
    KN = K * NN;
    KD = K * DD;
    ncol = KL * DD;
    ldh = ((M + 3) & ~3) + 4;
    // tensor-core epilogues walk rows one thread per row: odd row strides keep
    // those column sweeps free of bank conflicts (the FFMA GEMMs need ncol)
    ldv = tc_ ? ncol + 1 : ncol;
    ldg = tc_ ? ncol + 1 : ncol;
    nV = (size_t)M * ldv;
    nG = (size_t)KN * ldg;
    // resident: planar H (2 planes of KN x ldh); streamed: kStreamStages buffers of SB
    // interleaved complex = 2*kStreamStages*SB reals = 2 "planes" of kStreamStages*SB
    nH = hres ? (size_t)KN * ldh : (size_t)kStreamStages * SB;
    tc_a = 4 * (KN > M ? KN : M) * tcs::KW * 4;
    tc_b = 4 * ncol * tcs::KW * 4;
    if (tc) nH = ((size_t)kTcStages * (tc_a + tc_b) / sizeof(R) + 1) / 2;  // ring reals = 2 nH
    oH = 0;
    oV0 = oH + 2 * nH;
    oV1 = oV0 + 2 * nV;
    oG0 = oV1 + (vglob ? 0 : 2 * nV);
    oG1 = oG0 + 2 * nG;
    oUall = oG1 + 2 * nG;                       // RC<R>[K*NN*DD]
    oPall = oUall + (size_t)2 * K * NN * DD;
    oDown = oPall + (size_t)2 * K * NN * DD;    // RC<R>[KL*NN*DD]
    const size_t nR = oDown + (size_t)2 * KL * NN * DD;
    dbl_off = ((nR * sizeof(R)) + 15) & ~(size_t)15;
    bytes = dbl_off + dbl_count() * sizeof(double);
  }
  // fp64 region: gx[2] (K*NN*NN cd each), ucache[2] (KL*NN*DD cd each),
  // wcache[2] (KL*DD*DD cd each), lndetw[2], alpha_own, fu, fw, fv, rate,
  // ust, ust2 (KL each), xs (XS_COUNT), red (32).  [2] = bank by iteration
  // parity: WSR(t) and K1(t+1) run concurrently.
  __host__ __device__ size_t dbl_count() const {
    return (size_t)2 * 2 * K * NN * NN + 2 * 2 * KL * NN * DD + 2 * 2 * KL * DD * DD + 9 * KL +
           XS_COUNT + k1w_count() + 32;
  }
  // split-K1 exchange (k1_pipelined; the N = d = 2 closed form does not use it)
  __host__ __device__ size_t k1w_count() const {
    return (NN == 2 && DD == 2) ? 0 : (size_t)KL * (2 * DD * DD + NN + 1);
  }
};

// TC = true: the tcgen05 GEMM variant (separate instantiation, so the FFMA
// kernel carries none of its code, registers or local arrays).
// MC, KC, CC != 0: shape-specialised instantiation (M, K, cluster size and
// the 256-thread block known at compile time; the planner selects it when the
// dims and its plan match, entries.h).
// SBC != 0 (specialisations only): the plan's placement is fixed too (H streamed,
// V_old in the global slot, SBC-byte staging buffers).
template <typename R, int NN, int DD, bool TC = false, int MC = 0, int KC = 0, int CC = 0,
          int SBC = 0>
__global__ void __launch_bounds__(kClusterThreads<NN, DD>, 1) ammmse_cluster_kernel(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Ctl ctl;
  __shared__ unsigned long long s_r;
  if constexpr (MC > 0) __builtin_assume(blockDim.x == kClusterThreads<NN, DD>);
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int C = CC > 0 ? CC : (int)cl.num_blocks();
  const int tid = threadIdx.x;

  CLayout<R, NN, DD> L;
  L.init(MC > 0 ? MC : a.M, KC > 0 ? KC : a.K, C, SBC > 0 ? 0 : a.hres, SBC > 0 ? 1 : a.vold_glob,
         SBC > 0 ? SBC : a.sb_bytes, TC ? 1 : 0);
  const bool hres = SBC > 0 ? false : a.hres != 0;
  const int M = L.M, K = L.K, KL = L.KL, KN = L.KN, ncol = L.ncol;
  const int ldh = L.ldh, ldv = L.ldv, ldg = L.ldg;
  const int k0 = crank * KL;       // first own user
  const int col0 = crank * ncol;   // first own global column

  R* base = reinterpret_cast<R*>(smem);
  R* Hr = base + L.oH;
  R* Hi = Hr + L.nH;
  RC<R>* stage = reinterpret_cast<RC<R>*>(base + L.oH);  // streamed mode
  const RC<R>* Hcur = nullptr;                            // this realization's H in global
  R *Vr[2], *Vi[2], *Gr[2], *Gi[2];
  Vr[0] = base + L.oV0; Vi[0] = Vr[0] + L.nV;
  if (L.vglob) {  // V_old slot in global scratch (generic pointers: every path works)
    Vr[1] = reinterpret_cast<R*>(a.scratch) + (size_t)blockIdx.x * 2 * L.nV;
  } else {
    Vr[1] = base + L.oV1;
  }
  Vi[1] = Vr[1] + L.nV;
  Gr[0] = base + L.oG0; Gi[0] = Gr[0] + L.nG;
  Gr[1] = base + L.oG1; Gi[1] = Gr[1] + L.nG;
  RC<R>* Uall = reinterpret_cast<RC<R>*>(base + L.oUall);
  RC<R>* Pall = reinterpret_cast<RC<R>*>(base + L.oPall);
  RC<R>* Down = reinterpret_cast<RC<R>*>(base + L.oDown);
  double* dp = reinterpret_cast<double*>(smem + L.dbl_off);
  cd* gx[2];
  gx[0] = reinterpret_cast<cd*>(dp); dp += 2 * K * NN * NN;
  gx[1] = reinterpret_cast<cd*>(dp); dp += 2 * K * NN * NN;
  const Pair<cd> ucb{reinterpret_cast<cd*>(dp), (size_t)KL * NN * DD};  // bank b: ucb[b]
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
  double* k1w = dp; dp += L.k1w_count();  // split-K1 exchange
  double* red = dp;

  // ---- tensor-core mode: bulk-copy ring with full / done mbarriers, TMEM accumulators ----
  __shared__ uint64_t tc_full[kTcStages], tc_bready[kTcStages], tc_done[kTcStages], tc_fin;
  __shared__ uint32_t tc_tmem_slot;
  tcs::Pipe pipe;
  pipe.ring = reinterpret_cast<unsigned char*>(base + L.oH);
  pipe.S = kTcStages;
  pipe.a_bytes = L.tc_a;
  pipe.stage_bytes = L.tc_a + L.tc_b;
  pipe.full = tc_full;
  pipe.bready = tc_bready;
  pipe.done = tc_done;
  pipe.fin = &tc_fin;
  pipe.tmem = 0;
  tcs::Seq tc_seq;             // pipeline position (identical in every thread)
  const float* hpB = nullptr;  // pre-split H planes (rows r, K = m), this cluster's slot
  const float* hpA = nullptr;  // pre-split H^T planes (rows m, K = r)
  const int tmA = tc_tm(M), tmB = tc_tm(KN);
  if constexpr (TC) {
    if (tid == 0) {
      for (int q = 0; q < kTcStages; ++q) {
        umma::mbar_init(&tc_full[q], 1);
        umma::mbar_init(&tc_bready[q], 1);  // the producing warp (tcs::gemm)
        umma::mbar_init(&tc_done[q], 1);
      }
      umma::mbar_init(&tc_fin, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if ((tid >> 5) == 0) umma::tmem_alloc<512>(&tc_tmem_slot);  // one CTA per SM
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    pipe.tmem = tc_tmem_slot;
    const size_t hp = (size_t)8 * L.KN * L.M;
    float* slot = a.hplanes + (size_t)(blockIdx.x / C) * hp;
    hpB = slot;
    hpA = slot + (size_t)4 * L.KN * L.M;
  }

  // fixed-order cluster sum / first-nonzero of an exchange slot
  auto xsum = [&](int slot) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += cl.map_shared_rank(xs, c)[slot];
    return s;
  };
  auto xfirst = [&](int slot) {
    for (int c = 0; c < C; ++c) {
      const double v = cl.map_shared_rank(xs, c)[slot];
      if (v != 0.0) return (int)v;
    }
    return 0;
  };
  // partial Grams over own columns for ALL users: gx[buf][k] (warp per user)
  auto gram_partials = [&](const R* Xr, const R* Xi, int buf) {
    user_grams<R, NN>(Xr, Xi, ldg, ncol, K, gx[buf]);
  };
  // cluster sum of the own users' Gram partials, all threads in parallel (the
  // remote DSMEM loads are independent; fixed rank order), written back over
  // this CTA's own-user slots of gx[buf]: only this CTA reads those slots
  // (every CTA sums the slots of ITS users), and each element is read and
  // rewritten by one thread.  Called after the cluster barrier that publishes
  // gx[buf]; the partials are not rewritten before the next cluster barrier.
  auto gram_reduce = [&](int buf) {
    constexpr int per = NN * NN;
    for (int i = tid; i < KL * per; i += blockDim.x) {
      const size_t gi = (size_t)k0 * per + i;
      cd s = cl.map_shared_rank(gx[buf], 0)[gi];
      for (int c = 1; c < C; ++c) s = cadd(s, cl.map_shared_rank(gx[buf], c)[gi]);
      gx[buf][gi] = s;
    }
  };
  // reduced Gram of own user kl (after gram_reduce(buf) and a block barrier)
  auto gram_of = [&](int buf, int kl, cd (&Tg)[NN][NN]) {
    const cd* g = gx[buf] + (size_t)(k0 + kl) * NN * NN;
#pragma unroll
    for (int p = 0; p < NN; ++p)
#pragma unroll
      for (int q = 0; q < NN; ++q) Tg[p][q] = g[p * NN + q];
  };
  // per-user K1 of own users kl = first, first + step, ... from the reduced
  // Gram gx[0] and the work Ĝ in G[gsrc]; W_prev / ln det W_prev from bank
  // bin, U / W / ln det W to bank bout (solvers.py:210-254)
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
        const int ig = ((k0 + kl) * NN + p) * DD + q, il = (kl * NN + p) * DD + q;
        Uall[ig] = RC<R>{(R)o.U[p][q].r, (R)o.U[p][q].i};
        Pall[ig] = RC<R>{(R)o.P[p][q].r, (R)o.P[p][q].i};
        Down[il] = RC<R>{(R)o.D[p][q].r, (R)o.D[p][q].i};
        ucache[il] = o.U[p][q];
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
  // K1(t+1) of the pipelined loop, run by threads 32.. (warp 0 is on WSR(t)).
  // Generic N, d in the weighted stage: the receiver half (k1_part_u) on warp 1
  // and the Woodbury weight half (k1_part_w) on warp 2 run concurrently, one
  // lane per user, then warp 1 combines (same arithmetic as k1_math, so the
  // results are identical to the one-thread path).
  auto k1_pipelined = [&](int gsrc, bool weighted, int bin, int bout) {
    constexpr bool closed = NN == 2 && DD == 2;
    const int warp = tid >> 5, lane = tid & 31;
    if (closed || !weighted || KL > 32 || blockDim.x < 96) {
      if (tid >= 32) k1_users(gsrc, weighted, true, bin, bout, tid - 32, blockDim.x - 32);
      return;
    }
    if constexpr (!closed) {
      constexpr int wstride = 2 * DD * DD + NN + 1;  // doubles per user in k1w
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
          for (int a = 0; a < NN; ++a) pv[a] = w[2 * DD * DD + a];
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
          for (int a = 0; a < NN; ++a) w[2 * DD * DD + a] = wv.piv[a];
          w[2 * DD * DD + NN] = (double)wv.pd;
        }
        asm volatile("bar.sync 1, 64;\n" ::: "memory");
      }
    }
  };
  // per-CTA K1 sums -> exchange slots (one thread, after the K1 writes are visible)
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
  // gather the other owners' U and α U W (after a cluster barrier)
  auto k1_gather = [&]() {
    const int per = NN * DD;
    for (int i = tid; i < K * per; i += blockDim.x) {
      const int owner = (i / per) / KL;
      if (owner != crank) {
        Uall[i] = cl.map_shared_rank(Uall, owner)[i];
        Pall[i] = cl.map_shared_rank(Pall, owner)[i];
      }
    }
  };
  // one non-overlapped K1 pass + publication + gather
  auto k1_phase = [&](int gsrc, bool weighted, bool want_f, int bin, int bout) {
    k1_users(gsrc, weighted, want_f, bin, bout, tid, blockDim.x);
    __syncthreads();
    if (tid == 0) k1_publish();
    cl.sync();
    k1_gather();
  };
  // Ŷ over own columns, in place over G[g]
  auto build_yhat = [&](int g) {
    R* Yr = Gr[g];
    R* Yi = Gi[g];
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
        R gr[NN], gi[NN], qr[DD], qi[DD];
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          gr[p] = Yr[(m * NN + p) * ldg + jl];
          gi[p] = Yi[(m * NN + p) * ldg + jl];
        }
#pragma unroll
        for (int q = 0; q < DD; ++q) {
          R sr = 0, si = 0;
#pragma unroll
          for (int p = 0; p < NN; ++p) {
            const RC<R> u = Uall[(m * NN + p) * DD + q];
            sr = fma(u.r, gr[p], fma(u.i, gi[p], sr));
            si = fma(u.r, gi[p], fma(-u.i, gr[p], si));
          }
          qr[q] = sr;
          qi[q] = si;
        }
#pragma unroll
        for (int p = 0; p < NN; ++p) {
          R sr = 0, si = 0;
#pragma unroll
          for (int q = 0; q < DD; ++q) {
            const RC<R> pp = Pall[(m * NN + p) * DD + q];
            sr = fma(pp.r, qr[q], fma(-pp.i, qi[q], sr));
            si = fma(pp.r, qi[q], fma(pp.i, qr[q], si));
          }
          yr[p] = sr;
          yi[p] = si;
        }
      }
#pragma unroll
      for (int p = 0; p < NN; ++p) {
        Yr[(m * NN + p) * ldg + jl] = yr[p];
        Yi[(m * NN + p) * ldg + jl] = yi[p];
      }
    }
  };
  // GEMM-A + extrapolation + step, returns cluster-wide ‖X‖².
  //   V̂ = V[vc] + ω (V[vc] − V[vo]);  X = V̂ − step ∇ -> V[vx];  save: V[vo] <- old V[vc]
  // With V_old in global scratch (L.vglob) the current precoders stay pinned in
  // the SMEM slot 0 (vc = vx = 0, vo = 1, save): GEMM-B always reads SMEM.
  auto grad_step = [&](int ysrc, int vc, int vo, int vx, bool save, double step, double omega,
                       bool extrap) {
    const R* vcr = Vr[vc];
    const R* vci = Vi[vc];
    R* vor = Vr[vo];
    R* voi = Vi[vo];
    R* xr = Vr[vx];
    R* xi = Vi[vx];
    const R st = (R)step, om = (R)omega;
    double pw = 0.0;
    // V_old in global scratch (h_placement 3): staged into the free H ring
    // after the K loop, so the epilogue reads it from shared memory
    const size_t ring_reals = TC ? 2 * L.nH : (size_t)2 * kStreamStages * L.SB;
    const bool stage_vold = extrap && L.vglob && vo == 1 && !hres && 2 * L.nV <= ring_reals &&
                            (2 * L.nV * sizeof(R)) % 16 == 0;
    const R* rdr = stage_vold ? reinterpret_cast<const R*>(stage) : vor;
    const R* rdi = stage_vold ? rdr + L.nV : voi;
    // tensor-core epilogues run one thread per row p: the global V_old slot is
    // then column-major (q * M + p) so the per-row saves coalesce
    const bool vo_cm = TC && L.vglob && vo == 1;
    auto pre = [&]() {
      if (stage_vold) {
        const int n16 = (int)((2 * L.nV * sizeof(R)) / 16);
        constexpr int per = 16 / (int)sizeof(R);
        R* dst = reinterpret_cast<R*>(stage);
        for (int i = tid; i < n16; i += blockDim.x) cp_async16(dst + i * per, vor + i * per);
        cp_async_commit();
        cp_async_wait0();
        __syncthreads();
      }
    };
    auto epi = [&](int p, int q, R gr, R gi) {
      const int o = p * ldv + q;
      const int ov = vo_cm ? q * M + p : o;
      const R cr0 = vcr[o], ci0 = vci[o];
      R vr = cr0, vi = ci0;
      if (extrap) {
        vr = vr + om * (vr - rdr[ov]);
        vi = vi + om * (vi - rdi[ov]);
      }
      const R x_r = vr - st * gr, x_i = vi - st * gi;
      if (save) {
        vor[ov] = cr0;
        voi[ov] = ci0;
      }
      xr[o] = x_r;
      xi[o] = x_i;
      pw += (double)x_r * (double)x_r + (double)x_i * (double)x_i;
    };
    if constexpr (TC) {  // ∇' = H^H Ŷ on tcgen05 (conj A), epilogue one thread per row
      tcs::gemm(pipe, tc_seq, hpA, tmA, M / tmA, KN, ncol, (const float*)Gr[ysrc],
                (const float*)Gi[ysrc], ldg);
      pre();
      tcs::for_each(pipe, tmA, M / tmA, ncol, KN, true,
                    [&](int p, int q, float gr, float gi) { epi(p, q, (R)gr, (R)gi); });
    } else if (hres)
      cgemm_any<R, 4, 4, true>(M, ncol, KN, Hr, Hi, ldh, Gr[ysrc], Gi[ysrc], ldg, epi);
    else if ((M / 4) * (ncol / 4) < (int)blockDim.x &&
             stream2_ok<R, 2, 4, true>(M, ncol, KN, ldg, L.SB, blockDim.x))
      cgemm_stream2<R, 2, 4, kStreamStages, true>(M, ncol, KN, Hcur, M, stage, L.SB, Gr[ysrc],
                                                   Gi[ysrc], ldg, epi, pre);
    else if (stream2_ok<R, 4, 4, true>(M, ncol, KN, ldg, L.SB, blockDim.x))
      cgemm_stream2<R, 4, 4, kStreamStages, true>(M, ncol, KN, Hcur, M, stage, L.SB, Gr[ysrc],
                                                   Gi[ysrc], ldg, epi, pre);
    else if (stream2_ok<R, 8, 4, true>(M, ncol, KN, ldg, L.SB, blockDim.x))
      cgemm_stream2<R, 8, 4, kStreamStages, true>(M, ncol, KN, Hcur, M, stage, L.SB, Gr[ysrc],
                                                   Gi[ysrc], ldg, epi, pre);
    else
      cgemm_stream<R, kStreamRY, kStreamRX, kStreamTPT, true>(M, ncol, KN, Hcur, M, stage, L.SB,
                                                              Gr[ysrc], Gi[ysrc], ldg, epi, pre);
    pw = block_sum(pw, red);
    if (tid == 0) xs[XS_POWER] = pw;
    cl.sync();
    return xsum(XS_POWER);
  };
  // GEMM-B: G[dst] = H V[src].  With ghat >= 0 the epilogue also writes the
  // next iteration's extrapolated Ĝ = G + ω (G − G_prev) over G[ghat], which
  // holds G_prev (solvers.py:380-390 by linearity).
  auto gemm_hv = [&](int src, int dst, int ghat, double omega) {
    R* gr = Gr[dst];
    R* gi = Gi[dst];
    R* hr = ghat >= 0 ? Gr[ghat] : nullptr;
    R* hi = ghat >= 0 ? Gi[ghat] : nullptr;
    const R om = (R)omega;
    auto epi = [&](int p, int q, R cr, R ci) {
      const int o = p * ldg + q;
      gr[o] = cr;
      gi[o] = ci;
      if (hr) {  // ω = 0: plain copy (G_prev may be uninitialised shared memory)
        hr[o] = om == R(0) ? cr : cr + om * (cr - hr[o]);
        hi[o] = om == R(0) ? ci : ci + om * (ci - hi[o]);
      }
    };
    if constexpr (TC) {  // G = H V on tcgen05, epilogue one thread per row
      tcs::gemm(pipe, tc_seq, hpB, tmB, KN / tmB, M, ncol, (const float*)Vr[src],
                (const float*)Vi[src], ldv);
      tcs::for_each(pipe, tmB, KN / tmB, ncol, M, false,
                    [&](int p, int q, float cr, float ci) { epi(p, q, (R)cr, (R)ci); });
    } else if (hres)
      cgemm_any<R, 2, 4, false>(KN, ncol, M, Hr, Hi, ldh, Vr[src], Vi[src], ldv, epi);
    else if (stream2_ok<R, 2, 4, false>(KN, ncol, M, ldv, L.SB, blockDim.x))
      cgemm_stream2<R, 2, 4, kStreamStages, false>(KN, ncol, M, Hcur, M, stage, L.SB, Vr[src],
                                                    Vi[src], ldv, epi);
    else if (stream2_ok<R, 4, 4, false>(KN, ncol, M, ldv, L.SB, blockDim.x))
      cgemm_stream2<R, 4, 4, kStreamStages, false>(KN, ncol, M, Hcur, M, stage, L.SB, Vr[src],
                                                    Vi[src], ldv, epi);
    else
      cgemm_stream<R, kStreamRY, kStreamRX, kStreamTPT, false>(KN, ncol, M, Hcur, M, stage, L.SB,
                                                               Vr[src], Vi[src], ldv, epi);
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
    // ---------------- load realization r: full H, own columns of V0 ----------------
    {
      const RC<R>* Hg = reinterpret_cast<const RC<R>*>(a.H) + (size_t)r * KN * M;
      Hcur = Hg;
      if constexpr (sizeof(R) == 4) {
        if (TC) {  // this CTA's share of the pre-split H / H^T planes (rows r0..r1)
          const int r0 = crank * (KN / C), r1 = (crank + 1) * (KN / C);
          const float2* H2 = reinterpret_cast<const float2*>(Hg);
          tcs::split_h(H2, KN, M, false, const_cast<float*>(hpB), r0, r1);
          tcs::split_h(H2, KN, M, true, const_cast<float*>(hpA), r0, r1);
          umma::fence_proxy_async_global();  // generic writes -> the cluster's bulk copies
          __threadfence();  // visible to the other CTAs before the next cluster barrier
        }
      }
      if (hres) {
        for (int i = tid; i < KN * M; i += blockDim.x) {
          const int row = i / M, col = i - row * M;
          const RC<R> v = Hg[i];
          Hr[row * ldh + col] = v.r;
          Hi[row * ldh + col] = v.i;
        }
      }
      const RC<R>* Vg = reinterpret_cast<const RC<R>*>(a.V0) + ((size_t)r * K + k0) * M * DD;
      for (int i = tid; i < KL * M * DD; i += blockDim.x) {
        const int kl = i / (M * DD), rem = i - kl * M * DD, m = rem / DD, s = rem - m * DD;
        const RC<R> v = Vg[i];
        Vr[0][m * ldv + kl * DD + s] = v.r;
        Vi[0][m * ldv + kl * DD + s] = v.i;
      }
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
      // Grams of H rows of ALL users over M would duplicate work; own users only
      const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
      for (int kl = warp; kl < KL; kl += nw) {
        const int k = k0 + kl;
        double sr[NN][NN], si[NN][NN];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < NN; ++q) sr[p][q] = si[p][q] = 0.0;
        for (int m = lane; m < M; m += 32) {
          double hr[NN], hi[NN];
          for (int p = 0; p < NN; ++p) {
            if (hres) {
              hr[p] = (double)Hr[(k * NN + p) * ldh + m];
              hi[p] = (double)Hi[(k * NN + p) * ldh + m];
            } else {
              const RC<R> v = Hcur[(size_t)(k * NN + p) * M + m];
              hr[p] = (double)v.r;
              hi[p] = (double)v.i;
            }
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
        if (lane == 0) rate[kl] = herm_eig_max<NN>(G);
      }
      __syncthreads();
      if (tid == 0) {
        double kap = 0.0;
        for (int kl = 0; kl < KL; ++kl) kap = fmax(kap, rate[kl]);
        xs[XS_KAPPA] = kap;
      }
      cl.sync();
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
    gemm_hv(0, 0, 1, 0.0);
    __syncthreads();

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
    // ---------------- K1(1) (solvers.py:440-460 at t = 1) ----------------
    bool wn = stage_flag();  // the flag K1(t) was computed with
    gram_partials(Gr[1], Gi[1], 0);
    cl.sync();
    gram_reduce(0);
    __syncthreads();
    k1_phase(1, wn, true, 0, 1);
    pc.mark(9);  // setup: load, bounds, G = H V0, K1(1)

    // ---------------- main loop (solvers.py:440-505), software-pipelined ----------------
    // Per iteration t: [K1(t) status] | Ŷ(t) | GEMM-A + ‖X‖² (cluster sum) |
    // projection | GEMM-B (+ Ĝ(t+1) in its epilogue) | Gram partials of G_new
    // and Ĝ(t+1) | warp 0: WSR(t) of own users while warps 1..: K1(t+1) with a
    // speculated stage flag | exchange | every CTA: state machine of t (fixed
    // rank order, identical decisions), K1(t+1) redone if mis-speculated, U/P
    // gather.  U/W/ln det W double-buffered by iteration parity.  Three cluster
    // barriers per iteration (four at a stage switch).
    for (int t = 1; t <= a.max_iters; ++t) {
      const int cur = ctl.cur, oth = 1 - cur;
      const int bk = t & 1;  // bank holding K1(t)'s U / W / ln det W
      if (tid == 0) {  // K1(t) results (published before the last cluster barrier)
        ctl.f_u = xsum(XS_FU);
        ctl.f_w = xsum(XS_FW);
        const int st = xfirst(XS_ST1);
        if (st) {  // update_weight_matrices raised inside iteration t (solvers.py:455-460)
          if (!ctl.latched && wn) {
            if (a.latch) ctl.latched = 1;
            if (ctl.switch_it < 0) ctl.switch_it = t;
          }
          ctl.status = st;
          ctl.stop = 1;
        }
      }
      const bool extrap = (t >= 2) && (ctl.omega > 0.0);
      __syncthreads();
      pc.mark(0);
      if (ctl.stop) break;
      build_yhat(oth);
      __syncthreads();
      pc.mark(1);
      const bool pin = L.vglob;  // current precoders pinned in SMEM slot 0
      const int vx = pin ? 0 : oth;
      const double power = pin ? grad_step(oth, 0, 1, 0, true, ctl.step, ctl.omega, extrap)
                               : grad_step(oth, cur, oth, oth, false, ctl.step, ctl.omega, extrap);
      double scale = 1.0;
      if (!(power <= ctl.pmax)) scale = sqrt(ctl.pmax / power);
      if (scale != 1.0) {
        const R sc = (R)scale;
        for (int i = tid; i < M * ldv; i += blockDim.x) {  // (padding columns too)
          Vr[vx][i] *= sc;
          Vi[vx][i] *= sc;
        }
      }
      __syncthreads();
      pc.mark(2);
      const bool more = t < a.max_iters;
      // G_new over Ŷ; Ĝ(t+1) over G_cur (which becomes G_old)
      gemm_hv(vx, oth, more ? cur : -1, ctl.omega);
      __syncthreads();
      pc.mark(3);
      {  // Gram partials of G_new -> gx[1] and of Ĝ(t+1) -> gx[0], all warps
        const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
        for (int k = warp; k < K; k += nw)
          gram_pair<R, NN>(k, Gr[oth], Gi[oth], gx[1], more ? Gr[cur] : nullptr, Gi[cur], gx[0],
                           ldg, ncol, lane);
      }
      // speculated stage flag of t+1 (thread 0 updates ctl.latched below)
      const bool wn_spec = ctl.latched || wn;
      cl.sync();
      gram_reduce(1);
      if (more) gram_reduce(0);
      __syncthreads();
      pc.mark(4);
      if (tid < 32) {  // warp 0: rates / f_after_v of own users (lanes), CTA partials
        const int lane = tid;
        const cd* ucache = ucb[bk];
        const cd* wcache = wcb[bk];
        for (int kl = lane; kl < KL; kl += 32) {
          cd Tg[NN][NN], Gkk[NN][DD], U[NN][DD], W[DD][DD];
          gram_of(1, kl, Tg);
#pragma unroll
          for (int p = 0; p < NN; ++p)
#pragma unroll
            for (int s = 0; s < DD; ++s) {
              const int idx = ((k0 + kl) * NN + p) * ldg + kl * DD + s;
              Gkk[p][s] = cmk((double)Gr[oth][idx], (double)Gi[oth][idx]);
              U[p][s] = ucache[(kl * NN + p) * DD + s];
            }
#pragma unroll
          for (int p = 0; p < DD; ++p)
#pragma unroll
            for (int q = 0; q < DD; ++q) W[p][q] = wcache[(kl * DD + p) * DD + q];
          double rr, ff;
          int st;
          wsr_math<NN, DD>(Tg, Gkk, ctl.sigma2, alpha[kl], U, W, lndb[bk][kl], rr, ff, st);
          rate[kl] = rr;
          fv[kl] = ff;
          ust2[kl] = st;
        }
        __syncwarp();
        double sr = 0.0, sv = 0.0;
        int f2 = KL;
        for (int kl = lane; kl < KL; kl += 32) {  // lane-strided, then a fixed shuffle tree
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
      } else if (more) {  // warps 1..: K1(t+1) with the speculated stage flag
        k1_pipelined(cur, wn_spec, bk, bk ^ 1);
      }
      __syncthreads();
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
        for (int i = tid; i < KL * M * DD; i += blockDim.x) {
          const int kl = i / (M * DD), rem = i - kl * M * DD, m = rem / DD, s = rem - m * DD;
          const int o = m * ldv + kl * DD + s;
          dV[2 * i] = (double)Vr[vx][o];
          dV[2 * i + 1] = (double)Vi[vx][o];
        }
      }
      if (tid == 0) {  // state machine of iteration t, identical in every CTA
        if (!ctl.latched && wn) {
          if (a.latch) ctl.latched = 1;
          if (ctl.switch_it < 0) ctl.switch_it = t;
        }
        const double wsr = xsum(XS_RATE);
        const double sv = xsum(XS_FV);
        int st = xfirst(XS_ST2);
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
        ctl.weighted_now = wn;
        ctl.last_weighted = wn;
        if (a.trace && crank == 0) {
          double* tr = a.trace + ((size_t)r * a.max_iters + (t - 1)) * kTraceFields;
          tr[AMMMSE_TRACE_T] = (double)t;
          tr[AMMMSE_TRACE_WSR_BITS] = wsr / kLn2;
          tr[AMMMSE_TRACE_F_VALUE] = sv;
          tr[AMMMSE_TRACE_TOTAL_POWER] = total_power;
          tr[AMMMSE_TRACE_STAGE] = wn ? 1.0 : 0.0;
          tr[AMMMSE_TRACE_F_AFTER_U] = ctl.f_u;
          tr[AMMMSE_TRACE_F_AFTER_W] = ctl.f_w;
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
        ctl.wn_next = stage_flag();
      }
      __syncthreads();
      pc.mark(6);
      if (ctl.stop) break;
      wn = ctl.wn_next != 0;
      if (more && wn != wn_spec) {  // mis-speculated stage flag: redo K1(t+1) (same inputs)
        k1_phase(cur, wn, true, bk, bk ^ 1);
      } else if (more) {
        k1_gather();
      }
      __syncthreads();
      pc.mark(7);
    }

    // ---------------- exit: stationarity residual (solvers.py:400-412) ----------------
    double residual = NAN;
    if (ctl.status == 0) {
      const int cur = ctl.cur, oth = 1 - cur;
      const bool weighted = ctl.latched || ctl.last_weighted;
      for (int i = tid; i < KN * ldg; i += blockDim.x) {
        Gr[oth][i] = Gr[cur][i];
        Gi[oth][i] = Gi[cur][i];
      }
      __syncthreads();
      gram_partials(Gr[oth], Gi[oth], 0);
      cl.sync();
      gram_reduce(0);
      __syncthreads();
      k1_phase(oth, weighted, false, 0, 0);
      int st = xfirst(XS_ST1);
      __syncthreads();
      if (st == 0) {
        build_yhat(oth);
        __syncthreads();
        const int rc = L.vglob ? 0 : cur, rx = L.vglob ? 1 : oth;
        const double power = grad_step(oth, rc, rx, rx, false, 2.0 * ctl.gamma_safe, 0.0, false);
        double scale = 1.0;
        if (!(power <= ctl.pmax)) scale = sqrt(ctl.pmax / power);
        double dsum = 0.0, vsum = 0.0;
        for (int i = tid; i < M * ldv; i += blockDim.x) {
          if (i % ldv >= ncol) continue;  // padding column (tensor-core layout)
          const double a_r = (double)Vr[rc][i], a_i = (double)Vi[rc][i];
          const double dr = a_r - (double)((R)(Vr[rx][i] * (R)scale));
          const double di = a_i - (double)((R)(Vi[rx][i] * (R)scale));
          dsum += dr * dr + di * di;
          vsum += a_r * a_r + a_i * a_i;
        }
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
    __syncthreads();
    // ---------------- write results (own users' precoders) ----------------
    {
      const int cur = ctl.cur;
      if (a.Vout) {
        RC<R>* Vg = reinterpret_cast<RC<R>*>(a.Vout) + ((size_t)r * K + k0) * M * DD;
        for (int i = tid; i < KL * M * DD; i += blockDim.x) {
          const int kl = i / (M * DD), rem = i - kl * M * DD, m = rem / DD, s = rem - m * DD;
          const int vcur = L.vglob ? 0 : cur;
          Vg[i] = RC<R>{Vr[vcur][m * ldv + kl * DD + s], Vi[vcur][m * ldv + kl * DD + s]};
        }
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
    // all remote reads of this realization's exchange buffers are complete
    // before any CTA starts the next realization (its first writes)
    cl.sync();
    pc.mark(8);
  }
  pc.flush();
  if constexpr (TC) {
    __syncthreads();
    if ((tid >> 5) == 0) umma::tmem_dealloc<512>(pipe.tmem);
  }
}

}  // namespace ammmse
