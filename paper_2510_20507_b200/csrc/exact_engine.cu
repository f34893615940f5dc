// exact_engine.cu — batched exact-update drivers on the device (SURVEY.md §8(f)
// row 1): run_wmmse / run_mmmse, i.e. _run_bcd with exact=True,
// use_extrapolation=False (pkg/src/wsrbeam/solvers.py:415-518, :521-537):
//
//   U_k = (H_k Q H_k^H + σ² I)^{-1} H_k V_k              update_receivers (:210-225)
//   W_k = herm((I − U_k^H H_k V_k)^{-1}) or I              update_weight_matrices (:228-254)
//   A   = herm(Σ_m α_m H_m^H U_m W_m U_m^H H_m)  (M x M)   weighted_gram (objective.py:172-187)
//   B_k = α_k H_k^H U_k W_k                                update_precoders_exact (:332-348)
//   V_k = (A + λ I)^{-1} B_k, λ by dual bisection          bisect_dual (:276-329)
//   WSR / rel / switch / stop as in the A-MMMSE engine     (:465-518; no divergence test)
//
// One CTA (256 threads) per realization at a time (persistent grid over an
// atomic counter), everything in fp64.  The M x M system matrix, its Cholesky
// factor, the stacked targets and the solves live in a per-CTA global scratch
// slot (L1 / L2 resident); the per-user N x N / d x d algebra reuses the fp64
// routines of the A-MMMSE engine (user_algebra.cuh: the receiver half is the
// same Cholesky solve, the weight half the Woodbury form of W = T^{-1}).
// The Cholesky factorisation is right-looking, one column per step (3 block
// barriers); it reports failure exactly where LAPACK zpotrf (scipy cho_factor)
// raises: a non-positive or non-finite pivot.  The min-norm least-squares
// fallback of bisect_dual (np.linalg.lstsq, :324-327) is a pseudo-inverse from
// a cyclic Jacobi eigendecomposition of the real 2M x 2M embedding of A with
// numpy's default cutoff (eps * M * sigma_max).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ammmse.h"
#include "small_linalg.cuh"
#include "user_algebra.cuh"

namespace ammmse {
namespace exact {

constexpr int kThreads = 256;
constexpr double kLn2x = 0.69314718055994530942;

struct Args {
  const void* H;
  const void* V0;
  int c64;  // inputs complex64 (converted to complex128 on load)
  const double* sigma2;
  const double* pmax;
  const double* alpha;
  void* Vout;
  double* wsr_bits;
  int* iterations;
  unsigned char* converged;
  double* residual;
  int* switch_it;
  int* status;
  double* trace;
  double* itU;
  double* itW;
  double* itV;
  double eps1, eps2, bisect_tol;
  int max_iters, latch, start_weighted, bisect_max;
  int M, K;
  long long B;
  cd* scratch;  // per-CTA slot of slot_cd complex128 elements
  size_t slot_cd;
  unsigned long long* counter;
};

// per-CTA scratch layout (cd elements)
struct Slot {
  cd *H, *V, *X, *Y, *Z, *G, *A, *L, *T;  // T: bisection candidate / residual work
  double* J;                              // 2M x 2M real Jacobi workspace (lstsq fallback)
  double* Q;                              // 2M x 2M eigenvectors
  __host__ __device__ static size_t count(int M, int K, int N, int d) {
    const size_t KN = (size_t)K * N, KD = (size_t)K * d, m = M;
    return KN * m + 5 * m * KD + KN * KD + 2 * m * m + (2 * (2 * m) * (2 * m) + 1) / 2 + 16;
  }
  __device__ void init(cd* base, int M, int K, int N, int d) {
    const size_t KN = (size_t)K * N, KD = (size_t)K * d, m = M;
    H = base;
    V = H + KN * m;
    X = V + m * KD;
    Y = X + m * KD;
    Z = Y + m * KD;
    T = Z + m * KD;
    G = T + m * KD;
    A = G + KN * KD;
    L = A + m * m;
    J = reinterpret_cast<double*>(L + m * m);
    Q = J + (2 * m) * (2 * m);
  }
};

__device__ __forceinline__ double warp_allsum_x(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];  // fixed order: identical in every thread
  __syncthreads();
  return s;
}

// In-place lower Cholesky of the M x M Hermitian matrix in L (lower triangle
// valid).  Returns false (in every thread) on a non-positive / non-finite pivot.
__device__ bool chol_block(cd* L, int M, int* flag) {
  const int tid = threadIdx.x;
  for (int j = 0; j < M; ++j) {
    if (tid == 0) {
      const double dj = L[(size_t)j * M + j].r;
      if (!(dj > 0.0) || !isfinite(dj)) {
        *flag = 1;
      } else {
        L[(size_t)j * M + j] = cmk(sqrt(dj));
      }
    }
    __syncthreads();
    if (*flag) return false;
    const double inv = 1.0 / L[(size_t)j * M + j].r;
    for (int i = j + 1 + tid; i < M; i += blockDim.x) L[(size_t)i * M + j] = cscale(L[(size_t)i * M + j], inv);
    __syncthreads();
    const int n = M - j - 1;  // trailing lower triangle, row-major over (i, k), k <= i
    for (int e = tid; e < n * (n + 1) / 2; e += blockDim.x) {
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      if ((i + 1) * (i + 2) / 2 <= e) ++i;
      if (i * (i + 1) / 2 > e) --i;
      const int k = e - i * (i + 1) / 2;
      const int ii = j + 1 + i, kk = j + 1 + k;
      L[(size_t)ii * M + kk] = csub(L[(size_t)ii * M + kk], cmulcb(L[(size_t)ii * M + j], L[(size_t)kk * M + j]));
    }
    __syncthreads();
  }
  return true;
}

// X (M x KD) = (L L^H)^{-1} B, one RHS column per thread (cho_solve)
__device__ void chol_solve_block(const cd* L, int M, const cd* B, cd* X, int KD) {
  for (int q = threadIdx.x; q < KD; q += blockDim.x) {
    for (int i = 0; i < M; ++i) {
      cd t = B[(size_t)i * KD + q];
      for (int p = 0; p < i; ++p) t = csub(t, cmul(L[(size_t)i * M + p], X[(size_t)p * KD + q]));
      X[(size_t)i * KD + q] = cscale(t, 1.0 / L[(size_t)i * M + i].r);
    }
    for (int i = M - 1; i >= 0; --i) {
      cd t = X[(size_t)i * KD + q];
      for (int p = i + 1; p < M; ++p) t = csub(t, cmulc(L[(size_t)p * M + i], X[(size_t)p * KD + q]));
      X[(size_t)i * KD + q] = cscale(t, 1.0 / L[(size_t)i * M + i].r);
    }
  }
  __syncthreads();
}

// solve_hpd(A + lam I, B) -> X; false if the factorisation fails
__device__ bool solve_shifted(const cd* A, cd* L, int M, double lam, const cd* B, cd* X, int KD,
                              int* flag) {
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int i = e / M, k = e - i * M;
    if (k <= i) {
      cd v = A[e];
      if (i == k) v.r += lam;
      L[e] = v;
    }
  }
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  if (!chol_block(L, M, flag)) return false;
  chol_solve_block(L, M, B, X, KD);
  return true;
}

__device__ double power_of(const cd* X, size_t n, double* red) {
  double s = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) s += cabs2(X[i]);
  return block_sum_d(s, red);
}

// Min-norm least squares X = A^+ B (np.linalg.lstsq, rcond = eps * M): cyclic
// Jacobi on the real embedding S = [[Ar, -Ai], [Ai, Ar]] by thread 0 (rare
// fallback path), then X = Q diag(1/λ) Q^T applied by all threads.
__device__ void lstsq_block(const cd* A, int M, const cd* B, cd* X, int KD, double* S, double* Q) {
  const int n = 2 * M;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    const cd a = A[(size_t)(i % M) * M + (j % M)];
    double v;
    if ((i < M) == (j < M)) v = a.r;
    else v = i < M ? -a.i : a.i;
    S[e] = v;
    Q[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int sweep = 0; sweep < 80; ++sweep) {
      double off = 0.0, diag = 0.0;
      for (int p = 0; p < n; ++p) {
        diag += S[p * n + p] * S[p * n + p];
        for (int q = p + 1; q < n; ++q) off += S[p * n + q] * S[p * n + q];
      }
      if (off <= 1e-32 * diag || off == 0.0) break;
      for (int p = 0; p < n; ++p)
        for (int q = p + 1; q < n; ++q) {
          const double apq = S[p * n + q];
          if (apq == 0.0) continue;
          const double theta = (S[q * n + q] - S[p * n + p]) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
          for (int r = 0; r < n; ++r) {
            const double srp = S[r * n + p], srq = S[r * n + q];
            S[r * n + p] = c * srp - s * srq;
            S[r * n + q] = s * srp + c * srq;
          }
          for (int r = 0; r < n; ++r) {
            const double spr = S[p * n + r], sqr = S[q * n + r];
            S[p * n + r] = c * spr - s * sqr;
            S[q * n + r] = s * spr + c * sqr;
          }
          for (int r = 0; r < n; ++r) {
            const double qrp = Q[r * n + p], qrq = Q[r * n + q];
            Q[r * n + p] = c * qrp - s * qrq;
            Q[r * n + q] = s * qrp + c * qrq;
          }
        }
    }
  }
  __syncthreads();
  double smax = 0.0;
  for (int p = 0; p < n; ++p) smax = fmax(smax, fabs(S[p * n + p]));
  const double cut = 2.220446049250313e-16 * M * smax;
  // X = Q diag(1/λ) Q^T [Br; Bi] per RHS column (thread per column)
  for (int q = threadIdx.x; q < KD; q += blockDim.x) {
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int p = 0; p < n; ++p) {
        const double lam = S[p * n + p];
        if (fabs(lam) <= cut) continue;
        double proj = 0.0;  // Q[:, p]^T b
        for (int r = 0; r < n; ++r) {
          const cd b = B[(size_t)(r % M) * KD + q];
          proj += Q[r * n + p] * (r < M ? b.r : b.i);
        }
        acc += Q[i * n + p] * proj / lam;
      }
      if (i < M) X[(size_t)i * KD + q].r = acc;
      else X[(size_t)(i - M) * KD + q].i = acc;
    }
  }
  __syncthreads();
}

template <int NN, int DD>
__global__ void __launch_bounds__(kThreads) exact_solve_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[32];
  __shared__ int flag;
  __shared__ unsigned long long s_r;
  __shared__ int s_stop, s_status, s_latched, s_switch, s_weighted, s_last_weighted, s_conv,
      s_iters, s_nhist;
  __shared__ double s_wsr_last, s_wsr_prev, s_wsr, s_sigma2, s_pmax, s_gsafe;
  const int M = a.M, K = a.K, KN = K * NN, KD = K * DD;
  const int tid = threadIdx.x;
  // shared memory: per-user fp64 state
  cd* gram = reinterpret_cast<cd*>(smem);        // K*NN*NN
  cd* Uc = gram + (size_t)K * NN * NN;           // K*NN*DD
  cd* Wc = Uc + (size_t)K * NN * DD;             // K*DD*DD
  cd* Wp = Wc + (size_t)K * DD * DD;             // K*DD*DD (previous W)
  double* lnw = reinterpret_cast<double*>(Wp + (size_t)K * DD * DD);  // K
  double* lnwp = lnw + K;
  double* fu = lnwp + K;
  double* fw = fu + K;
  double* fv = fw + K;
  double* rate = fv + K;
  int* ust = reinterpret_cast<int*>(rate + K);

  Slot sl;
  sl.init(a.scratch + (size_t)blockIdx.x * a.slot_cd, M, K, NN, DD);

  auto gemm_hv = [&]() {  // G = H V (KN x KD)
    for (int e = tid; e < KN * KD; e += blockDim.x) {
      const int r = e / KD, q = e - r * KD;
      cd s = cmk(0.0);
      for (int m = 0; m < M; ++m) cfma(s, sl.H[(size_t)r * M + m], sl.V[(size_t)m * KD + q]);
      sl.G[e] = s;
    }
    __syncthreads();
  };
  auto grams = [&]() {  // per-user N x N Grams of G's rows over all KD columns
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int k = warp; k < K; k += nw) {
      double sr[NN][NN], si[NN][NN];
      for (int p = 0; p < NN; ++p)
        for (int q = 0; q < NN; ++q) sr[p][q] = si[p][q] = 0.0;
      for (int j = lane; j < KD; j += 32) {
        cd g[NN];
        for (int p = 0; p < NN; ++p) g[p] = sl.G[(size_t)(k * NN + p) * KD + j];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q <= p; ++q) {
            sr[p][q] = fma(g[p].r, g[q].r, fma(g[p].i, g[q].i, sr[p][q]));
            si[p][q] = fma(g[p].i, g[q].r, fma(-g[p].r, g[q].i, si[p][q]));
          }
      }
      for (int p = 0; p < NN; ++p)
        for (int q = 0; q <= p; ++q) {
          const double re = warp_allsum_x(sr[p][q]), im = warp_allsum_x(si[p][q]);
          if (lane == 0) {
            gram[(k * NN + p) * NN + q] = cmk(re, q < p ? im : 0.0);
            gram[(k * NN + q) * NN + p] = cmk(re, q < p ? -im : 0.0);
          }
        }
    }
    __syncthreads();
  };
  auto load_user = [&](int k, cd (&Tg)[NN][NN], cd (&Gkk)[NN][DD]) {
    for (int p = 0; p < NN; ++p)
      for (int q = 0; q < NN; ++q) Tg[p][q] = gram[(k * NN + p) * NN + q];
    for (int p = 0; p < NN; ++p)
      for (int s = 0; s < DD; ++s) Gkk[p][s] = sl.G[(size_t)(k * NN + p) * KD + k * DD + s];
  };
  // U / W (weighted or I) of every user at the current G; f terms; status
  auto k1 = [&](bool weighted, bool want_f) {
    for (int k = tid; k < K; k += blockDim.x) {
      cd Tg[NN][NN], Gkk[NN][DD], Wpk[DD][DD];
      load_user(k, Tg, Gkk);
      for (int p = 0; p < DD; ++p)
        for (int q = 0; q < DD; ++q) Wpk[p][q] = Wp[(k * DD + p) * DD + q];
      K1Out<NN, DD> o;
      k1_math<NN, DD>(Tg, Gkk, s_sigma2, a.alpha[(size_t)s_r * K + k], Wpk, lnwp[k], weighted,
                      want_f, o);
      for (int p = 0; p < NN; ++p)
        for (int q = 0; q < DD; ++q) Uc[(k * NN + p) * DD + q] = o.U[p][q];
      for (int p = 0; p < DD; ++p)
        for (int q = 0; q < DD; ++q) Wc[(k * DD + p) * DD + q] = o.W[p][q];
      lnw[k] = o.lndetw;
      fu[k] = o.fu;
      fw[k] = o.fw;
      ust[k] = o.status;
    }
    __syncthreads();
  };
  // Z_k = H_k^H U_k, Y_k = α_k Z_k W_k (M x KD), A = herm(Σ_k Y_k Z_k^H) (M x M)
  auto system = [&]() {
    for (int e = tid; e < M * KD; e += blockDim.x) {
      const int m = e / KD, q = e - m * KD, k = q / DD, s = q - k * DD;
      cd z = cmk(0.0);
      for (int p = 0; p < NN; ++p) cfmac(z, sl.H[(size_t)(k * NN + p) * M + m], Uc[(k * NN + p) * DD + s]);
      sl.Z[e] = z;
    }
    __syncthreads();
    for (int e = tid; e < M * KD; e += blockDim.x) {
      const int m = e / KD, q = e - m * KD, k = q / DD, s = q - k * DD;
      cd y = cmk(0.0);
      for (int p = 0; p < DD; ++p) cfma(y, sl.Z[(size_t)m * KD + k * DD + p], Wc[(k * DD + p) * DD + s]);
      sl.Y[e] = cscale(y, a.alpha[(size_t)s_r * K + k]);
    }
    __syncthreads();
    for (int e = tid; e < M * M; e += blockDim.x) {
      const int i = e / M, j = e - i * M;
      if (j > i) continue;
      cd s1 = cmk(0.0), s2 = cmk(0.0);  // (Y Z^H)_ij and (Y Z^H)_ji
      for (int q = 0; q < KD; ++q) {
        s1 = cadd(s1, cmulcb(sl.Y[(size_t)i * KD + q], sl.Z[(size_t)j * KD + q]));
        s2 = cadd(s2, cmulcb(sl.Y[(size_t)j * KD + q], sl.Z[(size_t)i * KD + q]));
      }
      const cd h = cmk(0.5 * (s1.r + s2.r), 0.5 * (s1.i - s2.i));  // hermitianize
      sl.A[(size_t)i * M + j] = h;
      sl.A[(size_t)j * M + i] = cconj(h);
    }
    __syncthreads();
  };
  // bisect_dual (solvers.py:276-329): V <- (A + λ I)^{-1} Y.  false: the
  // factorisation at the bracket's upper end failed (the reference raises
  // ConfigError("system matrix is not positive semidefinite"), :311-312)
  auto bisect = [&]() -> bool {
    const size_t nv = (size_t)M * KD;
    const double P = s_pmax;
    if (solve_shifted(sl.A, sl.L, M, 0.0, sl.Y, sl.X, KD, &flag) &&
        power_of(sl.X, nv, red) <= P) {
      for (size_t i = tid; i < nv; i += blockDim.x) sl.V[i] = sl.X[i];
      __syncthreads();
      return true;
    }
    const double lam_hi0 = sqrt(power_of(sl.Y, nv, red) / P);
    if (lam_hi0 == 0.0) {
      for (size_t i = tid; i < nv; i += blockDim.x) sl.V[i] = cmk(0.0);
      __syncthreads();
      return true;
    }
    double lo = 0.0, hi = lam_hi0;
    // x_hi lives in V, candidates in X
    if (!solve_shifted(sl.A, sl.L, M, hi, sl.Y, sl.V, KD, &flag)) return false;
    double p_hi = power_of(sl.V, nv, red);
    const double band = (1.0 - 1e-3) * P;
    int its = 0;
    while (its < a.bisect_max && !(p_hi >= band && (hi - lo) < a.bisect_tol)) {
      const double mid = 0.5 * (lo + hi);
      ++its;
      const bool good = solve_shifted(sl.A, sl.L, M, mid, sl.Y, sl.X, KD, &flag);
      const double pm = good ? power_of(sl.X, nv, red) : INFINITY;
      if (!good || pm > P) {
        lo = mid;
      } else {
        hi = mid;
        p_hi = pm;
        for (size_t i = tid; i < nv; i += blockDim.x) sl.V[i] = sl.X[i];
        __syncthreads();
      }
    }
    const bool conv = p_hi >= band && (hi - lo) < a.bisect_tol;
    if (!conv) {  // interior optimum with singular A: min-norm least squares (:324-327)
      lstsq_block(sl.A, M, sl.Y, sl.X, KD, sl.J, sl.Q);
      if (power_of(sl.X, nv, red) <= P) {
        for (size_t i = tid; i < nv; i += blockDim.x) sl.V[i] = sl.X[i];
        __syncthreads();
      }
    }
    return true;
  };

  for (;;) {
    if (tid == 0) s_r = atomicAdd(a.counter, 1ULL);
    __syncthreads();
    const long long r = (long long)s_r;
    if (r >= a.B) break;
    // ---- load (complex128 working copies) ----
    for (int e = tid; e < KN * M; e += blockDim.x) {
      if (a.c64) {
        const float2 v = reinterpret_cast<const float2*>(a.H)[(size_t)r * KN * M + e];
        sl.H[e] = cmk(v.x, v.y);
      } else {
        sl.H[e] = reinterpret_cast<const cd*>(a.H)[(size_t)r * KN * M + e];
      }
    }
    for (int e = tid; e < M * KD; e += blockDim.x) {  // V0 (K, M, d) -> V (M x KD)
      const int k = e / (M * DD), rem = e - k * M * DD, m = rem / DD, s = rem - m * DD;
      cd v;
      if (a.c64) {
        const float2 f = reinterpret_cast<const float2*>(a.V0)[(size_t)r * K * M * DD + e];
        v = cmk(f.x, f.y);
      } else {
        v = reinterpret_cast<const cd*>(a.V0)[(size_t)r * K * M * DD + e];
      }
      sl.V[(size_t)m * KD + k * DD + s] = v;
    }
    for (int e = tid; e < K * DD * DD; e += blockDim.x) {
      const int p = (e / DD) % DD, q = e % DD;
      Wp[e] = cmk(p == q ? 1.0 : 0.0);
    }
    for (int k = tid; k < K; k += blockDim.x) lnwp[k] = 0.0;
    if (tid == 0) {
      s_sigma2 = a.sigma2[r];
      s_pmax = a.pmax[r];
      s_stop = 0;
      s_status = 0;
      s_latched = a.start_weighted;
      s_switch = -1;
      s_weighted = 0;
      s_last_weighted = 0;
      s_conv = 0;
      s_iters = 0;
      s_nhist = 0;
      s_wsr_last = s_wsr_prev = s_wsr = 0.0;
    }
    __syncthreads();
    // ---- γ_safe for the stationarity residual (compute_bounds, objective.py:216-240) ----
    {
      const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
      for (int k = warp; k < K; k += nw) {
        double sr[NN][NN], si[NN][NN];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < NN; ++q) sr[p][q] = si[p][q] = 0.0;
        for (int m = lane; m < M; m += 32) {
          cd h[NN];
          for (int p = 0; p < NN; ++p) h[p] = sl.H[(size_t)(k * NN + p) * M + m];
          for (int p = 0; p < NN; ++p)
            for (int q = 0; q < NN; ++q) {
              sr[p][q] = fma(h[p].r, h[q].r, fma(h[p].i, h[q].i, sr[p][q]));
              si[p][q] = fma(h[p].i, h[q].r, fma(-h[p].r, h[q].i, si[p][q]));
            }
        }
        cd Gm[NN][NN];
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < NN; ++q) Gm[p][q] = cmk(warp_allsum_x(sr[p][q]), warp_allsum_x(si[p][q]));
        if (lane == 0) rate[k] = herm_eig_max<NN>(Gm);
      }
      __syncthreads();
      if (tid == 0) {
        double kap = 0.0, abar = a.alpha[(size_t)r * K];
        for (int k = 0; k < K; ++k) {
          kap = fmax(kap, rate[k]);
          abar = fmax(abar, a.alpha[(size_t)r * K + k]);
        }
        s_gsafe = 1.0 / (2.0 * abar * K * kap / s_sigma2);
      }
      __syncthreads();
    }
    // ---- main loop (solvers.py:440-505, exact=True, no extrapolation) ----
    for (int t = 1; t <= a.max_iters; ++t) {
      gemm_hv();
      grams();
      if (tid == 0) {  // stage flag (solvers.py:449-459)
        bool w;
        if (s_latched) {
          w = true;
        } else {
          double rs = INFINITY;
          if (s_nhist >= 2) {
            const double den = fabs(s_wsr_prev);
            rs = den == 0.0 ? INFINITY : fabs(s_wsr_last - s_wsr_prev) / den;
          }
          w = rs <= a.eps1;
          if (w) {
            if (a.latch) s_latched = 1;
            if (s_switch < 0) s_switch = t;
          }
        }
        s_weighted = w ? 1 : 0;
      }
      __syncthreads();
      const bool weighted = s_weighted != 0;
      k1(weighted, true);
      if (tid == 0) {  // update_weight_matrices raised (solvers.py:243-252)
        int st = 0;
        for (int k = 0; k < K; ++k)
          if (st == 0 && ust[k] != 0) st = ust[k];
        if (st) {
          s_status = st;
          s_stop = 1;
        }
      }
      __syncthreads();
      if (s_stop) break;
      double f_u = 0.0, f_w = 0.0;
      for (int k = 0; k < K; ++k) {
        f_u += fu[k];
        f_w += fw[k];
      }
      system();
      if (!bisect()) {
        if (tid == 0) s_status = AMMMSE_STATUS_NONFINITE;
        __syncthreads();
        break;
      }
      // ---- WSR / f_after_v at V_new (objective.py:108-169) ----
      gemm_hv();
      grams();
      for (int k = tid; k < K; k += blockDim.x) {
        cd Tg[NN][NN], Gkk[NN][DD], U[NN][DD], W[DD][DD];
        load_user(k, Tg, Gkk);
        for (int p = 0; p < NN; ++p)
          for (int q = 0; q < DD; ++q) U[p][q] = Uc[(k * NN + p) * DD + q];
        for (int p = 0; p < DD; ++p)
          for (int q = 0; q < DD; ++q) W[p][q] = Wc[(k * DD + p) * DD + q];
        double rr, ff;
        int st;
        wsr_math<NN, DD>(Tg, Gkk, s_sigma2, a.alpha[(size_t)r * K + k], U, W, lnw[k], rr, ff, st);
        rate[k] = rr;
        fv[k] = ff;
        ust[k] = st;
      }
      const double power = power_of(sl.V, (size_t)M * KD, red);  // (barriers inside)
      if (a.itU) {  // block iterate of t (solvers.py:487-488)
        const size_t it = (size_t)r * a.max_iters + (t - 1);
        double* dU = a.itU + it * (size_t)K * NN * DD * 2;
        double* dW = a.itW + it * (size_t)K * DD * DD * 2;
        double* dV = a.itV + it * (size_t)K * M * DD * 2;
        for (int i = tid; i < K * NN * DD; i += blockDim.x) {
          dU[2 * i] = Uc[i].r;
          dU[2 * i + 1] = Uc[i].i;
        }
        for (int i = tid; i < K * DD * DD; i += blockDim.x) {
          dW[2 * i] = Wc[i].r;
          dW[2 * i + 1] = Wc[i].i;
        }
        for (int i = tid; i < K * M * DD; i += blockDim.x) {
          const int k = i / (M * DD), rem = i - k * M * DD, m = rem / DD, s = rem - m * DD;
          const cd v = sl.V[(size_t)m * KD + k * DD + s];
          dV[2 * i] = v.r;
          dV[2 * i + 1] = v.i;
        }
      }
      if (tid == 0) {
        double wsr = 0.0, sv = 0.0;
        int st = 0;
        for (int k = 0; k < K; ++k) {  // fixed user order (objective.py:144-146)
          wsr += rate[k];
          sv += fv[k];
          if (st == 0 && ust[k] != 0) st = ust[k];
        }
        if (!isfinite(wsr) || !isfinite(power)) st = AMMMSE_STATUS_NONFINITE;
        double rel = INFINITY;
        if (t > 1) {
          const double den = fabs(s_wsr_last);
          rel = den == 0.0 ? INFINITY : fabs(wsr - s_wsr_last) / den;
        }
        s_wsr_prev = s_wsr_last;
        s_wsr_last = wsr;
        s_nhist += 1;
        s_iters = t;
        s_wsr = wsr;
        s_last_weighted = weighted ? 1 : 0;
        if (a.trace) {
          double* tr = a.trace + ((size_t)r * a.max_iters + (t - 1)) * AMMMSE_TRACE_FIELDS;
          tr[AMMMSE_TRACE_T] = (double)t;
          tr[AMMMSE_TRACE_WSR_BITS] = wsr / kLn2x;
          tr[AMMMSE_TRACE_F_VALUE] = sv;
          tr[AMMMSE_TRACE_TOTAL_POWER] = power;
          tr[AMMMSE_TRACE_STAGE] = weighted ? 1.0 : 0.0;
          tr[AMMMSE_TRACE_F_AFTER_U] = f_u;
          tr[AMMMSE_TRACE_F_AFTER_W] = f_w;
          tr[AMMMSE_TRACE_F_AFTER_V] = sv;
          tr[AMMMSE_TRACE_REL_CHANGE] = rel;
        }
        if (st) {
          s_status = st;
          s_stop = 1;
        } else if (weighted && rel <= a.eps2) {  // stop test (:503-505)
          s_conv = 1;
          s_stop = 1;
        }
      }
      // W_prev <- W (solvers.py:502)
      for (int i = tid; i < K * DD * DD; i += blockDim.x) Wp[i] = Wc[i];
      for (int k = tid; k < K; k += blockDim.x) lnwp[k] = lnw[k];
      __syncthreads();
      if (s_stop) break;
    }
    // ---- exit: stationarity residual (solvers.py:400-412) ----
    double residual = NAN;
    if (s_status == 0) {
      gemm_hv();
      grams();
      k1(s_latched || s_last_weighted, false);
      if (tid == 0) {
        int st = 0;
        for (int k = 0; k < K; ++k)
          if (st == 0 && ust[k] != 0) st = ust[k];
        s_status = st;
      }
      __syncthreads();
      if (s_status == 0) {
        system();
        // X = V − γ_safe · 2 (A V − Y), projected (pgd_precoder_step, :358-377)
        const double g = s_gsafe;
        for (int e = tid; e < M * KD; e += blockDim.x) {
          const int i = e / KD, q = e - i * KD;
          cd av = cmk(0.0);
          for (int j = 0; j < M; ++j) cfma(av, sl.A[(size_t)i * M + j], sl.V[(size_t)j * KD + q]);
          const cd gr = cscale(csub(av, sl.Y[e]), 2.0);
          sl.X[e] = csub(sl.V[e], cscale(gr, g));
        }
        __syncthreads();
        const size_t nv = (size_t)M * KD;
        const double px = power_of(sl.X, nv, red);
        const double sc = px <= s_pmax ? 1.0 : sqrt(s_pmax / px);
        double ds = 0.0;
        for (size_t i = tid; i < nv; i += blockDim.x) ds += cabs2(csub(sl.V[i], cscale(sl.X[i], sc)));
        ds = block_sum_d(ds, red);
        const double vs = power_of(sl.V, nv, red);
        residual = sqrt(ds) / fmax(1.0, sqrt(fmax(vs, 0.0)));
      }
    }
    // ---- results ----
    if (a.Vout) {
      for (int e = tid; e < K * M * DD; e += blockDim.x) {
        const int k = e / (M * DD), rem = e - k * M * DD, m = rem / DD, s = rem - m * DD;
        const cd v = sl.V[(size_t)m * KD + k * DD + s];
        if (a.c64)
          reinterpret_cast<float2*>(a.Vout)[(size_t)r * K * M * DD + e] = make_float2((float)v.r, (float)v.i);
        else
          reinterpret_cast<cd*>(a.Vout)[(size_t)r * K * M * DD + e] = v;
      }
    }
    if (tid == 0) {
      if (a.wsr_bits) a.wsr_bits[r] = s_wsr / kLn2x;
      if (a.iterations) a.iterations[r] = s_iters;
      if (a.converged) a.converged[r] = (unsigned char)s_conv;
      if (a.residual) a.residual[r] = residual;
      if (a.switch_it) a.switch_it[r] = s_switch;
      if (a.status) a.status[r] = s_status;
    }
    __syncthreads();
  }
}

template <int NN, int DD>
size_t smem_bytes(int K) {
  return (size_t)K * (NN * NN + NN * DD + 2 * DD * DD) * sizeof(cd) + (size_t)K * 6 * sizeof(double) +
         (size_t)K * sizeof(int) + 16;
}

template <int NN>
const void* kernel_n(int d) {
  switch (d) {
    case 1: return (const void*)exact_solve_kernel<NN, 1>;
    case 2: return (const void*)exact_solve_kernel<NN, 2>;
    case 3: return (const void*)exact_solve_kernel<NN, 3>;
    default: return (const void*)exact_solve_kernel<NN, 4>;
  }
}
template <int NN>
size_t smem_n(int d, int K) {
  switch (d) {
    case 1: return smem_bytes<NN, 1>(K);
    case 2: return smem_bytes<NN, 2>(K);
    case 3: return smem_bytes<NN, 3>(K);
    default: return smem_bytes<NN, 4>(K);
  }
}
const void* kernel_for(int N, int d) {
  switch (N) {
    case 1: return kernel_n<1>(d);
    case 2: return kernel_n<2>(d);
    case 3: return kernel_n<3>(d);
    default: return kernel_n<4>(d);
  }
}
size_t smem_for(int N, int d, int K) {
  switch (N) {
    case 1: return smem_n<1>(d, K);
    case 2: return smem_n<2>(d, K);
    case 3: return smem_n<3>(d, K);
    default: return smem_n<4>(d, K);
  }
}

int grid_for(const AmmmseDims* d) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 148;
  const long long g = d->batch < sms ? d->batch : sms;
  return (int)(g < 1 ? 1 : g);
}

bool dims_ok(const AmmmseDims* d) {
  return d && d->batch >= 1 && d->M >= 1 && d->N >= 1 && d->N <= 4 && d->d >= 1 && d->d <= 4 &&
         d->K >= 1 && d->K <= 1024 && (d->dtype == AMMMSE_COMPLEX64 || d->dtype == AMMMSE_COMPLEX128);
}

}  // namespace exact
}  // namespace ammmse

extern "C" {

size_t ammmse_exact_workspace_size(const AmmmseDims* dims) {
  using namespace ammmse::exact;
  if (!dims_ok(dims)) return 0;
  return 256 + (size_t)grid_for(dims) * Slot::count(dims->M, dims->K, dims->N, dims->d) * sizeof(ammmse::cd);
}

int ammmse_solve_exact(const AmmmseDims* dims, const AmmmseProblem* prob, const AmmmseOptions* opt,
                       int algorithm, double bisect_tol, int bisect_max, AmmmseResult* res,
                       void* workspace, size_t workspace_bytes, void* stream) {
  using namespace ammmse::exact;
  if (!dims_ok(dims) || !prob || !opt || !res || !prob->channels || !prob->noise_power ||
      !prob->p_max || !prob->weights || !prob->init_precoders)
    return AMMMSE_ERR_INVALID;
  if (algorithm != AMMMSE_ALGO_WMMSE && algorithm != AMMMSE_ALGO_MMMSE) return AMMMSE_ERR_INVALID;
  if (!(opt->eps1 > 0) || !(opt->eps2 > 0 && isfinite(opt->eps2)) || opt->eps2 > opt->eps1 ||
      opt->max_iters < 1 || !(bisect_tol > 0) || bisect_max < 1)
    return AMMMSE_ERR_INVALID;
  if ((res->iter_receivers != nullptr) != (res->iter_weights != nullptr) ||
      (res->iter_receivers != nullptr) != (res->iter_precoders != nullptr))
    return AMMMSE_ERR_INVALID;
  const size_t need = ammmse_exact_workspace_size(dims);
  if (!workspace || workspace_bytes < need) return AMMMSE_ERR_WORKSPACE;
  const void* f = kernel_for(dims->N, dims->d);
  const size_t smem = smem_for(dims->N, dims->d, dims->K);
  cudaStream_t s = (cudaStream_t)stream;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return AMMMSE_ERR_UNSUPPORTED;
  if (cudaMemsetAsync(workspace, 0, 8, s) != cudaSuccess) return AMMMSE_ERR_CUDA;
  Args a{};
  a.H = prob->channels;
  a.V0 = prob->init_precoders;
  a.c64 = dims->dtype == AMMMSE_COMPLEX64 ? 1 : 0;
  a.sigma2 = prob->noise_power;
  a.pmax = prob->p_max;
  a.alpha = prob->weights;
  a.Vout = res->final_precoders;
  a.wsr_bits = res->wsr_bits;
  a.iterations = res->iterations;
  a.converged = res->converged;
  a.residual = res->stationarity_residual;
  a.switch_it = res->switch_iteration;
  a.status = res->status;
  a.trace = res->trace;
  a.itU = res->iter_receivers;
  a.itW = res->iter_weights;
  a.itV = res->iter_precoders;
  a.eps1 = opt->eps1;
  a.eps2 = opt->eps2;
  a.bisect_tol = bisect_tol;
  a.max_iters = opt->max_iters;
  a.latch = opt->latch_stage ? 1 : 0;
  a.start_weighted = algorithm == AMMMSE_ALGO_WMMSE ? 1 : 0;  // solvers.py:521-537
  a.bisect_max = bisect_max;
  a.M = dims->M;
  a.K = dims->K;
  a.B = dims->batch;
  a.scratch = reinterpret_cast<ammmse::cd*>(reinterpret_cast<unsigned char*>(workspace) + 256);
  a.slot_cd = Slot::count(dims->M, dims->K, dims->N, dims->d);
  a.counter = reinterpret_cast<unsigned long long*>(workspace);
  void* args[] = {&a};
  if (cudaLaunchKernel(f, dim3((unsigned)grid_for(dims)), dim3(kThreads), args, smem, s) != cudaSuccess)
    return AMMMSE_ERR_CUDA;
  return AMMMSE_OK;
}

}  // extern "C"
