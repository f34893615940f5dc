// small_linalg.cuh — per-user dense algebra on N x N / d x d complex matrices
// (N, d <= 4), one thread per user, fp64 in registers.
//
// These are the device restatements of the reference's L0 helpers
// (pkg/src/wsrbeam/linalg.py): hermitianize (:12-14), solve_hpd via a lower
// Cholesky factor (:17-24, scipy cho_factor/cho_solve = LAPACK zpotrf/zpotrs),
// lndet_hpd from the Cholesky diagonal (:27-30); plus the eigvalsh used by
// compute_bounds (objective.py:231).
#pragma once
#include <math.h>

namespace ammmse {

struct cd {
  double r, i;
};

__device__ __forceinline__ cd cmk(double r, double i = 0.0) { return cd{r, i}; }
__device__ __forceinline__ cd cadd(cd a, cd b) { return cd{a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return cd{a.r - b.r, a.i - b.i}; }
__device__ __forceinline__ cd cmul(cd a, cd b) { return cd{a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
// conj(a) * b
__device__ __forceinline__ cd cmulc(cd a, cd b) { return cd{a.r * b.r + a.i * b.i, a.r * b.i - a.i * b.r}; }
// a * conj(b)
__device__ __forceinline__ cd cmulcb(cd a, cd b) { return cd{a.r * b.r + a.i * b.i, a.i * b.r - a.r * b.i}; }
__device__ __forceinline__ cd cconj(cd a) { return cd{a.r, -a.i}; }
__device__ __forceinline__ cd cscale(cd a, double s) { return cd{a.r * s, a.i * s}; }
__device__ __forceinline__ double cabs2(cd a) { return a.r * a.r + a.i * a.i; }
// a += b * c
__device__ __forceinline__ void cfma(cd& a, cd b, cd c) {
  a.r = fma(b.r, c.r, fma(-b.i, c.i, a.r));
  a.i = fma(b.r, c.i, fma(b.i, c.r, a.i));
}
// a += conj(b) * c
__device__ __forceinline__ void cfmac(cd& a, cd b, cd c) {
  a.r = fma(b.r, c.r, fma(b.i, c.i, a.r));
  a.i = fma(b.r, c.i, fma(-b.i, c.r, a.i));
}
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  // Smith-free plain division: |b| is a pivot magnitude well away from 0 here
  double den = 1.0 / cabs2(b);
  return cd{(a.r * b.r + a.i * b.i) * den, (a.i * b.r - a.r * b.i) * den};
}

// In-place lower Cholesky of a Hermitian positive definite matrix whose
// lower triangle (incl. diagonal) is valid.  Returns false if a pivot is not
// strictly positive or not finite (numpy/scipy raise LinAlgError there).
template <int n>
__device__ __forceinline__ bool chol_lower(cd (&A)[n][n]) {
#pragma unroll
  for (int j = 0; j < n; ++j) {
    double s = A[j][j].r;
#pragma unroll
    for (int p = 0; p < j; ++p) s -= cabs2(A[j][p]);
    if (!(s > 0.0) || !isfinite(s)) return false;
    const double l = sqrt(s);
    const double inv = 1.0 / l;
    A[j][j] = cmk(l);
#pragma unroll
    for (int i = j + 1; i < n; ++i) {
      cd t = A[i][j];
#pragma unroll
      for (int p = 0; p < j; ++p) t = csub(t, cmulcb(A[i][p], A[j][p]));
      A[i][j] = cscale(t, inv);
    }
  }
  return true;
}

// ln det of the matrix whose Cholesky factor is L (linalg.py:27-30): one log
// of the product of the pivots (the per-user algebra is latency bound and an
// fp64 log is a long dependent routine), the sum of logs only when the
// product leaves the normal range.
template <int n>
__device__ __forceinline__ double chol_lndet(const cd (&L)[n][n]) {
  double p = 1.0;
#pragma unroll
  for (int j = 0; j < n; ++j) p *= L[j][j].r * L[j][j].r;
  if (p >= 2.2250738585072014e-308 && p <= 1.7976931348623157e308) return log(p);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < n; ++j) s += log(L[j][j].r);
  return 2.0 * s;
}

// ln det(A) - ln det(C) from their Cholesky factors with a single log
template <int n>
__device__ __forceinline__ double chol_lndet_diff(const cd (&LA)[n][n], const cd (&LC)[n][n]) {
  double q = 1.0;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const double r = LA[j][j].r / LC[j][j].r;
    q *= r * r;
  }
  if (q >= 2.2250738585072014e-308 && q <= 1.7976931348623157e308) return log(q);
  return chol_lndet<n>(LA) - chol_lndet<n>(LC);
}

// Solve (L L^H) X = B in place, B is n x m (scipy cho_solve).
template <int n, int m>
__device__ __forceinline__ void chol_solve(const cd (&L)[n][n], cd (&B)[n][m]) {
#pragma unroll
  for (int c = 0; c < m; ++c) {
#pragma unroll
    for (int i = 0; i < n; ++i) {  // forward: L y = b
      cd t = B[i][c];
#pragma unroll
      for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], B[p][c]));
      B[i][c] = cscale(t, 1.0 / L[i][i].r);
    }
#pragma unroll
    for (int i = n - 1; i >= 0; --i) {  // backward: L^H x = y
      cd t = B[i][c];
#pragma unroll
      for (int p = i + 1; p < n; ++p) t = csub(t, cmulc(L[p][i], B[p][c]));
      B[i][c] = cscale(t, 1.0 / L[i][i].r);
    }
  }
}

// Largest eigenvalue of a Hermitian n x n matrix (full storage), via cyclic
// Jacobi on the 2n x 2n real symmetric embedding [[Ar, -Ai], [Ai, Ar]]
// (same spectrum, each eigenvalue doubled).  Once per realization only.
template <int n>
__device__ double herm_eig_max(const cd (&A)[n][n]) {
  if (n == 1) return A[0][0].r;
  constexpr int m = 2 * n;
  double S[m][m];
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < n; ++j) {
      // hermitianize (linalg.py:12-14)
      const double re = 0.5 * (A[i][j].r + A[j][i].r);
      const double im = 0.5 * (A[i][j].i - A[j][i].i);
      S[i][j] = re; S[i + n][j + n] = re;
      S[i + n][j] = im; S[i][j + n] = -im;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < m; ++p) {
      diag += S[p][p] * S[p][p];
      for (int q = p + 1; q < m; ++q) off += S[p][q] * S[p][q];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = S[p][q];
        if (apq == 0.0) continue;
        const double theta = (S[q][q] - S[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int r = 0; r < m; ++r) {  // columns p, q
          const double srp = S[r][p], srq = S[r][q];
          S[r][p] = c * srp - s * srq;
          S[r][q] = s * srp + c * srq;
        }
        for (int r = 0; r < m; ++r) {  // rows p, q
          const double spr = S[p][r], sqr = S[q][r];
          S[p][r] = c * spr - s * sqr;
          S[q][r] = s * spr + c * sqr;
        }
      }
  }
  double mx = S[0][0];
  for (int p = 1; p < m; ++p) mx = fmax(mx, S[p][p]);
  return mx;
}

}  // namespace ammmse
