// user_algebra.cuh — per-user fp64 algebra of one A-MMMSE iteration, shared by
// the single-CTA engine and the cluster engine.  One thread per user.
//
//   k1_math : receiver, weight, gradient factor and objective terms of user k
//             (update_receivers solvers.py:210-225, update_weight_matrices
//             :228-254, the Ŷ factors of gradient_v objective.py:196-213,
//             wmmse_objective / mse_matrix objective.py:84-169)
//   wsr_math: rate and f_after_v terms of user k at the new precoders
//             (user_rate objective.py:108-128, wmmse_objective)
//
// Inputs are the user's N x N Gram  T_k = sum_j G_kj G_kj^H  (all columns)
// and its diagonal block G_kk (N x d); everything is fp64.
#pragma once

#include "ammmse.h"
#include "small_linalg.cuh"

namespace ammmse {

constexpr double kCondLimitUA = 1e12;  // solvers.py:71

template <int NN, int DD>
struct K1Out {
  cd U[NN][DD];
  cd W[DD][DD];
  cd P[NN][DD];  // α U W
  cd D[NN][DD];  // −α U W (I − U^H G_kk): diagonal block of Ŷ
  double lndetw;
  double fu, fw;
  int status;
};

// ---------------------------------------------------------------------------
// Closed-form N = d = 2 path (the BASELINE medium / massive / sweep shapes).
// Same mathematics as the generic Cholesky / Gauss-Jordan path: 2x2 Hermitian
// inverses through the adjugate, log-determinants and positive-definiteness
// tests through the determinant (for 2x2: PD <=> a00 > 0 and det > 0; the
// Cholesky log-det 2*sum(log L_jj) equals log(det)).  Cuts the serial fp64
// latency per user from ~10 sqrt/div/log to 2-3 divisions and one log.
// ---------------------------------------------------------------------------
struct H2 {  // Hermitian 2x2: [[a, b], [conj(b), c]], a, c real
  double a, c;
  cd b;
};
__device__ __forceinline__ double det_h2(const H2& m) { return m.a * m.c - cabs2(m.b); }
__device__ __forceinline__ bool pd_h2(const H2& m, double det) { return m.a > 0.0 && det > 0.0 && isfinite(det); }

__device__ __forceinline__ void k1_math_22(const cd (&Tg)[2][2], const cd (&G)[2][2], double sigma2,
                                           double ak, const cd (&Wp)[2][2], double lndet_wprev,
                                           bool weighted, bool want_f, K1Out<2, 2>& o) {
  H2 A{Tg[0][0].r + sigma2, Tg[1][1].r + sigma2, Tg[0][1]};
  const double detA = det_h2(A);
  o.status = pd_h2(A, detA) ? 0 : AMMMSE_STATUS_NONFINITE;
  const double id = 1.0 / detA;
  // U = A^{-1} G, A^{-1} = [[c, -b], [-conj(b), a]] / det
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const cd g0 = G[0][s], g1 = G[1][s];
    const cd u0 = csub(cscale(g0, A.c), cmul(A.b, g1));
    const cd u1 = csub(cscale(g1, A.a), cmul(cconj(A.b), g0));
    o.U[0][s] = cscale(u0, id);
    o.U[1][s] = cscale(u1, id);
  }
  cd T[2][2];  // T = I - U^H G
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cd s = cmk(0.0);
      cfmac(s, o.U[0][p], G[0][q]);
      cfmac(s, o.U[1][p], G[1][q]);
      T[p][q] = csub(cmk(p == q ? 1.0 : 0.0), s);
    }
  cd E[2][2];
  if (want_f) {
    // At the MMSE receiver U = A^{-1} G:  U^H A U = U^H G, so the MSE matrix
    // E = I - U^H G - G^H U + U^H A U  reduces to  I - G^H U = T^H  (T is
    // Hermitian there up to rounding; its Hermitian part is used).
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        E[p][q] = cmk(0.5 * (T[p][q].r + T[q][p].r), 0.5 * (T[p][q].i - T[q][p].i));
    double tr = 0.0;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q) tr += Wp[p][q].r * E[q][p].r - Wp[p][q].i * E[q][p].i;
    o.fu = ak * (tr - lndet_wprev);
  } else {
    o.fu = 0.0;
  }
  o.lndetw = 0.0;
  if (weighted) {
    // T^{-1} = adj(T) / det(T)  (np.linalg.solve(T, I))
    const cd detT = csub(cmul(T[0][0], T[1][1]), cmul(T[0][1], T[1][0]));
    const double adet = cabs2(detT);
    const double nT = cabs2(T[0][0]) + cabs2(T[0][1]) + cabs2(T[1][0]) + cabs2(T[1][1]);
    cd Ti[2][2];
    if (adet > 0.0 && isfinite(adet)) {
      const cd inv = cdiv(cmk(1.0), detT);
      Ti[0][0] = cmul(T[1][1], inv);
      Ti[1][1] = cmul(T[0][0], inv);
      Ti[0][1] = cmul(cmk(-T[0][1].r, -T[0][1].i), inv);
      Ti[1][0] = cmul(cmk(-T[1][0].r, -T[1][0].i), inv);
    } else {
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 2; ++q) Ti[p][q] = cmk(0.0);
    }
    // ‖T‖_F ‖T^{-1}‖_F = ‖T‖_F^2 / |det T| for 2x2 (the adjugate has T's entries)
    const double cond = nT / sqrt(adet);
    if ((!(adet > 0.0) || !isfinite(cond) || cond > kCondLimitUA) && o.status == 0)
      o.status = AMMMSE_STATUS_ILL_CONDITIONED;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        o.W[p][q] = cmk(0.5 * (Ti[p][q].r + Ti[q][p].r), 0.5 * (Ti[p][q].i - Ti[q][p].i));
    const H2 Wh{o.W[0][0].r, o.W[1][1].r, o.W[0][1]};
    const double detW = det_h2(Wh);
    if (!pd_h2(Wh, detW)) {
      if (o.status == 0) o.status = AMMMSE_STATUS_ILL_CONDITIONED;
    } else {
      o.lndetw = log(detW);
    }
  } else {
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q) o.W[p][q] = cmk(p == q ? 1.0 : 0.0);
  }
  if (want_f) {
    double tr = 0.0;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q) tr += o.W[p][q].r * E[q][p].r - o.W[p][q].i * E[q][p].i;
    o.fw = ak * (tr - o.lndetw);
  } else {
    o.fw = 0.0;
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cd acc = cmk(0.0);
      cfma(acc, o.U[a][0], o.W[0][q]);
      cfma(acc, o.U[a][1], o.W[1][q]);
      o.P[a][q] = cscale(acc, ak);
    }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cd acc = cmk(0.0);
      cfma(acc, o.P[a][0], T[0][q]);
      cfma(acc, o.P[a][1], T[1][q]);
      o.D[a][q] = cmk(-acc.r, -acc.i);
    }
}

__device__ __forceinline__ void wsr_math_22(const cd (&Tg)[2][2], const cd (&G)[2][2], double sigma2,
                                            double ak, const cd (&U)[2][2], const cd (&W)[2][2],
                                            double lndetw, double& rate, double& fv, int& status) {
  const H2 A{Tg[0][0].r + sigma2, Tg[1][1].r + sigma2, Tg[0][1]};
  cd own01 = cmk(0.0);
  double own00 = 0.0, own11 = 0.0;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    own00 += cabs2(G[0][s]);
    own11 += cabs2(G[1][s]);
    own01 = cadd(own01, cmulcb(G[0][s], G[1][s]));
  }
  const H2 Cv{A.a - own00, A.c - own11, csub(A.b, own01)};
  double tr = 0.0;  // Tr(W E) with E = I - U^H G - G^H U + U^H A U
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cd uhg = cmk(0.0), ghu = cmk(0.0);
      cfmac(uhg, U[0][p], G[0][q]);
      cfmac(uhg, U[1][p], G[1][q]);
      cfmac(ghu, G[0][p], U[0][q]);
      cfmac(ghu, G[1][p], U[1][q]);
      const cd au0 = cadd(cscale(U[0][q], A.a), cmul(A.b, U[1][q]));
      const cd au1 = cadd(cmul(cconj(A.b), U[0][q]), cscale(U[1][q], A.c));
      cd uau = cmk(0.0);
      cfmac(uau, U[0][p], au0);
      cfmac(uau, U[1][p], au1);
      cd e = csub(csub(uau, uhg), ghu);
      if (p == q) e.r += 1.0;
      tr += W[q][p].r * e.r - W[q][p].i * e.i;
    }
  fv = ak * (tr - lndetw);
  const double dA = det_h2(A), dC = det_h2(Cv);
  status = 0;
  rate = 0.0;
  if (pd_h2(A, dA) && pd_h2(Cv, dC)) {
    const double r = log(dA / dC);  // lndet(cov + own) - lndet(cov)
    rate = ak * (r > 0.0 ? r : 0.0);
  } else {
    status = AMMMSE_STATUS_NONFINITE;
  }
}

// weighted: W update (else W = I).  want_f: compute f_after_u / f_after_w
// terms (the exit residual pass does not need them).
template <int NN, int DD>
__device__ __forceinline__ void k1_math(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                        double sigma2, double ak, const cd (&Wprev)[DD][DD],
                                        double lndet_wprev, bool weighted, bool want_f,
                                        K1Out<NN, DD>& o) {
  if constexpr (NN == 2 && DD == 2) {
    k1_math_22(Tg, Gkk, sigma2, ak, Wprev, lndet_wprev, weighted, want_f, o);
    return;
  }
  cd A[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) A[a][b] = Tg[a][b];
#pragma unroll
  for (int a = 0; a < NN; ++a) A[a][a].r += sigma2;
  cd Lc[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) Lc[a][b] = A[a][b];
  o.status = 0;
  if (!chol_lower<NN>(Lc)) o.status = AMMMSE_STATUS_NONFINITE;
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int s = 0; s < DD; ++s) o.U[a][s] = Gkk[a][s];
  chol_solve<NN, DD>(Lc, o.U);  // U = A^{-1} G_kk (cho_solve)
  // T = I − U^H G_kk  (solvers.py:242)
  cd T[DD][DD];
#pragma unroll
  for (int p = 0; p < DD; ++p)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      cd s = cmk(0.0);
#pragma unroll
      for (int a = 0; a < NN; ++a) cfmac(s, o.U[a][p], Gkk[a][q]);
      T[p][q] = csub(cmk(p == q ? 1.0 : 0.0), s);
    }
  // MSE matrix E = I − U^H G_kk − G_kk^H U + U^H A U at the MMSE receiver:
  // U^H A U = U^H G_kk, so E = T^H (Hermitian part used, as in the 2x2 path)
  cd E[DD][DD];
  if (want_f) {
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q)
        E[p][q] = cmk(0.5 * (T[p][q].r + T[q][p].r), 0.5 * (T[p][q].i - T[q][p].i));
    double tr = 0.0;  // Tr(W_prev E): f_after_u uses the previous W (solvers.py:447)
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) tr += Wprev[p][q].r * E[q][p].r - Wprev[p][q].i * E[q][p].i;
    o.fu = ak * (tr - lndet_wprev);
  } else {
    o.fu = 0.0;
  }
  o.lndetw = 0.0;
  if (weighted) {
    // W = herm(T^{-1}) (np.linalg.solve(T, I) then hermitianize, linalg.py:12-14).
    // T's anti-Hermitian part is rounding-level at the MMSE point, and
    // herm(T^{-1}) = herm(T)^{-1} to second order in it, so W is formed from
    // one Cholesky factorisation of herm(T): W = L^{-H} L^{-1}.  The same
    // factor gives ln det W = -ln det herm(T) and the PD test of W
    // (eigvalsh(W)[0] > 0, solvers.py:249-252): W is PD iff herm(T) is.
    cd LT[DD][DD];
    double nT = 0.0;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        nT += cabs2(T[p][q]);
        LT[p][q] = cmk(0.5 * (T[p][q].r + T[q][p].r), 0.5 * (T[p][q].i - T[q][p].i));
      }
    const bool pd = chol_lower<DD>(LT);
    cd Ti[DD][DD];
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) Ti[p][q] = cmk(p == q ? 1.0 : 0.0);
    double nTi = 0.0;
    if (pd) {
      chol_solve<DD, DD>(LT, Ti);
#pragma unroll
      for (int p = 0; p < DD; ++p)
#pragma unroll
        for (int q = 0; q < DD; ++q) nTi += cabs2(Ti[p][q]);
    }
    // ‖T‖_F ‖T^{-1}‖_F: an upper bound (within a factor d) of np.linalg.cond
    const double cond = sqrt(nT) * sqrt(nTi);
    if ((!pd || !isfinite(cond) || cond > kCondLimitUA) && o.status == 0)
      o.status = AMMMSE_STATUS_ILL_CONDITIONED;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q)
        o.W[p][q] = cmk(0.5 * (Ti[p][q].r + Ti[q][p].r), 0.5 * (Ti[p][q].i - Ti[q][p].i));
    if (pd) o.lndetw = -chol_lndet<DD>(LT);
  } else {
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) o.W[p][q] = cmk(p == q ? 1.0 : 0.0);
  }
  if (want_f) {
    double tr = 0.0;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) tr += o.W[p][q].r * E[q][p].r - o.W[p][q].i * E[q][p].i;
    o.fw = ak * (tr - o.lndetw);
  } else {
    o.fw = 0.0;
  }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      cd acc = cmk(0.0);
#pragma unroll
      for (int p = 0; p < DD; ++p) cfma(acc, o.U[a][p], o.W[p][q]);
      o.P[a][q] = cscale(acc, ak);
    }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      cd acc = cmk(0.0);
#pragma unroll
      for (int p = 0; p < DD; ++p) cfma(acc, o.P[a][p], T[p][q]);
      o.D[a][q] = cmk(-acc.r, -acc.i);
    }
}

// Rate (clipped at 0, in nats, times alpha) and f_after_v term of user k.
// Tg = sum_j G_kj G_kj^H over all columns of the new G.
template <int NN, int DD>
__device__ __forceinline__ void wsr_math(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                         double sigma2, double ak, const cd (&U)[NN][DD],
                                         const cd (&W)[DD][DD], double lndetw, double& rate,
                                         double& fv, int& status) {
  if constexpr (NN == 2 && DD == 2) {
    wsr_math_22(Tg, Gkk, sigma2, ak, U, W, lndetw, rate, fv, status);
    return;
  }
  cd A[NN][NN], Cv[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      A[a][b] = Tg[a][b];
      cd own = cmk(0.0);
#pragma unroll
      for (int s = 0; s < DD; ++s) own = cadd(own, cmulcb(Gkk[a][s], Gkk[b][s]));
      Cv[a][b] = csub(A[a][b], own);  // interference-plus-noise (j != k)
    }
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    A[a][a].r += sigma2;
    A[a][a].i = 0.0;
    Cv[a][a].r += sigma2;
    Cv[a][a].i = 0.0;
  }
  double tr = 0.0;
#pragma unroll
  for (int p = 0; p < DD; ++p)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      cd uhg = cmk(0.0), ghu = cmk(0.0), uau = cmk(0.0);
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        cfmac(uhg, U[a][p], Gkk[a][q]);
        cfmac(ghu, Gkk[a][p], U[a][q]);
        cd au = cmk(0.0);
#pragma unroll
        for (int b = 0; b < NN; ++b) cfma(au, A[a][b], U[b][q]);
        cfmac(uau, U[a][p], au);
      }
      cd e = csub(csub(uau, uhg), ghu);
      if (p == q) e.r += 1.0;
      tr += W[q][p].r * e.r - W[q][p].i * e.i;
    }
  fv = ak * (tr - lndetw);
  status = 0;
  rate = 0.0;
  if (chol_lower<NN>(A) && chol_lower<NN>(Cv)) {
    double r = chol_lndet_diff<NN>(A, Cv);
    rate = ak * (r > 0.0 ? r : 0.0);
  } else {
    status = AMMMSE_STATUS_NONFINITE;
  }
}

}  // namespace ammmse
