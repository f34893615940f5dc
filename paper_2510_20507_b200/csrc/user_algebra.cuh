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

// ---------------------------------------------------------------------------
// Generic N x N / d x d path (Cholesky based), in three parts so that the
// receiver half and the weight half of one user can run on two threads:
//   k1_part_u : A = T_k + σ² I = L_A L_A^H,  U = A^{-1} G_kk (solvers.py:210-225),
//               T = I − U^H G_kk (solvers.py:242) and f_after_u (MSE matrix E = herm(T))
//   k1_part_w : C = A − G_kk G_kk^H (interference + noise) = L_C L_C^H,
//               W = I + Y^H Y with Y = L_C^{-1} G_kk
//   k1_combine: W (weighted stage) or I, ln det W, the ill-conditioning test,
//               f_after_w, P = α U W and D = −P T
// W = T^{-1} at the MMSE receiver by the Woodbury identity
//   (I − G^H A^{-1} G)^{-1} = I + G^H (A − G G^H)^{-1} G,
// and ln det W = ln det A − ln det C (determinant lemma): the weight update of
// solvers.py:228-254 (np.linalg.solve(T, I), hermitianize) without forming or
// factoring T, and independent of the receiver half.  W is Hermitian by
// construction and PD iff C is; the cond > 1e12 test uses ‖T‖_F ‖W‖_F.
// ---------------------------------------------------------------------------
// Re Tr(W E) with E = herm(T) (E[q][p] formed on the fly, same arithmetic as
// storing E first)
template <int DD>
__device__ __forceinline__ double trace_w_herm(const cd (&W)[DD][DD], const cd (&T)[DD][DD]) {
  double tr = 0.0;
#pragma unroll
  for (int p = 0; p < DD; ++p)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      const double er = 0.5 * (T[q][p].r + T[p][q].r), ei = 0.5 * (T[q][p].i - T[p][q].i);
      tr += W[p][q].r * er - W[p][q].i * ei;
    }
  return tr;
}

template <int NN, int DD>
struct K1U {
  cd U[NN][DD];
  cd T[DD][DD];    // E = herm(T) is formed on the fly where needed
  double piv[NN];  // Cholesky pivots of A
  double fu;
  int status;
};

template <int NN, int DD>
struct K1W {
  cd W[DD][DD];
  double piv[NN];  // Cholesky pivots of C
  int pd;
};

template <int NN, int DD>
__device__ __forceinline__ void k1_part_u(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                          double sigma2, double ak, const cd (&Wprev)[DD][DD],
                                          double lndet_wprev, bool want_f, K1U<NN, DD>& o) {
  cd L[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) L[a][b] = Tg[a][b];
#pragma unroll
  for (int a = 0; a < NN; ++a) L[a][a].r += sigma2;
  o.status = chol_lower<NN>(L) ? 0 : AMMMSE_STATUS_NONFINITE;
#pragma unroll
  for (int a = 0; a < NN; ++a) o.piv[a] = L[a][a].r;
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int s = 0; s < DD; ++s) o.U[a][s] = Gkk[a][s];
  chol_solve<NN, DD>(L, o.U);  // U = A^{-1} G_kk (cho_solve)
#pragma unroll
  for (int p = 0; p < DD; ++p)
#pragma unroll
    for (int q = 0; q < DD; ++q) {
      cd s = cmk(0.0);
#pragma unroll
      for (int a = 0; a < NN; ++a) cfmac(s, o.U[a][p], Gkk[a][q]);
      o.T[p][q] = csub(cmk(p == q ? 1.0 : 0.0), s);
    }
  // MSE matrix E = I − U^H G_kk − G_kk^H U + U^H A U at the MMSE receiver:
  // U^H A U = U^H G_kk, so E = T^H (Hermitian part used, as in the 2x2 path)
  o.fu = 0.0;
  if (want_f) {
    const double tr = trace_w_herm<DD>(Wprev, o.T);  // f_after_u uses the previous W (solvers.py:447)
    o.fu = ak * (tr - lndet_wprev);
  }
}

template <int NN, int DD>
__device__ __forceinline__ void k1_part_w(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                          double sigma2, K1W<NN, DD>& o) {
  cd L[NN][NN];  // lower triangle of C = T_k + σ² I − G_kk G_kk^H
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      cd own = cmk(0.0);
#pragma unroll
      for (int s = 0; s < DD; ++s) own = cadd(own, cmulcb(Gkk[a][s], Gkk[b][s]));
      L[a][b] = csub(Tg[a][b], own);
    }
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    L[a][a].r += sigma2;
    L[a][a].i = 0.0;
  }
  o.pd = chol_lower<NN>(L) ? 1 : 0;
#pragma unroll
  for (int a = 0; a < NN; ++a) o.piv[a] = L[a][a].r;
  cd Y[NN][DD];  // Y = L_C^{-1} G_kk (forward substitution)
#pragma unroll
  for (int s = 0; s < DD; ++s)
#pragma unroll
    for (int i = 0; i < NN; ++i) {
      cd t = Gkk[i][s];
#pragma unroll
      for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], Y[p][s]));
      Y[i][s] = cscale(t, 1.0 / L[i][i].r);
    }
#pragma unroll
  for (int p = 0; p < DD; ++p)
#pragma unroll
    for (int q = p; q < DD; ++q) {  // W = I + Y^H Y, Hermitian by construction
      cd s = cmk(p == q ? 1.0 : 0.0);
#pragma unroll
      for (int a = 0; a < NN; ++a) cfmac(s, Y[a][p], Y[a][q]);
      if (p == q) s.i = 0.0;
      o.W[p][q] = s;
      o.W[q][p] = cconj(s);
    }
}

template <int NN, int DD>
__device__ __forceinline__ void k1_combine(const K1U<NN, DD>& u, const cd (&Wm)[DD][DD],
                                           const double (&pivc)[NN], int pdc, double ak,
                                           bool weighted, bool want_f, K1Out<NN, DD>& o) {
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int s = 0; s < DD; ++s) o.U[a][s] = u.U[a][s];
  o.status = u.status;
  o.fu = u.fu;
  o.lndetw = 0.0;
  if (weighted) {
    double nT = 0.0, nW = 0.0;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        nT += cabs2(u.T[p][q]);
        nW += cabs2(Wm[p][q]);
        o.W[p][q] = Wm[p][q];
      }
    // ‖T‖_F ‖W‖_F: an upper bound (within a factor d) of np.linalg.cond(T)
    const double cond = sqrt(nT) * sqrt(nW);
    if ((!pdc || !isfinite(cond) || cond > kCondLimitUA) && o.status == 0)
      o.status = AMMMSE_STATUS_ILL_CONDITIONED;
    if (pdc && u.status == 0) {  // ln det W = ln det A − ln det C, one log
      double q = 1.0;
#pragma unroll
      for (int j = 0; j < NN; ++j) {
        const double r = u.piv[j] / pivc[j];
        q *= r * r;
      }
      if (q >= 2.2250738585072014e-308 && q <= 1.7976931348623157e308) {
        o.lndetw = log(q);
      } else {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NN; ++j) s += log(u.piv[j]) - log(pivc[j]);
        o.lndetw = 2.0 * s;
      }
    }
  } else {
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) o.W[p][q] = cmk(p == q ? 1.0 : 0.0);
  }
  o.fw = 0.0;
  if (want_f) o.fw = ak * (trace_w_herm<DD>(o.W, u.T) - o.lndetw);
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
      for (int p = 0; p < DD; ++p) cfma(acc, o.P[a][p], u.T[p][q]);
      o.D[a][q] = cmk(-acc.r, -acc.i);
    }
}

// weighted: W update (else W = I).  want_f: compute f_after_u / f_after_w
// terms (the exit residual pass does not need them).  One thread per user.
template <int NN, int DD>
__device__ __forceinline__ void k1_math(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                        double sigma2, double ak, const cd (&Wprev)[DD][DD],
                                        double lndet_wprev, bool weighted, bool want_f,
                                        K1Out<NN, DD>& o) {
  if constexpr (NN == 2 && DD == 2) {
    k1_math_22(Tg, Gkk, sigma2, ak, Wprev, lndet_wprev, weighted, want_f, o);
    return;
  } else {
    K1U<NN, DD> u;
    k1_part_u<NN, DD>(Tg, Gkk, sigma2, ak, Wprev, lndet_wprev, want_f, u);
    if (weighted) {
      K1W<NN, DD> w;
      k1_part_w<NN, DD>(Tg, Gkk, sigma2, w);
      k1_combine<NN, DD>(u, w.W, w.piv, w.pd, ak, true, want_f, o);
    } else {
      const cd (&Wm)[DD][DD] = u.T;  // unused when not weighted
      const double (&pv)[NN] = u.piv;
      k1_combine<NN, DD>(u, Wm, pv, 1, ak, false, want_f, o);
    }
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
