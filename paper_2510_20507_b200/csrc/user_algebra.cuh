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

// weighted: W update (else W = I).  want_f: compute f_after_u / f_after_w
// terms (the exit residual pass does not need them).
template <int NN, int DD>
__device__ __forceinline__ void k1_math(const cd (&Tg)[NN][NN], const cd (&Gkk)[NN][DD],
                                        double sigma2, double ak, const cd (&Wprev)[DD][DD],
                                        double lndet_wprev, bool weighted, bool want_f,
                                        K1Out<NN, DD>& o) {
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
  // MSE matrix in Gram form: E = I − U^H G_kk − G_kk^H U + U^H A U
  cd E[DD][DD];
  if (want_f) {
    cd AU[NN][DD];
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int s = 0; s < DD; ++s) {
        cd acc = cmk(0.0);
#pragma unroll
        for (int b = 0; b < NN; ++b) cfma(acc, A[a][b], o.U[b][s]);
        AU[a][s] = acc;
      }
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        cd uau = cmk(0.0);
#pragma unroll
        for (int a = 0; a < NN; ++a) cfmac(uau, o.U[a][p], AU[a][q]);
        const cd ghu = cconj(csub(cmk(p == q ? 1.0 : 0.0), T[q][p]));
        E[p][q] = cadd(csub(T[p][q], ghu), uau);
      }
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
    cd Tc[DD][DD], Ti[DD][DD];
    double nT = 0.0;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) {
        Tc[p][q] = T[p][q];
        nT += cabs2(T[p][q]);
      }
    const bool ok = inverse_gj<DD>(Tc, Ti);  // np.linalg.solve(T, I)
    double nTi = 0.0;
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) nTi += cabs2(Ti[p][q]);
    // ‖T‖_F ‖T^{-1}‖_F: an upper bound (within a factor d) of np.linalg.cond
    const double cond = sqrt(nT) * sqrt(nTi);
    if ((!ok || !isfinite(cond) || cond > kCondLimitUA) && o.status == 0)
      o.status = AMMMSE_STATUS_ILL_CONDITIONED;
#pragma unroll
    for (int p = 0; p < DD; ++p)  // hermitianize (linalg.py:12-14)
#pragma unroll
      for (int q = 0; q < DD; ++q)
        o.W[p][q] = cmk(0.5 * (Ti[p][q].r + Ti[q][p].r), 0.5 * (Ti[p][q].i - Ti[q][p].i));
    cd LW[DD][DD];
#pragma unroll
    for (int p = 0; p < DD; ++p)
#pragma unroll
      for (int q = 0; q < DD; ++q) LW[p][q] = o.W[p][q];
    if (!chol_lower<DD>(LW)) {  // eigvalsh(W)[0] <= 0 (solvers.py:249-252)
      if (o.status == 0) o.status = AMMMSE_STATUS_ILL_CONDITIONED;
    } else {
      o.lndetw = chol_lndet<DD>(LW);
    }
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
    double r = chol_lndet<NN>(A) - chol_lndet<NN>(Cv);
    rate = ak * (r > 0.0 ? r : 0.0);
  } else {
    status = AMMMSE_STATUS_NONFINITE;
  }
}

}  // namespace ammmse
