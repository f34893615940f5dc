// user_algebra_quad.cuh — per-user fp64 algebra of one A-MMMSE iteration for
// N = d = 4 with FOUR LANES PER USER (lane s of a quad owns column s of the
// user's N x d matrices), eight users per warp.  Same mathematics as
// user_algebra.cuh (update_receivers solvers.py:210-225, update_weight_matrices
// :228-254 in the Woodbury form, the Ŷ factors of objective.py:196-213,
// wmmse_objective / user_rate objective.py:84-169), reorganised so that a warp
// issues each instruction for 32 useful lanes instead of 8:
//   * the 4 x 4 Cholesky factorisations are replicated in the quad's lanes,
//   * everything that is column separable (triangular solves, U^H G, A U, U W,
//     P T, the traces) is split by column,
//   * the few full matrices a lane needs from its neighbours (U, Y, P) go through
//     a per-user shared-memory scratch and __syncwarp.
// Traces use  Re Tr(W herm(T)) = Re Tr(W T)  (W Hermitian) and
//   Re Tr(W E) = Tr W + Re Σ conj(UW) ∘ (A U − 2 G),  E = I − U^H G − G^H U + U^H A U.
#pragma once

#include "user_algebra.cuh"

namespace ammmse {
namespace quad {

constexpr int kScratch = 72;  // doubles per user: Y, P (16 cd each), pivots of C, flag

__device__ __forceinline__ double qsum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// ln(Π pa_j² / Π pc_j²) with one log (chol_lndet_diff)
__device__ __forceinline__ double lndet_diff4(const double (&pa)[4], const double (&pc)[4]) {
  double q = 1.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double r = pa[j] / pc[j];
    q *= r * r;
  }
  if (q >= 2.2250738585072014e-308 && q <= 1.7976931348623157e308) return log(q);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += log(pa[j]) - log(pc[j]);
  return 2.0 * s;
}

// lower triangle of G G^H
__device__ __forceinline__ void own_gram4(const cd (&G)[4][4], cd (&O)[4][4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      cd o = cmk(0.0);
#pragma unroll
      for (int q = 0; q < 4; ++q) o = cadd(o, cmulcb(G[a][q], G[b][q]));
      O[a][b] = o;
    }
}

// Rate and f_after_v term of one user (wsr_math), lane s = column s.
//   Tg: Gram of the new G rows; G: diagonal block; U, W: the iteration's receiver / weight.
// Results valid in every lane of the quad.
// Column-s vectors (gs = G[:, s], us = U[:, s], ws = W[:, s]) are passed
// separately: indexing a register array with the runtime lane column would
// push it to local memory.
__device__ __forceinline__ void wsr_quad(const cd (&Tg)[4][4], const cd (&G)[4][4], const cd (&gs)[4],
                                         double sigma2, double ak, const cd (&U)[4][4], const cd (&us)[4],
                                         const cd (&ws)[4], double wss, double lndetw, int s, double& rate,
                                         double& fv, int& status) {
  // column s of A U and of U W
  cd au[4], uw[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cd x = cscale(us[a], sigma2), y = cmk(0.0);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      cfma(x, Tg[a][b], us[b]);
      cfma(y, U[a][b], ws[b]);
    }
    au[a] = x;
    uw[a] = y;
  }
  double term = wss;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const cd z = cmk(au[a].r - 2.0 * gs[a].r, au[a].i - 2.0 * gs[a].i);
    term += uw[a].r * z.r + uw[a].i * z.i;  // Re(conj(uw) z)
  }
  fv = ak * (qsum(term) - lndetw);
  // lanes 0, 1 factor A = Tg + σ² I, lanes 2, 3 factor C = A − G G^H
  cd O[4][4], Mx[4][4];
  own_gram4(G, O);
  const double sel = s >= 2 ? 1.0 : 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) Mx[a][b] = cmk(Tg[a][b].r - sel * O[a][b].r, Tg[a][b].i - sel * O[a][b].i);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    Mx[a][a].r += sigma2;
    Mx[a][a].i = 0.0;
  }
  const bool ok = chol_lower<4>(Mx);
  double pa[4], pc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double pv = Mx[j][j].r;
    pa[j] = __shfl_sync(0xffffffffu, pv, 0, 4);
    pc[j] = __shfl_sync(0xffffffffu, pv, 2, 4);
  }
  const unsigned okm = __ballot_sync(0xffffffffu, ok);
  const int lane = threadIdx.x & 31;
  const bool okq = ((okm >> (lane & ~3)) & 0xFu) == 0xFu;
  status = 0;
  rate = 0.0;
  if (okq) {
    const double r = lndet_diff4(pa, pc);
    rate = ak * (r > 0.0 ? r : 0.0);
  } else {
    status = AMMMSE_STATUS_NONFINITE;
  }
}

// Receiver half of K1 (k1_part_u), lane s = column s.  Outputs: u (column s of U,
// also written to ucol[a * 4 + s]), tcol (column s of T = I − U^H G), fu, nT
// (‖T‖_F², quad sum), piv (Cholesky pivots of A), status.  `Ufull` returns the
// whole U (read back from `ucol` after a warp barrier).
__device__ __forceinline__ void k1u_quad(const cd (&Tg)[4][4], const cd (&gs)[4], double sigma2, double ak,
                                         const cd (&Wprow)[4], double lndet_wprev, int s, cd* ucol,
                                         cd (&Ufull)[4][4], cd (&u)[4], cd (&tcol)[4], double& fu, double& nT,
                                         double (&piv)[4], int& status) {
  cd L[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) L[a][b] = Tg[a][b];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    L[a][a].r += sigma2;
    L[a][a].i = 0.0;
  }
  status = chol_lower<4>(L) ? 0 : AMMMSE_STATUS_NONFINITE;
#pragma unroll
  for (int a = 0; a < 4; ++a) piv[a] = L[a][a].r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // forward: L y = g_s
    cd t = gs[i];
#pragma unroll
    for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], u[p]));
    u[i] = cscale(t, 1.0 / L[i][i].r);
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {  // backward: L^H x = y
    cd t = u[i];
#pragma unroll
    for (int p = i + 1; p < 4; ++p) t = csub(t, cmulc(L[p][i], u[p]));
    u[i] = cscale(t, 1.0 / L[i][i].r);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) ucol[a * 4 + s] = u[a];
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) Ufull[a][q] = ucol[a * 4 + q];
  double nt = 0.0, tr = 0.0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    cd acc = cmk(0.0);
#pragma unroll
    for (int a = 0; a < 4; ++a) cfmac(acc, Ufull[a][p], gs[a]);
    tcol[p] = cmk((p == s ? 1.0 : 0.0) - acc.r, -acc.i);
    nt += cabs2(tcol[p]);
    tr += Wprow[p].r * tcol[p].r - Wprow[p].i * tcol[p].i;  // Re(Wprev[s][p] T[p][s])
  }
  nT = qsum(nt);
  fu = ak * (qsum(tr) - lndet_wprev);
}

// Weight half of K1 (k1_part_w), lane s = column s: C = Tg + σ² I − G G^H = Lc Lc^H,
// Y = Lc^{-1} G, W = I + Y^H Y.  Writes column s of W to wcol[p * 4 + s]; returns
// the pivots of C and the positive-definiteness flag.  `yscr`: 16 cd of scratch.
__device__ __forceinline__ void k1w_quad(const cd (&Tg)[4][4], const cd (&G)[4][4], const cd (&gs)[4],
                                         double sigma2, int s, cd* yscr, cd* wcol, double (&piv)[4], int& pd) {
  cd O[4][4], L[4][4];
  own_gram4(G, O);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) L[a][b] = csub(Tg[a][b], O[a][b]);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    L[a][a].r += sigma2;
    L[a][a].i = 0.0;
  }
  pd = chol_lower<4>(L) ? 1 : 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) piv[a] = L[a][a].r;
  cd y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cd t = gs[i];
#pragma unroll
    for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], y[p]));
    y[i] = cscale(t, 1.0 / L[i][i].r);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) yscr[a * 4 + s] = y[a];
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    cd acc = cmk(p == s ? 1.0 : 0.0);
#pragma unroll
    for (int a = 0; a < 4; ++a) cfmac(acc, yscr[a * 4 + p], y[a]);
    if (p == s) acc.i = 0.0;
    wcol[p * 4 + s] = acc;
  }
}

// K1 combine (k1_combine), lane s = column s, after the W columns are visible.
//   wcol_s[p] = W[p][s];  Ufull, tcol, nT, piva from k1u_quad;  pivc, pdc from k1w_quad.
// Outputs column s of P = α U W and D = −P T, fw, lndetw, and the updated status.
__device__ __forceinline__ void k1c_quad(const cd (&Ufull)[4][4], const cd (&us)[4], const cd (&tcol)[4], double nT,
                                         const double (&piva)[4], const cd (&wcol_s)[4],
                                         const double (&pivc)[4], int pdc, double ak, bool weighted, int s,
                                         cd* pscr, cd (&pcol)[4], cd (&dcol)[4], double& fw, double& lndetw,
                                         int& status) {
  lndetw = 0.0;
  double trw = 0.0;
  if (weighted) {
    double nw = 0.0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      nw += cabs2(wcol_s[p]);
      // Re(W[s][p] T[p][s]) with W[s][p] = conj(W[p][s])
      trw += wcol_s[p].r * tcol[p].r + wcol_s[p].i * tcol[p].i;
    }
    const double nW = qsum(nw);
    const double cond = sqrt(nT) * sqrt(nW);  // ‖T‖_F ‖W‖_F >= cond_2(T)
    if ((!pdc || !isfinite(cond) || cond > kCondLimitUA) && status == 0)
      status = AMMMSE_STATUS_ILL_CONDITIONED;
    if (pdc && status != AMMMSE_STATUS_NONFINITE) lndetw = lndet_diff4(piva, pivc);
  } else {
    trw = s == 0 ? tcol[0].r : (s == 1 ? tcol[1].r : (s == 2 ? tcol[2].r : tcol[3].r));  // W = I
  }
  fw = ak * (qsum(trw) - lndetw);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cd acc = cmk(0.0);
    if (weighted) {
#pragma unroll
      for (int p = 0; p < 4; ++p) cfma(acc, Ufull[a][p], wcol_s[p]);
    } else {
      acc = us[a];
    }
    pcol[a] = cscale(acc, ak);
    pscr[a * 4 + s] = pcol[a];
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cd acc = cmk(0.0);
#pragma unroll
    for (int p = 0; p < 4; ++p) cfma(acc, pscr[a * 4 + p], tcol[p]);
    dcol[a] = cmk(-acc.r, -acc.i);
  }
}

}  // namespace quad
}  // namespace ammmse
