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

// doubles per user: Y [0,32), P [32,64), T [64,96) (16 cd each), then ‖T‖², pivots of A, status
constexpr int kScratch = 104;

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

// In-place lower Cholesky (chol_lower) that also returns the inverse pivots:
// one rsqrt per column instead of sqrt + division, and no divisions in the
// triangular solves that follow (the per-user algebra is a chain of dependent
// fp64 operations; a division or square root costs ~20 of them).
__device__ __forceinline__ bool chol4_inv(cd (&A)[4][4], double (&inv)[4]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double s = A[j][j].r;
#pragma unroll
    for (int p = 0; p < j; ++p) s -= cabs2(A[j][p]);
    ok = ok && (s > 0.0) && isfinite(s);
    const double r = rsqrt(s);
    inv[j] = r;
    A[j][j] = cmk(s * r);
#pragma unroll
    for (int i = j + 1; i < 4; ++i) {
      cd t = A[i][j];
#pragma unroll
      for (int p = 0; p < j; ++p) t = csub(t, cmulcb(A[i][p], A[j][p]));
      A[i][j] = cscale(t, r);
    }
  }
  return ok;
}

// ln(Π (pa_j ic_j)²): log-det difference from pivots of A and inverse pivots of C
__device__ __forceinline__ double lndet_diff4i(const double (&pa)[4], const double (&ic)[4]) {
  double q = 1.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double r = pa[j] * ic[j];
    q *= r * r;
  }
  if (q >= 2.2250738585072014e-308 && q <= 1.7976931348623157e308) return log(q);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += log(pa[j]) + log(ic[j]);
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
                                         const cd (&ws)[4], double wss, double lndetw, int s, bool want_f,
                                         double& rate, double& fv, int& status) {
  fv = 0.0;
  if (want_f) {  // f_after_v feeds the trace only
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
  }
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
  double ivp[4];
  const bool ok = chol4_inv(Mx, ivp);
  double pa[4], pc[4];  // pivots of A, INVERSE pivots of C
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pa[j] = __shfl_sync(0xffffffffu, Mx[j][j].r, 0, 4);
    pc[j] = __shfl_sync(0xffffffffu, ivp[j], 2, 4);
  }
  const unsigned okm = __ballot_sync(0xffffffffu, ok);
  const int lane = threadIdx.x & 31;
  const bool okq = ((okm >> (lane & ~3)) & 0xFu) == 0xFu;
  status = 0;
  rate = 0.0;
  if (okq) {
    const double r = lndet_diff4i(pa, pc);
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
                                         const cd (&Wprow)[4], double lndet_wprev, int s, bool want_f, cd* ucol,
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
  double ivp[4];
  status = chol4_inv(L, ivp) ? 0 : AMMMSE_STATUS_NONFINITE;
#pragma unroll
  for (int a = 0; a < 4; ++a) piv[a] = L[a][a].r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // forward: L y = g_s
    cd t = gs[i];
#pragma unroll
    for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], u[p]));
    u[i] = cscale(t, ivp[i]);
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {  // backward: L^H x = y
    cd t = u[i];
#pragma unroll
    for (int p = i + 1; p < 4; ++p) t = csub(t, cmulc(L[p][i], u[p]));
    u[i] = cscale(t, ivp[i]);
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
  fu = want_f ? ak * (qsum(tr) - lndet_wprev) : 0.0;
}

// Weight half of K1 (k1_part_w), lane s = column s: C = Tg + σ² I − G G^H = Lc Lc^H,
// Y = Lc^{-1} G, W = I + Y^H Y.  Writes column s of W to wcol[p * 4 + s]; returns
// the INVERSE pivots of C and the positive-definiteness flag.  `yscr`: 16 cd of scratch.
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
  pd = chol4_inv(L, piv) ? 1 : 0;  // piv: INVERSE pivots of C
  cd y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cd t = gs[i];
#pragma unroll
    for (int p = 0; p < i; ++p) t = csub(t, cmul(L[i][p], y[p]));
    y[i] = cscale(t, piv[i]);
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

// K1 combine (k1_combine), statistics half, lane s = column s: the ill-conditioning
// test on ‖T‖_F ‖W‖_F, ln det W = ln det A − ln det C and f_after_w.
//   wcol_s[p] = W[p][s], tcol[p] = T[p][s], nT = ‖T‖_F²; piva: pivots of A; ipivc:
//   INVERSE pivots of C.  want_f = false skips the log and the trace (they feed
//   the recorded trace only).
__device__ __forceinline__ void k1c_stat(const cd (&tcol)[4], double nT, const double (&piva)[4],
                                         const cd (&wcol_s)[4], const double (&ipivc)[4], int pdc, double ak,
                                         bool weighted, bool want_f, int s, double& fw, double& lndetw,
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
    const double c2 = nT * nW;  // (‖T‖_F ‖W‖_F)² >= cond_2(T)²: no square roots
    if ((!pdc || !isfinite(c2) || c2 > kCondLimitUA * kCondLimitUA) && status == 0)
      status = AMMMSE_STATUS_ILL_CONDITIONED;
    if (want_f && pdc && status != AMMMSE_STATUS_NONFINITE) lndetw = lndet_diff4i(piva, ipivc);
  } else {
    trw = s == 0 ? tcol[0].r : (s == 1 ? tcol[1].r : (s == 2 ? tcol[2].r : tcol[3].r));  // W = I
  }
  fw = want_f ? ak * (qsum(trw) - lndetw) : 0.0;
}

// K1 combine, product half: column s of P = α U W and D = −P T (the Ŷ factors of
// objective.py:196-213).  pscr: 16 cd of per-user scratch.
__device__ __forceinline__ void k1c_pd(const cd (&Ufull)[4][4], const cd (&us)[4], const cd (&tcol)[4],
                                       const cd (&wcol_s)[4], double ak, bool weighted, int s, cd* pscr,
                                       cd (&pcol)[4], cd (&dcol)[4]) {
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

// ---------------------------------------------------------------------------
// Warp-level drivers.  NOT inlined on purpose: inside the persistent solver
// kernel the register allocator is saturated (255 registers, spills around
// every fp64 chain, and every cluster barrier flushes L1, where the spills
// live); as separate functions they get their own allocation.  All operands
// are shared-memory pointers.
//   G: the own users' N x d diagonal blocks, fp32, addressed through QuadArgs
//   strides (in place in a G plane, or a compact saved copy).
//   gram: reduced Grams, 16 cd per GLOBAL user.  ucache / wcache: 16 cd per own user.
// ---------------------------------------------------------------------------
struct QuadArgs {
  const float* Gr;  // diagonal blocks: element (own user kl, row p, column c) at Gr[kl * ustride + p * rstride + c]
  const float* Gi;
  int ustride, rstride, k0, KL;
  const cd* gram;
  double sigma2;
  const double* alpha;
  int want_f;  // compute the f_after_u / w / v terms and ln det W (they feed the trace only)
};

// WSR(t): rate[kl], fv[kl], ust2[kl] of the own users (one full warp)
static __device__ __noinline__ void wsr_users(QuadArgs q, const cd* ucache, const cd* wcache, const double* lndetw,
                                       double* rate, double* fv, double* ust2) {
  __builtin_assume(__isShared(q.Gr));
  __builtin_assume(__isShared(q.Gi));
  __builtin_assume(__isShared(q.gram));
  __builtin_assume(__isShared(q.alpha));
  __builtin_assume(__isShared(ucache));
  __builtin_assume(__isShared(wcache));
  __builtin_assume(__isShared(lndetw));
  __builtin_assume(__isShared(rate));
  const int lane = threadIdx.x & 31, ul = lane >> 2, sc = lane & 3;
  for (int kl0 = 0; kl0 < q.KL; kl0 += 8) {
    const bool act = kl0 + ul < q.KL;
    const int kl = act ? kl0 + ul : 0;
    cd Tg[4][4], G[4][4], U[4][4], gs[4], us[4], ws[4];
    const cd* g = q.gram + (size_t)(q.k0 + kl) * 16;
    const size_t gbase = (size_t)kl * q.ustride;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        Tg[p][c] = g[p * 4 + c];
        G[p][c] = cmk((double)q.Gr[gbase + p * q.rstride + c], (double)q.Gi[gbase + p * q.rstride + c]);
        U[p][c] = ucache[kl * 16 + p * 4 + c];
      }
#pragma unroll
    for (int p = 0; p < 4; ++p) {  // column sc (no dynamic register indexing)
      gs[p] = cmk((double)q.Gr[gbase + p * q.rstride + sc], (double)q.Gi[gbase + p * q.rstride + sc]);
      us[p] = ucache[kl * 16 + p * 4 + sc];
      ws[p] = wcache[kl * 16 + p * 4 + sc];
    }
    const double wss = wcache[kl * 16 + sc * 4 + sc].r;
    double rr, ff;
    int st;
    wsr_quad(Tg, G, gs, q.sigma2, q.alpha[kl], U, us, ws, wss, lndetw[kl], sc, q.want_f != 0, rr, ff, st);
    if (act && sc == 0) {
      rate[kl] = rr;
      fv[kl] = ff;
      ust2[kl] = st;
    }
  }
}


// ---------------------------------------------------------------------------
// WSR(t) split over two warps (the rate needs two independent 4 x 4 Cholesky
// factorisations per user, A = T + σ² I and C = A − G G^H, each a chain of
// dependent fp64 operations): warp "A" factors A (and forms the f_after_v term
// when a trace is recorded), warp "C" forms G G^H — row s on lane s, exchanged
// through the scratch — and factors C; they meet at named barrier 2 (64 threads)
// once per pass of 8 users and warp A finishes the rate.
//   wscr: kWsrScratch doubles per own user.
// ---------------------------------------------------------------------------
constexpr int kWsrScratch = 40;  // G G^H rows (16 cd), inverse pivots of C (4), ok flag

static __device__ __noinline__ void wsr_users_c(QuadArgs q, double* wscr) {
  const int lane = threadIdx.x & 31, ul = lane >> 2, sc = lane & 3;
  for (int kl0 = 0; kl0 < q.KL; kl0 += 8) {
    const bool act = kl0 + ul < q.KL;
    const int kl = act ? kl0 + ul : 0;
    const cd* g = q.gram + (size_t)(q.k0 + kl) * 16;
    const size_t gbase = (size_t)kl * q.ustride;
    cd G[4][4], grow[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        G[p][c] = cmk((double)q.Gr[gbase + p * q.rstride + c], (double)q.Gi[gbase + p * q.rstride + c]);
      grow[p] = cmk((double)q.Gr[gbase + sc * q.rstride + p], (double)q.Gi[gbase + sc * q.rstride + p]);
    }
    double* scr = wscr + (size_t)kl * kWsrScratch;
    cd* orow = reinterpret_cast<cd*>(scr);
#pragma unroll
    for (int b = 0; b < 4; ++b) {  // (G G^H)[sc][b]
      cd o = cmk(0.0);
#pragma unroll
      for (int c = 0; c < 4; ++c) o = cadd(o, cmulcb(grow[c], G[b][c]));
      orow[sc * 4 + b] = o;
    }
    __syncwarp();
    cd L[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) L[a][b] = csub(g[a * 4 + b], orow[a * 4 + b]);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      L[a][a].r += q.sigma2;
      L[a][a].i = 0.0;
    }
    double ic[4];
    const bool ok = chol4_inv(L, ic);
    if (sc == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) scr[32 + j] = ic[j];
      scr[36] = ok ? 1.0 : 0.0;
    }
    asm volatile("bar.sync 2, 64;\n" ::: "memory");
  }
}

static __device__ __noinline__ void wsr_users_a(QuadArgs q, const cd* ucache, const cd* wcache,
                                                const double* lndetw, const double* wscr, double* rate,
                                                double* fv, double* ust2) {
  const int lane = threadIdx.x & 31, ul = lane >> 2, sc = lane & 3;
  for (int kl0 = 0; kl0 < q.KL; kl0 += 8) {
    const bool act = kl0 + ul < q.KL;
    const int kl = act ? kl0 + ul : 0;
    const cd* g = q.gram + (size_t)(q.k0 + kl) * 16;
    const size_t gbase = (size_t)kl * q.ustride;
    cd Tg[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c) Tg[p][c] = g[p * 4 + c];
    double ff = 0.0;
    if (q.want_f) {  // f_after_v (trace only): Tr W + Re Σ conj(UW) ∘ (A U − 2 G), column sc
      cd U[4][4], gs[4], us[4], ws[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
#pragma unroll
        for (int c = 0; c < 4; ++c) U[p][c] = ucache[kl * 16 + p * 4 + c];
        gs[p] = cmk((double)q.Gr[gbase + p * q.rstride + sc], (double)q.Gi[gbase + p * q.rstride + sc]);
        us[p] = ucache[kl * 16 + p * 4 + sc];
        ws[p] = wcache[kl * 16 + p * 4 + sc];
      }
      double term = wcache[kl * 16 + sc * 4 + sc].r;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        cd x = cscale(us[a], q.sigma2), y = cmk(0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          cfma(x, Tg[a][b], us[b]);
          cfma(y, U[a][b], ws[b]);
        }
        const cd z = cmk(x.r - 2.0 * gs[a].r, x.i - 2.0 * gs[a].i);
        term += y.r * z.r + y.i * z.i;  // Re(conj(uw) z)
      }
      ff = q.alpha[kl] * (qsum(term) - lndetw[kl]);
    }
    cd L[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) L[a][b] = Tg[a][b];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      L[a][a].r += q.sigma2;
      L[a][a].i = 0.0;
    }
    double ia[4], pa[4], ic[4];
    const bool okA = chol4_inv(L, ia);
#pragma unroll
    for (int j = 0; j < 4; ++j) pa[j] = L[j][j].r;
    asm volatile("bar.sync 2, 64;\n" ::: "memory");
    const double* scr = wscr + (size_t)kl * kWsrScratch;
#pragma unroll
    for (int j = 0; j < 4; ++j) ic[j] = scr[32 + j];
    const bool ok = okA && scr[36] != 0.0;
    double rr = 0.0;
    int st = 0;
    if (ok) {
      const double r = lndet_diff4i(pa, ic);
      rr = q.alpha[kl] * (r > 0.0 ? r : 0.0);
    } else {
      st = AMMMSE_STATUS_NONFINITE;
    }
    if (act && sc == 0) {
      rate[kl] = rr;
      fv[kl] = ff;
      ust2[kl] = st;
    }
  }
}

struct K1Out4 {  // destinations of K1 (own users unless noted)
  cd* ucache;        // 16 cd per user
  cd* wcache;        // 16 cd per user
  double* lndetw;
  double* fu;
  double* fw;
  double* ust;
  float2* Mall;      // fp32, 16 per GLOBAL user: M = P U^H = α U W U^H
  float2* Down;      // fp32, 16 per own user
  double* scratch;   // kScratch doubles per own user
};

// K1(t+1) in the weighted stage, warp 2: the weight half (W = I + Y^H Y), then — after
// the named barrier 1 (64 threads, once per pass of 8 users) it shares with
// k1_recv_users — the statistics half of the combine (ill-conditioning test,
// ln det W, f_after_w) while warp 1 forms P and D.
static __device__ __noinline__ void k1_weight_users(QuadArgs q, K1Out4 o) {
  const int lane = threadIdx.x & 31, ul = lane >> 2, sc = lane & 3;
  for (int kl0 = 0; kl0 < q.KL; kl0 += 8) {
    const bool act = kl0 + ul < q.KL;
    const int kl = act ? kl0 + ul : 0;
    cd Tg[4][4], G[4][4], gs[4];
    const cd* g = q.gram + (size_t)(q.k0 + kl) * 16;
    const size_t gbase = (size_t)kl * q.ustride;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        Tg[p][c] = g[p * 4 + c];
        G[p][c] = cmk((double)q.Gr[gbase + p * q.rstride + c], (double)q.Gi[gbase + p * q.rstride + c]);
      }
#pragma unroll
    for (int p = 0; p < 4; ++p)
      gs[p] = cmk((double)q.Gr[gbase + p * q.rstride + sc], (double)q.Gi[gbase + p * q.rstride + sc]);
    double* scr = o.scratch + (size_t)kl * kScratch;
    cd* wcol = o.wcache + (size_t)kl * 16;
    double ipivc[4];
    int pd;
    k1w_quad(Tg, G, gs, q.sigma2, sc, reinterpret_cast<cd*>(scr), wcol, ipivc, pd);
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
    // warp 1 has left T (column sc), ‖T‖², the pivots of A and its status in the scratch
    const cd* tsc = reinterpret_cast<const cd*>(scr + 64);
    cd tcol[4], wcs[4];
    double piva[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      tcol[p] = tsc[p * 4 + sc];
      wcs[p] = wcol[p * 4 + sc];
      piva[p] = scr[97 + p];
    }
    int st = (int)scr[101];
    double fw_, lnw;
    k1c_stat(tcol, scr[96], piva, wcs, ipivc, pd, q.alpha[kl], true, q.want_f != 0, sc, fw_, lnw, st);
    if (act && sc == 0) {
      o.lndetw[kl] = lnw;
      o.fw[kl] = fw_;
      o.ust[kl] = st;
    }
  }
}

// K1(t+1), warp 1: the receiver half, then P = α U W and D = −P T.  In the weighted
// stage the statistics half runs on warp 2 (k1_weight_users); otherwise (W = I) here.
// wprev / lndet_wprev: the previous iteration's W bank (f_after_u, solvers.py:447).
static __device__ __noinline__ void k1_recv_users(QuadArgs q, K1Out4 o, const cd* wprev, const double* lndet_wprev,
                                           bool weighted) {
  const int lane = threadIdx.x & 31, ul = lane >> 2, sc = lane & 3;
  for (int kl0 = 0; kl0 < q.KL; kl0 += 8) {
    const bool act = kl0 + ul < q.KL;
    const int kl = act ? kl0 + ul : 0;
    cd Tg[4][4], gs[4], Wprow[4];
    const cd* g = q.gram + (size_t)(q.k0 + kl) * 16;
    const size_t gbase = (size_t)kl * q.ustride;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
      for (int c = 0; c <= p; ++c) Tg[p][c] = g[p * 4 + c];
      gs[p] = cmk((double)q.Gr[gbase + p * q.rstride + sc], (double)q.Gi[gbase + p * q.rstride + sc]);
      Wprow[p] = wprev[kl * 16 + sc * 4 + p];
    }
    double* scr = o.scratch + (size_t)kl * kScratch;
    cd* ucol = o.ucache + (size_t)kl * 16;
    cd* wcol = o.wcache + (size_t)kl * 16;
    cd Ufull[4][4], us[4], tcol[4];
    double fu_, nT, piva[4];
    int st;
    k1u_quad(Tg, gs, q.sigma2, q.alpha[kl], Wprow, lndet_wprev[kl], sc, q.want_f != 0, ucol, Ufull, us, tcol,
             fu_, nT, piva, st);
    cd wcs[4];
    if (weighted) {
      cd* tsc = reinterpret_cast<cd*>(scr + 64);
#pragma unroll
      for (int p = 0; p < 4; ++p) tsc[p * 4 + sc] = tcol[p];
      if (sc == 0) {
        scr[96] = nT;
#pragma unroll
        for (int j = 0; j < 4; ++j) scr[97 + j] = piva[j];
        scr[101] = (double)st;
      }
      asm volatile("bar.sync 1, 64;\n" ::: "memory");
#pragma unroll
      for (int p = 0; p < 4; ++p) wcs[p] = wcol[p * 4 + sc];
    } else {
#pragma unroll
      for (int p = 0; p < 4; ++p) wcs[p] = cmk(p == sc ? 1.0 : 0.0);
      const double one[4] = {1.0, 1.0, 1.0, 1.0};
      double fw_, lnw;
      k1c_stat(tcol, nT, piva, wcs, one, 1, q.alpha[kl], false, q.want_f != 0, sc, fw_, lnw, st);
      if (act && sc == 0) {
        o.lndetw[kl] = lnw;
        o.fw[kl] = fw_;
        o.ust[kl] = st;
      }
    }
    cd pcol[4], dcol[4];
    const cd* pscr_c = reinterpret_cast<const cd*>(scr + 32);
    k1c_pd(Ufull, us, tcol, wcs, q.alpha[kl], weighted, sc, reinterpret_cast<cd*>(scr + 32), pcol, dcol);
    if (act) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {  // row p, column sc
        const int ig = ((q.k0 + kl) * 4 + p) * 4 + sc, il = (kl * 4 + p) * 4 + sc;
        // column sc of M = P U^H: M[p][sc] = Σ_c P[p][c] conj(U[sc][c]) (P full in the scratch)
        cd mm = cmk(0.0);
#pragma unroll
        for (int c = 0; c < 4; ++c) mm = cadd(mm, cmulcb(pscr_c[p * 4 + c], ucol[sc * 4 + c]));
        o.Mall[ig] = make_float2((float)mm.r, (float)mm.i);
        o.Down[il] = make_float2((float)dcol[p].r, (float)dcol[p].i);
        if (!weighted) wcol[p * 4 + sc] = wcs[p];
      }
      if (sc == 0) o.fu[kl] = fu_;
    }
  }
}

}  // namespace quad
}  // namespace ammmse
