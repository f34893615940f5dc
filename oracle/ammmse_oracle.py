"""CPU ORACLE for the A-MMMSE hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
/ ``--impl reference`` leg may import this module, and only as the checker or
the timed CPU reference arm; the product path (paper_2510_20507_b200) never
routes through it.

What it is: a numpy (complex128, fp64) restatement of the reference
``wsrbeam.run_ammmse`` (pkg/src/wsrbeam/solvers.py:540-550 →
``_run_bcd`` :415-518 with exact=False, use_extrapolation=True,
start_weighted=False) and of every block it calls.  Each function cites the
reference lines it follows.  The per-user Python loops of the reference are
written as batched numpy contractions over the user axis; the arithmetic is
the same (same matrices, same Cholesky / LU solves, same fp64), only the
summation order inside a few contractions differs.

Pinning: tests/test_oracle_golden.py checks this restatement against golden
vectors produced by running the unmodified reference
(tests/golden/make_golden.py, generated in the build container where
/root/reference is importable).  Third-party arithmetic: numpy 2.3 /
scipy 1.18 (OpenBLAS zgemm, LAPACK zpotrf/zpotrs/zgesv/zheevd), the same
libraries the reference calls (pkg/pyproject.toml:10-13 lower-bounds only).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

STATUS_OK = 0
STATUS_ILL_CONDITIONED = 1
STATUS_UNSTABLE = 2
STATUS_NONFINITE = 3

COND_LIMIT = 1e12          # solvers.py:71
LN2 = math.log(2.0)        # objective.py:21

STEP_TABLE = {             # solvers.py:61-69 (omega, gamma)
    -10.0: (0.6, 0.4), -5.0: (0.6, 0.4), 0.0: (0.6, 0.4), 5.0: (0.6, 0.4),
    10.0: (0.8, 0.05), 15.0: (0.8, 0.005), 20.0: (0.8, 0.003),
}


class _Fail(Exception):
    def __init__(self, status):
        super().__init__(status)
        self.status = status


def _herm(a):
    """hermitianize, linalg.py:12-14"""
    return 0.5 * (a + np.conj(np.swapaxes(a, -1, -2)))


def _lndet(a):
    """lndet_hpd, linalg.py:27-30 (batched over leading axes)"""
    try:
        c = np.linalg.cholesky(a)
    except np.linalg.LinAlgError:
        raise _Fail(STATUS_NONFINITE)
    return 2.0 * np.sum(np.log(np.real(np.diagonal(c, axis1=-2, axis2=-1))), axis=-1)


def table_step(snr_db):
    """default_step_parameters, solvers.py:185-193"""
    key = min(STEP_TABLE, key=lambda s: (abs(s - float(snr_db)), -s))
    return STEP_TABLE[key]


def bounds(H, alpha, p_max, s2):
    """compute_bounds, objective.py:216-240 -> (kappa, l_v, gamma_safe, ek_floor, alpha_bar)"""
    K, N, M = H.shape
    kappa = 0.0
    for k in range(K):
        hk = H[k]
        g = hk @ hk.conj().T if N <= M else hk.conj().T @ hk
        kappa = max(kappa, float(np.linalg.eigvalsh(_herm(g))[-1]))
    abar = float(np.max(alpha))
    l_v = 2.0 * abar * K * kappa / s2
    return kappa, l_v, 1.0 / l_v, s2 / (p_max * kappa + s2), abar


def receivers(H, V, s2):
    """update_receivers, solvers.py:210-225: U_k = (H_k Q H_k^H + s2 I)^-1 H_k V_k,
    Q = sum_j V_j V_j^H, HPD solve by Cholesky (linalg.py:17-24)."""
    K, N, _ = H.shape
    Q = np.einsum("jmd,jnd->mn", V, V.conj())
    A = _herm(H @ Q @ np.conj(np.swapaxes(H, 1, 2))) + s2 * np.eye(N)
    B = H @ V                                           # (K, N, d): H_k V_k
    U = np.empty_like(B)
    for k in range(K):
        U[k] = sla.cho_solve(sla.cho_factor(A[k], lower=True), B[k])
    return U


def weight_update(H, U, V):
    """update_weight_matrices, solvers.py:228-254"""
    K, _, d = V.shape
    eye = np.eye(d)
    T = eye - np.conj(np.swapaxes(U, 1, 2)) @ (H @ V)   # I - U_k^H H_k V_k
    cond = np.linalg.cond(T)
    if not np.all(np.isfinite(cond)) or np.any(cond > COND_LIMIT):
        raise _Fail(STATUS_ILL_CONDITIONED)
    W = _herm(np.linalg.solve(T, np.broadcast_to(eye, T.shape)))
    if np.any(np.linalg.eigvalsh(W)[:, 0] <= 0.0):
        raise _Fail(STATUS_ILL_CONDITIONED)
    return W


def cross_blocks(H, V):
    """C[k, j] = H_k V_j, the per-pair terms of user_rate / mse_matrix (K, K, N, d)."""
    return np.einsum("knm,jmd->kjnd", H, V)


def objective(H, U, W, V, alpha, s2):
    """wmmse_objective + mse_matrix, objective.py:84-105, :151-169"""
    K, N, d = U.shape
    C = cross_blocks(H, V)
    R = np.einsum("knd,kjne->kjde", U.conj(), C)            # U_k^H H_k V_j
    idx = np.arange(K)
    T = np.eye(d) - R[idx, idx]                               # I - U_k^H H_k V_k
    E = T @ np.conj(np.swapaxes(T, 1, 2)) + s2 * (np.conj(np.swapaxes(U, 1, 2)) @ U)
    off = R @ np.conj(np.swapaxes(R, 2, 3))                   # (K, K, d, d)
    off[idx, idx] = 0.0
    E = _herm(E + off.sum(axis=1))
    try:
        lw = _lndet(W)
    except _Fail:
        raise _Fail(STATUS_ILL_CONDITIONED)                   # ObjectiveDomainError
    tr = np.real(np.einsum("kab,kba->k", W, E))
    return float(np.sum(alpha * (tr - lw)))


def wsr(H, V, alpha, s2):
    """weighted_sum_rate + user_rate, objective.py:108-148 -> (wsr_nats, total_power)"""
    K, N, _ = H.shape
    C = cross_blocks(H, V)
    S = C @ np.conj(np.swapaxes(C, 2, 3))                     # (K, K, N, N)
    idx = np.arange(K)
    own = S[idx, idx]
    S[idx, idx] = 0.0
    cov = _herm(s2 * np.eye(N) + S.sum(axis=1))
    rates = _lndet(_herm(cov + own)) - _lndet(cov)
    rates = np.maximum(rates, 0.0)
    total = 0.0
    for k in range(K):                                        # fixed user order (:144-146)
        total += float(alpha[k]) * float(rates[k])
    return total, float(np.real(np.vdot(V, V)))


def project(X, p_max):
    """project_sum_power, solvers.py:257-263"""
    power = float(np.real(np.vdot(X, X)))
    if power <= p_max:
        return X
    return X * math.sqrt(p_max / power)


def pgd_step(Vhat, U, W, H, alpha, gamma, p_max):
    """pgd_precoder_step, solvers.py:358-377 with weighted_gram /
    gradient_common_factor, objective.py:172-193"""
    HU = np.conj(np.swapaxes(H, 1, 2)) @ U                    # H_k^H U_k (K, M, d)
    common = 2.0 * _herm(np.einsum("k,kmd,kde,kne->mn", alpha, HU, W, HU.conj()))
    grad = common @ Vhat - 2.0 * alpha[:, None, None] * (HU @ W)
    return project(Vhat - gamma * grad, p_max)


def stationarity(H, V, alpha, s2, p_max, gamma_safe, weighted):
    """_stationarity_residual, solvers.py:400-412"""
    K, _, d = V.shape
    U = receivers(H, V, s2)
    W = weight_update(H, U, V) if weighted else np.broadcast_to(np.eye(d), (K, d, d)).copy()
    stepped = pgd_step(V, U, W, H, alpha, gamma_safe, p_max)
    nv = math.sqrt(max(float(np.real(np.vdot(V, V))), 0.0))
    return float(np.linalg.norm(V - stepped)) / max(1.0, nv)


def _rel(new, old):
    """_rel_change, solvers.py:393-397"""
    den = abs(old)
    return math.inf if den == 0.0 else abs(new - old) / den


def solve(H, s2, alpha, p_max, V0, gamma, omega, eps1=0.1, eps2=1e-3, max_iters=1000,
          latch_stage=True, snr_db=10.0):
    """_run_bcd for A-MMMSE, solvers.py:415-518.

    gamma: float, "safe" or None (table by snr_db); omega: float or None.
    Returns a dict with the SolveResult fields plus status / trace / V."""
    H = np.asarray(H, dtype=np.complex128)
    V = np.asarray(V0, dtype=np.complex128).copy()
    alpha = np.asarray(alpha, dtype=np.float64)
    K, N, M = H.shape
    d = V.shape[2]
    bnd = bounds(H, alpha, p_max, s2)
    om_d, g_d = table_step(snr_db)
    om = om_d if omega is None else float(omega)
    if gamma is None:
        g = g_d
    elif gamma == "safe":
        g = bnd[2]
    else:
        g = float(gamma)
    eye_w = np.broadcast_to(np.eye(d), (K, d, d)).copy()
    v_cur, v_old, w_prev = V, V, eye_w
    latched, switch_it = False, None
    hist, trace = [], []
    running_max, streak, converged = -math.inf, 0, False
    status = STATUS_OK
    last_weighted = False
    try:
        for t in range(1, max_iters + 1):
            vhat = v_cur + om * (v_cur - v_old) if (t >= 2 and om > 0.0) else v_cur
            U = receivers(H, vhat, s2)
            f_u = objective(H, U, w_prev, vhat, alpha, s2)
            if latched:
                weighted = True
            else:
                rs = math.inf if len(hist) < 2 else _rel(hist[-1], hist[-2])
                weighted = rs <= eps1
                if weighted:
                    if latch_stage:
                        latched = True
                    if switch_it is None:
                        switch_it = t
            W = weight_update(H, U, vhat) if weighted else eye_w
            f_w = objective(H, U, W, vhat, alpha, s2)
            v_new = pgd_step(vhat, U, W, H, alpha, g, p_max)
            f_v = objective(H, U, W, v_new, alpha, s2)
            w_nats, power = wsr(H, v_new, alpha, s2)
            rel = math.inf if t == 1 else _rel(w_nats, hist[-1])
            hist.append(w_nats)
            trace.append((t, w_nats / LN2, f_v, power, 1.0 if weighted else 0.0, f_u, f_w, f_v, rel))
            last_weighted = weighted
            running_max = max(running_max, w_nats)
            streak = streak + 1 if w_nats < 0.5 * running_max else 0
            if streak >= 5:
                raise _Fail(STATUS_UNSTABLE)
            v_old, v_cur, w_prev = v_cur, v_new, W
            if weighted and rel <= eps2:
                converged = True
                break
        residual = stationarity(H, v_cur, alpha, s2, p_max, bnd[2], latched or last_weighted)
    except _Fail as f:
        status = f.status
        residual = math.nan
    tr = np.asarray(trace, dtype=np.float64).reshape(-1, 9)
    return dict(
        final_precoders=v_cur, wsr_bits=float(tr[-1, 1]) if len(tr) else math.nan,
        iterations=len(trace), converged=converged, stationarity_residual=residual,
        switch_iteration=-1 if switch_it is None else switch_it, status=status,
        gamma_used=g, omega_used=om, trace=tr, bounds=bnd)


def solve_batch(H, s2, alpha, p_max, V0, gamma, omega, eps1=0.1, eps2=1e-3, max_iters=1000,
                latch_stage=True, snr_db=10.0, record_trace=False):
    """Loop :func:`solve` over a batch; returns SoA numpy arrays."""
    B = H.shape[0]
    s2 = np.broadcast_to(np.asarray(s2, dtype=np.float64), (B,))
    pm = np.broadcast_to(np.asarray(p_max, dtype=np.float64), (B,))
    al = np.broadcast_to(np.asarray(alpha, dtype=np.float64), (B, H.shape[1]))
    outs = [solve(H[b], float(s2[b]), al[b], float(pm[b]), V0[b], gamma, omega, eps1, eps2,
                  max_iters, latch_stage, snr_db) for b in range(B)]
    res = dict(
        final_precoders=np.stack([o["final_precoders"] for o in outs]),
        wsr_bits=np.array([o["wsr_bits"] for o in outs]),
        iterations=np.array([o["iterations"] for o in outs], dtype=np.int32),
        converged=np.array([o["converged"] for o in outs], dtype=bool),
        stationarity_residual=np.array([o["stationarity_residual"] for o in outs]),
        switch_iteration=np.array([o["switch_iteration"] for o in outs], dtype=np.int32),
        status=np.array([o["status"] for o in outs], dtype=np.int32),
        gamma_used=np.array([o["gamma_used"] for o in outs]),
    )
    if record_trace:
        T = max(o["trace"].shape[0] for o in outs)
        tr = np.full((B, max(T, 1), 9), np.nan)
        for b, o in enumerate(outs):
            tr[b, : o["trace"].shape[0]] = o["trace"]
        res["trace"] = tr
    return res
