"""Verification oracles at batch scale on the GPU.

Restates the reference's acceptance oracles (pkg/src/wsrbeam/verify.py) for
batches of solves on the device, in complex128 torch arithmetic that does not
share code with the solve kernels (an independent route, as the reference's
docstring asks of an oracle):

  * :class:`OracleReport`        verify.py:25-44 (same fields and consistency rule)
  * :func:`check_lemma_bounds`   verify.py:147-207, reference signature (one
                                 SolveResult with recorded iterates)
  * :func:`lemma_bound_scan`     the same four bound families over a whole batch
                                 of recorded iterates (BatchResult.iterates),
                                 one device pass
  * :func:`gradient_fd_report`   harness.py:397-432 (``_gradient_fd_report``):
                                 central finite differences of the WMMSE
                                 objective (verify.py:54-76) against the
                                 closed-form gradient (objective.py:196-213),
                                 all 4 K M d perturbed objectives as one batch
  * :class:`BoundsReport` / :func:`compute_bounds`  objective.py:40-66, :216-240,
                                 through the engine's batched ``ammmse_bounds``
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

FD_COORD_BUDGET = 1024  # harness.py:60 (_FD_COORD_BUDGET)
FAMILIES = ("mse_eigenvalue_floor", "receiver_norm", "weight_norm", "gradient_factor_norm")


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class OracleReport:
    """Outcome of one oracle sweep (ref verify.py:25-44)."""

    name: str
    max_abs_error: float
    max_rel_error: float
    instances: int
    passed: bool
    tolerance: float
    detail: str = ""

    def __post_init__(self) -> None:
        if self.passed != (self.max_rel_error <= self.tolerance):
            raise ConfigError("OracleReport.passed inconsistent with its errors")


@dataclass(frozen=True)
class BoundsReport:
    """Spectral quantities controlling smoothness and safe step sizes
    (ref objective.py:40-66, same fields and checks)."""

    kappa: float
    l_v: float
    gamma_safe: float
    ek_floor: float
    alpha_bar: float

    def __post_init__(self) -> None:
        for name in ("kappa", "l_v", "gamma_safe", "ek_floor", "alpha_bar"):
            v = getattr(self, name)
            if not (math.isfinite(v) and v > 0):
                raise ConfigError(f"BoundsReport.{name} must be a positive real, got {v!r}")
        if abs(self.gamma_safe * self.l_v - 1.0) > 1e-12:
            raise ConfigError("gamma_safe must equal 1 / l_v")
        if not (0.0 < self.ek_floor <= 1.0):
            raise ConfigError(f"ek_floor must lie in (0, 1], got {self.ek_floor!r}")


def compute_bounds(channels, weights, p_max: float, noise_power: float, device=None) -> BoundsReport:
    """compute_bounds (ref objective.py:216-240) of one realization through the
    device kernel ``ammmse_bounds`` (AmmmseEngine.bounds)."""
    torch = _torch()
    from .solvers import engine

    eng = engine(device)
    H = np.asarray(getattr(channels, "channels", channels))
    dt = torch.complex64 if H.dtype == np.complex64 else torch.complex128
    dev = eng.device
    K = H.shape[0]
    out = eng.bounds(torch.from_numpy(np.ascontiguousarray(H[None])).to(dev, dt),
                     torch.from_numpy(np.asarray(weights, dtype=np.float64).reshape(1, K)).to(dev),
                     torch.full((1,), float(p_max), dtype=torch.float64, device=dev),
                     torch.full((1,), float(noise_power), dtype=torch.float64, device=dev))
    b = out[0].cpu().numpy()
    return BoundsReport(float(b[0]), float(b[1]), float(b[2]), float(b[3]), float(b[4]))


def _default_device():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else \
        torch.device("cpu")


def _herm(a):
    return 0.5 * (a + a.conj().transpose(-1, -2))


def lemma_bound_scan(H, noise_power, weights, bounds, U, W, V, iterations, t_chunk: int = 64):
    """Worst excess of each bound family over every recorded iterate of every
    realization (ref verify.py:147-207, the four families and slacks):
        λ_min(E_k) >= ek_floor - 1e-9          ‖U_k‖_F² <= d / σ² + 1e-9
        ‖W_k‖_F² <= d / ek_floor² + 1e-6       ‖herm(2 Σ α_k H_k^H U_k W_k U_k^H H_k)‖_2 <= l_v + 1e-6
    H (B, K, N, M); noise_power (B,); weights (B, K); bounds (B, 5) rows of
    [kappa, l_v, gamma_safe, ek_floor, alpha_bar]; U (B, T, K, N, d),
    W (B, T, K, d, d), V (B, T, K, M, d); iterations (B,): iterates t <
    iterations[b] are scanned.  Torch tensors (their device) or numpy arrays (the
    current CUDA device, or the CPU without one: verification, not the solve).
    Returns (worst (B, 4) float64 excess, limits (B, 4)), numpy; excess > 0
    means a violated bound."""
    torch = _torch()
    dev = U.device if torch.is_tensor(U) else _default_device()
    c128 = lambda x: (x if torch.is_tensor(x) else torch.from_numpy(np.asarray(x))).to(
        dev, torch.complex128)
    f64 = lambda x: (x if torch.is_tensor(x) else torch.from_numpy(np.asarray(x))).to(
        dev, torch.float64)
    H, U, W, V = c128(H), c128(U), c128(W), c128(V)
    s2, alpha, bnd = f64(noise_power), f64(weights), f64(bounds)
    iters = torch.as_tensor(np.asarray(iterations.cpu() if torch.is_tensor(iterations) else iterations),
                            device=dev)
    B, T, K, N, d = U.shape
    M = H.shape[3]
    lim = torch.stack([bnd[:, 3] - 1e-9, d / s2 + 1e-9, d / bnd[:, 3] ** 2 + 1e-6, bnd[:, 1] + 1e-6],
                      dim=1)  # (B, 4)
    worst = torch.full((B, 4), -math.inf, dtype=torch.float64, device=dev)
    eye = torch.eye(d, dtype=torch.complex128, device=dev)
    for t0 in range(0, T, t_chunk):
        t1 = min(T, t0 + t_chunk)
        valid = (torch.arange(t0, t1, device=dev)[None, :] < iters[:, None])  # (B, t)
        # iterates past a realization's last iteration are unwritten (NaN): zero them
        keep = valid[:, :, None, None, None]
        u = torch.where(keep, U[:, t0:t1], torch.zeros((), dtype=U.dtype, device=dev))
        w = torch.where(keep, W[:, t0:t1], torch.zeros((), dtype=W.dtype, device=dev))
        v = torch.where(keep, V[:, t0:t1], torch.zeros((), dtype=V.dtype, device=dev))
        # R[k, j] = U_k^H H_k V_j  (B, t, K, K, d, d)
        hv = torch.einsum("bknm,btjmd->btkjnd", H, v)
        R = torch.einsum("btkna,btkjnd->btkjad", u.conj(), hv)
        Rkk = torch.diagonal(R, dim1=2, dim2=3).permute(0, 1, 4, 2, 3)  # (B, t, K, d, d)
        Tm = eye - Rkk
        E = Tm @ Tm.conj().transpose(-1, -2)
        E = E + s2[:, None, None, None, None] * (u.conj().transpose(-1, -2) @ u)
        RR = R @ R.conj().transpose(-1, -2)  # (B, t, K, K, d, d)
        off = RR.sum(dim=3) - torch.diagonal(RR, dim1=2, dim2=3).permute(0, 1, 4, 2, 3)
        E = _herm(E + off)
        lam_min = torch.linalg.eigvalsh(E)[..., 0]                      # (B, t, K)
        un = (u.abs() ** 2).sum(dim=(-1, -2))                            # (B, t, K)
        wn = (w.abs() ** 2).sum(dim=(-1, -2))
        hu = torch.einsum("bknm,btkna->btkma", H.conj(), u)              # H_k^H U_k (B, t, K, M, d)
        F = 2.0 * torch.einsum("bk,btkma,btkac,btknc->btmn", alpha.to(torch.complex128), hu, w,
                               hu.conj())
        fn = torch.linalg.eigvalsh(_herm(F)).abs().amax(dim=-1)          # (B, t)
        ex = torch.stack([
            (lim[:, 0, None, None] - lam_min).amax(dim=2),
            (un - lim[:, 1, None, None]).amax(dim=2),
            (wn - lim[:, 2, None, None]).amax(dim=2),
            fn - lim[:, 3, None]], dim=2)                                # (B, t, 4)
        ex = torch.where(valid[..., None], ex, torch.full_like(ex, -math.inf))
        worst = torch.maximum(worst, ex.amax(dim=1))
    return worst.cpu().numpy(), lim.cpu().numpy()


def lemma_report(worst, limits, instances: int, name: str = "lemma_bounds") -> OracleReport:
    """OracleReport of scanned excesses (ref verify.py:196-207); several rows
    (realizations) merge as harness._merge_lemma_reports does (harness.py:434-445):
    max errors over the realizations, details = sorted distinct per-realization
    "violated: ..." strings joined by "; "."""
    worst = np.atleast_2d(worst)
    limits = np.atleast_2d(limits)
    max_abs, max_rel, details = 0.0, 0.0, set()
    for w, lim in zip(worst, limits):
        viol = [FAMILIES[j] for j in range(4) if w[j] > 0.0]
        max_abs = max(max_abs, max(0.0, float(np.max(w))))
        max_rel = max([max_rel] + [float(w[j] / abs(lim[j])) for j in range(4) if w[j] > 0.0])
        if viol:
            details.add("violated: " + ", ".join(sorted(viol)))
    return OracleReport(name=name, max_abs_error=max_abs, max_rel_error=max_rel, instances=instances,
                        passed=not details, tolerance=0.0, detail="; ".join(sorted(details)))


def check_lemma_bounds(channels, trace, bounds, weights=None) -> OracleReport:
    """Scan every recorded block iterate of one solve against the convergence
    bounds (ref verify.py:147-207 signature).  ``trace`` is a SolveResult run
    with ``record_iterates=True``; ``bounds`` a BoundsReport."""
    if trace.iterates is None or len(trace.iterates) == 0:
        raise ConfigError("solve result carries no recorded iterates; run with record_iterates=True")
    if channels.noise_power is None:
        raise ConfigError("channels carry no noise power")
    H = channels.channels
    K = H.shape[0]
    alpha = np.ones(K) if weights is None else np.asarray(weights, dtype=np.float64)
    U = np.stack([it.receivers.receivers for it in trace.iterates])[None]
    W = np.stack([it.weight_matrices.weight_matrices for it in trace.iterates])[None]
    V = np.stack([it.precoders.precoders for it in trace.iterates])[None]
    b = np.array([[bounds.kappa, bounds.l_v, bounds.gamma_safe, bounds.ek_floor, bounds.alpha_bar]])
    worst, lim = lemma_bound_scan(H[None], np.array([channels.noise_power]), alpha[None], b, U, W, V,
                                  np.array([U.shape[1]]))
    return lemma_report(worst, lim, instances=len(trace.iterates))


# --------------------------------------------------------------------------- FD gradient
def _receivers(H, V, s2):
    """MMSE receivers (ref solvers.py:210-225), batched over a leading axis."""
    torch = _torch()
    Q = torch.einsum("...jmd,...jnd->...mn", V, V.conj())
    A = _herm(H @ Q @ H.conj().transpose(-1, -2))
    A = A + s2 * torch.eye(H.shape[-2], dtype=A.dtype, device=A.device)
    return torch.linalg.solve(A, H @ V)


def _weights(H, U, V):
    """update_weight_matrices (ref solvers.py:228-254) without the raise paths."""
    torch = _torch()
    d = V.shape[-1]
    eye = torch.eye(d, dtype=V.dtype, device=V.device)
    Tm = eye - U.conj().transpose(-1, -2) @ (H @ V)
    return _herm(torch.linalg.solve(Tm, eye.expand_as(Tm)))


def _objective(H, U, W, V, alpha, s2):
    """wmmse_objective (ref objective.py:151-169) of a batch of precoder sets
    V (P, K, M, d) at fixed U, W: f = Σ α_k (Tr(W_k E_k) − ln det W_k)."""
    torch = _torch()
    R = torch.einsum("kna,knm,pjmd->pkjad", U.conj(), H, V)  # U_k^H H_k V_j
    K, d = U.shape[0], U.shape[2]
    idx = torch.arange(K, device=V.device)
    eye = torch.eye(d, dtype=V.dtype, device=V.device)
    Tm = eye - R[:, idx, idx]
    E = Tm @ Tm.conj().transpose(-1, -2) + s2 * (U.conj().transpose(-1, -2) @ U)
    RR = R @ R.conj().transpose(-1, -2)
    E = _herm(E + RR.sum(dim=2) - RR[:, idx, idx])
    lndet = 2.0 * torch.log(torch.linalg.cholesky(W).diagonal(dim1=-2, dim2=-1).real).sum(-1)
    tr = torch.einsum("kab,pkba->pk", W, E).real
    return ((tr - lndet) * alpha).sum(-1)


def gradient_fd_report(config, device=None, h: float = 1e-5) -> OracleReport | None:
    """Finite-difference check of the closed-form gradient on the experiment's
    base system (ref harness.py:397-432): channels / noise power / weights / V0
    of ``config``, receivers and weights at V0, every real and imaginary
    coordinate perturbed by ±h (verify.py:54-76), all 4 K M d objectives
    evaluated as one device batch.  None above the coordinate budget."""
    torch = _torch()
    from .model import compute_noise_power, generate_channels, init_precoders, project_sum_power

    if config.K * config.M * config.d > FD_COORD_BUDGET:
        return None
    dev = _default_device() if device is None else torch.device(device)
    ch = generate_channels(config)
    s2 = compute_noise_power(ch, config.snr_db, config)
    H = torch.from_numpy(ch.channels.astype(np.complex128)).to(dev)
    V0 = torch.from_numpy(init_precoders(config, project_sum_power).precoders.astype(np.complex128)).to(dev)
    alpha = torch.from_numpy(np.asarray(config.weight_vector, dtype=np.float64)).to(dev)
    U = _receivers(H, V0, s2)
    W = _weights(H, U, V0)
    n = V0.numel()
    steps = torch.zeros((2 * n,) + V0.shape, dtype=V0.dtype, device=dev)
    flat = steps.view(2 * n, n)
    ar = torch.arange(n, device=dev)
    flat[ar, ar] = h
    flat[n + ar, ar] = 1j * h
    Vp = torch.cat([V0 + steps, V0 - steps])
    f = _objective(H, U, W, Vp, alpha, s2)
    d_re = (f[:n] - f[2 * n:3 * n]) / (2.0 * h)
    d_im = (f[n:2 * n] - f[3 * n:]) / (2.0 * h)
    fd = (d_re + 1j * d_im).view(V0.shape)
    hu = H.conj().transpose(-1, -2) @ U                                   # H_k^H U_k
    common = 2.0 * _herm(torch.einsum("k,kma,kab,knb->mn", alpha.to(V0.dtype), hu, W, hu.conj()))
    grad = common @ V0 - 2.0 * alpha[:, None, None] * (hu @ W)          # gradient_v, all k
    num = torch.linalg.norm((grad - fd).reshape(config.K, -1), dim=1)
    den = torch.clamp(torch.linalg.norm(grad.reshape(config.K, -1), dim=1), min=1e-12)
    worst = float((num / den).max())
    tol = 1e-6
    return OracleReport(name="gradient_finite_difference", max_abs_error=worst, max_rel_error=worst,
                        instances=config.K, passed=worst <= tol, tolerance=tol)
