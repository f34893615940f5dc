"""Seeded batch inputs for the BASELINE.json workloads.

Realization r of a batch uses channel_seed = init_seed = seed0 + r, the
reference harness's rule (pkg/src/wsrbeam/harness.py:474-480).  Channels and
V0 come from the reference generators restated in :mod:`.model`
(generate_channels, init_precoders; bit-identical Philox streams), so the
GPU engine and the CPU oracle see identical inputs.  Extra draws the
reference has no generator for (BASELINE configs 2-5):

  * user priorities alpha_{r,k} ~ U[0.5, 1.5] from Philox [r, ALPHA_STREAM];
  * Kronecker channels (config 4): H_k = sqrt(beta_k) G_k R^{1/2}, G_k from
    generate_channels, R_ij = 0.5^{|i-j|}, R^{1/2} the symmetric PSD root by
    eigh, beta_k = 10^{U[-2, 0]} from Philox [r, BETA_STREAM].

complex64 workloads are generated in complex128 and rounded once; V0 is
rounded after its projection onto the power ball (both sides then start from
the same complex64 V0).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor

from dataclasses import dataclass

import numpy as np

from .model import ALPHA_STREAM, BETA_STREAM, CHANNEL_STREAM, INIT_STREAM, philox


@dataclass
class Batch:
    """Host arrays of one batched solve."""

    channels: np.ndarray        # (B, K, N, M) complex
    noise_power: np.ndarray     # (B,) float64
    p_max: np.ndarray           # (B,) float64
    weights: np.ndarray         # (B, K) float64
    init_precoders: np.ndarray  # (B, K, M, d) complex
    gamma: np.ndarray | None = None  # (B,) per-realization step (optional)
    omega: np.ndarray | None = None  # (B,) per-realization extrapolation (optional)

    @property
    def B(self) -> int:
        return self.channels.shape[0]

    def subset(self, idx) -> "Batch":
        sel = lambda a: None if a is None else a[idx]
        return Batch(self.channels[idx], self.noise_power[idx], self.p_max[idx], self.weights[idx],
                     self.init_precoders[idx], sel(self.gamma), sel(self.omega))

    @staticmethod
    def concat(parts) -> "Batch":
        cat = lambda f: np.concatenate([getattr(p, f) for p in parts])
        return Batch(cat("channels"), cat("noise_power"), cat("p_max"), cat("weights"),
                     cat("init_precoders"), cat("gamma"), cat("omega"))


def uniform_weights(r: int, K: int) -> np.ndarray:
    return philox(r, ALPHA_STREAM).uniform(0.5, 1.5, size=K)


def kronecker_root(M: int, rho: float = 0.5) -> np.ndarray:
    """Symmetric PSD square root of R_ij = rho^{|i-j|} (eigh)."""
    i = np.arange(M)
    R = rho ** np.abs(i[:, None] - i[None, :])
    w, Q = np.linalg.eigh(R)
    return (Q * np.sqrt(np.clip(w, 0.0, None))) @ Q.T


def build_batch(M: int, N: int, K: int, d: int, B: int, *, p_max: float, sigma2: float = 1.0,
                weights: str = "ones", channel: str = "iid", dtype=np.complex64,
                seed0: int = 0) -> Batch:
    """Batch of B realizations, seeds seed0 .. seed0+B-1.

    Per realization the Philox draws are exactly those of generate_channels /
    init_precoders (model.py); the Kronecker product, the power projection and
    the rounding are applied batch-wise (same arithmetic per element)."""
    rt = np.sqrt(0.5)
    Hc = np.empty((B, K, N, M), dtype=np.complex128)
    Vc = np.empty((B, K, M, d), dtype=np.complex128)
    W = np.ones((B, K), dtype=np.float64)
    beta = np.empty((B, K)) if channel == "kronecker" else None
    if channel not in ("iid", "kronecker"):
        raise ValueError(f"unknown channel model {channel!r}")
    root = kronecker_root(M) if channel == "kronecker" else None
    for b in range(B):
        r = seed0 + b
        g = philox(r, CHANNEL_STREAM)
        re = g.standard_normal((K, N, M))
        im = g.standard_normal((K, N, M))
        Hc[b] = (re + 1j * im) * rt
        g = philox(r, INIT_STREAM)
        re = g.standard_normal((K, M, d))
        im = g.standard_normal((K, M, d))
        v = (re + 1j * im) * rt
        power = float(np.real(np.vdot(v, v)))  # project_sum_power (solvers.py:257-263)
        Vc[b] = v if power <= p_max else v * math.sqrt(p_max / power)
        if beta is not None:  # H_k = sqrt(beta_k) G_k R^{1/2}, per realization
            beta[b] = 10.0 ** philox(r, BETA_STREAM).uniform(-2.0, 0.0, size=K)
            Hc[b] = np.sqrt(beta[b])[:, None, None] * (Hc[b] @ root)
        if weights == "uniform":
            W[b] = uniform_weights(r, K)
    return Batch(Hc.astype(dtype), np.full(B, float(sigma2)), np.full(B, float(p_max)), W,
                 Vc.astype(dtype))


def _build_chunk(args):
    from threadpoolctl import threadpool_limits

    kw, seed0, B = args
    with threadpool_limits(1):  # one BLAS thread per worker process
        return build_batch(B=B, seed0=seed0, **kw)


def build_batch_parallel(M: int, N: int, K: int, d: int, B: int, *, workers: int | None = None,
                         seed0: int = 0, **kw) -> Batch:
    """build_batch over a process pool (chunks of consecutive seeds); identical
    output to build_batch."""
    workers = workers or os.cpu_count() or 1
    if workers <= 1 or B < 64:
        return build_batch(M, N, K, d, B, seed0=seed0, **kw)
    chunk = -(-B // (4 * workers))
    jobs = [(dict(M=M, N=N, K=K, d=d, **kw), seed0 + s, min(chunk, B - s))
            for s in range(0, B, chunk)]
    with ProcessPoolExecutor(max_workers=workers) as pool:
        parts = list(pool.map(_build_chunk, jobs))
    cat = lambda f: np.concatenate([getattr(p, f) for p in parts])
    return Batch(cat("channels"), cat("noise_power"), cat("p_max"), cat("weights"),
                 cat("init_precoders"))


# Named workloads of BASELINE.json "configs" (index in brackets) with the
# (gamma, omega) fixed for them.  BASELINE.json leaves the step unspecified;
# the reference SNR table is unstable at sigma^2 = 1 (SURVEY.md §8(d),
# Appendix A), so each workload records the step chosen by the pilot study
# in DESIGN.md §Step parameters; both arms use these values.
@dataclass(frozen=True)
class Workload:
    name: str
    M: int
    N: int
    K: int
    d: int
    B: int
    p_max: float
    weights: str
    channel: str
    dtype: object
    eps2: float
    max_iters: int
    gamma: float
    omega: float
    eps1: float = 0.1
    snr_db: float = 20.0

    def batch(self, B: int | None = None, seed0: int = 0, workers: int = 1) -> Batch:
        b = build_batch_parallel(self.M, self.N, self.K, self.d, self.B if B is None else B,
                                 p_max=self.p_max, weights=self.weights, channel=self.channel,
                                 dtype=self.dtype, seed0=seed0, workers=workers)
        b.gamma = np.full(b.B, self.gamma)
        b.omega = np.full(b.B, self.omega)
        return b


TINY = np.finfo(np.float64).tiny * np.finfo(np.float64).eps  # smallest positive double (5e-324)

WORKLOADS = {
    # [0] small CPU-oracle case, complex128
    "small": Workload("small", 16, 2, 4, 2, 64, 100.0, "ones", "iid", np.complex128,
                      1e-6, 200, gamma=0.016, omega=0.8, snr_db=20.0),
    # [1] medium case, one entry per SNR point of the sweep {0,10,20,30} dB
    "medium_snr0": Workload("medium_snr0", 64, 2, 16, 2, 4096, 1.0, "uniform", "iid",
                            np.complex64, 1e-5, 300, gamma=0.001, omega=0.8, snr_db=0.0),
    "medium_snr10": Workload("medium_snr10", 64, 2, 16, 2, 4096, 10.0, "uniform", "iid",
                             np.complex64, 1e-5, 300, gamma=0.004, omega=0.8, snr_db=10.0),
    "medium_snr20": Workload("medium_snr20", 64, 2, 16, 2, 4096, 100.0, "uniform", "iid",
                             np.complex64, 1e-5, 300, gamma=0.002, omega=0.8, snr_db=20.0),
    "medium_snr30": Workload("medium_snr30", 64, 2, 16, 2, 4096, 1000.0, "uniform", "iid",
                             np.complex64, 1e-5, 300, gamma=0.002, omega=0.8, snr_db=30.0),
    # [2] large-array case
    "large": Workload("large", 128, 4, 32, 4, 8192, 100.0, "uniform", "iid", np.complex64,
                      1e-5, 500, gamma=0.002, omega=0.8, snr_db=20.0),
    # [3] massive MIMO, Kronecker-correlated
    "massive": Workload("massive", 256, 2, 64, 2, 16384, 100.0, "ones", "kronecker",
                        np.complex64, 1e-5, 500, gamma=0.002, omega=0.8, snr_db=20.0),
}
# [4] throughput sweep: exactly 50 iterations (eps2 = smallest positive double)
for _M, _g in ((32, 0.008), (64, 0.004), (128, 0.002), (256, 0.001), (512, 0.0005)):
    WORKLOADS[f"sweep{_M}"] = Workload(f"sweep{_M}", _M, 2, _M // 4, 2, 65536, 10 ** 1.5, "uniform",
                                       "iid", np.complex64, TINY, 50, gamma=_g, omega=0.8,
                                       snr_db=15.0)

MEDIUM = ("medium_snr0", "medium_snr10", "medium_snr20", "medium_snr30")
