"""On-device synthetic inputs (ammmse_generate_iid):
counter-based determinism, CN(0,1) moments, the sum-power projection of V0,
the weight distribution, and solver parity on device-generated inputs (the
oracle solves the same inputs copied to the host)."""

import numpy as np
import pytest

from oracle import ammmse_oracle as orc
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch
from paper_2510_20507_b200.solvers import AmmmseEngine

pytestmark = pytest.mark.gpu


def _gen(cuda, *a, **kw):
    import torch

    H, V0, A = AmmmseEngine(cuda).generate_iid(*a, **kw)
    torch.cuda.synchronize()
    return H.cpu().numpy(), V0.cpu().numpy(), A.cpu().numpy()


def test_counter_based_determinism(cuda):
    a = _gen(cuda, 6, 3, 2, 8, 2, seed0=11, p_max=5.0)
    b = _gen(cuda, 6, 3, 2, 8, 2, seed0=11, p_max=5.0)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    # realization r of seed0 is realization 0 of seed0 + r (seeds by global index)
    c = _gen(cuda, 2, 3, 2, 8, 2, seed0=14, p_max=5.0)
    for x, y in zip(a, c):
        np.testing.assert_array_equal(x[3:5], y)
    d = _gen(cuda, 6, 3, 2, 8, 2, seed0=12, p_max=5.0)
    assert not np.array_equal(a[0], d[0])


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_cn01_moments_and_projection(cuda, dtype):
    B, K, N, M, d, P = 2048, 4, 2, 16, 2, 10.0
    H, V0, A = _gen(cuda, B, K, N, M, d, seed0=0, p_max=P, dtype=dtype)
    assert H.dtype == np.dtype(dtype) and H.shape == (B, K, N, M) and V0.shape == (B, K, M, d)
    x = H.astype(np.complex128).ravel()
    n = x.size
    for comp in (x.real, x.imag):
        assert abs(comp.mean()) < 5 / np.sqrt(n)
        assert abs(comp.var() - 0.5) < 0.01
        assert abs(np.mean(comp ** 4) / comp.var() ** 2 - 3.0) < 0.05  # Gaussian kurtosis
    assert abs(np.mean(x.real * x.imag)) < 5 * 0.5 / np.sqrt(n)
    # V0 on the power ball: ||V0||^2 = P whenever the CN(0,1) draw exceeded it
    # (K M d = 128 >> P here, so always)
    pw = np.sum(np.abs(V0.astype(np.complex128)) ** 2, axis=(1, 2, 3))
    np.testing.assert_allclose(pw, P, rtol=1e-5 if dtype == "complex64" else 1e-12)
    assert A.shape == (B, K) and (A >= 0.5).all() and (A < 1.5).all()
    assert abs(A.mean() - 1.0) < 0.02


def test_weights_ones(cuda):
    _, _, A = _gen(cuda, 8, 5, 1, 4, 1, seed0=3, p_max=1.0, weights="ones")
    np.testing.assert_array_equal(A, 1.0)


def test_solver_parity_on_device_generated_inputs(cuda):
    H, V0, A = _gen(cuda, 5, 4, 2, 16, 2, seed0=100, p_max=100.0, dtype="complex128")
    s2 = np.ones(5)
    opts = SolverOptions(algorithm="ammmse", gamma=0.01, omega=0.8, eps2=1e-6, max_iters=150)
    g = run_ammmse_batch(H, s2, 100.0, A, V0, opts)
    r = orc.solve_batch(H, s2, A, 100.0, V0, 0.01, 0.8, eps2=1e-6, max_iters=150)
    assert np.array_equal(g.iterations, r["iterations"])
    assert np.array_equal(g.status, r["status"])
    np.testing.assert_allclose(g.wsr_bits, r["wsr_bits"], rtol=1e-9)


def test_kronecker_generation(cuda):
    """H_k = sqrt(beta_k) G_k R^{1/2}: undoing R^{1/2} leaves white rows whose
    power is beta_k, log-uniform over [0.01, 1); deterministic in the seed."""
    import torch

    from paper_2510_20507_b200.inputs import kronecker_root

    B, K, N, M = 512, 3, 2, 16
    eng = AmmmseEngine(cuda)
    H, V0, A = eng.generate_kronecker(B, K, N, M, 2, seed0=5, p_max=10.0, dtype="complex128")
    torch.cuda.synchronize()
    H = H.cpu().numpy()
    np.testing.assert_array_equal(A.cpu().numpy(), 1.0)
    # undo the correlation: G = H R^{-1/2} / sqrt(beta) must be white with equal row power
    root = kronecker_root(M)
    G = H @ np.linalg.inv(root)
    p = np.mean(np.abs(G) ** 2, axis=(2, 3))  # (B, K) = beta_k
    assert (p > 0.004).all() and (p < 1.6).all()
    lb = np.log10(p).ravel()
    # per-(b, k) power estimated from N M = 32 samples: allow the chi-square spread
    assert -2.7 < lb.min() and lb.max() < 0.35 and abs(lb.mean() + 1.0) < 0.1
    Gn = G / np.sqrt(p)[:, :, None, None]
    C = np.einsum("bkni,bknj->ij", Gn, Gn.conj()) / (B * K * N)
    np.testing.assert_allclose(C, np.eye(M), atol=0.08)
    # deterministic
    H2 = eng.generate_kronecker(B, K, N, M, 2, seed0=5, p_max=10.0, dtype="complex128")[0]
    np.testing.assert_array_equal(H, H2.cpu().numpy())
