"""Exact-update drivers on the device (run_wmmse /
run_mmmse, ref solvers.py:521-537) through ammmse_solve_exact against the
unmodified reference's outputs on the same inputs
(tests/golden/make_exact_golden.py): fp64 engine, so status, iteration /
switch counts and convergence flags must be identical, WSR within 1e-9,
traces within 1e-8, residuals within 1e-6.  The fixtures cover both drivers,
d = 1..3, N = 1..4, user weights, and the singular-Gram interior optimum where
bisect_dual falls back to np.linalg.lstsq every iteration."""

import glob
import json
import os

import numpy as np
import pytest

from paper_2510_20507_b200 import (ChannelSet, SolverOptions, SystemConfig, run_exact_batch,
                                   run_mmmse, run_wmmse, solve)
from paper_2510_20507_b200.errors import ConfigError

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "exact")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz")))


def _load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", NAMES)
def test_exact_driver_matches_reference(cuda, name):
    g = _load(name)
    opts = SolverOptions(algorithm=str(g["algorithm"]), **json.loads(str(g["opts"])))
    r = run_exact_batch(g["channels"], g["noise_power"], g["p_max"], g["weights"],
                        g["init_precoders"], opts, record_trace=True)
    assert np.array_equal(r.status, g["ref_status"])
    ok = g["ref_status"] == 0
    assert np.array_equal(r.iterations[ok], g["ref_iterations"][ok])
    assert np.array_equal(r.switch_iteration[ok], g["ref_switch_iteration"][ok])
    assert np.array_equal(r.converged.astype(bool)[ok], g["ref_converged"][ok])
    np.testing.assert_allclose(r.wsr_bits[ok], g["ref_wsr_bits"][ok], rtol=1e-9)
    np.testing.assert_allclose(r.stationarity_residual[ok], g["ref_residual"][ok], rtol=1e-6,
                               atol=1e-12)
    for b in np.nonzero(ok)[0]:
        n = int(g["ref_iterations"][b])
        np.testing.assert_allclose(r.trace[b, :n, :8], g["ref_trace"][b, :n, :8], rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(r.final_precoders[ok], g["ref_final_precoders"][ok], rtol=0, atol=1e-8)


def test_reference_signature_and_dispatch(cuda):
    g = _load("mmmse_small")
    H = g["channels"][0]
    K, N, M = H.shape
    d = g["init_precoders"].shape[3]
    cfg = SystemConfig(M=M, N=N, K=K, d=d, p_max=float(g["p_max"][0]), snr_db=10.0)
    ch = ChannelSet(H, float(g["noise_power"][0]))
    opts = SolverOptions(algorithm="mmmse", **json.loads(str(g["opts"])))
    res = run_mmmse(ch, cfg, opts, init=g["init_precoders"][0])
    assert res.iterations == int(g["ref_iterations"][0])
    assert abs(res.trace[-1].wsr_bits - g["ref_wsr_bits"][0]) <= 1e-9 * abs(g["ref_wsr_bits"][0])
    with pytest.raises(ConfigError):
        run_wmmse(ch, cfg, opts)  # algorithm mismatch (solvers.py:524-525)
    w = solve(ch, cfg, SolverOptions(algorithm="wmmse", eps2=1e-5, max_iters=50))
    assert w.switch_iteration is None and all(r.stage.value == 1 for r in w.trace)
