"""Boundary demonstration: the UNMODIFIED reference,
installed in baseline/_ref (pip install --no-index --target baseline/_ref of
/root/reference/pkg), runs its stock experiment harness
(wsrbeam.harness.run_experiment) once on its own CPU drivers and once with the
device drivers swapped into wsrbeam.solvers._DRIVERS by the reference-side
ctypes stub (integration/wsrbeam_b200.py, C-ABI of include/ammmse.h, no torch).
The two runs' summary.json and per-realization trace CSVs must agree (fp64 on
both sides)."""

import csv
import dataclasses
import json
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def wsrbeam_ref():
    if not os.path.isdir(os.path.join(REF, "wsrbeam")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import wsrbeam

    return wsrbeam


def _rows(path):
    with open(path) as f:
        return [[float(x) for x in r] for r in list(csv.reader(f))[1:]]


@pytest.mark.parametrize("algorithm,extra", [("ammmse", dict(gamma=0.02, omega=0.5)),
                                             ("wmmse", dict()), ("mmmse", dict())])
def test_stock_harness_on_device_drivers(cuda, wsrbeam_ref, tmp_path, algorithm, extra):
    wb = wsrbeam_ref
    from wsrbeam import harness as H
    from wsrbeam import solvers as ws

    sys.path.insert(0, ROOT)
    from integration import wsrbeam_b200 as b200

    if algorithm == "ammmse":
        base = wb.SystemConfig(M=8, N=2, K=2, d=1, p_max=10.0, snr_db=10.0, channel_seed=5,
                               init_seed=7)
        sweep = (("snr_db", (5.0, 15.0)), ("K", (2.0, 3.0)))
    else:
        # exact drivers on full-rank systems (K d >= M): with a rank-deficient weighted
        # Gram the reference's first cho_factor(A) at lambda = 0 succeeds or fails on
        # rounding-level pivot signs (LAPACK's blocked order vs ours), which decides
        # between its lambda = 0 answer and the bisection
        base = wb.SystemConfig(M=6, N=2, K=3, d=2, p_max=10.0, snr_db=10.0, channel_seed=5,
                               init_seed=7)
        sweep = (("snr_db", (5.0, 15.0)), ("K", (3.0, 4.0)))
    solver = wb.SolverOptions(algorithm=algorithm, eps1=0.1, eps2=1e-4, max_iters=80, **extra)
    spec = H.ExperimentSpec(base=base, solver=solver, n_realizations=3, sweep=sweep,
                            parallel_workers=1, output_dir=tmp_path / "stock")
    H.run_experiment(spec)
    prev = b200.install()
    try:
        assert ws._DRIVERS[ws.Algorithm.AMMMSE] is b200.run_ammmse_b200
        H.run_experiment(dataclasses.replace(spec, output_dir=tmp_path / "b200"))
    finally:
        ws._DRIVERS.clear()
        ws._DRIVERS.update(prev)
    a = json.load(open(tmp_path / "stock" / "summary.json"))
    b = json.load(open(tmp_path / "b200" / "summary.json"))
    assert [p["label"] for p in a["points"]] == [p["label"] for p in b["points"]]
    for pa, pb in zip(a["points"], b["points"]):
        for key in ("n_realizations", "n_completed", "n_converged", "iterations_mean",
                    "switch_iteration_mean", "failures"):
            assert pa[key] == pb[key], (pa["label"], key)
        np.testing.assert_allclose(pb["wsr_bits_mean"], pa["wsr_bits_mean"], rtol=1e-9)
        np.testing.assert_allclose(pb["stationarity_residual_max"], pa["stationarity_residual_max"],
                                   rtol=1e-6)
    files = sorted(f for f in os.listdir(tmp_path / "stock") if f.endswith(".csv"))
    assert files == sorted(f for f in os.listdir(tmp_path / "b200") if f.endswith(".csv"))
    for f in files:
        ra, rb = _rows(tmp_path / "stock" / f), _rows(tmp_path / "b200" / f)
        assert len(ra) == len(rb), f
        for x, y in zip(ra, rb):
            assert x[0] == y[0] and x[4] == y[4], f  # iteration index, stage
            np.testing.assert_allclose(np.array(y[:4] + y[5:-1], dtype=float),
                                       np.array(x[:4] + x[5:-1], dtype=float), rtol=1e-8, atol=1e-10)
