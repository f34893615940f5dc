"""Harness integration against fixtures made by the
unmodified reference runner (tests/golden/make_harness_golden.py):
trace CSV format, sweep expansion and summary.json of a batched run."""

import dataclasses
import json
import os

import numpy as np
import pytest

from paper_2510_20507_b200 import ConfigError, SolverOptions, SystemConfig
from paper_2510_20507_b200 import harness as H
from paper_2510_20507_b200.solvers import SolveResult

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness")


def _spec(outdir):
    """The spec of make_harness_golden.py, in this package's types."""
    base = SystemConfig(M=8, N=2, K=2, d=1, p_max=10.0, snr_db=10.0, weights=None, channel_seed=5,
                        init_seed=7)
    solver = SolverOptions(algorithm="ammmse", gamma=0.02, omega=0.5, eps1=0.1, eps2=1e-4,
                           max_iters=80)
    return H.ExperimentSpec(base=base, solver=solver, n_realizations=3,
                            sweep=(("snr_db", (5.0, 15.0)), ("K", (2.0, 3.0))), parallel_workers=1,
                            output_dir=outdir)


def _ref_traces():
    return sorted(f for f in os.listdir(GOLD) if f.endswith(".csv"))


class TestTraceFormat:
    def test_round_trip_is_byte_identical_to_reference(self, tmp_path):
        for name in _ref_traces():
            recs = H.read_trace(os.path.join(GOLD, name))
            res = SolveResult(final_precoders=None, trace=recs, iterations=len(recs),
                              converged=False, stationarity_residual=0.0)
            out = tmp_path / name
            H.emit_trace(res, out)
            assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read(), name

    def test_bad_header_rejected(self, tmp_path):
        p = tmp_path / "x.csv"
        p.write_text("iter,wsr\n1,2\n")
        with pytest.raises(ConfigError):
            H.read_trace(p)


class TestSpec:
    def test_sweep_labels_match_reference(self, tmp_path):
        ref = json.load(open(os.path.join(GOLD, "sweep_labels.json")))["labels"]
        s = _spec(tmp_path)
        big = H.ExperimentSpec(base=s.base, solver=s.solver, n_realizations=1,
                               sweep=(("M", (8.0, 16.0)), ("snr_db", (0.0, 12.5)), ("K", (2.0, 4.0))))
        pts = H.sweep_points(big)
        assert [lab for lab, _ in pts] == ref
        for lab, cfg in pts:  # K sweep resets the weight vector to the new length
            assert len(cfg.weights) == cfg.K

    @pytest.mark.parametrize("kw", [dict(n_realizations=0), dict(parallel_workers=-1),
                                    dict(sweep=(("d", (1.0,)),)), dict(sweep=(("K", ()),)),
                                    dict(sweep=(("K", (2.5,)),)),
                                    dict(sweep=(("snr_db", (float("nan"),)),))])
    def test_invalid_specs(self, tmp_path, kw):
        s = _spec(tmp_path)
        with pytest.raises(ConfigError):
            dataclasses.replace(s, **kw)

    def test_other_algorithms_rejected(self, tmp_path):
        s = _spec(tmp_path)
        with pytest.raises(ConfigError):
            H.run_experiment(dataclasses.replace(s, solver=dataclasses.replace(s.solver,
                                                                               algorithm="wmmse")))

    def test_point_inputs_use_consecutive_seeds(self, tmp_path):
        s = _spec(tmp_path)
        Hs, s2, alpha, V0, cfgs = H.point_inputs(s.base, 3)
        assert [c.channel_seed for c in cfgs] == [5, 6, 7]
        assert [c.init_seed for c in cfgs] == [7, 8, 9]
        assert Hs.shape == (3, 2, 2, 8) and V0.shape == (3, 2, 8, 1) and s2.shape == (3,)


@pytest.mark.gpu
def test_batched_run_matches_reference_summary(cuda, tmp_path):
    summary = H.run_experiment(_spec(tmp_path))
    ours = json.load(open(tmp_path / "summary.json"))
    ref = json.load(open(os.path.join(GOLD, "summary.json")))
    assert ours["spec"]["sweep"] == ref["spec"]["sweep"]
    assert len(ours["points"]) == len(ref["points"]) == len(summary.points)
    for p, q in zip(ours["points"], ref["points"]):
        assert p["label"] == q["label"]
        assert p["config"] == q["config"] and p["solver"] == q["solver"]
        for k in ("n_realizations", "n_completed", "n_converged", "convergence_rate",
                  "iterations_mean", "iterations_std", "switch_iteration_mean", "failures"):
            assert p[k] == q[k], (p["label"], k)
        np.testing.assert_allclose(p["wsr_bits_mean"], q["wsr_bits_mean"], rtol=1e-9)
        np.testing.assert_allclose(p["wsr_bits_std"], q["wsr_bits_std"], rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(p["stationarity_residual_max"], q["stationarity_residual_max"],
                                   rtol=1e-6, atol=1e-12)
    assert sorted(f for f in os.listdir(tmp_path) if f.endswith(".csv")) == _ref_traces()
    for name in _ref_traces():
        a = H.read_trace(tmp_path / name)
        b = H.read_trace(os.path.join(GOLD, name))
        assert [r.t for r in a] == [r.t for r in b]
        assert [r.stage for r in a] == [r.stage for r in b]
        for fld, tol in (("wsr_bits", 1e-9), ("f_value", 1e-8), ("total_power", 1e-9),
                         ("f_after_u", 1e-8), ("f_after_w", 1e-8), ("f_after_v", 1e-8)):
            np.testing.assert_allclose([getattr(r, fld) for r in a], [getattr(r, fld) for r in b],
                                       rtol=tol, atol=1e-10, err_msg=f"{name} {fld}")
