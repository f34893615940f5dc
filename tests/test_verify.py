"""Verification oracles (paper_2510_20507_b200/verify.py)
against fixtures of the unmodified reference (tests/golden/make_verify_golden.py):
the batched lemma-bound scan reproduces the reference check_lemma_bounds report
on the reference's own recorded iterates, flags injected violations family by
family with the reference's slack arithmetic, and the finite-difference gradient
oracle agrees with the reference harness's.  The scan runs on the CPU here (the
same torch code runs on the device in the harness)."""

import json
import math
import os

import numpy as np
import pytest

from paper_2510_20507_b200 import SystemConfig
from paper_2510_20507_b200.verify import (FAMILIES, BoundsReport, OracleReport, gradient_fd_report,
                                          lemma_bound_scan, lemma_report)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "verify")


def _load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k: z[k] for k in z.files}


def _scan(g, U=None, W=None):
    U = g["U"] if U is None else U
    W = g["W"] if W is None else W
    return lemma_bound_scan(g["channels"][None], np.array([float(g["noise_power"])]),
                            g["weights"][None], g["bounds"][None], U[None], W[None], g["V"][None],
                            np.array([U.shape[0]]))


@pytest.mark.parametrize("name", ["lemma_d1", "lemma_d2"])
def test_lemma_scan_matches_reference_report(name):
    g = _load(name)
    worst, lim = _scan(g)
    rep = lemma_report(worst, lim, instances=g["U"].shape[0])
    ref = json.loads(str(g["ref_report"]))
    assert rep.name == ref["name"] and rep.instances == ref["instances"]
    assert rep.passed == ref["passed"] and rep.detail == ref["detail"]
    assert rep.max_abs_error == ref["max_abs_error"] and rep.max_rel_error == ref["max_rel_error"]
    # every family holds with margin on a healthy run
    assert (worst < 0).all(), worst


def test_lemma_scan_flags_each_family():
    g = _load("lemma_d2")
    s2, b = float(g["noise_power"]), g["bounds"]
    d = g["U"].shape[-1]
    # receivers scaled past d / sigma^2
    U = g["U"].copy()
    U[5, 1] *= math.sqrt(2.0 * (d / s2) / max(np.sum(np.abs(U[5, 1]) ** 2), 1e-300))
    worst, lim = _scan(g, U=U)
    rep = lemma_report(worst, lim, instances=U.shape[0])
    assert not rep.passed and "receiver_norm" in rep.detail
    assert worst[0, FAMILIES.index("receiver_norm")] > 0
    # weights scaled past d / ek_floor^2 (also breaks the gradient-factor bound)
    W = g["W"].copy()
    W[7] *= 10.0 * math.sqrt(d) / b[3]
    worst, lim = _scan(g, W=W)
    rep = lemma_report(worst, lim, instances=W.shape[0])
    assert "weight_norm" in rep.detail and "gradient_factor_norm" in rep.detail
    # the reported relative error is the largest normalised excess (verify.py:199-200)
    j = FAMILIES.index("weight_norm")
    assert rep.max_rel_error >= worst[0, j] / abs(lim[0, j])


def test_report_consistency_rule():
    with pytest.raises(Exception):
        OracleReport("x", 1.0, 1.0, 1, True, 0.0)
    with pytest.raises(Exception):
        BoundsReport(1.0, 2.0, 0.4, 0.5, 1.0)  # gamma_safe != 1 / l_v


def test_gradient_fd_matches_reference_harness():
    ref = json.load(open(os.path.join(GOLD, "harness_verify", "summary.json")))["oracles"]
    ref_fd = [o for o in ref if o["name"] == "gradient_finite_difference"][0]
    cfg = SystemConfig(M=8, N=2, K=2, d=1, p_max=10.0, snr_db=10.0, weights=None, channel_seed=5,
                       init_seed=7)
    rep = gradient_fd_report(cfg, device="cpu")
    assert rep.name == ref_fd["name"] and rep.instances == ref_fd["instances"]
    assert rep.passed and ref_fd["passed"]
    # both are finite-difference truncation / rounding noise far below the 1e-6 tolerance
    assert rep.max_abs_error < 1e-9 and ref_fd["max_abs_error"] < 1e-9


def test_gradient_fd_skipped_above_budget():
    cfg = SystemConfig(M=64, N=2, K=16, d=2)
    assert gradient_fd_report(cfg, device="cpu") is None
