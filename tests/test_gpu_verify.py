"""GPU side of the verification oracles:
  * the engine's recorded block iterates (record_iterates, C-ABI iter_* buffers)
    equal the unmodified reference's on the same inputs (complex128), and the
    batched lemma-bound scan passes on them;
  * the batched bounds kernel (ammmse_bounds) equals compute_bounds (oracle);
  * harness.run_experiment(verify=True) reproduces the reference run's oracle
    reports (tests/golden/harness_verify/summary.json)."""

import json
import os

import numpy as np
import pytest

from oracle import ammmse_oracle as orc
from paper_2510_20507_b200 import ChannelSet, SolverOptions, SystemConfig, run_ammmse_batch
from paper_2510_20507_b200 import harness as Hn
from paper_2510_20507_b200.inputs import build_batch
from paper_2510_20507_b200.verify import check_lemma_bounds, compute_bounds

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "verify")


def _load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", ["lemma_d1", "lemma_d2"])
def test_recorded_iterates_match_reference(cuda, name):
    g = _load(name)
    sk = json.loads(str(g["opts"]))
    opts = SolverOptions(algorithm="ammmse", record_iterates=True, **sk)
    r = run_ammmse_batch(g["channels"][None], float(g["noise_power"]), float(g["p_max"]),
                         g["weights"][None], g["V0"][None], opts)
    n = int(r.iterations[0])
    assert n == int(g["iterations"])
    U, W, V = r.iterates
    np.testing.assert_allclose(U[0, :n], g["U"], rtol=0, atol=1e-8)
    np.testing.assert_allclose(W[0, :n], g["W"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(V[0, :n], g["V"], rtol=0, atol=1e-8)
    # reference-signature oracle on the engine's SolveResult view
    res = r.solve_result(0)
    assert len(res.iterates) == n
    ch = ChannelSet(g["channels"], float(g["noise_power"]))
    b = compute_bounds(ch, g["weights"], float(g["p_max"]), float(g["noise_power"]))
    rep = check_lemma_bounds(ch, res, b, g["weights"])
    assert rep.passed and rep.instances == n and rep.max_abs_error == 0.0
    ref = json.loads(str(g["ref_report"]))
    assert (rep.name, rep.passed, rep.detail) == (ref["name"], ref["passed"], ref["detail"])


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("M,N,K", [(16, 2, 4), (9, 3, 2), (6, 4, 3), (3, 4, 2), (128, 4, 32)])
def test_bounds_kernel_matches_oracle(cuda, dtype, M, N, K):
    import torch

    from paper_2510_20507_b200.solvers import engine

    b = build_batch(M, N, K, 1, 5, p_max=37.0, weights="uniform", dtype=dtype, seed0=11)
    s2 = np.linspace(0.5, 2.0, b.B)
    out = engine().bounds(torch.from_numpy(b.channels).to(cuda), torch.from_numpy(b.weights).to(cuda),
                          torch.from_numpy(b.p_max).to(cuda), torch.from_numpy(s2).to(cuda)).cpu().numpy()
    tol = 1e-10 if dtype == np.complex128 else 1e-5
    for i in range(b.B):
        ref = orc.bounds(b.channels[i].astype(np.complex128), b.weights[i], b.p_max[i], s2[i])
        np.testing.assert_allclose(out[i], ref, rtol=tol)


def test_harness_verify_matches_reference(cuda, tmp_path):
    base = SystemConfig(M=8, N=2, K=2, d=1, p_max=10.0, snr_db=10.0, weights=None, channel_seed=5,
                        init_seed=7)
    solver = SolverOptions(algorithm="ammmse", gamma=0.02, omega=0.5, eps1=0.1, eps2=1e-4,
                           max_iters=80)
    spec = Hn.ExperimentSpec(base=base, solver=solver, n_realizations=3,
                             sweep=(("snr_db", (5.0, 15.0)), ("K", (2.0, 3.0))), parallel_workers=1,
                             output_dir=tmp_path)
    Hn.run_experiment(spec, verify=True)
    got = json.load(open(tmp_path / "summary.json"))["oracles"]
    ref = json.load(open(os.path.join(GOLD, "harness_verify", "summary.json")))["oracles"]
    assert [o["name"] for o in got] == [o["name"] for o in ref]
    for a, b in zip(got, ref):
        assert (a["instances"], a["passed"], a["tolerance"], a["detail"]) == \
            (b["instances"], b["passed"], b["tolerance"], b["detail"]), a["name"]
        if a["name"].startswith("lemma_bounds"):
            assert a["max_abs_error"] == b["max_abs_error"] == 0.0
        else:
            assert a["max_abs_error"] < 1e-9 and b["max_abs_error"] < 1e-9
