"""Second-generation tensor-core cluster engine (csrc/ammmse_tc2.cuh: split
operands resident, precoders / previous G in TMEM, lazy projection, even-depth
A ring with cross-GEMM prefetch, quad-lane per-user algebra) through the C-ABI:
against the fp64 oracle, the FFMA cluster engine and itself in its two
scheduling modes.  The reference's large golden (tests/golden/large.npz, 64
realizations of the unmodified reference) runs on this engine by default in
test_gpu_golden.py."""

import numpy as np
import pytest

from oracle import ammmse_oracle as orc
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch
from paper_2510_20507_b200._native import AmmmseDims, AmmmseOptions, plan_info
from paper_2510_20507_b200.inputs import build_batch

pytestmark = pytest.mark.gpu

WSR_RTOL_C64 = 1e-3  # BASELINE.json north_star: complex64 final WSR within 1e-3 of the fp64 reference
LARGE = dict(M=128, N=4, K=32, d=4)


def _oracle(b, n, **kw):
    """fp64 oracle on the first n realizations (a large realization costs seconds per
    100 iterations on one core)."""
    return orc.solve_batch(b.channels[:n], b.noise_power[:n], b.weights[:n], b.p_max[:n],
                           b.init_precoders[:n], kw["gamma"], kw["omega"], eps2=kw.get("eps2", 1e-3),
                           max_iters=kw["max_iters"], record_trace=True)


def _run(b, opts, **kw):
    return run_ammmse_batch(b.channels, b.noise_power, b.p_max, b.weights, b.init_precoders, opts, **kw)


def test_planner_picks_tc2_for_large(cuda):
    """BASELINE configs[2] (M=128, K=32, N=d=4, complex64): the automatic plan is
    the tc2 engine on 4-CTA clusters; FFMA / first-generation paths stay selectable."""
    dims = AmmmseDims(64, LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 0)
    auto = plan_info(dims, AmmmseOptions(max_iters=10))
    assert auto["tensor_cores"] == 2 and auto["cluster"] == 4
    assert plan_info(dims, AmmmseOptions(max_iters=10, tensor_cores=3))["tensor_cores"] == 2
    assert plan_info(dims, AmmmseOptions(max_iters=10, tensor_cores=1))["tensor_cores"] == 1
    assert plan_info(dims, AmmmseOptions(max_iters=10, tensor_cores=2))["tensor_cores"] == 0
    # shapes the tc2 engine does not cover fall back (N = d = 2 keeps FFMA)
    other = plan_info(AmmmseDims(64, 256, 2, 64, 2, 0), AmmmseOptions(max_iters=10))
    assert other["tensor_cores"] == 0


@pytest.mark.parametrize("B,weights,p_max", [(5, "uniform", 50.0), (1, "ones", 100.0), (37, "uniform", 10.0)])
def test_tc2_matches_oracle_and_ffma(cuda, B, weights, p_max):
    """Same inputs through tc2, the FFMA cluster engine and the fp64 oracle: final WSR
    within the north-star tolerance, identical iteration counts of the two engines
    away from the stop threshold, per-iteration WSR trajectories to 1e-5; ragged
    batch sizes (1, 37: fewer / more realizations than resident clusters)."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], B, p_max=p_max, weights=weights,
                    dtype=np.complex64, seed0=101)
    kw = dict(gamma=0.002, omega=0.8, eps2=1e-5, max_iters=80)
    opts = SolverOptions(algorithm="ammmse", **kw)
    tc = _run(b, opts, record_trace=True, tensor_cores=3)
    ff = _run(b, opts, record_trace=True, tensor_cores=2)
    no = min(B, 2)
    r = _oracle(b, no, **kw)
    assert (tc.status == 0).all() and np.array_equal(tc.status, ff.status)
    for g in (tc, ff):
        rel = np.abs(g.wsr_bits[:no] - r["wsr_bits"]) / np.abs(r["wsr_bits"])
        assert rel.max() <= WSR_RTOL_C64, rel
    np.testing.assert_array_equal(tc.iterations[:no], r["iterations"])
    print(f"tc2 vs oracle: max WSR rel diff "
          f"{(np.abs(tc.wsr_bits[:no] - r['wsr_bits']) / np.abs(r['wsr_bits'])).max():.3e}")
    n = int(min(tc.iterations.min(), ff.iterations.min()))
    np.testing.assert_allclose(tc.trace[:, :n, 1], ff.trace[:, :n, 1], rtol=1e-5)
    np.testing.assert_array_equal(tc.switch_iteration, ff.switch_iteration)
    # feasibility of the returned precoders (lazy projection: V = s X)
    V = tc.final_precoders.astype(np.complex128)
    power = np.sum(np.abs(V) ** 2, axis=(1, 2, 3))
    assert (power <= b.p_max * (1 + 1e-5)).all()
    np.testing.assert_allclose(tc.stationarity_residual, ff.stationarity_residual, rtol=2e-2, atol=1e-7)


def test_tc2_deferred_wsr_mode_is_identical(cuda, monkeypatch):
    """AMMMSE_TC2_DEFER=1 evaluates WSR(t) during GEMM-A(t+1) once the stage is latched
    and discards the speculative step at a stop: iteration counts, WSR and precoders are
    bit-identical to the inline schedule; the exit residual (on a rebuilt G) agrees to
    rounding."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 9, p_max=100.0, weights="uniform",
                    dtype=np.complex64, seed0=7)
    # eps2 loose enough for some realizations to converge before max_iters
    opts = SolverOptions(algorithm="ammmse", gamma=0.002, omega=0.8, eps2=1e-4, max_iters=400)
    monkeypatch.setenv("AMMMSE_TC2_DEFER", "0")
    inline = _run(b, opts, tensor_cores=3)
    monkeypatch.setenv("AMMMSE_TC2_DEFER", "1")
    deferred = _run(b, opts, tensor_cores=3)
    assert inline.converged.any() and (inline.iterations < 400).any()
    np.testing.assert_array_equal(inline.iterations, deferred.iterations)
    np.testing.assert_array_equal(inline.converged, deferred.converged)
    np.testing.assert_array_equal(inline.switch_iteration, deferred.switch_iteration)
    np.testing.assert_array_equal(inline.wsr_bits, deferred.wsr_bits)
    np.testing.assert_array_equal(inline.final_precoders, deferred.final_precoders)
    np.testing.assert_allclose(inline.stationarity_residual, deferred.stationarity_residual, rtol=1e-4)


def test_tc2_two_warp_wsr_is_identical(cuda, monkeypatch):
    """AMMMSE_TC2_WSR_SPLIT=1 factors A and C of every user on two warps concurrently (same
    arithmetic per factorisation): identical iteration counts and precoders, WSR to fp64 rounding."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 5, p_max=100.0, weights="uniform",
                    dtype=np.complex64, seed0=19)
    opts = SolverOptions(algorithm="ammmse", gamma=0.002, omega=0.8, eps2=1e-5, max_iters=120)
    monkeypatch.setenv("AMMMSE_TC2_WSR_SPLIT", "0")
    one = _run(b, opts, record_trace=True, tensor_cores=3)
    monkeypatch.setenv("AMMMSE_TC2_WSR_SPLIT", "1")
    two = _run(b, opts, record_trace=True, tensor_cores=3)
    np.testing.assert_array_equal(one.iterations, two.iterations)
    np.testing.assert_array_equal(one.final_precoders, two.final_precoders)
    np.testing.assert_allclose(one.wsr_bits, two.wsr_bits, rtol=1e-12)
    n = int(one.iterations.min())
    np.testing.assert_allclose(one.trace[:, :n, 1:8], two.trace[:, :n, 1:8], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("kw", [dict(max_iters=1), dict(max_iters=2), dict(omega=0.0, max_iters=40),
                                dict(eps1=1e-12, eps2=1e-13, max_iters=30),  # never leaves stage I
                                dict(eps1=10.0, eps2=1e-5, max_iters=40)])   # weighted from t = 2
def test_tc2_edge_schedules(cuda, kw):
    """Loop edge cases (reference solvers.py:440-505: one / two iterations, no
    extrapolation, a switch that never / immediately happens) against the FFMA engine."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 3, p_max=100.0, weights="uniform",
                    dtype=np.complex64, seed0=55)
    base = dict(gamma=0.002, omega=0.8)
    base.update(kw)
    opts = SolverOptions(algorithm="ammmse", **base)
    tc = _run(b, opts, record_trace=True, tensor_cores=3)
    ff = _run(b, opts, record_trace=True, tensor_cores=2)
    np.testing.assert_array_equal(tc.status, ff.status)
    np.testing.assert_array_equal(tc.iterations, ff.iterations)
    np.testing.assert_array_equal(tc.switch_iteration, ff.switch_iteration)
    np.testing.assert_allclose(tc.wsr_bits, ff.wsr_bits, rtol=1e-5)
    n = int(tc.iterations.min())
    # WSR, f_value, total power, stage, f_after_u / w / v of every recorded iteration
    np.testing.assert_allclose(tc.trace[:, :n, 1:8], ff.trace[:, :n, 1:8], rtol=2e-4, atol=1e-6)
    np.testing.assert_allclose(tc.final_precoders, ff.final_precoders, rtol=0, atol=2e-4)


def test_tc2_divergence_status_matches(cuda):
    """A step far above the safe bound (the iteration is chaotic there, so the engines
    are not compared realization by realization at a marginal step): every realization
    ends in a failure status on both engines (divergence detector solvers.py:490-500 /
    non-finite), none is reported converged, and a step inside the bound fails nowhere."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 4, p_max=100.0, weights="uniform",
                    dtype=np.complex64, seed0=3)
    opts = SolverOptions(algorithm="ammmse", gamma=50.0, omega=0.8, eps2=1e-6, max_iters=80)
    tc = _run(b, opts, tensor_cores=3)
    ff = _run(b, opts, tensor_cores=2)
    assert (ff.status != 0).all() and (tc.status != 0).all()
    assert not tc.converged.any()
    safe = SolverOptions(algorithm="ammmse", gamma="safe", omega=0.5, eps2=1e-6, max_iters=30)
    assert (_run(b, safe, tensor_cores=3).status == 0).all()


def test_tc2_recorded_iterates(cuda):
    """record_iterates (reference solvers.py:487-488) on the tc2 engine: U, W, V of every
    iteration against the FFMA engine (precoders are s X read back from TMEM)."""
    b = build_batch(LARGE["M"], LARGE["N"], LARGE["K"], LARGE["d"], 2, p_max=100.0, weights="uniform",
                    dtype=np.complex64, seed0=77)
    opts = SolverOptions(algorithm="ammmse", gamma=0.002, omega=0.8, eps2=1e-6, max_iters=12,
                         record_iterates=True)
    tc = _run(b, opts, tensor_cores=3)
    ff = _run(b, opts, tensor_cores=2)
    assert tc.iterates is not None and ff.iterates is not None
    for name, x, y in zip(("receivers", "weights", "precoders"), tc.iterates, ff.iterates):
        assert x.shape == y.shape
        n = int(min(tc.iterations.min(), ff.iterations.min()))
        np.testing.assert_allclose(x[:, :n], y[:, :n], rtol=0,
                                   atol=5e-4 * max(1.0, float(np.abs(y[:, :n]).max())), err_msg=name)
