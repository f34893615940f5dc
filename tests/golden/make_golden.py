"""Generate the golden fixtures tests/golden/*.npz by running the UNMODIFIED
reference (`wsrbeam.run_ammmse`, /root/reference/pkg/src) on seeded inputs.

Runs only in the build container, where /root/reference is importable; the
fixtures are committed and travel to the GPU box, the reference does not.

Inputs come from paper_2510_20507_b200.inputs (restated generators; the
script asserts they are bit-identical to the reference's generate_channels /
init_precoders).  V0 is injected by replacing the module-level name
`wsrbeam.solvers.init_precoders` that `_run_bcd` calls (solvers.py:41, :427),
so both sides start from the identical (possibly complex64-rounded) V0.

    python tests/golden/make_golden.py [case ...]
"""

import math
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from concurrent.futures import ProcessPoolExecutor  # noqa: E402

import numpy as np  # noqa: E402

from paper_2510_20507_b200.inputs import WORKLOADS, Batch, build_batch  # noqa: E402

TRACE_KEEP = 8      # realizations per case whose full trace is stored
WORKERS = int(os.environ.get("GOLDEN_WORKERS", "8"))
V_KEEP = 4          # realizations per case whose final precoders are stored


def _case(name, batch: Batch, opts: dict, snr_db=10.0, note="", workload=""):
    """workload != "": inputs are WORKLOADS[workload].batch(B) and are regenerated
    by the tests instead of being stored (bit-identical Philox streams)."""
    return dict(name=name, batch=batch, opts=opts, snr_db=snr_db, note=note, workload=workload)


def cases():
    out = []
    w = WORKLOADS["small"]
    out.append(_case("small", w.batch(), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1, eps2=w.eps2,
                                              max_iters=w.max_iters), note="BASELINE configs[0], full batch",
                     workload="small"))
    for n in ("medium_snr0", "medium_snr10", "medium_snr20", "medium_snr30"):
        w = WORKLOADS[n]
        out.append(_case(n, w.batch(B=64), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1,
                                                eps2=w.eps2, max_iters=w.max_iters),
                         note="BASELINE configs[1], seeds 0-63", workload=n))
    # the same SNR points with room to converge (at max_iters = 300 every 20 / 30 dB
    # realization stops at the cap, so their stop test is never exercised)
    # (max_iters bounded: over thousands of extrapolated, non-monotone iterations of
    # this non-convex problem an fp32 trajectory can settle on another stationary
    # point than the fp64 one)
    for n, T in (("medium_snr20", 1500), ("medium_snr30", 1000)):
        w = WORKLOADS[n]
        out.append(_case(n + "_long", w.batch(B=24), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1,
                                                          eps2=w.eps2, max_iters=T),
                         note=f"BASELINE configs[1] inputs, max_iters {T} (converging)", workload=n))
    w = WORKLOADS["large"]
    out.append(_case("large", w.batch(B=64), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1,
                                                  eps2=w.eps2, max_iters=w.max_iters),
                     note="BASELINE configs[2], seeds 0-63", workload="large"))
    w = WORKLOADS["massive"]
    out.append(_case("massive", w.batch(B=32), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1,
                                                    eps2=w.eps2, max_iters=w.max_iters),
                     note="BASELINE configs[3], seeds 0-31", workload="massive"))
    for M, B in ((32, 32), (64, 32), (128, 16), (256, 16), (512, 4)):
        w = WORKLOADS[f"sweep{M}"]
        out.append(_case(f"sweep{M}", w.batch(B=B), dict(gamma=w.gamma, omega=w.omega, eps1=w.eps1,
                                                          eps2=w.eps2, max_iters=w.max_iters),
                         note="BASELINE configs[4]", workload=f"sweep{M}"))
    # edge cases of the reference's own tests (test_solvers.py)
    b = build_batch(16, 2, 4, 2, 4, p_max=10.0, dtype=np.complex128, seed0=100)
    out.append(_case("edge_safe_monotone", b, dict(gamma="safe", omega=0.0, eps1=math.inf, eps2=1e-3,
                                                   max_iters=400),
                     note="test_solvers.py:402-415 monotone regime"))
    out.append(_case("edge_safe_tight", build_batch(16, 2, 4, 2, 2, p_max=10.0, dtype=np.complex128,
                                                    seed0=1),
                     dict(gamma="safe", omega=0.0, eps2=1e-6, max_iters=5000),
                     note="test_solvers.py:471-477 stationarity at tight tolerance"))
    b = build_batch(16, 2, 4, 2, 3, p_max=10.0, dtype=np.complex128, seed0=11)
    out.append(_case("edge_unlatched", b, dict(gamma=0.01, omega=0.6, eps2=1e-4, max_iters=300,
                                               latch_stage=False)))
    # Table I at 10 dB (0.05) is chaotic at sigma^2 = 1; 20 dB is not
    out.append(_case("edge_table_snr20", b, dict(gamma=None, omega=None, eps2=1e-4, max_iters=300),
                     snr_db=20.0, note="Table I defaults at 20 dB (0.8, 0.003)"))
    out.append(_case("edge_switch_eq_stop", b, dict(gamma=0.01, omega=0.6, eps1=1e-3, eps2=1e-3,
                                                    max_iters=500),
                     note="eps1 == eps2 (test_solvers.py:361-382 analogue)"))
    out.append(_case("edge_max_iters_1", build_batch(16, 2, 4, 2, 2, p_max=100.0,
                                                     dtype=np.complex128),
                     dict(gamma=0.01, omega=0.8, eps2=1e-6, max_iters=1)))
    for (M, N, K, d) in ((6, 1, 2, 1), (12, 4, 3, 2), (10, 3, 2, 3), (9, 2, 1, 1), (5, 2, 3, 2),
                         (16, 4, 4, 4)):
        b = build_batch(M, N, K, d, 3, p_max=10.0, weights="uniform", dtype=np.complex128, seed0=7)
        out.append(_case(f"edge_shape_M{M}N{N}K{K}d{d}", b,
                         dict(gamma=0.005, omega=0.5, eps2=1e-5, max_iters=150)))
    # divergence (test_solvers.py:438-449): two users on one channel, gamma=1000
    rng = np.random.default_rng(3)
    h1 = (rng.standard_normal((1, 6)) + 1j * rng.standard_normal((1, 6))) * np.sqrt(0.5)
    H = np.stack([h1, h1])[None]
    import wsrbeam as wb
    cfg = wb.SystemConfig(M=6, N=1, K=2, d=1, snr_db=30.0, channel_seed=0, init_seed=0)
    s2 = wb.compute_noise_power(wb.ChannelSet(H[0]), cfg.snr_db, cfg)
    V0 = wb.init_precoders(cfg, wb.project_sum_power).precoders[None]
    bd = Batch(H, np.array([s2]), np.array([cfg.p_max]), np.ones((1, 2)), V0)
    out.append(_case("edge_divergence", bd, dict(gamma=1000.0, omega=0.9, eps1=1e-8, eps2=1e-10,
                                                 max_iters=300),
                     note="UnstableParametersError expected"))
    return out


def _ref_one(args):
    import wsrbeam as wb
    import wsrbeam.solvers as ws

    H, s2, alpha, p_max, V0, opts, snr_db, r = args
    M, N, K, d = H.shape[2], H.shape[1], H.shape[0], V0.shape[2]
    cfg = wb.SystemConfig(M=M, N=N, K=K, d=d, p_max=float(p_max), snr_db=snr_db,
                          weights=tuple(float(a) for a in alpha), channel_seed=r, init_seed=r)
    ch = wb.ChannelSet(H, noise_power=float(s2))
    v0 = wb.PrecoderSet(V0)
    ws.init_precoders = lambda config, project: v0  # V0 injection (solvers.py:427)
    so = wb.SolverOptions(algorithm=wb.Algorithm.AMMMSE, **opts)
    try:
        res = wb.run_ammmse(ch, cfg, so)
    except (wb.UnstableParametersError, wb.IllConditionedWeightError) as exc:
        status = 2 if isinstance(exc, wb.UnstableParametersError) else 1
        return dict(status=status, iterations=-1, wsr_bits=math.nan, converged=False,
                    switch_iteration=-1, residual=math.nan, trace=np.zeros((0, 9)),
                    V=np.full_like(V0, np.nan), error=f"{type(exc).__name__}: {exc}")
    tr = np.array([[x.t, x.wsr_bits, x.f_value, x.total_power, x.stage.value, x.f_after_u,
                    x.f_after_w, x.f_after_v, x.rel_change] for x in res.trace])
    return dict(status=0, iterations=res.iterations, wsr_bits=res.trace[-1].wsr_bits,
                converged=res.converged,
                switch_iteration=-1 if res.switch_iteration is None else res.switch_iteration,
                residual=res.stationarity_residual, trace=tr, V=res.final_precoders.precoders,
                error="")


def check_generators():
    import wsrbeam as wb

    from paper_2510_20507_b200.model import SystemConfig, generate_channels, init_precoders
    for r in (0, 5, 77):
        for (M, N, K, d) in ((16, 2, 4, 2), (7, 3, 2, 1)):
            a = wb.SystemConfig(M=M, N=N, K=K, d=d, p_max=3.0, channel_seed=r, init_seed=r + 1)
            b = SystemConfig(M=M, N=N, K=K, d=d, p_max=3.0, channel_seed=r, init_seed=r + 1)
            assert np.array_equal(wb.generate_channels(a).channels, generate_channels(b).channels)
            assert np.array_equal(wb.init_precoders(a, wb.project_sum_power).precoders,
                                  init_precoders(b).precoders)


def main():
    check_generators()
    want = set(sys.argv[1:])
    for c in cases():
        if want and c["name"] not in want:
            continue
        b = c["batch"]
        t0 = time.time()
        jobs = [(b.channels[i], b.noise_power[i], b.weights[i], b.p_max[i], b.init_precoders[i],
                 c["opts"], c["snr_db"], i) for i in range(b.B)]
        with ProcessPoolExecutor(max_workers=min(WORKERS, len(jobs))) as pool:
            res = list(pool.map(_ref_one, jobs))
        nT = min(TRACE_KEEP, b.B)
        T = max([r["trace"].shape[0] for r in res[:nT]] + [1])
        trace = np.full((nT, T, 9), np.nan)
        for i in range(nT):
            trace[i, : res[i]["trace"].shape[0]] = res[i]["trace"]
        # rel_change of every realization (marginal stop / switch decisions)
        TA = max([r["trace"].shape[0] for r in res] + [1])
        rel_all = np.full((b.B, TA), np.nan)
        for i, r in enumerate(res):
            rel_all[i, : r["trace"].shape[0]] = r["trace"][:, 8] if r["trace"].size else []
        nV = min(V_KEEP, b.B, (1 << 16) // max(1, 2 * b.init_precoders[0].nbytes))
        opts = c["opts"]
        inputs = {} if c["workload"] else dict(
            channels=b.channels, noise_power=b.noise_power, p_max=b.p_max, weights=b.weights,
            init_precoders=b.init_precoders)
        np.savez_compressed(
            os.path.join(HERE, f"{c['name']}.npz"), workload=np.array(c["workload"]),
            batch_size=np.array(b.B), **inputs,
            gamma=np.array(np.nan if opts.get("gamma") is None else
                           (-1.0 if opts["gamma"] == "safe" else opts["gamma"])),
            omega=np.array(np.nan if opts.get("omega") is None else opts["omega"]),
            eps1=np.array(opts.get("eps1", 0.1)), eps2=np.array(opts.get("eps2", 1e-3)),
            max_iters=np.array(opts.get("max_iters", 1000)),
            latch_stage=np.array(opts.get("latch_stage", True)), snr_db=np.array(c["snr_db"]),
            ref_status=np.array([r["status"] for r in res], dtype=np.int32),
            ref_iterations=np.array([r["iterations"] for r in res], dtype=np.int32),
            ref_wsr_bits=np.array([r["wsr_bits"] for r in res]),
            ref_converged=np.array([r["converged"] for r in res]),
            ref_switch_iteration=np.array([r["switch_iteration"] for r in res], dtype=np.int32),
            ref_residual=np.array([r["residual"] for r in res]),
            ref_trace=trace, ref_rel=rel_all, ref_final_precoders=(np.stack([res[i]["V"] for i in range(nV)]) if nV else
                                 np.zeros((0,) + b.init_precoders.shape[1:], np.complex128)),
            note=np.array(c["note"]))
        print(f"{c['name']}: B={b.B} {time.time() - t0:.1f}s status={[r['status'] for r in res][:8]} "
              f"iters={[r['iterations'] for r in res][:8]}", flush=True)


if __name__ == "__main__":
    main()
