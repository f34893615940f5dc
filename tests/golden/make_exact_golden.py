"""Fixtures for the exact-update drivers from the
UNMODIFIED reference (run here, where /root/reference exists):

  python tests/golden/make_exact_golden.py

Writes tests/golden/exact/<case>.npz: inputs (channels, noise power, weights,
p_max, V0 exactly as init_precoders draws them), options, and the reference
run_wmmse / run_mmmse outputs per realization (status, iterations, WSR,
converged, switch iteration, stationarity residual, trace, final precoders),
plus how many bisections fell back to np.linalg.lstsq (solvers.py:324-327).
"""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import wsrbeam  # noqa: E402
import wsrbeam.solvers as ws  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "exact")

CASES = {  # name: (algorithm, SystemConfig kwargs (seed base), SolverOptions kwargs, B)
    "wmmse_small": ("wmmse", dict(M=8, N=2, K=3, d=2, p_max=10.0, snr_db=10.0), dict(eps2=1e-5, max_iters=100), 4),
    "mmmse_small": ("mmmse", dict(M=8, N=2, K=3, d=2, p_max=10.0, snr_db=10.0), dict(eps2=1e-5, max_iters=150), 4),
    "wmmse_m16": ("wmmse", dict(M=16, N=2, K=4, d=2, p_max=100.0, snr_db=20.0), dict(eps2=1e-6, max_iters=200), 3),
    "mmmse_m16": ("mmmse", dict(M=16, N=2, K=4, d=2, p_max=100.0, snr_db=20.0), dict(eps2=1e-6, max_iters=300), 3),
    "wmmse_d1": ("wmmse", dict(M=6, N=1, K=2, d=1, p_max=5.0, snr_db=5.0), dict(eps2=1e-6, max_iters=200), 3),
    "mmmse_n4d3": ("mmmse", dict(M=12, N=4, K=3, d=3, p_max=20.0, snr_db=12.0,
                                 weights=(1.0, 0.5, 1.5)), dict(eps2=1e-5, max_iters=200), 3),
    # K d < M: the weighted Gram is singular; a large power budget makes the
    # unconstrained optimum interior (bisection cannot reach the band -> lstsq)
    "wmmse_interior": ("wmmse", dict(M=12, N=2, K=2, d=1, p_max=1e4, snr_db=0.0),
                       dict(eps2=1e-6, max_iters=60), 3),
}


def run_case(name, algo, ck, sk, B):
    calls = {"lstsq": 0}
    real_lstsq = np.linalg.lstsq

    def counting_lstsq(*a, **k):
        calls["lstsq"] += 1
        return real_lstsq(*a, **k)

    np.linalg.lstsq = counting_lstsq
    recs = []
    try:
        for r in range(B):
            cfg = wsrbeam.SystemConfig(**ck, channel_seed=100 + r, init_seed=200 + r)
            ch = wsrbeam.generate_channels(cfg)
            ch = ch.with_noise_power(wsrbeam.compute_noise_power(ch, cfg.snr_db, cfg))
            V0 = wsrbeam.init_precoders(cfg, wsrbeam.project_sum_power).precoders
            opts = wsrbeam.SolverOptions(algorithm=algo, **sk)
            try:
                res = ws.solve(ch, cfg, opts)
                tr = np.array([[x.t, x.wsr_bits, x.f_value, x.total_power, x.stage.value, x.f_after_u,
                                x.f_after_w, x.f_after_v, x.rel_change] for x in res.trace])
                recs.append(dict(H=ch.channels, s2=ch.noise_power, w=cfg.weight_vector, V0=V0, status=0,
                                 it=res.iterations, wsr=res.trace[-1].wsr_bits, conv=res.converged,
                                 sw=-1 if res.switch_iteration is None else res.switch_iteration,
                                 resid=res.stationarity_residual, trace=tr,
                                 V=res.final_precoders.precoders))
            except wsrbeam.IllConditionedWeightError:
                recs.append(dict(H=ch.channels, s2=ch.noise_power, w=cfg.weight_vector, V0=V0, status=1,
                                 it=-1, wsr=math.nan, conv=False, sw=-1, resid=math.nan,
                                 trace=np.zeros((0, 9)), V=np.full_like(V0, np.nan)))
    finally:
        np.linalg.lstsq = real_lstsq
    T = max([r["trace"].shape[0] for r in recs] + [1])
    trace = np.full((B, T, 9), np.nan)
    for i, r in enumerate(recs):
        trace[i, : r["trace"].shape[0]] = r["trace"]
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"), algorithm=np.array(algo),
        channels=np.stack([r["H"] for r in recs]), noise_power=np.array([r["s2"] for r in recs]),
        weights=np.stack([r["w"] for r in recs]), p_max=np.full(B, float(ck["p_max"])),
        init_precoders=np.stack([r["V0"] for r in recs]), opts=np.array(json.dumps(sk)),
        ref_status=np.array([r["status"] for r in recs], dtype=np.int32),
        ref_iterations=np.array([r["it"] for r in recs], dtype=np.int32),
        ref_wsr_bits=np.array([r["wsr"] for r in recs]),
        ref_converged=np.array([r["conv"] for r in recs]),
        ref_switch_iteration=np.array([r["sw"] for r in recs], dtype=np.int32),
        ref_residual=np.array([r["resid"] for r in recs]), ref_trace=trace,
        ref_final_precoders=np.stack([r["V"] for r in recs]), lstsq_calls=np.array(calls["lstsq"]))
    print(name, [r["it"] for r in recs], [round(r["wsr"], 4) for r in recs], "lstsq", calls["lstsq"])


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    want = set(sys.argv[1:])
    for n, (a, ck, sk, B) in CASES.items():
        if not want or n in want:
            run_case(n, a, ck, sk, B)
