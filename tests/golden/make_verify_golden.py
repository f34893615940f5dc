"""Fixtures for the verification oracles from the
UNMODIFIED reference (run here, where /root/reference exists):

  python tests/golden/make_verify_golden.py

  * verify/lemma_<name>.npz: a reference run_ammmse with record_iterates=True
    (channels, noise power, weights, bounds, every recorded (U, W, V) block
    iterate) and the reference check_lemma_bounds report of those iterates;
  * verify/harness_verify/summary.json: the reference run_experiment(spec, verify=True)
    of the harness fixture's spec (lemma-bound and finite-difference oracles).
"""
import json
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import wsrbeam  # noqa: E402
from wsrbeam import harness as H  # noqa: E402
from wsrbeam import verify as V  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_harness_golden import spec  # noqa: E402

CASES = {  # name: (SystemConfig kwargs, SolverOptions kwargs)
    "lemma_d1": (dict(M=8, N=2, K=3, d=1, p_max=10.0, snr_db=10.0, channel_seed=3, init_seed=4),
                 dict(gamma=0.02, omega=0.5, eps2=1e-4, max_iters=60)),
    "lemma_d2": (dict(M=12, N=2, K=3, d=2, p_max=30.0, snr_db=15.0, channel_seed=9, init_seed=2,
                      weights=(1.0, 0.7, 1.3)),
                 dict(gamma=0.01, omega=0.8, eps2=1e-5, max_iters=80)),
}


def lemma_case(name, ck, sk):
    cfg = wsrbeam.SystemConfig(**ck)
    ch = wsrbeam.generate_channels(cfg)
    ch = ch.with_noise_power(wsrbeam.compute_noise_power(ch, cfg.snr_db, cfg))
    opts = wsrbeam.SolverOptions(algorithm="ammmse", record_iterates=True, **sk)
    res = wsrbeam.run_ammmse(ch, cfg, opts)
    b = wsrbeam.compute_bounds(ch, cfg.weight_vector, cfg.p_max, ch.noise_power)
    rep = V.check_lemma_bounds(ch, res, b, cfg.weight_vector)
    its = res.iterates
    np.savez_compressed(
        os.path.join(HERE, "verify", f"{name}.npz"), channels=ch.channels, noise_power=ch.noise_power,
        weights=cfg.weight_vector, p_max=cfg.p_max,
        bounds=np.array([b.kappa, b.l_v, b.gamma_safe, b.ek_floor, b.alpha_bar]),
        U=np.stack([i.receivers.receivers for i in its]),
        W=np.stack([i.weight_matrices.weight_matrices for i in its]),
        V=np.stack([i.precoders.precoders for i in its]),
        V0=wsrbeam.init_precoders(cfg, wsrbeam.project_sum_power).precoders,
        opts=json.dumps(sk), iterations=res.iterations,
        ref_report=json.dumps(dict(name=rep.name, max_abs_error=rep.max_abs_error,
                                   max_rel_error=rep.max_rel_error, instances=rep.instances,
                                   passed=rep.passed, tolerance=rep.tolerance, detail=rep.detail)))
    print(name, res.iterations, rep)


if __name__ == "__main__":
    for n, (ck, sk) in CASES.items():
        lemma_case(n, ck, sk)
    out = os.path.join(HERE, "verify", "harness_verify")
    shutil.rmtree(out, ignore_errors=True)
    os.makedirs(out)
    H.run_experiment(spec(out), verify=True)
    for f in os.listdir(out):
        if f != "summary.json":
            os.remove(os.path.join(out, f))
    print(json.load(open(os.path.join(out, "summary.json")))["oracles"])
