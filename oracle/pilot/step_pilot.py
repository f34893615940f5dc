"""Pilot study for the (gamma, omega) of each BASELINE workload — TEST/DESIGN
INFRASTRUCTURE (runs the CPU oracle only).

Rule: the largest gamma (omega = 0.8) whose weighted-stage
WSR never decreases on a pilot set, checked also for sensitivity: the final
WSR under a 1e-7 relative (fp32-level) perturbation of H must move by less
than 1e-5 relative and the iteration count must not change.
Usage: python oracle/pilot/step_pilot.py <workload> <gamma> [<gamma> ...]
"""
import os, sys, json
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from concurrent.futures import ProcessPoolExecutor
from oracle import ammmse_oracle as orc
from paper_2510_20507_b200.inputs import WORKLOADS


def run(args):
    name, gamma, r, max_iters = args
    w = WORKLOADS[name]
    b = w.batch(B=1, seed0=r)
    H = b.channels[0].astype(np.complex128)
    V0 = b.init_precoders[0].astype(np.complex128)
    out = []
    for pert in (0.0, 1e-7):
        Hp = H
        if pert:
            g = np.random.default_rng(1000 + r)
            Hp = H * (1 + pert * g.standard_normal(H.shape))
        o = orc.solve(Hp, 1.0, b.weights[0], w.p_max, V0, gamma, w.omega, eps1=w.eps1,
                      eps2=w.eps2, max_iters=max_iters)
        tr = o["trace"]
        wsr = tr[:, 1]
        st = tr[:, 4]
        dec = 0.0
        for t in range(1, len(wsr)):
            if st[t] > 0.5 and st[t - 1] > 0.5:
                dec = max(dec, (wsr[t - 1] - wsr[t]) / abs(wsr[t - 1]))
        out.append(dict(wsr=o["wsr_bits"], it=o["iterations"], conv=bool(o["converged"]),
                        sw=o["switch_iteration"], status=o["status"], maxdec=dec))
    a, p = out
    return dict(workload=name, gamma=gamma, r=r, wsr=a["wsr"], iters=a["it"], conv=a["conv"],
                switch=a["sw"], status=a["status"], maxdec=a["maxdec"],
                sens=abs(a["wsr"] - p["wsr"]) / abs(a["wsr"]), it_pert=p["it"])


if __name__ == "__main__":
    name = sys.argv[1]
    gammas = [float(g) for g in sys.argv[2:]]
    seeds = int(os.environ.get("PILOT_SEEDS", "4"))
    mi = int(os.environ.get("PILOT_MAX_ITERS", WORKLOADS[name].max_iters))
    jobs = [(name, g, r, mi) for g in gammas for r in range(seeds)]
    with ProcessPoolExecutor(max_workers=int(os.environ.get("PILOT_WORKERS", "8"))) as pool:
        for res in pool.map(run, jobs):
            print(json.dumps(res), flush=True)
