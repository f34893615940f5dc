"""Harness fixtures from the UNMODIFIED reference (run here, where
/root/reference exists; the GPU box only reads the committed outputs).

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness_golden.py

Writes tests/golden/harness/: the reference run_experiment outputs
(summary.json + trace CSVs) of a small A-MMMSE spec with an SNR x K sweep, and
the sweep-point labels of a larger grid (sweep_labels.json)."""
import json
import os
import shutil
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import wsrbeam  # noqa: E402
from wsrbeam import harness as H  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness")


def spec(outdir):
    base = wsrbeam.SystemConfig(M=8, N=2, K=2, d=1, p_max=10.0, snr_db=10.0, weights=None,
                                channel_seed=5, init_seed=7)
    solver = wsrbeam.SolverOptions(algorithm="ammmse", gamma=0.02, omega=0.5, eps1=0.1,
                                   eps2=1e-4, max_iters=80)
    return H.ExperimentSpec(base=base, solver=solver, n_realizations=3,
                            sweep=(("snr_db", (5.0, 15.0)), ("K", (2.0, 3.0))),
                            parallel_workers=1, output_dir=outdir)


if __name__ == "__main__":
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    H.run_experiment(spec(OUT))
    os.remove(os.path.join(OUT, "timing.json"))
    big = H.ExperimentSpec(base=spec(OUT).base, solver=spec(OUT).solver, n_realizations=1,
                           sweep=(("M", (8.0, 16.0)), ("snr_db", (0.0, 12.5)), ("K", (2.0, 4.0))))
    labels = [lab for lab, _ in H._sweep_points(big)]
    json.dump({"labels": labels}, open(os.path.join(OUT, "sweep_labels.json"), "w"), indent=1)
    print(sorted(os.listdir(OUT)))
