"""fp32 engine vs fp64 reference: deviation of rel_change along the stored traces
(c64 golden fixtures), to calibrate the marginal band of the iteration-count test."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import golden_util as gu
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch
for name in gu.names():
    g = gu.load(name)
    if not gu.is_c64(g):
        continue
    opts = SolverOptions(algorithm="ammmse", gamma=g["opt_gamma"], omega=g["opt_omega"], **g["opt"])
    r = run_ammmse_batch(g["channels"], g["noise_power"], g["p_max"], g["weights"],
                         g["init_precoders"], opts, snr_db=float(g["snr_db"]), record_trace=True)
    eps = g["opt"]["eps2"]
    tr = g["ref_trace"]
    for b in range(tr.shape[0]):
        n = int(min(g["ref_iterations"][b], r.iterations[b]))
        rr, rg = tr[b, 1:n, 8], r.trace[b, 1:n, 8]
        near = rr < 10 * eps
        dev = np.abs(rg[near] - rr[near]) / eps if near.any() else np.array([0.0])
        print(f"{name} b={b} iters ref={int(g['ref_iterations'][b])} gpu={int(r.iterations[b])} "
              f"max|rel_gpu-rel_ref|/eps2 (rel<10eps2) = {dev.max():.3g}  median {np.median(dev):.3g}")
