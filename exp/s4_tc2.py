"""tc2 engine on the large golden: deferred mode (no trace) vs inline mode (trace) vs the reference."""
import sys
import numpy as np
sys.path.insert(0, "tests")
import golden_util as gu
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch

g = gu.load("large")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
opts = SolverOptions(algorithm="ammmse", gamma=g["opt_gamma"], omega=g["opt_omega"], **g["opt"])
out = {}
for trace in (False, True):
    r = run_ammmse_batch(g["channels"][:n], g["noise_power"][:n], g["p_max"][:n], g["weights"][:n],
                         g["init_precoders"][:n], opts, snr_db=float(g["snr_db"]), record_trace=trace)
    out[trace] = r
    rel = np.abs(r.wsr_bits - g["ref_wsr_bits"][:n]) / np.abs(g["ref_wsr_bits"][:n])
    print(f"trace={trace}: status {np.unique(r.status)} max WSR rel {rel.max():.3e} median {np.median(rel):.3e}")
    print("  iters    ", r.iterations[:16])
    print("  ref iters", g["ref_iterations"][:16])
    print("  converged", r.converged[:16].astype(int), "ref", g["ref_converged"][:16].astype(int))
    print("  residual ", r.stationarity_residual[:4], "ref", g["ref_residual"][:4])
    V = r.final_precoders.astype(np.complex128)
    print("  power", np.sum(np.abs(V) ** 2, axis=(1, 2, 3))[:4])
a, b = out[False], out[True]
print("deferred vs inline: iter mismatches", int((a.iterations != b.iterations).sum()),
      "max wsr rel", float(np.max(np.abs(a.wsr_bits - b.wsr_bits) / np.abs(b.wsr_bits))),
      "V max abs diff", float(np.max(np.abs(a.final_precoders - b.final_precoders))),
      "residual max rel", float(np.nanmax(np.abs(a.stationarity_residual - b.stationarity_residual) / np.abs(b.stationarity_residual))),
      "switch mismatches", int((a.switch_iteration != b.switch_iteration).sum()))
