# per-realization comparison of the TC and FFMA engines against the large golden
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import golden_util as gu
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch
g = gu.load(sys.argv[1] if len(sys.argv) > 1 else "large")
opts = SolverOptions(algorithm="ammmse", gamma=g["opt_gamma"], omega=g["opt_omega"], **g["opt"])
for tc in (1, 2):
    r = run_ammmse_batch(g["channels"], g["noise_power"], g["p_max"], g["weights"], g["init_precoders"], opts,
                         tensor_cores=tc)
    rel = np.abs(r.wsr_bits - g["ref_wsr_bits"]) / np.abs(g["ref_wsr_bits"])
    bad = np.argsort(-rel)[:4]
    print("tc", tc, "max rel", rel.max(), "worst", [(int(i), float(rel[i]), int(r.iterations[i]), int(g["ref_iterations"][i])) for i in bad],
          "iter mismatches", int((r.iterations != g["ref_iterations"]).sum()))
