# tiny sweep128-shape solve (cluster C=1 spec kernel) for crash triage
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2510_20507_b200 import SolverOptions, run_ammmse_batch
from paper_2510_20507_b200.inputs import build_batch
M, K = int(sys.argv[1]), int(sys.argv[2])
b = build_batch(M, 2, K, 2, 2, p_max=30.0, weights="uniform", dtype=np.complex64, seed0=1)
opts = SolverOptions(algorithm="ammmse", gamma=0.002, omega=0.8, eps2=1e-5, max_iters=int(sys.argv[3]))
r = run_ammmse_batch(b.channels, b.noise_power, b.p_max, b.weights, b.init_precoders, opts)
print("ok", r.iterations, r.wsr_bits, r.status)
