"""Loading helpers for the golden fixtures produced by tests/golden/make_golden.py
(unmodified reference outputs on seeded inputs)."""

import glob
import math
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
# fixtures the CPU oracle needs minutes for; their oracle pin runs with AMMMSE_SLOW=1
SLOW = {"large", "massive", "sweep256", "sweep512", "edge_safe_tight", "medium_snr20_long",
        "medium_snr30_long"}


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    g = {k: z[k] for k in z.files}
    wl = str(g.get("workload", ""))
    if wl:  # inputs regenerated from the seeds (bit-identical to what the reference saw)
        from paper_2510_20507_b200.inputs import WORKLOADS

        b = WORKLOADS[wl].batch(B=int(g["batch_size"]))
        g.update(channels=b.channels, noise_power=b.noise_power, p_max=b.p_max, weights=b.weights,
                 init_precoders=b.init_precoders)
    gam = float(g["gamma"])
    g["opt_gamma"] = None if math.isnan(gam) else ("safe" if gam == -1.0 else gam)
    om = float(g["omega"])
    g["opt_omega"] = None if math.isnan(om) else om
    g["opt"] = dict(eps1=float(g["eps1"]), eps2=float(g["eps2"]), max_iters=int(g["max_iters"]),
                    latch_stage=bool(g["latch_stage"]))
    g["name"] = name
    return g


def is_c64(g):
    return g["channels"].dtype == np.complex64


def nonmarginal(g, margin=1e-2):
    """Realizations whose stored trace keeps every rel_change outside
    [eps(1-margin), eps(1+margin)] for eps in {eps1, eps2}.
    Realizations without a stored trace count as non-marginal."""
    B = g["ref_iterations"].shape[0]
    ok = np.ones(B, dtype=bool)
    # every realization's rel_change when the fixture stores it, else the traced ones
    rels = g["ref_rel"] if "ref_rel" in g else g["ref_trace"][:, :, 8]
    for b in range(min(B, rels.shape[0])):
        n = int(g["ref_iterations"][b])
        rel = rels[b, : max(n, 0)]
        for eps in (g["opt"]["eps1"], g["opt"]["eps2"]):
            if np.isfinite(eps):
                fin = np.isfinite(rel)
                if np.any(np.abs(rel[fin] - eps) <= margin * eps):
                    ok[b] = False
    return ok
