"""CPU baseline timing of the oracle port — TEST / BENCH INFRASTRUCTURE ONLY.

Used by bench.py's ``cpu_baseline`` leg and by ``bench.py --impl reference``.
It times the reference algorithm restated in :mod:`oracle.ammmse_oracle`
(complex128 numpy/scipy, the reference's own arithmetic) the way the
reference harness runs a batch: one realization per task in a
ProcessPoolExecutor with one BLAS thread per worker and
workers = os.cpu_count() (pkg/src/wsrbeam/harness.py:482-490).  Worker
processes are spawned with OPENBLAS/OMP threads pinned to 1 before numpy is
imported (SURVEY.md §8(d) CPU path timing).
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import time
from concurrent.futures import ProcessPoolExecutor

_THREAD_VARS = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")


def _solve_task(task):
    import numpy as np

    from oracle import ammmse_oracle as orc

    H, s2, alpha, p_max, V0, opts = task
    o = orc.solve(np.asarray(H, dtype=np.complex128), s2, alpha, p_max,
                  np.asarray(V0, dtype=np.complex128), **opts)
    return (o["wsr_bits"], o["iterations"], o["status"], o["switch_iteration"],
            marginal(o["trace"][:, 8], opts.get("eps1", 0.1), opts.get("eps2", 1e-3)))


MARGIN = 1e-2  # |rel - eps| <= 1e-2 eps is a marginal stop / switch decision


def marginal(rel, eps1, eps2) -> bool:
    """True if any rel_change of the trace lies within ±1 % of eps1 or eps2,
    i.e. the iteration / switch count is not a robust comparison point."""
    import numpy as np

    rel = np.asarray(rel, dtype=np.float64)
    rel = rel[np.isfinite(rel)]
    near = lambda eps: math.isfinite(eps) and bool(np.any(np.abs(rel - eps) <= MARGIN * eps))
    return near(eps1) or near(eps2)


def _warm(_):
    return os.getpid()


class CpuPool:
    """Spawned process pool with single-threaded BLAS per worker."""

    def __init__(self, workers: int | None = None):
        self.workers = workers or os.cpu_count() or 1
        saved = {v: os.environ.get(v) for v in _THREAD_VARS}
        for v in _THREAD_VARS:
            os.environ[v] = "1"
        try:
            self.pool = ProcessPoolExecutor(max_workers=self.workers, mp_context=mp.get_context("spawn"))
            list(self.pool.map(_warm, range(self.workers)))  # start workers outside timing
            list(self.pool.map(_solve_task, [_tiny_task()] * self.workers))  # import numpy/scipy
        finally:
            for v, val in saved.items():
                if val is None:
                    os.environ.pop(v, None)
                else:
                    os.environ[v] = val

    def solve(self, tasks):
        return list(self.pool.map(_solve_task, tasks, chunksize=1))

    def close(self):
        self.pool.shutdown()


def _tiny_task():
    import numpy as np

    H = np.ones((1, 1, 2), dtype=np.complex128)
    V0 = np.ones((1, 2, 1), dtype=np.complex128) * 0.1
    return (H, 1.0, np.ones(1), 1.0, V0, dict(gamma=0.01, omega=0.0, eps2=1e-3, max_iters=2))


def tasks_from_batch(batch, idx, opts):
    """One task per realization; per-realization (gamma, omega) from the batch."""
    tasks = []
    for i in idx:
        o = dict(opts, gamma=float(batch.gamma[i]), omega=float(batch.omega[i]))
        tasks.append((batch.channels[i], float(batch.noise_power[i]), batch.weights[i],
                      float(batch.p_max[i]), batch.init_precoders[i], o))
    return tasks


def time_tasks(pool: CpuPool, tasks):
    t0 = time.perf_counter()
    out = pool.solve(tasks)
    return time.perf_counter() - t0, out
