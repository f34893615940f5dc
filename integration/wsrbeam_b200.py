"""Reference-side binding of the B200 engine.

This is the module a ``wsrbeam`` maintainer would add to the reference code
base: a ctypes stub over the C-ABI of ``libammmse.so`` (include/ammmse.h)
that runs the reference's own types through the GPU engine, and an
``install()`` that swaps it into the reference's solver table
(``wsrbeam.solvers._DRIVERS``, solvers.py:553-557 — the seam the reference's
own test monkeypatches, test_harness.py:181).  After ``install()`` the stock
``wsrbeam.solve`` / ``wsrbeam.harness.run_experiment`` solve A-MMMSE (and
WMMSE / MMMSE through ``ammmse_solve_exact``) on the device.

No torch: device memory through the CUDA runtime (cudaMalloc / cudaMemcpy),
plain pointers and sizes across the ABI.  Tested against the unmodified
reference installed in ``baseline/_ref`` (tests/test_gpu_integration.py).
"""

from __future__ import annotations

import ctypes
import glob
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("AMMMSE_LIB", os.path.join(HERE, os.pardir, "paper_2510_20507_b200", "libammmse.so"))


def _cudart():
    cands = ["libcudart.so", "libcudart.so.12"] + sorted(glob.glob("/usr/local/cuda*/lib64/libcudart.so*"))
    try:  # the runtime torch ships, if present
        import nvidia.cuda_runtime as ncr  # type: ignore

        cands += glob.glob(os.path.join(os.path.dirname(ncr.__file__), "lib", "libcudart.so*"))
    except Exception:
        pass
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    raise OSError("libcudart not found")


class Dims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("M", ctypes.c_int32), ("N", ctypes.c_int32),
                ("K", ctypes.c_int32), ("d", ctypes.c_int32), ("dtype", ctypes.c_int32)]


class Problem(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("channels", "noise_power", "p_max", "weights",
                                              "init_precoders", "gamma", "omega")]


class Options(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("gamma_safe", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("omega", ctypes.c_double),
                ("eps1", ctypes.c_double), ("eps2", ctypes.c_double),
                ("latch_stage", ctypes.c_int32), ("cluster_size", ctypes.c_int32),
                ("h_placement", ctypes.c_int32), ("tensor_cores", ctypes.c_int32)]


class Result(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "final_precoders", "wsr_bits", "iterations", "converged", "stationarity_residual",
        "switch_iteration", "status", "gamma_used", "trace", "iter_receivers", "iter_weights",
        "iter_precoders")]


_lib = None
_rt = None


def _libs():
    global _lib, _rt
    if _lib is None:
        _lib = ctypes.CDLL(LIB)
        _rt = _cudart()
        _lib.ammmse_workspace_size.restype = ctypes.c_size_t
        _lib.ammmse_exact_workspace_size.restype = ctypes.c_size_t
        _lib.ammmse_error_string.restype = ctypes.c_char_p
    return _lib, _rt


class _Device:
    """Owned device allocations of one call (freed on exit)."""

    def __init__(self):
        self.ptrs = []

    def alloc(self, nbytes):
        _, rt = _libs()
        p = ctypes.c_void_p()
        if rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(max(int(nbytes), 16))) != 0:
            raise MemoryError("cudaMalloc failed")
        self.ptrs.append(p)
        return p

    def put(self, a):
        a = np.ascontiguousarray(a)
        p = self.alloc(a.nbytes)
        _libs()[1].cudaMemcpy(p, a.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(a.nbytes), 1)
        return p

    def get(self, p, shape, dtype):
        out = np.empty(shape, dtype=dtype)
        _libs()[1].cudaMemcpy(out.ctypes.data_as(ctypes.c_void_p), p, ctypes.c_size_t(out.nbytes), 2)
        return out

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        rt = _libs()[1]
        rt.cudaDeviceSynchronize()
        for p in self.ptrs:
            rt.cudaFree(p)


def _solve(channels, config, options, algorithm):
    """One realization through the C-ABI; returns a wsrbeam SolveResult or
    raises the reference's exceptions for failed solves."""
    import wsrbeam
    from wsrbeam import solvers as ws

    lib, _ = _libs()
    if channels.noise_power is None:
        raise wsrbeam.ConfigError("channels carry no noise power; call compute_noise_power first")
    K, N, M, d = config.K, config.N, config.M, config.d
    T = options.max_iters
    H = channels.channels.astype(np.complex128)[None]
    V0 = ws.init_precoders(config, ws.project_sum_power).precoders.astype(np.complex128)[None]
    dims = Dims(1, M, N, K, d, 1)  # AMMMSE_COMPLEX128 (the reference's precision)
    gamma, omega, safe = 0.0, 0.0, 0
    if algorithm == 0:  # A-MMMSE: resolve (gamma, omega) exactly as the reference does
        b = wsrbeam.compute_bounds(channels, config.weight_vector, config.p_max, channels.noise_power)
        gamma, omega = ws.resolve_step_parameters(options, config.snr_db, b)
    opts = Options(float(gamma), safe, int(T), float(omega), float(options.eps1), float(options.eps2),
                   int(options.latch_stage), 0, 0, 0)
    with _Device() as dev:
        prob = Problem(dev.put(H), dev.put(np.array([channels.noise_power])),
                       dev.put(np.array([config.p_max])), dev.put(config.weight_vector[None]),
                       dev.put(V0), None, None)
        f = lambda shape, dt: dev.alloc(int(np.prod(shape)) * np.dtype(dt).itemsize)
        rv = dict(final_precoders=f((1, K, M, d), np.complex128), wsr_bits=f((1,), np.float64),
                  iterations=f((1,), np.int32), converged=f((1,), np.uint8),
                  stationarity_residual=f((1,), np.float64), switch_iteration=f((1,), np.int32),
                  status=f((1,), np.int32), gamma_used=f((1,), np.float64),
                  trace=f((1, T, 9), np.float64))
        res = Result(**rv)
        if algorithm == 0:
            wsb = lib.ammmse_workspace_size(ctypes.byref(dims))
            ws_ptr = dev.alloc(wsb)
            rc = lib.ammmse_solve(ctypes.byref(dims), ctypes.byref(prob), ctypes.byref(opts),
                                  ctypes.byref(res), ws_ptr, ctypes.c_size_t(wsb), None)
        else:
            wsb = lib.ammmse_exact_workspace_size(ctypes.byref(dims))
            ws_ptr = dev.alloc(wsb)
            rc = lib.ammmse_solve_exact(ctypes.byref(dims), ctypes.byref(prob), ctypes.byref(opts),
                                        ctypes.c_int(algorithm), ctypes.c_double(options.bisect_tol),
                                        ctypes.c_int(options.bisect_max), ctypes.byref(res), ws_ptr,
                                        ctypes.c_size_t(wsb), None)
        if rc != 0:
            raise wsrbeam.ConfigError(lib.ammmse_error_string(rc).decode())
        status = int(dev.get(rv["status"], (1,), np.int32)[0])
        n = int(dev.get(rv["iterations"], (1,), np.int32)[0])
        trace = dev.get(rv["trace"], (1, T, 9), np.float64)[0, :n]
        V = dev.get(rv["final_precoders"], (1, K, M, d), np.complex128)[0]
        conv = bool(dev.get(rv["converged"], (1,), np.uint8)[0])
        resid = float(dev.get(rv["stationarity_residual"], (1,), np.float64)[0])
        sw = int(dev.get(rv["switch_iteration"], (1,), np.int32)[0])
    if status == 2:  # solvers.py:496-500
        raise wsrbeam.UnstableParametersError(
            f"weighted sum rate fell below half its running maximum for 5 consecutive iterations: "
            f"gamma={gamma!r}, omega={omega!r} are too aggressive for this instance")
    if status in (1, 3):  # solvers.py:243-252
        raise wsrbeam.IllConditionedWeightError("weight update ill-conditioned (device status "
                                                f"{status})")
    records = tuple(ws.IterationRecord(
        t=int(r[0]), wsr_bits=float(r[1]), f_value=float(r[2]), total_power=float(r[3]),
        stage=wsrbeam.Stage.WEIGHTED if r[4] > 0.5 else wsrbeam.Stage.UNWEIGHTED,
        f_after_u=float(r[5]), f_after_w=float(r[6]), f_after_v=float(r[7]),
        rel_change=float(r[8]) if math.isfinite(r[8]) else math.inf) for r in trace)
    return ws.SolveResult(final_precoders=wsrbeam.PrecoderSet(V), trace=records, iterations=n,
                          converged=conv, stationarity_residual=resid,
                          switch_iteration=None if sw < 0 else sw)


def run_ammmse_b200(channels, config, options):
    """Same contract as wsrbeam.run_ammmse (solvers.py:540-550), on the device."""
    from wsrbeam.solvers import Algorithm

    if options.algorithm is not Algorithm.AMMMSE:
        import wsrbeam

        raise wsrbeam.ConfigError("options.algorithm must be AMMMSE")
    return _solve(channels, config, options, 0)


def run_wmmse_b200(channels, config, options):
    """Same contract as wsrbeam.run_wmmse (solvers.py:521-527), on the device."""
    return _solve(channels, config, options, 1)


def run_mmmse_b200(channels, config, options):
    """Same contract as wsrbeam.run_mmmse (solvers.py:530-537), on the device."""
    return _solve(channels, config, options, 2)


def install(algorithms=("ammmse", "wmmse", "mmmse")):
    """Swap the device drivers into wsrbeam.solvers._DRIVERS (solvers.py:553-557).
    Returns the previous table so callers can restore it."""
    from wsrbeam import solvers as ws

    prev = dict(ws._DRIVERS)
    table = {"ammmse": (ws.Algorithm.AMMMSE, run_ammmse_b200),
             "wmmse": (ws.Algorithm.WMMSE, run_wmmse_b200),
             "mmmse": (ws.Algorithm.MMMSE, run_mmmse_b200)}
    for a in algorithms:
        alg, fn = table[a]
        ws._DRIVERS[alg] = fn
    return prev
