"""ctypes binding of the in-tree CUDA engine ``libammmse.so`` (include/ammmse.h).

The library is built by ``__graft_entry__.build()`` / ``make`` into this
package directory.  There is no CPU fallback: :func:`lib` raises
:class:`NativeLibraryError` when the library is missing.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

from .errors import NativeLibraryError

LIB_PATH = pathlib.Path(__file__).resolve().with_name("libammmse.so")

ABI_VERSION = 2
ALGO_WMMSE = 1
ALGO_MMMSE = 2
COMPLEX64 = 0
COMPLEX128 = 1
TRACE_FIELDS = 9
BOUND_FIELDS = 5

OK = 0
ERR_INVALID = -1
ERR_UNSUPPORTED = -2
ERR_WORKSPACE = -3
ERR_CUDA = -4

# every symbol include/ammmse.h declares
EXPORTED_SYMBOLS = (
    "ammmse_abi_version",
    "ammmse_check_dims",
    "ammmse_workspace_size",
    "ammmse_workspace_size_opts",
    "ammmse_solve",
    "ammmse_bounds",
    "ammmse_error_string",
    "ammmse_phase_profile",
    "ammmse_plan_info",
    "ammmse_exact_workspace_size",
    "ammmse_solve_exact",
    "ammmse_generate_iid",
)


class AmmmseDims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("M", ctypes.c_int32), ("N", ctypes.c_int32),
                ("K", ctypes.c_int32), ("d", ctypes.c_int32), ("dtype", ctypes.c_int32)]


class AmmmseProblem(ctypes.Structure):
    _fields_ = [("channels", ctypes.c_void_p), ("noise_power", ctypes.c_void_p),
                ("p_max", ctypes.c_void_p), ("weights", ctypes.c_void_p),
                ("init_precoders", ctypes.c_void_p), ("gamma", ctypes.c_void_p),
                ("omega", ctypes.c_void_p)]


class AmmmseOptions(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("gamma_safe", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("omega", ctypes.c_double),
                ("eps1", ctypes.c_double), ("eps2", ctypes.c_double),
                ("latch_stage", ctypes.c_int32), ("cluster_size", ctypes.c_int32),
                ("h_placement", ctypes.c_int32), ("tensor_cores", ctypes.c_int32)]


class AmmmseResult(ctypes.Structure):
    _fields_ = [("final_precoders", ctypes.c_void_p), ("wsr_bits", ctypes.c_void_p),
                ("iterations", ctypes.c_void_p), ("converged", ctypes.c_void_p),
                ("stationarity_residual", ctypes.c_void_p), ("switch_iteration", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("gamma_used", ctypes.c_void_p),
                ("trace", ctypes.c_void_p), ("iter_receivers", ctypes.c_void_p),
                ("iter_weights", ctypes.c_void_p), ("iter_precoders", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libammmse.so once (raises NativeLibraryError if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("AMMMSE_LIB", str(LIB_PATH))
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"CUDA engine not built: {path} is missing (run __graft_entry__.build() or `make`)")
        try:
            h = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        h.ammmse_generate_iid.restype = ctypes.c_int
        h.ammmse_generate_iid.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.c_ulonglong,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        h.ammmse_plan_info.restype = ctypes.c_int
        h.ammmse_plan_info.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.POINTER(AmmmseOptions),
                                       ctypes.POINTER(ctypes.c_int)]
        h.ammmse_phase_profile.restype = ctypes.c_int
        h.ammmse_phase_profile.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                           ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]
        h.ammmse_abi_version.restype = ctypes.c_int
        h.ammmse_abi_version.argtypes = []
        h.ammmse_check_dims.restype = ctypes.c_int
        h.ammmse_check_dims.argtypes = [ctypes.POINTER(AmmmseDims)]
        h.ammmse_workspace_size.restype = ctypes.c_size_t
        h.ammmse_workspace_size.argtypes = [ctypes.POINTER(AmmmseDims)]
        h.ammmse_workspace_size_opts.restype = ctypes.c_size_t
        h.ammmse_workspace_size_opts.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.POINTER(AmmmseOptions)]
        h.ammmse_solve.restype = ctypes.c_int
        h.ammmse_solve.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.POINTER(AmmmseProblem),
                                   ctypes.POINTER(AmmmseOptions), ctypes.POINTER(AmmmseResult),
                                   ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        h.ammmse_exact_workspace_size.restype = ctypes.c_size_t
        h.ammmse_exact_workspace_size.argtypes = [ctypes.POINTER(AmmmseDims)]
        h.ammmse_solve_exact.restype = ctypes.c_int
        h.ammmse_solve_exact.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.POINTER(AmmmseProblem),
                                         ctypes.POINTER(AmmmseOptions), ctypes.c_int, ctypes.c_double,
                                         ctypes.c_int, ctypes.POINTER(AmmmseResult), ctypes.c_void_p,
                                         ctypes.c_size_t, ctypes.c_void_p]
        h.ammmse_bounds.restype = ctypes.c_int
        h.ammmse_bounds.argtypes = [ctypes.POINTER(AmmmseDims), ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p]
        h.ammmse_error_string.restype = ctypes.c_char_p
        h.ammmse_error_string.argtypes = [ctypes.c_int]
        if h.ammmse_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libammmse.so ABI version mismatch; rebuild")
        _lib = h
        return h


def error_string(code: int) -> str:
    return lib().ammmse_error_string(int(code)).decode(errors="replace")


PLAN_FIELDS = ("cluster", "h_resident", "vold_global", "stage_bytes", "tensor_cores", "smem_bytes",
               "threads", "specialised")


def plan_info(dims: AmmmseDims, options: AmmmseOptions | None = None) -> dict:
    """The engine configuration ammmse_solve would launch (ammmse_plan_info)."""
    info = (ctypes.c_int * 8)()
    rc = lib().ammmse_plan_info(dims, options or AmmmseOptions(), info)
    if rc != 0:
        raise NativeLibraryError(f"ammmse_plan_info: {error_string(rc)}")
    return dict(zip(PLAN_FIELDS, list(info)))
