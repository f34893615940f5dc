"""Exception types of the batched A-MMMSE engine.

Names and base classes follow the reference's error module
(`pkg/src/wsrbeam/errors.py:4-24`) so callers that catch
``ConfigError`` / ``IllConditionedWeightError`` / ``UnstableParametersError``
keep working when they switch solvers.  The engine itself never raises the
numerical ones from device code: each realization carries a status code
(:data:`STATUS_*`) and :func:`raise_for_status` maps a code back to the
exception the reference would have raised for that realization.
"""


class ConfigError(ValueError):
    """Invalid configuration, options or input arrays (ref errors.py:7-8)."""


class DegenerateChannelError(ValueError):
    """A channel matrix is identically zero (ref errors.py:11-12)."""


class ObjectiveDomainError(ValueError):
    """Objective evaluated at a singular / indefinite weight (ref errors.py:15-16)."""


class IllConditionedWeightError(RuntimeError):
    """Weight update argument ill conditioned or W not PD (ref errors.py:19-22,
    raised at solvers.py:243-252)."""


class UnstableParametersError(RuntimeError):
    """WSR fell below half its running max for 5 iterations (ref errors.py:23-24,
    raised at solvers.py:490-500)."""


class NativeLibraryError(RuntimeError):
    """The CUDA engine (libammmse.so) is missing or a CUDA call failed.

    There is no CPU fallback: the product path fails loudly instead."""


# Per-realization status codes written by the device engine (include/ammmse.h).
STATUS_OK = 0
STATUS_ILL_CONDITIONED = 1
STATUS_UNSTABLE = 2
STATUS_NONFINITE = 3

STATUS_NAMES = {
    STATUS_OK: "ok",
    STATUS_ILL_CONDITIONED: "IllConditionedWeightError",
    STATUS_UNSTABLE: "UnstableParametersError",
    STATUS_NONFINITE: "non-finite iterate",
}


def raise_for_status(status: int, gamma=None, omega=None) -> None:
    """Raise the exception the reference raises for a failed realization."""
    status = int(status)
    if status == STATUS_OK:
        return
    if status == STATUS_ILL_CONDITIONED:
        raise IllConditionedWeightError(
            "weight update is ill conditioned (cond > 1e12) or produced a non positive "
            "definite matrix; receivers are not MMSE-consistent with the precoders")
    if status == STATUS_UNSTABLE:
        raise UnstableParametersError(
            "weighted sum rate fell below half its running maximum for 5 consecutive "
            f"iterations: gamma={gamma!r}, omega={omega!r} are too aggressive for this instance")
    if status == STATUS_NONFINITE:
        raise UnstableParametersError("iterate became non-finite (gamma/omega too aggressive)")
    raise RuntimeError(f"unknown realization status {status}")
