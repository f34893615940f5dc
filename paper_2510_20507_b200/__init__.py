"""B200-native batched A-MMMSE engine (arXiv 2510.20507).

Drop-in for the reference's A-MMMSE path (`wsrbeam.run_ammmse`,
pkg/src/wsrbeam/solvers.py:540-550): same call signature and result layout,
executed for a whole batch of channel realizations by hand-written sm_100a
CUDA kernels (libammmse.so, C-ABI in include/ammmse.h).  No CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (
    ConfigError,
    DegenerateChannelError,
    IllConditionedWeightError,
    NativeLibraryError,
    ObjectiveDomainError,
    UnstableParametersError,
)
from .model import (
    ChannelSet,
    PrecoderSet,
    Stage,
    SystemConfig,
    compute_noise_power,
    generate_channels,
    init_precoders,
    project_sum_power,
)
from .solvers import (
    GAMMA_SAFE,
    STEP_DEFAULTS_BY_SNR,
    Algorithm,
    AmmmseEngine,
    BatchResult,
    IterationRecord,
    SolveResult,
    SolverOptions,
    default_step_parameters,
    resolve_step_parameters,
    run_ammmse,
    run_ammmse_batch,
    run_exact_batch,
    run_mmmse,
    run_wmmse,
    solve,
)

__all__ = [n for n in dir() if not n.startswith("_")]
