"""Drop-in A-MMMSE driver backed by the B200 engine.

Mirrors the reference solver interface for the A-MMMSE path
(`pkg/src/wsrbeam/solvers.py`): ``SolverOptions`` (:88-136),
``IterationRecord`` (:139-156), ``SolveResult`` (:174-182),
``default_step_parameters`` / ``resolve_step_parameters`` (:185-207),
``run_ammmse`` (:540-550) and ``solve`` (:560-562) keep their names,
argument meaning and error behaviour.  The loop itself runs on the GPU
(libammmse.so) for a whole batch of realizations per call:

  * :func:`run_ammmse`        one realization, reference signature, raises the
                              reference's exceptions;
  * :func:`run_ammmse_batch`  B realizations (SoA in, SoA out, per-realization
                              status codes instead of exceptions, as the
                              reference harness records them, harness.py:277-278);
  * :class:`AmmmseEngine`     device-resident entry point (torch tensors in
                              HBM, stream-ordered) used by the benchmark.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np

from . import _native
from .errors import ConfigError, NativeLibraryError, raise_for_status
from .model import (ChannelSet, PrecoderSet, ReceiverSet, Stage, SystemConfig, WeightMatrixSet,
                    init_precoders, project_sum_power)

GAMMA_SAFE = "safe"

#: (omega, gamma) per SNR in dB, paper Table I (ref solvers.py:61-69)
STEP_DEFAULTS_BY_SNR: dict = {
    -10.0: (0.6, 0.4),
    -5.0: (0.6, 0.4),
    0.0: (0.6, 0.4),
    5.0: (0.6, 0.4),
    10.0: (0.8, 0.05),
    15.0: (0.8, 0.005),
    20.0: (0.8, 0.003),
}


class Algorithm(Enum):
    WMMSE = "wmmse"
    MMMSE = "mmmse"
    AMMMSE = "ammmse"

    @classmethod
    def from_name(cls, name: str) -> "Algorithm":
        key = str(name).strip().lower()
        for a in cls:
            if a.value == key:
                return a
        raise ConfigError(f"unknown algorithm {name!r}; expected one of {[a.value for a in cls]}")


@dataclass(frozen=True)
class SolverOptions:
    """Options of one solve (ref solvers.py:88-136, same fields and checks).

    ``bisect_*`` belong to the exact drivers and are accepted but unused by
    A-MMMSE; ``record_iterates`` keeps every (U, W, V_new) block iterate in
    device buffers of (B, max_iters, ...) complex128 (meant for small B: the
    bound scans of verify.py).
    """

    algorithm: Algorithm = Algorithm.WMMSE
    gamma: float | str | None = None
    omega: float | None = None
    eps1: float = 0.1
    eps2: float = 0.001
    max_iters: int = 1000
    bisect_tol: float = 1e-4
    bisect_max: int = 100
    record_iterates: bool = False
    latch_stage: bool = True

    def __post_init__(self) -> None:
        if not isinstance(self.algorithm, Algorithm):
            object.__setattr__(self, "algorithm", Algorithm.from_name(self.algorithm))
        g = self.gamma
        if isinstance(g, str):
            if g != GAMMA_SAFE:
                raise ConfigError(f"gamma must be positive, {GAMMA_SAFE!r}, or None; got {g!r}")
        elif g is not None:
            gf = float(g)
            if not (math.isfinite(gf) and gf > 0):
                raise ConfigError(f"gamma must be positive, got {g!r}")
            object.__setattr__(self, "gamma", gf)
        if self.omega is not None:
            om = float(self.omega)
            if not (0.0 <= om < 1.0):
                raise ConfigError(f"omega must lie in [0, 1), got {self.omega!r}")
            object.__setattr__(self, "omega", om)
        if not (self.eps1 > 0):
            raise ConfigError(f"eps1 must be positive, got {self.eps1!r}")
        if not (self.eps2 > 0 and math.isfinite(self.eps2)):
            raise ConfigError(f"eps2 must be positive and finite, got {self.eps2!r}")
        if self.eps2 > self.eps1:
            raise ConfigError(f"eps2 ({self.eps2}) must not exceed eps1 ({self.eps1})")
        if self.max_iters < 1:
            raise ConfigError("max_iters must be at least 1")
        if not (self.bisect_tol > 0):
            raise ConfigError("bisect_tol must be positive")
        if self.bisect_max < 1:
            raise ConfigError("bisect_max must be at least 1")


@dataclass(frozen=True)
class IterationRecord:
    """One completed iteration (ref solvers.py:139-156)."""

    t: int
    wsr_bits: float
    f_value: float
    total_power: float
    stage: Stage
    f_after_u: float
    f_after_w: float
    f_after_v: float
    rel_change: float


class BlockIterate(NamedTuple):
    """Full block variables of one completed iteration (ref solvers.py:159-164)."""

    receivers: ReceiverSet
    weight_matrices: WeightMatrixSet
    precoders: PrecoderSet


@dataclass(frozen=True, eq=False)
class SolveResult:
    """Result of one realization (ref solvers.py:174-182)."""

    final_precoders: PrecoderSet
    trace: tuple
    iterations: int
    converged: bool
    stationarity_residual: float
    switch_iteration: int | None = None
    iterates: tuple | None = None


def default_step_parameters(snr_db: float) -> tuple[float, float]:
    """(omega, gamma) at the nearest tabulated SNR, ties toward the higher SNR
    (ref solvers.py:185-193)."""
    snr = float(snr_db)
    best = None
    for s in STEP_DEFAULTS_BY_SNR:
        key = (abs(s - snr), -s)
        if best is None or key < best[0]:
            best = (key, s)
    return STEP_DEFAULTS_BY_SNR[best[1]]


def resolve_step_parameters(options: SolverOptions, snr_db: float, bounds=None):
    """Concrete (gamma, omega) (ref solvers.py:196-207).

    ``gamma == "safe"`` resolves to ``bounds.gamma_safe`` when a bounds object
    is given, else to the string sentinel (the engine resolves it on device
    per realization)."""
    omega_default, gamma_default = default_step_parameters(snr_db)
    omega = omega_default if options.omega is None else options.omega
    if options.gamma is None:
        gamma = gamma_default
    elif options.gamma == GAMMA_SAFE:
        gamma = bounds.gamma_safe if bounds is not None else GAMMA_SAFE
    else:
        gamma = float(options.gamma)
    return gamma, omega


# ---------------------------------------------------------------------------
# device engine
# ---------------------------------------------------------------------------


def _torch():
    import torch

    return torch


@dataclass
class BatchResult:
    """SoA result of a batched solve (device or host arrays).

    Field order follows SolveResult; ``status`` holds AMMMSE_STATUS_* codes
    (0 ok, 1 IllConditionedWeightError, 2 UnstableParametersError, 3 non-finite)
    and ``switch_iteration`` uses -1 for None."""

    final_precoders: object
    wsr_bits: object
    iterations: object
    converged: object
    stationarity_residual: object
    switch_iteration: object
    status: object
    gamma_used: object
    trace: object = None
    omega: float = 0.0
    # recorded iterates (record_iterates): (U (B,T,K,N,d), W (B,T,K,d,d), V (B,T,K,M,d)) complex128
    iterates: tuple | None = None

    def to_host(self) -> "BatchResult":
        def h(x):
            if x is None:
                return None
            return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)

        return BatchResult(*(h(getattr(self, f)) for f in (
            "final_precoders", "wsr_bits", "iterations", "converged", "stationarity_residual",
            "switch_iteration", "status", "gamma_used", "trace")), omega=self.omega,
            iterates=None if self.iterates is None else tuple(h(x) for x in self.iterates))

    def solve_result(self, i: int) -> SolveResult:
        """Per-realization SolveResult view (needs a host result with a trace)."""
        h = self if isinstance(self.wsr_bits, np.ndarray) else self.to_host()
        n = int(h.iterations[i])
        records = ()
        if h.trace is not None:
            rows = h.trace[i, :n]
            records = tuple(IterationRecord(
                t=int(row[0]), wsr_bits=float(row[1]), f_value=float(row[2]),
                total_power=float(row[3]), stage=Stage.WEIGHTED if row[4] > 0.5 else Stage.UNWEIGHTED,
                f_after_u=float(row[5]), f_after_w=float(row[6]), f_after_v=float(row[7]),
                rel_change=float(row[8])) for row in rows)
        sw = int(h.switch_iteration[i])
        iterates = None
        if h.iterates is not None:
            U, W, V = h.iterates
            stages = [records[t].stage if records else Stage.WEIGHTED for t in range(n)]
            iterates = tuple(BlockIterate(
                ReceiverSet(U[i, t]),
                WeightMatrixSet(W[i, t], stages[t]) if stages[t] is Stage.WEIGHTED
                else WeightMatrixSet.identity(W.shape[2], W.shape[3]),
                PrecoderSet(V[i, t])) for t in range(n))
        return SolveResult(
            final_precoders=PrecoderSet(h.final_precoders[i]),
            trace=records,
            iterations=n,
            converged=bool(h.converged[i]),
            stationarity_residual=float(h.stationarity_residual[i]),
            switch_iteration=None if sw < 0 else sw,
            iterates=iterates,
        )


class AmmmseEngine:
    """Stream-ordered batched A-MMMSE on one CUDA device.

    Inputs are torch tensors already in HBM: channels (B, K, N, M) and
    init_precoders (B, K, M, d), both complex64 or both complex128;
    noise_power, p_max (B,) and weights (B, K) float64.  All outputs are
    allocated on the same device.  The call is asynchronous on ``stream``
    (default: torch's current stream)."""

    def __init__(self, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise NativeLibraryError("the A-MMMSE engine needs a CUDA device (no CPU fallback)")
        self.lib = _native.lib()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.type != "cuda":
            raise ConfigError(f"the engine runs on a CUDA device, got {dev}")
        self.device = dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = {}

    def dims(self, channels, init_precoders) -> _native.AmmmseDims:
        torch = _torch()
        if channels.dim() != 4 or init_precoders.dim() != 4:
            raise ConfigError("channels must be (B, K, N, M) and init_precoders (B, K, M, d)")
        B, K, N, M = channels.shape
        if init_precoders.shape[:3] != (B, K, M):
            raise ConfigError(f"init_precoders shape {tuple(init_precoders.shape)} does not match "
                              f"channels {tuple(channels.shape)}")
        if channels.dtype != init_precoders.dtype:
            raise ConfigError("channels and init_precoders must share a complex dtype")
        if channels.dtype == torch.complex64:
            dt = _native.COMPLEX64
        elif channels.dtype == torch.complex128:
            dt = _native.COMPLEX128
        else:
            raise ConfigError(f"unsupported dtype {channels.dtype}; use complex64 or complex128")
        return _native.AmmmseDims(B, M, N, K, int(init_precoders.shape[3]), dt)

    def check(self, dims) -> None:
        rc = self.lib.ammmse_check_dims(dims)
        if rc != 0:
            raise ConfigError(f"shape (M={dims.M}, N={dims.N}, K={dims.K}, d={dims.d}) not supported "
                              f"by the engine: {_native.error_string(rc)}")

    def _workspace(self, nbytes: int, stream=None):
        """Engine-owned workspace, one per stream (it holds the persistent
        kernel's work counter, so two solves in flight on different streams
        must not share it).  Growing it first waits for the stream's pending
        work on the old buffer."""
        torch = _torch()
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        if not isinstance(self._ws, dict):
            self._ws = {}
        key = int(stream.cuda_stream)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            if ws is not None:
                stream.synchronize()
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def _check_out(self, out, init_precoders, B: int, max_iters: int) -> None:
        """A caller-supplied result must match this call (the kernel writes B
        entries of every field and (B, max_iters, 9) trace rows)."""
        torch = _torch()
        want = {"final_precoders": (tuple(init_precoders.shape), init_precoders.dtype),
                "wsr_bits": ((B,), torch.float64), "iterations": ((B,), torch.int32),
                "converged": ((B,), torch.uint8), "stationarity_residual": ((B,), torch.float64),
                "switch_iteration": ((B,), torch.int32), "status": ((B,), torch.int32),
                "gamma_used": ((B,), torch.float64)}
        for f, (shape, dt) in want.items():
            t = getattr(out, f)
            if t is None:
                continue
            if (tuple(t.shape) != shape or t.dtype != dt or t.device != self.device
                    or not t.is_contiguous()):
                raise ConfigError(f"out.{f} must be a contiguous {dt} tensor of shape {shape} on "
                                  f"{self.device}")
        if out.iterates is not None:
            K, M, d = init_precoders.shape[1], init_precoders.shape[2], init_precoders.shape[3]
            U, W, V = out.iterates
            N = U.shape[3] if U.dim() == 5 else -1
            for nm, t, shape in (("U", U, (B, max_iters, K, N, d)), ("W", W, (B, max_iters, K, d, d)),
                                 ("V", V, (B, max_iters, K, M, d))):
                if (tuple(t.shape) != shape or t.dtype != torch.complex128 or t.device != self.device
                        or not t.is_contiguous()):
                    raise ConfigError(f"out.iterates {nm} must be a contiguous complex128 tensor of "
                                      f"shape {shape}")
        if out.trace is not None:
            shape = (B, max_iters, _native.TRACE_FIELDS)
            if (tuple(out.trace.shape) != shape or out.trace.dtype != torch.float64
                    or out.trace.device != self.device or not out.trace.is_contiguous()):
                raise ConfigError(f"out.trace must be a contiguous float64 tensor of shape {shape}")

    def solve(self, channels, noise_power, p_max, weights, init_precoders, *, gamma, omega,
              eps1=0.1, eps2=1e-3, max_iters=1000, latch_stage=True, record_trace=False,
              record_iterates=False,
              out: BatchResult | None = None, stream=None, cluster_size: int = 0,
              h_placement: int = 0, tensor_cores: int = 0, workspace=None,
              algorithm: str = "ammmse", bisect_tol: float = 1e-4,
              bisect_max: int = 100) -> BatchResult:
        """algorithm "ammmse" (ammmse_solve) or the exact-update drivers
        "wmmse" / "mmmse" (ammmse_solve_exact: bisect_tol / bisect_max apply,
        gamma / omega and the engine knobs are ignored)."""
        torch = _torch()
        dims = self.dims(channels, init_precoders)
        self.check(dims)
        B = dims.batch
        dev = self.device
        K = dims.K
        if channels.device != dev or init_precoders.device != dev:
            raise ConfigError(f"channels / init_precoders must live on the engine's device {dev}")
        for name, t, shape in (("noise_power", noise_power, (B,)), ("p_max", p_max, (B,)),
                               ("weights", weights, (B, K))):
            if (t.dtype != torch.float64 or t.device != dev or not t.is_contiguous()
                    or tuple(t.shape) != shape):
                raise ConfigError(f"{name} must be a contiguous float64 tensor of shape {shape} "
                                  f"on {dev}")
        if not channels.is_contiguous() or not init_precoders.is_contiguous():
            raise ConfigError("channels / init_precoders must be contiguous")
        if out is not None:
            self._check_out(out, init_precoders, B, int(max_iters))
        if out is None:
            out = BatchResult(
                final_precoders=torch.empty_like(init_precoders),
                wsr_bits=torch.empty(B, dtype=torch.float64, device=dev),
                iterations=torch.empty(B, dtype=torch.int32, device=dev),
                converged=torch.empty(B, dtype=torch.uint8, device=dev),
                stationarity_residual=torch.empty(B, dtype=torch.float64, device=dev),
                switch_iteration=torch.empty(B, dtype=torch.int32, device=dev),
                status=torch.empty(B, dtype=torch.int32, device=dev),
                gamma_used=torch.empty(B, dtype=torch.float64, device=dev),
                trace=(torch.full((B, int(max_iters), _native.TRACE_FIELDS), float("nan"),
                                  dtype=torch.float64, device=dev) if record_trace else None),
            )
            if record_iterates:
                T, N, d, M = int(max_iters), dims.N, dims.d, dims.M
                z = lambda *s: torch.full(s, complex("nan+nanj"), dtype=torch.complex128, device=dev)
                out.iterates = (z(B, T, K, N, d), z(B, T, K, d, d), z(B, T, K, M, d))
        # gamma: float | "safe" | (B,) float64 tensor;  omega: float | (B,) float64 tensor
        g_arr = gamma if torch.is_tensor(gamma) else None
        o_arr = omega if torch.is_tensor(omega) else None
        for name, t in (("gamma", g_arr), ("omega", o_arr)):
            if t is not None and (t.dtype != torch.float64 or t.device != dev or t.shape != (B,)
                                  or not t.is_contiguous()):
                raise ConfigError(f"per-realization {name} must be a contiguous ({B},) float64 tensor on {dev}")
        safe = g_arr is None and isinstance(gamma, str)
        if safe and gamma != GAMMA_SAFE:
            raise ConfigError(f"gamma must be positive or {GAMMA_SAFE!r}")
        opts = _native.AmmmseOptions(
            gamma=0.0 if (safe or g_arr is not None) else float(gamma), gamma_safe=1 if safe else 0,
            max_iters=int(max_iters), omega=0.0 if o_arr is not None else float(omega),
            eps1=float(eps1), eps2=float(eps2), latch_stage=1 if latch_stage else 0,
            cluster_size=int(cluster_size), h_placement=int(h_placement),
            tensor_cores=int(tensor_cores))
        prob = _native.AmmmseProblem(channels.data_ptr(), noise_power.data_ptr(), p_max.data_ptr(),
                                     weights.data_ptr(), init_precoders.data_ptr(),
                                     None if g_arr is None else g_arr.data_ptr(),
                                     None if o_arr is None else o_arr.data_ptr())
        ptr = lambda t: None if t is None else t.data_ptr()
        its = out.iterates if out.iterates is not None else (None, None, None)
        res = _native.AmmmseResult(
            ptr(out.final_precoders), ptr(out.wsr_bits), ptr(out.iterations), ptr(out.converged),
            ptr(out.stationarity_residual), ptr(out.switch_iteration), ptr(out.status),
            ptr(out.gamma_used), ptr(out.trace), ptr(its[0]), ptr(its[1]), ptr(its[2]))
        exact = {"ammmse": 0, "wmmse": _native.ALGO_WMMSE, "mmmse": _native.ALGO_MMMSE}.get(
            str(algorithm).lower())
        if exact is None:
            raise ConfigError(f"unknown algorithm {algorithm!r}")
        with torch.cuda.device(dev):  # the C-ABI launches on the current device
            ws_bytes = int(self.lib.ammmse_exact_workspace_size(dims) if exact
                           else self.lib.ammmse_workspace_size_opts(dims, opts))
            if ws_bytes == 0:
                raise ConfigError(f"no engine configuration fits (cluster_size={cluster_size}, "
                                  f"h_placement={h_placement}, tensor_cores={tensor_cores})")
            if workspace is not None:
                # caller-owned (concurrent solves on several streams each own one)
                if workspace.device != dev or workspace.numel() < ws_bytes:
                    raise ConfigError(f"workspace must be a tensor of >= {ws_bytes} bytes on {dev}")
                ws = workspace
            else:
                ws = self._workspace(ws_bytes, stream)
            if stream is None:
                stream = torch.cuda.current_stream(dev)
            if exact:
                rc = self.lib.ammmse_solve_exact(dims, prob, opts, exact, float(bisect_tol),
                                                 int(bisect_max), res, ws.data_ptr(), ws.numel(),
                                                 ctypes_stream(stream))
            else:
                rc = self.lib.ammmse_solve(dims, prob, opts, res, ws.data_ptr(), ws.numel(),
                                           ctypes_stream(stream))
        if rc != 0:
            if rc == _native.ERR_INVALID:
                raise ConfigError(_native.error_string(rc))
            raise NativeLibraryError(f"ammmse_solve failed: {_native.error_string(rc)}")
        out.omega = omega if o_arr is None else o_arr
        return out

    def generate_iid(self, B: int, K: int, N: int, M: int, d: int, *, seed0: int = 0,
                     p_max: float = 10.0, weights: str = "uniform", dtype="complex64",
                     stream=None):
        """On-device synthetic batch (ammmse_generate_iid): channels (B, K, N, M)
        and projected init_precoders (B, K, M, d) i.i.d. CN(0,1) from a Philox
        stream keyed by seed0 + r, weights (B, K) Uniform[0.5, 1.5) or ones.
        Distributionally identical to generate_channels / init_precoders,
        not bit-identical (the host generators stay the bit-exact path)."""
        torch = _torch()
        ct = torch.complex64 if str(dtype).endswith("64") else torch.complex128
        dev = self.device
        H = torch.empty((B, K, N, M), dtype=ct, device=dev)
        V0 = torch.empty((B, K, M, d), dtype=ct, device=dev)
        A = torch.empty((B, K), dtype=torch.float64, device=dev)
        if weights not in ("uniform", "ones"):
            raise ConfigError("weights must be 'uniform' or 'ones'")
        if not (p_max > 0 and math.isfinite(p_max)):
            raise ConfigError("p_max must be a positive real")
        dims = _native.AmmmseDims(B, M, N, K, d,
                                  _native.COMPLEX64 if ct == torch.complex64 else _native.COMPLEX128)
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        with torch.cuda.device(dev):
            rc = self.lib.ammmse_generate_iid(dims, int(seed0), float(p_max),
                                              1 if weights == "uniform" else 0, H.data_ptr(),
                                              V0.data_ptr(), A.data_ptr(), ctypes_stream(stream))
        if rc != 0:
            raise NativeLibraryError(f"ammmse_generate_iid failed: {_native.error_string(rc)}")
        return H, V0, A

    def generate_kronecker(self, B: int, K: int, N: int, M: int, d: int, *, seed0: int = 0,
                           p_max: float = 10.0, weights: str = "ones", rho: float = 0.5,
                           dtype="complex64", stream=None):
        """On-device Kronecker-correlated batch (BASELINE configs[3]):
        H_k = sqrt(beta_k) G_k R^{1/2} with G_k i.i.d. CN(0,1) from
        ammmse_generate_iid, R_ij = rho^|i-j| (symmetric PSD root by eigh on the
        host, inputs.kronecker_root), beta_k = 10^U[-2,0) from a second Philox
        stream (seed tag 0xBE7A); V0 / weights as generate_iid.  The R^{1/2}
        product is one batched library GEMM (input generation, not the solve)."""
        torch = _torch()
        from .inputs import kronecker_root

        H, V0, A = self.generate_iid(B, K, N, M, d, seed0=seed0, p_max=p_max, weights=weights,
                                     dtype=dtype, stream=stream)
        _, _, U = self.generate_iid(B, K, 1, 1, 1, seed0=(int(seed0) ^ 0xBE7A) << 20, p_max=1.0,
                                    weights="uniform", dtype=dtype, stream=stream)
        beta = torch.pow(10.0, 2.0 * (U - 1.5))  # U in [0.5, 1.5) -> beta in [0.01, 1)
        root = torch.from_numpy(kronecker_root(M, rho)).to(device=self.device, dtype=H.dtype)
        cs = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(
            torch.cuda.current_stream(self.device))
        with cs:
            H = torch.matmul(H.reshape(B * K * N, M), root).reshape(B, K, N, M)
            H *= torch.sqrt(beta).to(H.real.dtype)[:, :, None, None]
        return H.contiguous(), V0, A

    _RESULT_FIELDS = ("final_precoders", "wsr_bits", "iterations", "converged",
                      "stationarity_residual", "switch_iteration", "status")

    def solve_host(self, host_inputs, host_out, dev_inputs, dev_out: BatchResult, *, gamma, omega,
                   chunks: int = 4, stream=None, **kw) -> BatchResult:
        """End-to-end solve of HOST (pinned) arrays, pipelined in `chunks`
        slices over two CUDA streams: the host->device copy of slice i+1 and the
        device->host copy of slice i-1 overlap the solve of slice i, and the
        next slice's kernel fills the SMs the previous one's tail leaves idle.

        host_inputs / dev_inputs: (channels, noise_power, p_max, weights,
        init_precoders); host_out: dict of pinned tensors keyed by the
        BatchResult fields in _RESULT_FIELDS; dev_out: device BatchResult;
        gamma / omega: scalars or (B,) device tensors.  Stream-ordered on
        `stream` (default: the current stream); returns dev_out."""
        torch = _torch()
        dev = self.device
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        B = int(host_inputs[0].shape[0])
        chunks = max(1, min(int(chunks), B))
        if not hasattr(self, "_side"):
            self._side = [torch.cuda.Stream(dev) for _ in range(2)]
            self._side_ws = [None, None]
        start = torch.cuda.Event()
        start.record(stream)
        bounds = [B * c // chunks for c in range(chunks + 1)]
        for c in range(chunks):
            a, b = bounds[c], bounds[c + 1]
            if b <= a:
                continue
            s = self._side[c % 2]
            s.wait_event(start)
            with torch.cuda.stream(s):
                for d_, h_ in zip(dev_inputs, host_inputs):
                    d_[a:b].copy_(h_[a:b], non_blocking=True)
                sub = BatchResult(*(getattr(dev_out, f)[a:b] for f in self._RESULT_FIELDS),
                                  gamma_used=dev_out.gamma_used[a:b])
                g = gamma[a:b] if torch.is_tensor(gamma) else gamma
                o = omega[a:b] if torch.is_tensor(omega) else omega
                dims = self.dims(dev_inputs[0][a:b], dev_inputs[4][a:b])
                opts_kw = {k: kw[k] for k in ("cluster_size", "h_placement", "tensor_cores") if k in kw}
                need = int(self.lib.ammmse_workspace_size_opts(dims, _native.AmmmseOptions(
                    max_iters=int(kw.get("max_iters", 1000)), **opts_kw)))
                wsb = self._side_ws[c % 2]
                if wsb is None or wsb.numel() < need:
                    wsb = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
                    self._side_ws[c % 2] = wsb
                self.solve(*(x[a:b] for x in dev_inputs), gamma=g, omega=o, out=sub, stream=s,
                           workspace=wsb, **kw)
                for f, h_ in host_out.items():
                    h_[a:b].copy_(getattr(dev_out, f)[a:b], non_blocking=True)
        for s in self._side:
            stream.wait_stream(s)
        return dev_out

    def bounds(self, channels, weights, p_max, noise_power, stream=None):
        """Batched compute_bounds (ref objective.py:216-240): (B, 5) float64
        [kappa, l_v, gamma_safe, ek_floor, alpha_bar]."""
        torch = _torch()
        if channels.dim() != 4 or channels.dtype not in (torch.complex64, torch.complex128):
            raise ConfigError("channels must be a (B, K, N, M) complex64 / complex128 tensor")
        B, K, N, M = channels.shape
        dev = self.device
        for name, t, shape in (("weights", weights, (B, K)), ("p_max", p_max, (B,)),
                               ("noise_power", noise_power, (B,))):
            if (t.dtype != torch.float64 or t.device != dev or not t.is_contiguous()
                    or tuple(t.shape) != shape):
                raise ConfigError(f"{name} must be a contiguous float64 tensor of shape {shape} "
                                  f"on {dev}")
        if channels.device != dev or not channels.is_contiguous():
            raise ConfigError(f"channels must be contiguous on {dev}")
        dt = _native.COMPLEX64 if channels.dtype == torch.complex64 else _native.COMPLEX128
        dims = _native.AmmmseDims(B, M, N, K, 1, dt)
        out = torch.empty((B, _native.BOUND_FIELDS), dtype=torch.float64, device=dev)
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        with torch.cuda.device(dev):
            rc = self.lib.ammmse_bounds(dims, channels.data_ptr(), weights.data_ptr(),
                                        p_max.data_ptr(), noise_power.data_ptr(), out.data_ptr(),
                                        ctypes_stream(stream))
        if rc != 0:
            raise NativeLibraryError(f"ammmse_bounds failed: {_native.error_string(rc)}")
        return out


def ctypes_stream(stream) -> int:
    return int(stream.cuda_stream)


_ENGINES: dict = {}


def engine(device=None) -> AmmmseEngine:
    torch = _torch()
    if not torch.cuda.is_available():
        raise NativeLibraryError("the A-MMMSE engine needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = torch.cuda.current_device() if dev.index is None else dev.index
    if key not in _ENGINES:
        _ENGINES[key] = AmmmseEngine(torch.device("cuda", key))
    return _ENGINES[key]


def _validate_host_inputs(H, sigma2, p_max, weights, V0):
    if not np.all(np.isfinite(H)):
        raise ConfigError("channels contains non-finite entries")
    if not np.all(np.isfinite(V0)):
        raise ConfigError("precoders contains non-finite entries")
    if not np.all((sigma2 > 0) & np.isfinite(sigma2)):
        raise ConfigError("noise_power must be positive")
    if not np.all((p_max > 0) & np.isfinite(p_max)):
        raise ConfigError("p_max must be a positive real")
    if not np.all((weights > 0) & np.isfinite(weights)):
        raise ConfigError("weights must all be strictly positive")


def run_ammmse_batch(channels, noise_power, p_max, weights, init_precoders, options: SolverOptions,
                     snr_db: float = 10.0, record_trace: bool = False, device=None,
                     step_gamma=None, step_omega=None, cluster_size: int = 0,
                     h_placement: int = 0, tensor_cores: int = 0) -> BatchResult:
    """Solve B realizations from host arrays; returns a host BatchResult.

    channels (B, K, N, M), init_precoders (B, K, M, d): complex64 or
    complex128 numpy arrays (the engine computes in that precision);
    noise_power, p_max: (B,) or scalars; weights: (B, K) or (K,).
    ``snr_db`` only feeds the (omega, gamma) table when options leave them unset;
    ``step_gamma`` / ``step_omega`` ((B,) arrays) override the options per
    realization, the way the harness resolves them per sweep point
    (harness.py:466-472)."""
    torch = _torch()
    if options.algorithm is not Algorithm.AMMMSE:
        raise ConfigError("options.algorithm must be AMMMSE")
    return _run_batch(channels, noise_power, p_max, weights, init_precoders, options, snr_db,
                      record_trace, device, step_gamma, step_omega, cluster_size, h_placement,
                      tensor_cores)


def run_exact_batch(channels, noise_power, p_max, weights, init_precoders, options: SolverOptions,
                    record_trace: bool = False, device=None) -> BatchResult:
    """B realizations of the exact-update drivers run_wmmse / run_mmmse (ref
    solvers.py:521-537) on the device (ammmse_solve_exact): host arrays in,
    host BatchResult out, per-realization status codes; the algorithm,
    eps1 / eps2 / max_iters / latch_stage / bisect_tol / bisect_max come from
    ``options``."""
    if options.algorithm not in (Algorithm.WMMSE, Algorithm.MMMSE):
        raise ConfigError("options.algorithm must be WMMSE or MMMSE")
    return _run_batch(channels, noise_power, p_max, weights, init_precoders, options, 10.0,
                      record_trace, device, None, None, 0, 0, 0)


def _run_batch(channels, noise_power, p_max, weights, init_precoders, options, snr_db,
               record_trace, device, step_gamma, step_omega, cluster_size, h_placement,
               tensor_cores) -> BatchResult:
    torch = _torch()
    H = np.asarray(channels)
    V0 = np.asarray(init_precoders)
    if H.ndim != 4 or V0.ndim != 4:
        raise ConfigError("channels must be (B, K, N, M) and init_precoders (B, K, M, d)")
    dt = np.complex64 if (H.dtype == np.complex64 and V0.dtype == np.complex64) else np.complex128
    H = np.array(H, dtype=dt, order="C", copy=True)
    V0 = np.array(V0, dtype=dt, order="C", copy=True)
    B, K = H.shape[0], H.shape[1]
    s2 = np.broadcast_to(np.asarray(noise_power, dtype=np.float64), (B,)).copy()
    pm = np.broadcast_to(np.asarray(p_max, dtype=np.float64), (B,)).copy()
    al = np.broadcast_to(np.asarray(weights, dtype=np.float64), (B, K)).copy()
    _validate_host_inputs(H, s2, pm, al, V0)
    exact = options.algorithm is not Algorithm.AMMMSE
    gamma, omega = (0.0, 0.0) if exact else resolve_step_parameters(options, snr_db)
    eng = engine(device)
    dev = eng.device
    if step_gamma is not None:
        g = np.broadcast_to(np.asarray(step_gamma, dtype=np.float64), (B,)).copy()
        if not np.all((g > 0) & np.isfinite(g)):
            raise ConfigError("gamma must be positive")
        gamma = torch.from_numpy(g).to(dev)
    if step_omega is not None:
        o = np.broadcast_to(np.asarray(step_omega, dtype=np.float64), (B,)).copy()
        if not np.all((o >= 0) & (o < 1)):
            raise ConfigError("omega must lie in [0, 1)")
        omega = torch.from_numpy(o).to(dev)
    out = eng.solve(torch.from_numpy(H).to(dev), torch.from_numpy(s2).to(dev),
                    torch.from_numpy(pm).to(dev), torch.from_numpy(al).to(dev),
                    torch.from_numpy(V0).to(dev), gamma=gamma, omega=omega, eps1=options.eps1,
                    eps2=options.eps2, max_iters=options.max_iters, latch_stage=options.latch_stage,
                    record_trace=record_trace or options.record_iterates,
                    record_iterates=options.record_iterates, cluster_size=cluster_size,
                    h_placement=h_placement, tensor_cores=tensor_cores,
                    algorithm=options.algorithm.value, bisect_tol=options.bisect_tol,
                    bisect_max=options.bisect_max)
    return out.to_host()


def run_ammmse(channels: ChannelSet, config: SystemConfig, options: SolverOptions,
               init=None) -> SolveResult:
    """Reference-signature A-MMMSE solve of one realization (ref solvers.py:540-550).

    ``init`` optionally injects V0 (PrecoderSet or array); by default V0 is
    ``init_precoders(config)`` exactly as the reference draws it
    (solvers.py:427).  Raises the reference's exceptions for failed solves."""
    if options.algorithm is not Algorithm.AMMMSE:
        raise ConfigError("options.algorithm must be AMMMSE")
    if channels.noise_power is None:
        raise ConfigError("channels carry no noise power; call compute_noise_power first")
    if init is None:
        init = init_precoders(config, project_sum_power)
    v0 = init.precoders if isinstance(init, PrecoderSet) else np.asarray(init)
    H = channels.channels
    if H.shape != (config.K, config.N, config.M):
        raise ConfigError(f"channels shape {H.shape} does not match config "
                          f"(K={config.K}, N={config.N}, M={config.M})")
    dt = np.complex64 if (H.dtype == np.complex64 and v0.dtype == np.complex64) else np.complex128
    res = run_ammmse_batch(H[None].astype(dt), channels.noise_power, config.p_max,
                           config.weight_vector[None], v0[None].astype(dt), options,
                           snr_db=config.snr_db, record_trace=True)
    raise_for_status(int(res.status[0]), gamma=float(res.gamma_used[0]), omega=res.omega)
    return res.solve_result(0)


def _run_exact(channels: ChannelSet, config: SystemConfig, options: SolverOptions,
               init=None) -> SolveResult:
    if channels.noise_power is None:
        raise ConfigError("channels carry no noise power; call compute_noise_power first")
    if init is None:
        init = init_precoders(config, project_sum_power)
    v0 = init.precoders if isinstance(init, PrecoderSet) else np.asarray(init)
    H = channels.channels
    if H.shape != (config.K, config.N, config.M):
        raise ConfigError(f"channels shape {H.shape} does not match config "
                          f"(K={config.K}, N={config.N}, M={config.M})")
    res = run_exact_batch(H[None].astype(np.complex128), channels.noise_power, config.p_max,
                          config.weight_vector[None], v0[None].astype(np.complex128), options,
                          record_trace=True)
    raise_for_status(int(res.status[0]), gamma=0.0, omega=0.0)
    return res.solve_result(0)


def run_wmmse(channels: ChannelSet, config: SystemConfig, options: SolverOptions,
              init=None) -> SolveResult:
    """Exact block-coordinate WMMSE (ref solvers.py:521-527) on the device:
    MMSE receivers, the standard weight update from t = 1, precoders by dual
    bisection; stops on the relative WSR change."""
    if options.algorithm is not Algorithm.WMMSE:
        raise ConfigError("options.algorithm must be WMMSE")
    return _run_exact(channels, config, options, init)


def run_mmmse(channels: ChannelSet, config: SystemConfig, options: SolverOptions,
              init=None) -> SolveResult:
    """Two-stage warm-started exact solver (ref solvers.py:530-537): identity
    weights until the relative WSR change first drops below eps1, then the
    weighted updates until eps2."""
    if options.algorithm is not Algorithm.MMMSE:
        raise ConfigError("options.algorithm must be MMMSE")
    return _run_exact(channels, config, options, init)


_DRIVERS = {  # ref solvers.py:553-557
    Algorithm.WMMSE: run_wmmse,
    Algorithm.MMMSE: run_mmmse,
    Algorithm.AMMMSE: run_ammmse,
}


def solve(channels: ChannelSet, config: SystemConfig, options: SolverOptions) -> SolveResult:
    """Dispatch on options.algorithm (ref solvers.py:553-562)."""
    return _DRIVERS[options.algorithm](channels, config, options)
