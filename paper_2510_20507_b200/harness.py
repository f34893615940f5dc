"""Experiment harness on the batched engine.

Mirror of the reference runner (pkg/src/wsrbeam/harness.py) for the A-MMMSE
path: the same experiment spec, sweep expansion, per-realization seeds, trace
CSV format and ``summary.json`` schema, with one batched device solve per
sweep point instead of one process-pool job per realization
(``_solve_one``, harness.py:262-278).

    spec = ExperimentSpec(base=SystemConfig(...), solver=SolverOptions(...),
                          n_realizations=100, sweep=(("snr_db", (0, 10, 20)),),
                          output_dir="out")
    summary = run_experiment(spec)

``verify=True`` runs the reference's oracles (harness.py:459-460, :509-517,
:540-545) at batch scale on the device (verify.py): every realization is solved
with recorded iterates, the four lemma-bound families are scanned over all of
them in one pass per sweep point, and the finite-difference gradient check
runs on the base system.

Differences from the reference, by design:
  * only ``Algorithm.AMMMSE`` (the exact drivers are out of scope);
  * ``parallel_workers`` is kept for the schema but unused (one device call
    per point);
  * failure strings carry the reference's exception class and the engine's
    message (the device engine reports a status code per realization, not the
    offending user index / condition number);
  * ``stamps.package`` names this package.
"""

from __future__ import annotations

import dataclasses
import json
import math
import platform
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import __version__
from .errors import (
    STATUS_OK,
    ConfigError,
    IllConditionedWeightError,
    UnstableParametersError,
    raise_for_status,
)
from .model import RNG_ALGORITHM, Stage, SystemConfig, compute_noise_power, generate_channels, \
    init_precoders, project_sum_power
from .solvers import Algorithm, IterationRecord, SolveResult, SolverOptions, \
    default_step_parameters, run_ammmse_batch

TRACE_HEADER = "iter,wsr_bpcu,f_nats,power,stage,f_after_u,f_after_w,f_after_v,rel_change"  # harness.py:50

_SWEEPABLE = ("K", "M", "snr_db")  # harness.py:52


@dataclass(frozen=True)
class ExperimentSpec:
    """One experiment: base system, solver options, sweep grid, I/O (harness.py:63-87)."""

    base: SystemConfig
    solver: SolverOptions
    n_realizations: int = 20
    sweep: tuple = ()
    parallel_workers: int = 0
    output_dir: Path = Path("out")

    def __post_init__(self) -> None:
        if self.n_realizations < 1:
            raise ConfigError("n_realizations must be at least 1")
        if self.parallel_workers < 0:
            raise ConfigError("parallel_workers must be nonnegative")
        object.__setattr__(self, "output_dir", Path(self.output_dir))
        object.__setattr__(self, "sweep", tuple((str(n), tuple(v)) for n, v in self.sweep))
        for name, values in self.sweep:
            if name not in _SWEEPABLE:
                raise ConfigError(f"sweep parameter must be one of {_SWEEPABLE}, got {name!r}")
            if len(values) == 0:
                raise ConfigError(f"sweep over {name} has no values")
            for v in values:
                if not math.isfinite(v):
                    raise ConfigError(f"sweep value for {name} must be finite, got {v!r}")
                if name in ("K", "M") and (v <= 0 or int(v) != v):
                    raise ConfigError(f"sweep values for {name} must be positive integers, got {v!r}")


# --------------------------------------------------------------------------- traces
def _fmt(x: float) -> str:
    return repr(float(x))  # round-trips exactly (harness.py:188-191)


def emit_trace(result: SolveResult, path) -> None:
    """One CSV row per iteration, exact decimal text (harness.py:194-209)."""
    lines = [TRACE_HEADER]
    for rec in result.trace:
        lines.append(",".join([
            str(rec.t), _fmt(rec.wsr_bits), _fmt(rec.f_value), _fmt(rec.total_power),
            str(rec.stage.value), _fmt(rec.f_after_u), _fmt(rec.f_after_w), _fmt(rec.f_after_v),
            _fmt(rec.rel_change),
        ]))
    Path(path).write_text("\n".join(lines) + "\n")


def read_trace(path) -> tuple:
    """Parse a trace CSV back into iteration records (harness.py:212-230)."""
    text = Path(path).read_text()
    lines = [ln for ln in text.splitlines() if ln]
    if not lines or lines[0] != TRACE_HEADER:
        raise ConfigError(f"{path}: not a trace file (bad header)")
    records = []
    for ln in lines[1:]:
        p = ln.split(",")
        if len(p) != 9:
            raise ConfigError(f"{path}: malformed trace row {ln!r}")
        records.append(IterationRecord(
            t=int(p[0]), wsr_bits=float(p[1]), f_value=float(p[2]), total_power=float(p[3]),
            stage=Stage(int(p[4])), f_after_u=float(p[5]), f_after_w=float(p[6]),
            f_after_v=float(p[7]), rel_change=float(p[8])))
    return tuple(records)


# --------------------------------------------------------------------------- sweep
def sweep_points(spec: ExperimentSpec) -> list:
    """Cross product of the sweep grid; label "base" without a sweep (harness.py:232-259)."""
    points = [("base", spec.base)]
    for name, values in spec.sweep:
        expanded = []
        for label, cfg in points:
            for v in values:
                overrides: dict = {}
                if name in ("K", "M"):
                    value = int(v)
                    tag = f"{name}{value}"
                    if name == "K" and len(cfg.weights) != value:  # K invalidates the weights
                        overrides["weights"] = None
                else:
                    value = float(v)
                    tag = f"snr{value:g}"
                overrides[name] = value
                new_cfg = dataclasses.replace(cfg, **overrides)
                expanded.append((tag if label == "base" else f"{label}_{tag}", new_cfg))
        points = expanded
    return points


# --------------------------------------------------------------------------- summary
def _config_dict(c: SystemConfig) -> dict:
    return {"M": c.M, "N": c.N, "K": c.K, "d": c.d, "p_max": c.p_max, "snr_db": c.snr_db,
            "weights": list(c.weights), "channel_seed": c.channel_seed, "init_seed": c.init_seed}


def _solver_dict(o: SolverOptions) -> dict:
    return {"algorithm": o.algorithm.value, "gamma": o.gamma, "omega": o.omega, "eps1": o.eps1,
            "eps2": o.eps2, "max_iters": o.max_iters, "bisect_tol": o.bisect_tol,
            "bisect_max": o.bisect_max}


def _mean_std(values):
    if not values:
        return None, None
    a = np.asarray(values, dtype=np.float64)
    return float(a.mean()), float(a.std())


@dataclass(frozen=True)
class PointSummary:
    """Aggregates of one sweep point (harness.py:322-344)."""

    label: str
    config: SystemConfig
    solver: SolverOptions
    n_realizations: int
    n_completed: int
    n_converged: int
    wsr_bits_mean: float | None
    wsr_bits_std: float | None
    iterations_mean: float | None
    iterations_std: float | None
    switch_iteration_mean: float | None
    stationarity_residual_max: float | None
    failures: tuple
    wall_time_mean: float | None
    wall_time_std: float | None

    def __post_init__(self) -> None:
        if self.n_completed + len(self.failures) != self.n_realizations:
            raise ConfigError("completed and failed realizations must account for "
                              f"all {self.n_realizations} runs")


@dataclass(frozen=True)
class RunSummary:
    """All points of one experiment; JSON schema of harness.py:347-394."""

    spec: ExperimentSpec
    points: tuple
    oracle_reports: tuple = ()

    def to_json_dict(self, include_timing: bool = False) -> dict:
        points = []
        for p in self.points:
            e = {"label": p.label, "config": _config_dict(p.config), "solver": _solver_dict(p.solver),
                 "n_realizations": p.n_realizations, "n_completed": p.n_completed,
                 "n_converged": p.n_converged, "convergence_rate": p.n_converged / p.n_realizations,
                 "wsr_bits_mean": p.wsr_bits_mean, "wsr_bits_std": p.wsr_bits_std,
                 "iterations_mean": p.iterations_mean, "iterations_std": p.iterations_std,
                 "switch_iteration_mean": p.switch_iteration_mean,
                 "stationarity_residual_max": p.stationarity_residual_max,
                 "failures": list(p.failures)}
            if include_timing:
                e["wall_time_mean_s"] = p.wall_time_mean
                e["wall_time_std_s"] = p.wall_time_std
            points.append(e)
        return {
            "spec": {"base": _config_dict(self.spec.base), "solver": _solver_dict(self.spec.solver),
                     "n_realizations": self.spec.n_realizations,
                     "sweep": [[n, list(v)] for n, v in self.spec.sweep],
                     "parallel_workers": self.spec.parallel_workers,
                     "output_dir": str(self.spec.output_dir)},
            "points": points,
            "oracles": [{"name": r.name, "max_abs_error": r.max_abs_error,
                         "max_rel_error": r.max_rel_error, "instances": r.instances,
                         "passed": r.passed, "tolerance": r.tolerance, "detail": r.detail}
                        for r in self.oracle_reports],
            "stamps": {"package": "paper_2510_20507_b200", "version": __version__,
                       "python": platform.python_version(), "numpy": np.__version__,
                       "rng": RNG_ALGORITHM},
        }


# --------------------------------------------------------------------------- runner
def point_inputs(cfg: SystemConfig, n: int, dtype=np.complex128):
    """Host inputs of realizations r = 0..n-1 of one sweep point, seeds
    base + r (harness.py:474-480), noise power from the SNR (harness.py:270-272)
    and V0 drawn as init_precoders draws it (solvers.py:427)."""
    H, s2, alpha, V0, cfgs = [], [], [], [], []
    for r in range(n):
        cfg_r = dataclasses.replace(cfg, channel_seed=cfg.channel_seed + r,
                                    init_seed=cfg.init_seed + r)
        ch = generate_channels(cfg_r)
        H.append(ch.channels)
        s2.append(compute_noise_power(ch, cfg_r.snr_db, cfg_r))
        alpha.append(cfg_r.weight_vector)
        V0.append(init_precoders(cfg_r, project_sum_power).precoders)
        cfgs.append(cfg_r)
    return (np.stack(H).astype(dtype), np.asarray(s2), np.stack(alpha), np.stack(V0).astype(dtype),
            cfgs)


def _failure(status: int, gamma, omega) -> str:
    try:
        raise_for_status(status, gamma=gamma, omega=omega)
    except (IllConditionedWeightError, UnstableParametersError) as exc:
        return f"{type(exc).__name__}: {exc}"
    return f"status {status}"


def _lemma_point_report(label, H, s2, alpha, p_max, res, device):
    """lemma_bounds[label]: check_lemma_bounds of every completed realization of
    the point merged as harness._merge_lemma_reports does (harness.py:434-445),
    in one batched device scan; bounds per realization from ammmse_bounds."""
    import torch

    from .solvers import engine
    from .verify import lemma_bound_scan, lemma_report

    ok = np.nonzero(res.status == STATUS_OK)[0]
    if ok.size == 0:
        return []
    eng = engine(device)
    dev = eng.device
    Hd = torch.from_numpy(np.ascontiguousarray(H[ok])).to(dev)
    s2d = torch.from_numpy(np.ascontiguousarray(s2[ok], dtype=np.float64)).to(dev)
    ald = torch.from_numpy(np.ascontiguousarray(alpha[ok], dtype=np.float64)).to(dev)
    pmd = torch.full((ok.size,), float(p_max), dtype=torch.float64, device=dev)
    bnd = eng.bounds(Hd, ald, pmd, s2d)
    U, W, V = (torch.from_numpy(np.ascontiguousarray(x[ok])).to(dev) for x in res.iterates)
    worst, lim = lemma_bound_scan(Hd, s2d, ald, bnd, U, W, V, res.iterations[ok])
    return [lemma_report(worst, lim, instances=int(res.iterations[ok].sum()),
                         name=f"lemma_bounds[{label}]")]


def run_experiment(spec: ExperimentSpec, verify: bool = False, dtype=np.complex128,
                   device=None) -> RunSummary:
    """Run every (sweep point x realization), write traces and summaries
    (harness.py:448-562), one batched device solve per sweep point.
    Realizations are reduced in realization order, so the outputs do not depend
    on the batch split."""
    if spec.solver.algorithm is not Algorithm.AMMMSE:
        raise ConfigError("the batched engine runs A-MMMSE only")
    outdir = spec.output_dir
    outdir.mkdir(parents=True, exist_ok=True)
    options = spec.solver
    if verify and not options.record_iterates:  # harness.py:459-460
        options = dataclasses.replace(options, record_iterates=True)
    summaries = []
    oracle_reports = []
    for label, point_cfg in sweep_points(spec):
        opts = options
        if options.gamma is None or options.omega is None:  # per point (harness.py:466-472)
            omega_d, gamma_d = default_step_parameters(point_cfg.snr_db)
            opts = dataclasses.replace(options,
                                       gamma=gamma_d if options.gamma is None else options.gamma,
                                       omega=omega_d if options.omega is None else options.omega)
        H, s2, alpha, V0, _ = point_inputs(point_cfg, spec.n_realizations, dtype)
        t0 = time.perf_counter()
        res = run_ammmse_batch(H, s2, point_cfg.p_max, alpha, V0, opts, snr_db=point_cfg.snr_db,
                               record_trace=True, device=device)
        wall = (time.perf_counter() - t0) / spec.n_realizations
        if verify:  # lemma bounds over every completed realization's iterates (:509-517)
            oracle_reports.extend(_lemma_point_report(label, H, s2, alpha, point_cfg.p_max, res,
                                                      device))
        wsr, iters, switches, residuals, walls, failures = [], [], [], [], [], []
        n_conv = 0
        for r in range(spec.n_realizations):
            st = int(res.status[r])
            if st != STATUS_OK:
                failures.append(f"seed {r}: {_failure(st, float(res.gamma_used[r]), res.omega)}")
                continue
            sr = res.solve_result(r)
            emit_trace(sr, outdir / f"{opts.algorithm.value}_{label}_seed{r}.csv")
            wsr.append(sr.trace[-1].wsr_bits)
            iters.append(float(sr.iterations))
            if sr.switch_iteration is not None:
                switches.append(float(sr.switch_iteration))
            residuals.append(sr.stationarity_residual)
            walls.append(wall)
            n_conv += int(sr.converged)
        wm, ws = _mean_std(wsr)
        im, isd = _mean_std(iters)
        sm, _ = _mean_std(switches)
        tm, tsd = _mean_std(walls)
        summaries.append(PointSummary(
            label=label, config=point_cfg, solver=opts, n_realizations=spec.n_realizations,
            n_completed=len(wsr), n_converged=n_conv, wsr_bits_mean=wm, wsr_bits_std=ws,
            iterations_mean=im, iterations_std=isd, switch_iteration_mean=sm,
            stationarity_residual_max=max(residuals) if residuals else None,
            failures=tuple(failures), wall_time_mean=tm, wall_time_std=tsd))
    if verify:  # finite-difference gradient check on the base system (:543-545)
        from .verify import gradient_fd_report

        fd = gradient_fd_report(spec.base)
        if fd is not None:
            oracle_reports.append(fd)
    summary = RunSummary(spec=spec, points=tuple(summaries), oracle_reports=tuple(oracle_reports))
    (outdir / "summary.json").write_text(
        json.dumps(summary.to_json_dict(include_timing=False), indent=2, sort_keys=True) + "\n")
    timing = {"note": "wall-clock statistics are non-normative and excluded from the "
                      "reproducibility contract (one batched device solve per point)",
              "points": [{"label": p.label, "wall_time_mean_s": p.wall_time_mean,
                          "wall_time_std_s": p.wall_time_std} for p in summary.points]}
    (outdir / "timing.json").write_text(json.dumps(timing, indent=2, sort_keys=True) + "\n")
    return summary
