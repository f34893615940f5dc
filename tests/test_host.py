"""CPU tests of the host layer: option validation and step-parameter
resolution mirror the reference (test_solvers.py:26-52), error mapping,
the C-ABI library loads and exports every symbol include/*.h declares, and
shape / argument validation happens before any GPU work."""

import math
import os
import re

import numpy as np
import pytest

import paper_2510_20507_b200 as pkg
from paper_2510_20507_b200 import _native
from paper_2510_20507_b200.errors import (STATUS_ILL_CONDITIONED, STATUS_OK, STATUS_UNSTABLE,
                                          ConfigError, IllConditionedWeightError,
                                          UnstableParametersError, raise_for_status)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestSolverOptions:
    def test_eps_ordering_enforced(self):
        with pytest.raises(ConfigError):
            pkg.SolverOptions(eps1=1e-4, eps2=1e-3)

    def test_omega_range(self):
        for bad in (1.0, -0.1):
            with pytest.raises(ConfigError):
                pkg.SolverOptions(omega=bad)

    def test_gamma_safe_sentinel(self):
        assert pkg.SolverOptions(gamma=pkg.GAMMA_SAFE).gamma == "safe"
        for bad in ("fast", -0.1, 0.0, math.inf):
            with pytest.raises(ConfigError):
                pkg.SolverOptions(gamma=bad)

    def test_eps2_positive_finite(self):
        for bad in (0.0, math.inf, -1.0):
            with pytest.raises(ConfigError):
                pkg.SolverOptions(eps2=bad, eps1=math.inf)

    def test_max_iters_and_algorithm_names(self):
        with pytest.raises(ConfigError):
            pkg.SolverOptions(max_iters=0)
        assert pkg.SolverOptions(algorithm=" AMMMSE ").algorithm is pkg.Algorithm.AMMMSE
        with pytest.raises(ConfigError):
            pkg.SolverOptions(algorithm="sgd")

    def test_step_defaults_by_snr(self):
        assert pkg.default_step_parameters(10.0) == (0.8, 0.05)
        assert pkg.default_step_parameters(20.0) == (0.8, 0.003)
        assert pkg.default_step_parameters(-10.0) == (0.6, 0.4)
        assert pkg.default_step_parameters(11.0) == (0.8, 0.05)
        assert pkg.default_step_parameters(-30.0) == (0.6, 0.4)
        assert pkg.default_step_parameters(12.5) == (0.8, 0.005)  # tie -> higher SNR

    def test_resolve(self):
        o = pkg.SolverOptions(algorithm="ammmse")
        assert pkg.resolve_step_parameters(o, 10.0) == (0.05, 0.8)
        o = pkg.SolverOptions(algorithm="ammmse", gamma="safe", omega=0.2)

        class B:
            gamma_safe = 0.123

        assert pkg.resolve_step_parameters(o, 10.0, B()) == (0.123, 0.2)
        assert pkg.resolve_step_parameters(o, 10.0) == ("safe", 0.2)


class TestModel:
    def test_config_validation(self):
        with pytest.raises(ConfigError):
            pkg.SystemConfig(M=0, N=1, K=1, d=1)
        with pytest.raises(ConfigError):
            pkg.SystemConfig(M=4, N=1, K=2, d=1, weights=(1.0,))
        with pytest.raises(ConfigError):
            pkg.SystemConfig(M=4, N=1, K=1, d=1, p_max=-1.0)
        c = pkg.SystemConfig(M=4, N=2, K=3, d=1)
        assert c.weights == (1.0, 1.0, 1.0)

    def test_generators_deterministic_and_projected(self):
        cfg = pkg.SystemConfig(M=8, N=2, K=3, d=2, p_max=2.0, channel_seed=4, init_seed=9)
        a = pkg.generate_channels(cfg).channels
        assert a.shape == (3, 2, 8) and np.array_equal(a, pkg.generate_channels(cfg).channels)
        v = pkg.init_precoders(cfg)
        assert v.total_power() <= 2.0 * (1 + 1e-12)

    def test_noise_power_formula(self):
        cfg = pkg.SystemConfig(M=4, N=2, K=2, d=1)
        h = np.zeros((2, 2, 4), dtype=complex)
        h[:, :, :2] = 1.0  # ||H_k||_F^2 = 4 = N * 2 -> 10^{log10 2 - 1}
        s2 = pkg.compute_noise_power(pkg.ChannelSet(h), 10.0, cfg)
        assert s2 == pytest.approx(0.2, rel=1e-12)
        with pytest.raises(pkg.DegenerateChannelError):
            pkg.compute_noise_power(pkg.ChannelSet(np.zeros((2, 2, 4))), 10.0, cfg)

    def test_channelset_rejects_nonfinite(self):
        h = np.ones((1, 1, 2), dtype=complex)
        h[0, 0, 0] = np.nan
        with pytest.raises(ConfigError):
            pkg.ChannelSet(h)


class TestErrors:
    def test_status_mapping(self):
        raise_for_status(STATUS_OK)
        with pytest.raises(IllConditionedWeightError):
            raise_for_status(STATUS_ILL_CONDITIONED)
        with pytest.raises(UnstableParametersError, match="gamma"):
            raise_for_status(STATUS_UNSTABLE, gamma=1000.0, omega=0.9)

    def test_drivers_reject_other_algorithms(self):
        # each driver checks its algorithm before any device work (solvers.py:524-548)
        cfg = pkg.SystemConfig(M=4, N=1, K=1, d=1)
        ch = pkg.ChannelSet(np.ones((1, 1, 4)), noise_power=1.0)
        with pytest.raises(ConfigError):
            pkg.run_ammmse(ch, cfg, pkg.SolverOptions(algorithm="mmmse"))
        with pytest.raises(ConfigError):
            pkg.run_wmmse(ch, cfg, pkg.SolverOptions(algorithm="ammmse"))
        with pytest.raises(ConfigError):
            pkg.run_mmmse(ch, cfg, pkg.SolverOptions(algorithm="wmmse"))
        from paper_2510_20507_b200.solvers import _DRIVERS

        assert _DRIVERS[pkg.Algorithm.WMMSE] is pkg.run_wmmse
        assert _DRIVERS[pkg.Algorithm.MMMSE] is pkg.run_mmmse
        assert _DRIVERS[pkg.Algorithm.AMMMSE] is pkg.run_ammmse


def _declared_functions(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(ammmse_\w+)\s*\(", text, flags=re.M))


class TestCAbi:
    def test_library_exports_every_declared_symbol(self):
        import ctypes

        h = _native.lib()
        decl = _declared_functions(os.path.join(ROOT, "include", "ammmse.h"))
        assert decl == set(_native.EXPORTED_SYMBOLS)
        for sym in decl:
            assert hasattr(h, sym), sym
        probe = ctypes.CDLL(os.path.join(ROOT, "paper_2510_20507_b200", "libammmse_probe.so"))
        for sym in _declared_functions(os.path.join(ROOT, "include", "ammmse_probe.h")):
            assert hasattr(probe, sym), sym

    def test_abi_version_and_workspace(self):
        h = _native.lib()
        assert h.ammmse_abi_version() == _native.ABI_VERSION
        d = _native.AmmmseDims(16, 64, 2, 16, 2, _native.COMPLEX64)
        assert h.ammmse_workspace_size(d) >= 8
        bad = _native.AmmmseDims(0, 64, 2, 16, 2, _native.COMPLEX64)
        assert h.ammmse_workspace_size(bad) == 0

    def test_check_dims_codes(self):
        h = _native.lib()
        D = _native.AmmmseDims
        assert h.ammmse_check_dims(D(4, 64, 2, 16, 2, 0)) == _native.OK
        assert h.ammmse_check_dims(D(4, 16, 2, 4, 2, 1)) == _native.OK
        assert h.ammmse_check_dims(D(0, 64, 2, 16, 2, 0)) == _native.ERR_INVALID
        assert h.ammmse_check_dims(D(4, 64, 2, 16, 2, 7)) == _native.ERR_INVALID
        assert h.ammmse_check_dims(D(4, 64, 5, 16, 2, 0)) == _native.ERR_UNSUPPORTED
        assert h.ammmse_check_dims(D(4, 64, 2, 16, 5, 0)) == _native.ERR_UNSUPPORTED
        assert "invalid" in _native.error_string(_native.ERR_INVALID)

    def test_planner_engine_choice(self):
        """ammmse_plan_info (no GPU needed): BASELINE large runs on the second-generation
        tensor-core engine (tensor_cores == 2) within the sm_100 shared-memory limit, the other
        BASELINE shapes keep their engines, and forcing tc2 on a shape outside its rules fails."""
        D, O = _native.AmmmseDims, _native.AmmmseOptions
        large = _native.plan_info(D(64, 128, 4, 32, 4, 0), O(max_iters=10))
        assert large["tensor_cores"] == 2 and large["cluster"] == 4 and large["threads"] == 256
        assert large["smem_bytes"] <= 232448 - 2048  # static shared (control block, barriers, slots)
        assert _native.plan_info(D(64, 128, 4, 32, 4, 0), O(max_iters=10, tensor_cores=2))["tensor_cores"] == 0
        assert _native.plan_info(D(64, 128, 4, 32, 4, 0), O(max_iters=10, tensor_cores=1))["tensor_cores"] == 1
        medium = _native.plan_info(D(64, 64, 2, 16, 2, 0), O(max_iters=10))
        assert medium["cluster"] == 0 and medium["tensor_cores"] == 0
        massive = _native.plan_info(D(64, 256, 2, 64, 2, 0), O(max_iters=10))
        assert massive["cluster"] == 4 and massive["tensor_cores"] == 0
        with pytest.raises(Exception):
            _native.plan_info(D(64, 256, 2, 64, 2, 0), O(max_iters=10, tensor_cores=3))
        # complex128 never takes a tensor-core engine
        assert _native.plan_info(D(8, 128, 4, 32, 4, 1), O(max_iters=10))["tensor_cores"] == 0

    def test_solve_rejects_null_problem_without_touching_gpu(self):
        h = _native.lib()
        d = _native.AmmmseDims(4, 64, 2, 16, 2, 0)
        rc = h.ammmse_solve(d, None, None, None, None, 0, None)
        assert rc in (_native.ERR_INVALID, _native.ERR_UNSUPPORTED)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    b = np.ones((1, 1, 1, 2), dtype=np.complex64)
    v = np.ones((1, 1, 2, 1), dtype=np.complex64)
    with pytest.raises(pkg.NativeLibraryError):
        pkg.run_ammmse_batch(b, 1.0, 1.0, np.ones((1, 1)), v,
                             pkg.SolverOptions(algorithm="ammmse", gamma=0.01, omega=0.0))


def test_product_path_does_not_import_oracle():
    """The product package never imports the CPU oracle."""
    pkgdir = os.path.join(ROOT, "paper_2510_20507_b200")
    for f in os.listdir(pkgdir):
        if f.endswith(".py"):
            src = open(os.path.join(pkgdir, f)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
