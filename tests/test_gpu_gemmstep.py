"""The cluster engine's tensor-core GEMM (csrc/tc_stream.cuh: bulk-copied
pre-split H planes, warp-specialised B split, tcgen05 kind::tf32 3xTF32,
TMEM accumulators) driven standalone through libammmse_gemmstep.so on the
engine's layouts, against a complex128 numpy product of the same operands:
    mode 0 (GEMM-B):  D = H X        mode 1 (GEMM-A):  D = H^H Y
mode 2 / 3: the same products with the gemm_sync schedule.
Bar: error / (|H| |B| column scale) <= 1e-5, i.e. fp32-class accuracy
(1xTF32 would be ~1e-3)."""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gslib():
    h = ctypes.CDLL(os.path.join(ROOT, "paper_2510_20507_b200", "libammmse_gemmstep.so"))
    h.ammmse_gemmstep_scratch.restype = ctypes.c_size_t
    h.ammmse_gemmstep_scratch.argtypes = [ctypes.c_int] * 3
    h.ammmse_gemmstep_run.restype = ctypes.c_int
    h.ammmse_gemmstep_run.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 8 + [ctypes.c_void_p]
    return h


def run(gslib, cuda, H, B, mode, reps=1):
    import torch

    nprob, KN, M = H.shape
    ncol = B.shape[2]
    rows = KN if mode % 2 == 0 else M
    dH = torch.from_numpy(H).to(cuda)
    dB = torch.from_numpy(B).to(cuda)
    dD = torch.full((nprob, rows, ncol), complex(float("nan"), 0), dtype=torch.complex64, device=cuda)
    grid = min(nprob, torch.cuda.get_device_properties(cuda).multi_processor_count)
    scr = torch.empty(gslib.ammmse_gemmstep_scratch(KN, M, grid), dtype=torch.uint8, device=cuda)
    rc = gslib.ammmse_gemmstep_run(dH.data_ptr(), dB.data_ptr(), dD.data_ptr(), scr.data_ptr(), nprob,
                                   KN, M, ncol, mode, reps, grid, 1,
                                   torch.cuda.current_stream(cuda).cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    return dD.cpu().numpy()


@pytest.mark.parametrize("KN,M,ncol", [(128, 128, 32), (64, 128, 32), (128, 256, 32), (64, 128, 64),
                                       (128, 128, 16), (64, 64, 16)])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_tc_gemm_matches_complex128(cuda, gslib, KN, M, ncol, mode):
    rng = np.random.default_rng(KN * 7 + M + ncol + mode)
    nprob = 3
    c = lambda *s: ((rng.standard_normal(s) + 1j * rng.standard_normal(s)) / np.sqrt(2)).astype(np.complex64)
    H = c(nprob, KN, M)
    kd = M if mode % 2 == 0 else KN
    B = c(nprob, kd, ncol)
    got = run(gslib, cuda, H, B, mode)
    H64, B64 = H.astype(np.complex128), B.astype(np.complex128)
    ref = H64 @ B64 if mode % 2 == 0 else np.conj(np.swapaxes(H64, 1, 2)) @ B64
    scale = np.sqrt(kd)  # |entries| ~ sqrt(kd)
    err = np.abs(got - ref).max() / scale
    # fp32 FFMA-class reference: the same product in complex64 numpy (BLAS fp32)
    H32, B32 = H, B
    f32 = H32 @ B32 if mode % 2 == 0 else np.conj(np.swapaxes(H32, 1, 2)) @ B32
    err32 = np.abs(f32.astype(np.complex128) - ref).max() / scale
    print(f"KN={KN} M={M} ncol={ncol} mode={mode}: 3xTF32 err {err:.2e}, fp32 BLAS err {err32:.2e}")
    assert np.isfinite(got).all()
    assert err < 4 * err32 + 1e-7, (err, err32)
