"""Validation of the hand-written tcgen05 toolkit (csrc/tc_umma.cuh) on B200:
3xTF32 D = A·B through UMMA with TMEM accumulators (K-major A and B in the
canonical no-swizzle layout), both accumulator heights (M = 64, 128) and the
negate-B instruction bit, against fp64.

Measured facts (round 1):
  * K-major A/B: correct; normalised error ~2-3e-6 (tensor-core fp32
    accumulation is ~5x noisier than an FFMA dot product of the same length);
  * MN-major kind::tf32 operands in the no-swizzle layout read back as zeros
    (either LBO/SBO assignment), so the engine keeps every operand K-major
    (H and H^T are pre-split separately, tc_stream.cuh) and no test pins the
    MN-major behaviour.
"""

import ctypes
import itertools
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tclib():
    return ctypes.CDLL(os.path.join(ROOT, "paper_2510_20507_b200", "libammmse_tctest.so"))


CASES = list(itertools.product([128, 64], [16, 32], [32, 64], [0], [0], [0, 1]))


@pytest.mark.parametrize("P,Q,K,a_mn,b_mn,neg_b", CASES)
def test_umma_3xtf32(cuda, tclib, P, Q, K, a_mn, b_mn, neg_b):
    import torch

    rng = np.random.default_rng(P * 1000 + Q * 10 + K + 7 * a_mn + 3 * b_mn + neg_b)
    A = rng.standard_normal((P, K)).astype(np.float32)
    B = rng.standard_normal((K, Q)).astype(np.float32)
    dA, dB = torch.from_numpy(A).to(cuda), torch.from_numpy(B).to(cuda)
    dD = torch.full((P, Q), float("nan"), dtype=torch.float32, device=cuda)
    rc = tclib.ammmse_tc_selftest(ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                                  ctypes.c_void_p(dD.data_ptr()), P, Q, K, a_mn, b_mn, neg_b,
                                  int(os.environ.get("AMMMSE_TC_SWAP", "0")))
    assert rc == 0
    ref = A.astype(np.float64) @ B.astype(np.float64) * (-1.0 if neg_b else 1.0)
    got = dD.cpu().numpy().astype(np.float64)
    scale = np.sqrt(K)  # |entries| ~ sqrt(K)
    err = np.abs(got - ref).max() / scale
    assert err < 1e-5, (err, got[:2, :4], ref[:2, :4])
