#!/usr/bin/env python
"""GEMM-step measurement (SURVEY.md §8(d) "GEMM-step fraction"): the cluster
engine's tensor-core GEMM (csrc/tc_stream.cuh) alone, on the engine's layouts
and a CTA's column slice at the BASELINE shapes, one CTA per SM, timed with
CUDA events.  Each CTA runs `reps` back-to-back GEMM + TMEM epilogue passes on
its problem (A = pre-split H planes streamed from L2 by bulk copies, B = the
fp32 column slice split hi/lo in shared memory), exactly what the solve does
twice per BCGD iteration.

    python bench_gemmstep.py [--reps 200]      # one JSON line per shape

Reported per shape: algorithmic TFLOP/s (8 flop per complex MAC, i.e. the
F = 16 K^2 N d M accounting of bench.py restricted to one GEMM of one column
slice), the tensor-pipe work actually issued (3xTF32: 3 real tf32 products per
real fp32 product), and the fraction of the 3xTF32 fp32-equivalent peak =
(dense tf32 peak) / 3, with tf32 dense = MEASURED_PEAKS bf16 burst / 2.
"""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))

# (label, KN, M, ncol, C): a CTA's slice of the BASELINE shapes on the cluster
# engine; the C CTAs of a cluster share one realization's H planes (L2 footprint
# as in the solve)
SHAPES = [("large C=4", 128, 128, 32, 4), ("massive C=4", 128, 256, 32, 4),
          ("sweep128 C=1", 64, 128, 64, 1), ("large C=2", 128, 128, 64, 2)]


def main():
    import numpy as np
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--ablate", type=int, nargs="*", default=[0],
                    help="tcs::gemm<DBG> variants to time: 1 no A copies, 2 no B split, "
                         "4 no MMAs, 7 none of them (diagnostics)")
    args = ap.parse_args()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2510_20507_b200", "libammmse_gemmstep.so"))
    lib.ammmse_gemmstep_scratch.restype = ctypes.c_size_t
    lib.ammmse_gemmstep_scratch.argtypes = [ctypes.c_int] * 3
    lib.ammmse_gemmstep_run.restype = ctypes.c_int
    lib.ammmse_gemmstep_run.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 8 + [ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    tf32 = peaks["bf16_tflops"] / 2
    peak3 = tf32 / 3
    stream = torch.cuda.current_stream(dev)
    for label, KN, M, ncol, share in SHAPES:
        for (mode, name), abl in ((m, a) for m in ((0, "GEMM-B G = H X"), (1, "GEMM-A grad = H^H Y"))
                                  for a in args.ablate):
            rows, kd = (KN, M) if mode == 0 else (M, KN)
            rng = np.random.default_rng(0)
            H = torch.from_numpy((rng.standard_normal((sms, KN, M)) + 1j * rng.standard_normal(
                (sms, KN, M))).astype(np.complex64)).to(dev)
            B = torch.from_numpy((rng.standard_normal((sms, kd, ncol)) + 1j * rng.standard_normal(
                (sms, kd, ncol))).astype(np.complex64)).to(dev)
            D = torch.empty((sms, rows, ncol), dtype=torch.complex64, device=dev)
            scr = torch.empty(lib.ammmse_gemmstep_scratch(KN, M, sms), dtype=torch.uint8, device=dev)
            # (slots beyond sms / share stay unused)
            run = lambda reps: lib.ammmse_gemmstep_run(H.data_ptr(), B.data_ptr(), D.data_ptr(),
                                                       scr.data_ptr(), sms, KN, M, ncol,
                                                       mode | (abl << 2), reps,
                                                       sms, share, stream.cuda_stream)
            assert run(2) == 0
            torch.cuda.synchronize()
            ts = []
            for reps in (1, 1 + args.reps):  # difference removes the per-problem split / load
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                assert run(reps) == 0
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            t = (ts[1] - ts[0]) / args.reps  # one GEMM + epilogue on every SM
            flops = 8.0 * rows * kd * ncol * sms
            achieved = flops / t
            print(json.dumps({
                "shape": label, "gemm": name, "rows": rows, "K": kd, "ncol": ncol, "ctas": sms,
                "ctas_per_h": share, "ablate": abl,
                "us_per_gemm": t * 1e6, "cycles_per_gemm_at_1965MHz": t * 1.965e9,
                "achieved_tflops": achieved / 1e12,
                "tensor_tflops_issued": 3 * achieved / 1e12,
                "peak_3xtf32_tflops": peak3, "frac_of_3xtf32_peak": achieved / 1e12 / peak3,
                "peak_note": f"tf32 dense = MEASURED_PEAKS bf16 burst {peaks['bf16_tflops']} / 2; "
                             "3xTF32 fp32-equivalent = tf32 / 3"}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
