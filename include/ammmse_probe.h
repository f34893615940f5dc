/*
 * ammmse_probe.h — measurement helper library (libammmse_probe.so), used by
 * bench.py to obtain the FP32 FMA-pipe roofline denominator live on the box
 * (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).  Not part of
 * the solver ABI and never on the solve path.
 */
#ifndef AMMMSE_PROBE_H_
#define AMMMSE_PROBE_H_
#ifdef __cplusplus
extern "C" {
#endif
/* Runs an FFMA throughput kernel on the current device and returns the
   achieved FP32 FLOP/s (2 per FMA), or a negative value on error. */
double ammmse_probe_fp32_flops(int reps);
/* Same for the FP64 DFMA pipe. */
double ammmse_probe_fp64_flops(int reps);
#ifdef __cplusplus
}
#endif
#endif
