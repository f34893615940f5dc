/*
 * ammmse.h — C-ABI of the B200-native batched A-MMMSE engine (libammmse.so).
 *
 * One call solves B independent channel realizations of the weighted
 * sum-rate precoder problem with the A-MMMSE algorithm (arXiv 2510.20507),
 * i.e. it replaces, per realization, the reference call
 *
 *     wsrbeam.run_ammmse(channels, config, options) -> SolveResult
 *         pkg/src/wsrbeam/solvers.py:540-550  (driver)
 *         pkg/src/wsrbeam/solvers.py:415-518  (_run_bcd loop, exact=False,
 *                                              use_extrapolation=True,
 *                                              start_weighted=False)
 *
 * and its once-per-solve helper
 *
 *     wsrbeam.compute_bounds(channels, weights, p_max, noise_power)
 *         pkg/src/wsrbeam/objective.py:216-240
 *
 * The reference is pure Python (no FFI exists upstream); the binding a
 * maintainer would add on the reference side is a ctypes stub, shown in
 * INTEGRATION.md.  Signatures carry plain pointers and sizes only.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers on the current CUDA device.
 *   - Complex arrays are interleaved (re, im) pairs: complex64 = 2 x float,
 *     complex128 = 2 x double (numpy / torch memory layout).
 *   - Layouts follow the reference containers: channels (B, K, N, M)
 *     (model.py:110), precoders (B, K, M, d) (model.py:141).
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     stream-ordered and asynchronous.  No global mutable state: calls are
 *     reentrant across streams and devices.
 *   - Return value: 0 on success, a negative AMMMSE_ERR_* code otherwise.
 *     Numerical failures of individual realizations are NOT call errors:
 *     they are reported per realization in `status` (AMMMSE_STATUS_*), the
 *     way the reference harness records per-realization exceptions
 *     (harness.py:277-278).
 */
#ifndef AMMMSE_H_
#define AMMMSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMMMSE_ABI_VERSION 2

/* element type of channels / precoders */
enum {
  AMMMSE_COMPLEX64 = 0,  /* fp32 GEMMs, fp64 small algebra + WSR */
  AMMMSE_COMPLEX128 = 1  /* fp64 throughout (reference precision, model.py:93) */
};

/* call status */
enum {
  AMMMSE_OK = 0,
  AMMMSE_ERR_INVALID = -1,      /* bad pointer / dims / options (ConfigError) */
  AMMMSE_ERR_UNSUPPORTED = -2,  /* shape not instantiated (N or d > 4, SMEM) */
  AMMMSE_ERR_WORKSPACE = -3,    /* workspace NULL or smaller than ammmse_workspace_size */
  AMMMSE_ERR_CUDA = -4          /* a CUDA runtime call failed */
};

/* per-realization status (result.status) */
enum {
  AMMMSE_STATUS_OK = 0,              /* converged or reached max_iters */
  AMMMSE_STATUS_ILL_CONDITIONED = 1, /* IllConditionedWeightError, solvers.py:243-252 */
  AMMMSE_STATUS_UNSTABLE = 2,        /* UnstableParametersError, solvers.py:490-500 */
  AMMMSE_STATUS_NONFINITE = 3        /* non-finite iterate / failed Cholesky */
};

/* trace record fields, in IterationRecord order (solvers.py:139-156) */
enum {
  AMMMSE_TRACE_T = 0, AMMMSE_TRACE_WSR_BITS, AMMMSE_TRACE_F_VALUE,
  AMMMSE_TRACE_TOTAL_POWER, AMMMSE_TRACE_STAGE, AMMMSE_TRACE_F_AFTER_U,
  AMMMSE_TRACE_F_AFTER_W, AMMMSE_TRACE_F_AFTER_V, AMMMSE_TRACE_REL_CHANGE,
  AMMMSE_TRACE_FIELDS
};

typedef struct AmmmseDims {
  int64_t batch;  /* B, number of realizations (>= 1) */
  int32_t M;      /* BS antennas */
  int32_t N;      /* receive antennas per user (1..4) */
  int32_t K;      /* users */
  int32_t d;      /* streams per user (1..4) */
  int32_t dtype;  /* AMMMSE_COMPLEX64 | AMMMSE_COMPLEX128 */
} AmmmseDims;

/* inputs (ChannelSet + SystemConfig + V0 of each realization) */
typedef struct AmmmseProblem {
  const void* channels;        /* (B, K, N, M) complex                         */
  const double* noise_power;   /* (B,)   sigma^2 > 0      (ChannelSet.noise_power) */
  const double* p_max;         /* (B,)   P > 0            (SystemConfig.p_max)     */
  const double* weights;       /* (B, K) alpha_k > 0      (SystemConfig.weights)   */
  const void* init_precoders;  /* (B, K, M, d) complex, V0 (init_precoders(), model.py:225-235) */
  /* Optional per-realization step parameters (B,), NULL = use AmmmseOptions.
     The reference resolves (gamma, omega) per sweep point (harness.py:466-472);
     a batch mixing sweep points carries them per realization. */
  const double* gamma;         /* > 0; overrides options.gamma and options.gamma_safe */
  const double* omega;         /* [0, 1); overrides options.omega */
} AmmmseProblem;

/* SolverOptions (solvers.py:88-136) after resolve_step_parameters (:196-207) */
typedef struct AmmmseOptions {
  double gamma;        /* step size, used when gamma_safe == 0 (> 0, finite)           */
  int32_t gamma_safe;  /* 1: gamma = per-realization gamma_safe (GAMMA_SAFE sentinel)  */
  int32_t max_iters;   /* >= 1                                                         */
  double omega;        /* extrapolation, [0, 1)                                        */
  double eps1;         /* stage-switch threshold, > 0, may be +inf                     */
  double eps2;         /* stop threshold, > 0, finite, <= eps1                         */
  int32_t latch_stage; /* 1: latch the weighted stage (default); 0: re-test every iteration */
  int32_t cluster_size;/* 0: automatic engine choice.  c >= 1: force the thread-block-cluster
                          engine with c CTAs per realization (c in {1,2,4,8,16}, c | K) —
                          a tuning / testing knob, results are identical up to rounding */
  int32_t h_placement; /* cluster engine only: 0 auto, 1 H resident in every CTA's SMEM,
                          2 H streamed from HBM/L2 through a cp.async ring, 3 streamed H and
                          the previous precoders in a per-CTA global scratch slot */
  int32_t tensor_cores;/* cluster engine, complex64: 0 automatic (N = d = 4: the second-generation
                          tcgen05 engine, csrc/ammmse_tc2.cuh, where its shape rules hold — M = K N =
                          128 as in BASELINE large — else the first-generation one; other N, d: FFMA,
                          where measured faster); 1 first-generation tcgen05 3xTF32 GEMMs (bulk-copied
                          pre-split H planes, TMEM accumulators) where shape and shared memory allow;
                          2 FP32 FFMA GEMMs; 3 the second-generation engine or an error */
} AmmmseOptions;

/* SolveResult (solvers.py:174-182), struct-of-arrays.  Any pointer may be NULL. */
typedef struct AmmmseResult {
  void* final_precoders;          /* (B, K, M, d) complex, same dtype as inputs    */
  double* wsr_bits;               /* (B,)  trace[-1].wsr_bits                      */
  int32_t* iterations;            /* (B,)  len(trace)                              */
  uint8_t* converged;             /* (B,)                                          */
  double* stationarity_residual;  /* (B,)                                          */
  int32_t* switch_iteration;      /* (B,)  first weighted iteration, -1 = None     */
  int32_t* status;                /* (B,)  AMMMSE_STATUS_*                         */
  double* gamma_used;             /* (B,)  resolved step size                      */
  double* trace;                  /* (B, max_iters, AMMMSE_TRACE_FIELDS), rows past
                                     `iterations` are left untouched              */
  /* Recorded block iterates (SolverOptions.record_iterates, solvers.py:106, :487-488):
     per completed iteration t the (U, W, V_new) the reference appends as
     BlockIterate, complex128 (interleaved doubles) whatever the input dtype.
     Rows past `iterations` are left untouched.  All three NULL = not recorded. */
  double* iter_receivers;         /* (B, max_iters, K, N, d) complex128           */
  double* iter_weights;           /* (B, max_iters, K, d, d) complex128           */
  double* iter_precoders;         /* (B, max_iters, K, M, d) complex128           */
} AmmmseResult;

/* BoundsReport (objective.py:40-66) per realization, (B, 5) row-major */
enum {
  AMMMSE_BOUND_KAPPA = 0, AMMMSE_BOUND_L_V, AMMMSE_BOUND_GAMMA_SAFE,
  AMMMSE_BOUND_EK_FLOOR, AMMMSE_BOUND_ALPHA_BAR, AMMMSE_BOUND_FIELDS
};

/* ABI version (AMMMSE_ABI_VERSION) */
int ammmse_abi_version(void);

/* 0 if the dims are supported by the compiled engine, else AMMMSE_ERR_* */
int ammmse_check_dims(const AmmmseDims* dims);

/* bytes of device workspace ammmse_solve needs with automatic engine choice
   (0 on invalid dims) */
size_t ammmse_workspace_size(const AmmmseDims* dims);

/* same, for the engine configuration `options` selects (cluster_size /
   h_placement knobs); 0 if no configuration fits */
size_t ammmse_workspace_size_opts(const AmmmseDims* dims, const AmmmseOptions* options);

/* Solve all B realizations.  Replaces run_ammmse (solvers.py:540-550). */
int ammmse_solve(const AmmmseDims* dims, const AmmmseProblem* problem,
                 const AmmmseOptions* options, AmmmseResult* result,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Spectral bounds.  Replaces compute_bounds (objective.py:216-240).
   out: device (B, AMMMSE_BOUND_FIELDS) doubles. */
int ammmse_bounds(const AmmmseDims* dims, const void* channels, const double* weights,
                  const double* p_max, const double* noise_power, double* out, void* stream);

/* Human-readable text for an AMMMSE_ERR_* code, plus the last CUDA error of
   this thread if any. */
const char* ammmse_error_string(int code);

/* On-device synthetic inputs: for realization r of
   the batch, H (B, K, N, M) and V0 (B, K, M, d) i.i.d. CN(0,1) drawn from
   Philox4x32-10 keyed by (seed0 + r, stream tag), V0 scaled onto the power
   ball ||V0||^2 <= p_max (generate_channels model.py:197-207,
   init_precoders model.py:225-235, project_sum_power solvers.py:257-263);
   weights (B, K), optional: Uniform[0.5, 1.5) if uniform_weights else 1.
   Distributionally (not bit-) identical to the reference's numpy streams.
   Device pointers, stream-ordered. */
int ammmse_generate_iid(const AmmmseDims* dims, unsigned long long seed0, double p_max,
                        int uniform_weights, void* channels, void* init_precoders,
                        double* weights, void* stream);

/* Exact-update drivers: replace run_wmmse / run_mmmse
   (solvers.py:521-537 -> _run_bcd :415-518 with exact=True, no extrapolation):
   MMSE receivers, the standard weight update (WMMSE: weighted from t = 1;
   MMMSE: identity weights until the eps1 switch), and the exact precoder
   update (A + lambda I)^{-1} B by dual bisection (bisect_dual :276-329,
   update_precoders_exact :332-348).  fp64 throughout (complex64 inputs are
   promoted).  Same problem / result layout as ammmse_solve; options.gamma,
   gamma_safe, omega, cluster_size, h_placement, tensor_cores are ignored;
   per-realization status as for ammmse_solve (no divergence test). */
enum { AMMMSE_ALGO_WMMSE = 1, AMMMSE_ALGO_MMMSE = 2 };

size_t ammmse_exact_workspace_size(const AmmmseDims* dims);

int ammmse_solve_exact(const AmmmseDims* dims, const AmmmseProblem* problem,
                       const AmmmseOptions* options, int algorithm, double bisect_tol,
                       int bisect_max, AmmmseResult* result, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Diagnostics: the engine configuration ammmse_solve would launch for these
   dims / options.  info[8] = {cluster size (0 = single-CTA engine), H resident,
   V_old in global scratch, staging bytes, tensor-core GEMMs, shared memory bytes
   per CTA, threads per CTA, shape-specialised kernel}. */
int ammmse_plan_info(const AmmmseDims* dims, const AmmmseOptions* options, int* info);

/* Diagnostics (no reference counterpart).  In a library built with
   AMMMSE_PHASES=1 (`make PHASES=1`), ammmse_solve run with the environment
   variable AMMMSE_PROFILE_PHASES=1 accumulates per-phase thread-0 clock64
   totals of the solve kernel into the call's workspace.  This copies them
   back (synchronising `stream`), writes up to n shares into `shares` and
   returns the number of phases (0 in production builds or when nothing was
   recorded); *bcgd_first / *bcgd_count name the phases of the BCGD precoder
   step (GEMM-A + step + projection, GEMM-B).  No library-global state. */
int ammmse_phase_profile(const void* workspace, double* shares, int n, int* bcgd_first,
                         int* bcgd_count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* AMMMSE_H_ */
