// ammmse_capi.cu — extern "C" boundary of libammmse.so (include/ammmse.h).
//
// Validation mirrors the reference's construction-time checks:
//   SolverOptions.__post_init__  (pkg/src/wsrbeam/solvers.py:109-136)
//   SystemConfig.__post_init__   (pkg/src/wsrbeam/model.py:60-85)
// Per-array value checks (finite entries, sigma^2 > 0, alpha > 0) are the
// host layer's job (it owns the host copies); the ABI checks shapes, pointers
// and option ranges.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ammmse.h"
#include "ammmse_tc2.cuh"
#include "entries.h"

namespace {

thread_local char g_err[256];  // per-thread text of the last error (ammmse_error_string)

// workspace layout: [0, 8) persistent-kernel work counter, [64, 192) phase
// counters (diagnostic builds), scratch from byte 256
constexpr size_t kPhaseOff = 64;
constexpr int kPhaseN = 20;

const ammmse::KernelEntry* lookup(const AmmmseDims* d) {
  if (d->N < 1 || d->N > 4 || d->d < 1 || d->d > 4) return nullptr;
  const ammmse::KernelEntry* t = nullptr;
  if (d->dtype == AMMMSE_COMPLEX64) {
    switch (d->N) {
      case 1: t = ammmse::entries_float_1(); break;
      case 2: t = ammmse::entries_float_2(); break;
      case 3: t = ammmse::entries_float_3(); break;
      case 4: t = ammmse::entries_float_4(); break;
    }
  } else if (d->dtype == AMMMSE_COMPLEX128) {
    switch (d->N) {
      case 1: t = ammmse::entries_double_1(); break;
      case 2: t = ammmse::entries_double_2(); break;
      case 3: t = ammmse::entries_double_3(); break;
      case 4: t = ammmse::entries_double_4(); break;
    }
  }
  return t ? &t[d->d - 1] : nullptr;
}

int dims_valid(const AmmmseDims* d) {
  if (!d) return AMMMSE_ERR_INVALID;
  if (d->batch < 1 || d->M < 1 || d->N < 1 || d->K < 1 || d->d < 1) return AMMMSE_ERR_INVALID;
  if (d->dtype != AMMMSE_COMPLEX64 && d->dtype != AMMMSE_COMPLEX128) return AMMMSE_ERR_INVALID;
  return AMMMSE_OK;
}

int max_smem_optin() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  return v;
}

// Engine choice: one CTA per realization when its state fits one SM's shared
// memory, else the smallest thread-block cluster (C | K) whose per-CTA slice
// fits.  force_c >= 1 forces the cluster engine with that many CTAs.
struct Plan {
  const ammmse::KernelEntry* e;
  int cluster;  // 0: single-CTA engine; >= 1: cluster engine with that many CTAs
  int hres;     // cluster engine: H resident (1) or streamed (0)
  int vglob;    // cluster engine: V_old in global scratch
  int sb;       // cluster engine: staging bytes per buffer
  int tc;       // cluster engine: tcgen05 GEMMs (1: ammmse_cluster_kernel<TC>, 2: ammmse_tc2_kernel)
  int stages;   // tc == 2: A ring depth
  size_t smem;
  int threads;
};

int pick_threads(const AmmmseDims* d);

int make_plan(const AmmmseDims* d, int force_c, int h_placement, int tensor_cores, Plan* p) {
  const ammmse::KernelEntry* e = lookup(d);
  if (!e || !e->smem_bytes || !e->cluster_smem_bytes) return AMMMSE_ERR_UNSUPPORTED;  // (empty: dev builds)
  int lim = max_smem_optin();
  if (lim <= 0) lim = 232448;  // sm_100 opt-in limit (no device to query)
  p->e = e;
  p->hres = 1;
  p->vglob = 0;
  p->sb = 20480;
  p->tc = 0;
  p->stages = 0;
  if (force_c == 0 && h_placement == 0 && tensor_cores != 1) {
    const size_t s1 = e->smem_bytes(d->M, d->K);
    if (s1 <= (size_t)lim) {
      p->cluster = 0;
      p->smem = s1;
      p->threads = pick_threads(d);
      return AMMMSE_OK;
    }
  }
  // Smallest cluster first (per-realization cost ~ C x serial per-CTA time +
  // GEMM work, measured: massive C=4 1.55x faster than C=8), then placement:
  // H resident in every CTA; H streamed (20 KB staging buffers); H streamed with
  // V_old in a per-CTA global scratch slot (20 KB, then 12 KB staging).
  const int cands[5] = {1, 2, 4, 8, 16};
  const int modes[4][3] = {{1, 0, 20480}, {0, 0, 20480}, {0, 1, 20480}, {0, 1, 12288}};
  for (int i = 0; i < 5; ++i) {
    const int c = cands[i];
    if (force_c && c != force_c) continue;
    if (d->K % c) continue;
    for (int mi = 0; mi < 4; ++mi) {
      const int hres = modes[mi][0], vglob = modes[mi][1], sb = modes[mi][2];
      if ((h_placement == 1 && !hres) || (h_placement == 2 && (hres || vglob)) ||
          (h_placement == 3 && (hres || !vglob)))
        continue;
      // streamed H moves 16-byte pieces: complex64 rows need an even length
      if (!hres && d->dtype == AMMMSE_COMPLEX64 && (d->M % 2)) continue;
      // tensor-core GEMMs (bulk-copied pre-split H planes, TMEM accumulators):
      // forced with tensor_cores = 1; chosen automatically (tensor_cores = 0)
      // where measured faster than the FFMA GEMMs: N = d = 4 (BASELINE large,
      // 1185 vs 1052 realizations/s).  The N = d = 2 shapes keep FFMA (massive
      // 733 vs 1045, sweep256 5.6k vs 8.1k: their FFMA GEMMs already run at
      // 0.4 of the FMA peak while the per-chunk handoffs of the tensor-core
      // ring are latency bound, bench_gemmstep.py).
      const int ncol = (d->K / c) * d->d;
      // second-generation tensor-core engine (ammmse_tc2.cuh: split operands
      // resident, precoders in TMEM, one-thread A ring with cross-GEMM
      // prefetch): tensor_cores = 3, or automatically for N = d = 4
      if (mi == 0 && d->dtype == AMMMSE_COMPLEX64 && e->cluster_solve_tc2 && h_placement == 0 &&
          (tensor_cores == 3 || (tensor_cores == 0 && d->N == 4 && d->d == 4)) &&
          ammmse::tc2::shape_ok(d->M, d->K * d->N, ncol)) {
        const int st = e->tc2_stages(d->M, d->K, c, (size_t)lim - 2048);  // static shared: ctl, barriers, exchange copy
        if (st >= 2) {
          p->cluster = c;
          p->hres = 0;
          p->vglob = 0;
          p->sb = 0;
          p->tc = 2;
          p->stages = st;
          p->smem = e->tc2_smem_bytes(d->M, d->K, c, st);
          p->threads = 256;
          return AMMMSE_OK;
        }
      }
      if (tensor_cores == 3) continue;
      const bool tc_auto = tensor_cores == 0 && d->N == 4 && d->d == 4;
      if (!hres && d->dtype == AMMMSE_COMPLEX64 && (tensor_cores == 1 || tc_auto) &&
          ammmse::tc_shape_ok(d->M, d->K * d->N, ncol)) {
        const size_t st = e->cluster_smem_bytes(d->M, d->K, c, hres, vglob, sb, 1);
        if (st <= (size_t)lim) {
          p->cluster = c;
          p->hres = hres;
          p->vglob = vglob;
          p->sb = sb;
          p->tc = 1;
          p->smem = st;
          p->threads = 256;
          return AMMMSE_OK;
        }
      }
      if (tensor_cores == 1) continue;
      const size_t s = e->cluster_smem_bytes(d->M, d->K, c, hres, vglob, sb, 0);
      if (s <= (size_t)lim) {
        p->cluster = c;
        p->hres = hres;
        p->vglob = vglob;
        p->sb = sb;
        p->smem = s;
        p->threads = 256;  // kClusterThreads
        return AMMMSE_OK;
      }
    }
  }
  return AMMMSE_ERR_UNSUPPORTED;
}

// Threads per CTA: about one 2x2 output tile of the larger GEMM per thread,
// 64..256, multiple of 32.
int pick_threads(const AmmmseDims* d) {
  const long tiles_a = (long)((d->M + 1) / 2) * (((long)d->K * d->d + 1) / 2);
  const long tiles_b = (long)((d->K * d->N + 1) / 2) * (((long)d->K * d->d + 1) / 2);
  long t = tiles_a > tiles_b ? tiles_a : tiles_b;
  t = (t + 31) / 32 * 32;
  if (t < 64) t = 64;
  if (t > 256) t = 256;
  return (int)t;
}

int cuda_fail(cudaError_t e, const char* what) {
  snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return AMMMSE_ERR_CUDA;
}

// tensor-core mode: pre-split H / H^T planes (8 planes of KN x M floats) per
// resident cluster (one CTA per SM -> at most sms / C clusters), after the
// V_old slots
size_t tc_planes_bytes(const AmmmseDims* d, const Plan& p, int sms) {
  const size_t per = (size_t)8 * d->K * d->N * d->M * 4;
  return (size_t)((sms + p.cluster - 1) / p.cluster) * per + 256;
}

// row stride of the per-CTA V_old slot (CLayout::ldv: padded in tensor-core mode)
size_t vold_ld(const AmmmseDims* d, const Plan& p) {
  const size_t ncol = (size_t)(d->K / p.cluster) * d->d;
  return p.tc ? ncol + 1 : ncol;
}

// bytes of per-CTA V_old scratch (cluster engine, vglob plans); one CTA per SM
// is resident for those plans, so the slot count is bounded by the SM count
size_t scratch_bytes(const AmmmseDims* d, const Plan& p) {
  if (!p.cluster || (!p.vglob && !p.tc)) return 0;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 160;
  const size_t rsz = d->dtype == AMMMSE_COMPLEX64 ? 4 : 8;
  size_t b = p.vglob ? (size_t)sms * 2 * (size_t)d->M * vold_ld(d, p) * rsz : 0;
  if (p.tc) b = ((b + 255) & ~(size_t)255) + tc_planes_bytes(d, p, sms);
  return b;
}

}  // namespace

extern "C" {

int ammmse_abi_version(void) { return AMMMSE_ABI_VERSION; }

int ammmse_check_dims(const AmmmseDims* dims) {
  int rc = dims_valid(dims);
  if (rc) return rc;
  Plan p;
  return make_plan(dims, 0, 0, 0, &p);
}

size_t ammmse_workspace_size(const AmmmseDims* dims) {
  if (dims_valid(dims)) return 0;
  Plan p;
  if (make_plan(dims, 0, 0, 0, &p) != AMMMSE_OK) return 256;
  return 256 + scratch_bytes(dims, p);  // work counter (padded) + V_old scratch
}

size_t ammmse_workspace_size_opts(const AmmmseDims* dims, const AmmmseOptions* opt) {
  if (dims_valid(dims) || !opt) return 0;
  Plan p;
  if (make_plan(dims, opt->cluster_size, opt->h_placement, opt->tensor_cores, &p) != AMMMSE_OK)
    return 0;
  return 256 + scratch_bytes(dims, p);
}

int ammmse_solve(const AmmmseDims* dims, const AmmmseProblem* prob, const AmmmseOptions* opt,
                 AmmmseResult* res, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = ammmse_check_dims(dims);
  if (rc) {
    snprintf(g_err, sizeof g_err, "unsupported or invalid dims");
    return rc;
  }
  if (!prob || !opt || !res || !prob->channels || !prob->noise_power || !prob->p_max ||
      !prob->weights || !prob->init_precoders) {
    snprintf(g_err, sizeof g_err, "null problem/options/result pointer");
    return AMMMSE_ERR_INVALID;
  }
  // SolverOptions checks (solvers.py:112-132)
  if (!prob->gamma && !opt->gamma_safe && !(isfinite(opt->gamma) && opt->gamma > 0)) {
    snprintf(g_err, sizeof g_err, "gamma must be positive, got %g", opt->gamma);
    return AMMMSE_ERR_INVALID;
  }
  if (!prob->omega && !(opt->omega >= 0.0 && opt->omega < 1.0)) {
    snprintf(g_err, sizeof g_err, "omega must lie in [0, 1), got %g", opt->omega);
    return AMMMSE_ERR_INVALID;
  }
  if (!(opt->eps1 > 0)) {
    snprintf(g_err, sizeof g_err, "eps1 must be positive");
    return AMMMSE_ERR_INVALID;
  }
  if (!(opt->eps2 > 0 && isfinite(opt->eps2)) || opt->eps2 > opt->eps1) {
    snprintf(g_err, sizeof g_err, "eps2 must be positive, finite and <= eps1");
    return AMMMSE_ERR_INVALID;
  }
  if (opt->max_iters < 1) {
    snprintf(g_err, sizeof g_err, "max_iters must be at least 1");
    return AMMMSE_ERR_INVALID;
  }
  if (!workspace || workspace_bytes < 256) {
    snprintf(g_err, sizeof g_err, "workspace missing or too small");
    return AMMMSE_ERR_WORKSPACE;
  }
  Plan plan;
  if (opt->cluster_size < 0 || opt->h_placement < 0 || opt->h_placement > 3 ||
      opt->tensor_cores < 0 || opt->tensor_cores > 3 ||
      make_plan(dims, opt->cluster_size, opt->h_placement, opt->tensor_cores, &plan) != AMMMSE_OK) {
    snprintf(g_err, sizeof g_err, "no engine configuration fits (cluster_size %d)", opt->cluster_size);
    return AMMMSE_ERR_UNSUPPORTED;
  }
  if (workspace_bytes < 256 + scratch_bytes(dims, plan)) {
    snprintf(g_err, sizeof g_err, "workspace missing or too small");
    return AMMMSE_ERR_WORKSPACE;
  }
  const void* func = plan.cluster ? (plan.tc == 2   ? plan.e->cluster_solve_tc2
                                     : plan.tc ? plan.e->cluster_solve_tc
                                               : plan.e->cluster_solve)
                                  : plan.e->solve;
  {  // shape-specialised single-CTA kernel (AMMMSE_NO_SPEC=1 disables it, for A/B)
    const char* ns = getenv("AMMMSE_NO_SPEC");
    const bool use_spec = !(ns && ns[0] == '1');
    if (use_spec && !plan.cluster)
      for (int i = 0; i < plan.e->n_solve_specs; ++i) {
        const ammmse::SpecEntry& sp = plan.e->solve_specs[i];
        if (sp.M == dims->M && sp.K == dims->K && sp.T == plan.threads) func = sp.f;
      }
    if (use_spec && plan.cluster && !plan.tc)
      for (int i = 0; i < plan.e->n_cluster_specs; ++i) {
        const ammmse::SpecEntry& sp = plan.e->cluster_specs[i];
        const bool place_ok = sp.sb == 0 || (!plan.hres && plan.vglob && plan.sb == sp.sb);
        if (sp.M == dims->M && sp.K == dims->K && sp.C == plan.cluster && sp.T == plan.threads &&
            place_ok)
          func = sp.f;
      }
  }
  if (!func) {
    snprintf(g_err, sizeof g_err, "no kernel instantiation for this plan");
    return AMMMSE_ERR_UNSUPPORTED;
  }
  const size_t smem = plan.smem;
  const int threads = plan.threads;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

  cudaError_t ce = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaFuncSetAttribute");
  long long grid = 0;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cudaLaunchAttribute attr[1];
  if (plan.cluster) {
    if (plan.cluster > 8) {
      ce = cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (ce != cudaSuccess) return cuda_fail(ce, "non-portable cluster size");
    }
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)plan.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.gridDim = dim3((unsigned)(plan.cluster * sms));
    int nclusters = 0;
    ce = cudaOccupancyMaxActiveClusters(&nclusters, func, &cfg);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaOccupancyMaxActiveClusters");
    if (nclusters < 1) {
      snprintf(g_err, sizeof g_err, "cluster of %d CTAs with %zu B smem cannot be resident", plan.cluster, smem);
      return AMMMSE_ERR_UNSUPPORTED;
    }
    long long nc = nclusters < dims->batch ? nclusters : dims->batch;
    // per-CTA global scratch slots (V_old, tensor-core H planes) are sized for
    // at most one CTA per SM (scratch_bytes): never launch more
    if ((plan.vglob || plan.tc) && nc * plan.cluster > sms) nc = sms / plan.cluster;
    grid = nc * plan.cluster;
    cfg.gridDim = dim3((unsigned)grid);
  } else {
    int per_sm = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
    if (ce != cudaSuccess) return cuda_fail(ce, "occupancy");
    if (per_sm < 1) {
      snprintf(g_err, sizeof g_err, "kernel does not fit on an SM (smem %zu)", smem);
      return AMMMSE_ERR_UNSUPPORTED;
    }
    grid = (long long)sms * per_sm;
    if (grid > dims->batch) grid = dims->batch;
  }

  ce = cudaMemsetAsync(workspace, 0, 8, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemsetAsync");

  ammmse::EngineArgs a;
  memset(&a, 0, sizeof a);
  a.H = prob->channels;
  a.sigma2 = prob->noise_power;
  a.pmax = prob->p_max;
  a.alpha = prob->weights;
  a.V0 = prob->init_precoders;
  a.gamma_arr = prob->gamma;
  a.omega_arr = prob->omega;
  a.Vout = res->final_precoders;
  a.wsr_bits = res->wsr_bits;
  a.iterations = res->iterations;
  a.converged = res->converged;
  a.residual = res->stationarity_residual;
  a.switch_it = res->switch_iteration;
  a.status = res->status;
  a.gamma_used = res->gamma_used;
  a.trace = res->trace;
  if ((res->iter_receivers != nullptr) != (res->iter_weights != nullptr) ||
      (res->iter_receivers != nullptr) != (res->iter_precoders != nullptr)) {
    snprintf(g_err, sizeof g_err, "iterate buffers must be all set or all NULL");
    return AMMMSE_ERR_INVALID;
  }
  a.itU = res->iter_receivers;
  a.itW = res->iter_weights;
  a.itV = res->iter_precoders;
  a.gamma = opt->gamma;
  a.gamma_safe = opt->gamma_safe ? 1 : 0;
  a.omega = opt->omega;
  a.eps1 = opt->eps1;
  a.eps2 = opt->eps2;
  a.max_iters = opt->max_iters;
  a.latch = opt->latch_stage ? 1 : 0;
  a.M = dims->M;
  a.K = dims->K;
  a.B = dims->batch;
  a.hres = plan.cluster ? plan.hres : 1;
  a.vold_glob = plan.cluster ? plan.vglob : 0;
  a.sb_bytes = plan.sb;
  a.scratch = reinterpret_cast<unsigned char*>(workspace) + 256;
  a.tcm = plan.cluster ? plan.tc : 0;
  a.tc_stages = plan.stages;
  {  // tuning knob (A/B measurements): AMMMSE_TC2_DEFER=1 moves WSR(t) into GEMM-A(t+1)
     // once the stage is latched.  Off by default: measured 1872 vs 1980 realizations/s on
     // BASELINE large (K1(t+1) is as long as WSR(t), so hiding WSR alone does not pay).
    const char* de = getenv("AMMMSE_TC2_DEFER");
    a.tc_defer = (de && de[0] == '1') ? 1 : 0;
    // A/B knob: AMMMSE_TC2_WSR_SPLIT=1 runs WSR(t) on two warps (A / C factorisations
    // concurrently).  Off by default: measured 2 158 vs 2 212 realizations/s (K1(t+1) on
    // warps 1-2 bounds the phase; the extra warp and named barrier only add contention).
    const char* ws = getenv("AMMMSE_TC2_WSR_SPLIT");
    a.tc_wsr_split = (ws && ws[0] == '1') ? 1 : 0;
  }
  if (a.tcm) {  // H planes after the V_old slots, 256-byte aligned
    int sms2 = 0;
    cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev);
    const size_t rsz = dims->dtype == AMMMSE_COMPLEX64 ? 4 : 8;
    size_t off = plan.vglob ? (size_t)sms2 * 2 * (size_t)dims->M * vold_ld(dims, plan) * rsz : 0;
    off = (off + 255) & ~(size_t)255;
    a.hplanes = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(workspace) + 256 + off);
  }
  a.counter = reinterpret_cast<unsigned long long*>(workspace);
  // diagnostic builds (AMMMSE_PHASES=1) with AMMMSE_PROFILE_PHASES=1: per-phase
  // thread-0 clock64 totals into the caller's workspace (ammmse_phase_profile)
  if (AMMMSE_PHASES) {
    const char* de = getenv("AMMMSE_DBG");
    a.dbg = de ? atoi(de) : 0;
    const char* pe = getenv("AMMMSE_PROFILE_PHASES");
    if (pe && pe[0] == '1') {
      a.prof = reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(workspace) + kPhaseOff);
      ce = cudaMemsetAsync(a.prof, 0, kPhaseN * sizeof(unsigned long long), s);
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemsetAsync(phases)");
    }
  }
  void* args[] = {&a};
  if (plan.cluster)
    ce = cudaLaunchKernelExC(&cfg, func, args);
  else
    ce = cudaLaunchKernel(func, dim3((unsigned)grid), dim3(threads), args, smem, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "kernel launch (solve)");
  return AMMMSE_OK;
}

int ammmse_plan_info(const AmmmseDims* dims, const AmmmseOptions* opt, int* info) {
  int rc = dims_valid(dims);
  if (rc) return rc;
  if (!opt || !info) return AMMMSE_ERR_INVALID;
  Plan p;
  rc = make_plan(dims, opt->cluster_size, opt->h_placement, opt->tensor_cores, &p);
  if (rc) return rc;
  int spec = 0;
  if (!p.cluster) {
    for (int i = 0; i < p.e->n_solve_specs; ++i)
      if (p.e->solve_specs[i].M == dims->M && p.e->solve_specs[i].K == dims->K &&
          p.e->solve_specs[i].T == p.threads)
        spec = 1;
  } else if (!p.tc) {
    for (int i = 0; i < p.e->n_cluster_specs; ++i) {
      const ammmse::SpecEntry& sp = p.e->cluster_specs[i];
      const bool place_ok = sp.sb == 0 || (!p.hres && p.vglob && p.sb == sp.sb);
      if (sp.M == dims->M && sp.K == dims->K && sp.C == p.cluster && sp.T == p.threads && place_ok)
        spec = 1;
    }
  }
  info[0] = p.cluster;
  info[1] = p.hres;
  info[2] = p.vglob;
  info[3] = p.sb;
  info[4] = p.tc;
  info[5] = (int)p.smem;
  info[6] = p.threads;
  info[7] = spec;
  return AMMMSE_OK;
}

int ammmse_phase_profile(const void* workspace, double* shares, int n, int* bcgd_first,
                         int* bcgd_count, void* stream) {
  if (bcgd_first) *bcgd_first = 2;
  if (bcgd_count) *bcgd_count = 2;
  if (!AMMMSE_PHASES) return 0;
  if (!workspace) return AMMMSE_ERR_INVALID;
  unsigned long long h[kPhaseN];
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t ce = cudaMemcpyAsync(h, reinterpret_cast<const unsigned char*>(workspace) + kPhaseOff,
                                   sizeof h, cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return cuda_fail(ce, "phase counters");
  double tot = 0;
  for (int i = 0; i < kPhaseN; ++i) tot += (double)h[i];
  if (shares)
    for (int i = 0; i < n && i < kPhaseN; ++i) shares[i] = tot > 0 ? (double)h[i] / tot : 0.0;
  return tot > 0 ? kPhaseN : 0;
}

int ammmse_bounds(const AmmmseDims* dims, const void* channels, const double* weights,
                  const double* p_max, const double* noise_power, double* out, void* stream) {
  int rc = dims_valid(dims);
  if (rc) return rc;
  const ammmse::KernelEntry* e = lookup(dims);
  if (!e) return AMMMSE_ERR_UNSUPPORTED;
  if (dims->K > 1024) return AMMMSE_ERR_UNSUPPORTED;
  if (!channels || !weights || !p_max || !noise_power || !out) return AMMMSE_ERR_INVALID;
  const void* H = channels;
  int M = dims->M, K = dims->K;
  long long B = dims->batch;
  void* args[] = {(void*)&H, (void*)&weights, (void*)&p_max, (void*)&noise_power, &M, &K, &B, &out};
  cudaError_t ce = cudaLaunchKernel(e->bounds, dim3((unsigned)B), dim3(128), args, 0, (cudaStream_t)stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaLaunchKernel(bounds)");
  return AMMMSE_OK;
}

const char* ammmse_error_string(int code) {
  static thread_local char buf[384];
  const char* base = "unknown error";
  switch (code) {
    case AMMMSE_OK: base = "ok"; break;
    case AMMMSE_ERR_INVALID: base = "invalid argument"; break;
    case AMMMSE_ERR_UNSUPPORTED: base = "unsupported shape"; break;
    case AMMMSE_ERR_WORKSPACE: base = "workspace too small"; break;
    case AMMMSE_ERR_CUDA: base = "CUDA error"; break;
  }
  snprintf(buf, sizeof buf, "%s%s%s", base, g_err[0] ? ": " : "", g_err);
  return buf;
}

}  // extern "C"
