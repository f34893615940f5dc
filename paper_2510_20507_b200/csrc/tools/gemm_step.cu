// gemm_step.cu — standalone driver of the cluster engine's tensor-core GEMM
// (tc_stream.cuh) for validation and for the GEMM-step measurement
// (bench_gemmstep.py, tests/test_gpu_gemmstep.py).  Built into
// libammmse_gemmstep.so; not on the solve path.
//
// One CTA of 256 threads per problem, `nprob` problems (a persistent grid of
// one CTA per SM loops over them), exactly the engine's data layout:
//   H   (KN x M) interleaved complex64 in global, split once per problem into
//       the chunk-major planes of H (rows r, K = m) and H^T (rows m, K = r);
//   B   fp32 planar in shared memory, element (k, q) at k * ldb + q, ldb = ncol + 1;
//   D   written back interleaved (rows x ncol complex).
// mode 0: D = H X   (GEMM-B, K = M, X is M x ncol)
// mode 1: D = H^H Y (GEMM-A, K = KN, Y is KN x ncol)
// reps > 1 repeats the GEMM + epilogue on the same operands (timing);
// mode | 2 selects the gemm_sync schedule; mode | (DBG << 2) the tcs::gemm<DBG>
// ablations (timing only: results are not meaningful).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../tc_stream.cuh"

using namespace ammmse;

namespace {

constexpr int kStages = 4;

__global__ void __launch_bounds__(256, 1)
    gemm_step_kernel(const float2* __restrict__ H, const float2* __restrict__ Bsrc,
                     float2* __restrict__ D, float* __restrict__ planes, int nprob, int KN, int M,
                     int ncol, int mode, int reps, int share) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kStages], bready[kStages], done[kStages], fin;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  const int sched = mode & 2;           // 2: gemm_sync schedule (A/B)
  const int ablate = (mode >> 2) & 7;   // tcs::gemm<DBG> diagnostics (timing only)
  mode &= 1;
  const int rows = mode == 0 ? KN : M;  // output rows
  const int kd = mode == 0 ? M : KN;    // contraction
  const int tm = rows >= 128 ? 128 : 64;
  const int ldb = ncol + 1;
  const int maxr = KN > M ? KN : M;
  tcs::Pipe p;
  p.ring = smem;
  p.S = kStages;
  p.a_bytes = 4 * maxr * tcs::KW * 4;
  p.stage_bytes = p.a_bytes + 4 * ncol * tcs::KW * 4;
  p.full = full;
  p.bready = bready;
  p.done = done;
  p.fin = &fin;
  float* Bs = reinterpret_cast<float*>(smem + (size_t)kStages * p.stage_bytes);
  float* Bsi = Bs + (size_t)kd * ldb;
  if (tid == 0) {
    for (int q = 0; q < kStages; ++q) {
      umma::mbar_init(&full[q], 1);
      umma::mbar_init(&bready[q], 1);
      umma::mbar_init(&done[q], 1);
    }
    umma::mbar_init(&fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if ((tid >> 5) == 0) umma::tmem_alloc<512>(&tslot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  p.tmem = tslot;
  tcs::Seq seq;
  // `share` consecutive CTAs use one plane slot (a realization's cluster shares
  // its H planes in the engine); they split identical values into it
  float* slot = planes + (size_t)(blockIdx.x / share) * 8 * KN * M;
  const float* hp = slot + (mode == 0 ? 0 : (size_t)4 * KN * M);
  for (int pb = blockIdx.x; pb < nprob; pb += gridDim.x) {
    const float2* Hg = H + (size_t)(pb / share * share) * KN * M;
    tcs::split_h(Hg, KN, M, mode == 1, slot + (mode == 0 ? 0 : (size_t)4 * KN * M), 0, KN);
    umma::fence_proxy_async_global();
    __threadfence();
    const float2* Bg = Bsrc + (size_t)pb * kd * ncol;
    for (int i = tid; i < kd * ncol; i += blockDim.x) {
      const int k = i / ncol, q = i - k * ncol;
      Bs[k * ldb + q] = Bg[i].x;
      Bsi[k * ldb + q] = Bg[i].y;
    }
    __syncthreads();
    float2* Dg = D + (size_t)pb * rows * ncol;
    for (int r = 0; r < reps; ++r) {
      if (sched)
        tcs::gemm_sync(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      else if (ablate == 1)
        tcs::gemm<1>(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      else if (ablate == 2)
        tcs::gemm<2>(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      else if (ablate == 4)
        tcs::gemm<4>(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      else if (ablate == 7)
        tcs::gemm<7>(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      else
        tcs::gemm(p, seq, hp, tm, rows / tm, kd, ncol, Bs, Bsi, ldb);
      tcs::for_each(p, tm, rows / tm, ncol, kd, mode == 1, [&](int row, int q, float re, float im) {
        if (r == reps - 1) Dg[(size_t)row * ncol + q] = make_float2(re, im);
      });
      __syncthreads();
    }
  }
  __syncthreads();
  if ((tid >> 5) == 0) umma::tmem_dealloc<512>(p.tmem);
}

bool tcs_shape_ok_host(int KN, int M, int ncol) {
  auto rows_ok = [](int r) { return r == 64 || (r % 128 == 0 && r > 0); };
  if (!rows_ok(M) || !rows_ok(KN) || ncol % 16 || 4 * ncol > 256) return false;
  const int t = (M > KN ? M : KN) / 128 > 0 ? (M > KN ? M : KN) / 128 : 1;
  return 8 * ncol * t <= 512;
}

}  // namespace

extern "C" {

// Bytes of the per-CTA plane scratch for `grid` CTAs.
size_t ammmse_gemmstep_scratch(int KN, int M, int grid) { return (size_t)grid * 8 * KN * M * 4; }

// Returns 0 or a CUDA error code.  grid <= 0: one CTA per SM.  share: CTAs per
// H-plane slot (problems pb of a group use H of the group's first problem).
int ammmse_gemmstep_run(const void* H, const void* B, void* D, void* scratch, int nprob, int KN,
                        int M, int ncol, int mode, int reps, int grid, int share, void* stream) {
  if (share < 1) share = 1;
  if (!tcs_shape_ok_host(KN, M, ncol)) return -1;
  const int maxr = KN > M ? KN : M;
  const int kd = (mode & 1) == 0 ? M : KN;
  const size_t smem = (size_t)kStages * (4 * maxr * tcs::KW * 4 + 4 * ncol * tcs::KW * 4) +
                      (size_t)2 * kd * (ncol + 1) * 4;
  cudaError_t e = cudaFuncSetAttribute(gemm_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  if (grid <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev);
  }
  if (grid > nprob) grid = nprob;
  gemm_step_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(
      (const float2*)H, (const float2*)B, (float2*)D, (float*)scratch, nprob, KN, M, ncol, mode, reps,
      share);
  return (int)cudaGetLastError();
}

}  // extern "C"
