// Latency / throughput probes for the tc2 pipeline building blocks (one CTA per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_20507_b200/csrc/tc_umma.cuh"
using namespace ammmse;

__device__ __forceinline__ void wait_try(uint64_t* b, uint32_t par) { umma::mbar_wait(b, par); }
__device__ __forceinline__ void wait_test(uint64_t* b, uint32_t par) { umma::mbar_wait_spin(b, par); }

// out[0]: ping-pong round trip (try_wait), out[1]: (test_wait), out[2]: commit->arrive latency,
// out[3]: bulk copy 16 KB latency, out[4]: 16 x 16 KB through a 3-stage ring (cycles total),
// out[5..7]: cycles per MMA for N = 64 / 128 / 256 (32 back-to-back, same accumulator)
// out[8]: ring with 6 stages of 8 KB
__global__ void __launch_bounds__(256, 1) probe(const unsigned char* g, long long* out, int iters) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t ba, bb, bf[8], bd[8];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    umma::mbar_init(&ba, 1);
    umma::mbar_init(&bb, 1);
    for (int i = 0; i < 8; ++i) { umma::mbar_init(&bf[i], 1); umma::mbar_init(&bd[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc<512>(&tslot);
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;
  long long t0, t1;
  // ---- A: ping-pong ----
  for (int variant = 0; variant < 2; ++variant) {
    __syncthreads();
    if (warp == 0 && lane == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        umma::mbar_arrive(&ba);
        const uint32_t par = (uint32_t)((variant * iters + i) & 1);
        if (variant == 0) wait_try(&bb, par); else wait_test(&bb, par);
      }
      t1 = clock64();
      if (blockIdx.x == 0) out[variant] = (t1 - t0) / iters;
    } else if (warp == 1 && lane == 0) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t par = (uint32_t)((variant * iters + i) & 1);
        if (variant == 0) wait_try(&ba, par); else wait_test(&ba, par);
        umma::mbar_arrive(&bb);
      }
    }
  }
  __syncthreads();
  // ---- B: commit latency (no MMAs pending) ----
  if (tid == 0) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      umma::commit(&bf[0]);
      wait_test(&bf[0], (uint32_t)(i & 1));
    }
    t1 = clock64();
    if (blockIdx.x == 0) out[2] = (t1 - t0) / iters;
  }
  __syncthreads();
  // ---- C: bulk copy latency, 16 KB, L2 warm (bf[1]) ----
  const unsigned char* src = g + (size_t)(blockIdx.x / 4) * (512 * 1024);
  if (tid == 0) {
    uint32_t ph = 0;
    for (int i = 0; i < 4; ++i) {  // warm
      umma::mbar_arrive_expect_tx(&bf[1], 16384);
      umma::bulk_g2s(smem, src + i * 16384, 16384, &bf[1]);
      wait_test(&bf[1], ph & 1); ++ph;
    }
    t0 = clock64();
    for (int i = 0; i < 16; ++i) {
      umma::mbar_arrive_expect_tx(&bf[1], 16384);
      umma::bulk_g2s(smem, src + i * 16384, 16384, &bf[1]);
      wait_test(&bf[1], ph & 1); ++ph;
    }
    t1 = clock64();
    if (blockIdx.x == 0) out[3] = (t1 - t0) / 16;
  }
  __syncthreads();
  // ---- C2: 16 chunks of 16 KB through S stages (consumer releases immediately) ----
  for (int cfg = 0; cfg < 3; ++cfg) {
    const int S = cfg == 0 ? 3 : (cfg == 1 ? 6 : 8);
    const uint32_t bytes = cfg == 0 ? 16384 : (cfg == 1 ? 8192 : 16384);
    const int n = cfg == 1 ? 32 : 16;
    __syncthreads();
    // fresh barriers for each cfg
    if (tid == 0) {
      for (int i = 0; i < 8; ++i) { umma::mbar_init(&bf[i], 1); umma::mbar_init(&bd[i], 1); }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 1 && lane == 0) {
      for (int rep = 0; rep < 8; ++rep)
        for (int c = 0; c < n; ++c) {
          const int q = rep * n + c, s = q % S, use = q / S;
          if (use > 0) wait_test(&bd[s], (uint32_t)((use - 1) & 1));
          umma::mbar_arrive_expect_tx(&bf[s], bytes);
          umma::bulk_g2s(smem + (size_t)s * bytes, src + (size_t)c * bytes, bytes, &bf[s]);
        }
    } else if (tid == 0) {
      t0 = clock64();
      for (int rep = 0; rep < 8; ++rep)
        for (int c = 0; c < n; ++c) {
          const int q = rep * n + c, s = q % S;
          wait_test(&bf[s], (uint32_t)((q / S) & 1));
          umma::mbar_arrive(&bd[s]);
        }
      t1 = clock64();
      if (blockIdx.x == 0) out[cfg == 0 ? 4 : (cfg == 1 ? 8 : 9)] = (t1 - t0) / 8;
    }
  }
  __syncthreads();
  // ---- D: MMA issue/execute time ----
  for (int v = 0; v < 3; ++v) {
    const int N = 64 << v;
    __syncthreads();
    if (tid == 0) {
      umma::mbar_init(&bf[2], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      const uint32_t idesc = umma::make_idesc_tf32(128, N, false, false, false, false);
      const uint64_t ad = umma::make_sdesc(umma::smem_u32(smem), 128, 256);
      const uint64_t bd2 = umma::make_sdesc(umma::smem_u32(smem + 65536), 128, 256);
      t0 = clock64();
      for (int i = 0; i < 64; ++i) umma::mma_tf32(tmem, ad, bd2, idesc, i ? 1u : 0u);
      umma::commit(&bf[2]);
      const long long t_issue = clock64();
      wait_test(&bf[2], 0);
      t1 = clock64();
      if (blockIdx.x == 0) { out[5 + v] = (t1 - t0) / 64; out[10 + v] = (t_issue - t0) / 64; }
    }
  }
  __syncthreads();
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<512>(tmem);
}

int main() {
  unsigned char* g;
  long long* out;
  cudaMalloc(&g, 64 << 20);
  cudaMemset(g, 0, 64 << 20);
  cudaMallocManaged(&out, 64 * sizeof(long long));
  for (int i = 0; i < 64; ++i) out[i] = -1;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 132}) {
    probe<<<grid, 256, 200 * 1024>>>(g, out, 1000);
    cudaError_t e = cudaDeviceSynchronize();
    printf("grid %d: %s\n", grid, cudaGetErrorString(e));
    printf(" pingpong try_wait %lld  test_wait %lld  commit %lld  bulk16K latency %lld\n", out[0], out[1], out[2], out[3]);
    printf(" ring 3x16K: %lld cycles / 256 KB   6x8K: %lld   8x16K: %lld\n", out[4], out[8], out[9]);
    printf(" MMA cycles each (exec / issue): N=64 %lld/%lld  N=128 %lld/%lld  N=256 %lld/%lld\n", out[5], out[10], out[6], out[11], out[7], out[12]);
  }
  return 0;
}
