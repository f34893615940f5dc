// mbarrier op cost: default (acquire/release) vs relaxed; 2-thread ring of S=3, no copies
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_20507_b200/csrc/tc_umma.cuh"
using namespace ammmse;
template <bool RELAXED>
__device__ __forceinline__ void wait_u32(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  do {
    if (RELAXED)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(mbar), "r"(parity) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(mbar), "r"(parity) : "memory");
  } while (!ok);
}
template <bool RELAXED>
__device__ __forceinline__ void arrive_u32(uint32_t mbar) {
  if (RELAXED) asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
  else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}
constexpr int S = 3, N = 256;
template <bool RELAXED>
__global__ void __launch_bounds__(256, 1) probe(long long* out, int slot) {
  __shared__ uint64_t bf[4], bd[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { umma::mbar_init(&bf[i], 1); umma::mbar_init(&bd[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint32_t f0 = umma::smem_u32(bf), d0 = umma::smem_u32(bd);
  if (warp == 1) {
    if (lane == 0) {
      uint32_t par = 1;  // first pass: no wait
      bool first = true;
      for (int q = 0; q < N; q += 3) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          if (!first) wait_u32<RELAXED>(d0 + 8 * s, par);
          arrive_u32<RELAXED>(f0 + 8 * s);
        }
        if (!first) par ^= 1; else { first = false; par = 0; }
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    if (lane == 0) {
      long long t0 = clock64();
      uint32_t par = 0;
      for (int q = 0; q < N; q += 3) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          wait_u32<RELAXED>(f0 + 8 * s, par);
          arrive_u32<RELAXED>(d0 + 8 * s);
        }
        par ^= 1;
      }
      long long t1 = clock64();
      if (blockIdx.x == 0) out[slot] = (t1 - t0) / N;
    }
    __syncwarp();
  }
  __syncthreads();
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 64 * sizeof(long long));
  probe<false><<<132, 256>>>(out, 0);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  probe<true><<<132, 256>>>(out, 1);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  printf("ring S=3 handshake only, unrolled: default %lld cycles/chunk, relaxed %lld cycles/chunk\n", out[0], out[1]);
  return 0;
}
