// bulk-copy throughput vs copy size (one CTA per SM), L2-warm source
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_20507_b200/csrc/tc_umma.cuh"
using namespace ammmse;
__global__ void __launch_bounds__(256, 1) probe(const unsigned char* g, long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bf;
  const int tid = threadIdx.x;
  const unsigned char* src = g + (size_t)(blockIdx.x / 4) * (512 * 1024);
  int slot = 0;
  uint32_t ph = 0;
  if (tid == 0) { umma::mbar_init(&bf, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  __syncthreads();
  for (int rep = 0; rep < 2; ++rep)
  for (uint32_t bytes = 2048; bytes <= 65536; bytes *= 2) {
    const int total = 128 * 1024;
    const int n = total / bytes;
    if (tid == 0) {
      long long t0 = clock64();
      umma::mbar_arrive_expect_tx(&bf, total);
      for (int i = 0; i < n; ++i) umma::bulk_g2s(smem + (size_t)i * bytes, src + (size_t)i * bytes, bytes, &bf);
      long long t1 = clock64();
      umma::mbar_wait_spin(&bf, ph & 1); ++ph;
      long long t2 = clock64();
      if (blockIdx.x == 0 && rep == 1) { out[slot] = t2 - t0; out[slot + 16] = t1 - t0; }
      ++slot;
    }
    __syncthreads();
  }
}
int main() {
  unsigned char* g; long long* out;
  cudaMalloc(&g, 64 << 20); cudaMemset(g, 0, 64 << 20);
  cudaMallocManaged(&out, 64 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 132}) {
    probe<<<grid, 256, 200 * 1024>>>(g, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("grid %d: %s\n", grid, cudaGetErrorString(e));
    int slot = 6;  // rep 1 slots
    for (uint32_t bytes = 2048; bytes <= 65536; bytes *= 2, ++slot)
      printf("  128 KB in %5u-byte copies: %lld cycles total (issue %lld) -> %.1f B/clk\n", bytes, out[slot], out[slot + 16], 131072.0 / out[slot]);
  }
  return 0;
}
