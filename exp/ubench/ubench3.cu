// handshake-loop probes: 2 role threads (warp 0 lane 0 = consumer/MMA, warp 1 lane 0 = producer)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_20507_b200/csrc/tc_umma.cuh"
using namespace ammmse;
constexpr int S = 3, NCH = 16, REPS = 16;
__global__ void __launch_bounds__(256, 1) probe(const unsigned char* g, long long* out, int variant, int copies, int spinners) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bf[8], bd[8], fin;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) { umma::mbar_init(&bf[i], 1); umma::mbar_init(&bd[i], 1); }
    umma::mbar_init(&fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc<512>(&tslot);
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;
  const unsigned char* src = g + (size_t)(blockIdx.x / 4) * (512 * 1024);
  const uint32_t idesc = umma::make_idesc_tf32(128, 64, false, false, false, false);
  long long t0 = 0, t1 = 0;
  if (warp == 1) {
    if (lane == 0) {
      for (int q = 0; q < REPS * NCH; ++q) {
        const int s = q % S, use = q / S;
        if (use > 0) umma::mbar_wait_spin(&bd[s], (uint32_t)((use - 1) & 1));
        if (copies) {
          umma::mbar_arrive_expect_tx(&bf[s], 16384);
          umma::bulk_g2s(smem + (size_t)s * 16384, src + (size_t)(q % NCH) * 16384, 16384, &bf[s]);
        } else {
          umma::mbar_arrive(&bf[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    if (lane == 0) {
      t0 = clock64();
      for (int q = 0; q < REPS * NCH; ++q) {
        const int s = q % S;
        umma::mbar_wait_spin(&bf[s], (uint32_t)((q / S) & 1));
        if (variant >= 1) umma::fence_after();
        if (variant >= 3) {
          const uint64_t ad = umma::make_sdesc(umma::smem_u32(smem + (size_t)s * 16384), 128, 256);
          const uint64_t bdsc = umma::make_sdesc(umma::smem_u32(smem + 65536 + (q % NCH) * 4128), 128, 256);
          for (int i = 0; i < 6; ++i) umma::mma_tf32(tmem + (i / 3) * 64, ad, bdsc, idesc, 1u);
        }
        if (variant >= 2) umma::commit(&bd[s]); else umma::mbar_arrive(&bd[s]);
      }
      umma::commit(&fin);
      umma::mbar_wait_spin(&fin, 0);
      t1 = clock64();
      if (blockIdx.x == 0) out[0] = (t1 - t0) / (REPS * NCH);
    }
    __syncwarp();
  } else if (warp < 2 + spinners) {
    // optional: other warps spin on try_wait of a barrier that completes at the end
    umma::mbar_wait(&fin, 0);
  }
  __syncthreads();
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<512>(tmem);
}
int main() {
  unsigned char* g; long long* out;
  cudaMalloc(&g, 64 << 20); cudaMemset(g, 0, 64 << 20);
  cudaMallocManaged(&out, 64 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int copies = 0; copies < 2; ++copies)
    for (int variant = 0; variant < 4; ++variant)
      for (int spinners : {0, 6}) {
        probe<<<132, 256, 200 * 1024>>>(g, out, variant, copies, spinners);
        cudaError_t e = cudaDeviceSynchronize();
        printf("copies %d variant %d (0 arrive, 1 +fence, 2 +commit, 3 +6 MMAs) spinners %d: %lld cycles/chunk  %s\n", copies, variant, spinners, out[0], cudaGetErrorString(e));
      }
  return 0;
}
