// 7-stage A ring + MMA loop in isolation (uniform role warps, elect, fused asm) — cycles per chunk
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_20507_b200/csrc/tc_umma.cuh"
using namespace ammmse;
constexpr int S = 7, NCH = 16, REPS = 32;
__device__ __forceinline__ uint32_t test_u32(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(mbar), "r"(parity) : "memory");
  return ok;
}
__device__ __forceinline__ void try_u32(uint32_t mbar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" :: "r"(mbar), "r"(parity) : "memory");
}
// variant bits: 1 = early poll fused, 2 = MMAs on, 4 = copies on, 8 = commit only every 2nd chunk (producer waits pair)
__global__ void __launch_bounds__(256, 1) probe(const unsigned char* g, long long* out, int variant) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bf[8], bd[8], fin;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
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
  const uint32_t f0 = umma::smem_u32(bf), d0 = umma::smem_u32(bd), sm0 = umma::smem_u32(smem);
  const bool early = variant & 1, mmas = variant & 2, copies = variant & 4;
  if (warp == 1) {
    uint32_t pm = 0, ever = 0;
    for (int q = 0; q < REPS * NCH; ++q) {
      const uint32_t s = q % S, bit = 1u << s;
      if (ever & bit) { uint32_t ok; do { ok = test_u32(d0 + 8 * s, ((pm >> s) & 1) ^ 1); } while (!ok); }
      if (copies) {
        asm volatile("{\n\t.reg .pred Pe;\n\telect.sync _|Pe, 0xffffffff;\n\t"
                     "@Pe cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t"
                     "@Pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t}\n"
                     :: "r"(sm0 + s * 16384), "l"(src + (size_t)(q % NCH) * 16384), "r"(16384), "r"(f0 + 8 * s) : "memory");
      } else {
        asm volatile("{\n\t.reg .pred Pe;\n\telect.sync _|Pe, 0xffffffff;\n\t@Pe mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}\n" :: "r"(f0 + 8 * s) : "memory");
      }
      pm ^= bit; ever |= bit;
    }
  } else if (warp == 0) {
    long long t0 = clock64();
    uint32_t cm = 0;
    uint32_t ok = early ? test_u32(f0, 0) : 0;
    const uint64_t dproto = umma::make_sdesc(0, 128, 256);
    const uint64_t dhi = (uint64_t)(uint32_t)(dproto >> 32) << 32;
    const uint32_t dlo = (uint32_t)dproto;
    for (int q = 0; q < REPS * NCH; ++q) {
      const uint32_t s = q % S, nx = (s + 1) % S;
      const uint32_t par = (cm >> s) & 1;
      if (early) { while (!ok) ok = test_u32(f0 + 8 * s, par); }
      else try_u32(f0 + 8 * s, par);
      cm ^= 1u << s;
      const uint32_t al = dlo | (((sm0 + s * 16384) >> 4) & 0x3FFF);
      const uint32_t bl = dlo | (((sm0 + 7 * 16384 + (q % NCH) * 4128) >> 4) & 0x3FFF);
      const uint64_t a_rh = dhi | al, a_ih = dhi | (al + 256), a_rl = dhi | (al + 512), a_il = dhi | (al + 768);
      const uint64_t bhi = dhi | bl, blo = dhi | (bl + 128);
      const uint32_t d1 = tmem + (q & 1) * 128, d2 = d1 + 64;
      const uint32_t npar = (cm >> nx) & 1;
      asm volatile(
          "{\n\t.reg .pred Pn, Pe, Pa, Pt;\n\t"
          "setp.ne.b32 Pt, %12, 0;\n\t"
          "@Pt mbarrier.test_wait.parity.shared::cta.b64 Pn, [%10], %11;\n\t"
          "elect.sync _|Pe, 0xffffffff;\n\t"
          "setp.ne.b32 Pa, %13, 0;\n\t"
          "and.pred Pa, Pe, Pa;\n\t"
          "setp.eq.b32 Pt, 0, 0;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %7, %9, Pt;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %8, %9, Pt;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %7, %9, Pt;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%2], %4, %7, %9, Pt;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%2], %4, %8, %9, Pt;\n\t"
          "@Pa tcgen05.mma.cta_group::1.kind::tf32 [%2], %6, %7, %9, Pt;\n\t"
          "@Pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%14];\n\t"
          "selp.u32 %0, 1, 0, Pn;\n\t}\n"
          : "=r"(ok)
          : "r"(d1), "r"(d2), "l"(a_rh), "l"(a_ih), "l"(a_rl), "l"(a_il), "l"(bhi), "l"(blo), "r"(idesc),
            "r"(f0 + 8 * nx), "r"(npar), "r"(early ? 1 : 0), "r"(mmas ? 1 : 0), "r"(d0 + 8 * s)
          : "memory");
      if (!early) ok = 0;
    }
    asm volatile("{\n\t.reg .pred Pe;\n\telect.sync _|Pe, 0xffffffff;\n\t@Pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" :: "r"(umma::smem_u32(&fin)) : "memory");
    umma::mbar_wait_spin(&fin, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) out[0] = (t1 - t0) / (REPS * NCH);
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
  for (int variant = 0; variant < 8; ++variant) {
    probe<<<132, 256, 200 * 1024>>>(g, out, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("early-poll %d  MMAs %d  copies %d : %lld cycles/chunk  %s\n", variant & 1, (variant >> 1) & 1, (variant >> 2) & 1, out[0], cudaGetErrorString(e));
  }
  return 0;
}
