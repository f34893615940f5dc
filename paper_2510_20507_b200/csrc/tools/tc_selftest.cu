// tc_selftest.cu — validation kernel for the hand-written tcgen05 toolkit
// (tc_umma.cuh): D = A · B with 3xTF32 (hi·hi + hi·lo + lo·hi), operands in
// canonical no-swizzle layouts (K-major or MN-major), accumulator in TMEM.
// Built into libammmse_tctest.so and driven by tests/test_gpu_tc.py; not
// on the solve path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../tc_umma.cuh"

using namespace ammmse;

namespace {

__global__ void __launch_bounds__(128) tc_selftest_kernel(const float* A, const float* B, float* D,
                                                         int P, int Q, int K, int a_mn, int b_mn,
                                                         int neg_b, int mn_swap) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  float* Ahi = reinterpret_cast<float*>(smem);
  float* Alo = Ahi + P * K;
  float* Bhi = Alo + P * K;
  float* Blo = Bhi + K * Q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // operands -> canonical layouts (byte offsets / 4)
  for (int i = tid; i < P * K; i += blockDim.x) {
    const int p = i / K, k = i - p * K;
    float hi, lo;
    umma::split_tf32(A[i], hi, lo);
    const uint32_t off = a_mn ? umma::cm_offset(k, p, P) : umma::cm_offset(p, k, K);
    Ahi[off >> 2] = hi;
    Alo[off >> 2] = lo;
  }
  for (int i = tid; i < K * Q; i += blockDim.x) {
    const int k = i / Q, q = i - k * Q;
    float hi, lo;
    umma::split_tf32(B[i], hi, lo);
    const uint32_t off = b_mn ? umma::cm_offset(k, q, Q) : umma::cm_offset(q, k, K);
    Bhi[off >> 2] = hi;
    Blo[off >> 2] = lo;
  }
  if (tid == 0) umma::mbar_init(&mbar, 1);
  if (warp == 0) umma::tmem_alloc<64>(&tslot);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tbase = tslot;

  if (tid == 0) {
    const uint32_t idesc = umma::make_idesc_tf32(P, Q, a_mn, b_mn, false, neg_b != 0);
    uint32_t a_lbo = a_mn ? (uint32_t)(P / 4) * 128 : 128u;
    uint32_t a_sbo = a_mn ? 128u : (uint32_t)(K / 4) * 128;
    uint32_t b_lbo = b_mn ? (uint32_t)(Q / 4) * 128 : 128u;
    uint32_t b_sbo = b_mn ? 128u : (uint32_t)(K / 4) * 128;
    if (mn_swap) {  // probe: swapped LBO / SBO roles for MN-major operands
      if (a_mn) { const uint32_t t = a_lbo; a_lbo = a_sbo; a_sbo = t; }
      if (b_mn) { const uint32_t t = b_lbo; b_lbo = b_sbo; b_sbo = t; }
    }
    const float* aops[3] = {Ahi, Ahi, Alo};
    const float* bops[3] = {Bhi, Blo, Bhi};
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t a_step = a_mn ? s * (P / 4) * 128 : s * 256;
      const uint32_t b_step = b_mn ? s * (Q / 4) * 128 : s * 256;
      for (int term = 0; term < 3; ++term) {
        const uint64_t ad = umma::make_sdesc(umma::smem_u32(aops[term]) + a_step, a_lbo, a_sbo);
        const uint64_t bd = umma::make_sdesc(umma::smem_u32(bops[term]) + b_step, b_lbo, b_sbo);
        umma::mma_tf32(tbase, ad, bd, idesc, (s > 0 || term > 0) ? 1u : 0u);
      }
    }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after();
  // readback: warp w holds TMEM lanes 32w..32w+31
  for (int c0 = 0; c0 < Q; c0 += 16) {
    float v[16];
    umma::tmem_ld16(tbase + ((uint32_t)(32 * warp) << 16) + c0, v);
    int row;
    if (P == 128) row = 32 * warp + lane;
    else row = lane < 16 ? 16 * warp + lane : -1;  // M = 64: lanes 0-15 of each quadrant
    if (row >= 0 && row < P)
      for (int j = 0; j < 16 && c0 + j < Q; ++j) D[row * Q + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<64>(tbase);
}

}  // namespace

extern "C" int ammmse_tc_selftest(const float* A, const float* B, float* D, int P, int Q, int K,
                                  int a_mn, int b_mn, int neg_b, int mn_swap) {
  if (!(P == 64 || P == 128) || Q < 16 || Q > 64 || Q % 16 || K % 8) return -1;
  const size_t smem = (size_t)2 * (P * K + K * Q) * sizeof(float);
  if (cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return -2;
  tc_selftest_kernel<<<1, 128, smem>>>(A, B, D, P, Q, K, a_mn, b_mn, neg_b, mn_swap);
  if (cudaGetLastError() != cudaSuccess) return -3;
  if (cudaDeviceSynchronize() != cudaSuccess) return -4;
  return 0;
}
