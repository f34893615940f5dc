// ammmse_gen.cu — on-device synthetic inputs.
//
// Counterpart of the reference's host generators for one realization
// (generate_channels model.py:197-207: H_k i.i.d. CN(0,1); init_precoders
// model.py:225-235 + project_sum_power solvers.py:257-263: V0 i.i.d. CN(0,1)
// scaled onto the power ball), for whole batches, so throughput runs at
// BASELINE's full batch sizes need no host generation or H2D copy.
//
// Random stream: Philox4x32-10 (Salmon et al., SC'11: 10 rounds of the
// 2 x 32-bit multiply-xorshift bijection with Weyl key schedule), keyed by
// (seed0 + realization, stream tag), counter = element index; Box-Muller turns
// each 4-word block into two standard normals per complex element pair.
// This is NOT numpy's stream (numpy draws normals with a ziggurat), so inputs
// are distributionally, not bit-, identical to the reference generators; the
// host generators (model.py / inputs.py) stay the bit-exact path.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "ammmse.h"

namespace {

struct P4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ P4 philox4x32_10(P4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = P4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// (0, 1] uniform from 32 bits
__device__ __forceinline__ double u01(uint32_t v) { return ((double)v + 1.0) * 2.3283064365386963e-10; }

// Two CN(0,1) draws (variance 1/2 per real component) from counter (idx, tag)
__device__ __forceinline__ void cn01_pair(uint64_t key, uint32_t tag, uint64_t idx, double (&re)[2],
                                          double (&im)[2]) {
  const P4 v = philox4x32_10(P4{(uint32_t)idx, (uint32_t)(idx >> 32), tag, 0u}, (uint32_t)key,
                             (uint32_t)(key >> 32));
  // Box-Muller: sqrt(-2 ln u1) * (cos, sin)(2 pi u2) has unit variance per component
  const double r0 = sqrt(-log(u01(v.x))), r1 = sqrt(-log(u01(v.z)));
  double s0, c0, s1, c1;
  sincospi(2.0 * u01(v.y), &s0, &c0);
  sincospi(2.0 * u01(v.w), &s1, &c1);
  re[0] = r0 * c0;  // r = sqrt(-ln u) gives variance 1/2 per component
  im[0] = r0 * s0;
  re[1] = r1 * c1;
  im[1] = r1 * s1;
}

constexpr uint32_t kTagH = 0xC4A77E1u, kTagV = 0x1417C0DEu, kTagA = 0xA1FAu;

template <typename R>
__global__ void __launch_bounds__(256) gen_iid_kernel(long long B, int K, int N, int M, int d,
                                                      unsigned long long seed0, double p_max,
                                                      int uniform_weights, R* H, R* V0,
                                                      double* alpha) {
  __shared__ double red[8];
  const long long r = blockIdx.x;
  if (r >= B) return;
  const uint64_t key = (uint64_t)(seed0 + (unsigned long long)r);
  const long long nh = (long long)K * N * M, nv = (long long)K * M * d;
  R* h = H + 2 * r * nh;
  for (long long e = 2 * (long long)threadIdx.x; e < nh; e += 2 * blockDim.x) {
    double re[2], im[2];
    cn01_pair(key, kTagH, (uint64_t)e, re, im);
    h[2 * e] = (R)re[0];
    h[2 * e + 1] = (R)im[0];
    if (e + 1 < nh) {
      h[2 * e + 2] = (R)re[1];
      h[2 * e + 3] = (R)im[1];
    }
  }
  // V0 ~ CN(0,1), then the sum-power projection (scale iff ||V0||^2 > P)
  R* v = V0 + 2 * r * nv;
  double pw = 0.0;
  for (long long e = 2 * (long long)threadIdx.x; e < nv; e += 2 * blockDim.x) {
    double re[2], im[2];
    cn01_pair(key, kTagV, (uint64_t)e, re, im);
    const R a0 = (R)re[0], b0 = (R)im[0];
    v[2 * e] = a0;
    v[2 * e + 1] = b0;
    pw += (double)a0 * a0 + (double)b0 * b0;
    if (e + 1 < nv) {
      const R a1 = (R)re[1], b1 = (R)im[1];
      v[2 * e + 2] = a1;
      v[2 * e + 3] = b1;
      pw += (double)a1 * a1 + (double)b1 * b1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  if (tot > p_max) {
    const double sc = sqrt(p_max / tot);
    for (long long e = threadIdx.x; e < 2 * nv; e += blockDim.x) v[e] = (R)((double)v[e] * sc);
  }
  if (alpha) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      double a = 1.0;
      if (uniform_weights) {
        const P4 u = philox4x32_10(P4{(uint32_t)k, 0u, kTagA, 0u}, (uint32_t)key,
                                   (uint32_t)(key >> 32));
        a = 0.5 + (u01(u.x) - 2.3283064365386963e-10);  // Uniform[0.5, 1.5)
      }
      alpha[r * K + k] = a;
    }
  }
}

}  // namespace

extern "C" int ammmse_generate_iid(const AmmmseDims* dims, unsigned long long seed0, double p_max,
                                   int uniform_weights, void* channels, void* init_precoders,
                                   double* weights, void* stream) {
  if (!dims || dims->batch < 1 || dims->M < 1 || dims->N < 1 || dims->K < 1 || dims->d < 1)
    return AMMMSE_ERR_INVALID;
  if (!channels || !init_precoders || !(p_max > 0) || !isfinite(p_max)) return AMMMSE_ERR_INVALID;
  const long long B = dims->batch;
  if (B > 0x7fffffffLL) return AMMMSE_ERR_UNSUPPORTED;
  cudaError_t ce;
  if (dims->dtype == AMMMSE_COMPLEX64) {
    gen_iid_kernel<float><<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>(
        B, dims->K, dims->N, dims->M, dims->d, seed0, p_max, uniform_weights,
        (float*)channels, (float*)init_precoders, weights);
  } else if (dims->dtype == AMMMSE_COMPLEX128) {
    gen_iid_kernel<double><<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>(
        B, dims->K, dims->N, dims->M, dims->d, seed0, p_max, uniform_weights,
        (double*)channels, (double*)init_precoders, weights);
  } else {
    return AMMMSE_ERR_INVALID;
  }
  ce = cudaGetLastError();
  return ce == cudaSuccess ? AMMMSE_OK : AMMMSE_ERR_CUDA;
}
