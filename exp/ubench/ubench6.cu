// fp64 latency / throughput probes (one warp, one CTA)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double x0) {
  double a = x0, b = x0 * 1.0000001, c0 = x0, c1 = x0 + 1, c2 = x0 + 2, c3 = x0 + 3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a = fma(a, b, 1e-9);  // dependent chain
  }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // 4 independent chains
      c0 = fma(c0, b, 1e-9); c1 = fma(c1, b, 1e-9); c2 = fma(c2, b, 1e-9); c3 = fma(c3, b, 1e-9);
    }
  }
  long long t2 = clock64();
  double r = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) r = rsqrt(r + 1.5);
  long long t3 = clock64();
  double d = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) d = 1.0 / (d + 1.5);
  long long t4 = clock64();
  double s = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) s = sqrt(s + 1.5);
  long long t5 = clock64();
  double l = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) l = log(l + 1.5);
  long long t6 = clock64();
  float f = (float)x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) f = fmaf(f, 1.0000001f, 1e-9f);
  }
  long long t7 = clock64();
  double sh = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) sh += __shfl_xor_sync(0xffffffffu, sh, 1);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 2048; cyc[1] = (t2 - t1) / 2048; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
    cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256; cyc[6] = (t7 - t6) / 2048; cyc[7] = (t8 - t7) / 256;
  }
  out[threadIdx.x] = a + c0 + c1 + c2 + c3 + r + d + s + l + f + sh;
}
int main() {
  double* out; long long* cyc;
  cudaMallocManaged(&out, 1024 * 8); cudaMallocManaged(&cyc, 64 * 8);
  for (int nt : {32, 256}) {
    probe<<<1, nt>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    printf("threads %d: DFMA dependent %lld cyc, DFMA 4-chain %lld cyc/op, rsqrt %lld, 1/x %lld, sqrt %lld, log %lld, FFMA dependent %lld, shfl+dadd(64-bit) %lld\n",
           nt, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
  }
  return 0;
}
