// probe.cu — FMA-pipe throughput probes for the roofline denominator.
#include <cuda_runtime.h>
#include "ammmse_probe.h"

namespace {
constexpr int kChains = 8;
constexpr int kInner = 256;

template <typename T>
__global__ void __launch_bounds__(256) fma_probe(T* out, int reps, T a, T b) {
  T acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = (T)(threadIdx.x + c);
  T x = a + (T)threadIdx.x * (T)1e-7, y = b * ((T)1 + (T)threadIdx.x * (T)1e-9);
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < kInner; ++i) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], x, y);  // register-operand FMA
    }
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == (T)-1.2345) out[0] = s;  // keep the chains alive
}

template <typename T>
double run(int reps) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* out = nullptr;
  if (cudaMalloc(&out, sizeof(T)) != cudaSuccess) return -1.0;
  const int blocks = sms * 8, threads = 256;
  fma_probe<T><<<blocks, threads>>>(out, 2, (T)0.999999, (T)1e-6);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_probe<T><<<blocks, threads>>>(out, reps, (T)0.999999, (T)1e-6);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
  const double fmas = (double)blocks * threads * reps * kInner * kChains;
  return 2.0 * fmas / (ms * 1e-3);
}
}  // namespace

extern "C" double ammmse_probe_fp32_flops(int reps) { return run<float>(reps > 0 ? reps : 400); }
extern "C" double ammmse_probe_fp64_flops(int reps) { return run<double>(reps > 0 ? reps : 100); }
