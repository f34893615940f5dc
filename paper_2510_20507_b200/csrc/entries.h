// entries.h — table of compiled engine instantiations (one .cu per (R, N)).
#pragma once
#include <stddef.h>

namespace ammmse {

struct SpecEntry {  // shape-specialised kernel for fixed (M, K, cluster size C, block size T)
  const void* f;
  int M, K, C, T;
  int sb = 0;  // cluster: > 0 = compiled for the streamed-H / global-V_old plan with sb-byte stages
};

struct KernelEntry {
  const void* solve;                           // ammmse_solve_kernel<R, N, d>   (1 CTA / realization)
  const void* bounds;                          // ammmse_bounds_kernel<R, N>
  size_t (*smem_bytes)(int M, int K);          // Layout<R, N, d>::bytes
  const void* cluster_solve;                   // ammmse_cluster_kernel<R, N, d> (1 cluster / realization)
  size_t (*cluster_smem_bytes)(int M, int K, int C, int hres, int vglob, int sb, int tc);  // CLayout::bytes
  const void* cluster_solve_tc;                // ammmse_cluster_kernel<float, N, d, true> (nullptr for fp64)
  const SpecEntry* solve_specs = nullptr;      // ammmse_solve_kernel<R, N, d, M, K, T> (C = 0)
  int n_solve_specs = 0;
  const SpecEntry* cluster_specs = nullptr;    // FFMA cluster kernels for fixed (M, K, C), T = 256
  int n_cluster_specs = 0;
  // second-generation tensor-core cluster engine (ammmse_tc2.cuh; float only)
  const void* cluster_solve_tc2 = nullptr;     // ammmse_tc2_kernel<N, d>
  int (*tc2_stages)(int M, int K, int C, size_t limit) = nullptr;   // A ring depth that fits (0: none)
  size_t (*tc2_smem_bytes)(int M, int K, int C, int stages) = nullptr;
};

// entries_<real>_<N>()[d - 1], d = 1..4
const KernelEntry* entries_float_1();
const KernelEntry* entries_float_2();
const KernelEntry* entries_float_3();
const KernelEntry* entries_float_4();
const KernelEntry* entries_double_1();
const KernelEntry* entries_double_2();
const KernelEntry* entries_double_3();
const KernelEntry* entries_double_4();

}  // namespace ammmse
