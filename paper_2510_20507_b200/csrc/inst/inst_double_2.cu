// Generated instantiation unit: engine kernels for R=double, N=2, d=1..4.
#include "../ammmse_cluster.cuh"
#include "../entries.h"

namespace ammmse {
namespace {
template <int DD>
size_t cluster_smem_fn(int M, int K, int C, int hres, int vglob, int sb, int tc) {
  CLayout<double, 2, DD> L;
  L.init(M, K, C, hres, vglob, sb, tc);
  return L.bytes;
}
template <int DD>
size_t smem_fn(int M, int K) {
  Layout<double, 2, DD> L;
  L.init(M, K);
  return L.bytes;
}
// single-CTA engine: BASELINE small case (M=16, K=4, complex128, 64 threads)
const SpecEntry kSolveSpecs22[1] = {
    {(const void*)ammmse_solve_kernel<double, 2, 2, 16, 4, 64>, 16, 4, 0, 64},
};
const KernelEntry kEntries[4] = {
    {(const void*)ammmse_solve_kernel<double, 2, 1>, (const void*)ammmse_bounds_kernel<double, 2>, smem_fn<1>,
     (const void*)ammmse_cluster_kernel<double, 2, 1>, cluster_smem_fn<1>, nullptr},
    {(const void*)ammmse_solve_kernel<double, 2, 2>, (const void*)ammmse_bounds_kernel<double, 2>, smem_fn<2>,
     (const void*)ammmse_cluster_kernel<double, 2, 2>, cluster_smem_fn<2>, nullptr, kSolveSpecs22, 1},
    {(const void*)ammmse_solve_kernel<double, 2, 3>, (const void*)ammmse_bounds_kernel<double, 2>, smem_fn<3>,
     (const void*)ammmse_cluster_kernel<double, 2, 3>, cluster_smem_fn<3>, nullptr},
    {(const void*)ammmse_solve_kernel<double, 2, 4>, (const void*)ammmse_bounds_kernel<double, 2>, smem_fn<4>,
     (const void*)ammmse_cluster_kernel<double, 2, 4>, cluster_smem_fn<4>, nullptr},
};
}  // namespace
const KernelEntry* entries_double_2() { return kEntries; }
}  // namespace ammmse
