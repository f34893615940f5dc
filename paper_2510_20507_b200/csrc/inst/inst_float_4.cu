// Generated instantiation unit: engine kernels for R=float, N=4, d=1..4.
#include "../ammmse_tc2.cuh"
#include "../entries.h"

namespace ammmse {
namespace {
template <int DD>
size_t cluster_smem_fn(int M, int K, int C, int hres, int vglob, int sb, int tc) {
  CLayout<float, 4, DD> L;
  L.init(M, K, C, hres, vglob, sb, tc);
  return L.bytes;
}
template <int DD>
size_t smem_fn(int M, int K) {
  Layout<float, 4, DD> L;
  L.init(M, K);
  return L.bytes;
}
// second-generation tensor-core engine (ammmse_tc2.cuh): N = d = 4
int tc2_stages44(int M, int K, int C, size_t limit) { return tc2::pick_stages<4, 4>(M, K, C, limit); }
size_t tc2_smem44(int M, int K, int C, int stages) {
  tc2::T2Layout<4, 4> L;
  L.init(M, K, C, stages);
  return L.bytes;
}
// BASELINE large case on the cluster engine: M=128, K=32, N=d=4 (C=4)
const SpecEntry kClusterSpecs44[1] = {
    {(const void*)ammmse_cluster_kernel<float, 4, 4, false, 128, 32, 4, 20480>, 128, 32, 4, 256, 20480},
};
const KernelEntry kEntries[4] = {
    {(const void*)ammmse_solve_kernel<float, 4, 1>, (const void*)ammmse_bounds_kernel<float, 4>, smem_fn<1>,
     (const void*)ammmse_cluster_kernel<float, 4, 1>, cluster_smem_fn<1>, (const void*)ammmse_cluster_kernel<float, 4, 1, true>},
    {(const void*)ammmse_solve_kernel<float, 4, 2>, (const void*)ammmse_bounds_kernel<float, 4>, smem_fn<2>,
     (const void*)ammmse_cluster_kernel<float, 4, 2>, cluster_smem_fn<2>, (const void*)ammmse_cluster_kernel<float, 4, 2, true>},
    {(const void*)ammmse_solve_kernel<float, 4, 3>, (const void*)ammmse_bounds_kernel<float, 4>, smem_fn<3>,
     (const void*)ammmse_cluster_kernel<float, 4, 3>, cluster_smem_fn<3>, (const void*)ammmse_cluster_kernel<float, 4, 3, true>},
    {(const void*)ammmse_solve_kernel<float, 4, 4>, (const void*)ammmse_bounds_kernel<float, 4>, smem_fn<4>,
     (const void*)ammmse_cluster_kernel<float, 4, 4>, cluster_smem_fn<4>, (const void*)ammmse_cluster_kernel<float, 4, 4, true>,
     nullptr, 0, kClusterSpecs44, 1, (const void*)ammmse_tc2_kernel<4, 4>, tc2_stages44, tc2_smem44},
};
}  // namespace
const KernelEntry* entries_float_4() { return kEntries; }
}  // namespace ammmse
