// Generated instantiation unit: engine kernels for R=float, N=2, d=1..4.
#include "../ammmse_cluster.cuh"
#include "../entries.h"

namespace ammmse {
namespace {
template <int DD>
size_t cluster_smem_fn(int M, int K, int C, int hres, int vglob, int sb, int tc) {
  CLayout<float, 2, DD> L;
  L.init(M, K, C, hres, vglob, sb, tc);
  return L.bytes;
}
template <int DD>
size_t smem_fn(int M, int K) {
  Layout<float, 2, DD> L;
  L.init(M, K);
  return L.bytes;
}
// BASELINE shapes on the cluster engine: massive / sweep M=256 (C=4), sweep M=128 (C=1),
// sweep M=512 (C=16)
// (placement fixed to the planner's choice for these shapes: H streamed, V_old in L2)
const SpecEntry kClusterSpecs22[3] = {
    {(const void*)ammmse_cluster_kernel<float, 2, 2, false, 256, 64, 4, 20480>, 256, 64, 4, 256, 20480},
    {(const void*)ammmse_cluster_kernel<float, 2, 2, false, 128, 32, 1, 20480>, 128, 32, 1, 256, 20480},
    {(const void*)ammmse_cluster_kernel<float, 2, 2, false, 512, 128, 16, 12288>, 512, 128, 16, 256, 12288},
};
// single-CTA engine: medium / sweep M=64 (256 threads; registers sized for 2 CTAs/SM,
// 128 regs without spills, measured +2 % over 3 CTAs/SM at 80 regs), sweep M=32
// (128 threads)
const SpecEntry kSolveSpecs22[2] = {
    {(const void*)ammmse_solve_kernel<float, 2, 2, 64, 16, 256, 2>, 64, 16, 0, 256},
    {(const void*)ammmse_solve_kernel<float, 2, 2, 32, 8, 128>, 32, 8, 0, 128},
};
const KernelEntry kEntries[4] = {
    {(const void*)ammmse_solve_kernel<float, 2, 1>, (const void*)ammmse_bounds_kernel<float, 2>, smem_fn<1>,
     (const void*)ammmse_cluster_kernel<float, 2, 1>, cluster_smem_fn<1>, (const void*)ammmse_cluster_kernel<float, 2, 1, true>},
    // d = 2 carries the M = 64, K = 16 specialisation (BASELINE medium / sweep M = 64)
    {(const void*)ammmse_solve_kernel<float, 2, 2>, (const void*)ammmse_bounds_kernel<float, 2>, smem_fn<2>,
     (const void*)ammmse_cluster_kernel<float, 2, 2>, cluster_smem_fn<2>, (const void*)ammmse_cluster_kernel<float, 2, 2, true>,
     kSolveSpecs22, 2, kClusterSpecs22, 3},
    {(const void*)ammmse_solve_kernel<float, 2, 3>, (const void*)ammmse_bounds_kernel<float, 2>, smem_fn<3>,
     (const void*)ammmse_cluster_kernel<float, 2, 3>, cluster_smem_fn<3>, (const void*)ammmse_cluster_kernel<float, 2, 3, true>},
    {(const void*)ammmse_solve_kernel<float, 2, 4>, (const void*)ammmse_bounds_kernel<float, 2>, smem_fn<4>,
     (const void*)ammmse_cluster_kernel<float, 2, 4>, cluster_smem_fn<4>, (const void*)ammmse_cluster_kernel<float, 2, 4, true>},
};
}  // namespace
const KernelEntry* entries_float_2() { return kEntries; }
}  // namespace ammmse
