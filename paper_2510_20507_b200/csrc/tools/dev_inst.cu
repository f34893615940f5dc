// Development-only instantiation unit (make dev): the float N = d = 4 cluster
// kernels alone (BASELINE large), every other table entry empty.  Cuts the
// edit-compile loop to one translation unit; never shipped.
#include "../ammmse_tc2.cuh"
#include "../entries.h"

namespace ammmse {
namespace {
size_t cluster_smem_fn44(int M, int K, int C, int hres, int vglob, int sb, int tc) {
  CLayout<float, 4, 4> L;
  L.init(M, K, C, hres, vglob, sb, tc);
  return L.bytes;
}
size_t smem_fn44(int M, int K) {
  Layout<float, 4, 4> L;
  L.init(M, K);
  return L.bytes;
}
int tc2_stages44(int M, int K, int C, size_t limit) { return tc2::pick_stages<4, 4>(M, K, C, limit); }
size_t tc2_smem44(int M, int K, int C, int stages) {
  tc2::T2Layout<4, 4> L;
  L.init(M, K, C, stages);
  return L.bytes;
}
const KernelEntry kEmpty[4] = {};
#ifdef AMMMSE_DEV_FFMA
const SpecEntry kClusterSpecs44[1] = {
    {(const void*)ammmse_cluster_kernel<float, 4, 4, false, 128, 32, 4, 20480>, 128, 32, 4, 256, 20480},
};
#endif
const KernelEntry kEntries4[4] = {
    {}, {}, {},
    {nullptr, (const void*)ammmse_bounds_kernel<float, 4>, smem_fn44,
#ifdef AMMMSE_DEV_FFMA
     (const void*)ammmse_cluster_kernel<float, 4, 4>,
#else
     nullptr,
#endif
     cluster_smem_fn44, (const void*)ammmse_cluster_kernel<float, 4, 4, true>,
#ifdef AMMMSE_DEV_FFMA
     nullptr, 0, kClusterSpecs44, 1,
#else
     nullptr, 0, nullptr, 0,
#endif
     (const void*)ammmse_tc2_kernel<4, 4>, tc2_stages44, tc2_smem44},
};
}  // namespace
const KernelEntry* entries_float_1() { return kEmpty; }
const KernelEntry* entries_float_2() { return kEmpty; }
const KernelEntry* entries_float_3() { return kEmpty; }
const KernelEntry* entries_float_4() { return kEntries4; }
const KernelEntry* entries_double_1() { return kEmpty; }
const KernelEntry* entries_double_2() { return kEmpty; }
const KernelEntry* entries_double_3() { return kEmpty; }
const KernelEntry* entries_double_4() { return kEmpty; }
}  // namespace ammmse
