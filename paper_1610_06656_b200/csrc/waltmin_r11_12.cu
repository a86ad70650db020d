// Explicit instantiations of the WAltMin persistent kernel for r = 11..12
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<11>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<12>(WMParams& p, cudaStream_t st);
}  // namespace smp
