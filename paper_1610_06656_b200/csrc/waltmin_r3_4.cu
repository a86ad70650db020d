// Explicit instantiations of the WAltMin persistent kernel for r = 3..4
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<3>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<4>(WMParams& p, cudaStream_t st);
}  // namespace smp
