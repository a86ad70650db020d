// Explicit instantiations of the WAltMin persistent kernel for r = 7..8
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<7>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<8>(WMParams& p, cudaStream_t st);
}  // namespace smp
