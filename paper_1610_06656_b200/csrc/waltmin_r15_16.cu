// Explicit instantiations of the WAltMin persistent kernel for r = 15..16
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<15>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<16>(WMParams& p, cudaStream_t st);
}  // namespace smp
