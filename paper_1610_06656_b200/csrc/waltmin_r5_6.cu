// Explicit instantiations of the WAltMin persistent kernel for r = 5..6
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<5>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<6>(WMParams& p, cudaStream_t st);
}  // namespace smp
