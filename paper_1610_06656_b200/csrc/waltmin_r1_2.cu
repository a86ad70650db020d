// Explicit instantiations of the WAltMin persistent kernel for r = 1..2
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<1>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<2>(WMParams& p, cudaStream_t st);
}  // namespace smp
