// Explicit instantiations of the WAltMin persistent kernel for r = 9..10
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<9>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<10>(WMParams& p, cudaStream_t st);
}  // namespace smp
