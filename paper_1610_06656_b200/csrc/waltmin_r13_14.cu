// Explicit instantiations of the WAltMin persistent kernel for r = 13..14
// (split for parallel compilation).
#include "waltmin_impl.cuh"

namespace smp {
template cudaError_t launch_wm<13>(WMParams& p, cudaStream_t st);
template cudaError_t launch_wm<14>(WMParams& p, cudaStream_t st);
}  // namespace smp
