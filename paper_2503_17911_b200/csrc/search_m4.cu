// search_m4.cu -- search kernel instantiations for tau_l mode L2W_8 (search_kernel.cuh).
#include "search_kernel.cuh"

namespace vsag {
template cudaError_t launch_search_mode<L2W_8>(int, int, int, int, int, const KParams &, int, cudaStream_t,
                                                SearchLaunch *, int64_t);
}  // namespace vsag
