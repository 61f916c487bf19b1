// search_m5.cu -- search kernel instantiations for tau_l mode L2W_4 (search_kernel.cuh).
#include "search_kernel.cuh"

namespace vsag {
template cudaError_t launch_search_mode<L2W_4>(int, int, int, int, int, const KParams &, int, cudaStream_t,
                                                SearchLaunch *, int64_t);
}  // namespace vsag
