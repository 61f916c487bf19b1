// search_m0.cu -- search kernel instantiations for tau_l mode L2_8 (search_kernel.cuh).
#include "search_kernel.cuh"

namespace vsag {
template cudaError_t launch_search_mode<L2_8>(int, int, int, int, int, const KParams &, int, cudaStream_t,
                                                SearchLaunch *, int64_t);
#ifdef VSAG_STATS
extern "C" __attribute__((visibility("default"))) int vsag_debug_stats(unsigned long long *out, int reset) {
    cudaMemcpyFromSymbol(out, g_stats, sizeof(unsigned long long) * 64);
    if (reset) {
        unsigned long long z[64] = {};
        cudaMemcpyToSymbol(g_stats, z, sizeof(z));
    }
    return 0;
}
#endif

}  // namespace vsag
