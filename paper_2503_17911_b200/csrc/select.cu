// select.cu -- row a5, part 2: per-query selection of the initial candidate pool.
//
// Alg. 1 line 3 inserts every initial node with its tau_l into C, keeping
// |C| <= L: the result is the L smallest (tau_l, id) keys of the entry set, sorted.
#include "keys.cuh"
#include "vsag_internal.cuh"

namespace vsag {
namespace {

// a5, part 2: per query, the top-L entry nodes by (tau_l, id) as a sorted key list.
// One warp per query.  Entry ids are sorted, so (tau_l, id) order is (tau_l, index)
// order.  (1) Radix-select (4 passes of 8 bits over the order-preserving u32 image of
// tau_l, warp-private 256-bin shared histograms) finds T = the need-th smallest tau_l
// and how many ties at T to keep; (2) the need = min(L, S) selected keys are compacted
// (ties at T taken in index order) and (3) bitonic-sorted in shared memory.
constexpr int SEL_WARPS = 8;

__global__ void __launch_bounds__(SEL_WARPS * 32) seed_select_kernel(const int32_t *__restrict__ seed_tau,
                                                                     const int32_t *__restrict__ entry, int S,
                                                                     int64_t nq, int L, uint64_t *init_keys,
                                                                     int *init_psz, int n2) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    uint8_t *wbase = smem + (threadIdx.x >> 5) * (1024 + n2 * 8);
    uint32_t *hist = reinterpret_cast<uint32_t *>(wbase);
    uint64_t *list = reinterpret_cast<uint64_t *>(wbase + 1024);
    const int need = min(L, S);
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += nwarps) {
        const uint32_t *st = reinterpret_cast<const uint32_t *>(seed_tau + q * S);
        uint32_t prefix = 0, pmask = 0;
        int k = need - 1;  // 0-based rank still to locate
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int i = lane; i < 256; i += 32) hist[i] = 0;
            __syncwarp();
            for (int i = lane; i < S; i += 32) {
                const uint32_t u = st[i] ^ 0x80000000u;
                if ((u & pmask) == prefix) atomicAdd(hist + ((u >> shift) & 255u), 1u);
            }
            __syncwarp();
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int t = 0; t < 8; t++) {
                c[t] = hist[lane * 8 + t];
                tot += c[t];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t excl = incl - tot;
            const bool mine = excl <= (uint32_t)k && (uint32_t)k < incl;
            const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
            uint32_t digit = 0, before = 0;
            if (mine) {
                uint32_t run = excl;
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    if (run + c[t] > (uint32_t)k) {
                        digit = lane * 8 + t;
                        before = run;
                        break;
                    }
                    run += c[t];
                }
            }
            digit = __shfl_sync(0xffffffffu, digit, owner);
            before = __shfl_sync(0xffffffffu, before, owner);
            k -= (int)before;
            prefix |= digit << shift;
            pmask |= 255u << shift;
            __syncwarp();
        }
        // keep every u < T and the first k+1 entries with u == T (index order = id order)
        int taken = 0, eq_seen = 0;
        for (int i0 = 0; i0 < S; i0 += 32) {
            const int i = i0 + lane;
            const uint32_t u = i < S ? (st[i] ^ 0x80000000u) : 0xffffffffu;
            const bool eq = i < S && u == prefix;
            const uint32_t beq = __ballot_sync(0xffffffffu, eq);
            const bool take = (i < S && u < prefix) || (eq && eq_seen + __popc(beq & lanemask_lt()) <= k);
            const uint32_t bt = __ballot_sync(0xffffffffu, take);
            if (take) list[taken + __popc(bt & lanemask_lt())] = ((uint64_t)u << 32) | (uint32_t)entry[i];
            taken += __popc(bt);
            eq_seen += __popc(beq);
        }
        for (int t = need + lane; t < n2; t += 32) list[t] = KEY_INF;
        __syncwarp();
        for (int kk = 2; kk <= n2; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < n2; i += 32) {
                    const int l = i ^ j;
                    if (l > i) {
                        const uint64_t x = list[i], y = list[l];
                        if ((x > y) == ((i & kk) == 0)) {
                            list[i] = y;
                            list[l] = x;
                        }
                    }
                }
                __syncwarp();
            }
        }
        for (int t = lane; t < need; t += 32) init_keys[q * L + t] = list[t];
        if (lane == 0) init_psz[q] = need;
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_seed_select(const int32_t *seed_tau, const int32_t *entry, int S, int64_t nq, int L,
                               uint64_t *init_keys, int *init_psz, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    int n2 = 32;
    while (n2 < (L < S ? L : S)) n2 <<= 1;
    const size_t sm = (size_t)SEL_WARPS * (1024 + n2 * 8);
    cudaError_t e = cudaFuncSetAttribute(seed_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (nq + SEL_WARPS - 1) / SEL_WARPS;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    seed_select_kernel<<<(unsigned)blocks, SEL_WARPS * 32, sm, s>>>(seed_tau, entry, S, nq, L, init_keys, init_psz, n2);
    return cudaGetLastError();
}

}  // namespace vsag
