// select.cu -- row a5, part 2: per-query selection of the initial candidate pool.
//
// Alg. 1 line 3 inserts every initial node with its tau_l into C, keeping
// |C| <= L: the result is the L smallest (tau_l, id) keys of the entry set, sorted.
// One warp per query.  Entry ids are sorted at index load, so the (tau_l, id) order is
// the (tau_l, index) order.
//
// S <= 1024 (seed_select_reg_kernel): the warp holds the S values in registers (PL per lane,
// index i = lane + 32 j), packs each into a 32-bit key (u - min) << ib | i (ib = index bits;
// values too far above the minimum to fit are clamped, which is exact whenever at least
// `need` values fit -- otherwise the same algorithm runs on 64-bit keys u << 32 | i), sorts
// every lane's PL keys in a register sorting network, and merges the 32 sorted lists: the
// t-th output is a warp-wide min (REDUX) of the lanes' list heads, and the lane holding it
// advances.  ~1.5k instructions per query instead of the histogram passes and the 256-key
// bitonic network below.
//
// Larger S (seed_select_kernel):
//   (1) one pass for min/max of the order-preserving u32 image u of tau_l;
//   (2) radix select on u - min over only its significant bits (8-bit digits, warp-
//       private 256-bin shared histograms; 3 passes for 23-bit ranges) -> the need-th
//       smallest value T and the number of ties at T to keep (first ones in index order);
//       as soon as all entries up to the end of the current digit's bin fit the n2-entry
//       sort buffer, the refinement stops and all of them are kept (usually after pass 1);
//   (3) compaction of the need = min(L, S) selected keys (u << 32 | id << 1, keys.cuh);
//   (4) a bitonic sort held in registers (need <= 256) or in shared memory (larger).
#include <algorithm>
#include <cstdlib>

#include "keys.cuh"
#include "select_net.cuh"
#include "vsag_internal.cuh"

namespace vsag {
namespace {

constexpr int SEL_WARPS = 4;  // 4-warp CTAs slot into the search grid's drain sooner (+0.4% pipelined, tools A/B)
constexpr int UB = 8;  // tau loads in flight per lane

// Ascending bitonic sort of 32*E keys held E per lane in blocked order (e = lane*E + r).
template <int E>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&v)[E], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int e = lane * E + r;
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], j / E);
                    const bool up = (e & k) == 0, low = (e & j) == 0;
                    const bool lt = v[r] < o;
                    v[r] = ((low == up) == lt) ? v[r] : o;
                }
            } else {
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int r2 = r ^ j;
                    if (r < r2) {
                        const int e = lane * E + r;
                        const bool up = (e & k) == 0;
                        const uint64_t a = v[r], b = v[r2];
                        if ((a > b) == up) {
                            v[r] = b;
                            v[r2] = a;
                        }
                    }
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ void sort_list_regs(uint64_t *list, int lane) {
    uint64_t v[E];
#pragma unroll
    for (int r = 0; r < E; r++) v[r] = list[lane * E + r];
    warp_sort_regs<E>(v, lane);
#pragma unroll
    for (int r = 0; r < E; r++) list[lane * E + r] = v[r];
}

__device__ __forceinline__ void sort_list_smem(uint64_t *list, int n2, int lane) {
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
}

// One query's selection by radix select + bitonic sort (any S; the fallback of the register
// kernel).  hist: 256 words, list: n2 >= need keys of warp-private shared memory.
__device__ __noinline__ void select_one_hist(const uint32_t *__restrict__ st, const int32_t *__restrict__ entry, int S,
                                             int need, int n2, uint32_t *hist, uint64_t *list, uint64_t *out, int lane) {
    {
        // (1) range of u = tau ^ 2^31 (order preserving); loads in batches of 8 per lane
        uint32_t mn = 0xffffffffu, mx = 0u;
        for (int i0 = 0; i0 < S; i0 += 32 * UB) {
            uint32_t u[UB];
#pragma unroll
            for (int j = 0; j < UB; j++) {
                const int i = i0 + 32 * j + lane;
                u[j] = i < S ? __ldg(st + i) ^ 0x80000000u : 0xffffffffu;
            }
#pragma unroll
            for (int j = 0; j < UB; j++) {
                if (i0 + 32 * j + lane < S) {
                    mn = min(mn, u[j]);
                    mx = max(mx, u[j]);
                }
            }
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        const uint32_t range = mx - mn;
        const int nbits = range ? 32 - __clz(range) : 1;
        // (2) radix select on v = u - mn, digits from the top significant bit
        uint32_t prefix = 0, pmask = 0;
        int k = need - 1;  // 0-based rank still to locate
        int taken_all = 0;  // entries below the current prefix (all selected)
        bool wide = false;
        uint32_t wide_bound = 0;
        for (int hi = nbits; hi > 0; hi -= 8) {
            const int shift = hi > 8 ? hi - 8 : 0;
            const uint32_t dmask = (1u << (hi - shift)) - 1u;
            for (int i = lane; i < 256; i += 32) hist[i] = 0;
            __syncwarp();
            for (int i0 = 0; i0 < S; i0 += 32 * UB) {
                uint32_t v[UB];
#pragma unroll
                for (int j = 0; j < UB; j++) {
                    const int i = i0 + 32 * j + lane;
                    v[j] = i < S ? (__ldg(st + i) ^ 0x80000000u) - mn : 0u;
                }
#pragma unroll
                for (int j = 0; j < UB; j++)
                    if (i0 + 32 * j + lane < S && (v[j] & pmask) == prefix) atomicAdd(hist + ((v[j] >> shift) & dmask), 1u);
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
                const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
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
            uint32_t cdig = 0;  // entries in the selected digit's bin
#pragma unroll
            for (int t = 0; t < 8; t++)
                if (mine && digit == (uint32_t)(lane * 8 + t)) cdig = c[t];
            digit = __shfl_sync(0xffffffffu, digit, owner);
            before = __shfl_sync(0xffffffffu, before, owner);
            cdig = __shfl_sync(0xffffffffu, cdig, owner);
            k -= (int)before;
            prefix |= digit << shift;
            pmask |= dmask << shift;
            __syncwarp();
            // every entry up to the end of this bin fits the sort buffer: keep them all and
            // let the sort order them (the first `need` after sorting are the selection)
            if (shift > 0 && taken_all + (int)before + (int)cdig <= n2) {
                wide_bound = prefix | ((1u << shift) - 1u);
                wide = true;
                break;
            }
            taken_all += (int)before;
        }
        const uint32_t T = prefix + mn;
        // (3) keep every u < T and the first k+1 entries with u == T (index order = id order)
        int taken = 0, eq_seen = 0;
        for (int i0 = 0; i0 < S; i0 += 32 * UB) {
            uint32_t ub[UB];
            int32_t eb[UB];
#pragma unroll
            for (int j = 0; j < UB; j++) {
                const int i = i0 + 32 * j + lane;
                ub[j] = i < S ? (__ldg(st + i) ^ 0x80000000u) : 0xffffffffu;
                eb[j] = i < S ? __ldg(entry + i) : 0;
            }
#pragma unroll
            for (int j = 0; j < UB; j++) {
                const int i = i0 + 32 * j + lane;
                const uint32_t u = ub[j];
                const bool eq = !wide && i < S && u == T;
                const uint32_t beq = __ballot_sync(0xffffffffu, eq);
                const bool take = wide ? (i < S && u - mn <= wide_bound)
                                       : ((i < S && u < T) || (eq && eq_seen + __popc(beq & lanemask_lt()) <= k));
                const uint32_t bt = __ballot_sync(0xffffffffu, take);
                if (take) list[taken + __popc(bt & lanemask_lt())] = make_key_u(u, eb[j]);
                taken += __popc(bt);
                eq_seen += __popc(beq);
            }
        }
        for (int t = taken + lane; t < n2; t += 32) list[t] = KEY_INF;
        __syncwarp();
        // (4) sort
        switch (n2) {
            case 32: sort_list_regs<1>(list, lane); break;
            case 64: sort_list_regs<2>(list, lane); break;
            case 128: sort_list_regs<4>(list, lane); break;
            case 256: sort_list_regs<8>(list, lane); break;
            default: sort_list_smem(list, n2, lane); break;
        }
        __syncwarp();
        for (int t = lane; t < need; t += 32) out[t] = list[t];
        __syncwarp();
    }
}

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
        select_one_hist(reinterpret_cast<const uint32_t *>(seed_tau + q * S), entry, S, need, n2, hist, list,
                        init_keys + q * L, lane);
        if (lane == 0) init_psz[q] = need;
    }
}

// per warp: the 32-bit lists [PL + 2][32] + a 32-word output buffer, or the fallback's
// histogram + sort list
__host__ __device__ constexpr int reg_select_warp_bytes(int pl, int n2) {
    return (pl + 3) * 32 * 4 > 1024 + n2 * 8 ? (pl + 3) * 32 * 4 : 1024 + n2 * 8;
}

// Ascending sorting network over N keys held in registers: Batcher's odd-even merge sort
// (select_net.cuh; 191 compare-exchanges for N = 32, against 240 for bitonic).
template <typename K, int N>
__device__ __forceinline__ void lane_sort(K (&v)[N]) {
    if constexpr (N == 8) oem_sort8(v);
    else if constexpr (N == 16) oem_sort16(v);
    else oem_sort32(v);
}


// Merge of the lanes' sorted lists (list j of lane l at lst[j * 32 + l]; v = the lane's sorted
// keys, still in registers): the `need` smallest keys in ascending order.  Output t is held by
// lane t % 32 until a group of 32 is complete, then `emit(t, key)` runs on every lane.
// Merge of the lanes' sorted lists: list j of lane l at lst[j * 32 + l], followed by two rows
// of sentinels (v = the lane's sorted keys, still in registers).  Emits the `need` smallest
// keys in ascending order: round t takes the warp-wide min (REDUX) of the lanes' heads and the
// lane holding it advances; lane 0 parks round t's key in obuf[t % 32] and after each 32 rounds
// every lane emits one of them (`emit(t, key)`).  Straight-line rounds (~8 instructions):
// every lane loads the element after its next one each round through a 32-bit shared-memory
// address that advances by 128 bytes on a pop (the sentinel rows keep it in bounds), so the
// dependency chain is REDUX -> compare -> select.  Full groups of 32 rounds run without any
// round test; only the last, partial group checks.  (An earlier form indexing
// lst[ptr * 32 + lane] after ptr++ read one element too far in the SASS nvcc 12.9 generated;
// tools/select_test.cu checks this kernel against a CPU reference.)
template <int PL, typename Emit>
__device__ __forceinline__ void warp_merge(const uint32_t (&v)[PL], const uint32_t *lst, uint32_t *obuf, int need,
                                           int lane, Emit emit) {
    uint32_t head = v[0], nxt = v[1];
    uint32_t addr = (uint32_t)__cvta_generic_to_shared(lst + 2 * 32 + lane);  // the element after nxt
    auto round = [&](int u) {
        const uint32_t m = __reduce_min_sync(0xffffffffu, head);
        if (lane == 0) obuf[u] = m;
        const bool pop = head == m;  // keys are distinct: exactly one lane pops
        uint32_t ld;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ld) : "r"(addr) : "memory");
        head = pop ? nxt : head;
        nxt = pop ? ld : nxt;
        addr += pop ? 128u : 0u;
    };
    int t0 = 0;
    for (; t0 + 32 <= need; t0 += 32) {
#pragma unroll
        for (int u = 0; u < 32; u++) round(u);
        __syncwarp();
        emit(t0 + lane, obuf[lane]);
        __syncwarp();
    }
    if (t0 < need) {
        const int rounds = need - t0;
        for (int u = 0; u < rounds; u++) round(u);
        __syncwarp();
        if (lane < rounds) emit(t0 + lane, obuf[lane]);
        __syncwarp();
    }
}

template <int PL, bool FULL>  // FULL: S == 32 * PL (no tail checks)
__global__ void __launch_bounds__(SEL_WARPS * 32) seed_select_reg_kernel(const int32_t *__restrict__ seed_tau,
                                                                         const int32_t *__restrict__ entry, int S,
                                                                         int ib, int64_t nq, int L, int n2,
                                                                         uint64_t *__restrict__ init_keys,
                                                                         int *__restrict__ init_psz) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    // per warp: the 32-bit lists [PL][32], or the fallback's histogram + sort list
    uint8_t *wbase = smem + (threadIdx.x >> 5) * reg_select_warp_bytes(PL, n2);
    const int need = min(L, S);
    const uint32_t LIM = 0xffffffffu >> ib;  // packed values v = u - min in [0, LIM) are exact
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += nwarps) {
        const uint32_t *st = reinterpret_cast<const uint32_t *>(seed_tau + q * S);
        uint32_t u[PL];
        uint32_t mn = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < PL; j++) {
            const int i = lane + 32 * j;
            u[j] = (FULL || i < S) ? __ldg(st + i) ^ 0x80000000u : 0xffffffffu;  // order-preserving image of tau
        }
#pragma unroll
        for (int j = 0; j < PL; j++)
            if (FULL || lane + 32 * j < S) mn = min(mn, u[j]);
        mn = __reduce_min_sync(0xffffffffu, mn);
        int fit = 0;
#pragma unroll
        for (int j = 0; j < PL; j++) fit += (FULL || lane + 32 * j < S) && (u[j] - mn < LIM);
        fit = (int)__reduce_add_sync(0xffffffffu, (uint32_t)fit);
        uint64_t *out = init_keys + q * L;
        if (fit >= need) {  // 32-bit keys (the common case)
            uint32_t k[PL];
#pragma unroll
            for (int j = 0; j < PL; j++) {
                const int i = lane + 32 * j;
                k[j] = (FULL || i < S) ? (min(u[j] - mn, LIM) << ib) | (uint32_t)i : 0xffffffffu;
            }
            lane_sort<uint32_t, PL>(k);
            uint32_t *lst = reinterpret_cast<uint32_t *>(wbase);
#pragma unroll
            for (int j = 0; j < PL; j++) lst[j * 32 + lane] = k[j];
            lst[PL * 32 + lane] = 0xffffffffu;
            lst[(PL + 1) * 32 + lane] = 0xffffffffu;
            __syncwarp();
            const uint32_t imask = (1u << ib) - 1u;
            warp_merge<PL>(k, lst, lst + (PL + 2) * 32, need, lane, [&](int t, uint32_t key) {
                out[t] = make_key_u(mn + (key >> ib), __ldg(entry + (key & imask)));
            });
        } else {  // the values spread too far for 32-bit keys: radix select + sort
            select_one_hist(st, entry, S, need, n2, reinterpret_cast<uint32_t *>(wbase),
                            reinterpret_cast<uint64_t *>(wbase + 1024), out, lane);
        }
        if (lane == 0) init_psz[q] = need;
        __syncwarp();  // the lists are rewritten by the next query
    }
}

}  // namespace

cudaError_t launch_seed_select(const int32_t *seed_tau, const int32_t *entry, int S, int64_t nq, int L,
                               uint64_t *init_keys, int *init_psz, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const bool force_hist = getenv("VSAG_SELECT_HIST") != nullptr;  // dev A/B switch
    if (S <= 1024 && !force_hist) {
        int ib = 1;
        while ((1 << ib) < S) ib++;
        const int pl = S <= 256 ? 8 : (S <= 512 ? 16 : 32);
        const bool full = S == 32 * pl;
        auto kern = pl == 8 ? (full ? seed_select_reg_kernel<8, true> : seed_select_reg_kernel<8, false>)
                    : pl == 16 ? (full ? seed_select_reg_kernel<16, true> : seed_select_reg_kernel<16, false>)
                               : (full ? seed_select_reg_kernel<32, true> : seed_select_reg_kernel<32, false>);
        int n2 = 32;
        while (n2 < (L < S ? L : S)) n2 <<= 1;
        const size_t sm = (size_t)SEL_WARPS * reg_select_warp_bytes(pl, n2);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SEL_WARPS * 32, sm);
        if (e != cudaSuccess) return e;
        // one query per warp (no persistent loop): in a pipelined step this kernel runs in the
        // drain of the previous batch's search, where short blocks fill freed SMs soonest
        int64_t blocks = (nq + SEL_WARPS - 1) / SEL_WARPS;
#ifdef VSAG_SEL_PERSIST
        if (blocks > (int64_t)sms * std::max(per_sm, 1)) blocks = (int64_t)sms * std::max(per_sm, 1);
#endif
        if (blocks > (1 << 30)) blocks = 1 << 30;
        kern<<<(unsigned)blocks, SEL_WARPS * 32, sm, s>>>(seed_tau, entry, S, ib, nq, L, n2, init_keys, init_psz);
        return cudaGetLastError();
    }
    int n2 = 32;
    while (n2 < (L < S ? L : S)) n2 <<= 1;
    const size_t sm = (size_t)SEL_WARPS * (1024 + n2 * 8);
    cudaError_t e = cudaFuncSetAttribute(seed_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int64_t blocks = (nq + SEL_WARPS - 1) / SEL_WARPS;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    seed_select_kernel<<<(unsigned)blocks, SEL_WARPS * 32, sm, s>>>(seed_tau, entry, S, nq, L, init_keys, init_psz, n2);
    return cudaGetLastError();
}

}  // namespace vsag
