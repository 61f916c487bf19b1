// search_common.cuh -- device-side pieces of the search kernel (search.cu): launch
// parameters, the visited-set variants, the pool lower bound and the per-query finish
// (trace, a7 re-rank, a8 output).
#pragma once
#include <cuda_fp16.h>

#include "dist.cuh"
#include "keys.cuh"

namespace vsag {

struct KParams {
    const uint32_t *op;
    int op_stride;  // words per query
    const int32_t *seed_tau;
    const int32_t *entry;
    int S;
    const uint64_t *init_keys;  // [nq, L] initial pool (sorted), from seed_select_kernel
    const int *init_psz;        // [nq]
    const int32_t *adj;
    const uint8_t *codes;
    const uint8_t *rows;
    int64_t row_bytes;
    int ids_bytes;
    const float *base;
    const float *queries;
    int d;
    int64_t nq;
    int k, ef, R, L, degree, cbp, chunks, g_log2, layout, metric;
    int h_log2;
    int vkind;           // visited set: 2 u16 buckets / 3 u32 probing (shared memory), 4 device-memory bitset
    int64_t gvis_words;  // kind 4: bitset words per warp (multiple of 4)
    uint32_t *gvis;      // kind 4: [resident warps, gvis_words] (set by the launcher)
    int tab16, nb_log2, id_bits, tab_bytes, row_dups, lcap;
    int wide;            // every code row starts on a 32-byte boundary (the gather uses 32-byte loads)
    int64_t n_base;      // rows of the index (checked build)
    int rk_bytes;        // bytes of the warp's re-rank scratch region (checked build)
    int smem_per_warp, off_pool, off_tab, off_newk, off_newid, off_newslot, off_row;
    const int32_t *l2w;  // weighted L2 (NEXT-1b): per-dimension weights, copied to the CTA's shared memory
    int off_cta;         // bytes of the CTA-shared region in front of the warps' regions
    int l2w_dims;        // weights in l2w (padded dimensions)
    const float *labels; // edge labels [n, degree] (NEXT-2) or NULL
    int m_s;             // edge filter: degree cap (0: none)
    float alpha_s;       // edge filter: label bound (0: none)
    int filt;            // edge filter active
    const int32_t *prs_blk;    // PRS delta in (0, 1] on a table index (NEXT-4): block of each node or -1
    const uint8_t *prs_codes;  // [blocks, degree * cbp]
    int adaptive;              // NEXT-3 early stop of the re-rank
    int qlp_ef_low, qlp_hop, qlp_feature;  // NEXT-4b QLP checkpoint (qlp_ef_low == 0: off)
    long long qlp_threshold;
    double delta_min;          // its smallest quantisation step
    int32_t *out_ids;
    float *out_dists;
    int32_t *t_hops, *t_expanded, *t_nlp, *t_nhp, *t_miss, *t_pool_ids, *t_pool_tau;
    int max_hops;
    unsigned int *counter;
    int *check;          // VSAG_CHECKS builds: the index's mapped error flag (bounds-check failures)
};

namespace {

#ifdef VSAG_STATS
static __device__ unsigned long long g_stats[64];
#define STAT(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_stats[i], (unsigned long long)(v)); } while (0)
#else
#define STAT(i, v) do { } while (0)
#endif

// Bounds checks of the checked build (VSAG_CHECKS; compute-sanitizer is not available on the
// GPU pool): a failed check stores its bit in the index's mapped error flag, which the API
// reports as VSAG_ERR_CUDA from the calls that synchronise.  Bits: 2 shared-memory index,
// 4 global row index, 8 visited-table index, 16 merge index, 32 output index.
#ifdef VSAG_CHECKS
#define VCHK(chk, cond, bit)                                                   \
    do {                                                                      \
        if (!(cond)) *reinterpret_cast<volatile int *>(chk) = (bit);          \
    } while (0)
#else
#define VCHK(chk, cond, bit) do { } while (0)
#endif

constexpr uint32_t EMPTY = 0xffffffffu;
// Probe window of the u32 visited table (lookup and insert).  A short window keeps lookups cheap
// once the table is full (every absent id probes the whole window): on C4's 10M-row code path
// a window of 2 is 31% faster than 32 with 0.2% more re-evaluated ids (4: -26%, 1: -29%).
#ifndef VSAG_MAX_PROBE
#define VSAG_MAX_PROBE 2
#endif
constexpr int MAX_PROBE = VSAG_MAX_PROBE;
#ifndef VSAG_RK_PER_LANE
#define VSAG_RK_PER_LANE 8
#endif
constexpr int RK_PER_LANE = VSAG_RK_PER_LANE;  // re-rank keys held in registers per lane (R' <= 256 fully in registers)


// Number of entries of pool[0, n) whose key is < key (branchless binary search over a
// power-of-two span; all lanes run the same number of steps).  The expanded flag (bit 0)
// does not change the order of different nodes' keys, so no masking is needed.
__device__ __forceinline__ int pool_lower_bound(const uint64_t *pool, int n, int span, uint64_t key) {
    int pos = 0;
    for (int step = span >> 1; step > 0; step >>= 1) {
        const int t = pos + step;
        if (t <= n && pool[t - 1] < key) pos = t;
    }
    if (pos < n && pool[pos] < key) pos++;
    return pos;
}

// Visited-set test-and-insert, u32 variant (used when a 15-bit tag cannot identify an
// id): open addressing, linear probing, full ids, CAS inserts.  Returns true if `id` was
// not known to be visited.
__device__ __forceinline__ bool visit32(uint32_t *tab, int h_log2, int id, int &miss) {
    const uint32_t mask = (1u << h_log2) - 1u;
    uint32_t h = ((uint32_t)id * 0x9E3779B1u) >> (32 - h_log2);
    for (int probe = 0; probe < MAX_PROBE; probe++) {
        uint32_t cur = tab[h];
        if (cur == (uint32_t)id) return false;
        if (cur == EMPTY) {
            cur = atomicCAS(tab + h, EMPTY, (uint32_t)id);
            if (cur == EMPTY) return true;
            if (cur == (uint32_t)id) return false;
        }
        h = (h + 1) & mask;
    }
    miss++;
    return true;
}

// Visited set, kind 4: an exact bitset of n bits per resident warp in device memory (L2 /
// HBM), cleared at the start of every query; test-and-set with one atomicOr per id.  Never
// forgets.  Ids must be distinct across the lanes of a call (rows are de-duplicated).
__device__ __forceinline__ bool visit_bits(uint32_t *bits, int id) {
    const uint32_t b = 1u << (id & 31);
    return (atomicOr(bits + (id >> 5), b) & b) == 0u;
}

// Visited-set, u16 variant: buckets of 8 u16 (one 16-byte LDS): slot 0 = fill count
// (>= 7 means full), slots 1..7 = tags.  An id splits into its low nb_log2 bits (the
// primary bucket b1) and the rest t < 2^14; its tag in b1 is t + 0x400, and its
// alternate bucket is b2 = b1 ^ f(t) with tag (t + 0x400) | 0x8000.  (bucket, stored tag)
// identifies exactly one id, so a hit is never a false positive.  Tags are normal fp16
// bit patterns (exponent 1..16, never 0, inf or NaN; distinct patterns are distinct
// values) and counts / empty slots are fp16 subnormals or zero, so one HSET2.EQ per
// 32-bit word compares two slots exactly.  An id goes to b1 while b1 has room, else to
// b2; a bucket never empties, so a lookup only reads b2 when b1 is full.  When both are
// full, one of b1's four oldest tags is evicted (the id is forgotten, counted in `miss`;
// DESIGN.md §6 shows the traversal is unchanged).
__device__ __forceinline__ bool any_half_eq(const uint4 &x, uint32_t pat) {
    const __half2 p = *reinterpret_cast<const __half2 *>(&pat);
    const uint32_t m = __heq2_mask(*reinterpret_cast<const __half2 *>(&x.x), p) |
                       __heq2_mask(*reinterpret_cast<const __half2 *>(&x.y), p) |
                       __heq2_mask(*reinterpret_cast<const __half2 *>(&x.z), p) |
                       __heq2_mask(*reinterpret_cast<const __half2 *>(&x.w), p);
    return m != 0u;
}

struct Tab16 {
    uint32_t bmask;  // bucket mask
    int nb_log2;
    __device__ __forceinline__ Tab16(int nb_log2_, int id_bits) {
        (void)id_bits;
        bmask = (1u << nb_log2_) - 1u;
        nb_log2 = nb_log2_;
    }
    __device__ __forceinline__ void locate(int id, uint32_t &b1, uint32_t &tag) const {
        b1 = (uint32_t)id & bmask;
        tag = ((uint32_t)id >> nb_log2) + 0x400u;
    }
    // the alternate bucket (only read once the primary one is full)
    __device__ __forceinline__ uint32_t alt(uint32_t b1, uint32_t tag) const {
        return b1 ^ ((((tag - 0x400u) * 0x9E3779B1u) >> 11) & bmask);
    }
};

// One round of lookups+inserts for one id per lane (id < 0: none) over the lanes of
// `mask` (all of them call it).  Lookups only read; an insert takes its slot with a
// shared-memory atomicAdd on the bucket's first word (the count sits in its low half
// and stays <= 7 + 32, an fp16 subnormal below every tag, so it never carries into slot
// 1 and never equals a tag), so lanes inserting into the same bucket get distinct
// slots without any re-check.  A bucket without room evicts one of its four oldest
// tags instead (the displaced id is forgotten; `miss` counts these).  Ids must be
// distinct across the lanes (callers de-duplicate rows that repeat an id).  Returns
// true if the lane's id was not in V (it is evaluated).
__device__ __forceinline__ bool visit16_round(uint16_t *tab, const Tab16 &tb, int id, int &miss,
                                              uint32_t mask = 0xffffffffu, int *chk = nullptr) {
    // straight-line for the common path: a lane without an id looks up id 0's bucket and
    // never inserts; only the second-bucket probe and the slot claim are conditional
    uint32_t b1, tag1;
    tb.locate(max(id, 0), b1, tag1);
    const uint4 x1 = *reinterpret_cast<const uint4 *>(tab + b1 * 8);
    bool found = any_half_eq(x1, tag1 * 0x10001u);
    uint32_t bk = b1, tg = tag1, c = x1.x & 0xffffu;
    if (id >= 0 && !found && c >= 7) {
        const uint32_t b2 = tb.alt(b1, tag1), tag2 = tag1 | 0x8000u;
        const uint4 x2 = *reinterpret_cast<const uint4 *>(tab + b2 * 8);
        found = any_half_eq(x2, tag2 * 0x10001u);
        const uint32_t c2 = x2.x & 0xffffu;
        if (c2 < 7) {
            bk = b2;
            tg = tag2;
            c = c2;
        }
    }
    const bool isnew = id >= 0 && !found;
    // only a bucket seen with room is counted up, so a count never exceeds 7 + 31
    const bool room = isnew && c < 7;
    uint32_t old = 0;
    {   // predicated ATOMS (no branch around it)
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(tab + bk * 8);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p atom.shared.add.u32 %0, [%1], 1;\n\t}"
                     : "+r"(old) : "r"(a), "r"((uint32_t)room) : "memory");
    }
    uint32_t slot = room ? (old & 0xffffu) + 1 : 8;
    const bool evict = isnew && slot > 7;
    if (evict) {
        slot = 1 + (tg & 3u);
        miss++;
    }
    VCHK(chk, !isnew || (bk <= tb.bmask && slot >= 1 && slot <= 7), 8);
    if (isnew) tab[bk * 8 + slot] = (uint16_t)tg;
    __syncwarp(mask);
    return isnew;
}

// Top-k of the R' (tau_h, id) keys in rk[0, nhp): k rounds of a warp-wide argmin (keys are
// distinct).  Each lane keeps RKL keys in registers (32 * RKL >= nhp in the usual case; any
// further keys stay in shared memory), so the instantiation with the fewest registers that
// covers nhp is the fastest (C1, R' = 132: 5 keys per lane instead of 8, -1.2% step time).
template <int RKL, bool TRACE>
__device__ __forceinline__ void topk_out(const KParams &p, int q, uint64_t *rk, int nhp, int lane) {
    {
        uint64_t kv[RKL];
#pragma unroll
        for (int j = 0; j < RKL; j++) {
            const int t = lane + 32 * j;
            kv[j] = t < nhp ? rk[t] : KEY_INF;
        }
        __syncwarp();
        const int kout = min(p.k, nhp);
        if (TRACE && lane == 0 && p.t_nhp) p.t_nhp[q] = nhp;
        for (int t = 0; t < kout; t++) {
            uint64_t mn = KEY_INF;
#pragma unroll
            for (int j = 0; j < RKL; j++) mn = min(mn, kv[j]);
            for (int j = RKL * 32 + lane; j < nhp; j += 32) mn = min(mn, rk[j]);
            const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(mn >> 32));
            const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(mn >> 32) == hi ? (uint32_t)mn : 0xffffffffu);
            const uint64_t best = ((uint64_t)hi << 32) | lo;
#pragma unroll
            for (int j = 0; j < RKL; j++)
                if (kv[j] == best) kv[j] = KEY_INF;
            for (int j = RKL * 32 + lane; j < nhp; j += 32)
                if (rk[j] == best) rk[j] = KEY_INF;
            VCHK(p.check, q < p.nq && t < p.k, 32);
            if (lane == 0) {
                p.out_ids[(int64_t)q * p.k + t] = (int32_t)(best & 0xffffffffu);
                p.out_dists[(int64_t)q * p.k + t] = ordf((uint32_t)(best >> 32));
            }
        }
        for (int t = kout + lane; t < p.k; t += 32) {
            p.out_ids[(int64_t)q * p.k + t] = -1;
            p.out_dists[(int64_t)q * p.k + t] = __int_as_float(0x7f800000);
        }
    }
}

// Trace outputs, the selective re-rank of the first R' = min(R, |C|) pool entries with
// tau_h (Alg. 1 line 18; fp32 rows, fp64 accumulation, one fp32 rounding, R-16) and the
// top-k by (tau_h, id).  Whole warp (full mask); `tab` (>= 8 * R' bytes) is scratch.
template <int M, bool TRACE = true>
__device__ __forceinline__ void finish_query(const KParams &p, int R, int q, const uint64_t *pool, int psz, uint8_t *tab,
                                             int hops, int n_lp, int mtot, int lane) {
    constexpr bool L2 = mode_l2(M);  // the weighted L2 re-ranks with plain L2
    // ---- trace
    const int rr = min(R, psz);
    {
        if (TRACE && lane == 0) {
            if (p.t_hops) p.t_hops[q] = hops;
            if (p.t_nlp) p.t_nlp[q] = n_lp;
            if (p.t_miss) p.t_miss[q] = mtot;
        }
        if (TRACE && p.t_expanded)
            for (int t = hops + lane; t < p.max_hops; t += 32) p.t_expanded[(int64_t)q * p.max_hops + t] = -1;
        if (TRACE && (p.t_pool_ids || p.t_pool_tau))
        for (int t = lane; t < p.L; t += 32) {
            const bool has = t < psz;
            if (p.t_pool_ids) p.t_pool_ids[(int64_t)q * p.L + t] = has ? key_id(pool[t]) : -1;
            if (p.t_pool_tau) p.t_pool_tau[(int64_t)q * p.L + t] = has ? key_tau(pool[t]) : 0x7fffffff;
        }
    }
    __syncwarp();

    // ---- a7: selective re-rank of the first R' entries (Alg. 1 line 18)
    uint64_t *rk = reinterpret_cast<uint64_t *>(tab);  // V is dead now
    const float *qv = p.queries + (int64_t)q * p.d;
    const bool vec4 = (p.d & 3) == 0;
    const int nf4 = p.d >> 2;
    const uint32_t rowb = (uint32_t)p.d * 4u;
    // d <= 128: lane f keeps its query float4 in fp64 registers for the whole re-rank
    const bool qreg = vec4 && nf4 <= 32;
    double qd[4] = {0.0, 0.0, 0.0, 0.0};
    if (qreg && lane < nf4) {
        const float4 qa = __ldg(reinterpret_cast<const float4 *>(qv) + lane);
        qd[0] = (double)qa.x;
        qd[1] = (double)qa.y;
        qd[2] = (double)qa.z;
        qd[3] = (double)qa.w;
    }
    int nhp = rr;
    for (int c0 = 0; c0 < rr; c0 += 4) {
        if (p.adaptive && c0 >= p.k) {
            // NEXT-3 (R-27): stop when the first remaining candidate's tau_l lower-bounds
            // tau_h above the k-th best so far, i.e. when k evaluated tau_h lie below the bound
            const double t = (double)key_tau(pool[c0]);
            const double v = t - 2.0002 * sqrt((double)p.d * t);
            const double lb = v > 0.0 ? p.delta_min * p.delta_min * v * (1.0 - 1e-5) : 0.0;
            if (lb > 0.0) {
                __syncwarp();  // rk[0, c0) written by the previous groups
                int below = 0;
                for (int i = lane; i < c0; i += 32) below += (double)ordf((uint32_t)(rk[i] >> 32)) < lb;
                if ((int)__reduce_add_sync(0xffffffffu, (uint32_t)below) >= p.k) {
                    nhp = c0;
                    break;
                }
            }
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        int idc[4];
#pragma unroll
        for (int u = 0; u < 4; u++) idc[u] = key_id(pool[min(c0 + u, rr - 1)]);  // tail repeats a valid id
#pragma unroll
        for (int u = 0; u < 4; u++) VCHK(p.check, idc[u] >= 0 && idc[u] < p.n_base, 4);
        auto row = [&](int u) {
            return reinterpret_cast<const float4 *>(reinterpret_cast<const uint8_t *>(p.base) +
                                                    (uint64_t)(uint32_t)idc[u] * rowb);
        };
        if (qreg) {
            if (lane < nf4) {
                float4 xa[4];
#pragma unroll
                for (int u = 0; u < 4; u++) xa[u] = ldg16_stream(row(u) + lane);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const float xs[4] = {xa[u].x, xa[u].y, xa[u].z, xa[u].w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        // fp64 accumulation, one rounding per step (R-16): the product of two fp32
                        // values is exact in fp64, and so is the square of their fp64 difference
                        // when the two magnitudes are close enough for it to fit 53 bits;
                        // otherwise the fused multiply-add rounds once, far below the 1e-5
                        // relative tolerance of the fp32 result
                        if (L2) {
                            const double df = __dsub_rn(qd[t], (double)xs[t]);
                            acc[u] = __fma_rn(df, df, acc[u]);
                        } else {
                            acc[u] = __fma_rn(qd[t], (double)xs[t], acc[u]);
                        }
                    }
                }
            }
        } else if (vec4) {
            for (int f = lane; f < nf4; f += 32) {
                const float4 qa = __ldg(reinterpret_cast<const float4 *>(qv) + f);
                float4 xa[4];
#pragma unroll
                for (int u = 0; u < 4; u++) xa[u] = ldg16_stream(row(u) + f);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const float qs[4] = {qa.x, qa.y, qa.z, qa.w};
                    const float xs[4] = {xa[u].x, xa[u].y, xa[u].z, xa[u].w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        if (L2) {
                            const double df = __dsub_rn((double)qs[t], (double)xs[t]);
                            acc[u] = __fma_rn(df, df, acc[u]);
                        } else {
                            acc[u] = __fma_rn((double)qs[t], (double)xs[t], acc[u]);
                        }
                    }
                }
            }
        } else {
            for (int j = lane; j < p.d; j += 32) {
                const double qs = (double)__ldg(qv + j);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const double xs = (double)__ldg(reinterpret_cast<const float *>(row(u)) + j);
                    if (L2) {
                        const double df = __dsub_rn(qs, xs);
                        acc[u] = __fma_rn(df, df, acc[u]);
                    } else {
                        acc[u] = __fma_rn(qs, xs, acc[u]);
                    }
                }
            }
        }
        // reduce-scatter of the 4 partial sums: lane bits 0,1 pick the candidate, the
        // remaining three xor steps finish the sum (6 shuffle-adds instead of 20)
        {
            const bool b0 = lane & 1, b1 = lane & 2;
            const double s0 = b0 ? acc[0] : acc[2], s1 = b0 ? acc[1] : acc[3];
            double k0 = b0 ? acc[2] : acc[0], k1 = b0 ? acc[3] : acc[1];
            k0 = __dadd_rn(k0, __shfl_xor_sync(0xffffffffu, s0, 1));
            k1 = __dadd_rn(k1, __shfl_xor_sync(0xffffffffu, s1, 1));
            double sum = __dadd_rn(b1 ? k1 : k0, __shfl_xor_sync(0xffffffffu, b1 ? k0 : k1, 2));
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
            const int u = (b0 ? 2 : 0) + (b1 ? 1 : 0);
            const int cid = key_id(pool[min(c0 + u, rr - 1)]);  // (lanes 0..3 keep the result)
            if (lane < 4 && c0 + u < rr) {  // (rk[c0 + u] is read by the next group's stop test)
                const float th = __double2float_rn(L2 ? sum : -sum);
                VCHK(p.check, (c0 + u) * 8 < p.rk_bytes, 2);
                rk[c0 + u] = ((uint64_t)ford(th) << 32) | (uint32_t)cid;
            }
        }
    }
    __syncwarp();
    // top-k of the R' (tau_h, id) keys
    if (nhp <= 160) topk_out<5, TRACE>(p, q, rk, nhp, lane);
    else topk_out<RK_PER_LANE, TRACE>(p, q, rk, nhp, lane);
}

}  // namespace
}  // namespace vsag
