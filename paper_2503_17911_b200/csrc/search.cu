// search.cu -- rows a5 (seed selection), a6 (hop loop), a7 (re-rank), a8 (output).
//
// Deterministic Access Greedy Search (Alg. 1; App. A)
// for a batch of queries, one WARP per query, persistent grid (each warp pulls the
// next query from a global counter).  Per warp, shared memory holds:
//   pool   the candidate pool C as a sorted array of L = max(ef, R) u64 keys
//          key = (tau_l ^ 0x80000000) << 32 | id << 1 | x  (total order (tau_l, id),
//          R-8; x = "expanded" flag, below the id so it never reorders two nodes);
//   tab    the visited set V: u16 tag buckets (or u32 linear probing for very large
//          n with a small table), reused as the re-rank scratch after the hop loop;
//   new*   the <= R new candidates of the current hop.
// One hop (lines 5-17):
//   select    first unexpanded key in the window [0, ef) (ballot scan from a hint);
//   ids       one coalesced load of the node's R neighbour ids (layout 0: adjacency
//             table; layout 1: the id block of the node's PRS row), usually already
//             in registers: the previous hop predicted this node and loaded its row
//             while it merged;
//   filter    test-and-insert every id in V *before* touching any code -- the
//             paper's deterministic access: only unvisited neighbours
//             are gathered;
//   gather    each unvisited neighbour's code is read with 16-byte loads by a group
//             of G lanes (G = code bytes / 16 rounded up to a power of two), several
//             codes per warp instruction, several instructions in flight;
//   tau_l     VABSDIFF4 + IDP.4A (dist.cuh), int32, reduced over the G lanes;
//   merge     drop keys >= the current L-th key, rank the survivors by counting,
//             binary-search their positions, shift the pool in place.
// After the loop the first R' = min(R, |C|) entries are re-ranked with tau_h:
// fp32 rows gathered with 16-byte loads, fp64 accumulation, one fp32 rounding
// (R-16), k rounds of a warp argmin over (tau_h, id), top-k written out.
//
// Visited set exactness: a lookup HIT is always a truly visited id,
// so the table never drops a node Alg. 1 would have evaluated.  A full bucket forgets
// an id (counted in n_miss); evaluating an already-visited node again cannot change
// the pool, because the pool is always the top-L of every key ever inserted and, once
// anything was forgotten, the merge removes exact duplicates.  Pool and expansion
// order are therefore identical to Alg. 1 with an exact V.
#include <algorithm>

#include "search_common.cuh"

namespace vsag {
namespace {

// pool <- top_L(pool U new) (Alg. 1 line 17 for a whole batch of inserts: the result
// equals inserting them one by one).  Input: s candidate keys
// newk[0, s) (unsorted, each below the current L-th key when the pool is full).
// DEDUP (only once the visited cache has forgotten an id): drop keys that repeat an
// earlier new key or a node already in C.  Then (1) rank the m2 survivors by counting
// (all distinct) and scatter them sorted into sk; (2) merge-path merge of A = pool[0, na)
// and B = sk[0, m2) in place, top 32-block first: final position f takes j(f) elements
// from B, the largest j with j == 0 or B[j-1] < A[f-j] (a log2(m2+1)-step search per
// lane); blocks below the first position that takes a B element are unchanged, so the
// loop stops there.  Reads of a block happen before its writes, and lower blocks only
// read positions below it.  Updates psz and the first-unexpanded hint.
template <int E, bool DEDUP>
__device__ __forceinline__ void merge_new(int s, uint64_t *pool, int &psz, int L, int span, uint64_t *newk,
                                          uint64_t *sk, int &hint, int lane) {
    uint64_t v[E];
    bool valid[E];
#pragma unroll
    for (int r = 0; r < E; r++) {
        const int e = lane + 32 * r;
        v[r] = e < s ? newk[e] : KEY_INF;
        valid[r] = e < s;
    }
    int m2 = s;
    if (DEDUP) {
        for (int i = 0; i < s; i++) {
            const uint64_t o = newk[i];
#pragma unroll
            for (int r = 0; r < E; r++)
                if (o == v[r] && i < lane + 32 * r) valid[r] = false;
        }
#pragma unroll
        for (int r = 0; r < E; r++) {
            if (valid[r]) {
                const int lb = pool_lower_bound(pool, psz, span, v[r]);
                if (lb < psz && kmask(pool[lb]) == v[r]) valid[r] = false;  // already in C
            }
            if (!valid[r]) v[r] = KEY_INF;
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < E; r++)
            if (lane + 32 * r < s) newk[lane + 32 * r] = v[r];
        m2 = 0;
#pragma unroll
        for (int r = 0; r < E; r++) m2 += __popc(__ballot_sync(0xffffffffu, valid[r]));
        __syncwarp();
        if (m2 == 0) return;
    }
    int rank[E];
#pragma unroll
    for (int r = 0; r < E; r++) rank[r] = 0;
    for (int i = 0; i < s; i++) {
        const uint64_t o = newk[i];
#pragma unroll
        for (int r = 0; r < E; r++) rank[r] += o < v[r];
    }
#pragma unroll
    for (int r = 0; r < E; r++)
        if (valid[r]) sk[rank[r]] = v[r];
    __syncwarp();
    const int na = psz;
    const int total = min(L, na + m2);
    int first_b = L;
    STAT(6, m2);
    for (int base = (total - 1) & ~31; base >= 0; base -= 32) {
        const int f = base + lane;
        uint64_t val = 0;
        bool from_b = false;
        int j = 0;
        if (f < total) {
            int lo = max(0, f - na), hi = min(f, m2);
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (f - mid >= na || sk[mid - 1] < pool[f - mid]) lo = mid; else hi = mid - 1;
            }
            j = lo;
            const uint64_t a = f - j < na ? pool[f - j] : KEY_INF;
            const uint64_t bk = j < m2 ? sk[j] : KEY_INF;
            from_b = bk < a;
            val = from_b ? bk : a;
        }
        STAT(7, 1);
        const int j0 = __shfl_sync(0xffffffffu, j, 0);
        const uint32_t bb = __ballot_sync(0xffffffffu, from_b);
        if (bb) first_b = base + __ffs(bb) - 1;
        __syncwarp();
        if (f < total) pool[f] = val;
        if (j0 == 0) break;  // no B element below `base`: pool[0, base) is unchanged
        __syncwarp();
    }
    __syncwarp();
    psz = total;
    hint = min(hint, first_b);
}

template <int M, int CPL, int GL, int E>
__global__ void __launch_bounds__(128, 8) search_kernel(const KParams p) {
    constexpr int OPW = (M == L2_4 || M == IP_4) ? 2 : 1;
    constexpr int QW = 4 * OPW;  // operand words per 16-byte code chunk
    constexpr int UNR = CPL >= 2 ? 1 : 2;  // gather passes issued back to back
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    uint8_t *wbase = smem + (threadIdx.x >> 5) * p.smem_per_warp;
    uint64_t *pool = reinterpret_cast<uint64_t *>(wbase);
    uint8_t *tab = wbase + p.off_tab;
    uint64_t *newk = reinterpret_cast<uint64_t *>(wbase + p.off_newk);
    int *newid = reinterpret_cast<int *>(wbase + p.off_newid);
    int *newslot = reinterpret_cast<int *>(wbase + p.off_newslot);
    uint64_t *sk = reinterpret_cast<uint64_t *>(wbase + p.off_newid);  // aliases newid/newslot (dead by then)
    constexpr int G = 1 << GL;
    constexpr int npp = 32 >> GL;      // codes per gather pass
    const int gl = lane & (G - 1);     // lane within its code group
    const int gi = lane >> GL;         // code group index within the warp
    int span = 1;
    while (span < p.L) span <<= 1;
    uint16_t *tab16 = reinterpret_cast<uint16_t *>(tab);
    uint32_t *tab32 = reinterpret_cast<uint32_t *>(tab);
    const Tab16 tb{p.nb_log2, p.id_bits};

    for (;;) {
        int q = 0;
        if (lane == 0) q = (int)atomicAdd(p.counter, 1u);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= p.nq) break;

        // ---- query operand chunks into registers (a4 output)
        uint32_t qr[CPL][QW];
        const uint32_t *opq = p.op + (int64_t)q * p.op_stride;
#pragma unroll
        for (int mm = 0; mm < CPL; mm++) {
            const int c = gl + G * mm;
#pragma unroll
            for (int t = 0; t < QW; t += 4) {
                uint4 w = make_uint4(0, 0, 0, 0);
                if (c < p.chunks) w = *reinterpret_cast<const uint4 *>(opq + c * QW + t);
                qr[mm][t] = w.x;
                qr[mm][t + 1] = w.y;
                qr[mm][t + 2] = w.z;
                qr[mm][t + 3] = w.w;
            }
        }
        // ---- clear V
        {
            const uint32_t fill = p.tab16 ? 0u : EMPTY;
            for (int i = lane * 16; i < p.tab_bytes; i += 512)
                *reinterpret_cast<uint4 *>(tab + i) = make_uint4(fill, fill, fill, fill);
        }
        __syncwarp();

        // ---- a5: C <- top_L of the entry set by (tau_l, id)  (Alg. 1 line 3), selected
        // by seed_select_kernel; copy it into the pool (positions >= psz hold KEY_INF)
        int psz = p.init_psz[q], hint = 0;
        for (int t = lane; t < p.lcap; t += 32) pool[t] = t < psz ? p.init_keys[(int64_t)q * p.L + t] : KEY_INF;
        __syncwarp();
        int miss = 0;
        // V <- ids(C) (R-10)
        for (int t0 = 0; t0 < psz; t0 += 32) {
            const int t = t0 + lane;
            const int id = t < psz ? key_id(pool[t]) : -1;
            if (p.tab16) visit16_round(tab16, tb, id, miss);
            else if (id >= 0) visit32(tab32, p.h_log2, id, miss);
        }
        __syncwarp();
        int n_lp = p.S, hops = 0;

        // ---- a6: hop loop (Alg. 1 lines 4-17)
        int pred_node = -1;  // node whose id row is already in flight (nb_pref)
        int nb_pref[E];
        for (;;) {
            const int lim = min(p.ef, psz);
            int sel = -1;
            uint64_t next2 = KEY_INF;  // key of the second unexpanded entry of the window block
            for (int b = hint; b < lim; b += 32) {
                const int t = b + lane;
                const uint64_t pt = t < lim ? pool[t] : KEY_FLAG;
                const uint32_t bal = __ballot_sync(0xffffffffu, !(pt & KEY_FLAG));
                if (bal) {
                    sel = b + __ffs(bal) - 1;
                    const uint32_t bal2 = bal & (bal - 1);
                    const uint64_t k2 = __shfl_sync(0xffffffffu, pt, bal2 ? __ffs(bal2) - 1 : 0);
                    if (bal2) next2 = k2;
                    break;
                }
            }
            if (sel < 0) break;
            STAT(8, (sel - hint) / 32 + 1);
            const int node = key_id(pool[sel]);
            __syncwarp();
            if (lane == 0) pool[sel] |= KEY_FLAG;
            hint = sel + 1;
            if (p.t_expanded && lane == 0 && hops < p.max_hops) p.t_expanded[(int64_t)q * p.max_hops + hops] = node;
            hops++;

            // neighbour ids (lines 7-10: ids only, no vector data yet).  If the previous hop
            // predicted this node, its row is already in registers.
            int nb[E];
            STAT(0, 1);
            STAT(1, node == pred_node);
            if (node == pred_node) {
#pragma unroll
                for (int r = 0; r < E; r++) nb[r] = nb_pref[r];
            } else {
                const int32_t *ids = p.layout == 0 ? p.adj + (int64_t)node * p.degree
                                                   : reinterpret_cast<const int32_t *>(p.rows + (int64_t)node * p.row_bytes);
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int t = lane + 32 * r;
                    nb[r] = t < p.degree ? __ldg(ids + t) : -1;
                }
            }
            // visited filter, one 32-id slice at a time (a later slice sees the earlier one's
            // inserts); rows that repeat an id keep only its first lane per slice
            int m = 0;
#pragma unroll
            for (int r = 0; r < E; r++) {
                int id = nb[r];
                if (p.row_dups) {
                    const uint32_t mm = __match_any_sync(0xffffffffu, id);
                    if (mm & lanemask_lt()) id = -1;
                }
                bool isnew;
                if (p.tab16) {
                    isnew = visit16_round(tab16, tb, id, miss);
                } else {
                    isnew = id >= 0 && visit32(tab32, p.h_log2, id, miss);
                    __syncwarp();
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, isnew);
                if (isnew) {
                    const int rk = m + __popc(bal & lanemask_lt());
                    newid[rk] = id;
                    newslot[rk] = p.layout == 0 ? id : lane + 32 * r;  // code index in cbase
                }
                m += __popc(bal);
            }
            __syncwarp();
            if (m == 0) {  // nothing new: the next expansion is the window's next entry
                pred_node = next2 == KEY_INF ? -1 : key_id(next2);
                if (pred_node >= 0) {
                    const int32_t *ids2 = p.layout == 0 ? p.adj + (int64_t)pred_node * p.degree
                                                        : reinterpret_cast<const int32_t *>(p.rows + (int64_t)pred_node * p.row_bytes);
#pragma unroll
                    for (int r = 0; r < E; r++) {
                        const int t = lane + 32 * r;
                        nb_pref[r] = t < p.degree ? __ldg(ids2 + t) : -1;
                    }
                }
                continue;
            }
            n_lp += m;
            STAT(2, m);
            STAT(3, 1);
            const bool forgot = __any_sync(0xffffffffu, miss != 0);  // V has dropped an id: dedupe merges

            // lines 13-17: gather the unvisited codes, tau_l, keys.  A key that is not below
            // the current L-th key (pool full) cannot enter C and is dropped right here.
            const uint8_t *cbase = p.layout == 0 ? p.codes : p.rows + (int64_t)node * p.row_bytes + p.ids_bytes;
            const uint64_t worst = psz == p.L ? pool[p.L - 1] : KEY_INF;
            int ns = 0;
            for (int b0 = 0; b0 < m; b0 += npp * UNR) {
                uint4 cv[UNR][CPL];
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    const int idx = b0 + u * npp + gi;
                    const bool ok = idx < m;
                    const uint8_t *cp = nullptr;
                    if (ok) {
                        cp = cbase + (int64_t)newslot[idx] * p.cbp;
                    }
#pragma unroll
                    for (int mm = 0; mm < CPL; mm++) {
                        const int c = gl + G * mm;
                        cv[u][mm] = (ok && c < p.chunks) ? ldg16(cp + c * 16) : make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    int acc = 0;
#pragma unroll
                    for (int mm = 0; mm < CPL; mm++) {
                        const uint32_t c4[4] = {cv[u][mm].x, cv[u][mm].y, cv[u][mm].z, cv[u][mm].w};
#pragma unroll
                        for (int w = 0; w < 4; w++)
                            acc = word_dist<M>(acc, qr[mm][w * OPW], OPW == 2 ? qr[mm][w * OPW + 1] : 0u, c4[w]);
                    }
#pragma unroll
                    for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    const int idx = b0 + u * npp + gi;
                    const uint64_t key = make_key(finish_tau<M>(acc), idx < m ? newid[idx] : 0);
                    const bool ok = gl == 0 && idx < m && key < worst;
                    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                    if (ok) newk[ns + __popc(bal & lanemask_lt())] = key;
                    ns += __popc(bal);
                }
            }
            __syncwarp();
            // The next expansion is the smaller of the window's next unexpanded entry and the
            // best surviving new key (when it lands inside the window); start loading that
            // node's id row now so the load overlaps the merge.
            {
                uint64_t kb = KEY_INF;
#pragma unroll
                for (int r = 0; r < E; r++)
                    if (lane + 32 * r < ns) kb = min(kb, newk[lane + 32 * r]);
                const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(kb >> 32));
                const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(kb >> 32) == hi ? (uint32_t)kb : 0xffffffffu);
                kb = ((uint64_t)hi << 32) | lo;
                const uint64_t pk = min(kb, next2);
                pred_node = pk == KEY_INF ? -1 : key_id(pk);
                if (pred_node >= 0) {
                    const int32_t *ids2 = p.layout == 0 ? p.adj + (int64_t)pred_node * p.degree
                                                        : reinterpret_cast<const int32_t *>(p.rows + (int64_t)pred_node * p.row_bytes);
#pragma unroll
                    for (int r = 0; r < E; r++) {
                        const int t = lane + 32 * r;
                        nb_pref[r] = t < p.degree ? __ldg(ids2 + t) : -1;
                    }
                }
            }
            STAT(4, ns);
            STAT(12 + min(ns, 9), 1);
            if (ns > 0) {
                STAT(5, 1);
                STAT(10, forgot);
                if (forgot) merge_new<E, true>(ns, pool, psz, p.L, span, newk, sk, hint, lane);
                else merge_new<E, false>(ns, pool, psz, p.L, span, newk, sk, hint, lane);
            }
        }

        // ---- trace, a7 re-rank, a8 output
        finish_query(p, q, pool, psz, tab, hops, n_lp, __reduce_add_sync(0xffffffffu, miss), lane);
        __syncwarp();
    }
}

template <int M, int CPL, int GL, int E>
cudaError_t launch_typed(const KParams &kp, int wpb, cudaStream_t s, SearchLaunch *info, int64_t nq) {
    auto kern = search_kernel<M, CPL, GL, E>;
    const size_t smem = (size_t)wpb * kp.smem_per_warp;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wpb * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (nq + wpb - 1) / wpb;
    if (blocks > need) blocks = need;
    if (info) {
        info->warps_per_block = wpb;
        info->blocks = (int)blocks;
        info->smem_per_warp = kp.smem_per_warp;
    }
    kern<<<(unsigned)blocks, wpb * 32, smem, s>>>(kp);
    return cudaGetLastError();
}

// Code-group shapes: G = 2^GL lanes read one code (16 B each); CPL 16-byte chunks per lane.
template <int M, int E>
cudaError_t launch_cpl(int cpl, int gl, const KParams &kp, int wpb, cudaStream_t s, SearchLaunch *info, int64_t nq) {
    if (cpl == 1) {
        switch (gl) {
            case 2: return launch_typed<M, 1, 2, E>(kp, wpb, s, info, nq);
            case 3: return launch_typed<M, 1, 3, E>(kp, wpb, s, info, nq);
            case 4: return launch_typed<M, 1, 4, E>(kp, wpb, s, info, nq);
            default: return launch_typed<M, 1, 5, E>(kp, wpb, s, info, nq);
        }
    }
    if (cpl == 2) {
        switch (gl) {
            case 2: return launch_typed<M, 2, 2, E>(kp, wpb, s, info, nq);
            case 3: return launch_typed<M, 2, 3, E>(kp, wpb, s, info, nq);
            case 4: return launch_typed<M, 2, 4, E>(kp, wpb, s, info, nq);
            default: return launch_typed<M, 2, 5, E>(kp, wpb, s, info, nq);
        }
    }
    return launch_typed<M, 4, 5, E>(kp, wpb, s, info, nq);
}

template <int E>
cudaError_t launch_mode(int mode, int cpl, int gl, const KParams &kp, int wpb, cudaStream_t s, SearchLaunch *info,
                        int64_t nq) {
    switch (mode) {
        case L2_8: return launch_cpl<L2_8, E>(cpl, gl, kp, wpb, s, info, nq);
        case L2_4: return launch_cpl<L2_4, E>(cpl, gl, kp, wpb, s, info, nq);
        case IP_8: return launch_cpl<IP_8, E>(cpl, gl, kp, wpb, s, info, nq);
        default: return launch_cpl<IP_4, E>(cpl, gl, kp, wpb, s, info, nq);
    }
}

int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) r++;
    return r;
}

// Lanes per code (returns log2 G) and 16-byte chunks per lane for a code of `chunks`
// 16-byte chunks.  Default: two chunks per lane (one gather pass covers 32/G codes),
// which measured fastest on C1 (tools/sweep_launch.py); code_lanes overrides G.
int code_shape(int chunks, int code_lanes, int *cpl) {
    int G;
    if (code_lanes >= 4 && code_lanes <= 32) {
        G = code_lanes;
    } else if (chunks <= 4) {
        G = 4;
    } else {
        G = 4;
        while (G * 2 < chunks && G < 32) G <<= 1;
    }
    const int need = (chunks + G - 1) / G;
    *cpl = need <= 1 ? 1 : (need <= 2 ? 2 : 4);
    if (need > 4) return -1;
    return ilog2(G);
}

}  // namespace

// The u16 bucket table applies when a 14-bit tag plus the bucket index identify an id.
bool visited_u16(int H, int64_t n) {
    int id_bits = 1;
    while (id_bits < 31 && ((int64_t)1 << id_bits) < n) id_bits++;
    return id_bits - (ilog2(H) - 3) <= 14;
}

// Shared-memory bytes one warp needs for a given (L, R, H).
size_t search_smem_per_warp(int L, int R, int H, int64_t n, int degree, int cbp, int code_lanes) {
    (void)degree;
    (void)cbp;
    (void)code_lanes;
    const size_t lcap = ((size_t)L + 31) / 32 * 32;
    int rk = 32;
    while (rk < R) rk <<= 1;
    size_t tab = (size_t)H * (visited_u16(H, n) ? 2 : 4);
    if ((size_t)rk * 8 > tab) tab = (size_t)rk * 8;
    return lcap * 8 + tab + NEW_CAP * 8 + NEW_CAP * 4 * 2;
}

cudaError_t launch_search(const SearchArgs &a, int warps_per_block, cudaStream_t s, SearchLaunch *info) {
    const Index &ix = *a.ix;
    KParams kp{};
    kp.op = a.op;
    kp.op_stride = a.op_stride_words;
    kp.seed_tau = a.seed_tau;
    kp.entry = ix.entry;
    kp.S = ix.n_entry;
    kp.adj = ix.adj;
    kp.codes = ix.codes;
    kp.rows = ix.rows;
    kp.row_bytes = ix.row_bytes;
    kp.ids_bytes = ix.ids_bytes;
    kp.base = ix.base;
    kp.queries = a.queries;
    kp.d = ix.d;
    kp.nq = a.nq;
    kp.k = a.k;
    kp.ef = a.ef;
    kp.R = a.rerank_n;
    kp.L = a.L;
    kp.degree = ix.degree;
    kp.cbp = ix.cbp;
    kp.chunks = ix.cbp / 16;
    int cpl = 1;
    kp.g_log2 = code_shape(kp.chunks, a.code_lanes, &cpl);
    kp.layout = ix.layout;
    kp.metric = a.metric;
    kp.h_log2 = ilog2(a.visited_slots);
    kp.id_bits = 1;
    while (kp.id_bits < 31 && ((int64_t)1 << kp.id_bits) < ix.n) kp.id_bits++;
    kp.nb_log2 = kp.h_log2 - 3;
    kp.tab16 = visited_u16(a.visited_slots, ix.n);
    kp.tab_bytes = a.visited_slots * (kp.tab16 ? 2 : 4);
    kp.row_dups = ix.row_dups;
    const size_t lcap = ((size_t)a.L + 31) / 32 * 32;
    kp.lcap = (int)lcap;
    int rk = 32;
    while (rk < a.rerank_n) rk <<= 1;
    size_t tab = (size_t)kp.tab_bytes;
    if ((size_t)rk * 8 > tab) tab = (size_t)rk * 8;
    kp.off_tab = (int)(lcap * 8);
    kp.off_newk = kp.off_tab + (int)tab;
    kp.off_newid = kp.off_newk + NEW_CAP * 8;
    kp.off_newslot = kp.off_newid + NEW_CAP * 4;
    kp.smem_per_warp = kp.off_newslot + NEW_CAP * 4;
    kp.out_ids = a.out_ids;
    kp.out_dists = a.out_dists;
    if (a.has_trace) {
        kp.t_hops = a.trace.hops;
        kp.t_expanded = a.trace.expanded;
        kp.t_nlp = a.trace.n_lp;
        kp.t_nhp = a.trace.n_hp;
        kp.t_miss = a.trace.n_miss;
        kp.t_pool_ids = a.trace.pool_ids;
        kp.t_pool_tau = a.trace.pool_tau;
        kp.max_hops = a.trace.expanded ? a.trace.max_hops : 0;
    }
    kp.counter = a.counter;
    kp.init_keys = a.init_keys;
    kp.init_psz = a.init_psz;
    if (kp.g_log2 < 0) return cudaErrorInvalidValue;
    if (info) info->visited_kind = kp.tab16 ? 2 : 3;
    if (ix.degree <= 32) return launch_mode<1>(a.mode, cpl, kp.g_log2, kp, warps_per_block, s, info, a.nq);
    return launch_mode<2>(a.mode, cpl, kp.g_log2, kp, warps_per_block, s, info, a.nq);
}

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
