// search.cu -- rows a5 (seed selection), a6 (hop loop), a7 (re-rank), a8 (output).
//
// Deterministic Access Greedy Search (Alg. 1; App. A)
// for a batch of queries, one WARP per query, persistent grid (each warp pulls the
// next query from a global counter).  Per warp, shared memory holds:
//   pool   the candidate pool C as a sorted array of L = max(ef, R) u64 keys
//          key = (tau_l ^ 0x80000000) << 32 | id   (total order (tau_l, id), R-8),
//          bit 31 of the key = "expanded" flag (masked out of every comparison);
//   tab    the visited set V as an open-addressing u32 hash table (reused as the
//          re-rank scratch after the hop loop);
//   new*   the <= R new candidates of the current hop.
// One hop (lines 5-17):
//   select    first unexpanded key in the window [0, ef) (ballot scan from a hint);
//   ids       one coalesced load of the node's R neighbour ids (layout 0: adjacency
//             table; layout 1: the id block of the node's PRS row);
//   filter    test-and-insert every id in V *before* touching any code -- the
//             paper's deterministic access: only unvisited neighbours
//             are gathered;
//   gather    each unvisited neighbour's code is read with 16-byte loads by a group
//             of G lanes (G = code bytes / 16 rounded up to a power of two), several
//             codes per warp instruction, several instructions in flight;
//   tau_l     VABSDIFF4 + IDP.4A (dist.cuh), int32, reduced over the G lanes;
//   merge     warp bitonic sort of the new keys, drop duplicates / keys >= the
//             current L-th key, binary-search positions, in-place shift of the pool.
// After the loop the first R' = min(R, |C|) entries are re-ranked with tau_h:
// fp32 rows gathered with 16-byte loads, fp64 accumulation, one fp32 rounding
// (R-16), bitonic sort of (tau_h, id), top-k written out.
//
// Visited set exactness: a lookup HIT is always a truly visited id,
// so the table never drops a node Alg. 1 would have evaluated.  If a probe sequence
// is full the id is evaluated but not remembered (counted in n_miss); evaluating an
// already-visited node again cannot change the pool, because the pool is always the
// top-L of every key ever inserted and the merge removes exact duplicates.  Pool and
// expansion order are therefore identical to Alg. 1 with an exact V.
#include <algorithm>

#include "dist.cuh"
#include "keys.cuh"

namespace vsag {
namespace {

constexpr uint32_t EMPTY = 0xffffffffu;
constexpr int MAX_PROBE = 32;
constexpr int NEW_CAP = 64;  // >= VSAG_MAX_DEGREE
constexpr int RK_PER_LANE = 8;  // re-rank keys held in registers per lane (R' <= 256 fully in registers)

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
    int tab16, nb_log2, id_bits, tab_bytes;
    int smem_per_warp, off_tab, off_newk, off_newlb, off_newid, off_newslot;
    int32_t *out_ids;
    float *out_dists;
    int32_t *t_hops, *t_expanded, *t_nlp, *t_nhp, *t_miss, *t_pool_ids, *t_pool_tau;
    int max_hops;
    unsigned int *counter;
};

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}

// Number of entries of pool[0, n) whose masked key is < key (branchless binary search
// over a power-of-two span; all lanes run the same number of steps).
__device__ __forceinline__ int pool_lower_bound(const uint64_t *pool, int n, int span, uint64_t key) {
    int pos = 0;
    for (int step = span >> 1; step > 0; step >>= 1) {
        const int t = pos + step;
        if (t <= n && kmask(pool[t - 1]) < key) pos = t;
    }
    if (pos < n && kmask(pool[pos]) < key) pos++;
    return pos;
}

// pool <- top_L(pool U new) with exact duplicates removed (Alg. 1 line 17 for a whole
// batch of inserts: the result equals inserting them one by one).
// Input: s candidate keys newk[0, s) (unsorted, already known to be < the current
// L-th key when the pool is full).  Steps: (1) drop keys that repeat an earlier new key
// (only possible after a visited-cache miss, check_dups) or that are already in C;
// (2) rank the survivors by counting (all distinct), scatter them sorted into sk/slb;
// (3) shift pool entries p >= lb_0 up by #{r : lb_r <= p}, top block first; (4) write
// the new keys at lb_r + r.  Updates psz and the first-unexpanded hint.
template <int E>
__device__ __forceinline__ void merge_new(int s, bool check_dups, uint64_t *pool, int &psz, int L, int span,
                                          uint64_t *newk, uint64_t *sk, int *slb, int &hint, int lane) {
    if (s == 0) return;
    uint64_t v[E];
    int lb[E];
    bool valid[E];
#pragma unroll
    for (int r = 0; r < E; r++) {
        const int e = lane + 32 * r;
        v[r] = e < s ? newk[e] : KEY_INF;
        valid[r] = e < s;
    }
    if (check_dups) {
        for (int i = 0; i < s; i++) {
            const uint64_t o = newk[i];
#pragma unroll
            for (int r = 0; r < E; r++)
                if (o == v[r] && i < lane + 32 * r) valid[r] = false;
        }
    }
#pragma unroll
    for (int r = 0; r < E; r++) {
        lb[r] = 0;
        if (valid[r]) {
            lb[r] = pool_lower_bound(pool, psz, span, v[r]);
            if (lb[r] < psz && kmask(pool[lb[r]]) == v[r]) valid[r] = false;  // already in C
        }
        if (!valid[r]) v[r] = KEY_INF;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; r++)
        if (lane + 32 * r < s) newk[lane + 32 * r] = v[r];
    int m2 = 0;
#pragma unroll
    for (int r = 0; r < E; r++) m2 += __popc(__ballot_sync(0xffffffffu, valid[r]));
    __syncwarp();
    if (m2 == 0) return;
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
        if (valid[r]) {
            sk[rank[r]] = v[r];
            slb[rank[r]] = lb[r];
        }
    __syncwarp();
    const int lb0 = slb[0];
    for (int hi = psz; hi > lb0; hi -= 32) {
        const int p = hi - 32 + lane;
        const bool active = p >= lb0;
        uint64_t val = 0;
        int dest = L;
        if (active) {
            val = pool[p];
            int c = 0;
            if (m2 <= 8) {
                for (int r = 0; r < m2; r++) c += slb[r] <= p;
            } else {
                int lo = 0, h2 = m2;
                while (lo < h2) {
                    const int mid = (lo + h2) >> 1;
                    if (slb[mid] <= p) lo = mid + 1; else h2 = mid;
                }
                c = lo;
            }
            dest = p + c;
        }
        __syncwarp();
        if (active && dest < L) pool[dest] = val;
        __syncwarp();
    }
    for (int r = lane; r < m2; r += 32) {
        const int pos = slb[r] + r;
        if (pos < L) pool[pos] = sk[r];
    }
    __syncwarp();
    psz = min(L, psz + m2);
    hint = min(hint, lb0);
}

// Visited-set test-and-insert, u32 variant: open addressing, linear probing, full ids.
// Returns true if `id` was not known to be visited.
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

// Visited-set test-and-insert, u16 variant (half the shared memory, so more queries in
// flight).  Buckets of 8 u16 slots (one 16-byte LDS), two candidate buckets per id.
// An id is first mapped by a bijection h of [0, 2^id_bits) (odd multiply + xorshift);
// b1 = h mod NB, tag t = h / NB + 1 (<= 2^14), b2 = b1 ^ f(t).  A slot stores t plus a
// "choice" bit (0x8000 when the id sits in its alternate bucket), so (bucket, slot value)
// identifies exactly one id: a match is never a false positive.  A full pair of buckets
// forgets the id (miss), which the merge tolerates (see the file header).
__device__ __forceinline__ bool has16(const uint4 &x, uint32_t pat) {
    return (__vcmpeq2(x.x, pat) | __vcmpeq2(x.y, pat) | __vcmpeq2(x.z, pat) | __vcmpeq2(x.w, pat)) != 0u;
}
// Buckets fill strictly left to right (an insert always targets the first free slot, and
// a lost CAS re-reads), so the occupied slots are a prefix and the first free slot is the
// number of non-zero u16 entries.
__device__ __forceinline__ int fill16(const uint4 &x) {
    return (__popc(__vcmpne2(x.x, 0u)) + __popc(__vcmpne2(x.y, 0u)) + __popc(__vcmpne2(x.z, 0u)) +
            __popc(__vcmpne2(x.w, 0u))) >> 4;
}
__device__ __forceinline__ uint32_t word_sel(const uint4 &x, int w) {
    const uint32_t a = (w & 2) ? x.z : x.x, b = (w & 2) ? x.w : x.y;
    return (w & 1) ? b : a;
}
// Slots never empty again, so if b1 still has a free slot the id cannot have been placed in
// b2 (it would have gone to b1): the common lookup reads one bucket.  Inserts use a 32-bit
// CAS on the word holding the chosen 16-bit slot (retried if another lane won it).
__device__ __forceinline__ bool visit16(uint16_t *tab, int nb_log2, int id_bits, int id, int &miss) {
    const uint32_t imask = (id_bits >= 32) ? 0xffffffffu : ((1u << id_bits) - 1u);
    uint32_t h = ((uint32_t)id * 0x2545F491u) & imask;
    h ^= h >> ((id_bits + 1) >> 1);
    const uint32_t bmask = (1u << nb_log2) - 1u;
    const uint32_t b1 = h & bmask;
    const uint32_t t = (h >> nb_log2) + 1u;
    uint32_t *w1 = reinterpret_cast<uint32_t *>(tab + b1 * 8);
    for (int attempt = 0; attempt < 8; attempt++) {
        const uint4 x1 = *reinterpret_cast<const uint4 *>(w1);
        if (has16(x1, t * 0x10001u)) return false;
        int slot = fill16(x1);
        uint32_t *bw = w1;
        uint32_t ent = t;
        uint32_t old = word_sel(x1, slot >> 1);
        if (slot == 8) {
            const uint32_t b2 = b1 ^ (((t * 0x9E3779B1u) >> 11) & bmask);
            uint32_t *w2 = reinterpret_cast<uint32_t *>(tab + b2 * 8);
            const uint4 x2 = *reinterpret_cast<const uint4 *>(w2);
            ent = t | 0x8000u;
            if (has16(x2, ent * 0x10001u)) return false;
            slot = fill16(x2);
            if (slot == 8) break;
            bw = w2;
            old = word_sel(x2, slot >> 1);
        }
        const uint32_t nw = old | ((slot & 1) ? (ent << 16) : ent);
        if (atomicCAS(bw + (slot >> 1), old, nw) == old) return true;
    }
    miss++;
    return true;
}

__device__ __forceinline__ bool visit(uint8_t *tab, const KParams &p, int id, int &miss) {
    return p.tab16 ? visit16(reinterpret_cast<uint16_t *>(tab), p.nb_log2, p.id_bits, id, miss)
                   : visit32(reinterpret_cast<uint32_t *>(tab), p.h_log2, id, miss);
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
    int *newlb = reinterpret_cast<int *>(wbase + p.off_newlb);
    int *newid = reinterpret_cast<int *>(wbase + p.off_newid);
    int *newslot = reinterpret_cast<int *>(wbase + p.off_newslot);
    uint64_t *sk = reinterpret_cast<uint64_t *>(wbase + p.off_newid);  // aliases newid/newslot (dead by then)
    constexpr int G = 1 << GL;
    constexpr int npp = 32 >> GL;      // codes per gather pass
    const int gl = lane & (G - 1);     // lane within its code group
    const int gi = lane >> GL;         // code group index within the warp
    int span = 1;
    while (span < p.L) span <<= 1;

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
        // by seed_select_kernel; copy it into the pool
        int psz = p.init_psz[q], hint = 0;
        for (int t = lane; t < psz; t += 32) pool[t] = p.init_keys[(int64_t)q * p.L + t];
        __syncwarp();
        int miss = 0;
        for (int t = lane; t < psz; t += 32) visit(tab, p, key_id(pool[t]), miss);  // V <- ids(C) (R-10)
        __syncwarp();
        int n_lp = p.S, hops = 0;
        hint = 0;

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
                    if (bal2) next2 = kmask(k2);
                    break;
                }
            }
            if (sel < 0) break;
            const int node = key_id(pool[sel]);
            __syncwarp();
            if (lane == 0) pool[sel] |= KEY_FLAG;
            hint = sel + 1;
            if (p.t_expanded && lane == 0 && hops < p.max_hops) p.t_expanded[(int64_t)q * p.max_hops + hops] = node;
            hops++;

            // neighbour ids (lines 7-10: ids only, no vector data yet).  If the previous hop
            // predicted this node, its row is already in registers.
            int nb[E];
            bool isnew[E];
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
            const int miss0 = miss;
#pragma unroll
            for (int r = 0; r < E; r++) isnew[r] = nb[r] >= 0 && visit(tab, p, nb[r], miss);
            const bool hop_miss = __any_sync(0xffffffffu, miss != miss0);
            int m = 0;
#pragma unroll
            for (int r = 0; r < E; r++) {
                const uint32_t bal = __ballot_sync(0xffffffffu, isnew[r]);
                if (isnew[r]) {
                    const int rk = m + __popc(bal & lanemask_lt());
                    newid[rk] = nb[r];
                    newslot[rk] = p.layout == 0 ? nb[r] : lane + 32 * r;  // code index in cbase
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

            // lines 13-17: gather the unvisited codes, tau_l, keys.  A key that is not below
            // the current L-th key (pool full) cannot enter C and is dropped right here.
            const uint8_t *cbase = p.layout == 0 ? p.codes : p.rows + (int64_t)node * p.row_bytes + p.ids_bytes;
            const uint64_t worst = psz == p.L ? kmask(pool[p.L - 1]) : KEY_INF;
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
            merge_new<E>(ns, hop_miss, pool, psz, p.L, span, newk, sk, newlb, hint, lane);
        }

        // ---- trace
        const int rr = min(p.R, psz);
        {
            const int mtot = __reduce_add_sync(0xffffffffu, miss);
            if (lane == 0) {
                if (p.t_hops) p.t_hops[q] = hops;
                if (p.t_nlp) p.t_nlp[q] = n_lp;
                if (p.t_nhp) p.t_nhp[q] = rr;
                if (p.t_miss) p.t_miss[q] = mtot;
            }
            if (p.t_expanded)
                for (int t = hops + lane; t < p.max_hops; t += 32) p.t_expanded[(int64_t)q * p.max_hops + t] = -1;
            if (p.t_pool_ids || p.t_pool_tau)
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
        for (int c0 = 0; c0 < rr; c0 += 4) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            int idc[4];
#pragma unroll
            for (int u = 0; u < 4; u++) idc[u] = c0 + u < rr ? key_id(pool[c0 + u]) : -1;
            if (vec4) {
                const int nf4 = p.d >> 2;
                for (int f = lane; f < nf4; f += 32) {
                    const float4 qa = __ldg(reinterpret_cast<const float4 *>(qv) + f);
                    float4 xa[4];
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        xa[u] = idc[u] >= 0 ? __ldg(reinterpret_cast<const float4 *>(p.base + (int64_t)idc[u] * p.d) + f)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const float qs[4] = {qa.x, qa.y, qa.z, qa.w};
                        const float xs[4] = {xa[u].x, xa[u].y, xa[u].z, xa[u].w};
#pragma unroll
                        for (int t = 0; t < 4; t++) {
                            if (p.metric == VSAG_METRIC_L2) {
                                const double df = __dsub_rn((double)qs[t], (double)xs[t]);
                                acc[u] = __dadd_rn(acc[u], __dmul_rn(df, df));
                            } else {
                                acc[u] = __dadd_rn(acc[u], __dmul_rn((double)qs[t], (double)xs[t]));
                            }
                        }
                    }
                }
            } else {
                for (int j = lane; j < p.d; j += 32) {
                    const double qs = (double)__ldg(qv + j);
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (idc[u] < 0) continue;
                        const double xs = (double)__ldg(p.base + (int64_t)idc[u] * p.d + j);
                        if (p.metric == VSAG_METRIC_L2) {
                            const double df = __dsub_rn(qs, xs);
                            acc[u] = __dadd_rn(acc[u], __dmul_rn(df, df));
                        } else {
                            acc[u] = __dadd_rn(acc[u], __dmul_rn(qs, xs));
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
                const int cid = u == 0 ? idc[0] : (u == 1 ? idc[1] : (u == 2 ? idc[2] : idc[3]));
                if (lane < 4 && cid >= 0) {
                    const float th = __double2float_rn(p.metric == VSAG_METRIC_L2 ? sum : -sum);
                    rk[c0 + u] = ((uint64_t)ford(th) << 32) | (uint32_t)cid;
                }
            }
        }
        __syncwarp();
        // top-k of the R' (tau_h, id) keys: k rounds of a warp-wide argmin (keys are distinct)
        {
            uint64_t kv[RK_PER_LANE];
#pragma unroll
            for (int j = 0; j < RK_PER_LANE; j++) {
                const int t = lane + 32 * j;
                kv[j] = t < rr ? rk[t] : KEY_INF;
            }
            __syncwarp();
            const int kout = min(p.k, rr);
            for (int t = 0; t < kout; t++) {
                uint64_t mn = KEY_INF;
#pragma unroll
                for (int j = 0; j < RK_PER_LANE; j++) mn = min(mn, kv[j]);
                for (int j = RK_PER_LANE * 32 + lane; j < rr; j += 32) mn = min(mn, rk[j]);
                const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(mn >> 32));
                const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(mn >> 32) == hi ? (uint32_t)mn : 0xffffffffu);
                const uint64_t best = ((uint64_t)hi << 32) | lo;
#pragma unroll
                for (int j = 0; j < RK_PER_LANE; j++)
                    if (kv[j] == best) kv[j] = KEY_INF;
                for (int j = RK_PER_LANE * 32 + lane; j < rr; j += 32)
                    if (rk[j] == best) rk[j] = KEY_INF;
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
    return lcap * 8 + tab + NEW_CAP * 8 + NEW_CAP * 4 * 3;
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
    const size_t lcap = ((size_t)a.L + 31) / 32 * 32;
    int rk = 32;
    while (rk < a.rerank_n) rk <<= 1;
    size_t tab = (size_t)kp.tab_bytes;
    if ((size_t)rk * 8 > tab) tab = (size_t)rk * 8;
    kp.off_tab = (int)(lcap * 8);
    kp.off_newk = kp.off_tab + (int)tab;
    kp.off_newlb = kp.off_newk + NEW_CAP * 8;
    kp.off_newid = kp.off_newlb + NEW_CAP * 4;
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

}  // namespace vsag
