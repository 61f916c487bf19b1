// search_kernel.cuh -- rows a5 (pool init), a6 (hop loop), a7 (re-rank), a8 (output):
// the search kernel template.  Instantiated per tau_l mode in search_m*.cu (compiled in
// parallel); the host side (launch_search) is in search.cu.
//
// Deterministic Access Greedy Search (Alg. 1; App. A)
// for a batch of queries, one WARP per query, persistent grid (each warp pulls the
// next query from a global counter).  Per warp, shared memory holds:
//   pool   the candidate pool C as a sorted array of L = max(ef, R) u64 keys
//          key = (tau_l ^ 0x80000000) << 32 | id << 1 | x  (total order (tau_l, id),
//          R-8; x = "expanded" flag, below the id so it never reorders two nodes);
//          positions >= |C| hold KEY_INF;
//   tab    the visited set V: u16 tag buckets (or u32 linear probing for very large
//          n with a small table), reused as the re-rank scratch after the hop loop;
//   new*   the <= R new candidates of the current hop.
// One hop (lines 5-17):
//   select    first unexpanded key in the window [0, ef): the lowest bit of a register mask of
//             the current 32-entry pool block, or the smallest pending key (see the hop loop);
//   ids       the node's R neighbour ids (layout 0: adjacency table; layout 1: the id block
//             of the node's PRS row), usually already in the warp's shared-memory row
//             buffer: the previous hop predicted this node and started a cp.async copy of
//             its row (no register, nothing to spill, 94% of the hops);
//   filter    test-and-insert every id in V *before* touching any code -- the
//             paper's deterministic access: only unvisited neighbours
//             are gathered;
//   gather    each unvisited neighbour's code is read with 16-byte loads by a group
//             of G lanes (G = code bytes / 16 rounded up to a power of two), several
//             codes per warp instruction, several instructions in flight;
//   tau_l     VABSDIFF4 + IDP.4A (dist.cuh), int32, reduced over the G lanes;
//   keep      keys >= the pool's L-th key are dropped; the others are appended to the
//             pending buffer (lazy pool, see the hop loop), which is merged into the pool
//             when it could overflow: rank the keys, binary-search their pool positions,
//             rewrite the pool top-down in 32-entry blocks.
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
#pragma once
#include "search_common.cuh"

namespace vsag {
namespace {

constexpr uint32_t FULLMASK = 0xffffffffu;
#ifndef VSAG_UNR1
#define VSAG_UNR1 4  // gather passes in flight for one-chunk-per-lane codes (<= 64 B at 4 lanes): C4 at ef 32 +8% vs 2
#endif
#ifndef VSAG_UNR1G
#define VSAG_UNR1G 4  // the same in the generic variant
#endif
#ifndef VSAG_UNR2G
#define VSAG_UNR2G 2  // generic variant, SQ8 codes of two or four chunks per lane: gather passes in flight
#endif
#ifndef VSAG_MERGE_BSEARCH
#define VSAG_MERGE_BSEARCH 3  // merges of more new keys place them by per-lane binary search (tools/ab.sh: 3 beats 0, 6, 12)
#endif

// pool <- top_L(pool U new) (Alg. 1 line 17 for a whole batch of inserts: the result
// equals inserting them one by one).  Input: s candidate keys
// newk[0, s) (unsorted, each below the current L-th key when the pool is full).
// DEDUP (only once the visited cache has forgotten an id): drop keys that repeat an
// earlier new key or a node already in C.  Then every surviving key r gets its rank
// among the new keys and its pool lower bound lb_r (binary search), i.e. its final
// position pos_r = lb_r + rank_r.  The pool is rewritten top-down in 32-entry blocks
// from min(L, |C| + m2) - 1 down to the block of min pos_r: in a block the final
// positions holding new keys form a bitmask (OR-reduction of the lanes' pos_r), so
// final position f holds new key #k or old entry f - k, k = new keys before f.  Reads
// of a block happen before its writes and lower blocks only read below it.  Updates
// psz and the first-unexpanded hint.
template <int E, bool DEDUP>
__device__ __forceinline__ void merge_new(int s, uint64_t *pool, int &psz, int L, int span, uint64_t *newk,
                                          uint64_t *sk, int &hint, int lane, int *chk, int lcap, int nc) {
    uint64_t v[E];
    bool valid[E];
#pragma unroll
    for (int r = 0; r < E; r++) {
        const int e = lane + 32 * r;
        v[r] = e < s ? newk[e] : KEY_INF;
        valid[r] = e < s;
    }
    int m2 = s;
    int lb[E], pos[E];
#pragma unroll
    for (int r = 0; r < E; r++) lb[r] = 0;
    if (DEDUP || s > VSAG_MERGE_BSEARCH) {
        // per-lane binary search of each key's pool position, then ranks by counting
        if (DEDUP) {
            for (int i = 0; i < s; i++) {
                const uint64_t o = newk[i];
#pragma unroll
                for (int r = 0; r < E; r++)
                    if (o == v[r] && i < lane + 32 * r) valid[r] = false;
            }
        }
#pragma unroll
        for (int r = 0; r < E; r++) {
            if (valid[r]) {
                lb[r] = pool_lower_bound(pool, psz, span, v[r]);
                if (DEDUP && lb[r] < psz && kmask(pool[lb[r]]) == v[r]) valid[r] = false;  // already in C
            }
            if (DEDUP && !valid[r]) v[r] = KEY_INF;
        }
        if (DEDUP) {
            __syncwarp();
#pragma unroll
            for (int r = 0; r < E; r++)
                if (lane + 32 * r < s) newk[lane + 32 * r] = v[r];
            m2 = 0;
#pragma unroll
            for (int r = 0; r < E; r++) m2 += __popc(__ballot_sync(FULLMASK, valid[r]));
            __syncwarp();
            if (m2 == 0) return;
        }
#pragma unroll
        for (int r = 0; r < E; r++) pos[r] = lb[r];
#pragma unroll 4
        for (int i = 0; i < s; i++) {
            const uint64_t o = newk[i];
#pragma unroll
            for (int r = 0; r < E; r++) pos[r] += o < v[r];
        }
    } else {
        // few keys: the whole warp places one key at a time.  Lane l holds the pivot
        // pool[(l + 1) * st - 1] (st = pool entries per lane-block); one ballot finds the
        // block of the key, a second one (lanes < st) its position inside the block; the
        // same loop counts each lane's key rank among the new keys.
        const int st = (psz + 31) >> 5;
        const int pe = min((lane + 1) * st, psz) - 1;
        const uint64_t pv = pool[max(pe, 0)];  // unpredicated load (pe >= 0 whenever it is used)
        const uint64_t piv = lane * st < psz ? pv : KEY_INF;
#pragma unroll
        for (int r = 0; r < E; r++) pos[r] = 0;
        for (int j = 0; j < s; j++) {
            const uint64_t vj = newk[j];
#pragma unroll
            for (int r = 0; r < E; r++) pos[r] += vj < v[r];
            const int blk = __popc(__ballot_sync(FULLMASK, piv < vj));  // blocks entirely below vj
            const int f = blk * st + lane;
            const uint64_t pf = pool[min(f, psz - 1)];  // unpredicated load
            const bool below = lane < st && f < psz && pf < vj;
            const int lbj = min(blk * st, psz) + __popc(__ballot_sync(FULLMASK, below));
#pragma unroll
            for (int r = 0; r < E; r++)
                if (lane + 32 * r == j) lb[r] = lbj;
        }
#pragma unroll
        for (int r = 0; r < E; r++) pos[r] += lb[r];
    }
    __syncwarp();  // sk aliases newk
    int pmin = 0x7fffffff, pmax = -1;
#pragma unroll
    for (int r = 0; r < E; r++) {
        if (valid[r]) {
            VCHK(chk, pos[r] - lb[r] >= 0 && pos[r] - lb[r] < nc, 16);
            sk[pos[r] - lb[r]] = v[r];
            pmin = min(pmin, pos[r]);
            pmax = max(pmax, pos[r]);
        } else {
            pos[r] = 0x7fffffff;
        }
    }
    pmin = __reduce_min_sync(FULLMASK, pmin);
    pmax = __reduce_max_sync(FULLMASK, pmax);
    __syncwarp();
    const int total = min(L, psz + m2);
    VCHK(chk, total <= lcap && m2 <= nc, 16);
    // One __syncwarp per block orders its reads before its writes; a lower block only
    // reads below the blocks already written, and its own barrier orders those reads
    // after every lane's reads of the block above.
    int fb = (total - 1) & ~31;
    STAT(7, ((total - 1) >> 5) - (pmin >> 5) + 1);
    STAT(9, pmin);
    STAT(10, pmax);
    for (; fb > (pmax | 31); fb -= 32) {  // no new key at or above this block: a plain shift by m2
        const int f = fb + lane;
        const uint64_t val = f < total ? pool[f - m2] : 0;
        __syncwarp();
        if (f < total) pool[f] = val;
    }
    for (; fb >= (pmin & ~31); fb -= 32) {
        uint32_t bits = 0, below = 0;
#pragma unroll
        for (int r = 0; r < E; r++) {
            const uint32_t d = (uint32_t)(pos[r] - fb);
            if (d < 32u) bits |= 1u << d;
            below += pos[r] < fb;
        }
        const uint32_t mask = __reduce_or_sync(FULLMASK, bits);
        const int k = (int)__reduce_add_sync(FULLMASK, below) + __popc(mask & ((1u << lane) - 1u));
        const int f = fb + lane;
        // one load from either sk[k] (a new key lands here) or pool[f - k] (old entry)
        VCHK(chk, f >= total || (((mask >> lane) & 1u) ? (k >= 0 && k < nc) : (f - k >= 0 && f - k < lcap)), 16);
        const uint64_t *src = ((mask >> lane) & 1u) ? sk + k : pool + (f - k);
        const uint64_t val = f < total ? *src : 0;
        __syncwarp();
        if (f < total) pool[f] = val;
    }
    __syncwarp();
    psz = total;
    hint = min(hint, pmin);
}

// VAR 0: generic (visited-table kind, row de-duplication, expansion trace and the code
// chunk count are read at run time); VAR 1 / 2: the common case fixed at compile time
// (degree 32, u16 visited table, rows without repeated ids, codes filling all G * CPL chunks),
// without any trace output / with the trace outputs; VAR 3: the same common case with the u32
// visited table (indexes too large for 14-bit tags, e.g. C4's 10M rows), trace outputs
// checked at run time.  Same arithmetic, same results.
// BIG (generic variant only): compiled for 128 registers (16 warps per SM) instead of 56, for
// batches small enough to reside at once anyway (nq <= 16 warps x SMs, e.g. C2's 1,000 queries):
// nothing spills and SQ4 long codes also keep two gather passes in flight (C2: search -13 to -21%).
template <int M, int CPL, int GL, int E, int LAYOUT, int VAR, int BIG = 0>
#ifndef VSAG_SEARCH_MINB
#define VSAG_SEARCH_MINB 9  // 56 registers: 36 warps per SM (tools/ab.sh)
#endif
__global__ void __launch_bounds__(128, BIG ? 4 : VSAG_SEARCH_MINB) search_kernel(const KParams p) {
    constexpr bool FAST = VAR != 0;
    constexpr int OPW = mode_sq4(M) ? 2 : 1;
    constexpr int DPW = mode_sq4(M) ? 8 : 4;  // dimensions per code word
    constexpr int QW = 4 * OPW;  // operand words per 16-byte code chunk
    // gather passes issued back to back: long SQ8 codes of the generic variant keep two passes in
    // flight (C3: 10-19% faster; the SQ4 operand needs twice the registers and spills under the
    // 56-register cap: C2 1-17% slower, so SQ4 does it only in the 128-register BIG variant)
    constexpr int UNR = CPL >= 2 ? ((FAST || (mode_sq4(M) && !BIG)) ? 1 : VSAG_UNR2G) : (FAST ? VSAG_UNR1 : VSAG_UNR1G);
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const uint32_t ltm = (1u << lane) - 1u;  // lanes below this one
    uint8_t *wbase = smem + (mode_w(M) ? p.off_cta : 0) + (threadIdx.x >> 5) * p.smem_per_warp;
    const int32_t *wsm = reinterpret_cast<const int32_t *>(smem);  // weighted L2 weights (CTA-shared)
    if (mode_w(M)) {
        for (int i = threadIdx.x; i < p.l2w_dims; i += blockDim.x) reinterpret_cast<int32_t *>(smem)[i] = p.l2w[i];
        __syncthreads();
    }
    // (the common case, degree 32 and the table layout: newk at 0, newid at 256, row at 384, pool at 512)
    uint64_t *pool = reinterpret_cast<uint64_t *>(wbase + (FAST ? 512 : p.off_pool));
    uint8_t *tab = wbase + p.off_tab;
    uint64_t *newk = reinterpret_cast<uint64_t *>(wbase + (FAST ? 0 : p.off_newk));
    // (the common case has degree 32: newid follows the 32 new-key slots)
    int *newid = FAST ? reinterpret_cast<int *>(newk + 32) : reinterpret_cast<int *>(wbase + p.off_newid);
    // code index in cbase: the id for the global table, the row slot for layout 1 / PRS blocks
    int *newslot = (LAYOUT == 0 && (FAST || !p.prs_blk)) ? newid : reinterpret_cast<int *>(wbase + p.off_newslot);
    uint64_t *sk = newk;  // the merge's sorted new keys overwrite newk once it has been read
    // predicted next id row (cp.async target; follows newid)
    const int *rowbuf = FAST ? reinterpret_cast<const int *>(newk + 32) + 32 : reinterpret_cast<const int *>(wbase + p.off_row);
    const uint32_t rowbuf_s = (uint32_t)__cvta_generic_to_shared(rowbuf);
    constexpr int G = 1 << GL;
    constexpr int npp = 32 >> GL;      // codes per gather pass
    const int gl = lane & (G - 1);     // lane within its code group
    const int gi = lane >> GL;         // code group index within the warp
    int span = 1;
    while (span < p.L) span <<= 1;
    uint16_t *tab16 = reinterpret_cast<uint16_t *>(tab);
    uint32_t *tab32 = reinterpret_cast<uint32_t *>(tab);
    const Tab16 tb(p.nb_log2, p.id_bits);
    const bool use16 = FAST ? VAR != 3 : p.tab16 != 0;
    const bool usebits = !FAST && p.vkind == 4;
    uint32_t *gbits = usebits ? p.gvis + (int64_t)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * p.gvis_words
                              : nullptr;
    const bool row_dups = !FAST && p.row_dups != 0;
    const bool wide = p.wide != 0;  // code rows 32-byte aligned (32-byte loads)
    // Chunk mm of this lane.  Generic variant: a lane owns CPL adjacent 16-byte chunks of a code, read
    // with one 32-byte load per pair (LDG.E.256; both chunks in one request -- two 16-byte loads 512
    // bytes apart were issued one after the other's use under register pressure: C3 / C2 17-21%
    // faster).  Common case (C1's 128-byte codes, 4 lanes): chunks gl and gl + G, two 16-byte loads
    // of 64 contiguous bytes per code each (the 32-byte form measured 0.4% slower there).
    constexpr bool ADJ = !FAST && CPL >= 2;
    auto chunk_of = [&](int mm) { return ADJ ? CPL * gl + mm : gl + G * mm; };
    const bool trace_exp = (FAST && VAR != 3) ? VAR == 2 : p.t_expanded != nullptr;
    // the common case fixes these at compile time: degree 32, codes filling all G * CPL chunks
    const int degree = FAST ? 32 : p.degree, chunks = FAST ? G * CPL : p.chunks, cbp = FAST ? G * CPL * 16 : p.cbp;
    // id row / code base of a node: layout 0 (delta = 0) uses the global adjacency and
    // code tables; layout 1 (PRS, delta = 1) the node's own row [ids | neighbour codes]
    auto id_row = [&](int node) -> const int32_t * {
        // (opaque: otherwise the shift that extracts the id from a key is folded into a 64-bit
        // shift / mask / add sequence of 7 instructions instead of one wide multiply-add)
        asm("" : "+r"(node));
        if (LAYOUT == 0)  // one IMAD.WIDE.U32 (byte offset)
            return reinterpret_cast<const int32_t *>(reinterpret_cast<const uint8_t *>(p.adj) +
                                                     (uint64_t)(uint32_t)node * (uint32_t)(FAST ? 128 : degree * 4));
        return reinterpret_cast<const int32_t *>(p.rows + (uint64_t)(uint32_t)node * (uint32_t)p.row_bytes);
    };

    for (;;) {
        int q = 0;
        if (lane == 0) q = (int)atomicAdd(p.counter, 1u);
        q = __shfl_sync(FULLMASK, q, 0);
        if (q >= p.nq) break;

        // ---- query operand chunks into registers (a4 output)
        uint32_t qr[CPL][QW];
        const uint32_t *opq = p.op + (int64_t)q * p.op_stride;
#pragma unroll
        for (int mm = 0; mm < CPL; mm++) {
            const int c = chunk_of(mm);
#pragma unroll
            for (int t = 0; t < QW; t += 4) {
                uint4 w = make_uint4(0, 0, 0, 0);
                if (FAST || c < chunks) w = *reinterpret_cast<const uint4 *>(opq + c * QW + t);
                qr[mm][t] = w.x;
                qr[mm][t + 1] = w.y;
                qr[mm][t + 2] = w.z;
                qr[mm][t + 3] = w.w;
            }
        }
        // ---- clear V
        if (usebits) {
            for (int64_t i = lane * 4; i < p.gvis_words; i += 128)
                *reinterpret_cast<uint4 *>(gbits + i) = make_uint4(0, 0, 0, 0);
        } else {
            const uint32_t fill = use16 ? 0u : EMPTY;
            for (int i = lane * 16; i < p.tab_bytes; i += 512)
                *reinterpret_cast<uint4 *>(tab + i) = make_uint4(fill, fill, fill, fill);
        }
        __syncwarp();  // (also orders the bitset's clearing stores before the warp's atomics)

        // ---- a5: C <- top_L of the entry set by (tau_l, id)  (Alg. 1 line 3), selected
        // by seed_select_kernel; copy it into the pool (positions >= psz hold KEY_INF)
        int psz = p.init_psz[q];
        for (int t = lane; t < p.lcap; t += 32) pool[t] = t < psz ? p.init_keys[(int64_t)q * p.L + t] : KEY_INF;
        __syncwarp();
        int miss = 0;
        // V <- ids(C) (R-10)
        for (int t0 = 0; t0 < psz; t0 += 32) {
            const int t = t0 + lane;
            const int id = t < psz ? key_id(pool[t]) : -1;
            if (use16) visit16_round(tab16, tb, id, miss, 0xffffffffu, p.check);
            else if (usebits) { if (id >= 0) visit_bits(gbits, id); }
            else if (id >= 0) visit32(tab32, p.h_log2, id, miss);
        }
        __syncwarp();
        int n_lp = p.S, hops = 0;
        // window, pool capacity and re-rank count of this query (QLP may shrink them)
        int ef = p.ef, L = p.L, R = p.R;
        bool qlp_pending = !FAST && p.qlp_ef_low > 0;

        // ---- a6: hop loop (Alg. 1 lines 4-17)
        // Lazy pool: the new keys of a hop are not merged at once; they stay in newk
        // ("pending", unsorted, pcnt of them, pexp of them expanded and flagged) until the
        // buffer could overflow, and the pool proper [0, psz) stays as it was after the last
        // merge.  C of Alg. 1 is top_L(pool U pending); the next expansion is the smallest
        // unexpanded key of C inside the window, i.e. the smaller of the pool's first
        // unexpanded entry and the smallest unexpanded pending key pmink:
        //  - every expanded pending key was, when it was chosen, below every unexpanded key,
        //    and the pool has not changed since, so all pexp of them precede the pool's
        //    candidate: its rank in C is sel + pexp (the scan stops at ef - pexp);
        //  - pmink's rank is its pool lower bound plus the expanded pending keys below it.
        // Pending keys were below the pool's L-th key when they were added (a bound that is
        // only stale, never too tight), and the merge cuts C back to L entries.
        int pcnt = 0, pexp = 0;
        uint64_t pmink = KEY_INF;
        const bool lazy = !qlp_pending;  // (QLP reads the pool at its checkpoint: merge every hop)
        // Unexpanded-entry mask of the block pool[wb, wb + 32): bit i of um is set when entry
        // wb + i exists and has not been expanded.  Every entry below wb is expanded.  um is read
        // from the keys' flag bits when the block changes or the pool has been merged and lives
        // in a register in between; em collects the entries expanded meanwhile, whose flag bits
        // are written to the pool before a merge or a block change reads them.
        int wb = 0;
        uint32_t um = 0, em = 0;
        // (um is clipped to the window [0, min(ef - pexp, psz)) when it is loaded and when pexp grows)
        auto load_mask = [&](int base) {
            wb = base;
            // (reads up to 31 entries past the pool's capacity: the warp's visited table / re-rank
            // scratch follows it; such lanes fail the window test)
            const uint32_t lo = reinterpret_cast<const uint32_t *>(pool)[2 * (base + lane)];
            um = __ballot_sync(FULLMASK, base + lane < min(ef - pexp, psz) && !(lo & 1u));
            em = 0;
        };
        auto store_flags = [&]() {
            if ((em >> lane) & 1u) reinterpret_cast<uint32_t *>(pool)[2 * (wb + lane)] |= 1u;
            em = 0;
            __syncwarp();
        };
        // lowest pool position that may hold an unexpanded entry
        auto first_open = [&]() { return um ? wb + __ffs(um) - 1 : max(wb, min(wb + 32, min(ef - pexp, psz))); };
        // pool <- top_L(pool U newk[0, s)): all pending keys go in; the mask is reloaded from the
        // lowest position that may hold an unexpanded entry afterwards
        auto merge_pending = [&](int s, bool dedup) {
            int hint = first_open();
            store_flags();
            if (dedup) merge_new<E, true>(s, pool, psz, L, span, newk, sk, hint, lane, p.check, p.lcap, 32 * E);
            else merge_new<E, false>(s, pool, psz, L, span, newk, sk, hint, lane, p.check, p.lcap, 32 * E);
            pcnt = 0;
            pexp = 0;
            pmink = KEY_INF;
            load_mask(hint);
        };
        load_mask(0);
        int pred_node = -1;  // node whose id row the row buffer holds (or is being copied into it)
        // the smaller of two keys by tau alone: enough for a prefetch hint
        auto hint_min = [](uint64_t a, uint64_t b) { return (uint32_t)(a >> 32) < (uint32_t)(b >> 32) ? a : b; };
        // Start copying the id row of the likeliest next expansion (key pk, KEY_INF: none) into the
        // warp's row buffer: cp.async needs no register and nothing waits for it until the next
        // hop has selected its node.  (Round 1 loaded the row into a register that the 56-register
        // cap spilled, so the spill store waited for the load: 10% of all stall samples.)
        auto predict = [&](uint64_t pk) {
            pred_node = -1;
            if ((uint32_t)(pk >> 32) != 0xffffffffu) {  // (a key's high word is tau ^ 2^31 < 2^32 - 1, R-20)
                pred_node = key_id(pk);
                const int32_t *ids2 = id_row(pred_node);
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int t = lane + 32 * r;
                    if (FAST || t < degree)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(rowbuf_s + 4 * t), "l"(ids2 + t) : "memory");
                }
            }
        };
        for (;;) {
            if (!FAST && qlp_pending && hops == p.qlp_hop) {
                // NEXT-4b (R-28, §4.3): one checkpoint, a stump on an integer feature
                // of the (exact) pool: 1 = sum of the 5 best tau_l, 2 = tau_l(k-th) - tau_l(best);
                // every lane reads the same entries, so the decision is warp-uniform
                qlp_pending = false;
                long long f = 0;
                bool have;
                if (p.qlp_feature == 1) {
                    have = psz >= 5;
                    for (int t = 0; have && t < 5; t++) f += key_tau(pool[t]);
                } else {
                    have = psz >= p.k;
                    if (have) f = (long long)key_tau(pool[p.k - 1]) - key_tau(pool[0]);
                }
                if (have && f <= p.qlp_threshold) {  // shrink: the farthest entries are evicted
                    ef = p.qlp_ef_low;
                    L = p.qlp_ef_low;
                    R = min(R, p.qlp_ef_low);
                    const int open = first_open();
                    store_flags();
                    psz = min(psz, L);
                    load_mask(min(open, psz));
                }
            }
            // first unexpanded pool entry inside the window: the lowest bit of the mask; an
            // exhausted block hands over to the next one
            while (um == 0 && min(ef - pexp, psz) - wb > 32) {
                store_flags();
                load_mask(wb + 32);
            }
            uint64_t next2 = KEY_INF;  // the pool's next unexpanded entry after this hop's choice
            int node = -1;
            bool from_pool = false;
            if (um) {
                const int src = __ffs(um) - 1;
                const uint64_t ks = pool[wb + src];
                VCHK(p.check, wb + src < p.lcap, 4);
                if (pmink < ks) {  // a pending key goes first; the pool's candidate stays
                    next2 = ks;
                } else {
                    from_pool = true;
                    node = key_id(ks);
                    um &= um - 1;
                    em |= 1u << src;
                    if (um) next2 = pool[wb + __ffs(um) - 1];
                }
            }
            if (!from_pool) {
                if (pmink == KEY_INF) break;
                // expand the pending key pmink if it lies inside the window: its rank in C is
                // (pool entries below it) + (expanded pending keys below it)
                uint64_t pk[E];
                int cnt = 0;
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int t = lane + 32 * r;
                    pk[r] = t < pcnt ? newk[t] : KEY_INF;
                    cnt += __popc(__ballot_sync(FULLMASK, (pk[r] & KEY_FLAG) && pk[r] < pmink));
                }
                const int wpos = ef - cnt - 1;
                if (wpos < 0 || (wpos < psz && !(pmink < pool[wpos]))) break;  // outside: nothing left in the window
                node = key_id(pmink);
                uint64_t mn = KEY_INF;
#pragma unroll
                for (int r = 0; r < E; r++) {
                    if (pk[r] == pmink) reinterpret_cast<uint32_t *>(newk)[2 * (lane + 32 * r)] = (uint32_t)pk[r] | 1u;
                    else if (!(pk[r] & KEY_FLAG)) mn = min(mn, pk[r]);
                }
                const uint32_t hi = __reduce_min_sync(FULLMASK, (uint32_t)(mn >> 32));
                const uint32_t lo = __reduce_min_sync(FULLMASK, (uint32_t)(mn >> 32) == hi ? (uint32_t)mn : 0xffffffffu);
                pmink = ((uint64_t)hi << 32) | lo;
                pexp++;
                {  // the window shrank by one entry
                    const int room = min(ef - pexp, psz) - wb;
                    if (room < 32) um = room > 0 ? um & ((1u << room) - 1u) : 0u;
                }
                STAT(11, 1);
                __syncwarp();
            }
            VCHK(p.check, node >= 0 && node < p.n_base, 4);
            if (lane == 0 && trace_exp && hops < p.max_hops) p.t_expanded[(int64_t)q * p.max_hops + hops] = node;
            hops++;
            STAT(0, 1);

            // neighbour ids (lines 7-10: ids only, no vector data yet).  If the previous hop
            // predicted this node, its row is in the row buffer (every lane reads back the words
            // it copied itself: no warp barrier needed).
            int nb[E];
            asm volatile("cp.async.wait_all;" ::: "memory");  // (the buffer is rewritten at the end of this hop)
#pragma unroll
            for (int r = 0; r < E; r++) {
                const int t = lane + 32 * r;
                nb[r] = (FAST || t < degree) ? rowbuf[t] : -1;
            }
            if (node != pred_node) {  // mispredicted (6% of the hops): load the row now
                const int32_t *ids = id_row(node);
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int t = lane + 32 * r;
                    nb[r] = t < degree ? __ldg(ids + t) : -1;
                }
            }
            // edge filter of Alg. 1 line 8 (NEXT-2, R-23): label <= alpha_s, then the first m_s
            // label-valid edges of the row (in row order, visited or not)
            if (!FAST && p.filt) {
                int kept = 0;
#pragma unroll
                for (int r = 0; r < E; r++) {
                    const int t = lane + 32 * r;
                    bool ok = nb[r] >= 0;
                    if (ok && p.labels) ok = p.labels[(int64_t)node * degree + t] <= p.alpha_s;
                    const uint32_t bal = __ballot_sync(FULLMASK, ok);
                    if (!ok || (p.m_s > 0 && kept + __popc(bal & ltm) >= p.m_s)) nb[r] = -1;
                    kept += __popc(bal);
                }
            }
            // PRS (NEXT-4): a node with a co-located block reads its neighbours' codes there
            const int blk = (LAYOUT == 0 && !FAST && p.prs_blk) ? __ldg(p.prs_blk + node) : -1;
            // visited filter, one 32-id slice at a time (a later slice sees the earlier one's
            // inserts); rows that repeat an id keep only its first lane per slice
            int m = 0;
#pragma unroll
            for (int r = 0; r < E; r++) {
                int id = nb[r];
                if (row_dups) {
                    const uint32_t mm = __match_any_sync(FULLMASK, id);
                    if (mm & ltm) id = -1;
                }
                bool isnew;
                if (use16) {
                    isnew = visit16_round(tab16, tb, id, miss, 0xffffffffu, p.check);
                } else if (usebits) {
                    isnew = id >= 0 && visit_bits(gbits, id);
                } else {
                    isnew = id >= 0 && visit32(tab32, p.h_log2, id, miss);
                    __syncwarp();
                }
                const uint32_t bal = __ballot_sync(FULLMASK, isnew);
                if (isnew) {
                    const int rk = m + __popc(bal & ltm);
                    VCHK(p.check, rk < 32 * E && id >= 0 && id < p.n_base, 2);
                    newid[rk] = id;
                    // code index: the slot in the node's row (layout 1 / PRS block) or the id
                    if (!(LAYOUT == 0 && FAST)) newslot[rk] = (LAYOUT != 0 || blk >= 0) ? lane + 32 * r : id;
                }
                m += __popc(bal);
            }
            __syncwarp();
            if (m == 0) {  // nothing new: the next expansion is the window's next entry (or pending key)
                predict(hint_min(pmink, next2));
                continue;
            }
            n_lp += m;
            STAT(2, m);
            STAT(3, 1);

            // lines 13-17: gather the unvisited codes, tau_l, keys.  A key that is not below
            // the current L-th key (pool full) cannot enter C and is dropped right here.
            const uint8_t *cbase = LAYOUT != 0 ? p.rows + (int64_t)node * p.row_bytes + p.ids_bytes
                                   : (blk >= 0 ? p.prs_codes + (int64_t)blk * degree * cbp : p.codes);
            // the pending keys are merged first when this hop's candidates may not fit behind
            // them, or when V has just forgotten an id (from here on every hop merges at once
            // with the de-duplicating merge, which expects unflagged new keys)
            const bool forgot = __any_sync(FULLMASK, miss != 0);
            if (pcnt > 0 && (pcnt + m > 32 * E || forgot)) {
                STAT(5, 1);
                STAT(4, pcnt);
                merge_pending(pcnt, false);
            }
            const uint64_t worst = psz == L ? pool[L - 1] : KEY_INF;
            const uint8_t *cb2 = cbase + gl * 16;  // this lane's first chunk of code 0 (common case)
            // (the common case keeps it as one 64-bit addend of the wide multiply-add below)
            if (FAST) asm("" : "+l"(cb2));
            int ns = pcnt;
            uint64_t kbest = KEY_INF;
            for (int b0 = 0; b0 < m; b0 += npp * UNR) {
                uint4 cv[UNR][CPL];
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    // groups past the last new id re-read the last code (same sectors as its
                    // own group, no extra traffic) instead of predicating the loads
                    const int idc = min(b0 + u * npp + gi, m - 1);
                    VCHK(p.check, idc >= 0 && idc < 32 * E, 2);
                    VCHK(p.check, (LAYOUT != 0 || blk >= 0) ? (newslot[idc] >= 0 && newslot[idc] < p.degree)
                                                            : (newslot[idc] >= 0 && newslot[idc] < p.n_base), 4);
                    const uint8_t *cp = FAST ? cb2 + (uint64_t)(uint32_t)newslot[idc] * (uint32_t)cbp
                                             : cbase + (uint64_t)(uint32_t)newslot[idc] * (uint32_t)cbp +
                                                   gl * (ADJ ? 16 * CPL : 16);
                    if (!ADJ) {
#pragma unroll
                        for (int mm = 0; mm < CPL; mm++)
                            cv[u][mm] = (FAST || chunk_of(mm) < chunks) ? ldg16(cp + G * 16 * mm) : make_uint4(0, 0, 0, 0);
                    } else if (wide) {
#pragma unroll
                        for (int mm = 0; mm < CPL; mm += 2)
                            ldg32(cp + 16 * mm, chunk_of(mm) < chunks, cv[u][mm], cv[u][mm + 1]);
                    } else {
#pragma unroll
                        for (int mm = 0; mm < CPL; mm += 2)
                            ldg16x2(cp + 16 * mm, 16, chunk_of(mm) < chunks, chunk_of(mm + 1) < chunks, cv[u][mm],
                                    cv[u][mm + 1]);
                    }
                }
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    int acc = 0;
#pragma unroll
                    for (int mm = 0; mm < CPL; mm++) {
                        const uint32_t c4[4] = {cv[u][mm].x, cv[u][mm].y, cv[u][mm].z, cv[u][mm].w};
#pragma unroll
                        for (int w = 0; w < 4; w++) {
                            if (mode_w(M))
                                acc = word_dist_w<M>(acc, qr[mm][w * OPW], OPW == 2 ? qr[mm][w * OPW + 1] : 0u, c4[w],
                                                     wsm + (chunk_of(mm) * 4 + w) * DPW);
                            else
                                acc = word_dist<M>(acc, qr[mm][w * OPW], OPW == 2 ? qr[mm][w * OPW + 1] : 0u, c4[w]);
                        }
                    }
#pragma unroll
                    for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, o);
                    const int idx = b0 + u * npp + gi;
                    const uint64_t key = make_key(finish_tau<M>(acc), newid[min(idx, m - 1)]);
                    const bool ok = gl == 0 && idx < m && key < worst;
                    const uint32_t bal = __ballot_sync(FULLMASK, ok);
                    const int at = ns + __popc(bal & ltm);
                    VCHK(p.check, !ok || at < 32 * E, 2);
                    if (ok) newk[at] = key;  // (predicated store, no branch)
                    kbest = ok && key < kbest ? key : kbest;
                    ns += __popc(bal);
                }
            }
            __syncwarp();
            // The next expansion is the smallest of the window's next unexpanded entry, the
            // pending keys and the best surviving new key (when it lands inside the window);
            // start loading that node's id row now so the load overlaps the merge / the select.
            {
                uint64_t kb = kbest;  // this lane's best surviving new key
                const uint32_t hi = __reduce_min_sync(FULLMASK, (uint32_t)(kb >> 32));
                const uint32_t lo = __reduce_min_sync(FULLMASK, (uint32_t)(kb >> 32) == hi ? (uint32_t)kb : 0xffffffffu);
                kb = ((uint64_t)hi << 32) | lo;
                kb = pmink = min(pmink, kb);
                predict(hint_min(kb, next2));
            }
            pcnt = ns;
            if ((!lazy || forgot) && pcnt > 0) {  // immediate merge (QLP reads the pool; forgetful V)
                STAT(5, 1);
                STAT(4, pcnt);
                merge_pending(pcnt, forgot);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (pcnt > 0) merge_pending(pcnt, false);  // C = top_L(pool U pending) for the re-rank and the trace

        // ---- trace, a7 re-rank, a8 output
        finish_query<M, VAR != 1>(p, R, q, pool, psz, tab, hops, n_lp, __reduce_add_sync(FULLMASK, miss), lane);
    }
}

template <int M, int CPL, int GL, int E, int LAYOUT, int VAR>
cudaError_t launch_typed(const KParams &kp, int wpb, cudaStream_t s, SearchLaunch *info, int64_t nq) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void (*kern)(const KParams) = search_kernel<M, CPL, GL, E, LAYOUT, VAR, 0>;
    if constexpr (VAR == 0) {  // a batch that 16 warps per SM hold at once: the 128-register build
        if (nq <= (int64_t)16 * sms) kern = search_kernel<M, CPL, GL, E, LAYOUT, VAR, 1>;
    }
    const size_t smem = (size_t)kp.off_cta + (size_t)wpb * kp.smem_per_warp;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
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
    KParams kq = kp;
    if (kp.vkind == 4) {  // one exact bitset per resident warp (stream-ordered scratch)
        e = scratch_alloc(reinterpret_cast<void **>(&kq.gvis), (size_t)blocks * wpb * kp.gvis_words * 4, dev, s);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)blocks, wpb * 32, smem, s>>>(kq);
    e = cudaGetLastError();
    if (kq.gvis) cudaFreeAsync(kq.gvis, s);
    return e;
}

// Code-group shapes: G = 2^GL lanes read one code (16 B each); CPL 16-byte chunks per lane.
template <int M, int E, int LAYOUT, int VAR>
cudaError_t launch_shape(int cpl, int gl, const KParams &kp, int wpb, cudaStream_t s, SearchLaunch *info,
                         int64_t nq) {
    if (cpl == 1) {
        switch (gl) {
            case 2: return launch_typed<M, 1, 2, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            case 3: return launch_typed<M, 1, 3, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            case 4: return launch_typed<M, 1, 4, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            default: return launch_typed<M, 1, 5, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
        }
    }
    if (cpl == 2) {
        switch (gl) {
            case 2: return launch_typed<M, 2, 2, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            case 3: return launch_typed<M, 2, 3, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            case 4: return launch_typed<M, 2, 4, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
            default: return launch_typed<M, 2, 5, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
        }
    }
    return launch_typed<M, 4, 5, E, LAYOUT, VAR>(kp, wpb, s, info, nq);
}

}  // namespace

// One tau_l mode's instantiations (search_m<M>.cu).
template <int M>
cudaError_t launch_search_mode(int cpl, int gl, int e, int layout, int var, const KParams &kp, int wpb, cudaStream_t s,
                               SearchLaunch *info, int64_t nq) {
    if (var == 1) return launch_shape<M, 1, 0, 1>(cpl, gl, kp, wpb, s, info, nq);
    if (var == 2) return launch_shape<M, 1, 0, 2>(cpl, gl, kp, wpb, s, info, nq);
    if (var == 3) return launch_shape<M, 1, 0, 3>(cpl, gl, kp, wpb, s, info, nq);
    if (e == 1) return layout == 0 ? launch_shape<M, 1, 0, 0>(cpl, gl, kp, wpb, s, info, nq)
                                   : launch_shape<M, 1, 1, 0>(cpl, gl, kp, wpb, s, info, nq);
    return layout == 0 ? launch_shape<M, 2, 0, 0>(cpl, gl, kp, wpb, s, info, nq)
                       : launch_shape<M, 2, 1, 0>(cpl, gl, kp, wpb, s, info, nq);
}

}  // namespace vsag
