// search.cu -- host side of rows a5-a8: kernel parameters, shared-memory layout and the
// choice of the search kernel instantiation (search_kernel.cuh; instantiated per tau_l
// mode in search_m0.cu .. search_m3.cu so they compile in parallel).
#include <algorithm>
#include <cstdint>

#include "search_common.cuh"

namespace vsag {

template <int M>
cudaError_t launch_search_mode(int cpl, int gl, int e, int layout, int var, const KParams &kp, int wpb, cudaStream_t s,
                               SearchLaunch *info, int64_t nq);

namespace {

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
// Layout of one warp's shared memory: pool [lcap] u64 | tab (visited set, >= the re-rank
// scratch) | newk [nc] u64 | newid [nc] i32 | row [nc] i32 | newslot [nc] i32 (layout 1 only);
// nc = 32 * ceil(degree / 32) new ids per hop.
struct WarpSmem {
    int off_pool, off_tab, off_newk, off_newid, off_newslot, off_row, bytes;
};
WarpSmem warp_smem(int L, int R, int H, int vkind, int degree, int layout) {
    WarpSmem w{};
    const int lcap = (L + 7) / 8 * 8;  // (pool entries past L are never read for their value)
    const int nc = (degree + 31) / 32 * 32;
    int rk = 32;
    while (rk < R) rk <<= 1;
    int tab = vkind == 4 ? 0 : H * (vkind == 2 ? 2 : 4);  // (4: V lives in device memory)
    if (rk * 8 > tab) tab = rk * 8;
    // new-key scratch first, so that for degree <= 32 and the table layout every buffer but
    // the visited table sits at a compile-time offset from the warp's base
    w.off_newk = 0;
    w.off_newid = nc * 8;
    w.off_row = w.off_newid + nc * 4;   // the predicted next id row (cp.async target), nc ids
    w.off_newslot = w.off_row + nc * 4;
    w.off_pool = w.off_newslot + (layout == 0 ? 0 : nc * 4);  // newslot: layout 1 and PRS blocks (layout code 2)
    w.off_tab = w.off_pool + lcap * 8;
    w.bytes = w.off_tab + tab;
    return w;
}

size_t search_smem_per_warp(int L, int R, int H, int vkind, int degree, int layout) {
    return (size_t)warp_smem(L, R, H, vkind, degree, layout).bytes;
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
    kp.vkind = a.visited_kind;
    kp.tab16 = a.visited_kind == 2;
    kp.tab_bytes = a.visited_kind == 4 ? 0 : a.visited_slots * (kp.tab16 ? 2 : 4);
    kp.gvis_words = (ix.n + 127) / 128 * 4;  // bitset words per warp (16-byte multiple)
    kp.row_dups = ix.row_dups;
    {   // 32-byte aligned code rows: the table (layout 0), PRS blocks, or the rows of layout 1
        auto a32 = [](const void *q) { return (reinterpret_cast<uintptr_t>(q) & 31) == 0; };
        kp.wide = (ix.cbp % 32 == 0) &&
                  (ix.layout == 0 ? a32(ix.codes) && (!ix.prs_blk || a32(ix.prs_codes))
                                  : a32(ix.rows) && ix.row_bytes % 32 == 0 && ix.ids_bytes % 32 == 0);
    }
    kp.lcap = (a.L + 7) / 8 * 8;
    const WarpSmem w = warp_smem(a.L, a.rerank_n, a.visited_slots, a.visited_kind, ix.degree, ix.prs_blk ? 2 : ix.layout);
    kp.off_tab = w.off_tab;
    kp.off_pool = w.off_pool;
    kp.off_newk = w.off_newk;
    kp.off_newid = w.off_newid;
    kp.off_newslot = w.off_newslot;
    kp.off_row = w.off_row;
    kp.smem_per_warp = w.bytes;
    kp.n_base = ix.n;
    kp.rk_bytes = w.bytes - w.off_tab;
    kp.check = ix.err;
    if (mode_w(a.mode)) {
        kp.l2w = ix.l2w;
        kp.l2w_dims = ix.cbp * (ix.bits == 8 ? 1 : 2);
        kp.off_cta = (kp.l2w_dims * 4 + 15) / 16 * 16;
    }
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
    if (info) info->visited_kind = a.visited_kind;
    const int e = ix.degree <= 32 ? 1 : 2;
    // the compile-time common case (search_kernel VAR 1/2): degree 32 (one 32-id slice), table layout,
    // u16 visited table, rows without repeated ids, codes filling all G * CPL chunks
    kp.labels = a.alpha_s > 0.0f ? ix.labels : nullptr;
    kp.m_s = a.m_s;
    kp.alpha_s = a.alpha_s;
    kp.filt = (a.m_s > 0 && a.m_s < ix.degree) || kp.labels != nullptr;
    kp.prs_blk = ix.layout == 0 ? ix.prs_blk : nullptr;
    kp.prs_codes = ix.prs_codes;
    kp.adaptive = a.adaptive;
    kp.qlp_ef_low = a.qlp_ef_low;
    kp.qlp_hop = a.qlp_hop;
    kp.qlp_feature = a.qlp_feature;
    kp.qlp_threshold = a.qlp_threshold;
    kp.delta_min = ix.delta_min;
    const bool common = ix.degree == 32 && ix.layout == 0 && !ix.row_dups && !kp.filt && !kp.prs_blk &&
                        kp.chunks == (1 << kp.g_log2) * cpl && !a.qlp_ef_low;
    // VAR 1 writes no trace output at all; VAR 3 is the common case on the u32 visited table
    const int var = !common ? 0 : (kp.tab16 ? (a.has_trace ? 2 : 1) : (a.visited_kind == 3 ? 3 : 0));
    switch (a.mode) {
        case L2_8: return launch_search_mode<L2_8>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
        case L2_4: return launch_search_mode<L2_4>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
        case IP_8: return launch_search_mode<IP_8>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
        case IP_4: return launch_search_mode<IP_4>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
        case L2W_8: return launch_search_mode<L2W_8>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
        default: return launch_search_mode<L2W_4>(cpl, kp.g_log2, e, ix.layout, var, kp, warps_per_block, s, info, a.nq);
    }
}

}  // namespace vsag
