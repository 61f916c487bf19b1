// vsag_internal.cuh -- shared device/host definitions of libvsag (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "vsag.h"

namespace vsag {

// tau_l arithmetic modes (R-6 / R-7) x SQ bits.
enum Mode : int { L2_8 = 0, L2_4 = 1, IP_8 = 2, IP_4 = 3, L2W_8 = 4, L2W_4 = 5 };

__host__ __device__ inline int mode_of(int metric, int bits) {
    return (metric == VSAG_METRIC_L2 ? 0 : (metric == VSAG_METRIC_IP ? 2 : 4)) + (bits == 4 ? 1 : 0);
}
__host__ __device__ constexpr bool mode_sq4(int mode) { return mode == L2_4 || mode == IP_4 || mode == L2W_4; }
__host__ __device__ constexpr bool mode_l2(int mode) { return mode == L2_8 || mode == L2_4 || mode == L2W_8 || mode == L2W_4; }
__host__ __device__ constexpr bool mode_w(int mode) { return mode == L2W_8 || mode == L2W_4; }
// operand words per code word: SQ4 keeps (lo-nibble, hi-nibble) pairs (see query_prep).
__host__ __device__ inline int op_words_per_code_word(int mode) { return mode_sq4(mode) ? 2 : 1; }

struct Index {
    int64_t n = 0;
    int d = 0, bits = 0;
    int cb = 0;        // code bytes (unpadded, caller layout)
    int cbp = 0;       // code stride inside the index (cb rounded up to 16)
    int degree = 0;    // R (row width of the padded adjacency)
    int layout = 0;
    int device = 0;
    int row_dups = 0;  // some adjacency row holds an id twice (search de-duplicates rows)
    const float *base = nullptr;   // borrowed [n, d]
    const float *lower = nullptr;  // borrowed [d]
    const float *upper = nullptr;  // borrowed [d]
    const uint8_t *codes = nullptr;  // [n, cbp] (borrowed if cb == cbp and aligned)
    uint8_t *codes_owned = nullptr;
    int32_t *adj = nullptr;          // owned padded [n, degree]  (layout 0)
    uint8_t *rows = nullptr;         // owned [n, row_bytes]       (layout 1)
    int64_t row_bytes = 0;
    int ids_bytes = 0;               // degree * 4 rounded up to 16
    int32_t *entry = nullptr;        // owned, sorted unique [n_entry]
    int n_entry = 0;
    uint8_t *seed_codes = nullptr;   // owned [n_entry, cbp]
    uint8_t *seed_op = nullptr;      // owned tensor-core seed operand [n_entry, cbp (SQ8) or 2 cbp (SQ4)]
    float *lower_owned = nullptr;    // owned copies of the model (pointers above refer to them)
    float *labels = nullptr;         // owned [n, degree] edge labels (NEXT-2), +inf padding; NULL: none
    int32_t *prs_blk = nullptr;      // owned [n]: PRS block of each node or -1 (NEXT-4, partial delta)
    uint8_t *prs_codes = nullptr;    // owned [prs_nodes, degree * cbp] co-located neighbour codes
    int64_t prs_nodes = 0;
    int base_in_range = 0;           // every base value lies inside [lower, upper] (NEXT-3 bound valid)
    double delta_min = 0.0;          // smallest quantisation step over non-constant dimensions
    int32_t *l2w = nullptr;          // owned [cbp * 8 / bits] weights of the weighted L2 (NEXT-1b), 0-padded
    int l2w_W = 0;                   // their scale W (0: the weighted L2 would overflow int32)
    int64_t owned_bytes = 0;
    int *err_host = nullptr;         // owned mapped pinned error flag (1: seed-contraction MMA wait timed out)
    int *err = nullptr;              // its device alias
};

// ------------------------------------------------------------------ kernels (launchers)
cudaError_t launch_sq_minmax(const float *x, int64_t n, int d, uint32_t *ord_min, uint32_t *ord_max,
                             int *bad, cudaStream_t s);
cudaError_t launch_sq_finalize(const uint32_t *ord_min, const uint32_t *ord_max, int d, float *lower,
                               float *upper, cudaStream_t s);
cudaError_t launch_sq_encode(const float *x, int64_t n, int d, int bits, const float *lower,
                             const float *upper, uint8_t *codes, int64_t stride, cudaStream_t s);
cudaError_t launch_l2w_weights(const float *lower, const float *upper, int d, int dims_padded, int W,
                               int32_t *w, cudaStream_t s);
cudaError_t launch_train_quantile(const float *x, int64_t n, int d, int64_t il, int64_t iu, float *lower,
                                  float *upper, uint32_t *scratch, cudaStream_t s);
size_t train_quantile_scratch_words(int d);
cudaError_t launch_query_prep(const float *q, int64_t nq, int d, int bits, int metric, const float *lower,
                              const float *upper, int cbp, uint32_t *op, cudaStream_t s);
cudaError_t launch_check_adj(const int32_t *adj, int64_t count, int64_t n, int *bad, cudaStream_t s);
cudaError_t launch_csr_to_padded(const int64_t *row_ptr, const int32_t *col, int64_t n, int degree,
                                 int32_t *out, int *bad, cudaStream_t s);
cudaError_t launch_row_dups(const int32_t *adj, int64_t n, int degree, int *flag, cudaStream_t s);
cudaError_t launch_pad_labels(const int64_t *row_ptr, const float *src, int64_t n, int degree, float *dst, int *bad,
                              cudaStream_t s);
cudaError_t launch_range_check(const float *x, int64_t n, int d, const float *lower, const float *upper, int *bad,
                               cudaStream_t s);
cudaError_t launch_in_degree(const int32_t *adj, int64_t count, int32_t *indeg, cudaStream_t s);
cudaError_t launch_prs_build(const int32_t *adj, const uint8_t *codes, const int32_t *nodes, int64_t count, int degree,
                             int cbp, uint8_t *blocks, cudaStream_t s);
cudaError_t launch_copy_pad_codes(const uint8_t *src, int64_t n, int cb, int cbp, uint8_t *dst,
                                  cudaStream_t s);
cudaError_t launch_layout_build(const int32_t *adj, const uint8_t *codes, int64_t n, int degree, int cbp,
                                int ids_bytes, int64_t row_bytes, uint8_t *rows, cudaStream_t s);
cudaError_t launch_gather_codes(const int32_t *ids, int count, const uint8_t *codes, int cbp, uint8_t *dst,
                                cudaStream_t s);
cudaError_t launch_seed_tau(const uint32_t *op, const int32_t *l2w, int64_t nq, const uint8_t *seed_codes,
                            const uint8_t *seed_op, int n_seed, int cbp, int mode, int32_t *tau, int *err,
                            cudaStream_t s);
// the tensor-core seed operand: the seed codes (SQ8) or their nibbles in plane order (SQ4)
size_t seed_operand_bytes(int n_seed, int cbp, int bits);
cudaError_t launch_seed_operand(const uint8_t *seed_codes, int n_seed, int cbp, int bits, uint8_t *out, cudaStream_t s);
cudaError_t launch_seed_tau_umma(const uint8_t *op, int64_t nq, const uint8_t *seed_op, int n_seed, int kbytes, bool ip,
                                 int32_t *tau, int *err, cudaStream_t s);

struct SearchArgs {
    const Index *ix;
    const float *queries;
    const uint32_t *op;      // [nq, op_stride_words]
    int op_stride_words;
    const int32_t *seed_tau; // [nq, n_entry]
    uint64_t *init_keys;     // [nq, L] scratch: initial pools
    int *init_psz;           // [nq]
    int64_t nq;
    int k, ef, rerank_n, L, metric, mode;
    int visited_slots;
    int visited_kind;        // 2 u16 buckets, 3 u32 probing (shared memory), 4 device-memory bitset
    int code_lanes;          // 0 auto, else lanes per code (4..32)
    int m_s;                 // edge filter (NEXT-2): degree cap (0: none)
    float alpha_s;           // edge filter: label bound (0: none)
    int adaptive;            // NEXT-3 early stop of the re-rank
    int qlp_ef_low, qlp_hop, qlp_feature;  // NEXT-4b QLP checkpoint (qlp_ef_low == 0: off)
    long long qlp_threshold;
    int32_t *out_ids;
    float *out_dists;
    vsag_trace trace;        // pointers may be NULL
    int has_trace;
    unsigned int *counter;   // persistent-scheduler query counter (zeroed)
};

struct SearchLaunch {
    int warps_per_block;
    int blocks;
    size_t smem_per_warp;
    int visited_kind;  // 2 = u16 two-choice buckets, 3 = u32 linear probing, 4 = device-memory bitset
};

cudaError_t launch_seed_select(const int32_t *seed_tau, const int32_t *entry, int S, int64_t nq, int L,
                               uint64_t *init_keys, int *init_psz, cudaStream_t s);
cudaError_t launch_search(const SearchArgs &a, int warps_per_block, cudaStream_t s, SearchLaunch *info);
size_t search_smem_per_warp(int L, int R, int H, int vkind, int degree, int layout);
bool visited_u16(int H, int64_t n);
// stream-ordered device scratch from the library's own pool (api.cu)
cudaError_t scratch_alloc(void **p, size_t bytes, int device, cudaStream_t s);


}  // namespace vsag
