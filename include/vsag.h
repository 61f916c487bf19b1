/*
 * vsag.h -- C ABI of libvsag: the B200-native batched search hot path of VSAG
 * (arXiv 2503.17911, "VSAG: An Optimized Search Framework for Graph-based
 * Approximate Nearest Neighbor Search").
 *
 * The path (PAPER.md line numbers "P:n"):
 *   - SQ-b scalar quantisation, per-dimension [min, max] range, 2^b - 1 steps
 *     (App. G; §5.2 "FLOAT32 -> INT8/INT4");
 *   - Deterministic Access Greedy Search (Alg. 1; App. A)
 *     with low-precision distances tau_l on the SQ codes (exact int32);
 *   - selective re-rank of the best pool entries with full-precision tau_h
 *     (§5.3; Alg. 1 line 18);
 *   - optional PRS co-located neighbour-code layout (delta = 1, §3.3.2).
 * The exact arithmetic of every step is fixed by the readings R-1..R-22 in
 * DESIGN.md §3; the CPU oracle (oracle/) implements the same contract.
 *
 * Conventions for every entry point:
 *   - Pointers are CUDA DEVICE pointers unless stated otherwise.  Arrays are
 *     dense row-major with the shapes given.  `stream` is a cudaStream_t passed
 *     as void* (NULL = legacy default stream); work is enqueued stream-ordered
 *     and the call returns without synchronising unless stated otherwise.
 *   - Every call validates its arguments before launching anything and returns
 *     a vsag_status; on failure nothing is written to the outputs and
 *     vsag_last_error() returns a thread-local message.  No C++ exception
 *     crosses the ABI.
 *   - The caller owns every buffer it passes in.
 *   - Device scratch of a call comes from a stream-ordered memory pool owned by the
 *     library (one per device, freed blocks stay cached for the next call); the
 *     device's default pool (cudaMallocAsync) is not modified.
 */
#ifndef VSAG_H
#define VSAG_H
#include <stdint.h>

#if defined(__GNUC__)
#define VSAG_API __attribute__((visibility("default")))
#else
#define VSAG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t vsag_status;
enum {
    VSAG_OK = 0,
    VSAG_ERR_INVALID_ARG = 1,  /* bad sizes, null pointers, ids out of range, non-finite input */
    VSAG_ERR_UNSUPPORTED = 2,  /* a valid request outside this build's limits (e.g. degree > 64) */
    VSAG_ERR_OVERFLOW = 3,     /* tau_l could exceed int32 (R-20) */
    VSAG_ERR_OOM = 4,          /* device allocation failed */
    VSAG_ERR_CUDA = 5          /* any other CUDA runtime error (message has cudaGetErrorString) */
};
enum { VSAG_METRIC_L2 = 0, VSAG_METRIC_IP = 1,
       /* weighted code-space L2 traversal (NEXT-1b): tau_l = sum_j w_j (cq_j - c_j)^2 with
          w_j = round_half_away(W r_j^2 / max_k r_k^2), r_j = upper_j - lower_j (fp32, then fp64),
          W = min(8192, floor((2^31 - 1) / (d (2^b - 1)^2))); re-rank and outputs as L2 */
       VSAG_METRIC_L2W = 2 };
enum { VSAG_LAYOUT_TABLE = 0 /* delta = 0: global code table */,
       VSAG_LAYOUT_COLOCATED = 1 /* delta = 1: PRS, each node row = [ids | neighbour codes] */ };

/* Limits of this build. */
#define VSAG_MAX_DEGREE 64    /* out-degree R of the graph */
#define VSAG_MAX_POOL 1024    /* L = max(ef, rerank_n) */
#define VSAG_MAX_CODE_BYTES 2048
#define VSAG_MAX_BATCH (1LL << 30) /* queries per search call (the persistent scheduler's 32-bit
                                      query counter stays below 2^31 with every resident warp's
                                      final increment) */

typedef struct vsag_index vsag_index; /* opaque; immutable after load */

/* bits == 8 ? d : (d + 1) / 2  (SQ4 packs two codes per byte, low nibble first, R-5). */
VSAG_API int64_t vsag_code_bytes(int32_t d, int32_t bits);

/*
 * vsag_encode_sq -- SQ training (row a1) and encoding (row a2).
 *   x[n, d] fp32 (finite); bits in {4, 8}.
 *   train = 1: lower[j] = min_i x[i][j], upper[j] = max_i x[i][j] are computed from x
 *              and written to lower/upper (a zero bound is written as +0.0, R-1);
 *   train = 0: lower/upper[d] are read.
 *   codes[n, vsag_code_bytes(d, bits)] u8: per element clamp -> (v-l)/(u-l) ->
 *   *(2^b - 1) -> round half away from zero (fp32, one rounding per op, R-3);
 *   u == l encodes to 0 (R-4).
 * Errors: INVALID_ARG for null pointers, n < 0, d < 1, bits not in {4, 8}, or (train = 1)
 * a non-finite element (this check reads a device flag and synchronises `stream`).
 */
VSAG_API vsag_status vsag_encode_sq(const float *x, int64_t n, int32_t d, int32_t bits, int32_t train,
                           float *lower, float *upper, uint8_t *codes, void *stream);

/*
 * vsag_train_sq -- row a1 with truncation (App. G: "99th percentile statistics
 * rather than absolute extremes"; NEXT-1a).  x[n, d] fp32 (finite), 1 <= n < 2^32.
 * Per dimension j, with v_j its n values sorted ascending (ranks in fp64, no interpolation):
 *   lower[j] = v_j[floor((1 - quantile) * (n - 1))], upper[j] = v_j[floor(quantile * (n - 1))]
 * (a zero bound is written as +0.0).  quantile in (0.5, 1]; 1 gives the plain per-dimension
 * min/max of vsag_encode_sq(train = 1).  Encode with vsag_encode_sq(train = 0) afterwards.
 * Synchronises `stream`.  Errors: INVALID_ARG (null pointers, sizes, quantile, non-finite x).
 */
VSAG_API vsag_status vsag_train_sq(const float *x, int64_t n, int32_t d, double quantile, float *lower,
                                   float *upper, void *stream);

/*
 * vsag_index_load -- row a3.  Builds the device-side index and synchronises `stream`.
 *   base[n, d] fp32 (re-rank rows), codes[n, code_bytes] u8, lower/upper[d]: BORROWED --
 *   they must stay alive and unmodified until vsag_index_free.
 *   Graph G: if row_ptr != NULL it is CSR (row_ptr[n+1] int64, adj[row_ptr[n]]
 *   int32 column ids, every row length <= degree); otherwise adj is fixed-degree
 *   [n, degree] int32.  -1 marks an empty slot; other ids must be in [0, n).
 *   degree in [1, 64].  Self-loops and duplicate ids are allowed (absorbed by V, R-13).
 *   base must be 16-byte aligned (the re-rank reads it with 16-byte loads).
 *   entry[n_entry] int32: the initial nodes I of Alg. 1, ids in [0, n);
 *   duplicates are removed (R-11).
 *   layout: VSAG_LAYOUT_TABLE or VSAG_LAYOUT_COLOCATED.
 * The index OWNS (and frees) its derived buffers: the padded adjacency, the layout-1
 * rows, the seed-code block and any padded copy of the codes.
 * Errors: INVALID_ARG (bad sizes/ids, CSR row longer than degree), UNSUPPORTED (degree
 * > 64, code bytes > 2048), OVERFLOW (R-20), OOM, CUDA.
 */
VSAG_API vsag_status vsag_index_load(const float *base, const uint8_t *codes, const float *lower,
                            const float *upper, int64_t n, int32_t d, int32_t bits,
                            const int64_t *row_ptr, const int32_t *adj, int32_t degree,
                            const int32_t *entry, int32_t n_entry, int32_t layout,
                            void *stream, vsag_index **out);

/*
 * vsag_index_set_labels -- per-edge labels L of the graph (Alg. 2 prune-based labels,
 * P:518-568; NEXT-2).  labels fp32 (device), in the layout the adjacency had at
 * vsag_index_load: [n, degree] rows, or CSR [row_ptr[n]] aligned with the columns (pass
 * the same row_ptr again).  The index copies them (owned; padding slots get +inf) and
 * searches may then filter edges with vsag_search_params.alpha_s.  Synchronises `stream`.
 * Errors: INVALID_ARG (null pointers, NaN label, CSR rows inconsistent with the index).
 */
VSAG_API vsag_status vsag_index_set_labels(vsag_index *ix, const int64_t *row_ptr, const float *labels,
                                           void *stream);

/*
 * vsag_index_set_prs -- PRS with a redundancy ratio delta in [0, 1] (§3.3.3, P:430-436:
 * "dynamically tunable redundancy ratio"; NEXT-4) for a VSAG_LAYOUT_TABLE index: the
 * round(delta * n) nodes of highest in-degree (ties: lower id) get a block holding their
 * neighbours' codes in row order (zero for empty slots); expanding such a node reads the
 * block instead of the global table.  delta = 0 drops the blocks.  Results are identical
 * for every delta.  Synchronises `stream`.  Errors: INVALID_ARG (delta outside [0, 1],
 * layout-1 index), OOM.
 */
VSAG_API vsag_status vsag_index_set_prs(vsag_index *ix, double delta, void *stream);

/* Optional per-query parity/statistics outputs (device pointers; any may be NULL). */
typedef struct {
    int32_t max_hops;  /* columns of `expanded` */
    int32_t *hops;     /* [nq] expansions performed */
    int32_t *expanded; /* [nq, max_hops] expanded node ids in order, -1 pad */
    int32_t *n_lp;     /* [nq] tau_l evaluations (entry set + new neighbours) */
    int32_t *n_hp;     /* [nq] tau_h evaluations = R' */
    int32_t *n_miss;   /* [nq] visited-cache inserts that could not be stored */
    int32_t *pool_ids; /* [nq, L] final pool ids, ascending (tau_l, id), -1 pad */
    int32_t *pool_tau; /* [nq, L] final pool tau_l, INT32_MAX pad */
} vsag_trace;

typedef struct {
    int32_t k;               /* results per query, >= 1 */
    int32_t ef;              /* expansion window ef_s, >= 1 */
    int32_t rerank_n;        /* R: pool entries re-ranked in fp32 (0 => ef); k <= R */
    int32_t metric;          /* VSAG_METRIC_L2 (squared) or VSAG_METRIC_IP (negated) */
    int32_t visited_slots;   /* per-query visited-cache slots (power of two in [256, 65536]); 0 = auto:
                                max(1024, next_pow2(12 ef)) capped at 16384, halved while the table costs
                                more than 15% of the batch's resident warps, doubled (up to 4096) while
                                that costs none */
    int32_t warps_per_block; /* search-kernel CTA size in warps (1..4), 0 = auto */
    int32_t code_lanes;      /* lanes that gather one code (power of two 4..32), 0 = auto */
    /* edge filter of Alg. 1 line 8 (NEXT-2), applied to each expanded row before
       the visited test: keep edges with label <= alpha_s (needs vsag_index_set_labels), and
       of those only the first max_degree in row order (R-23) */
    int32_t max_degree;      /* m_s, 0 = no cap */
    float alpha_s;           /* 0 = no label bound; > 0 needs labels */
    /* exact early stop of the re-rank (NEXT-3, R-27; L2 only, and every base value
       must lie inside [lower, upper], which vsag_index_load checks): in groups of 4, stop
       before a candidate whose tau_l lower-bounds tau_h above the k-th best tau_h so far.
       Same ids and distances as the full re-rank; trace.n_hp counts the tau_h evaluated. */
    int32_t rerank_adaptive;
    /* QLP early termination (§4.3; NEXT-4b, R-28): after qlp_hop
       expansions, if feature qlp_feature of the pool (1 = sum of the 5 best tau_l, 2 =
       tau_l(k-th) - tau_l(best); feature 0 of the oracle, the points scanned, is not exact
       under a forgetful visited cache and returns UNSUPPORTED) is <= qlp_threshold, ef and
       the pool capacity drop to qlp_ef_low (in [k, ef]; farthest entries evicted) and the
       re-rank count to min(R, qlp_ef_low).  qlp_ef_low == 0: off. */
    int32_t qlp_ef_low;
    int32_t qlp_hop;         /* >= 0 */
    int32_t qlp_feature;     /* 1 or 2 */
    /* visited set V of Alg. 1: 0 = auto; 2 = u16 two-choice buckets in shared memory
       (only where a 14-bit tag identifies an id: INVALID_ARG otherwise); 3 = u32 linear
       probing in shared memory; both are bounded caches that may forget ids (never the
       traversal); 4 = an exact n-bit bitset per resident warp in device memory
       (cleared per query, ceil(n / 128) * 16 bytes per warp of call scratch), never forgets.
       auto: the shared-memory table (2 where valid, else 3), or 4 when dropping the table
       lets >= 1.25x more of the batch's warps reside and clearing n bits is <= 1/4 of the
       query's estimated gathers (only with an explicitly large visited_slots: the auto table
       size keeps residency) */
    int32_t visited_kind;
    int64_t qlp_threshold;
    /* optional caller-owned cudaEvent_t handles (NULL: none) recorded on `stream` right before
       and right after the search kernel (rows a6-a8), without any synchronisation: the
       caller reads cudaEventElapsedTime later, e.g. per launch inside a pipelined loop */
    void *ev_search_start;
    void *ev_search_stop;
} vsag_search_params;

/* Optional per-stage device times of one call, filled when the call returns
   (requesting it synchronises `stream`). */
typedef struct {
    float ms_query_prep;
    float ms_seed;
    float ms_search;
    float ms_total;
    int32_t launches;        /* kernels launched by the call */
    int32_t visited_slots;   /* value actually used */
    int32_t warps_per_block; /* value actually used */
    int32_t blocks;          /* search-kernel grid size */
    int32_t visited_kind;    /* visited set used: 2 = u16 buckets, 3 = u32 probing, 4 = device-memory bitset */
} vsag_timing;

/*
 * vsag_search_batch -- rows a4-a8 for a batch of queries (the hot entry point).
 *   queries[nq, d] fp32; out_ids[nq, k] int32 and out_dists[nq, k] fp32, ascending
 *   (tau_h, id); fewer than k results pad with -1 / +inf (R-18).  L2 distances are
 *   squared, IP distances are -<q, x> (R-17).  ef >= 1, k <= rerank_n (0 => ef),
 *   L = max(ef, rerank_n) <= 1024.  nq == 0 is a no-op; nq > VSAG_MAX_BATCH returns
 *   UNSUPPORTED.  queries must be 16-byte aligned (INVALID_ARG otherwise).  trace may be NULL.
 *   Every argument is validated before anything is allocated or launched.
 *   If a tensor-core completion wait of the seed contraction ever times out (a hardware
 *   fault; it never hangs the GPU and never traps), the kernel sets a device flag of the
 *   index and the outputs are invalid: the calls that synchronise anyway
 *   (vsag_search_batch_host, and _ex with timing != NULL) then return VSAG_ERR_CUDA.
 */
VSAG_API vsag_status vsag_search_batch(const vsag_index *ix, const float *queries, int64_t nq, int32_t k,
                              int32_t ef, int32_t rerank_n, int32_t metric, int32_t *out_ids,
                              float *out_dists, vsag_trace *trace, void *stream);

/* Same as vsag_search_batch with tuning knobs, trace and optional stage timing. */
VSAG_API vsag_status vsag_search_batch_ex(const vsag_index *ix, const float *queries, int64_t nq,
                                 const vsag_search_params *params, int32_t *out_ids,
                                 float *out_dists, vsag_trace *trace, vsag_timing *timing,
                                 void *stream);

/*
 * vsag_search_batch_host -- end-to-end form: queries, out_ids and out_dists are HOST
 * pointers (pinned memory recommended).  Copies queries host->device, searches and
 * copies the results device->host on `stream`, then synchronises `stream`.
 */
VSAG_API vsag_status vsag_search_batch_host(const vsag_index *ix, const float *queries_host, int64_t nq,
                                   const vsag_search_params *params, int32_t *out_ids_host,
                                   float *out_dists_host, void *stream);

typedef struct {
    int64_t n;
    int32_t d, bits, code_bytes, code_stride, degree, layout, n_entry;
    int64_t device_bytes; /* bytes owned by the index */
    int64_t prs_nodes;    /* nodes with a co-located neighbour-code block (vsag_index_set_prs) */
    int64_t prs_bytes;    /* bytes of those blocks */
} vsag_index_info;

VSAG_API vsag_status vsag_index_get_info(const vsag_index *ix, vsag_index_info *info);

/* Frees the index's owned buffers (synchronises the device).  NULL is a no-op. */
VSAG_API vsag_status vsag_index_free(vsag_index *ix);

/* Message for the last failed call on this thread ("" if none). */
VSAG_API const char *vsag_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* VSAG_H */
