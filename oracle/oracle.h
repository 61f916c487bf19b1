/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * A plain, slow, single-threaded CPU transcription of the VSAG search hot path
 * (arXiv 2503.17911): SQ training/encoding (App. G), the
 * low-precision distance tau_l on SQ codes (§5.2), Deterministic
 * Access Greedy Search (Alg. 1; App. A) and
 * the selective re-rank with fp32 vectors (§5.3; Alg. 1 line 18).
 * Every free choice is fixed by the readings in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load liboracle.so.  It shares no code with libvsag.
 * All pointers are HOST pointers.  Functions return 0 on success, a nonzero
 * ORACLE_ERR_* code on invalid input (no output is written in that case).
 */
#ifndef VSAG_ORACLE_H
#define VSAG_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_ERR_INVALID_ARG = 1, ORACLE_ERR_OVERFLOW = 3 };
enum { ORACLE_METRIC_L2 = 0, ORACLE_METRIC_IP = 1, ORACLE_METRIC_L2W = 2 };

/* bytes per code: bits == 8 ? d : (d + 1) / 2 (two 4-bit codes per byte, low nibble first). */
int64_t oracle_code_bytes(int32_t d, int32_t bits);

/* lower[j] = min_i x[i][j], upper[j] = max_i x[i][j] over the base set (quantile 1.0). */
int32_t oracle_train_sq(const float *x, int64_t n, int32_t d, float *lower, float *upper);

/* Truncated SQ training (App. G, "99th percentile statistics"; NEXT-1a):
   per dimension, with v the dimension's n values sorted ascending,
   lower[j] = v[floor((1 - q) * (n - 1))], upper[j] = v[floor(q * (n - 1))] (indices in fp64,
   no interpolation); q in (0.5, 1]; q = 1 is oracle_train_sq. */
int32_t oracle_train_sq_quantile(const float *x, int64_t n, int32_t d, double q, float *lower, float *upper);

/* Weighted code-space L2 (NEXT-1b): integer weights w[j] = round_half_away(W * r_j^2 / max_j r_j^2),
   r_j = upper[j] - lower[j] (fp32) widened to fp64, W = min(8192, floor((2^31 - 1) / (d (2^b - 1)^2))).
   tau_l = sum_j w_j (cq_j - c_j)^2 stays below 2^31.  Returns W (0 if W < 1: overflow). */
int32_t oracle_l2w_weights(const float *lower, const float *upper, int32_t d, int32_t bits, int32_t *w);

/* codes[n, code_bytes] from x[n, d] with the pinned fp32 sequence (R-3). */
int32_t oracle_encode_sq(const float *x, int64_t n, int32_t d, int32_t bits,
                         const float *lower, const float *upper, uint8_t *codes);

/* IP query weights w[d] in [-127, 127] (R-7). */
int32_t oracle_ip_weights(const float *q, int32_t d, const float *lower, const float *upper,
                          int32_t *w);

/* tau_l between one query and one base code (R-6/R-7; L2W: NEXT-1b); int64 result. */
int32_t oracle_tau_l(const float *q, const uint8_t *code, int32_t d, int32_t bits,
                     const float *lower, const float *upper, int32_t metric, int64_t *out);

/* tau_h between one query and one base row (fp64 accumulation, rounded once to fp32). */
float oracle_tau_h(const float *q, const float *x, int32_t d, int32_t metric);

/* NEXT-3 (R-27): lower bound on tau_h (L2) from tau_l for base vectors inside [lower, upper]:
   D_min^2 * max(0, tau_l - 2.0002 sqrt(d tau_l)) * (1 - 1e-5), D_min the smallest step. */
double oracle_rerank_lower_bound(int64_t tau_l, int32_t d, const float *lower, const float *upper, int32_t bits);

/*
 * Batched search.  adjacency: if row_ptr != NULL it is CSR (row_ptr[n+1] int64,
 * adj = column ids), otherwise adj is fixed-degree [n, degree] with -1 = empty.
 * entry[n_entry]: initial nodes I (deduplicated internally).
 * rerank_n = R (0 => ef); pool capacity L = max(ef, R).
 * Outputs out_ids/out_dists [nq, k] (ids -1 / dists +inf pad).
 * Optional trace (any pointer may be NULL):
 *   hops[nq], n_lp[nq], n_hp[nq],
 *   expanded[nq, max_hops] (expansion order; -1 pad),
 *   pool_ids[nq, L], pool_tau[nq, L] (final pool, ascending (tau_l, id); -1 / INT32_MAX pad).
 * nthreads > 1 shards queries over std::threads (harness timing only; each thread
 * runs the same single-query function).
 */
int32_t oracle_search_batch(const float *base, const uint8_t *codes, const float *lower,
                            const float *upper, int64_t n, int32_t d, int32_t bits,
                            const int64_t *row_ptr, const int32_t *adj, int32_t degree,
                            const int32_t *entry, int32_t n_entry,
                            const float *queries, int64_t nq, int32_t k, int32_t ef,
                            int32_t rerank_n, int32_t metric,
                            int32_t *out_ids, float *out_dists,
                            int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                            int32_t *expanded, int32_t max_hops,
                            int32_t *pool_ids, int32_t *pool_tau,
                            int32_t nthreads);

/*
 * Same with the edge filter of Alg. 1 line 8 (NEXT-2): labels (per-edge, same
 * layout as adj; NULL = no filter) keep only edges with L_ij <= alpha_s, and of those only
 * the first m_s in row order (m_s <= 0: no cap), before the visited test (R-23).
 * adaptive != 0 (L2 only; NEXT-3, R-27): the re-rank runs in groups of 4 and stops
 * before a group whose first tau_l lower-bounds tau_h above the k-th best tau_h so far.
 */
int32_t oracle_search_batch_labels(const float *base, const uint8_t *codes, const float *lower,
                                   const float *upper, int64_t n, int32_t d, int32_t bits,
                                   const int64_t *row_ptr, const int32_t *adj, int32_t degree,
                                   const int32_t *entry, int32_t n_entry,
                                   const float *queries, int64_t nq, int32_t k, int32_t ef,
                                   int32_t rerank_n, int32_t metric,
                                   const float *labels, int32_t m_s, float alpha_s, int32_t adaptive,
                                   int32_t *out_ids, float *out_dists,
                                   int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                                   int32_t *expanded, int32_t max_hops,
                                   int32_t *pool_ids, int32_t *pool_tau,
                                   int32_t nthreads);

/*
 * Same with QLP early termination (§4.3; NEXT-4b, R-28): qlp_ef_low in
 * [k, ef] (0 = off); after qlp_hop expansions, if feature qlp_feature (0 = points scanned
 * n_lp, 1 = sum of the 5 best tau_l, 2 = tau_l(k-th) - tau_l(best)) is <= qlp_threshold,
 * ef and the pool capacity drop to qlp_ef_low and the re-rank count to min(R, qlp_ef_low).
 */
int32_t oracle_search_batch_qlp(const float *base, const uint8_t *codes, const float *lower,
                                const float *upper, int64_t n, int32_t d, int32_t bits,
                                const int64_t *row_ptr, const int32_t *adj, int32_t degree,
                                const int32_t *entry, int32_t n_entry,
                                const float *queries, int64_t nq, int32_t k, int32_t ef,
                                int32_t rerank_n, int32_t metric,
                                const float *labels, int32_t m_s, float alpha_s, int32_t adaptive,
                                int32_t qlp_hop, int32_t qlp_ef_low, int32_t qlp_feature, int64_t qlp_threshold,
                                int32_t *out_ids, float *out_dists,
                                int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                                int32_t *expanded, int32_t max_hops,
                                int32_t *pool_ids, int32_t *pool_tau,
                                int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif
