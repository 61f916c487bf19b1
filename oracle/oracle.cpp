// oracle.cpp -- TEST INFRASTRUCTURE ONLY (not the product path; see oracle.h).
//
// Plain, slow, single-threaded, obviously-correct CPU transcription of the VSAG
// search hot path (arXiv 2503.17911).  Built with -O2 -ffp-contract=off and no
// fast-math so every fp32/fp64 operation is one IEEE-rounded operation in the
// order written here.  It shares no code with the CUDA library (libvsag).
//
// Citations: PAPER.md line numbers ("P:n"); readings R-n are DESIGN.md §3.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

// ---------------------------------------------------------------- SQ (App. G)
// Value of dimension j of a packed code.  SQ8: one byte per dimension.  SQ4: two
// codes per byte, low nibble first (R-5).
int code_value(const uint8_t *code, int bits, int j) {
    if (bits == 8) return code[j];
    uint8_t b = code[j / 2];
    return (j % 2 == 0) ? (b & 0x0F) : (b >> 4);
}

// One dimension of SQ-b: "the dynamic range is uniformly partitioned",
// on the 2^b - 1 step grid (R-2), with the pinned fp32 order (R-3):
//   clamp, (v - lo) / (hi - lo), * (2^b - 1), round half away from zero.
// A constant dimension encodes to 0 (R-4).
int encode_value(float v, float lo, float hi, int bits) {
    const int levels = (1 << bits) - 1;
    if (hi == lo) return 0;
    float c = fminf(fmaxf(v, lo), hi);
    float t = (c - lo) / (hi - lo);
    t = t * (float)levels;
    int code = (int)roundf(t);
    if (code > levels) code = levels;
    return code;
}

// ---------------------------------------------------------------- tau_l (§5.2)
// The query side of tau_l.  L2 (R-6): the query is encoded with the base model
// and tau_l = sum_d (cq_d - c_d)^2 (symmetric code space, exact integers).
// IP (R-7): int8 weights w_d = round(127 * a_d / s), a_d = q_d * (u_d - l_d),
// s = max_d |a_d|, and tau_l = -sum_d w_d * c_d.
struct QueryOperand {
    std::vector<int> v;  // L2 / L2W: query codes; IP: weights
    std::vector<int> w;  // L2W: per-dimension integer weights
};

// NEXT-1b: W and the integer weights of the weighted code-space L2 (oracle.h).
int l2w_weights(const float *lower, const float *upper, int d, int bits, std::vector<int> &w) {
    const int64_t levels = (1 << bits) - 1;
    const int64_t cap = (((int64_t)1 << 31) - 1) / ((int64_t)d * levels * levels);
    const int W = (int)std::min<int64_t>(8192, cap);
    w.assign(d, 0);
    if (W < 1) return 0;
    double m = 0.0;
    for (int j = 0; j < d; j++) {
        double r = (double)(upper[j] - lower[j]);
        m = std::max(m, r * r);
    }
    for (int j = 0; j < d; j++) {
        double r = (double)(upper[j] - lower[j]);
        w[j] = m > 0.0 ? (int)std::llround((double)W * (r * r) / m) : 0;
    }
    return W;
}

QueryOperand make_operand(const float *q, int d, int bits, const float *lower, const float *upper,
                          int metric) {
    QueryOperand op;
    op.v.resize(d);
    if (metric == ORACLE_METRIC_L2 || metric == ORACLE_METRIC_L2W) {
        for (int j = 0; j < d; j++) op.v[j] = encode_value(q[j], lower[j], upper[j], bits);
        if (metric == ORACLE_METRIC_L2W) l2w_weights(lower, upper, d, bits, op.w);
    } else {
        std::vector<float> a(d);
        float s = 0.0f;
        for (int j = 0; j < d; j++) {
            a[j] = q[j] * (upper[j] - lower[j]);
            float m = fabsf(a[j]);
            if (m > s) s = m;
        }
        for (int j = 0; j < d; j++) {
            if (s == 0.0f) {
                op.v[j] = 0;
            } else {
                float t = a[j] / s;
                t = t * 127.0f;
                op.v[j] = (int)roundf(t);
            }
        }
    }
    return op;
}

int64_t tau_l(const QueryOperand &op, const uint8_t *code, int d, int bits, int metric) {
    int64_t s = 0;
    if (metric == ORACLE_METRIC_L2) {
        for (int j = 0; j < d; j++) {
            int64_t diff = (int64_t)op.v[j] - (int64_t)code_value(code, bits, j);
            s += diff * diff;
        }
        return s;
    }
    if (metric == ORACLE_METRIC_L2W) {  // NEXT-1b: sum_j w_j (cq_j - c_j)^2
        for (int j = 0; j < d; j++) {
            int64_t diff = (int64_t)op.v[j] - (int64_t)code_value(code, bits, j);
            s += (int64_t)op.w[j] * diff * diff;
        }
        return s;
    }
    for (int j = 0; j < d; j++) s += (int64_t)op.v[j] * (int64_t)code_value(code, bits, j);
    return -s;
}

// ---------------------------------------------------------------- tau_h (§5.3)
// Full-precision distance of the re-rank (R-16): fp32 inputs widened exactly to
// fp64, accumulated in fp64 in dimension order, rounded once to fp32.  L2 is
// squared (no sqrt); IP is negated so that smaller is nearer (R-17).
float tau_h(const float *q, const float *x, int d, int metric) {
    double s = 0.0;
    if (metric == ORACLE_METRIC_L2 || metric == ORACLE_METRIC_L2W) {  // L2W re-ranks with plain L2
        for (int j = 0; j < d; j++) {
            double diff = (double)q[j] - (double)x[j];
            s = s + diff * diff;
        }
        return (float)s;
    }
    for (int j = 0; j < d; j++) s = s + (double)q[j] * (double)x[j];
    return (float)(-s);
}

// ---------------------------------------------------------------- NEXT-3 bound (R-27)
// For L2 with every base value inside [l_d, u_d]: a value encodes to the grid point nearest
// to it, |v - (l + c*D)| <= D/2 (D = (u - l) / (2^b - 1)), and clamping the query only moves
// it towards the range, so |q_d - x_d| >= D_d * max(0, |cq_d - c_d| - 1).  Summing and
// Cauchy-Schwarz (sum |delta| <= sqrt(d * tau_l)) give
//   tau_h >= D_min^2 * max(0, tau_l - 2 sqrt(d * tau_l)),
// taken with margins for the fp32 encode and the fp32 rounding of tau_h.
double rerank_lower_bound(int64_t tau_l, int d, double delta_min) {
    const double t = (double)tau_l;
    const double v = t - 2.0002 * std::sqrt((double)d * t);
    return v > 0.0 ? delta_min * delta_min * v * (1.0 - 1e-5) : 0.0;
}

double min_step(const float *lower, const float *upper, int d, int bits) {
    const double levels = (double)((1 << bits) - 1);
    double m = 0.0;
    for (int j = 0; j < d; j++) {
        const double r = (double)(upper[j] - lower[j]);
        if (r > 0.0 && (m == 0.0 || r / levels < m)) m = r / levels;
    }
    return m;
}

// ---------------------------------------------------------------- Alg. 1
// Candidate pool C: kept as a list sorted ascending by the key
// (tau_l, id) -- ties broken by the smaller id (R-8) -- with an "expanded" flag
// per entry.  Its capacity is L = max(ef, R) (R-9); expansions only come from
// the first ef positions.
struct Cand {
    int64_t tau;
    int32_t id;
    bool expanded;
};

bool cand_less(const Cand &a, const Cand &b) {
    return a.tau < b.tau || (a.tau == b.tau && a.id < b.id);
}

// "insert (x_j, tau_l(x_j, x_q)) into C and keep |C| <= ef_s" (Alg. 1 line 17).
void insert_bounded(std::vector<Cand> &pool, Cand c, size_t cap) {
    auto it = std::upper_bound(pool.begin(), pool.end(), c, cand_less);
    pool.insert(it, c);
    if (pool.size() > cap) pool.pop_back();
}

struct Index {
    const float *base;
    const uint8_t *codes;
    const float *lower;
    const float *upper;
    int64_t n;
    int d;
    int bits;
    int64_t code_bytes;
    const int64_t *row_ptr;
    const int32_t *adj;
    int degree;
    std::vector<int32_t> entry;  // deduplicated, sorted
    const float *labels = nullptr;  // per-edge labels L (same layout as adj), or NULL
    bool adaptive = false;          // NEXT-3 exact early stop of the re-rank (L2, base inside [l, u])
    double delta_min = 0.0;         // smallest quantisation step over non-constant dimensions
    int m_s = 0;                    // degree cap of the search (<= 0: none)
    float alpha_s = 0.0f;           // label bound of the search
    // QLP early termination (NEXT-4b, R-28): at the checkpoint (after qlp_hop
    // expansions) a decision stump on one feature shrinks the candidate size to qlp_ef_low
    int qlp_hop = 0, qlp_ef_low = 0, qlp_feature = 0;  // qlp_ef_low == 0: off
    int64_t qlp_threshold = 0;
};

// Out-edges G_i of node i.  With labels (NEXT-2, the edge filter of Alg. 1
// line 8): only edges with L_ij <= alpha_s, and only the first m_s of those in
// row order (R-23: the cap counts label-valid edges whether visited or not, so the search
// equals a search on the graph built with m_c = m_s, alpha_c = alpha_s -- P:598).
std::vector<int32_t> row(const Index &ix, int32_t i) {
    std::vector<int32_t> r;
    int64_t a, b;
    if (ix.row_ptr) {
        a = ix.row_ptr[i];
        b = ix.row_ptr[i + 1];
    } else {
        a = (int64_t)i * ix.degree;
        b = a + ix.degree;
    }
    for (int64_t t = a; t < b; t++) {
        const int32_t j = ix.adj[t];
        if (ix.labels) {
            if (j < 0 || !(ix.labels[t] <= ix.alpha_s)) continue;
            if (ix.m_s > 0 && (int)r.size() >= ix.m_s) break;
        }
        r.push_back(j);
    }
    return r;
}

struct QueryResult {
    std::vector<int32_t> ids;
    std::vector<float> dists;
    std::vector<int32_t> expanded;
    std::vector<Cand> pool;
    int hops = 0;
    int n_lp = 0;
    int n_hp = 0;
};

QueryResult search_one(const Index &ix, const float *q, int k, int ef, int rerank_n, int metric) {
    QueryResult res;
    size_t cap = (size_t)std::max(ef, rerank_n);
    QueryOperand op = make_operand(q, ix.d, ix.bits, ix.lower, ix.upper, metric);
    auto tau = [&](int32_t j) { return tau_l(op, ix.codes + (int64_t)j * ix.code_bytes, ix.d, ix.bits, metric); };

    // Lines 1-3: C <- I with tau_l; V <- ids of the seeds that entered C (R-10).
    std::vector<Cand> pool;
    for (int32_t s : ix.entry) insert_bounded(pool, Cand{tau(s), s, false}, cap);
    std::unordered_set<int32_t> visited;
    for (const Cand &c : pool) visited.insert(c.id);
    res.n_lp = (int)ix.entry.size();

    // Lines 4-17.
    bool checked = false;
    while (true) {
        // QLP (§4.3: "after traversing certain hops in the graph, we employ the
        // decision tree along with the current features to determine whether the candidate
        // size should be reduced"), NEXT-4b / R-28: one checkpoint after qlp_hop expansions;
        // the decision is a stump "feature <= threshold" on one integer feature of the state:
        // 0 the points scanned so far (n_lp), 1 the sum of the 5 best tau_l (5 x their mean),
        // 2 the top-k spread tau_l(k-th) - tau_l(best).  Too few candidates: no decision.
        // Shrink: ef and the pool capacity drop to qlp_ef_low (farthest entries evicted),
        // the re-rank count to min(R, qlp_ef_low).
        if (ix.qlp_ef_low > 0 && !checked && res.hops == ix.qlp_hop) {
            checked = true;
            bool have = false;
            int64_t f = 0;
            if (ix.qlp_feature == 0) {
                have = true;
                f = res.n_lp;
            } else if (ix.qlp_feature == 1) {
                have = pool.size() >= 5;
                for (size_t t = 0; have && t < 5; t++) f += pool[t].tau;
            } else {
                have = pool.size() >= (size_t)k;
                if (have) f = pool[k - 1].tau - pool[0].tau;
            }
            if (have && f <= ix.qlp_threshold) {
                ef = ix.qlp_ef_low;
                cap = (size_t)ix.qlp_ef_low;
                rerank_n = std::min(rerank_n, ix.qlp_ef_low);
                if (pool.size() > cap) pool.resize(cap);
            }
        }
        // Line 5: closest un-expanded node of C, within the window [0, ef) (R-9, R-14).
        size_t lim = std::min(pool.size(), (size_t)ef);
        size_t p = lim;
        for (size_t t = 0; t < lim; t++) {
            if (!pool[t].expanded) {
                p = t;
                break;
            }
        }
        if (p == lim) break;
        pool[p].expanded = true;
        int32_t i = pool[p].id;
        res.expanded.push_back(i);
        res.hops++;

        // Lines 6-10: batch-filter the ids first, without touching vector data
        // (deterministic access).  -1 is padding (R-13); the label and
        // degree filters are off (alpha_s = inf, m_s = R; R-12).
        std::vector<int32_t> N;
        for (int32_t j : row(ix, i)) {
            if (j < 0) continue;
            if (visited.count(j)) continue;
            N.push_back(j);
            visited.insert(j);
        }
        // Lines 13-17: compute tau_l for each new neighbour and insert.
        for (int32_t j : N) {
            insert_bounded(pool, Cand{tau(j), j, false}, cap);
            res.n_lp++;
        }
    }
    res.pool = pool;

    // Line 18: selective re-rank of the first R' = min(R, |C|) entries (R-15).  NEXT-3
    // (R-27): in groups of 4, stop before a group whose first tau_l lower-bounds tau_h above
    // the k-th best tau_h so far -- no later candidate can enter the top-k.
    size_t rr = std::min(pool.size(), (size_t)rerank_n);
    std::vector<std::pair<float, int32_t>> hp;
    size_t done = 0;
    for (size_t t = 0; t < rr; t++) {
        if (ix.adaptive && t % 4 == 0 && t >= (size_t)k) {
            std::vector<float> best;
            for (const auto &e : hp) best.push_back(e.first);
            std::nth_element(best.begin(), best.begin() + (k - 1), best.end());
            const double tk = (double)best[k - 1];
            if (rerank_lower_bound(pool[t].tau, ix.d, ix.delta_min) > tk) break;
        }
        int32_t j = pool[t].id;
        hp.push_back({tau_h(q, ix.base + (int64_t)j * ix.d, ix.d, metric), j});
        done++;
    }
    res.n_hp = (int)done;
    std::sort(hp.begin(), hp.end(), [](const std::pair<float, int32_t> &a, const std::pair<float, int32_t> &b) {
        return a.first < b.first || (a.first == b.first && a.second < b.second);
    });
    for (int t = 0; t < k; t++) {
        if ((size_t)t < hp.size()) {
            res.ids.push_back(hp[t].second);
            res.dists.push_back(hp[t].first);
        } else {  // fewer than k reachable (R-18)
            res.ids.push_back(-1);
            res.dists.push_back(std::numeric_limits<float>::infinity());
        }
    }
    return res;
}

bool tau_fits_int32(int d, int bits, int metric) {
    const int64_t levels = (1 << bits) - 1;
    if (metric == ORACLE_METRIC_L2) return (int64_t)d * levels * levels < ((int64_t)1 << 31);
    if (metric == ORACLE_METRIC_L2W) return (int64_t)d * levels * levels < ((int64_t)1 << 31) - 1;  // W >= 1
    return (int64_t)d * 127 * levels < ((int64_t)1 << 31);
}

}  // namespace

extern "C" {

int64_t oracle_code_bytes(int32_t d, int32_t bits) { return bits == 8 ? d : (d + 1) / 2; }

int32_t oracle_train_sq(const float *x, int64_t n, int32_t d, float *lower, float *upper) {
    if (!x || !lower || !upper || n < 1 || d < 1) return ORACLE_ERR_INVALID_ARG;
    for (int64_t i = 0; i < n * d; i++)
        if (!std::isfinite(x[i])) return ORACLE_ERR_INVALID_ARG;
    for (int j = 0; j < d; j++) {
        float lo = x[j], hi = x[j];
        for (int64_t i = 1; i < n; i++) {
            float v = x[i * d + j];
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
        // The sign of a zero bound is immaterial to encoding; canonicalise to +0 (R-1).
        lower[j] = (lo == 0.0f) ? 0.0f : lo;
        upper[j] = (hi == 0.0f) ? 0.0f : hi;
    }
    return ORACLE_OK;
}

int32_t oracle_train_sq_quantile(const float *x, int64_t n, int32_t d, double q, float *lower, float *upper) {
    if (!x || !lower || !upper || n < 1 || d < 1 || !(q > 0.5 && q <= 1.0)) return ORACLE_ERR_INVALID_ARG;
    for (int64_t i = 0; i < n * d; i++)
        if (!std::isfinite(x[i])) return ORACLE_ERR_INVALID_ARG;
    const int64_t il = (int64_t)std::floor((1.0 - q) * (double)(n - 1));
    const int64_t iu = (int64_t)std::floor(q * (double)(n - 1));
    std::vector<float> col(n);
    for (int j = 0; j < d; j++) {
        for (int64_t i = 0; i < n; i++) col[i] = x[i * d + j];
        std::sort(col.begin(), col.end());
        const float lo = col[il], hi = col[iu];
        lower[j] = (lo == 0.0f) ? 0.0f : lo;  // +0 canonical zero (R-1)
        upper[j] = (hi == 0.0f) ? 0.0f : hi;
    }
    return ORACLE_OK;
}

int32_t oracle_l2w_weights(const float *lower, const float *upper, int32_t d, int32_t bits, int32_t *w) {
    if (!lower || !upper || !w || d < 1 || (bits != 4 && bits != 8)) return 0;
    std::vector<int> ww;
    const int W = l2w_weights(lower, upper, d, bits, ww);
    for (int j = 0; j < d; j++) w[j] = ww[j];
    return W;
}

int32_t oracle_encode_sq(const float *x, int64_t n, int32_t d, int32_t bits, const float *lower,
                         const float *upper, uint8_t *codes) {
    if (!x || !lower || !upper || !codes || n < 0 || d < 1 || (bits != 4 && bits != 8))
        return ORACLE_ERR_INVALID_ARG;
    const int64_t cb = oracle_code_bytes(d, bits);
    for (int64_t i = 0; i < n; i++) {
        uint8_t *c = codes + i * cb;
        std::memset(c, 0, (size_t)cb);
        for (int j = 0; j < d; j++) {
            int v = encode_value(x[i * d + j], lower[j], upper[j], bits);
            if (bits == 8)
                c[j] = (uint8_t)v;
            else
                c[j / 2] |= (uint8_t)(j % 2 == 0 ? v : (v << 4));
        }
    }
    return ORACLE_OK;
}

int32_t oracle_ip_weights(const float *q, int32_t d, const float *lower, const float *upper, int32_t *w) {
    if (!q || !lower || !upper || !w || d < 1) return ORACLE_ERR_INVALID_ARG;
    QueryOperand op = make_operand(q, d, 8, lower, upper, ORACLE_METRIC_IP);
    for (int j = 0; j < d; j++) w[j] = op.v[j];
    return ORACLE_OK;
}

int32_t oracle_tau_l(const float *q, const uint8_t *code, int32_t d, int32_t bits, const float *lower,
                     const float *upper, int32_t metric, int64_t *out) {
    if (!q || !code || !lower || !upper || !out || d < 1 || (bits != 4 && bits != 8) ||
        (metric != ORACLE_METRIC_L2 && metric != ORACLE_METRIC_IP && metric != ORACLE_METRIC_L2W))
        return ORACLE_ERR_INVALID_ARG;
    QueryOperand op = make_operand(q, d, bits, lower, upper, metric);
    *out = tau_l(op, code, d, bits, metric);
    return ORACLE_OK;
}

float oracle_tau_h(const float *q, const float *x, int32_t d, int32_t metric) { return tau_h(q, x, d, metric); }

double oracle_rerank_lower_bound(int64_t tau_l, int32_t d, const float *lower, const float *upper, int32_t bits) {
    return rerank_lower_bound(tau_l, d, min_step(lower, upper, d, bits));
}

int32_t oracle_search_batch(const float *base, const uint8_t *codes, const float *lower, const float *upper,
                            int64_t n, int32_t d, int32_t bits, const int64_t *row_ptr, const int32_t *adj,
                            int32_t degree, const int32_t *entry, int32_t n_entry, const float *queries,
                            int64_t nq, int32_t k, int32_t ef, int32_t rerank_n, int32_t metric,
                            int32_t *out_ids, float *out_dists, int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                            int32_t *expanded, int32_t max_hops, int32_t *pool_ids, int32_t *pool_tau,
                            int32_t nthreads) {
    return oracle_search_batch_labels(base, codes, lower, upper, n, d, bits, row_ptr, adj, degree, entry, n_entry,
                                      queries, nq, k, ef, rerank_n, metric, nullptr, 0, 0.0f, 0, out_ids, out_dists,
                                      hops, n_lp, n_hp, expanded, max_hops, pool_ids, pool_tau, nthreads);
}

int32_t oracle_search_batch_labels(const float *base, const uint8_t *codes, const float *lower, const float *upper,
                                   int64_t n, int32_t d, int32_t bits, const int64_t *row_ptr, const int32_t *adj,
                                   int32_t degree, const int32_t *entry, int32_t n_entry, const float *queries,
                                   int64_t nq, int32_t k, int32_t ef, int32_t rerank_n, int32_t metric,
                                   const float *labels, int32_t m_s, float alpha_s, int32_t adaptive,
                                   int32_t *out_ids, float *out_dists, int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                                   int32_t *expanded, int32_t max_hops, int32_t *pool_ids, int32_t *pool_tau,
                                   int32_t nthreads) {
    return oracle_search_batch_qlp(base, codes, lower, upper, n, d, bits, row_ptr, adj, degree, entry, n_entry,
                                   queries, nq, k, ef, rerank_n, metric, labels, m_s, alpha_s, adaptive, 0, 0, 0, 0,
                                   out_ids, out_dists, hops, n_lp, n_hp, expanded, max_hops, pool_ids, pool_tau,
                                   nthreads);
}

int32_t oracle_search_batch_qlp(const float *base, const uint8_t *codes, const float *lower, const float *upper,
                                int64_t n, int32_t d, int32_t bits, const int64_t *row_ptr, const int32_t *adj,
                                int32_t degree, const int32_t *entry, int32_t n_entry, const float *queries,
                                int64_t nq, int32_t k, int32_t ef, int32_t rerank_n, int32_t metric,
                                const float *labels, int32_t m_s, float alpha_s, int32_t adaptive,
                                int32_t qlp_hop, int32_t qlp_ef_low, int32_t qlp_feature, int64_t qlp_threshold,
                                int32_t *out_ids, float *out_dists, int32_t *hops, int32_t *n_lp, int32_t *n_hp,
                                int32_t *expanded, int32_t max_hops, int32_t *pool_ids, int32_t *pool_tau,
                                int32_t nthreads) {
    if (rerank_n == 0) rerank_n = ef;
    if (qlp_ef_low != 0 && (qlp_ef_low < k || qlp_ef_low > ef || qlp_hop < 0 || qlp_feature < 0 || qlp_feature > 2))
        return ORACLE_ERR_INVALID_ARG;
    if (!base || !codes || !lower || !upper || !adj || !entry || n < 1 || d < 1 || (bits != 4 && bits != 8) ||
        nq < 0 || (nq > 0 && (!queries || !out_ids || !out_dists)) || k < 1 || k > n || ef < 1 ||
        rerank_n < k || n_entry < 1 ||
        (metric != ORACLE_METRIC_L2 && metric != ORACLE_METRIC_IP && metric != ORACLE_METRIC_L2W) ||
        (!row_ptr && degree < 1) || (expanded && max_hops < 0))
        return ORACLE_ERR_INVALID_ARG;
    if (!tau_fits_int32(d, bits, metric)) return ORACLE_ERR_OVERFLOW;
    Index ix{base, codes, lower, upper, n, d, bits, oracle_code_bytes(d, bits), row_ptr, adj, degree, {}};
    ix.labels = labels;
    ix.m_s = m_s;
    ix.alpha_s = alpha_s;
    if (adaptive && metric != ORACLE_METRIC_L2) return ORACLE_ERR_INVALID_ARG;
    ix.adaptive = adaptive != 0;
    ix.delta_min = min_step(lower, upper, d, bits);
    ix.qlp_hop = qlp_hop;
    ix.qlp_ef_low = qlp_ef_low;
    ix.qlp_feature = qlp_feature;
    ix.qlp_threshold = qlp_threshold;
    for (int t = 0; t < n_entry; t++) {
        if (entry[t] < 0 || entry[t] >= n) return ORACLE_ERR_INVALID_ARG;
        ix.entry.push_back(entry[t]);
    }
    std::sort(ix.entry.begin(), ix.entry.end());
    ix.entry.erase(std::unique(ix.entry.begin(), ix.entry.end()), ix.entry.end());
    const int64_t nnz = row_ptr ? row_ptr[n] : n * (int64_t)degree;
    if (row_ptr) {
        if (row_ptr[0] != 0) return ORACLE_ERR_INVALID_ARG;
        for (int64_t i = 0; i < n; i++)
            if (row_ptr[i + 1] < row_ptr[i]) return ORACLE_ERR_INVALID_ARG;
    }
    for (int64_t t = 0; t < nnz; t++)
        if (adj[t] < -1 || adj[t] >= n) return ORACLE_ERR_INVALID_ARG;

    const int64_t cap = std::max(ef, rerank_n);
    auto run = [&](int64_t q0, int64_t q1) {
        for (int64_t qi = q0; qi < q1; qi++) {
            QueryResult r = search_one(ix, queries + qi * d, k, ef, rerank_n, metric);
            for (int t = 0; t < k; t++) {
                out_ids[qi * k + t] = r.ids[t];
                out_dists[qi * k + t] = r.dists[t];
            }
            if (hops) hops[qi] = r.hops;
            if (n_lp) n_lp[qi] = r.n_lp;
            if (n_hp) n_hp[qi] = r.n_hp;
            if (expanded)
                for (int t = 0; t < max_hops; t++)
                    expanded[qi * max_hops + t] = t < (int)r.expanded.size() ? r.expanded[t] : -1;
            for (int64_t t = 0; t < cap; t++) {
                bool has = t < (int64_t)r.pool.size();
                if (pool_ids) pool_ids[qi * cap + t] = has ? r.pool[t].id : -1;
                if (pool_tau) pool_tau[qi * cap + t] = has ? (int32_t)r.pool[t].tau : INT32_MAX;
            }
        }
    };
    if (nthreads <= 1 || nq < 2) {
        run(0, nq);
    } else {
        std::vector<std::thread> th;
        int64_t per = (nq + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; t++) {
            int64_t a = t * per, b = std::min(nq, a + per);
            if (a < b) th.emplace_back(run, a, b);
        }
        for (auto &x : th) x.join();
    }
    return ORACLE_OK;
}

}  // extern "C"
