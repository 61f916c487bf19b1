// api.cu -- the C ABI of include/vsag.h: validation, ownership, orchestration.
// No C++ exception crosses this boundary; every entry point returns a vsag_status.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "vsag_internal.cuh"


using namespace vsag;

struct vsag_index {
    Index ix;
};

namespace {

thread_local std::string g_last_error;

vsag_status fail(vsag_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

vsag_status cuda_fail(cudaError_t e, const char *what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(VSAG_ERR_OOM, "%s: out of device memory", what);
    }
    return fail(VSAG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr, what)                                  \
    do {                                                \
        cudaError_t e_ = (expr);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline int64_t code_bytes(int d, int bits) { return bits == 8 ? d : (d + 1) / 2; }

// NEXT-1b weight scale W = min(8192, floor((2^31 - 1) / (d (2^b - 1)^2))): sum_j w_j (2^b - 1)^2 < 2^31.
int l2w_scale(int d, int bits) {
    const int64_t levels = (1 << bits) - 1;
    return (int)std::min<int64_t>(8192, (((int64_t)1 << 31) - 1) / ((int64_t)d * levels * levels));
}

bool tau_fits_int32(int d, int bits, int metric) {
    const int64_t levels = (1 << bits) - 1;
    if (metric == VSAG_METRIC_L2) return (int64_t)d * levels * levels < ((int64_t)1 << 31);
    if (metric == VSAG_METRIC_L2W) return l2w_scale(d, bits) >= 1;
    return (int64_t)d * 127 * levels < ((int64_t)1 << 31);
}

int next_pow2(int v) {
    int r = 1;
    while (r < v) r <<= 1;
    return r;
}

void free_index(Index &ix) {
    cudaFree(ix.codes_owned);
    cudaFree(ix.adj);
    cudaFree(ix.rows);
    cudaFree(ix.entry);
    cudaFree(ix.seed_codes);
    cudaFree(ix.seed_op);
    cudaFree(ix.l2w);
    cudaFree(ix.labels);
    cudaFree(ix.prs_blk);
    cudaFree(ix.prs_codes);
    cudaFreeHost(ix.err_host);
    ix = Index();
}

// Synchronous read of a device error flag.
cudaError_t read_flag(const int *flag, cudaStream_t s, int *out) {
    cudaError_t e = cudaMemcpyAsync(out, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(s);
}

}  // namespace

// Stream-ordered scratch comes from a memory pool owned by the library (one per device,
// created on first use, release threshold UINT64_MAX so freed scratch stays cached between
// calls).  The process-wide default pool of the device is never modified.
cudaError_t vsag::scratch_alloc(void **p, size_t bytes, int device, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[128] = {};
    if (device < 0 || device >= 128) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> g(mu);
        if (!pools[device]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = device;
            cudaError_t e = cudaMemPoolCreate(&pools[device], &props);
            if (e != cudaSuccess) {
                pools[device] = nullptr;
                return e;
            }
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = pools[device];
    }
#ifdef VSAG_DEFAULT_POOL
    (void)pool;
    return cudaMallocAsync(p, bytes, s);
#else
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
#endif
}

namespace {

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Error flags of an index: mapped pinned host memory (ix.err_host; ix.err is its device
// alias), 1 = a tensor-core completion wait of the seed contraction timed out
// (seed_umma.cuh).  Synchronises `s` (the calls that use it synchronise anyway), then reads
// the flag on the host: no copy.
vsag_status check_index_flags(const Index &ix, cudaStream_t s, const char *who) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, who);
    const int f = *reinterpret_cast<volatile int *>(ix.err_host);
    if (f & 1)
        return fail(VSAG_ERR_CUDA, "%s: tensor-core completion timeout in the seed contraction (outputs invalid)", who);
    if (f) return fail(VSAG_ERR_CUDA, "%s: device bounds check failed (VSAG_CHECKS build), code %d", who, f);
    return VSAG_OK;
}

}  // namespace

extern "C" {

int64_t vsag_code_bytes(int32_t d, int32_t bits) { return code_bytes(d, bits); }

const char *vsag_last_error(void) { return g_last_error.c_str(); }

vsag_status vsag_encode_sq(const float *x, int64_t n, int32_t d, int32_t bits, int32_t train, float *lower,
                           float *upper, uint8_t *codes, void *stream) {
    g_last_error.clear();
    if (n < 0 || d < 1 || (bits != 4 && bits != 8))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_encode_sq: need n >= 0, d >= 1, bits in {4, 8} (n=%lld d=%d bits=%d)",
                    (long long)n, d, bits);
    if (!lower || !upper || (n > 0 && (!x || !codes)))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_encode_sq: null pointer");
    if (train && n < 1) return fail(VSAG_ERR_INVALID_ARG, "vsag_encode_sq: training needs n >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    if (train) {
        uint8_t *scratch = nullptr;
        const size_t bytes = (size_t)d * 8 + 16;
        CK(scratch_alloc((void **)&scratch, bytes, current_device(), s), "vsag_encode_sq: scratch");
        uint32_t *omin = reinterpret_cast<uint32_t *>(scratch);
        uint32_t *omax = omin + d;
        int *bad = reinterpret_cast<int *>(omax + d);
        cudaError_t e = cudaMemsetAsync(omin, 0xff, (size_t)d * 4, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(omax, 0, (size_t)d * 4 + sizeof(int), s);
        if (e == cudaSuccess) e = launch_sq_minmax(x, n, d, omin, omax, bad, s);
        int hbad = 0;
        if (e == cudaSuccess) e = read_flag(bad, s, &hbad);
        if (e == cudaSuccess && !hbad) e = launch_sq_finalize(omin, omax, d, lower, upper, s);
        cudaFreeAsync(scratch, s);
        if (e != cudaSuccess) return cuda_fail(e, "vsag_encode_sq: train");
        if (hbad) return fail(VSAG_ERR_INVALID_ARG, "vsag_encode_sq: non-finite value in x");
    }
    CK(launch_sq_encode(x, n, d, bits, lower, upper, codes, code_bytes(d, bits), s), "vsag_encode_sq: encode");
    return VSAG_OK;
}

vsag_status vsag_train_sq(const float *x, int64_t n, int32_t d, double quantile, float *lower, float *upper,
                          void *stream) {
    g_last_error.clear();
    if (!x || !lower || !upper || n < 1 || n > 0xffffffffLL || d < 1)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_train_sq: need x/lower/upper, 1 <= n < 2^32, d >= 1");
    if (!(quantile > 0.5 && quantile <= 1.0))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_train_sq: quantile must be in (0.5, 1]");
    cudaStream_t s = (cudaStream_t)stream;
    // order statistics of the truncated range (ranks in fp64, no interpolation)
    const int64_t il = (int64_t)std::floor((1.0 - quantile) * (double)(n - 1));
    const int64_t iu = (int64_t)std::floor(quantile * (double)(n - 1));
    const size_t qwords = quantile < 1.0 ? train_quantile_scratch_words(d) : 0;
    uint8_t *scratch = nullptr;
    CK(scratch_alloc((void **)&scratch, (size_t)d * 8 + 16 + qwords * 4, current_device(), s), "vsag_train_sq: scratch");
    uint32_t *omin = reinterpret_cast<uint32_t *>(scratch);
    uint32_t *omax = omin + d;
    int *bad = reinterpret_cast<int *>(omax + d);
    cudaError_t e = cudaMemsetAsync(omin, 0xff, (size_t)d * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(omax, 0, (size_t)d * 4 + sizeof(int), s);
    if (e == cudaSuccess) e = launch_sq_minmax(x, n, d, omin, omax, bad, s);  // also the finiteness check
    int hbad = 0;
    if (e == cudaSuccess) e = read_flag(bad, s, &hbad);
    if (e == cudaSuccess && !hbad) {
        if (quantile == 1.0)
            e = launch_sq_finalize(omin, omax, d, lower, upper, s);
        else
            e = launch_train_quantile(x, n, d, il, iu, lower, upper,
                                      reinterpret_cast<uint32_t *>(scratch + (size_t)d * 8 + 16), s);
    }
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "vsag_train_sq");
    if (hbad) return fail(VSAG_ERR_INVALID_ARG, "vsag_train_sq: non-finite value in x");
    return VSAG_OK;
}

vsag_status vsag_index_load(const float *base, const uint8_t *codes, const float *lower, const float *upper,
                            int64_t n, int32_t d, int32_t bits, const int64_t *row_ptr, const int32_t *adj,
                            int32_t degree, const int32_t *entry, int32_t n_entry, int32_t layout, void *stream,
                            vsag_index **out) {
    g_last_error.clear();
    if (!out) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: out is NULL");
    *out = nullptr;
    if (!base || !codes || !lower || !upper || !adj || !entry)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: null pointer");
    if (n < 1 || n > 0x7fffffffLL || d < 1 || (bits != 4 && bits != 8) || n_entry < 1)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: need 1 <= n < 2^31, d >= 1, bits in {4,8}, n_entry >= 1");
    if (degree < 1) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: degree must be >= 1");
    if (degree > VSAG_MAX_DEGREE) return fail(VSAG_ERR_UNSUPPORTED, "vsag_index_load: degree %d > %d", degree, VSAG_MAX_DEGREE);
    if (layout != VSAG_LAYOUT_TABLE && layout != VSAG_LAYOUT_COLOCATED)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: unknown layout %d", layout);
    if (!aligned16(base)) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: base must be 16-byte aligned");
    const int cb = (int)code_bytes(d, bits);
    // code stride: whole 16-byte chunks; up to 128 B padded to a power of two of them, so the
    // search kernel's common-case variant (codes filling all of its lanes' 16-byte chunks)
    // applies and codes sit on aligned 32-byte sectors: SQ4 at d = 96 (C4) goes 48 -> 64 B and
    // searches 21-24% faster at 2M rows (neutral at 10M, where HBM latency dominates).
    // (Padding C2's 480-byte codes to 512 measured 7-25% slower.)
    int cbp = (cb + 15) / 16 * 16;
    if (cbp <= 128) {
        int p2 = 16;
        while (p2 < cbp) p2 <<= 1;
        cbp = p2;
    }
    if (cbp > VSAG_MAX_CODE_BYTES)
        return fail(VSAG_ERR_UNSUPPORTED, "vsag_index_load: code bytes %d > %d", cb, VSAG_MAX_CODE_BYTES);
    if (!tau_fits_int32(d, bits, VSAG_METRIC_L2))
        return fail(VSAG_ERR_OVERFLOW, "vsag_index_load: d=%d with %d-bit codes can overflow int32 tau_l", d, bits);
    cudaStream_t s = (cudaStream_t)stream;

    // entry set: sorted, deduplicated, range-checked (R-11)
    std::vector<int32_t> h_entry(n_entry);
    CK(cudaMemcpyAsync(h_entry.data(), entry, sizeof(int32_t) * n_entry, cudaMemcpyDeviceToHost, s), "entry copy");
    CK(cudaStreamSynchronize(s), "entry copy");
    for (int32_t v : h_entry)
        if (v < 0 || v >= n) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: entry id %d out of range", v);
    std::sort(h_entry.begin(), h_entry.end());
    h_entry.erase(std::unique(h_entry.begin(), h_entry.end()), h_entry.end());

    vsag_index *h = new (std::nothrow) vsag_index();
    if (!h) return fail(VSAG_ERR_OOM, "vsag_index_load: host allocation");
    Index &ix = h->ix;
    cudaGetDevice(&ix.device);
    ix.n = n;
    ix.d = d;
    ix.bits = bits;
    ix.cb = cb;
    ix.cbp = cbp;
    ix.degree = degree;
    ix.layout = layout;
    ix.base = base;
    ix.lower = lower;
    ix.upper = upper;
    ix.n_entry = (int)h_entry.size();
    int *flag = nullptr;
    auto bail = [&](vsag_status st) {
        cudaStreamSynchronize(s);
        cudaFree(flag);
        free_index(ix);
        delete h;
        return st;
    };
#define CKB(expr, what)                                          \
    do {                                                         \
        cudaError_t e_ = (expr);                                 \
        if (e_ != cudaSuccess) return bail(cuda_fail(e_, what)); \
    } while (0)

    CKB(cudaMalloc((void **)&flag, sizeof(int)), "flag");
    CKB(cudaHostAlloc((void **)&ix.err_host, sizeof(int), cudaHostAllocMapped), "error flag");
    *ix.err_host = 0;
    CKB(cudaHostGetDevicePointer((void **)&ix.err, ix.err_host, 0), "error flag");
    CKB(cudaMemsetAsync(flag, 0, sizeof(int), s), "flag");
    // padded fixed-degree adjacency
    CKB(cudaMalloc((void **)&ix.adj, (size_t)n * degree * 4), "adjacency");
    ix.owned_bytes += (int64_t)n * degree * 4;
    if (row_ptr) {
        CKB(launch_csr_to_padded(row_ptr, adj, n, degree, ix.adj, flag, s), "csr_to_padded");
    } else {
        CKB(cudaMemcpyAsync(ix.adj, adj, (size_t)n * degree * 4, cudaMemcpyDeviceToDevice, s), "adjacency copy");
        CKB(launch_check_adj(ix.adj, n * (int64_t)degree, n, flag, s), "check_adj");
    }
    int hflag = 0;
    CKB(read_flag(flag, s, &hflag), "adjacency check");
    if (hflag & 2) return bail(fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: CSR row longer than degree or row_ptr not monotone"));
    if (hflag & 1) return bail(fail(VSAG_ERR_INVALID_ARG, "vsag_index_load: adjacency id out of [-1, n)"));
    CKB(launch_row_dups(ix.adj, n, degree, flag, s), "row_dups");
    CKB(read_flag(flag, s, &hflag), "row_dups");
    ix.row_dups = (hflag & 4) ? 1 : 0;

    // codes with a 16-byte stride (borrowed when already laid out that way)
    if (cb == cbp && (reinterpret_cast<uintptr_t>(codes) & 15) == 0) {
        ix.codes = codes;
    } else {
        CKB(cudaMalloc((void **)&ix.codes_owned, (size_t)n * cbp), "padded codes");
        ix.owned_bytes += n * (int64_t)cbp;
        CKB(launch_copy_pad_codes(codes, n, cb, cbp, ix.codes_owned, s), "copy_pad_codes");
        ix.codes = ix.codes_owned;
    }
    // entry set + its code block
    CKB(cudaMalloc((void **)&ix.entry, sizeof(int32_t) * ix.n_entry), "entry");
    CKB(cudaMemcpyAsync(ix.entry, h_entry.data(), sizeof(int32_t) * ix.n_entry, cudaMemcpyHostToDevice, s), "entry");
    CKB(cudaMalloc((void **)&ix.seed_codes, (size_t)ix.n_entry * cbp), "seed codes");
    ix.owned_bytes += (int64_t)ix.n_entry * (4 + cbp);
    CKB(launch_gather_codes(ix.entry, ix.n_entry, ix.codes, cbp, ix.seed_codes, s), "gather_codes");
    {
        const size_t ob = seed_operand_bytes(ix.n_entry, cbp, bits);
        CKB(cudaMalloc((void **)&ix.seed_op, ob), "seed operand");
        ix.owned_bytes += (int64_t)ob;
        CKB(launch_seed_operand(ix.seed_codes, ix.n_entry, cbp, bits, ix.seed_op, s), "seed operand");
    }
    // NEXT-3: the re-rank bound needs the base inside the trained range; smallest step
    {
        CKB(cudaMemsetAsync(flag, 0, sizeof(int), s), "range check");
        CKB(launch_range_check(base, n, d, lower, upper, flag, s), "range check");
        int hout = 0;
        CKB(read_flag(flag, s, &hout), "range check");
        ix.base_in_range = hout ? 0 : 1;
        std::vector<float> hl(d), hu(d);
        CKB(cudaMemcpy(hl.data(), lower, (size_t)d * 4, cudaMemcpyDeviceToHost), "range");
        CKB(cudaMemcpy(hu.data(), upper, (size_t)d * 4, cudaMemcpyDeviceToHost), "range");
        const double levels = (double)((1 << bits) - 1);
        for (int j = 0; j < d; j++) {
            const double r = (double)(hu[j] - hl[j]);
            if (r > 0.0 && (ix.delta_min == 0.0 || r / levels < ix.delta_min)) ix.delta_min = r / levels;
        }
    }
    // weights of the weighted code-space L2 (NEXT-1b), one per (padded) dimension
    ix.l2w_W = l2w_scale(d, bits);
    if (ix.l2w_W >= 1) {
        const int dims_padded = cbp * (bits == 8 ? 1 : 2);
        CKB(cudaMalloc((void **)&ix.l2w, (size_t)dims_padded * 4), "l2w weights");
        ix.owned_bytes += (int64_t)dims_padded * 4;
        CKB(launch_l2w_weights(lower, upper, d, dims_padded, ix.l2w_W, ix.l2w, s), "l2w weights");
    }
    // layout 1: PRS rows [ids | neighbour codes]
    if (layout == VSAG_LAYOUT_COLOCATED) {
        ix.ids_bytes = (degree * 4 + 15) / 16 * 16;
        ix.row_bytes = ix.ids_bytes + (int64_t)degree * cbp;
        CKB(cudaMalloc((void **)&ix.rows, (size_t)(n * ix.row_bytes)), "layout-1 rows");
        ix.owned_bytes += n * ix.row_bytes;
        CKB(launch_layout_build(ix.adj, ix.codes, n, degree, cbp, ix.ids_bytes, ix.row_bytes, ix.rows, s), "layout_build");
        CKB(cudaStreamSynchronize(s), "layout_build");
        cudaFree(ix.adj);  // the rows carry the ids
        ix.adj = nullptr;
        ix.owned_bytes -= (int64_t)n * degree * 4;
    }
    CKB(cudaStreamSynchronize(s), "index load");
    cudaFree(flag);
    *out = h;
    return VSAG_OK;
#undef CKB
}

vsag_status vsag_index_get_info(const vsag_index *h, vsag_index_info *info) {
    g_last_error.clear();
    if (!h || !info) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_get_info: null pointer");
    const Index &ix = h->ix;
    info->n = ix.n;
    info->d = ix.d;
    info->bits = ix.bits;
    info->code_bytes = ix.cb;
    info->code_stride = ix.cbp;
    info->degree = ix.degree;
    info->layout = ix.layout;
    info->n_entry = ix.n_entry;
    info->device_bytes = ix.owned_bytes;
    info->prs_nodes = ix.prs_nodes;
    info->prs_bytes = ix.prs_nodes * (int64_t)ix.degree * ix.cbp;
    return VSAG_OK;
}

vsag_status vsag_index_set_prs(vsag_index *h, double delta, void *stream) {
    g_last_error.clear();
    if (!h) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_set_prs: null index");
    Index &ix = h->ix;
    if (!(delta >= 0.0 && delta <= 1.0)) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_set_prs: delta must be in [0, 1]");
    if (ix.layout != VSAG_LAYOUT_TABLE)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_index_set_prs: needs a VSAG_LAYOUT_TABLE index");
    DeviceGuard g(ix.device);
    cudaStream_t s = (cudaStream_t)stream;
    if (ix.prs_blk) {
        cudaFree(ix.prs_blk);
        cudaFree(ix.prs_codes);
        ix.owned_bytes -= ix.n * 4 + ix.prs_nodes * (int64_t)ix.degree * ix.cbp;
        ix.prs_blk = nullptr;
        ix.prs_codes = nullptr;
        ix.prs_nodes = 0;
    }
    const int64_t count = (int64_t)std::llround(delta * (double)ix.n);
    if (count == 0) return VSAG_OK;
    // in-degrees, then the count nodes of highest in-degree (ties: lower id)
    int32_t *indeg = nullptr;
    CK(cudaMalloc((void **)&indeg, (size_t)ix.n * 4), "vsag_index_set_prs: in-degree");
    cudaError_t e = cudaMemsetAsync(indeg, 0, (size_t)ix.n * 4, s);
    if (e == cudaSuccess) e = launch_in_degree(ix.adj, ix.n * (int64_t)ix.degree, indeg, s);
    std::vector<int32_t> hdeg(ix.n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hdeg.data(), indeg, (size_t)ix.n * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(indeg);
    if (e != cudaSuccess) return cuda_fail(e, "vsag_index_set_prs: in-degree");
    std::vector<int32_t> order(ix.n);
    for (int64_t i = 0; i < ix.n; i++) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return hdeg[a] > hdeg[b]; });
    order.resize(count);
    std::sort(order.begin(), order.end());  // blocks in id order
    std::vector<int32_t> blk(ix.n, -1);
    for (int64_t b = 0; b < count; b++) blk[order[b]] = (int32_t)b;
    int32_t *dnodes = nullptr;
    CK(cudaMalloc((void **)&ix.prs_blk, (size_t)ix.n * 4), "vsag_index_set_prs: block map");
    e = cudaMalloc((void **)&ix.prs_codes, (size_t)count * ix.degree * ix.cbp);
    if (e == cudaSuccess) e = cudaMalloc((void **)&dnodes, (size_t)count * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ix.prs_blk, blk.data(), (size_t)ix.n * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dnodes, order.data(), (size_t)count * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_prs_build(ix.adj, ix.codes, dnodes, count, ix.degree, ix.cbp, ix.prs_codes, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(dnodes);
    if (e != cudaSuccess) {
        cudaFree(ix.prs_blk);
        cudaFree(ix.prs_codes);
        ix.prs_blk = nullptr;
        ix.prs_codes = nullptr;
        return cuda_fail(e, "vsag_index_set_prs");
    }
    ix.prs_nodes = count;
    ix.owned_bytes += ix.n * 4 + count * (int64_t)ix.degree * ix.cbp;
    return VSAG_OK;
}

vsag_status vsag_index_free(vsag_index *h) {
    g_last_error.clear();
    if (!h) return VSAG_OK;
    DeviceGuard g(h->ix.device);
    cudaDeviceSynchronize();
    free_index(h->ix);
    delete h;
    return VSAG_OK;
}

vsag_status vsag_index_set_labels(vsag_index *h, const int64_t *row_ptr, const float *labels, void *stream) {
    g_last_error.clear();
    if (!h || !labels) return fail(VSAG_ERR_INVALID_ARG, "vsag_index_set_labels: null pointer");
    Index &ix = h->ix;
    DeviceGuard g(ix.device);
    cudaStream_t s = (cudaStream_t)stream;
    float *dst = nullptr;
    int *flag = nullptr;
    CK(cudaMalloc((void **)&dst, (size_t)ix.n * ix.degree * 4), "vsag_index_set_labels: labels");
    cudaError_t e = cudaMalloc((void **)&flag, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(int), s);
    if (e == cudaSuccess) e = launch_pad_labels(row_ptr, labels, ix.n, ix.degree, dst, flag, s);
    int hflag = 0;
    if (e == cudaSuccess) e = read_flag(flag, s, &hflag);
    cudaFree(flag);
    if (e != cudaSuccess || hflag) {
        cudaFree(dst);
        if (e != cudaSuccess) return cuda_fail(e, "vsag_index_set_labels");
        return fail(VSAG_ERR_INVALID_ARG, (hflag & 2) ? "vsag_index_set_labels: CSR row longer than degree"
                                                      : "vsag_index_set_labels: NaN label");
    }
    if (ix.labels) {
        cudaFree(ix.labels);
        ix.owned_bytes -= ix.n * (int64_t)ix.degree * 4;
    }
    ix.labels = dst;
    ix.owned_bytes += ix.n * (int64_t)ix.degree * 4;
    return VSAG_OK;
}

// visited_kind 0 (auto): the shared-memory table (u16 buckets where a 14-bit tag identifies
// an id, else u32 probing), unless the exact device-memory bitset lets clearly more warps
// reside for the batch at hand and clearing n bits per query is small next to the query's
// gathers (estimated as ef hops of degree / 5 new codes plus the id row).  With the
// residency-first auto table size (check_search) the table rarely limits residency, so this
// keeps the table in all of the measured configs (profiles/r02_config_sweep_v7.json: a small
// forgetful table beats the bitset by 17-25% at C3, ef 256 / 512); it still switches for
// explicitly large visited_slots.
int auto_visited_kind(const Index &ix, int64_t nq, int ef, int L, int R, int H) {
    const int table = visited_u16(H, ix.n) ? 2 : 3;
    int smem_sm = 0, reserve = 0, sms = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ix.device);
    cudaDeviceGetAttribute(&reserve, cudaDevAttrReservedSharedMemoryPerBlock, ix.device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix.device);
    if (smem_sm <= 0 || sms <= 0) return table;
    const int layout = ix.prs_blk ? 2 : ix.layout;
    const double reg_warps = 36.0;  // search_kernel: 56 registers (__launch_bounds__(128, 9))
    auto warps = [&](int kind) {    // resident warps for this batch, 2-warp CTAs
        const double per_warp = (double)search_smem_per_warp(L, R, H, kind, ix.degree, layout) + reserve / 2.0;
        const double per_sm = std::min(reg_warps, std::floor(smem_sm / per_warp));
        return std::min((double)nq, per_sm * sms);
    };
    const double clear = (double)ix.n / 8.0;
    const double gather = (double)ef * (ix.degree / 5.0 * ix.cbp + 4.0 * ix.degree);
    if (warps(4) >= 1.25 * warps(table) && clear * 4.0 <= gather) return 4;
    return table;
}

// Validation shared by the device and host entry points (nothing is allocated or launched
// before it passes).  Fills the derived sizes.
struct SearchCfg {
    int k, ef, R, L, H, wpb, metric, vkind;
};

vsag_status check_search(const Index &ix, int64_t nq, const vsag_search_params *sp, SearchCfg *c) {
    const int k = sp->k, ef = sp->ef, metric = sp->metric;
    const int R = sp->rerank_n ? sp->rerank_n : ef;
    if (nq < 0) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: nq < 0");
    if (nq > VSAG_MAX_BATCH)
        return fail(VSAG_ERR_UNSUPPORTED, "vsag_search_batch: nq = %lld > %lld per call", (long long)nq,
                    (long long)VSAG_MAX_BATCH);
    if (k < 1 || k > ix.n) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: need 1 <= k <= n (k=%d)", k);
    if (ef < 1) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: ef must be >= 1");
    if (R < k) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: rerank_n (%d) must be >= k (%d)", R, k);
    const int L = std::max(ef, R);
    if (L > VSAG_MAX_POOL) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: max(ef, rerank_n) = %d > %d", L, VSAG_MAX_POOL);
    if (metric != VSAG_METRIC_L2 && metric != VSAG_METRIC_IP && metric != VSAG_METRIC_L2W)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: unknown metric %d", metric);
    if (!tau_fits_int32(ix.d, ix.bits, metric)) return fail(VSAG_ERR_OVERFLOW, "vsag_search_batch: int32 tau_l overflow");
    const int code_lanes = sp->code_lanes;
    if (code_lanes != 0 && (code_lanes < 4 || code_lanes > 32 || (code_lanes & (code_lanes - 1))))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: code_lanes must be 0 or a power of two in [4, 32]");
    if (sp->qlp_ef_low != 0) {
        if (sp->qlp_ef_low < k || sp->qlp_ef_low > ef || sp->qlp_hop < 0)
            return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: QLP needs k <= qlp_ef_low <= ef and qlp_hop >= 0");
        if (sp->qlp_feature == 0)
            return fail(VSAG_ERR_UNSUPPORTED, "vsag_search_batch: QLP feature 0 (points scanned) is not exact under "
                                              "the forgetful visited cache; use feature 1 or 2");
        if (sp->qlp_feature != 1 && sp->qlp_feature != 2)
            return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: qlp_feature must be 1 or 2");
    }
    if (sp->rerank_adaptive && (metric != VSAG_METRIC_L2 || !ix.base_in_range))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: rerank_adaptive needs metric L2 and every base value "
                                          "inside [lower, upper]");
    if (sp->max_degree < 0) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: max_degree must be >= 0");
    if (!(sp->alpha_s >= 0.0f)) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: alpha_s must be >= 0");
    if (sp->alpha_s > 0.0f && !ix.labels)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: alpha_s needs edge labels (vsag_index_set_labels)");
    int H = sp->visited_slots;
    if (H == 0) {
        // auto: 12 slots per window entry (a query evaluates ~ 12 ef ids at degree 32), but resident
        // warps come first: the table is halved while it costs more than 15% of the warps that a
        // 1024-slot table would let reside for this batch (measured: C1 at ef 192 / 256 is 24% / 12%
        // faster with 2048 slots and 34 / 32 warps per SM than with 4096 slots and 20; C4's u32
        // table 26% faster with 1024 slots than with 2048), and doubled (up to 4096) while that
        // costs no resident warp (C4 at ef 32 / 64: 2048 u16 slots, which keeps the search on its
        // lazy-pool path).  A forgetful table never changes results.
        H = std::min(16384, std::max(1024, next_pow2(12 * ef)));
        int smem_sm = 0, reserve = 0, sms = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ix.device);
        cudaDeviceGetAttribute(&reserve, cudaDevAttrReservedSharedMemoryPerBlock, ix.device);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix.device);
        const int layout = ix.prs_blk ? 2 : ix.layout;
        auto warps = [&](int h) {  // resident warps of this batch with an h-slot table (2-warp CTAs)
            const double per_warp =
                (double)search_smem_per_warp(L, R, h, visited_u16(h, ix.n) ? 2 : 3, ix.degree, layout) + reserve / 2.0;
            return std::min((double)std::max<int64_t>(nq, 1), std::min(36.0, std::floor(smem_sm / per_warp)) * sms);
        };
        if (smem_sm > 0 && sms > 0) {
            const double w1 = warps(1024);
            while (H > 1024 && warps(H) < 0.85 * w1) H /= 2;
            while (H < 4096 && warps(2 * H) >= warps(H)) H *= 2;
        }
    }
    if (H < 256 || H > (1 << 16) || (H & (H - 1)))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: visited_slots must be a power of two in [256, 65536]");
    const int wpb = sp->warps_per_block ? sp->warps_per_block : 2;
    if (wpb < 1 || wpb > 4) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: warps_per_block must be in [1, 4]");
    int vk = sp->visited_kind;
    if (vk != 0 && vk != 2 && vk != 3 && vk != 4)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: visited_kind must be 0, 2, 3 or 4");
    if (vk == 2 && !visited_u16(H, ix.n))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: visited_kind 2 (u16 tags) cannot identify %lld ids with "
                                          "%d slots", (long long)ix.n, H);
    if (vk == 0) vk = auto_visited_kind(ix, nq, ef, L, R, H);
    *c = SearchCfg{k, ef, R, L, H, wpb, metric, vk};
    return VSAG_OK;
}

vsag_status vsag_search_batch_ex(const vsag_index *h, const float *queries, int64_t nq, const vsag_search_params *sp,
                                 int32_t *out_ids, float *out_dists, vsag_trace *trace, vsag_timing *timing,
                                 void *stream) {
    g_last_error.clear();
    if (!h || !sp) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: null index or params");
    const Index &ix = h->ix;
    SearchCfg cfg;
    {
        const vsag_status st = check_search(ix, nq, sp, &cfg);
        if (st != VSAG_OK) return st;
    }
    if (nq > 0 && (!queries || !out_ids || !out_dists)) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: null pointer");
    if (nq > 0 && !aligned16(queries)) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: queries must be 16-byte aligned");
    const int k = cfg.k, ef = cfg.ef, metric = cfg.metric, R = cfg.R, L = cfg.L, H = cfg.H;
    int wpb = cfg.wpb;
    const int code_lanes = sp->code_lanes;
    if (trace && trace->expanded && trace->max_hops < 0)
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch: trace.max_hops < 0");
    if (timing) std::memset(timing, 0, sizeof(*timing));
    if (nq == 0) return VSAG_OK;

    DeviceGuard g(ix.device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t per_warp = search_smem_per_warp(L, R, H, cfg.vkind, ix.degree, ix.prs_blk ? 2 : ix.layout);
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix.device);
    const size_t cta = mode_w(mode_of(metric, ix.bits)) ? (size_t)(ix.cbp * (ix.bits == 8 ? 1 : 2) * 4 + 15) / 16 * 16 : 0;
    while (wpb > 1 && cta + (size_t)wpb * per_warp > (size_t)max_smem) wpb--;
    if (cta + per_warp > (size_t)max_smem)
        return fail(VSAG_ERR_UNSUPPORTED, "vsag_search_batch: %zu B of shared memory per query exceeds %d", per_warp, max_smem);

    const int mode = mode_of(metric, ix.bits);
    const int op_stride = (ix.cbp / 4) * op_words_per_code_word(mode);
    const size_t op_bytes = (size_t)nq * op_stride * 4;
    const size_t tau_bytes = (size_t)nq * ix.n_entry * 4;
    const size_t init_bytes = (size_t)nq * L * 8, psz_bytes = (size_t)nq * 4;
    const size_t op_off = 256, tau_off = op_off + (op_bytes + 255) / 256 * 256;
    const size_t init_off = tau_off + (tau_bytes + 255) / 256 * 256;
    const size_t psz_off = init_off + (init_bytes + 255) / 256 * 256;
    uint8_t *scratch = nullptr;
    CK(scratch_alloc((void **)&scratch, psz_off + psz_bytes, ix.device, s), "vsag_search_batch: scratch");

    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    if (timing)
        for (auto &e : ev) cudaEventCreate(&e);
    SearchArgs a{};
    a.ix = &ix;
    a.queries = queries;
    a.op = reinterpret_cast<uint32_t *>(scratch + op_off);
    a.op_stride_words = op_stride;
    a.seed_tau = reinterpret_cast<int32_t *>(scratch + tau_off);
    a.init_keys = reinterpret_cast<uint64_t *>(scratch + init_off);
    a.init_psz = reinterpret_cast<int *>(scratch + psz_off);
    a.nq = nq;
    a.k = k;
    a.ef = ef;
    a.rerank_n = R;
    a.L = L;
    a.metric = metric;
    a.mode = mode;
    a.visited_slots = H;
    a.visited_kind = cfg.vkind;
    a.code_lanes = code_lanes;
    a.m_s = sp->max_degree;
    a.adaptive = sp->rerank_adaptive ? 1 : 0;
    a.qlp_ef_low = sp->qlp_ef_low;
    a.qlp_hop = sp->qlp_hop;
    a.qlp_feature = sp->qlp_feature;
    a.qlp_threshold = sp->qlp_threshold;
    a.alpha_s = sp->alpha_s;
    a.out_ids = out_ids;
    a.out_dists = out_dists;
    if (trace) {
        a.trace = *trace;
        a.has_trace = 1;
    }
    a.counter = reinterpret_cast<unsigned int *>(scratch);
    SearchLaunch info{};
    cudaError_t e = cudaMemsetAsync(scratch, 0, 256, s);
    if (timing && e == cudaSuccess) e = cudaEventRecord(ev[0], s);
    if (e == cudaSuccess)
        e = launch_query_prep(queries, nq, ix.d, ix.bits, metric, ix.lower, ix.upper, ix.cbp,
                              const_cast<uint32_t *>(a.op), s);
    if (timing && e == cudaSuccess) e = cudaEventRecord(ev[1], s);
    if (e == cudaSuccess)
        e = launch_seed_tau(a.op, ix.l2w, nq, ix.seed_codes, ix.seed_op, ix.n_entry, ix.cbp, mode,
                            const_cast<int32_t *>(a.seed_tau), ix.err, s);
    if (timing && e == cudaSuccess) e = cudaEventRecord(ev[2], s);
    if (e == cudaSuccess) e = launch_seed_select(a.seed_tau, ix.entry, ix.n_entry, nq, L, a.init_keys, a.init_psz, s);
    if (timing && e == cudaSuccess) e = cudaEventRecord(ev[4], s);
    if (e == cudaSuccess && sp->ev_search_start) e = cudaEventRecord((cudaEvent_t)sp->ev_search_start, s);
    if (e == cudaSuccess) e = launch_search(a, wpb, s, &info);
    if (e == cudaSuccess && sp->ev_search_stop) e = cudaEventRecord((cudaEvent_t)sp->ev_search_stop, s);
    if (timing && e == cudaSuccess) e = cudaEventRecord(ev[3], s);
    cudaFreeAsync(scratch, s);
    if (e == cudaSuccess && timing) {
        e = cudaEventSynchronize(ev[3]);
        if (e == cudaSuccess) {
            cudaEventElapsedTime(&timing->ms_query_prep, ev[0], ev[1]);
            cudaEventElapsedTime(&timing->ms_seed, ev[1], ev[4]);
            cudaEventElapsedTime(&timing->ms_search, ev[4], ev[3]);
            cudaEventElapsedTime(&timing->ms_total, ev[0], ev[3]);
            timing->launches = 4;
            timing->visited_slots = H;
            timing->warps_per_block = info.warps_per_block;
            timing->blocks = info.blocks;
            timing->visited_kind = info.visited_kind;
        }
    }
    if (timing)
        for (auto &x : ev) cudaEventDestroy(x);
    if (e != cudaSuccess) return cuda_fail(e, "vsag_search_batch");
    if (timing) return check_index_flags(ix, s, "vsag_search_batch");  // synchronised already
    return VSAG_OK;
}

vsag_status vsag_search_batch(const vsag_index *h, const float *queries, int64_t nq, int32_t k, int32_t ef,
                              int32_t rerank_n, int32_t metric, int32_t *out_ids, float *out_dists, vsag_trace *trace,
                              void *stream) {
    vsag_search_params sp{};
    sp.k = k;
    sp.ef = ef;
    sp.rerank_n = rerank_n;
    sp.metric = metric;
    return vsag_search_batch_ex(h, queries, nq, &sp, out_ids, out_dists, trace, nullptr, stream);
}

vsag_status vsag_search_batch_host(const vsag_index *h, const float *queries_host, int64_t nq,
                                   const vsag_search_params *sp, int32_t *out_ids_host, float *out_dists_host,
                                   void *stream) {
    g_last_error.clear();
    if (!h || !sp) return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch_host: null index or params");
    const Index &ix = h->ix;
    SearchCfg cfg;
    {
        const vsag_status st = check_search(ix, nq, sp, &cfg);  // before any allocation
        if (st != VSAG_OK) return st;
    }
    if (nq > 0 && (!queries_host || !out_ids_host || !out_dists_host))
        return fail(VSAG_ERR_INVALID_ARG, "vsag_search_batch_host: null pointer");
    if (nq == 0) return VSAG_OK;
    DeviceGuard g(ix.device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t qb = (size_t)nq * ix.d * 4, ob = (size_t)nq * cfg.k * 4;
    uint8_t *buf = nullptr;
    const size_t qoff = 0, ioff = (qb + 255) / 256 * 256, doff = ioff + (ob + 255) / 256 * 256;
    CK(scratch_alloc((void **)&buf, doff + ob, ix.device, s), "vsag_search_batch_host: buffers");
    cudaError_t e = cudaMemcpyAsync(buf + qoff, queries_host, qb, cudaMemcpyHostToDevice, s);
    vsag_status st = VSAG_OK;
    if (e == cudaSuccess) {
        st = vsag_search_batch_ex(h, reinterpret_cast<float *>(buf + qoff), nq, sp, reinterpret_cast<int32_t *>(buf + ioff),
                                  reinterpret_cast<float *>(buf + doff), nullptr, nullptr, stream);
    }
    if (e == cudaSuccess && st == VSAG_OK) e = cudaMemcpyAsync(out_ids_host, buf + ioff, ob, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && st == VSAG_OK) e = cudaMemcpyAsync(out_dists_host, buf + doff, ob, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(buf, s);
    if (st != VSAG_OK) {
        cudaStreamSynchronize(s);
        return st;
    }
    if (e != cudaSuccess) {
        cudaStreamSynchronize(s);
        return cuda_fail(e, "vsag_search_batch_host");
    }
    return check_index_flags(ix, s, "vsag_search_batch_host");  // the call's one synchronisation
}

}  // extern "C"
