// sq.cu -- rows a1 (SQ train), a2 (SQ encode) and a4 (query prep) for sm_100a.
//
// SQ-b (App. G; §5.2): per-dimension range [lower, upper]
// from the base set (R-1), 2^b - 1 steps (R-2), pinned fp32 op order with
// round-half-away (R-3), constant dimension -> 0 (R-4), SQ4 low nibble first (R-5).
// These kernels are bandwidth-bound one-pass streams (4d bytes in, cb bytes out per
// row); they run once per index build, not in the search step.
#include <vector>

#include "vsag_internal.cuh"

namespace vsag {
namespace {

__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u << 1) == 0) u = 0;  // -0 -> +0 (R-1)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// One SQ-b code (R-3): every op is an explicitly rounded fp32 op, roundf() rounds
// half away from zero (never __float2int_rn, which is half-to-even).
__device__ __forceinline__ int sq_code(float v, float lo, float hi, int levels) {
    if (hi == lo) return 0;
    float c = fminf(fmaxf(v, lo), hi);
    float t = __fdiv_rn(__fsub_rn(c, lo), __fsub_rn(hi, lo));
    t = __fmul_rn(t, (float)levels);
    int code = (int)roundf(t);
    return code > levels ? levels : code;
}

// a1: thread g owns column g % d and rows g / d, g / d + P, ... (coalesced along rows);
// exact min/max is order independent, so global atomics on order-preserving u32 keys
// give the same result as a sequential scan.
__global__ void sq_minmax_kernel(const float *__restrict__ x, int64_t n, int d, int64_t P,
                                 uint32_t *ord_min, uint32_t *ord_max, int *bad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P * d) return;
    const int col = (int)(g % d);
    int64_t r = g / d;
    uint32_t mn = 0xffffffffu, mx = 0u;
    bool nonfinite = false;
    for (; r < n; r += P) {
        float v = __ldg(x + r * d + col);
        nonfinite |= !isfinite(v);
        uint32_t o = f2ord(v);
        mn = min(mn, o);
        mx = max(mx, o);
    }
    if (nonfinite) atomicOr(bad, 1);
    atomicMin(ord_min + col, mn);
    atomicMax(ord_max + col, mx);
}

__global__ void sq_finalize_kernel(const uint32_t *ord_min, const uint32_t *ord_max, int d, float *lower,
                                   float *upper) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < d) {
        lower[j] = ord2f(ord_min[j]);
        upper[j] = ord2f(ord_max[j]);
    }
}

// a1, truncated variant (App. G, "99th percentile statistics"; NEXT-1a):
// per dimension the order statistics at ranks il and iu (0-based) of its n values, by a
// 4-pass radix select on the order-preserving u32 image (8-bit digits, most significant
// first).  Pass kernel: a CTA takes 16 consecutive dimensions and a slice of rows (a
// warp reads 64 contiguous bytes of two rows), counts the digit of every value whose
// higher digits match the target's prefix into shared histograms [2][16][256], then adds
// them to the global histograms.  State per (target, dimension): prefix, remaining rank.
constexpr int QDT = 16;
__global__ void __launch_bounds__(256) quantile_hist_kernel(const float *__restrict__ x, int64_t n, int d,
                                                            int64_t rows_per_cta, int shift,
                                                            const uint32_t *__restrict__ prefix,
                                                            uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[2][QDT][256];
    for (int i = threadIdx.x; i < 2 * QDT * 256; i += 256) (&h[0][0][0])[i] = 0;
    __syncthreads();
    const int dj = threadIdx.x & (QDT - 1), r0 = threadIdx.x / QDT;
    const int j = blockIdx.x * QDT + dj;
    const uint32_t pmask = shift >= 24 ? 0u : (0xffffffffu << (shift + 8));
    if (j < d) {
        const uint32_t p0 = prefix[j], p1 = prefix[d + j];
        const int64_t a = (int64_t)blockIdx.y * rows_per_cta, b = min(n, a + rows_per_cta);
        for (int64_t r = a + r0; r < b; r += 256 / QDT) {
            const uint32_t key = f2ord(__ldg(x + r * d + j));
            const uint32_t dig = (key >> shift) & 0xffu;
            if ((key & pmask) == p0) atomicAdd(&h[0][dj][dig], 1u);
            if ((key & pmask) == p1) atomicAdd(&h[1][dj][dig], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * QDT * 256; i += 256) {
        const int t = i / (QDT * 256), jj = (i / 256) % QDT, dig = i % 256;
        const uint32_t c = h[t][jj][dig];
        if (c && blockIdx.x * QDT + jj < d) atomicAdd(hist + ((int64_t)t * d + blockIdx.x * QDT + jj) * 256 + dig, c);
    }
}

// One thread per (target, dimension): the digit that holds the remaining rank; extends
// the prefix and clears the histogram for the next pass.
__global__ void quantile_step_kernel(uint32_t *hist, int d, int shift, uint32_t *prefix, uint32_t *rank) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * d) return;
    uint32_t *hh = hist + (int64_t)i * 256;
    uint32_t k = rank[i], run = 0, dig = 255;
    for (int t = 0; t < 256; t++) {
        const uint32_t c = hh[t];
        if (run + c > k) {
            dig = t;
            break;
        }
        run += c;
    }
    for (int t = 0; t < 256; t++) hh[t] = 0;
    prefix[i] |= dig << shift;
    rank[i] = k - run;
}

__global__ void quantile_finish_kernel(const uint32_t *prefix, int d, float *lower, float *upper) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < d) {
        lower[j] = ord2f(prefix[j]);
        upper[j] = ord2f(prefix[d + j]);
    }
}

// NEXT-1b weights: w_j = round_half_away(W * r_j^2 / max_k r_k^2), r_j = upper_j - lower_j
// (fp32) widened to fp64; 0 for the padding dimensions.  One warp.
__global__ void l2w_weights_kernel(const float *__restrict__ lower, const float *__restrict__ upper, int d,
                                   int dims_padded, int W, int32_t *w) {
    const int lane = threadIdx.x;
    double m = 0.0;
    for (int j = lane; j < d; j += 32) {
        const double r = (double)__fsub_rn(upper[j], lower[j]);
        m = fmax(m, r * r);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int j = lane; j < dims_padded; j += 32) {
        int v = 0;
        if (j < d && m > 0.0) {
            const double r = (double)__fsub_rn(upper[j], lower[j]);
            v = (int)llround(__ddiv_rn(__dmul_rn((double)W, __dmul_rn(r, r)), m));
        }
        w[j] = v;
    }
}

// Index load: flags (bit 1) any base value outside [lower_j, upper_j] (the NEXT-3 re-rank
// bound assumes the base lies inside the trained range).
__global__ void range_check_kernel(const float *__restrict__ x, int64_t n, int d, const float *__restrict__ lower,
                                   const float *__restrict__ upper, int *bad) {
    bool out = false;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n * d; g += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(g % d);
        const float v = __ldg(x + g);
        out |= !(v >= __ldg(lower + j) && v <= __ldg(upper + j));
    }
    if (__any_sync(0xffffffffu, out) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// a2: one thread per (row, 4 code bytes).  SQ8: byte b = dim b.  SQ4: byte b = dims
// (2b, 2b+1) as (lo, hi) nibbles.  Rows of `stride` bytes; bytes in [cb, stride) are
// written as 0 when stride > cb (internal padded copies).
__global__ void sq_encode_kernel(const float *__restrict__ x, int64_t n, int d, int bits,
                                 const float *__restrict__ lower, const float *__restrict__ upper,
                                 uint8_t *__restrict__ codes, int cb, int64_t stride) {
    const int words = (int)((stride + 3) / 4);
    const int levels = (1 << bits) - 1;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n * words;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / words;
        const int w = (int)(g % words);
        const float *xr = x + r * d;
        uint32_t packed = 0;
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int b = 4 * w + t;
            uint32_t byte = 0;
            if (b < cb) {
                if (bits == 8) {
                    byte = (uint32_t)sq_code(__ldg(xr + b), __ldg(lower + b), __ldg(upper + b), levels);
                } else {
                    const int j0 = 2 * b, j1 = 2 * b + 1;
                    byte = (uint32_t)sq_code(__ldg(xr + j0), __ldg(lower + j0), __ldg(upper + j0), levels);
                    if (j1 < d)
                        byte |= (uint32_t)sq_code(__ldg(xr + j1), __ldg(lower + j1), __ldg(upper + j1), levels) << 4;
                }
            }
            packed |= byte << (8 * t);
        }
        uint8_t *dst = codes + r * stride + 4 * w;
        if ((stride & 3) == 0) {
            *reinterpret_cast<uint32_t *>(dst) = packed;
        } else {
            for (int t = 0; t < 4 && 4 * w + t < stride; t++) dst[t] = (uint8_t)(packed >> (8 * t));
        }
    }
}

// a4: one warp per query.  Writes the "operand" the distance stage consumes, per code
// word k (4 code bytes) of the cbp-byte padded code:
//   L2_8: word k = query codes of dims 4k..4k+3                         (R-6)
//   L2_4: words (2k, 2k+1) = (lo, hi) nibble planes of dims 8k..8k+7 as bytes
//         lo = dims 8k, 8k+2, 8k+4, 8k+6 ; hi = dims 8k+1, 8k+3, 8k+5, 8k+7
//   IP_8: word k = int8 weights of dims 4k..4k+3                       (R-7)
//   IP_4: words (2k, 2k+1) = int8 weights in the lo/hi plane order above
// Padding dimensions get 0, matching the zero padding of the base codes.
__global__ void query_prep_kernel(const float *__restrict__ q, int64_t nq, int d, int bits, int metric,
                                  const float *__restrict__ lower, const float *__restrict__ upper, int cbp,
                                  uint32_t *__restrict__ op) {
    const int lane = threadIdx.x & 31;
    const int64_t qi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (qi >= nq) return;
    const float *qr = q + qi * d;
    const int levels = (1 << bits) - 1;
    const int cwords = cbp / 4;
    const int mode = mode_of(metric, bits);
    const int opw = op_words_per_code_word(mode);
    uint32_t *out = op + qi * (int64_t)cwords * opw;

    float s = 0.0f;  // IP: s = max_d |a_d|, exact (max is order independent)
    if (metric == VSAG_METRIC_IP) {
        for (int j = lane; j < d; j += 32) {
            float a = __fmul_rn(__ldg(qr + j), __fsub_rn(__ldg(upper + j), __ldg(lower + j)));
            s = fmaxf(s, fabsf(a));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
    }
    auto value = [&](int j) -> int {  // per-dimension operand value (0 beyond d)
        if (j >= d) return 0;
        if (metric != VSAG_METRIC_IP)  // L2 and the weighted L2 encode the query with the base model
            return sq_code(__ldg(qr + j), __ldg(lower + j), __ldg(upper + j), levels);
        if (s == 0.0f) return 0;
        float a = __fmul_rn(__ldg(qr + j), __fsub_rn(__ldg(upper + j), __ldg(lower + j)));
        return (int)roundf(__fmul_rn(__fdiv_rn(a, s), 127.0f));
    };
    for (int k = lane; k < cwords; k += 32) {
        if (bits == 8) {
            uint32_t w = 0;
#pragma unroll
            for (int t = 0; t < 4; t++) w |= ((uint32_t)value(4 * k + t) & 0xffu) << (8 * t);
            out[k] = w;
        } else {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int t = 0; t < 4; t++) {
                lo |= ((uint32_t)value(8 * k + 2 * t) & 0xffu) << (8 * t);
                hi |= ((uint32_t)value(8 * k + 2 * t + 1) & 0xffu) << (8 * t);
            }
            out[2 * k] = lo;
            out[2 * k + 1] = hi;
        }
    }
}

}  // namespace

cudaError_t launch_sq_minmax(const float *x, int64_t n, int d, uint32_t *ord_min, uint32_t *ord_max, int *bad,
                             cudaStream_t s) {
    int64_t P = (148LL * 2048 + d - 1) / d;
    if (P > n) P = n;
    if (P < 1) P = 1;
    const int64_t threads = P * d;
    const int block = 256;
    sq_minmax_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, s>>>(x, n, d, P, ord_min, ord_max, bad);
    return cudaGetLastError();
}

cudaError_t launch_sq_finalize(const uint32_t *ord_min, const uint32_t *ord_max, int d, float *lower, float *upper,
                               cudaStream_t s) {
    sq_finalize_kernel<<<(d + 255) / 256, 256, 0, s>>>(ord_min, ord_max, d, lower, upper);
    return cudaGetLastError();
}

cudaError_t launch_sq_encode(const float *x, int64_t n, int d, int bits, const float *lower, const float *upper,
                             uint8_t *codes, int64_t stride, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int cb = bits == 8 ? d : (d + 1) / 2;
    const int64_t work = n * ((stride + 3) / 4);
    int64_t blocks = (work + 255) / 256;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    sq_encode_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, n, d, bits, lower, upper, codes, cb, stride);
    return cudaGetLastError();
}

size_t train_quantile_scratch_words(int d) { return (size_t)2 * d * 256 + 4 * (size_t)d; }

cudaError_t launch_train_quantile(const float *x, int64_t n, int d, int64_t il, int64_t iu, float *lower,
                                  float *upper, uint32_t *scratch, cudaStream_t s) {
    uint32_t *hist = scratch, *prefix = scratch + (size_t)2 * d * 256, *rank = prefix + 2 * (size_t)d;
    cudaError_t e = cudaMemsetAsync(scratch, 0, train_quantile_scratch_words(d) * 4, s);
    if (e != cudaSuccess) return e;
    // ranks: targets 0 (lower) and 1 (upper)
    std::vector<uint32_t> hr(2 * (size_t)d);
    for (int j = 0; j < d; j++) {
        hr[j] = (uint32_t)il;
        hr[d + j] = (uint32_t)iu;
    }
    e = cudaMemcpyAsync(rank, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    int64_t rows_per_cta = 4096;
    const unsigned gx = (unsigned)((d + QDT - 1) / QDT);
    while ((int64_t)gx * ((n + rows_per_cta - 1) / rows_per_cta) > 148LL * 64 && rows_per_cta < (1 << 30))
        rows_per_cta *= 2;
    const dim3 grid(gx, (unsigned)((n + rows_per_cta - 1) / rows_per_cta));
    for (int shift = 24; shift >= 0; shift -= 8) {
        quantile_hist_kernel<<<grid, 256, 0, s>>>(x, n, d, rows_per_cta, shift, prefix, hist);
        quantile_step_kernel<<<(2 * d + 255) / 256, 256, 0, s>>>(hist, d, shift, prefix, rank);
    }
    quantile_finish_kernel<<<(d + 255) / 256, 256, 0, s>>>(prefix, d, lower, upper);
    e = cudaStreamSynchronize(s);  // the host rank vector must outlive the copy
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_range_check(const float *x, int64_t n, int d, const float *lower, const float *upper, int *bad,
                               cudaStream_t s) {
    int64_t blocks = (n * d + 255) / 256;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    range_check_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, n, d, lower, upper, bad);
    return cudaGetLastError();
}

cudaError_t launch_l2w_weights(const float *lower, const float *upper, int d, int dims_padded, int W, int32_t *w,
                               cudaStream_t s) {
    l2w_weights_kernel<<<1, 32, 0, s>>>(lower, upper, d, dims_padded, W, w);
    return cudaGetLastError();
}

cudaError_t launch_query_prep(const float *q, int64_t nq, int d, int bits, int metric, const float *lower,
                              const float *upper, int cbp, uint32_t *op, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const int block = 256;
    const int64_t blocks = (nq * 32 + block - 1) / block;
    query_prep_kernel<<<(unsigned)blocks, block, 0, s>>>(q, nq, d, bits, metric, lower, upper, cbp, op);
    return cudaGetLastError();
}

}  // namespace vsag
