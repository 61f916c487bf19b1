// layout.cu -- row a3 (index load): adjacency validation / padding, the PRS
// co-located layout (delta = 1, §3.3.2: "co-locating neighbor lists with
// their corresponding vectors within each node's data structure") and the seed-code
// block.  One-time, bandwidth-bound gathers.
#include "vsag_internal.cuh"

namespace vsag {
namespace {

__global__ void check_adj_kernel(const int32_t *__restrict__ adj, int64_t count, int64_t n, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = adj[t];
        if (v < -1 || v >= n) atomicOr(bad, 1);
    }
}

// CSR -> fixed-degree rows padded with -1 (one thread per row).
__global__ void csr_to_padded_kernel(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t n,
                                     int degree, int32_t *__restrict__ out, int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = row_ptr[i], b = row_ptr[i + 1];
        if (b < a || b - a > degree) {
            atomicOr(bad, 2);
            continue;
        }
        for (int t = 0; t < degree; t++) {
            int32_t v = (a + t < b) ? col[a + t] : -1;
            if (v < -1 || v >= n) atomicOr(bad, 1);
            out[i * degree + t] = v;
        }
    }
}

// Sets bit 4 of *flag if any row holds the same id twice (the search kernel then
// de-duplicates each id row before the visited filter).  One thread per row.
__global__ void row_dups_kernel(const int32_t *__restrict__ adj, int64_t n, int degree, int *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *row = adj + i * degree;
        bool dup = false;
        for (int t = 1; t < degree && !dup; t++) {
            const int32_t v = row[t];
            if (v < 0) continue;
            for (int u = 0; u < t; u++)
                if (row[u] == v) {
                    dup = true;
                    break;
                }
        }
        if (dup) atomicOr(flag, 4);
    }
}

// Edge labels into the padded [n, degree] layout of the index's adjacency (CSR rows are
// left-aligned like csr_to_padded, the tail gets +inf; the search ignores the labels of
// -1 slots).  bit 1: NaN label; bit 2: CSR row longer than degree.
__global__ void pad_labels_kernel(const int64_t *__restrict__ row_ptr, const float *__restrict__ src, int64_t n,
                                  int degree, float *__restrict__ dst, int *bad) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n * degree;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = g / degree;
        const int t = (int)(g % degree);
        float v;
        if (row_ptr) {
            const int64_t a = row_ptr[i], b = row_ptr[i + 1];
            if (b - a > degree) atomicOr(bad, 2);
            v = a + t < b ? src[a + t] : __int_as_float(0x7f800000);
        } else {
            v = src[g];
        }
        if (isnan(v)) atomicOr(bad, 1);
        dst[g] = v;
    }
}

__global__ void in_degree_kernel(const int32_t *__restrict__ adj, int64_t count, int32_t *indeg) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = adj[t];
        if (v >= 0) atomicAdd(indeg + v, 1);
    }
}

// PRS block b = codes of node nodes[b]'s neighbours in row order (one warp per block).
__global__ void prs_build_kernel(const int32_t *__restrict__ adj, const uint8_t *__restrict__ codes,
                                 const int32_t *__restrict__ nodes, int64_t count, int degree, int cbp,
                                 uint8_t *__restrict__ blocks) {
    const int lane = threadIdx.x & 31;
    const int chunks = cbp / 16;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < count;
         b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t i = nodes[b];
        uint4 *dst = reinterpret_cast<uint4 *>(blocks + b * (int64_t)degree * cbp);
        for (int e = lane; e < degree * chunks; e += 32) {
            const int t = e / chunks, c = e % chunks;
            const int32_t j = adj[(int64_t)i * degree + t];
            dst[e] = j >= 0 ? __ldg(reinterpret_cast<const uint4 *>(codes + (int64_t)j * cbp) + c) : make_uint4(0, 0, 0, 0);
        }
    }
}

// Copy codes [n, cb] into a 16-byte-strided [n, cbp] table with zero padding.
__global__ void copy_pad_codes_kernel(const uint8_t *__restrict__ src, int64_t n, int cb, int cbp,
                                      uint8_t *__restrict__ dst) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n * cbp; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / cbp;
        const int b = (int)(g % cbp);
        dst[g] = b < cb ? src[r * cb + b] : 0;
    }
}

// Layout 1 row of node i: [ids: degree int32, padded to ids_bytes | slot t: code of
// neighbour adj[i][t] (cbp bytes; zero for an empty slot)].  One warp per row,
// 16-byte copies.
__global__ void layout_build_kernel(const int32_t *__restrict__ adj, const uint8_t *__restrict__ codes, int64_t n,
                                    int degree, int cbp, int ids_bytes, int64_t row_bytes, uint8_t *__restrict__ rows) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int chunks = cbp / 16;
    for (int64_t i = warp; i < n; i += nwarps) {
        uint8_t *row = rows + i * row_bytes;
        int32_t *ids = reinterpret_cast<int32_t *>(row);
        for (int t = lane; t < ids_bytes / 4; t += 32) ids[t] = t < degree ? adj[i * degree + t] : -1;
        uint4 *dst = reinterpret_cast<uint4 *>(row + ids_bytes);
        for (int e = lane; e < degree * chunks; e += 32) {
            const int t = e / chunks, c = e % chunks;
            const int32_t j = adj[i * degree + t];
            uint4 v = make_uint4(0, 0, 0, 0);
            if (j >= 0) v = __ldg(reinterpret_cast<const uint4 *>(codes + (int64_t)j * cbp) + c);
            dst[e] = v;
        }
    }
}

__global__ void gather_codes_kernel(const int32_t *__restrict__ ids, int count, const uint8_t *__restrict__ codes,
                                    int cbp, uint8_t *__restrict__ dst) {
    const int chunks = cbp / 16;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < (int64_t)count * chunks;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = g / chunks;
        const int c = (int)(g % chunks);
        reinterpret_cast<uint4 *>(dst + s * cbp)[c] =
            __ldg(reinterpret_cast<const uint4 *>(codes + (int64_t)ids[s] * cbp) + c);
    }
}

inline unsigned grid_for(int64_t work, int block) {
    int64_t b = (work + block - 1) / block;
    if (b > 148LL * 32) b = 148LL * 32;
    if (b < 1) b = 1;
    return (unsigned)b;
}

}  // namespace

cudaError_t launch_check_adj(const int32_t *adj, int64_t count, int64_t n, int *bad, cudaStream_t s) {
    check_adj_kernel<<<grid_for(count, 256), 256, 0, s>>>(adj, count, n, bad);
    return cudaGetLastError();
}

cudaError_t launch_csr_to_padded(const int64_t *row_ptr, const int32_t *col, int64_t n, int degree, int32_t *out,
                                 int *bad, cudaStream_t s) {
    csr_to_padded_kernel<<<grid_for(n, 256), 256, 0, s>>>(row_ptr, col, n, degree, out, bad);
    return cudaGetLastError();
}

cudaError_t launch_row_dups(const int32_t *adj, int64_t n, int degree, int *flag, cudaStream_t s) {
    row_dups_kernel<<<grid_for(n, 256), 256, 0, s>>>(adj, n, degree, flag);
    return cudaGetLastError();
}

cudaError_t launch_pad_labels(const int64_t *row_ptr, const float *src, int64_t n, int degree, float *dst, int *bad,
                              cudaStream_t s) {
    pad_labels_kernel<<<grid_for(n * degree, 256), 256, 0, s>>>(row_ptr, src, n, degree, dst, bad);
    return cudaGetLastError();
}

cudaError_t launch_in_degree(const int32_t *adj, int64_t count, int32_t *indeg, cudaStream_t s) {
    in_degree_kernel<<<grid_for(count, 256), 256, 0, s>>>(adj, count, indeg);
    return cudaGetLastError();
}

cudaError_t launch_prs_build(const int32_t *adj, const uint8_t *codes, const int32_t *nodes, int64_t count, int degree,
                             int cbp, uint8_t *blocks, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    prs_build_kernel<<<grid_for(count * 32, 256), 256, 0, s>>>(adj, codes, nodes, count, degree, cbp, blocks);
    return cudaGetLastError();
}

cudaError_t launch_copy_pad_codes(const uint8_t *src, int64_t n, int cb, int cbp, uint8_t *dst, cudaStream_t s) {
    copy_pad_codes_kernel<<<grid_for(n * cbp, 256), 256, 0, s>>>(src, n, cb, cbp, dst);
    return cudaGetLastError();
}

cudaError_t launch_layout_build(const int32_t *adj, const uint8_t *codes, int64_t n, int degree, int cbp,
                                int ids_bytes, int64_t row_bytes, uint8_t *rows, cudaStream_t s) {
    layout_build_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(adj, codes, n, degree, cbp, ids_bytes, row_bytes, rows);
    return cudaGetLastError();
}

cudaError_t launch_gather_codes(const int32_t *ids, int count, const uint8_t *codes, int cbp, uint8_t *dst,
                                cudaStream_t s) {
    gather_codes_kernel<<<grid_for((int64_t)count * (cbp / 16), 256), 256, 0, s>>>(ids, count, codes, cbp, dst);
    return cudaGetLastError();
}

}  // namespace vsag
