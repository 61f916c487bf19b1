// seed.cu -- row a5, part 1: tau_l of every entry node for every query.  L2 and IP (SQ8 and
// SQ4) run on the tensor cores (tcgen05 kind::i8, seed_umma.cuh); the weighted L2 (NEXT-1b)
// uses the dp4a tile below.
//
// Alg. 1 line 3: "insert (x_i, tau_l(x_i, x_q)), for all x_i in I, into C".
// With |I| = S seeds shared by all queries this is a dense [nq x cb] . [cb x S]
// integer contraction, so it is tiled like a GEMM: a CTA stages 32 query operands
// and 128 seed codes in shared memory (32-word K chunks) and every thread keeps a 4 x 4
// register tile of int32 accumulators.  Output tau[nq, S] int32; the per-query top-L
// selection is seed_select_kernel (select.cu).
#include <cudaTypedefs.h>

#include "dist.cuh"
#include "seed_umma.cuh"

namespace vsag {
namespace {

constexpr int TQ = 32, TS = 128, KC = 32, THREADS = 256;

// CTA tile: 32 queries x 128 seeds, K (code words) in chunks of 32.  Thread (lane, warp)
// owns queries 4*warp .. 4*warp+3 and seeds lane, lane+32, lane+64, lane+96 (16 int32
// accumulators); per 4 code words it reads 4 seed chunks and 4 (SQ4: 8) query chunks as
// 16-byte shared loads (query rows are warp-uniform: broadcast; seed rows are padded to
// 36 words so the 16-byte loads of a quarter warp hit distinct banks).
template <int M>
__global__ void __launch_bounds__(THREADS) seed_tau_kernel(const uint32_t *__restrict__ op,
                                                           const int32_t *__restrict__ l2w, int64_t nq,
                                                           const uint8_t *__restrict__ seed_codes, int S, int cbp,
                                                           int32_t *__restrict__ tau) {
    constexpr int OPW = mode_sq4(M) ? 2 : 1;
    constexpr int DPW = mode_sq4(M) ? 8 : 4;  // dimensions per code word
    constexpr int SQW = KC * OPW + 4, SSW = KC + 4;  // padded row widths (words)
    __shared__ __align__(16) uint32_t sq[TQ * SQW];
    __shared__ __align__(16) uint32_t ss[TS * SSW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q0 = (int64_t)blockIdx.x * TQ;
    const int s0 = blockIdx.y * TS;
    const int cwords = cbp / 4;  // multiple of 4 (cbp is a multiple of 16)
    const uint4 *cw = reinterpret_cast<const uint4 *>(seed_codes);
    const uint4 *ow = reinterpret_cast<const uint4 *>(op);
    int acc[4][4] = {};
    for (int k0 = 0; k0 < cwords; k0 += KC) {
        const int kc = min(KC, cwords - k0);  // words in this chunk (multiple of 4)
        __syncthreads();
        for (int e = threadIdx.x; e < TS * (KC / 4); e += THREADS) {
            const int si = e / (KC / 4), w4 = e % (KC / 4);
            uint4 v = make_uint4(0, 0, 0, 0);
            if (s0 + si < S && 4 * w4 < kc) v = __ldg(cw + (int64_t)(s0 + si) * (cwords / 4) + k0 / 4 + w4);
            *reinterpret_cast<uint4 *>(ss + si * SSW + 4 * w4) = v;
        }
        for (int e = threadIdx.x; e < TQ * (KC * OPW / 4); e += THREADS) {
            const int qi = e / (KC * OPW / 4), w4 = e % (KC * OPW / 4);
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + qi < nq && 4 * w4 < kc * OPW)
                v = __ldg(ow + (q0 + qi) * (int64_t)(cwords * OPW / 4) + k0 * OPW / 4 + w4);
            *reinterpret_cast<uint4 *>(sq + qi * SQW + 4 * w4) = v;
        }
        __syncthreads();
#pragma unroll 2
        for (int w = 0; w < KC; w += 4) {
            uint4 c[4];
#pragma unroll
            for (int j = 0; j < 4; j++) c[j] = *reinterpret_cast<const uint4 *>(ss + (lane + 32 * j) * SSW + w);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t *qa = sq + (warp * 4 + i) * SQW + w * OPW;
                uint32_t a[4 * OPW];
                {
                    const uint4 a0 = *reinterpret_cast<const uint4 *>(qa);
                    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
                    if (OPW == 2) {
                        const uint4 a1 = *reinterpret_cast<const uint4 *>(qa + 4);
                        a[4 * OPW - 4] = a1.x; a[4 * OPW - 3] = a1.y; a[4 * OPW - 2] = a1.z; a[4 * OPW - 1] = a1.w;
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint32_t cc[4] = {c[j].x, c[j].y, c[j].z, c[j].w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        if (mode_w(M))  // weights of the word's dimensions (uniform across the CTA)
                            acc[i][j] = word_dist_w<M>(acc[i][j], a[t * OPW], OPW == 2 ? a[t * OPW + 1] : 0u, cc[t],
                                                       l2w + (int64_t)(k0 + w + t) * DPW);
                        else
                            acc[i][j] = word_dist<M>(acc[i][j], a[t * OPW], OPW == 2 ? a[t * OPW + 1] : 0u, cc[t]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t qq = q0 + warp * 4 + i;
        if (qq >= nq) continue;
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (s0 + lane + 32 * j < S) tau[qq * S + s0 + lane + 32 * j] = finish_tau<M>(acc[i][j]);
    }
}

// SQ4 seed operand for the tensor cores: one nibble per byte in the query operand's plane
// order (per 4-byte code word: its 4 low nibbles, then its 4 high nibbles), [S, 2 cbp].
__global__ void unpack_sq4_planes_kernel(const uint8_t *__restrict__ codes, int S, int cbp, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one code word
    const int64_t words = (int64_t)S * (cbp / 4);
    if (i >= words) return;
    const uint32_t w = reinterpret_cast<const uint32_t *>(codes)[i];
    reinterpret_cast<uint2 *>(out)[i] = make_uint2(w & 0x0F0F0F0Fu, (w >> 4) & 0x0F0F0F0Fu);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D u8 tensor [rows, inner] with row stride `stride` bytes; box 128 bytes x box_rows,
// 128-byte swizzle (the UMMA operand layout of seed_umma.cuh); out-of-range reads are zero.
bool make_map(CUtensorMap *m, const void *base, uint64_t inner, uint64_t rows, uint64_t stride, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {stride};
    const cuuint32_t box[2] = {(cuuint32_t)umma::KB, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t seed_operand_bytes(int n_seed, int cbp, int bits) { return (size_t)n_seed * cbp * (bits == 4 ? 2 : 1); }

cudaError_t launch_seed_operand(const uint8_t *seed_codes, int n_seed, int cbp, int bits, uint8_t *out, cudaStream_t s) {
    if (bits != 4) return cudaMemcpyAsync(out, seed_codes, (size_t)n_seed * cbp, cudaMemcpyDeviceToDevice, s);
    const int64_t words = (int64_t)n_seed * (cbp / 4);
    unpack_sq4_planes_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(seed_codes, n_seed, cbp, out);
    return cudaGetLastError();
}

// The tcgen05 contraction: op [nq, kbytes] (query operand), seed_op [n_seed, kbytes].
cudaError_t launch_seed_tau_umma(const uint8_t *op, int64_t nq, const uint8_t *seed_op, int n_seed, int kbytes, bool ip,
                                 int32_t *tau, int *err, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    if (nq > 0x7fffffffLL - umma::TM) return cudaErrorInvalidValue;
    CUtensorMap ta, tb;
    if (!make_map(&ta, op, (uint64_t)kbytes, (uint64_t)nq, (uint64_t)kbytes, umma::TM) ||
        !make_map(&tb, seed_op, (uint64_t)kbytes, (uint64_t)n_seed, (uint64_t)kbytes, umma::TN))
        return cudaErrorInvalidValue;
    auto kern = ip ? umma::seed_tau_umma_kernel<true> : umma::seed_tau_umma_kernel<false>;
    const size_t sm = umma::seed_tau_umma_smem(kbytes);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 g((unsigned)((nq + umma::TM - 1) / umma::TM), (unsigned)((n_seed + umma::TN - 1) / umma::TN));
    kern<<<g, 128, sm, s>>>(ta, tb, nq, n_seed, kbytes, tau, err);
    return cudaGetLastError();
}

cudaError_t launch_seed_tau(const uint32_t *op, const int32_t *l2w, int64_t nq, const uint8_t *seed_codes,
                            const uint8_t *seed_op, int n_seed, int cbp, int mode, int32_t *tau, int *err,
                            cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    if (mode == L2_8 || mode == IP_8 || mode == L2_4 || mode == IP_4) {
        // the contraction on the tensor cores (seed_umma.cuh); the query operand is one byte
        // per dimension (L2: code values, IP: int8 weights), in the nibble-plane order for SQ4
        const int kbytes = mode_sq4(mode) ? 2 * cbp : cbp;
        return launch_seed_tau_umma(reinterpret_cast<const uint8_t *>(op), nq, seed_op, n_seed, kbytes,
                                    mode == IP_8 || mode == IP_4, tau, err, s);
    }
    dim3 grid((unsigned)((nq + TQ - 1) / TQ), (unsigned)((n_seed + TS - 1) / TS));
    switch (mode) {
        case L2_8: seed_tau_kernel<L2_8><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
        case L2_4: seed_tau_kernel<L2_4><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
        case IP_8: seed_tau_kernel<IP_8><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
        case IP_4: seed_tau_kernel<IP_4><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
        case L2W_8: seed_tau_kernel<L2W_8><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
        default: seed_tau_kernel<L2W_4><<<grid, THREADS, 0, s>>>(op, l2w, nq, seed_codes, n_seed, cbp, tau); break;
    }
    return cudaGetLastError();
}

}  // namespace vsag
