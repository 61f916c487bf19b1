// seed.cu -- row a5, part 1: tau_l of every entry node for every query.
//
// Alg. 1 line 3: "insert (x_i, tau_l(x_i, x_q)), for all x_i in I, into C".
// With |I| = S seeds shared by all queries this is a dense [nq x cb] . [cb x S]
// integer contraction, so it is tiled like a GEMM: a CTA stages 32 query operands
// and 64 seed codes in shared memory (32-word K chunks, +1 word row padding so the
// 32 lanes of a warp hit 32 different banks) and every thread keeps a 4 x 2
// register tile of int32 accumulators.  Output tau[nq, S] int32; the per-query
// top-L selection happens at the start of search_kernel.
#include "dist.cuh"

namespace vsag {
namespace {

constexpr int TQ = 32, TS = 64, KC = 32, THREADS = 256;

template <int M>
__global__ void __launch_bounds__(THREADS) seed_tau_kernel(const uint32_t *__restrict__ op, int64_t nq,
                                                           const uint8_t *__restrict__ seed_codes, int S, int cbp,
                                                           int32_t *__restrict__ tau) {
    constexpr int OPW = (M == L2_4 || M == IP_4) ? 2 : 1;
    __shared__ uint32_t sq[TQ][KC * OPW + 1];
    __shared__ uint32_t ss[TS][KC + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 8 warps x 4 queries
    const int64_t q0 = (int64_t)blockIdx.x * TQ;
    const int s0 = blockIdx.y * TS;
    const int cwords = cbp / 4;
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(seed_codes);
    int acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int k0 = 0; k0 < cwords; k0 += KC) {
        __syncthreads();
        for (int e = threadIdx.x; e < TS * KC; e += THREADS) {
            const int s = e / KC, w = e % KC;
            ss[s][w] = (s0 + s < S && k0 + w < cwords) ? __ldg(cw + (int64_t)(s0 + s) * cwords + k0 + w) : 0u;
        }
        for (int e = threadIdx.x; e < TQ * KC * OPW; e += THREADS) {
            const int qq = e / (KC * OPW), w = e % (KC * OPW);
            sq[qq][w] = (q0 + qq < nq && k0 * OPW + w < cwords * OPW)
                            ? __ldg(op + (q0 + qq) * (int64_t)(cwords * OPW) + k0 * OPW + w)
                            : 0u;
        }
        __syncthreads();
#pragma unroll 8
        for (int w = 0; w < KC; w++) {
            const uint32_t c0 = ss[tx][w], c1 = ss[tx + 32][w];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t a0 = sq[ty * 4 + i][w * OPW];
                const uint32_t a1 = OPW == 2 ? sq[ty * 4 + i][w * OPW + 1] : 0u;
                acc[i][0] = word_dist<M>(acc[i][0], a0, a1, c0);
                acc[i][1] = word_dist<M>(acc[i][1], a0, a1, c1);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t qq = q0 + ty * 4 + i;
        if (qq >= nq) continue;
        if (s0 + tx < S) tau[qq * S + s0 + tx] = finish_tau<M>(acc[i][0]);
        if (s0 + tx + 32 < S) tau[qq * S + s0 + tx + 32] = finish_tau<M>(acc[i][1]);
    }
}

}  // namespace

cudaError_t launch_seed_tau(const uint32_t *op, int64_t nq, const uint8_t *seed_codes, int n_seed, int cbp, int mode,
                            int32_t *tau, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    dim3 grid((unsigned)((nq + TQ - 1) / TQ), (unsigned)((n_seed + TS - 1) / TS));
    switch (mode) {
        case L2_8: seed_tau_kernel<L2_8><<<grid, THREADS, 0, s>>>(op, nq, seed_codes, n_seed, cbp, tau); break;
        case L2_4: seed_tau_kernel<L2_4><<<grid, THREADS, 0, s>>>(op, nq, seed_codes, n_seed, cbp, tau); break;
        case IP_8: seed_tau_kernel<IP_8><<<grid, THREADS, 0, s>>>(op, nq, seed_codes, n_seed, cbp, tau); break;
        default: seed_tau_kernel<IP_4><<<grid, THREADS, 0, s>>>(op, nq, seed_codes, n_seed, cbp, tau); break;
    }
    return cudaGetLastError();
}

}  // namespace vsag
