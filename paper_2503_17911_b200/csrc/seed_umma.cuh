// seed_umma.cuh -- row a5, part 1 on the tensor cores: tau_l of every entry node for every
// query as an 8-bit contraction on tcgen05 (kind::i8): SQ8 L2 (u8 query codes x u8 codes) and
// SQ8 IP (s8 query weights x u8 codes, R-7: tau_l = -sum w_d c_d).
//
// Alg. 1 line 3 evaluates tau_l(x_q, s) for every initial node s.  For SQ8 L2 the
// code-space distance splits exactly, in integers, as |cq|^2 + |c_s|^2 - 2 cq.c_s (the
// decomposition of P:649; u8 products summed in int32 are exact), so the S x nq grid is a
// dense [nq x cb] . [cb x S] contraction: a CTA stages 128 query codes (A) and TN seed codes
// (B) in shared memory in the canonical K-major no-swizzle layout (8-row x 16-byte core
// matrices: K-adjacent core matrices 128 B apart, 8-row groups 1 KB apart), one thread
// issues tcgen05.mma (M 128, N TN, K 32 per instruction) into a 128 x TN int32
// accumulator in tensor memory, and each thread then reads its query's row back with
// tcgen05.ld and writes tau = |cq|^2 + |c_s|^2 - 2 dot.  K is processed in 128-byte blocks.
#pragma once
#include <stdint.h>

namespace vsag {
namespace umma {

constexpr int TM = 128, TN = 128, KB = 128;  // tile rows (queries), columns (seeds), K block (bytes)
constexpr int SMEM_A = TM * KB, SMEM_B = TN * KB;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Shared-memory matrix descriptor (sm_100): start >> 4 in [0, 14), leading-dimension byte
// offset >> 4 in [16, 30), stride-dimension byte offset >> 4 in [32, 46), version 1 at 46,
// base offset 0, legacy LBO mode, layout type 0 (no swizzle) in [61, 64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// Instruction descriptor, kind::i8: D s32 (c_format 2 at [4, 6)), A unsigned (0) or signed (1)
// 8-bit at [7, 10), B unsigned 8-bit at [10, 13), both K-major, N >> 3 at [17, 23), M >> 4 at
// [24, 29).
template <bool SIGNED_A>
__host__ __device__ constexpr uint32_t idesc() {
    return (2u << 4) | ((SIGNED_A ? 1u : 0u) << 7) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

// Wait for an mbarrier phase; false if it did not complete within ~2^26 polls (a lost
// tensor-core commit): the caller reports it through the index's error flag instead of
// hanging the GPU or trapping (a trap would leave a sticky context error).
__device__ __forceinline__ bool mbar_wait(uint32_t mbar, uint32_t phase) {
    uint32_t done = 0;
    for (long long spin = 0; !done; spin++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(mbar), "r"(phase));
        if (spin > (1ll << 26)) return false;
    }
    return true;
}

// tau[q, s] for q in [q0, q0 + 128), s in [s0, s0 + TN).  128 threads (4 warps); warp w
// reads tensor-memory lanes 32 w .. 32 w + 31 = the tile's queries 32 w .. 32 w + 31.
// IP: A holds the int8 weights and tau = -dot; L2: tau = |cq|^2 + |c_s|^2 - 2 dot.
// SQ4: K runs over the unpacked nibbles in the query operand's plane order (per code word:
// its low nibbles as 4 bytes, then its high nibbles), so B is unpacked while it is staged and
// A (the operand, 2 * cbp bytes per query) is used as it is.
template <bool IP, bool SQ4 = false>
__global__ void __launch_bounds__(128) seed_tau_umma_kernel(const uint8_t *__restrict__ qcodes, int64_t nq,
                                                            const uint8_t *__restrict__ scodes, int S, int cbp,
                                                            int32_t *__restrict__ tau, int *err) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sa = smem;                                  // [TM rows x KB] core-matrix layout
    uint8_t *sb = smem + SMEM_A;                         // [TN rows x KB]
    int32_t *snorm = reinterpret_cast<int32_t *>(smem + SMEM_A + SMEM_B);  // [TN]
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t q0 = (int64_t)blockIdx.x * TM;
    const int s0 = blockIdx.y * TN;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "n"(TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // |cq|^2 of this thread's query row and |c_s|^2 of its two seed rows, accumulated from the
    // staged tiles block by block (shared-memory reads; no extra global traffic)
    constexpr int NS = TN / 128;  // seed rows per thread
    int qn = 0, sn[NS] = {};
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;

    uint32_t phase = 0;
    const int kbytes = SQ4 ? 2 * cbp : cbp;  // K in bytes (= the operand's row stride)
    for (int kb = 0; kb < kbytes; kb += KB) {
        const int kw = min(KB, kbytes - kb);  // bytes of K in this block (multiple of 16)
        if (kb > 0) __syncthreads();  // every thread's norm reads of the previous block are done
        // stage A and B: 16-byte chunk i of row r goes to (r / 8) * 1024 + (i) * 128 + (r % 8) * 16;
        // chunks past kw (a partial last block) and rows past nq / S are zero
        for (int i = tid; i < TM * (KB / 16); i += 128) {
            const int r = i >> 3, c = i & 7;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (q0 + r < nq && c * 16 < kw)
                v = __ldg(reinterpret_cast<const uint4 *>(qcodes + (q0 + r) * kbytes + kb) + c);
            *reinterpret_cast<uint4 *>(sa + (r >> 3) * 1024 + c * 128 + (r & 7) * 16) = v;
        }
        for (int i = tid; i < TN * (KB / 16); i += 128) {
            const int r = i >> 3, c = i & 7;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (s0 + r < S && c * 16 < kw) {
                if (SQ4) {  // 8 packed bytes = 2 code words -> (lo0, hi0, lo1, hi1)
                    const uint2 p = __ldg(reinterpret_cast<const uint2 *>(scodes + (int64_t)(s0 + r) * cbp + kb / 2) + c);
                    v = make_uint4(p.x & 0x0F0F0F0Fu, (p.x >> 4) & 0x0F0F0F0Fu, p.y & 0x0F0F0F0Fu, (p.y >> 4) & 0x0F0F0F0Fu);
                } else {
                    v = __ldg(reinterpret_cast<const uint4 *>(scodes + (int64_t)(s0 + r) * cbp + kb) + c);
                }
            }
            *reinterpret_cast<uint4 *>(sb + (r >> 3) * 1024 + c * 128 + (r & 7) * 16) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy stores -> tensor core
        __syncthreads();
#pragma unroll
        for (int c = 0; c < (IP ? 0 : KB / 16); c++) {
            const uint4 a4 = *reinterpret_cast<const uint4 *>(sa + (tid >> 3) * 1024 + c * 128 + (tid & 7) * 16);
            qn = (int)__dp4a(a4.x, a4.x, __dp4a(a4.y, a4.y, __dp4a(a4.z, a4.z, __dp4a(a4.w, a4.w, (unsigned)qn))));
#pragma unroll
            for (int j = 0; j < NS; j++) {
                const int r = tid + 128 * j;
                const uint4 b = *reinterpret_cast<const uint4 *>(sb + (r >> 3) * 1024 + c * 128 + (r & 7) * 16);
                sn[j] = (int)__dp4a(b.x, b.x, __dp4a(b.y, b.y, __dp4a(b.z, b.z, __dp4a(b.w, b.w, (unsigned)sn[j]))));
            }
        }
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int ks = 0; ks < KB / 32; ks++) {
                const uint64_t ad = make_desc(smem_u32(sa) + ks * 256, 128, 1024);
                const uint64_t bd = make_desc(smem_u32(sb) + ks * 256, 128, 1024);
                const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                    ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc<IP>()), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mbar)));
        }
        if (!mbar_wait(smem_u32(&mbar), phase)) {
            if (tid == 0) *reinterpret_cast<volatile int *>(err) = 1;  // (mapped host flag) reported by the API
        }
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
    }

#pragma unroll
    for (int j = 0; j < NS; j++) snorm[tid + 128 * j] = sn[j];
    __syncthreads();
    // epilogue: this thread's query row, 32 columns at a time
    const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < TN; c0 += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(trow + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        // stage the warp's 32 x 32 block in shared memory (16-byte chunks XOR-swizzled by row,
        // the A tile is free now), then write it back row-contiguously: 8 lanes per 128-byte
        // row segment, so every global store fills whole sectors
        uint4 *stg = reinterpret_cast<uint4 *>(sa) + warp * 32 * 8;  // [32 rows][8 chunks]
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            uint4 o;
            o.x = (uint32_t)(IP ? -(int)v[j] : qn + snorm[c0 + j] - 2 * (int)v[j]);
            o.y = (uint32_t)(IP ? -(int)v[j + 1] : qn + snorm[c0 + j + 1] - 2 * (int)v[j + 1]);
            o.z = (uint32_t)(IP ? -(int)v[j + 2] : qn + snorm[c0 + j + 2] - 2 * (int)v[j + 2]);
            o.w = (uint32_t)(IP ? -(int)v[j + 3] : qn + snorm[c0 + j + 3] - 2 * (int)v[j + 3]);
            stg[(tid & 31) * 8 + ((j >> 2) ^ (tid & 7))] = o;
        }
        __syncwarp();
        const int lane = tid & 31, cj = lane & 7;
#pragma unroll
        for (int rr = 0; rr < 32; rr += 4) {
            const int rl = rr + (lane >> 3);  // row within the warp's block
            const int64_t q = q0 + warp * 32 + rl;
            const uint4 o = stg[rl * 8 + (cj ^ (rl & 7))];
            const int col = s0 + c0 + cj * 4;
            if (q < nq) {
                int32_t *out = tau + q * S + col;
                if (col + 4 <= S && (S & 3) == 0) {
                    *reinterpret_cast<uint4 *>(out) = o;
                } else {
                    const uint32_t e[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int t = 0; t < 4; t++)
                        if (col + t < S) out[t] = (int32_t)e[t];
                }
            }
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(TN));
}

inline size_t seed_tau_umma_smem() { return (size_t)SMEM_A + SMEM_B + TN * 4; }

}  // namespace umma
}  // namespace vsag
