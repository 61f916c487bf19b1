// seed_umma.cuh -- row a5, part 1 on the tensor cores: tau_l of every entry node for every
// query as an 8-bit contraction on tcgen05 (kind::i8): L2 (u8 query codes x u8 codes) and IP
// (s8 query weights x u8 codes, R-7: tau_l = -sum w_d c_d), SQ8 and SQ4.
//
// Alg. 1 line 3 evaluates tau_l(x_q, s) for every initial node s.  For L2 the
// code-space distance splits exactly, in integers, as |cq|^2 + |c_s|^2 - 2 cq.c_s (the
// decomposition of P:649; u8 products summed in int32 are exact), so the S x nq grid is a
// dense [nq x K] . [K x S] contraction.  A CTA owns 128 queries x 256 seeds:
//   - TMA (cp.async.bulk.tensor.2d, 128-byte swizzle) stages the query operand tile A
//     (128 rows x 128 bytes of K) and the seed operand tile B (256 rows x 128 bytes) per K
//     block into a two-stage ring, completion on an mbarrier (expect_tx);
//   - one thread issues tcgen05.mma.cta_group::1.kind::i8 (M 128, N 256, K 32; four per K
//     block; SWIZZLE_128B K-major shared-memory descriptors) into a 128 x 256 int32
//     accumulator in tensor memory and commits to a second mbarrier;
//   - every thread reads its query's row back with tcgen05.ld.32x32b.x32 and writes
//     tau = |cq|^2 + |c_s|^2 - 2 dot (IP: -dot), staged per warp in shared memory so that
//     global stores are row-contiguous whole sectors.
// The seed operand is the seed-code block for SQ8, and for SQ4 the codes unpacked to one
// nibble per byte in the query operand's plane order (per code word: its low nibbles as 4
// bytes, then its high nibbles), built once at index load (seed.cu).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace vsag {
namespace umma {

constexpr int TM = 128, TN = 256, KB = 128;  // tile rows (queries), columns (seeds), K block (bytes)
constexpr int SMEM_A = TM * KB, SMEM_B = TN * KB, STAGE = SMEM_A + SMEM_B;
constexpr int STAGES = 2;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Shared-memory matrix descriptor (sm_100), K-major with the 128-byte swizzle: start >> 4 in
// [0, 14), leading-dimension byte offset >> 4 in [16, 30) (unused for swizzled K-major, 1),
// stride-dimension byte offset >> 4 in [32, 46) (1024: 8 rows of 128 bytes), version 1 at 46,
// base offset 0 (tiles are 1024-byte aligned), layout type 2 (SWIZZLE_128B) in [61, 64).
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
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
// completion): the caller reports it through the index's error flag instead of hanging the
// GPU or trapping (a trap would leave a sticky context error).
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

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

// 16-byte chunk c of row r of a 128-byte-swizzled tile (8-row groups of 1 KB, chunk index
// XOR row % 8): what TMA wrote and what the MMA descriptor reads.
__device__ __forceinline__ const uint4 *sw128_chunk(const uint8_t *tile, int r, int c) {
    return reinterpret_cast<const uint4 *>(tile + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// tau[q, s] for q in [q0, q0 + 128), s in [s0, s0 + 256).  128 threads (4 warps); warp w
// reads tensor-memory lanes 32 w .. 32 w + 31 = the tile's queries 32 w .. 32 w + 31.
// ta: the query operand [nq rows x kbytes] (u8 codes for L2, s8 weights for IP); tb: the seed
// operand [S rows x kbytes] (u8).  Rows past nq / S and K past kbytes are zero-filled by TMA.
template <bool IP>
__global__ void __launch_bounds__(128) seed_tau_umma_kernel(const __grid_constant__ CUtensorMap ta,
                                                            const __grid_constant__ CUtensorMap tb, int64_t nq, int S,
                                                            int kbytes, int32_t *__restrict__ tau, int *err) {
    extern __shared__ uint8_t smem_raw[];
    // SWIZZLE_128B tiles need 1024-byte alignment
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int nk = (kbytes + KB - 1) / KB;
    int32_t *snorm = reinterpret_cast<int32_t *>(smem + (nk > 1 ? 2 : 1) * STAGE);  // [TN] |c_s|^2
    __shared__ __align__(8) uint64_t full[STAGES], mma_done[STAGES];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t q0 = (int64_t)blockIdx.x * TM;
    const int s0 = blockIdx.y * TN;

    auto issue_loads = [&](int kb) {  // (thread 0) K block kb -> stage kb % 2
        const int st = kb & 1;
        uint8_t *sa = smem + st * STAGE, *sb = sa + SMEM_A;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])),
                     "r"((uint32_t)STAGE)
                     : "memory");
        tma_load_2d(smem_u32(sa), &ta, kb * KB, (int)q0, smem_u32(&full[st]));
        tma_load_2d(smem_u32(sb), &tb, kb * KB, s0, smem_u32(&full[st]));
    };
    // the first loads go out before the tensor-memory allocation, which may wait for another
    // CTA on this SM to release its columns
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
        for (int i = 0; i < STAGES; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mma_done[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        issue_loads(0);
        if (nk > 1) issue_loads(1);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "n"(TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;
    // |cq|^2 of this thread's query row and |c_s|^2 of its two seed rows, accumulated from the
    // staged tiles block by block (shared-memory reads; no extra global traffic)
    int qn = 0, sn0 = 0, sn1 = 0;
    bool ok = true;
    for (int kb = 0; kb < nk; kb++) {
        const int st = kb & 1;
        const uint8_t *sa = smem + st * STAGE, *sb = sa + SMEM_A;
        ok &= mbar_wait(smem_u32(&full[st]), (uint32_t)((kb >> 1) & 1));
        if (!IP) {
#pragma unroll
            for (int c = 0; c < KB / 16; c++) {
                const uint4 a4 = *sw128_chunk(sa, tid, c);
                qn = (int)__dp4a(a4.x, a4.x, __dp4a(a4.y, a4.y, __dp4a(a4.z, a4.z, __dp4a(a4.w, a4.w, (unsigned)qn))));
                const uint4 b0 = *sw128_chunk(sb, tid, c), b1 = *sw128_chunk(sb, tid + 128, c);
                sn0 = (int)__dp4a(b0.x, b0.x, __dp4a(b0.y, b0.y, __dp4a(b0.z, b0.z, __dp4a(b0.w, b0.w, (unsigned)sn0))));
                sn1 = (int)__dp4a(b1.x, b1.x, __dp4a(b1.y, b1.y, __dp4a(b1.z, b1.z, __dp4a(b1.w, b1.w, (unsigned)sn1))));
            }
        }
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int ks = 0; ks < KB / 32; ks++) {  // K = 32 bytes per MMA: +32 bytes inside the swizzle atom
                const uint64_t ad = make_desc_sw128(smem_u32(sa) + ks * 32);
                const uint64_t bd = make_desc_sw128(smem_u32(sb) + ks * 32);
                const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                    "l"(ad), "l"(bd), "r"(idesc<IP>()), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mma_done[st])));
        }
        if (kb + 2 < nk) {
            __syncthreads();  // every thread's norm reads of this stage are done
            if (tid == 0) {
                ok &= mbar_wait(smem_u32(&mma_done[st]), (uint32_t)((kb >> 1) & 1));  // the MMAs read it
                issue_loads(kb + 2);
            }
        }
    }
    {  // the last commit tracks every MMA issued before it
        const int kl = nk - 1;
        ok &= mbar_wait(smem_u32(&mma_done[kl & 1]), (uint32_t)((kl >> 1) & 1));
    }
    if (!ok) *reinterpret_cast<volatile int *>(err) = 1;  // (mapped host flag) reported by the API (vsag.h)
    asm volatile("tcgen05.fence::after_thread_sync;");
    snorm[tid] = sn0;
    snorm[tid + 128] = sn1;
    __syncthreads();  // norms visible; the stage buffers are free for the epilogue
    // epilogue: this thread's query row, 32 columns at a time
    const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
    uint4 *stg = reinterpret_cast<uint4 *>(smem) + warp * 32 * 8;  // [32 rows][8 chunks] per warp
    const int lane = tid & 31, cj = lane & 7;
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
        // stage the warp's 32 x 32 block in shared memory (16-byte chunks XOR-swizzled by row),
        // then write it back row-contiguously: 8 lanes per 128-byte row segment, so every
        // global store fills whole sectors
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            uint4 o;
            o.x = (uint32_t)(IP ? -(int)v[j] : qn + snorm[c0 + j] - 2 * (int)v[j]);
            o.y = (uint32_t)(IP ? -(int)v[j + 1] : qn + snorm[c0 + j + 1] - 2 * (int)v[j + 1]);
            o.z = (uint32_t)(IP ? -(int)v[j + 2] : qn + snorm[c0 + j + 2] - 2 * (int)v[j + 2]);
            o.w = (uint32_t)(IP ? -(int)v[j + 3] : qn + snorm[c0 + j + 3] - 2 * (int)v[j + 3]);
            stg[lane * 8 + ((j >> 2) ^ (lane & 7))] = o;
        }
        __syncwarp();
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

// dynamic shared memory: the stages used (one for a single K block) + norms + alignment slack
inline size_t seed_tau_umma_smem(int kbytes) { return (size_t)(kbytes > KB ? 2 : 1) * STAGE + TN * 4 + 1024; }

}  // namespace umma
}  // namespace vsag
