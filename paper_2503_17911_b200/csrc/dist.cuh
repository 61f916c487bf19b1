// dist.cuh -- tau_l on packed SQ codes, one 32-bit code word at a time (R-6 / R-7).
//
// "SQ ... directly compressing vector dimensions (e.g., FLOAT32 -> INT8/INT4) without
// requiring lookup tables" (§5.2).  On sm_100a each 4 dimensions of SQ8 L2 cost
// two SASS ops, VABSDIFF4.U8 + IDP.4A.U8.U8; IP uses IDP.4A.S8.U8 (int8 weights x u8
// codes); SQ4 first splits a word into its lo/hi nibble planes with two LOP3s.
// Accumulation is exact int32 (the index load rejects inputs that could overflow, R-20).
#pragma once
#include <stdint.h>

#include "vsag_internal.cuh"

namespace vsag {

__device__ __forceinline__ int dp4a_s8u8(uint32_t a_s8, uint32_t b_u8, int c) {
    int r;
    asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a_s8), "r"(b_u8), "r"(c));
    return r;
}

__device__ __forceinline__ int dp4a_u8u8(uint32_t a, uint32_t b, int c) {
    return (int)__dp4a(a, b, (unsigned int)c);
}

// acc += contribution of one code word `c` (4 code bytes).  q0/q1 are the matching
// operand words written by query_prep (q1 only used by the SQ4 modes).
template <int M>
__device__ __forceinline__ int word_dist(int acc, uint32_t q0, uint32_t q1, uint32_t c) {
    if (M == L2_8 || M == L2W_8) {
        const uint32_t t = __vabsdiffu4(q0, c);
        return dp4a_u8u8(t, t, acc);
    } else if (M == L2_4 || M == L2W_4) {
        const uint32_t cl = c & 0x0F0F0F0Fu, ch = (c >> 4) & 0x0F0F0F0Fu;
        const uint32_t t0 = __vabsdiffu4(q0, cl), t1 = __vabsdiffu4(q1, ch);
        return dp4a_u8u8(t1, t1, dp4a_u8u8(t0, t0, acc));
    } else if (M == IP_8) {
        return dp4a_s8u8(q0, c, acc);
    } else {
        const uint32_t cl = c & 0x0F0F0F0Fu, ch = (c >> 4) & 0x0F0F0F0Fu;
        return dp4a_s8u8(q1, ch, dp4a_s8u8(q0, cl, acc));
    }
}

// Weighted code-space L2 (NEXT-1b): acc += sum_i w_i * |cq_i - c_i|^2 over the word's
// dimensions; wd = the integer weights of those dimensions (4 for SQ8, 8 for SQ4, in
// dimension order).  Exact int32 (the weights' scale W keeps the sum below 2^31).
template <int M>
__device__ __forceinline__ int word_dist_w(int acc, uint32_t q0, uint32_t q1, uint32_t c, const int32_t *wd) {
    if (M == L2W_8) {
        const uint32_t t = __vabsdiffu4(q0, c);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int di = (int)((t >> (8 * i)) & 0xffu);
            acc += wd[i] * (di * di);
        }
        return acc;
    } else if (M == L2W_4) {
        const uint32_t cl = c & 0x0F0F0F0Fu, ch = (c >> 4) & 0x0F0F0F0Fu;
        const uint32_t t0 = __vabsdiffu4(q0, cl), t1 = __vabsdiffu4(q1, ch);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int a = (int)((t0 >> (8 * i)) & 0xffu), b = (int)((t1 >> (8 * i)) & 0xffu);
            acc += wd[2 * i] * (a * a) + wd[2 * i + 1] * (b * b);
        }
        return acc;
    } else {
        return word_dist<M>(acc, q0, q1, c);
    }
}

template <int M>
__device__ __forceinline__ int finish_tau(int acc) {
    return (M == IP_8 || M == IP_4) ? -acc : acc;
}

}  // namespace vsag
