// keys.cuh -- candidate keys and small warp helpers shared by the search kernels.
//
// A candidate is the u64 key (tau ^ 2^31) << 32 | id << 1 | x: ascending key order is the
// total order (tau, id) of R-8 (ties to the smaller id; ids are < 2^31).  Bit 0 (x) is the
// pool's "expanded" flag.  It sits below the id, so it never changes the order of two
// different nodes' keys: no comparison needs to mask it.  Only an equality test between
// a new key and a pool entry of the same node (possible after the visited cache forgot
// an id) masks it (kmask).
#pragma once
#include <stdint.h>

namespace vsag {

constexpr uint64_t KEY_FLAG = 1ull;
constexpr uint64_t KEY_INF = 0xffffffffffffffffull;

__device__ __forceinline__ uint64_t kmask(uint64_t k) { return k & ~KEY_FLAG; }
__device__ __forceinline__ uint64_t make_key(int tau, int id) {
    return ((uint64_t)((uint32_t)tau ^ 0x80000000u) << 32) | ((uint32_t)id << 1);
}
// the same key from the order-preserving image u = tau ^ 2^31
__device__ __forceinline__ uint64_t make_key_u(uint32_t u, int id) { return ((uint64_t)u << 32) | ((uint32_t)id << 1); }
__device__ __forceinline__ int key_id(uint64_t k) { return (int)((uint32_t)k >> 1); }
__device__ __forceinline__ int key_tau(uint64_t k) { return (int)((uint32_t)(k >> 32) ^ 0x80000000u); }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
// 16-byte read-only global load (LDG.E.128.CONSTANT).
__device__ __forceinline__ uint4 ldg16(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
// Two predicated 16-byte read-only loads from one base (codes whose rows are not 32-byte
// aligned; aligned ones use ldg32).  A chunk whose flag is 0 is not loaded and reads as zero.
__device__ __forceinline__ void ldg16x2(const void *p, int stride, bool ok0, bool ok1, uint4 &a, uint4 &b) {
    a = make_uint4(0, 0, 0, 0);
    b = make_uint4(0, 0, 0, 0);
    const uint8_t *q = reinterpret_cast<const uint8_t *>(p);
    asm volatile(
        "{\n\t.reg .pred p0, p1;\n\t"
        "setp.ne.u32 p0, %10, 0;\n\tsetp.ne.u32 p1, %11, 0;\n\t"
        "@p0 ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%8];\n\t"
        "@p1 ld.global.nc.v4.u32 {%4, %5, %6, %7}, [%9];\n\t}"
        : "+r"(a.x), "+r"(a.y), "+r"(a.z), "+r"(a.w), "+r"(b.x), "+r"(b.y), "+r"(b.z), "+r"(b.w)
        : "l"(q), "l"(q + stride), "r"((uint32_t)ok0), "r"((uint32_t)ok1));
}
// Predicated 32-byte read-only global load (LDG.E.256 on sm_100; p must be 32-byte aligned):
// two adjacent 16-byte chunks of a code in one request.  Reads as zero when `ok` is false.
__device__ __forceinline__ void ldg32(const void *p, bool ok, uint4 &a, uint4 &b) {
    a = make_uint4(0, 0, 0, 0);
    b = make_uint4(0, 0, 0, 0);
    asm volatile(
        "{\n\t.reg .pred p0;\n\tsetp.ne.u32 p0, %9, 0;\n\t"
        "@p0 ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t}"
        : "+r"(a.x), "+r"(a.y), "+r"(a.z), "+r"(a.w), "+r"(b.x), "+r"(b.y), "+r"(b.z), "+r"(b.w)
        : "l"(p), "r"((uint32_t)ok));
}
// 16-byte read-only load that does not allocate in L1: re-rank rows are read once per query
// and would otherwise evict the codes that the SM's warps share (hub nodes).
__device__ __forceinline__ float4 ldg16_stream(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// Order-preserving float <-> u32 (-0 is mapped like +0).
__device__ __forceinline__ uint32_t ford(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u << 1) == 0) u = 0;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordf(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

}  // namespace vsag
