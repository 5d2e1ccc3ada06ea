// common.cuh -- shared device helpers for the trigpu engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace trigpu {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;  // kInvalidVertex (common.hpp:13)

// splitmix64 finaliser; identical to oracle/oracle.c:or_mix64 and to the
// reference-harness checksum sink.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Order-independent triangle hash over DENSE ids: h(a) * h(b) * h(c) mod
// 2^64 with the odd vertex hash h(v) = mix64(v) | 1. Symmetric, so the device
// never sorts, and it factors: the checksum of all triangles (s, x, y) of one
// row is h(s) h(x) * sum_y h(y) -- one 64-bit multiply per row chunk.
__host__ __device__ __forceinline__ uint64_t vertex_hash(uint32_t v) { return mix64(v) | 1ull; }
__host__ __device__ __forceinline__ uint64_t tri_hash(uint32_t a, uint32_t b, uint32_t c) {
    return vertex_hash(a) * vertex_hash(b) * vertex_hash(c);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(FULL, static_cast<uint32_t>(v), src);
    uint32_t hi = __shfl_sync(FULL, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(FULL, v, o);
        if (lane >= static_cast<unsigned>(o)) v += t;
    }
    return v;
}

// Shared-memory accesses through 32-bit shared-window addresses (keeps
// pointers out of 64-bit registers and guarantees LDS/STS).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint4 lds128(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(unsigned a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(unsigned a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts64(unsigned a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}

// Four predicated 16-byte read-only loads in ONE asm block (all four in
// flight before any use); a lane whose predicate is off keeps its old values.
// The _na variant does not allocate the lines in L1 (the CTA classes: their
// rows are streamed once per seed, and L1 is better left to the checksum's
// vertex-hash gathers; measured 3 % faster for C1 / C2, slower for H / R).
__device__ __forceinline__ void ldg4q(const uint4* const (&a)[4], const bool (&p)[4], uint4 (&v)[4]) {
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
        "setp.ne.u32 q0, %16, 0;\n\t"
        "setp.ne.u32 q1, %17, 0;\n\t"
        "setp.ne.u32 q2, %18, 0;\n\t"
        "setp.ne.u32 q3, %19, 0;\n\t"
        "@q0 ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%20];\n\t"
        "@q1 ld.global.nc.v4.u32 {%4, %5, %6, %7}, [%21];\n\t"
        "@q2 ld.global.nc.v4.u32 {%8, %9, %10, %11}, [%22];\n\t"
        "@q3 ld.global.nc.v4.u32 {%12, %13, %14, %15}, [%23];\n\t"
        "}"
        : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
          "+r"(v[1].w), "+r"(v[2].x), "+r"(v[2].y), "+r"(v[2].z), "+r"(v[2].w), "+r"(v[3].x), "+r"(v[3].y),
          "+r"(v[3].z), "+r"(v[3].w)
        : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "r"((unsigned)p[2]), "r"((unsigned)p[3]), "l"(a[0]), "l"(a[1]),
          "l"(a[2]), "l"(a[3]));
}


__device__ __forceinline__ void ldg4q_na(const uint4* const (&a)[4], const bool (&p)[4], uint4 (&v)[4]) {
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
        "setp.ne.u32 q0, %16, 0;\n\t"
        "setp.ne.u32 q1, %17, 0;\n\t"
        "setp.ne.u32 q2, %18, 0;\n\t"
        "setp.ne.u32 q3, %19, 0;\n\t"
        "@q0 ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%20];\n\t"
        "@q1 ld.global.nc.L1::no_allocate.v4.u32 {%4, %5, %6, %7}, [%21];\n\t"
        "@q2 ld.global.nc.L1::no_allocate.v4.u32 {%8, %9, %10, %11}, [%22];\n\t"
        "@q3 ld.global.nc.L1::no_allocate.v4.u32 {%12, %13, %14, %15}, [%23];\n\t"
        "}"
        : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
          "+r"(v[1].w), "+r"(v[2].x), "+r"(v[2].y), "+r"(v[2].z), "+r"(v[2].w), "+r"(v[3].x), "+r"(v[3].y),
          "+r"(v[3].z), "+r"(v[3].w)
        : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "r"((unsigned)p[2]), "r"((unsigned)p[3]), "l"(a[0]), "l"(a[1]),
          "l"(a[2]), "l"(a[3]));
}

__device__ __forceinline__ void ldg2q(const uint4* const (&a)[2], const bool (&p)[2], uint4 (&v)[2]) {
    asm volatile(
        "{\n\t.reg .pred q0, q1;\n\t"
        "setp.ne.u32 q0, %8, 0;\n\t"
        "setp.ne.u32 q1, %9, 0;\n\t"
        "@q0 ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%10];\n\t"
        "@q1 ld.global.nc.v4.u32 {%4, %5, %6, %7}, [%11];\n\t"
        "}"
        : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
          "+r"(v[1].w)
        : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "l"(a[0]), "l"(a[1]));
}
template <bool NA>
__device__ __forceinline__ void ldgq(const uint4* const (&a)[4], const bool (&p)[4], uint4 (&v)[4]) {
    if constexpr (NA) ldg4q_na(a, p, v);
    else ldg4q(a, p, v);
}
template <bool NA>
__device__ __forceinline__ void ldgq(const uint4* const (&a)[2], const bool (&p)[2], uint4 (&v)[2]) { ldg2q(a, p, v); }

}  // namespace trigpu
