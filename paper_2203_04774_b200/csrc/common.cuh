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
// Shared address of the 32-bit word holding bit o of a bitmap at `base`:
// base + (o >> 5) * 4 as SHF + LEA (written as mad so ptxas does not turn it
// into SHF + LOP3 + IADD).
__device__ __forceinline__ unsigned bit_word(unsigned base, uint32_t o) {
    unsigned a;
    asm("{\n\t.reg .u32 w;\n\tshr.u32 w, %1, 5;\n\tmad.lo.u32 %0, w, 4, %2;\n\t}" : "=r"(a) : "r"(o), "r"(base));
    return a;
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
// L2 eviction-priority policies (createpolicy): rows re-read by many seeds
// are loaded evict_last, the rest evict_first, so the hot rows stay in L2.
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ldg4q / ldg2q with a per-load L2 policy (NA: no L1 allocation as ldg4q_na)
template <bool NA>
__device__ __forceinline__ void ldgq_pol(const uint4* const (&a)[4], const bool (&p)[4], const uint64_t (&pol)[4],
                                         uint4 (&v)[4]) {
    if constexpr (NA)
        asm volatile(
            "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
            "setp.ne.u32 q0, %16, 0;\n\t"
            "setp.ne.u32 q1, %17, 0;\n\t"
            "setp.ne.u32 q2, %18, 0;\n\t"
            "setp.ne.u32 q3, %19, 0;\n\t"
            "@q0 ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%20], %24;\n\t"
            "@q1 ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%4, %5, %6, %7}, [%21], %25;\n\t"
            "@q2 ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%8, %9, %10, %11}, [%22], %26;\n\t"
            "@q3 ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%12, %13, %14, %15}, [%23], %27;\n\t"
            "}"
            : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
              "+r"(v[1].w), "+r"(v[2].x), "+r"(v[2].y), "+r"(v[2].z), "+r"(v[2].w), "+r"(v[3].x), "+r"(v[3].y),
              "+r"(v[3].z), "+r"(v[3].w)
            : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "r"((unsigned)p[2]), "r"((unsigned)p[3]), "l"(a[0]),
              "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(pol[0]), "l"(pol[1]), "l"(pol[2]), "l"(pol[3]));
    else
        asm volatile(
            "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
            "setp.ne.u32 q0, %16, 0;\n\t"
            "setp.ne.u32 q1, %17, 0;\n\t"
            "setp.ne.u32 q2, %18, 0;\n\t"
            "setp.ne.u32 q3, %19, 0;\n\t"
            "@q0 ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%20], %24;\n\t"
            "@q1 ld.global.nc.L2::cache_hint.v4.u32 {%4, %5, %6, %7}, [%21], %25;\n\t"
            "@q2 ld.global.nc.L2::cache_hint.v4.u32 {%8, %9, %10, %11}, [%22], %26;\n\t"
            "@q3 ld.global.nc.L2::cache_hint.v4.u32 {%12, %13, %14, %15}, [%23], %27;\n\t"
            "}"
            : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
              "+r"(v[1].w), "+r"(v[2].x), "+r"(v[2].y), "+r"(v[2].z), "+r"(v[2].w), "+r"(v[3].x), "+r"(v[3].y),
              "+r"(v[3].z), "+r"(v[3].w)
            : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "r"((unsigned)p[2]), "r"((unsigned)p[3]), "l"(a[0]),
              "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(pol[0]), "l"(pol[1]), "l"(pol[2]), "l"(pol[3]));
}
template <bool NA>
__device__ __forceinline__ void ldgq_pol(const uint4* const (&a)[2], const bool (&p)[2], const uint64_t (&pol)[2],
                                         uint4 (&v)[2]) {
    asm volatile(
        "{\n\t.reg .pred q0, q1;\n\t"
        "setp.ne.u32 q0, %8, 0;\n\t"
        "setp.ne.u32 q1, %9, 0;\n\t"
        "@q0 ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%10], %12;\n\t"
        "@q1 ld.global.nc.L2::cache_hint.v4.u32 {%4, %5, %6, %7}, [%11], %13;\n\t"
        "}"
        : "+r"(v[0].x), "+r"(v[0].y), "+r"(v[0].z), "+r"(v[0].w), "+r"(v[1].x), "+r"(v[1].y), "+r"(v[1].z),
          "+r"(v[1].w)
        : "r"((unsigned)p[0]), "r"((unsigned)p[1]), "l"(a[0]), "l"(a[1]), "l"(pol[0]), "l"(pol[1]));
}

template <bool NA>
__device__ __forceinline__ void ldgq(const uint4* const (&a)[4], const bool (&p)[4], uint4 (&v)[4]) {
    if constexpr (NA) ldg4q_na(a, p, v);
    else ldg4q(a, p, v);
}
template <bool NA>
__device__ __forceinline__ void ldgq(const uint4* const (&a)[2], const bool (&p)[2], uint4 (&v)[2]) { ldg2q(a, p, v); }

// ---- mbarrier + bulk asynchronous copies (TMA engine, SASS UBLKCP) ----------
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// make barrier inits visible to the async proxy (the bulk copies' complete_tx)
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// order this thread's earlier generic-proxy shared accesses before later
// async-proxy (bulk copy) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned both
// sides) completing `bytes` of transaction count on `bar`
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s_pol(unsigned dst, const void* src, unsigned bytes, unsigned bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

}  // namespace trigpu
