// normalize.cuh -- raw labeled edge list -> the reference's Graph CSR on the
// device.
//
// Reference: normalize (core/src/graph.cpp:115-151) + Graph::from_dense_edges
// (:13-56):
//   * loops dropped, each edge canonicalised to (min, max) label, duplicates
//     merged (stats: loops_removed, duplicates_removed);
//   * labels = the sorted distinct endpoint labels; dense id = rank of the
//     label (lower_bound);
//   * CSR rows = the sorted neighbour lists (uint64 offsets, uint32 ids).
// Device plan: canonicalise (loops -> a sentinel pair that sorts last), sort
// the pairs by (a, b) with two stable LSD radix sorts, flag first-of-run,
// compact; labels by radix sort + unique over the 2m endpoints; dense ids by
// binary search; the 2m directed pairs as 64-bit keys (src << 32 | dst), one
// radix sort gives the rows already sorted; offsets from a degree count + scan.
#pragma once

#include "common.cuh"

namespace trigpu {

constexpr long long kLoopSentinel = 0x7FFFFFFFFFFFFFFFll;

__global__ void k_canon_edges(uint64_t k, const long long* __restrict__ raw, long long* __restrict__ a,
                              long long* __restrict__ b, unsigned long long* loops) {
    unsigned long long lc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const long long x = raw[2 * i], y = raw[2 * i + 1];
        if (x == y) {
            a[i] = kLoopSentinel;
            b[i] = kLoopSentinel;
            ++lc;
        } else {
            a[i] = x < y ? x : y;
            b[i] = x < y ? y : x;
        }
    }
    lc = warp_sum64(lc);
    if (lane_id() == 0 && lc) atomicAdd(loops, lc);
}

// keep[i] = first of its (a, b) run and not a loop (pairs sorted by (a, b))
__global__ void k_first_of_run(uint64_t k, const long long* __restrict__ a, const long long* __restrict__ b,
                               unsigned char* __restrict__ keep) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const bool loop = a[i] == kLoopSentinel;
        keep[i] = !loop && (i == 0 || a[i] != a[i - 1] || b[i] != b[i - 1]);
    }
}

__global__ void k_interleave_endpoints(uint64_t m, const long long* __restrict__ a, const long long* __restrict__ b,
                                       long long* __restrict__ ends) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        ends[2 * i] = a[i];
        ends[2 * i + 1] = b[i];
    }
}

__device__ __forceinline__ uint32_t label_rank(const long long* __restrict__ labels, uint32_t n, long long x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (labels[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Directed pair keys (src << 32 | dst) for both directions of every edge,
// and the degree counts.
__global__ void k_dense_keys(uint64_t m, const long long* __restrict__ a, const long long* __restrict__ b,
                             const long long* __restrict__ labels, uint32_t n,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint32_t u = label_rank(labels, n, a[i]), v = label_rank(labels, n, b[i]);
        keys[2 * i] = (static_cast<unsigned long long>(u) << 32) | v;
        keys[2 * i + 1] = (static_cast<unsigned long long>(v) << 32) | u;
        atomicAdd(&deg[u], 1u);
        atomicAdd(&deg[v], 1u);
    }
}

__global__ void k_low_words(uint64_t k, const unsigned long long* __restrict__ keys, uint32_t* __restrict__ adj) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride)
        adj[i] = static_cast<uint32_t>(keys[i]);
}

// out[i] = labels[ids[i]] (list output mapped to the Graph's labels)
__global__ void k_map_labels(uint64_t cnt, const uint32_t* __restrict__ ids, const long long* __restrict__ labels,
                             long long* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += stride) out[i] = labels[ids[i]];
}

}  // namespace trigpu
