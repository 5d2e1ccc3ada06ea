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
// Device plan (64-bit item counts throughout; 48 bytes of scratch per raw edge):
//   1. endpoints of the non-loop edges (flags + DeviceSelect::Flagged), radix
//      sort, unique -> labels (the dedup cannot remove a label: duplicates
//      share endpoints, so this is the label set of the kept edges);
//   2. each raw edge -> one 64-bit key (min dense id << 32 | max dense id) by
//      binary search in the labels (the label -> id map is monotone, so the
//      min label gives the min id); loops -> ~0, which sorts last;
//   3. radix sort + unique of the keys: the kept edges in (a, b) order, i.e.
//      normalize's sorted, deduplicated edge list; the loop key is dropped;
//   4. both directions as (src << 32 | dst) keys, one radix sort gives the
//      sorted rows; offsets from degree counts + scan (from_dense_edges).
#pragma once

#include "common.cuh"

namespace trigpu {

constexpr unsigned long long kLoopKey = ~0ull;

// flags[2i] = flags[2i + 1] = edge i is not a loop
__global__ void k_loop_flags(uint64_t k, const long long* __restrict__ raw, unsigned char* __restrict__ flags,
                             unsigned long long* loops) {
    unsigned long long lc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const bool keep = raw[2 * i] != raw[2 * i + 1];
        flags[2 * i] = keep;
        flags[2 * i + 1] = keep;
        lc += !keep;
    }
    lc = warp_sum64(lc);
    if (lane_id() == 0 && lc) atomicAdd(loops, lc);
}

__device__ __forceinline__ uint32_t label_rank(const long long* __restrict__ labels, uint32_t n, long long x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (labels[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One undirected key per raw edge: (min id << 32 | max id), loops -> kLoopKey.
__global__ void k_edge_keys(uint64_t k, const long long* __restrict__ raw, const long long* __restrict__ labels,
                            uint32_t n, unsigned long long* __restrict__ keys) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const long long x = raw[2 * i], y = raw[2 * i + 1];
        if (x == y) {
            keys[i] = kLoopKey;
            continue;
        }
        const uint32_t u = label_rank(labels, n, x < y ? x : y), v = label_rank(labels, n, x < y ? y : x);
        keys[i] = (static_cast<unsigned long long>(u) << 32) | v;
    }
}

// Directed pair keys (src << 32 | dst) for both directions of the m kept
// edges, and the degree counts.
__global__ void k_directed_keys(uint64_t m, const unsigned long long* __restrict__ edges,
                                unsigned long long* __restrict__ keys, uint32_t* __restrict__ deg) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        const unsigned long long e = edges[i];
        const uint32_t u = static_cast<uint32_t>(e >> 32), v = static_cast<uint32_t>(e);
        keys[2 * i] = e;
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
