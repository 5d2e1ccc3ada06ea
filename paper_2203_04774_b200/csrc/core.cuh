// core.cuh -- k-core decomposition and a degeneracy (core) ordering on the device.
//
// Reference: core_decompose / core_order (core/src/ordering.cpp:141-188,
// ordering.hpp:56-64): Batagelj-Zaversnik bucket peeling, one vertex at a
// time; coreness[v] = degree of v at its removal, degeneracy = max coreness,
// order = the removal sequence.
//
// The bucket queue is sequential by construction (every decrement swaps two
// entries of one shared array), so the device peels level-synchronously
// instead: at level k every vertex of current degree <= k is removed, round by
// round, until none is left, then k moves to the smallest remaining degree.
//   * coreness and degeneracy are order-independent: they equal the
//     reference's bit for bit (tests compare them with core_decompose).
//   * the ORDER is (removal round, vertex id) ascending. It is a degeneracy
//     ordering with the reference order's defining property - every vertex has
//     at most coreness(v) successors, so max d+ = degeneracy - but among
//     vertices the reference removes at the same degree it differs from the
//     reference's swap-dependent sequence. Listing results do not depend on
//     pi; the costs c_pp / c_pm under the two orders are reported side by side.
#pragma once

#include "common.cuh"

namespace trigpu {

struct CoreState {
    const uint64_t* off;  // Graph CSR (graph.hpp:20-62)
    const uint32_t* adj;
    uint32_t* deg;        // current degree (<= k once a vertex is removed or queued)
    uint32_t* rnd;        // removal round (kNone: not removed yet)
    uint32_t* core;       // coreness
};

// acc: [0] frontier count, [1] kept count, [2] smallest degree among the kept
__global__ void k_core_init(uint32_t n, CoreState S, uint32_t* __restrict__ alive) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        S.deg[v] = static_cast<uint32_t>(S.off[v + 1] - S.off[v]);
        S.rnd[v] = kNone;
        alive[v] = static_cast<uint32_t>(v);
    }
}

// Start of level k (round r): the vertices of `alive` not removed yet are split
// into the level's first frontier (degree <= k; marked removed) and the kept
// list; the kept list's smallest degree is the next non-empty level.
__global__ void __launch_bounds__(256) k_core_scan(const uint32_t* __restrict__ alive, uint32_t nalive, CoreState S,
                                                   uint32_t k, uint32_t r, uint32_t* __restrict__ frontier,
                                                   uint32_t* __restrict__ kept, unsigned int* __restrict__ acc) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t start = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t trips = ((uint64_t)nalive + stride - 1) / stride;
    uint32_t mind = kNone;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t i = start + t * stride;
        int what = 0;  // 1: frontier, 2: kept
        uint32_t v = 0;
        if (i < nalive) {
            v = alive[i];
            if (S.rnd[v] == kNone) {
                const uint32_t d = S.deg[v];
                what = d <= k ? 1 : 2;
                if (what == 2) mind = min(mind, d);
            }
        }
#pragma unroll
        for (int w = 1; w <= 2; ++w) {
            const unsigned b = __ballot_sync(FULL, what == w);
            if (!b) continue;
            const unsigned leader = __ffs(b) - 1;
            unsigned base = 0;
            if (lane_id() == leader) base = atomicAdd(&acc[w - 1], __popc(b));
            base = __shfl_sync(FULL, base, leader);
            if (what == w) (w == 1 ? frontier : kept)[base + __popc(b & lanemask_lt())] = v;
        }
        if (what == 1) {
            S.rnd[v] = r;
            S.core[v] = k;
        }
    }
    mind = __reduce_min_sync(FULL, mind);
    if (lane_id() == 0 && mind != kNone) atomicMin(&acc[2], mind);
}

// One round of level k: every frontier vertex leaves the graph; a neighbour
// whose degree drops to k joins the next frontier (round r). A warp per
// frontier vertex; a decrement that finds the neighbour already at <= k
// (removed, queued, or raced) is undone.
__device__ __forceinline__ void core_relax(const CoreState& S, uint32_t u, uint32_t k, uint32_t r,
                                           uint32_t* __restrict__ next, unsigned int* __restrict__ next_count) {
    if (__ldcg(S.deg + u) <= k) return;  // L2 read: degrees change under this kernel's atomics
    const uint32_t old = atomicSub(&S.deg[u], 1u);
    if (old == k + 1u) {
        S.rnd[u] = r;
        S.core[u] = k;
        next[atomicAdd(next_count, 1u)] = u;
    } else if (old <= k) {
        atomicAdd(&S.deg[u], 1u);
    }
}

__global__ void __launch_bounds__(256) k_core_peel(const uint32_t* __restrict__ frontier, uint32_t count, CoreState S,
                                                   uint32_t k, uint32_t r, uint32_t* __restrict__ next,
                                                   unsigned int* __restrict__ next_count) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < count; i += warps) {
        const uint32_t v = frontier[i];
        const uint64_t b = S.off[v], e = S.off[v + 1];
        for (uint64_t j = b + lane; j < e; j += 32) core_relax(S, S.adj[j], k, r, next, next_count);
    }
}

// Small frontiers: one CTA runs the rounds of level k back to back (no host
// round trip per round) while the frontier fits its two shared queues. On exit
// state[0] = rounds run, state[1] = size of the frontier left in `spill`
// (0: the level is finished).
constexpr uint32_t kCoreQ = 2048;
__global__ void __launch_bounds__(1024) k_core_peel_small(const uint32_t* __restrict__ frontier, uint32_t count,
                                                          CoreState S, uint32_t k, uint32_t r0,
                                                          uint32_t* __restrict__ spill, unsigned int* __restrict__ state) {
    __shared__ uint32_t q[2][kCoreQ];
    __shared__ unsigned int qn[2];
    __shared__ unsigned int overflow;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) q[0][i] = frontier[i];
    if (threadIdx.x == 0) {
        qn[0] = count;
        qn[1] = 0;
        overflow = 0;
    }
    __syncthreads();
    uint32_t cur = 0, r = r0, rounds = 0;
    for (;;) {
        const uint32_t c = qn[cur];
        if (c == 0) break;
        // next frontier into q[cur ^ 1]; entries past kCoreQ go to `spill`
        for (uint32_t i = warp; i < c; i += nw) {
            const uint32_t v = q[cur][i];
            const uint64_t b = S.off[v], e = S.off[v + 1];
            for (uint64_t j = b + lane; j < e; j += 32) {
                const uint32_t u = S.adj[j];
                if (__ldcg(S.deg + u) <= k) continue;
                const uint32_t old = atomicSub(&S.deg[u], 1u);
                if (old == k + 1u) {
                    S.rnd[u] = r;
                    S.core[u] = k;
                    const unsigned slot = atomicAdd(&qn[cur ^ 1], 1u);
                    if (slot < kCoreQ) q[cur ^ 1][slot] = u;
                    else spill[slot] = u;
                } else if (old <= k) {
                    atomicAdd(&S.deg[u], 1u);
                }
            }
        }
        __syncthreads();
        ++rounds;
        ++r;
        const uint32_t nn = qn[cur ^ 1];
        if (nn > kCoreQ) {  // too big for the CTA: hand the frontier back
            for (uint32_t i = threadIdx.x; i < kCoreQ; i += blockDim.x) spill[i] = q[cur ^ 1][i];
            if (threadIdx.x == 0) overflow = nn;
            __syncthreads();
            break;
        }
        if (threadIdx.x == 0) qn[cur] = 0;
        cur ^= 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        state[0] = rounds;
        state[1] = overflow;
    }
}

__global__ void k_core_iota(uint32_t n, uint32_t* __restrict__ val) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride)
        val[v] = static_cast<uint32_t>(v);
}

}  // namespace trigpu
