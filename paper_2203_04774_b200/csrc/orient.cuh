// orient.cuh -- pi relabel, edge orientation and CSR construction (K1-K3, K7).
//
// Replaces OrientedView::OrientedView (reference core/src/oriented_view.cpp:7-47).
// The reference visits vertices by ascending rank so each successor /
// predecessor row comes out rank-ascending (:32-46). Here every id on the
// device is a RANK (the "pi relabel"): row r of the out-CSR holds the ranks of
// the successors of inverse[r], sorted ascending, which is exactly the
// reference's row order. Steps:
//   k_inverse         inverse[rank[v]] = v, bijection check (Ordering ctor checks,
//                     ordering.cpp:21-48; size check oriented_view.cpp:8-9)
//   k_relabel_count   warp per dense row: radj[e] = rank[adj[e]], out/in degree
//                     of rank[u] (oriented_view.cpp:18-26)
//   scan              degrees -> uint64 offsets (oriented_view.cpp:27-30)
//   k_scatter         warp per dense row: successor ranks into out row rank[u],
//                     predecessor ranks into in row rank[u] (oriented_view.cpp:34-46)
//   segmented sort    (segsort.cuh) makes every row ascending
//   k_cost            c_pp, c_pm, c_mm, sum_deg_sq (cost.cpp:27-38)
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace trigpu {

__global__ void k_inverse(uint32_t n, const uint32_t* __restrict__ rank, uint32_t* inv,
                          unsigned long long* err) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = rank[v];
        if (r >= n) {
            atomicOr(err, 1ull);
            continue;
        }
        if (atomicExch(&inv[r], static_cast<uint32_t>(v)) != kNone) atomicOr(err, 2ull);
    }
}

// Warp per dense row u: relabel neighbours to ranks (kept in radj for the
// scatter pass, so the random rank gather is paid once) and count d+ / d- of
// rank[u]. Also flags rows that are not strictly increasing / contain loops
// or out-of-range ids (the Graph invariants, graph.cpp:98-113) in *err.
__global__ void k_relabel_count(uint32_t n, const uint64_t* __restrict__ goff,
                                const uint32_t* __restrict__ gadj,
                                const uint32_t* __restrict__ rank, uint32_t* __restrict__ radj,
                                uint32_t* __restrict__ outdeg, uint32_t* __restrict__ indeg,
                                unsigned long long* err) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint64_t b = goff[u], e = goff[u + 1];
        const uint32_t ru = rank[u];
        uint32_t outc = 0;
        bool bad = e < b;
        for (uint64_t i = b + lane; i < e; i += 32) {
            const uint32_t v = gadj[i];
            bad |= v >= n || v == u || (i > b && gadj[i - 1] >= v);
            const uint32_t rv = v < n ? rank[v] : 0;
            radj[i] = rv;
            outc += rv > ru;
        }
        outc = __reduce_add_sync(FULL, outc);
        if (__any_sync(FULL, bad) && lane == 0) atomicOr(err, 4ull);
        if (lane == 0) {
            outdeg[ru] = outc;
            indeg[ru] = static_cast<uint32_t>(e - b) - outc;
        }
    }
}

// ---- exclusive scan of uint32 counts into uint64 offsets[0..n] ----------
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(uint32_t n, const uint32_t* __restrict__ cnt,
                                                                unsigned long long* __restrict__ part) {
    using BR = cub::BlockReduce<unsigned long long, kScanThreads>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
        if (i < n) s += cnt[i];
    }
    s = BR(tmp).Sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Single CTA: exclusive scan of the per-tile partials in place.
__global__ void __launch_bounds__(kScanThreads) k_scan_tops(uint64_t nparts, unsigned long long* part) {
    using BS = cub::BlockScan<unsigned long long, kScanThreads>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < nparts; base += kScanThreads) {
        const uint64_t i = base + threadIdx.x;
        unsigned long long v = i < nparts ? part[i] : 0, agg;
        BS(tmp).ExclusiveSum(v, v, agg);
        const unsigned long long c = carry;
        if (i < nparts) part[i] = v + c;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + agg;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(uint32_t n, const uint32_t* __restrict__ cnt,
                                                             const unsigned long long* __restrict__ part,
                                                             uint64_t* __restrict__ off) {
    using BS = cub::BlockScan<unsigned long long, kScanThreads>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    unsigned long long v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < n) ? cnt[base + k] : 0;
    unsigned long long agg;
    BS(tmp).ExclusiveSum(v, v, agg);
    const unsigned long long p = part[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) off[base + k] = p + v[k];
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) off[n] = p + agg;
}

// Warp per dense row u: successors go to out row rank[u], predecessors to in
// row rank[u], each in the row's dense-id order (sorted afterwards).
template <bool kIn>
__global__ void k_scatter(uint32_t n, const uint64_t* __restrict__ goff,
                          const uint32_t* __restrict__ radj, const uint32_t* __restrict__ rank,
                          const uint64_t* __restrict__ out_off, uint32_t* __restrict__ out_adj,
                          const uint64_t* __restrict__ in_off, uint32_t* __restrict__ in_adj) {
    const unsigned lane = lane_id();
    const unsigned lt = lanemask_lt();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint64_t b = goff[u], e = goff[u + 1];
        if (b == e) continue;
        const uint32_t ru = rank[u];
        uint64_t op = out_off[ru], ip = kIn ? in_off[ru] : 0;
        for (uint64_t base = b; base < e; base += 32) {
            const uint64_t i = base + lane;
            const bool act = i < e;
            const uint32_t rv = act ? radj[i] : 0;
            const bool isout = act && rv > ru;
            const unsigned mo = __ballot_sync(FULL, isout);
            if (isout) out_adj[op + __popc(mo & lt)] = rv;
            op += __popc(mo);
            if (kIn) {
                const bool isin = act && rv < ru;
                const unsigned mi = __ballot_sync(FULL, isin);
                if (isin) in_adj[ip + __popc(mi & lt)] = rv;
                ip += __popc(mi);
            }
        }
    }
}

// cost_report(view) (cost.cpp:27-38) from the rank-space degree arrays.
__global__ void __launch_bounds__(256) k_cost(uint32_t n, const uint32_t* __restrict__ outdeg,
                                              const uint32_t* __restrict__ indeg,
                                              unsigned long long* __restrict__ cost) {
    using BR = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename BR::TempStorage tmp;
    unsigned long long pp = 0, pm = 0, mm = 0, dd = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long o = outdeg[r], i = indeg[r];
        pp += o * o;
        pm += o * i;
        mm += i * i;
        dd += (o + i) * (o + i);
    }
    unsigned long long s;
    s = BR(tmp).Sum(pp);
    if (threadIdx.x == 0) atomicAdd(&cost[0], s);
    __syncthreads();
    s = BR(tmp).Sum(pm);
    if (threadIdx.x == 0) atomicAdd(&cost[1], s);
    __syncthreads();
    s = BR(tmp).Sum(mm);
    if (threadIdx.x == 0) atomicAdd(&cost[2], s);
    __syncthreads();
    s = BR(tmp).Sum(dd);
    if (threadIdx.x == 0) atomicAdd(&cost[3], s);
}

// max over rows of the out-degree (listing batch arithmetic is 32-bit).
// Checksum sink table: hv[r] = vertex_hash(inv[r]) (common.cuh).
__global__ void k_vertex_hash(uint32_t n, const uint32_t* __restrict__ inv, unsigned long long* __restrict__ hv) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) hv[r] = vertex_hash(inv[r]);
}

__global__ void k_maxdeg(uint32_t n, const uint32_t* __restrict__ deg, unsigned int* out) {
    uint32_t m = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, deg[r]);
    m = __reduce_max_sync(FULL, m);
    if (lane_id() == 0) atomicMax(out, m);
}

// ---- export helpers (tl_fetch_oriented / tl_fetch_vertex_counts) --------

// dense_deg[u] = deg[rank[u]]
__global__ void k_gather_u32(uint32_t n, const uint32_t* __restrict__ src,
                             const uint32_t* __restrict__ rank, uint32_t* __restrict__ dst) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        dst[u] = src[rank[u]];
}

__global__ void k_gather_u64(uint32_t n, const unsigned long long* __restrict__ src,
                             const uint32_t* __restrict__ rank, unsigned long long* __restrict__ dst) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        dst[u] = src[rank[u]];
}

// Warp per dense row u: copy rank-space row rank[u], mapped to dense ids.
__global__ void k_export_rows(uint32_t n, const uint32_t* __restrict__ rank,
                              const uint32_t* __restrict__ inv, const uint64_t* __restrict__ roff,
                              const uint32_t* __restrict__ radj, const uint64_t* __restrict__ doff,
                              uint32_t* __restrict__ dadj) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint32_t r = rank[u];
        const uint64_t b = roff[r], e = roff[r + 1], d = doff[u];
        for (uint64_t i = b + lane; i < e; i += 32) dadj[d + (i - b)] = inv[radj[i]];
    }
}

}  // namespace trigpu
