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

// Graph CSR offsets: offsets[0] == 0, non-decreasing, offsets[n] == 2m
// (graph.hpp:20-62). Flag 8 in *err otherwise; checked before any kernel
// indexes the adjacency through them.
__global__ void k_check_offsets(uint32_t n, uint64_t m2, const uint64_t* __restrict__ off,
                                unsigned long long* err) {
    bool bad = false;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = off[v];
        if (v == 0) bad |= o != 0;
        else bad |= off[v - 1] > o;
        if (v == n) bad |= o != m2;
    }
    if (bad) atomicOr(err, 8ull);
}

// Rows of one warp: 32 consecutive dense rows, one per lane. Rows of fewer
// than kLongDeg edges are compacted to the low lanes and walked as ONE
// flattened stream (lane f of a 32-wide window takes element f of the
// concatenated rows; its row comes from an OR-reduction of the row starts),
// two windows per step, so the many short rows of a power-law graph keep all
// lanes busy. Longer rows go to a list and get a whole CTA each (the *_long
// kernels): R-MAT's top hub alone has ~0.14 % of all edge endpoints, which one
// warp would walk serially.
constexpr uint32_t kLongDeg = 1024;
constexpr int kLongThreads = 512;

struct FlatRows {  // compacted short rows of a warp (lane j: row j)
    uint64_t rbase;   // element f of the stream lives at rbase(row) + f
    uint32_t start;   // stream position of the row's first element
    uint32_t deg, total;
    int cnt;          // rows
    int src;          // original lane of compacted row j
};

__device__ __forceinline__ FlatRows flat_rows(uint64_t b, uint32_t deg) {
    const unsigned lane = lane_id();
    const unsigned ne = __ballot_sync(FULL, deg != 0);
    FlatRows f;
    f.cnt = __popc(ne);
    f.src = lane < (unsigned)f.cnt ? (int)__fns(ne, 0, lane + 1) : 0;
    const uint64_t cb = shfl64(b, f.src);
    const uint32_t dsrc = __shfl_sync(FULL, deg, f.src);
    f.deg = lane < (unsigned)f.cnt ? dsrc : 0u;
    const uint32_t incl = warp_incl_scan(f.deg);
    f.total = __shfl_sync(FULL, incl, 31);
    f.start = incl - f.deg;
    f.rbase = cb - f.start;
    return f;
}

// Rows (compacted index) of stream elements base + lane and base + 32 + lane;
// `before` carries the rows started in earlier windows.
__device__ __forceinline__ void flat_row2(const FlatRows& f, uint32_t base, int& before, int& jA, int& jB) {
    const uint32_t rel = f.start - base;  // wraps when start < base: no bit
    const bool in = f.deg != 0 && f.start >= base;
    const unsigned bitA = (in && rel < 32u) ? (1u << rel) : 0u;
    const unsigned bitB = (in && rel - 32u < 32u) ? (1u << (rel - 32u)) : 0u;
    const unsigned MA = __reduce_or_sync(FULL, bitA);
    const unsigned MB = __reduce_or_sync(FULL, bitB);
    const unsigned le = lanemask_le();
    const int ca = __popc(MA);
    jA = before + __popc(MA & le) - 1;
    jB = before + ca + __popc(MB & le) - 1;
    before += ca + __popc(MB);
    jA = jA > 31 ? 31 : (jA < 0 ? 0 : jA);
    jB = jB > 31 ? 31 : (jB < 0 ? 0 : jB);
}

__device__ __forceinline__ void push_long(bool is_long, uint32_t u, uint32_t* list, unsigned int* count) {
    const unsigned b = __ballot_sync(FULL, is_long);
    if (!b) return;
    unsigned base = 0;
    if (lane_id() == 0) base = atomicAdd(count, __popc(b));
    base = __shfl_sync(FULL, base, 0);
    if (is_long) list[base + __popc(b & lanemask_lt())] = u;
}

// Relabel neighbours to ranks (kept in radj for the scatter pass, so the
// random rank gather is paid once) and count d+ / d- of rank[u]. Also flags
// rows that are not strictly increasing / contain loops or out-of-range ids
// (the Graph invariants, graph.cpp:98-113) in *err.
__global__ void __launch_bounds__(256) k_relabel_count(uint32_t n, const uint64_t* __restrict__ goff,
                                                       const uint32_t* __restrict__ gadj,
                                                       const uint32_t* __restrict__ rank, uint32_t* __restrict__ radj,
                                                       uint32_t* __restrict__ outdeg, uint32_t* __restrict__ indeg,
                                                       uint32_t* __restrict__ long_rows, unsigned int* long_count,
                                                       unsigned long long* err) {
    __shared__ uint32_t cnt_sm[8][32];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t groups = ((uint64_t)n + 31) >> 5;
    for (uint64_t grp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; grp < groups; grp += warps) {
        const uint64_t u = grp * 32 + lane;
        const bool valid = u < n;
        uint64_t b = 0, e = 0;
        uint32_t ru = 0;
        if (valid) {
            b = goff[u];
            e = goff[u + 1];
            ru = rank[u];
        }
        bool bad = e < b;
        const uint32_t deg = bad ? 0u : static_cast<uint32_t>(e - b);
        push_long(valid && deg >= kLongDeg, static_cast<uint32_t>(u), long_rows, long_count);
        if (valid && deg == 0) {
            outdeg[ru] = 0;
            indeg[ru] = 0;
        }
        const FlatRows f = flat_rows(b, deg < kLongDeg ? deg : 0u);
        const uint32_t cu = __shfl_sync(FULL, static_cast<uint32_t>(u), f.src);
        const uint32_t cr = __shfl_sync(FULL, ru, f.src);
        cnt_sm[warp][lane] = 0;
        __syncwarp();
        int before = 0;
        uint32_t carry = 0;  // last element of the previous window
        for (uint32_t base = 0; base < f.total; base += 64) {
            int jA, jB;
            flat_row2(f, base, before, jA, jB);
            const uint32_t fA = base + lane, fB = fA + 32;
            const bool actA = fA < f.total, actB = fB < f.total;
            const uint64_t iA = shfl64(f.rbase, jA) + fA, iB = shfl64(f.rbase, jB) + fB;
            const uint32_t vA = actA ? gadj[iA] : 0u, vB = actB ? gadj[iB] : 0u;
            const uint32_t rvA = actA && vA < n ? rank[vA] : 0u, rvB = actB && vB < n ? rank[vB] : 0u;
            const uint32_t uA = __shfl_sync(FULL, cu, jA), uB = __shfl_sync(FULL, cu, jB);
            const uint32_t rA = __shfl_sync(FULL, cr, jA), rB = __shfl_sync(FULL, cr, jB);
            const uint32_t sA = __shfl_sync(FULL, f.start, jA), sB = __shfl_sync(FULL, f.start, jB);
            uint32_t pA = __shfl_up_sync(FULL, vA, 1), pB = __shfl_up_sync(FULL, vB, 1);
            const uint32_t lastA = __shfl_sync(FULL, vA, 31), lastB = __shfl_sync(FULL, vB, 31);
            if (lane == 0) {
                pA = carry;
                pB = lastA;
            }
            carry = lastB;
            if (actA) {
                bad |= vA >= n || vA == uA || (fA > sA && pA >= vA);
                radj[iA] = rvA;
            }
            if (actB) {
                bad |= vB >= n || vB == uB || (fB > sB && pB >= vB);
                radj[iB] = rvB;
            }
            const bool oA = actA && rvA > rA, oB = actB && rvB > rB;
            const unsigned gA = __match_any_sync(FULL, actA ? jA : 64), gB = __match_any_sync(FULL, actB ? jB : 64);
            const unsigned cA = __popc(__ballot_sync(FULL, oA) & gA), cB = __popc(__ballot_sync(FULL, oB) & gB);
            if (actA && (gA & lt) == 0) cnt_sm[warp][jA] += cA;  // group leaders
            __syncwarp();
            if (actB && (gB & lt) == 0) cnt_sm[warp][jB] += cB;
            __syncwarp();
        }
        if (lane < (unsigned)f.cnt) {
            const uint32_t c = cnt_sm[warp][lane];
            outdeg[cr] = c;
            indeg[cr] = f.deg - c;
        }
        __syncwarp();
        if (__any_sync(FULL, bad) && lane == 0) atomicOr(err, 4ull);
    }
}

// The rows of kLongDeg or more edges: one CTA per row (dynamic queue), four
// loads in flight per thread.
__global__ void __launch_bounds__(kLongThreads) k_relabel_long(uint32_t n, const uint64_t* __restrict__ goff,
                                                               const uint32_t* __restrict__ gadj,
                                                               const uint32_t* __restrict__ rank,
                                                               uint32_t* __restrict__ radj, uint32_t* __restrict__ outdeg,
                                                               uint32_t* __restrict__ indeg,
                                                               const uint32_t* __restrict__ long_rows,
                                                               const unsigned int* long_count, unsigned int* queue,
                                                               unsigned long long* err) {
    using BR = cub::BlockReduce<unsigned, kLongThreads>;
    __shared__ typename BR::TempStorage tmp;
    __shared__ unsigned item;
    const unsigned total = *long_count;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) item = atomicAdd(queue, 1u);
        __syncthreads();
        if (item >= total) break;
        const uint32_t u = long_rows[item];
        const uint64_t b = goff[u], e = goff[u + 1];
        const uint32_t ru = rank[u];
        unsigned c = 0;
        bool bad = false;
        for (uint64_t i0 = b + threadIdx.x; i0 < e; i0 += 4 * kLongThreads) {
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t i = i0 + (uint64_t)k * kLongThreads;
                v[k] = i < e ? gadj[i] : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t i = i0 + (uint64_t)k * kLongThreads;
                if (i < e) {
                    bad |= v[k] >= n || v[k] == u || (i > b && gadj[i - 1] >= v[k]);
                    const uint32_t rv = v[k] < n ? rank[v[k]] : 0u;
                    radj[i] = rv;
                    c += rv > ru;
                }
            }
        }
        const unsigned tot = BR(tmp).Sum(c);
        if (threadIdx.x == 0) {
            outdeg[ru] = tot;
            indeg[ru] = static_cast<uint32_t>(e - b) - tot;
        }
        if (bad) atomicOr(err, 4ull);
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

// Successors of dense row u go to out row rank[u] (order within the row is
// free: rows are sorted afterwards). Same row layout as k_relabel_count.
__global__ void __launch_bounds__(256) k_scatter(uint32_t n, const uint64_t* __restrict__ goff,
                                                 const uint32_t* __restrict__ radj, const uint32_t* __restrict__ rank,
                                                 const uint64_t* __restrict__ out_off, const uint32_t* __restrict__ outdeg,
                                                 uint32_t* __restrict__ out_adj) {
    __shared__ uint32_t cnt_sm[8][32];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t groups = ((uint64_t)n + 31) >> 5;
    for (uint64_t grp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; grp < groups; grp += warps) {
        const uint64_t u = grp * 32 + lane;
        uint64_t b = 0, e = 0, op = 0;
        uint32_t ru = 0;
        if (u < n) {
            b = goff[u];
            e = goff[u + 1];
        }
        const uint32_t deg = static_cast<uint32_t>(e - b);
        if (deg && deg < kLongDeg) {
            ru = rank[u];
            op = out_off[ru];
            // the row's pad slots (out-rows are padded to a multiple of 4: quads)
            for (uint32_t k = outdeg[ru]; k & 3u; ++k) out_adj[op + k] = kNone;
        }
        const FlatRows f = flat_rows(b, deg < kLongDeg ? deg : 0u);
        const uint32_t cr = __shfl_sync(FULL, ru, f.src);
        const uint64_t cop = shfl64(op, f.src);
        cnt_sm[warp][lane] = 0;
        __syncwarp();
        int before = 0;
        for (uint32_t base = 0; base < f.total; base += 64) {
            int jA, jB;
            flat_row2(f, base, before, jA, jB);
            const uint32_t fA = base + lane, fB = fA + 32;
            const bool actA = fA < f.total, actB = fB < f.total;
            const uint64_t iA = shfl64(f.rbase, jA) + fA, iB = shfl64(f.rbase, jB) + fB;
            const uint32_t rvA = actA ? radj[iA] : 0u, rvB = actB ? radj[iB] : 0u;
            const uint32_t rA = __shfl_sync(FULL, cr, jA), rB = __shfl_sync(FULL, cr, jB);
            const uint64_t opA = shfl64(cop, jA), opB = shfl64(cop, jB);
            const bool oA = actA && rvA > rA, oB = actB && rvB > rB;
            const unsigned gA = __match_any_sync(FULL, actA ? jA : 64), gB = __match_any_sync(FULL, actB ? jB : 64);
            const unsigned bA = __ballot_sync(FULL, oA) & gA, bB = __ballot_sync(FULL, oB) & gB;
            const uint32_t cA = cnt_sm[warp][jA];
            if (oA) out_adj[opA + cA + __popc(bA & lt)] = rvA;
            __syncwarp();
            if (actA && (gA & lt) == 0) cnt_sm[warp][jA] = cA + __popc(bA);  // group leaders
            __syncwarp();
            const uint32_t cB = cnt_sm[warp][jB];
            if (oB) out_adj[opB + cB + __popc(bB & lt)] = rvB;
            __syncwarp();
            if (actB && (gB & lt) == 0) cnt_sm[warp][jB] = cB + __popc(bB);
            __syncwarp();
        }
    }
}

// Long rows: one CTA per row, positions from a shared cursor.
__global__ void __launch_bounds__(kLongThreads) k_scatter_long(const uint64_t* __restrict__ goff,
                                                               const uint32_t* __restrict__ radj,
                                                               const uint32_t* __restrict__ rank,
                                                               const uint64_t* __restrict__ out_off,
                                                               const uint32_t* __restrict__ outdeg,
                                                               uint32_t* __restrict__ out_adj,
                                                               const uint32_t* __restrict__ long_rows,
                                                               const unsigned int* long_count, unsigned int* queue) {
    __shared__ unsigned item, cursor;
    const unsigned lt = lanemask_lt();
    const unsigned total = *long_count;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            item = atomicAdd(queue, 1u);
            cursor = 0;
        }
        __syncthreads();
        if (item >= total) break;
        const uint32_t u = long_rows[item];
        const uint64_t b = goff[u], e = goff[u + 1];
        const uint32_t ru = rank[u];
        const uint64_t op = out_off[ru];
        if (threadIdx.x == 0)
            for (uint32_t k = outdeg[ru]; k & 3u; ++k) out_adj[op + k] = kNone;  // pad slots
        // whole warps stride over the row (the loop bound is warp-uniform)
        const uint64_t wb = b + (threadIdx.x & ~31u);
        for (uint64_t i0 = wb; i0 < e; i0 += 4 * kLongThreads) {
            uint32_t rv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t i = i0 + lane_id() + (uint64_t)k * kLongThreads;
                rv[k] = i < e ? radj[i] : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t i = i0 + lane_id() + (uint64_t)k * kLongThreads;
                const bool o = i < e && rv[k] > ru;
                const unsigned bo = __ballot_sync(FULL, o);
                unsigned pos = 0;
                if (bo && lane_id() == 0) pos = atomicAdd(&cursor, __popc(bo));
                pos = __shfl_sync(FULL, pos, 0);
                if (o) out_adj[op + pos + __popc(bo & lt)] = rv[k];
            }
        }
    }
}

// cost_report(view) (cost.cpp:27-38) from the rank-space degree arrays.
__global__ void __launch_bounds__(256) k_cost(uint32_t n, const uint32_t* __restrict__ outdeg,
                                              const uint32_t* __restrict__ indeg,
                                              unsigned long long* __restrict__ cost,
                                              unsigned long long* __restrict__ sum_out) {
    using BR = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename BR::TempStorage tmp;
    unsigned long long pp = 0, pm = 0, mm = 0, dd = 0, so = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long o = outdeg[r], i = indeg[r];
        pp += o * o;
        pm += o * i;
        mm += i * i;
        dd += (o + i) * (o + i);
        so += o;
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
    __syncthreads();
    s = BR(tmp).Sum(so);  // = m for a symmetric adjacency (checked on the host)
    if (threadIdx.x == 0) atomicAdd(sum_out, s);
}

// max over rows of the out-degree (listing batch arithmetic is 32-bit).
// ---- device orderings (ordering.cpp:66-109) ----------------------------------
// Sort keys of the reference's bucket sort: degree ascending (degree order)
// or descending via ~degree (split order); the values are the vertex ids in
// ascending order and the radix sort is stable, so ties keep ascending ids,
// exactly as the reference's counting sort fills each degree bucket.
__global__ void k_degree_keys(uint32_t n, const uint64_t* __restrict__ off, bool desc, uint32_t* __restrict__ key,
                              uint32_t* __restrict__ val) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        const uint32_t d = static_cast<uint32_t>(off[v + 1] - off[v]);
        key[v] = desc ? ~d : d;
        val[v] = static_cast<uint32_t>(v);
    }
}

// Position p of the sorted sequence -> rank. Split: ordering.cpp:103-106
// (0-based parity formula).
__global__ void k_rank_from_sequence(uint32_t n, const uint32_t* __restrict__ seq, bool split,
                                     uint32_t* __restrict__ rank) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += stride) {
        const uint32_t pp = static_cast<uint32_t>(p);
        rank[seq[p]] = !split ? pp : ((pp & 1u) == 0 ? pp / 2 : n - 1 - pp / 2);
    }
}

// Padded out-row lengths: rows start on 16-byte boundaries (quads) so the
// listing reads them as whole quads; pad slots hold kNone.
__global__ void k_pad_len(uint32_t n, const uint32_t* __restrict__ deg, uint32_t* __restrict__ plen) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride)
        plen[r] = (deg[r] + 3u) & ~3u;
}

// Lowest rank r whose out-rows [r, n) fit in `budget_elems` padded elements:
// the rows the listing loads with L2 evict_last (the top ranks are the rows
// re-read by the most seeds). One thread, binary search over out_off.
__global__ void k_hot_rank(uint32_t n, const uint64_t* __restrict__ out_off, uint64_t budget_elems,
                           unsigned long long* __restrict__ out) {
    const uint64_t end = out_off[n];
    uint32_t lo = 0, hi = n;  // find min r with end - out_off[r] <= budget
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (end - out_off[mid] <= budget_elems) hi = mid;
        else lo = mid + 1;
    }
    *out = lo;
}

// Checksum sink table: hv[r] = vertex_hash(inv[r]) (common.cuh).
__global__ void k_vertex_hash(uint32_t n, const uint32_t* __restrict__ inv, unsigned long long* __restrict__ hv) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= n; r += stride)
        hv[r] = r < n ? vertex_hash(inv[r]) : 0ull;  // hv[n] = 0: the no-hit lanes' load target
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
                              const uint32_t* __restrict__ rlen, const uint32_t* __restrict__ radj,
                              const uint64_t* __restrict__ doff, uint32_t* __restrict__ dadj) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint32_t r = rank[u];
        const uint64_t b = roff[r], e = b + rlen[r], d = doff[u];
        for (uint64_t i = b + lane; i < e; i += 32) dadj[d + (i - b)] = inv[radj[i]];
    }
}

}  // namespace trigpu
