// segsort.cuh -- per-row segmented sort of the rank-space CSR rows.
//
// The reference gets rank-ascending rows for free from its sequential
// rank-order scatter (oriented_view.cpp:32-46); the parallel scatter writes
// rows in dense-id order, so every row is sorted here. Values in a row are
// distinct ranks (simple graph), which the bitmap path relies on. Size classes:
//   L <= 16            thread per row, bitonic network in registers
//   16 < L <= 32       16 lanes per row, cub::WarpMergeSort (2 keys / lane)
//   32 < L <= 64       warp per row, cub::WarpMergeSort (2 keys / lane)
//   64 < L <= 256      warp per row, cub::WarpMergeSort (8 keys / lane)
//   256 < L <= 1024    CTA per row, cub::BlockRadixSort (4 keys / thread)
//   1024 < L <= 4096   CTA per row, cub::BlockRadixSort (16 keys / thread)
// (radix sorts use 6-bit digits over bits(n) + 1 key bits)
//   L > 4096           CTA per row: bucket by 2^19-value window into a temp
//                      row, then per window either BlockRadixSort (<= 2048
//                      entries) or a 64 KB shared-memory bitmap + popc compaction
#pragma once

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/warp/warp_merge_sort.cuh>

#include "common.cuh"

namespace trigpu {

enum : int { kSortW32 = 0, kSortW64, kSortW256, kSortB1K, kSortB4K, kSortBig, kSortClasses };
struct SortLists {
    uint32_t* rows[kSortClasses];  // row ids per size class
    unsigned int* counts;          // [kSortClasses]
};

// Row r is adj[off[r], off[r] + L): L = len[r] when a length array is given
// (the out-CSR, whose rows are padded to quads), else off[r + 1] - off[r].
__device__ __forceinline__ uint64_t row_len(const uint64_t* off, const uint32_t* len, uint64_t r) {
    return len ? static_cast<uint64_t>(len[r]) : off[r + 1] - off[r];
}

constexpr uint32_t kSortThreadMax = 16;
constexpr uint32_t kSortWarpMax = 256;
constexpr uint32_t kSortBlockMax = 4096;
// upper bound of each listed class
__device__ __forceinline__ uint32_t sort_class_max(int c) {
    return c == 0 ? 32u : c == 1 ? 64u : c == 2 ? 256u : c == 3 ? 1024u : c == 4 ? 4096u : 0xFFFFFFFFu;
}

__device__ __forceinline__ void warp_append(uint32_t* list, unsigned int* count, bool pred, uint32_t v) {
    const unsigned b = __ballot_sync(FULL, pred);
    if (!b) return;
    const unsigned leader = __ffs(b) - 1;
    unsigned base = 0;
    if (lane_id() == leader) base = atomicAdd(count, __popc(b));
    base = __shfl_sync(FULL, base, leader);
    if (pred) list[base + __popc(b & lanemask_lt())] = v;
}

// Thread per row: sorts rows of length <= 16 in registers, lists the others.
__global__ void __launch_bounds__(256) k_sort_small(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                                    uint32_t* __restrict__ adj, SortLists lists) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t start = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    // warp-uniform trip count so the ballots in warp_append stay converged
    const uint64_t trips = (n + stride - 1) / stride;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t r = start + t * stride;
        uint64_t b = 0, L = 0;
        if (r < n) {
            b = off[r];
            L = row_len(off, len, r);
        }
        if (L >= 2 && L <= kSortThreadMax) {
            uint32_t a[kSortThreadMax];
            uint32_t* p = adj + b;
#pragma unroll
            for (int i = 0; i < (int)kSortThreadMax; ++i) a[i] = (uint64_t)i < L ? p[i] : kNone;
#pragma unroll
            for (int k = 2; k <= (int)kSortThreadMax; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                    for (int i = 0; i < (int)kSortThreadMax; ++i) {
                        const int l = i ^ j;
                        if (l > i) {
                            const uint32_t x = a[i], y = a[l];
                            const uint32_t lo = min(x, y), hi = max(x, y);
                            if ((i & k) == 0) { a[i] = lo; a[l] = hi; }
                            else { a[i] = hi; a[l] = lo; }
                        }
                    }
#pragma unroll
            for (int i = 0; i < (int)kSortThreadMax; ++i)
                if ((uint64_t)i < L) p[i] = a[i];
        }
        uint32_t lo = kSortThreadMax;
#pragma unroll
        for (int c = 0; c < kSortClasses; ++c) {
            warp_append(lists.rows[c], &lists.counts[c], L > lo && L <= sort_class_max(c), (uint32_t)r);
            lo = sort_class_max(c);
        }
    }
}

struct U32Less {
    __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const { return a < b; }
};

// Logical warp of LW lanes per row, ITEMS keys per lane (rows up to LW * ITEMS).
template <int ITEMS, int LW>
__global__ void __launch_bounds__(256) k_sort_warp(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                                   uint32_t* __restrict__ adj, const uint32_t* __restrict__ rows,
                                                   const unsigned int* __restrict__ count) {
    constexpr int kGroups = 256 / LW;
    using WS = cub::WarpMergeSort<uint32_t, ITEMS, LW>;
    __shared__ typename WS::TempStorage tmp[kGroups];
    const unsigned grp = threadIdx.x / LW, gl = threadIdx.x % LW;
    const unsigned total = *count;
    // uniform trip count per physical warp (the logical warps of a warp stay converged)
    const unsigned stride = gridDim.x * kGroups;
    const unsigned first = blockIdx.x * kGroups + grp;
    const unsigned warp_first = blockIdx.x * kGroups + (threadIdx.x / 32) * (32 / LW);
    for (unsigned base = warp_first; base < total; base += stride) {
        const unsigned i = first + (base - warp_first);
        const bool act = i < total;
        uint32_t* p = adj;
        int L = 0;
        if (act) {
            const uint32_t r = rows[i];
            p = adj + off[r];
            L = (int)row_len(off, len, r);
        }
        uint32_t k[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int idx = gl * ITEMS + j;
            k[j] = idx < L ? p[idx] : kNone;
        }
        WS(tmp[grp]).Sort(k, U32Less(), L, kNone);
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int idx = gl * ITEMS + j;
            if (idx < L) p[idx] = k[j];
        }
        __syncwarp();
    }
}

constexpr int kBlockSortThreads = 256;
constexpr int kRadixBits = 6;

template <int ITEMS>
__global__ void __launch_bounds__(kBlockSortThreads) k_sort_block(const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                                                  uint32_t* __restrict__ adj,
                                                                  const uint32_t* __restrict__ rows,
                                                                  const unsigned int* __restrict__ count,
                                                                  int end_bit) {
    using BRS = cub::BlockRadixSort<uint32_t, kBlockSortThreads, ITEMS, cub::NullType, kRadixBits>;
    __shared__ typename BRS::TempStorage tmp;
    const unsigned total = *count;
    for (unsigned i = blockIdx.x; i < total; i += gridDim.x) {
        const uint32_t r = rows[i];
        const uint64_t b = off[r];
        const int L = (int)row_len(off, len, r);
        uint32_t* p = adj + b;
        uint32_t k[ITEMS];
        // blocked arrangement; padding (all ones) sorts last under end_bit > bits(n-1)
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int idx = threadIdx.x * ITEMS + j;
            k[j] = idx < L ? p[idx] : kNone;
        }
        BRS(tmp).Sort(k, 0, end_bit);
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int idx = threadIdx.x * ITEMS + j;
            if (idx < L) p[idx] = k[j];
        }
        __syncthreads();
    }
}

constexpr int kBigThreads = 512;
constexpr int kWinBits = 19;                       // 2^19-value windows
constexpr int kWinWords = (1 << kWinBits) / 32;    // 16384 words = 64 KB bitmap
constexpr int kMaxWindows = 8192;                  // covers n < 2^32
constexpr int kBigSmallItems = 4;                  // small-window radix sort: 2048 keys
constexpr int kBigSmallMax = kBigThreads * kBigSmallItems;

struct BigSortSmem {
    uint32_t bitmap[kWinWords];
    uint32_t cursor[kMaxWindows];
    union {
        typename cub::BlockRadixSort<uint32_t, kBigThreads, kBigSmallItems>::TempStorage sort;
        typename cub::BlockScan<uint32_t, kBigThreads>::TempStorage scan;
    } u;
};

__global__ void __launch_bounds__(kBigThreads) k_sort_big(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ len,
                                                          uint32_t* __restrict__ adj, uint32_t* __restrict__ tmpbuf,
                                                          const uint32_t* __restrict__ rows,
                                                          const unsigned int* __restrict__ count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BigSortSmem& S = *reinterpret_cast<BigSortSmem*>(smem_raw);
    using BRS = cub::BlockRadixSort<uint32_t, kBigThreads, kBigSmallItems>;
    using BS = cub::BlockScan<uint32_t, kBigThreads>;
    const unsigned tid = threadIdx.x;
    const uint32_t H = (uint32_t)(((uint64_t)n + (1u << kWinBits) - 1) >> kWinBits);
    for (int i = tid; i < kWinWords; i += kBigThreads) S.bitmap[i] = 0;
    const unsigned total = *count;
    for (unsigned ri = blockIdx.x; ri < total; ri += gridDim.x) {
        const uint32_t r = rows[ri];
        const uint64_t b = off[r];
        const uint64_t L = row_len(off, len, r);
        uint32_t* p = adj + b;
        uint32_t* t = tmpbuf + b;
        for (uint32_t w = tid; w < H; w += kBigThreads) S.cursor[w] = 0;
        __syncthreads();
        for (uint64_t i = tid; i < L; i += kBigThreads) atomicAdd(&S.cursor[p[i] >> kWinBits], 1u);
        __syncthreads();
        // exclusive scan of window counts (H <= 8192 = 16 per thread)
        {
            constexpr int PER = kMaxWindows / kBigThreads;
            uint32_t v[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t w = tid * PER + k;
                v[k] = w < H ? S.cursor[w] : 0;
            }
            BS(S.u.scan).ExclusiveSum(v, v);
            __syncthreads();
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t w = tid * PER + k;
                if (w < H) S.cursor[w] = v[k];
            }
        }
        __syncthreads();
        for (uint64_t i = tid; i < L; i += kBigThreads) {
            const uint32_t v = p[i];
            t[atomicAdd(&S.cursor[v >> kWinBits], 1u)] = v;
        }
        __syncthreads();
        // window w now spans [cursor[w-1], cursor[w])
        for (uint32_t w = 0; w < H; ++w) {
            const uint32_t s = w ? S.cursor[w - 1] : 0, e = S.cursor[w];
            const uint32_t c = e - s;
            if (c == 0) continue;
            const uint32_t wbase = w << kWinBits;
            if (c <= (uint32_t)kBigSmallMax) {
                uint32_t k[kBigSmallItems];
#pragma unroll
                for (int j = 0; j < kBigSmallItems; ++j) {
                    const uint32_t idx = tid * kBigSmallItems + j;
                    k[j] = idx < c ? (t[s + idx] - wbase) : ((1u << kWinBits) | 0xFFFu);
                }
                BRS(S.u.sort).Sort(k, 0, kWinBits + 1);
#pragma unroll
                for (int j = 0; j < kBigSmallItems; ++j) {
                    const uint32_t idx = tid * kBigSmallItems + j;
                    if (idx < c) p[s + idx] = wbase + k[j];
                }
                __syncthreads();
            } else {
                for (uint32_t i = s + tid; i < e; i += kBigThreads) {
                    const uint32_t v = t[i] - wbase;
                    atomicOr(&S.bitmap[v >> 5], 1u << (v & 31));
                }
                __syncthreads();
                constexpr int WPT = kWinWords / kBigThreads;  // 32 words per thread
                uint32_t cnt = 0;
#pragma unroll 8
                for (int k = 0; k < WPT; ++k) cnt += __popc(S.bitmap[tid * WPT + k]);
                uint32_t pos;
                BS(S.u.scan).ExclusiveSum(cnt, pos);
                pos += s;
                for (int k = 0; k < WPT; ++k) {
                    uint32_t word = S.bitmap[tid * WPT + k];
                    while (word) {
                        const int bit = __ffs(word) - 1;
                        word &= word - 1;
                        p[pos++] = wbase + (uint32_t)((tid * WPT + k) * 32 + bit);
                    }
                }
                __syncthreads();
                for (int k = 0; k < WPT; ++k) S.bitmap[tid * WPT + k] = 0;
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

}  // namespace trigpu
