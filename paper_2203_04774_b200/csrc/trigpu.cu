// trigpu.cu -- context, device memory and the C-ABI (include/trigpu.h).
//
// One tl_ctx = one device + two CUDA streams + grow-only device buffers laid
// out for HBM residency (SURVEY §8 byte table):
//   input graph   goff u64[n+1], gadj u32[2m]        (owned copy, tl_orient only)
//   pi            rank u32[n], inv u32[n]
//   relabelled    radj u32[2m]  (rank[adj[e]]; reused as the sort temp row)
//   out-CSR       out_off u64[n+1], out_adj u32[m]   (rank space, rows ascending)
//   in-CSR        in_off u64[n+1], in_adj u32[m]     (built on first A++ / export)
//   degrees       outdeg u32[n], indeg u32[n]
//   work lists    lists u32[4n] (sort classes during orient, seed classes
//                 during listing)
//   sinks         acc u64[8], vcount u64[n], tri u32[3T]
// Host <-> device crossings: the input copy in tl_orient, small scalar
// read-backs (error flags, class counts, stats) and the explicit fetches.

#include <cuda_runtime.h>

#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "listing.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "core.cuh"
#include "normalize.cuh"
#include "orient.cuh"
#include "segsort.cuh"
#include "trigpu.h"

using namespace trigpu;

namespace {

thread_local std::string g_create_error;

#ifndef TRIGPU_HOT_MB
#define TRIGPU_HOT_MB 64
#endif
// L2 budget for the evict_last rows (126 MB L2: leave room for the checksum
// table gathers and the cold streaming)
constexpr uint64_t kHotRowBytes = uint64_t{TRIGPU_HOT_MB} << 20;

enum Phase {
    PH_H2D = 0,
    PH_RELABEL,
    PH_SCAN,
    PH_SCATTER,
    PH_SORT,
    PH_COST,
    PH_IN_CSR,
    PH_CLASSIFY,
    PH_LIST,
    PH_LIST_R,  // per seed class (the last pass of the last tl_list); G runs on the side stream
    PH_LIST_H,
    PH_LIST_C1,
    PH_LIST_C2,
    PH_LIST_G,
    PH_SORT_SMALL,  // segmented-sort classes of the last orientation's out-CSR
    PH_SORT_WARP,
    PH_SORT_BLOCK,
    PH_SORT_BIG,
    PH_WORK_R,  // per-class inner_ops of the last tl_list (TL_DEBUG_CLASS_WORK only; a count, not ms)
    PH_WORK_H,
    PH_WORK_C1,
    PH_WORK_C2,
    PH_WORK_G,
    PH_COUNT
};
const char* kPhaseNames[PH_COUNT] = {"h2d",    "relabel_count", "scan",    "scatter", "segsort", "cost",
                                     "in_csr", "classify",      "list",    "list_R",  "list_H",  "list_C1",
                                     "list_C2", "list_G", "sort_small", "sort_warp", "sort_block", "sort_big",
                                     "work_R", "work_H", "work_C1", "work_C2", "work_G"};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

}  // namespace

struct tl_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t s = nullptr, s2 = nullptr;
    cudaEvent_t ev[2 * PH_COUNT + 8] = {};
    cudaEvent_t timer0 = nullptr, timer1 = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaEvent_t cls_ev[10] = {};  // start / end of each seed-class launch
    cudaEvent_t sort_ev[8] = {};  // start / end of the segmented-sort class kernels
    bool sort_run[4] = {};
    bool cls_run[5] = {};
    std::string err;
    double phase_ms[PH_COUNT] = {};
    uint64_t launches = 0, orient_launches = 0;

    uint32_t n = 0;
    uint64_t m = 0;
    bool oriented = false, in_built = false, hv_built = false;
    bool normalized = false;       // goff / gadj / labels hold a tl_normalize result
    bool view_normalized = false;  // the oriented view was built from that graph (labels apply)
    uint32_t norm_n = 0;
    uint64_t norm_m = 0;
    uint32_t max_out = 0;
    uint32_t hot_rank = 0;  // rows of ranks >= hot_rank fit the L2 evict_last budget
    unsigned long long cost[4] = {0, 0, 0, 0};
    double h2d_ms = 0, orient_ms = 0;

    DevBuf holes, segs;  // list compaction: chunk tails {start, len}; move segments
    DevBuf goff, gadj, rank, inv, hv, sort_tmp, labels, radj, out_off, out_adj, in_off, in_adj, outdeg, indeg, lists, acc,
        vcount, tri, scan_part, bitmaps, small;
    bool have_vcounts = false, have_tri = false;
    int variant = 0;         // TL_DEBUG_VARIANT: probe flavour of an experiments build (A/B timing)
    uint32_t bm_shrink = 0;  // TL_DEBUG_BM_SHRINK: smaller bitmaps (tests force the filter path)
    bool class_work = false; // TL_DEBUG_CLASS_WORK: per-class inner_ops into the phase table
    uint32_t h_split = kHSplit;        // TL_DEBUG_H_SPLIT: largest class-H |S| left on the warp kernel above h_cta_min_n
    uint32_t h_cta_min_n = kHCtaMinN;  // TL_DEBUG_H_WIDE_MIN_N sets both thresholds (tests force the paths with 0):
    uint32_t wide_min_n = kWideMinN;   //   class H split above h_cta_min_n, C1's 2^19 window above wide_min_n
    unsigned long long tri_count = 0;

    tl_status fail(tl_status st, const std::string& what) {
        err = what;
        return st;
    }
    tl_status cuda_fail(const char* what, cudaError_t e) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        (void)cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? TL_ERR_OUT_OF_MEMORY : TL_ERR_CUDA;
    }
};

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return ctx->cuda_fail(#call, e_); \
    } while (0)
#define LAUNCHED()                                                                  \
    do {                                                                            \
        ++ctx->launches;                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess) return ctx->cuda_fail("kernel launch", e_);          \
    } while (0)

namespace {

tl_status ensure(tl_ctx* ctx, DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return TL_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return ctx->fail(TL_ERR_OUT_OF_MEMORY,
                         "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    }
    b.cap = bytes;
    return TL_OK;
}

#define ENSURE(buf, bytes)                                 \
    do {                                                   \
        tl_status st_ = ensure(ctx, ctx->buf, (bytes));    \
        if (st_ != TL_OK) return st_;                      \
    } while (0)

template <class T>
T* P(DevBuf& b) {
    return static_cast<T*>(b.p);
}

unsigned grid_for(uint64_t items, unsigned threads, unsigned cap) {
    uint64_t g = (items + threads - 1) / threads;
    if (g < 1) g = 1;
    return static_cast<unsigned>(std::min<uint64_t>(g, cap));
}

double ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// offsets[0..n] = exclusive scan of cnt[0..n)
tl_status scan_offsets(tl_ctx* ctx, uint32_t n, const uint32_t* cnt, uint64_t* off) {
    const uint64_t tiles = std::max<uint64_t>(1, (static_cast<uint64_t>(n) + kScanTile - 1) / kScanTile);
    ENSURE(scan_part, tiles * sizeof(unsigned long long));
    auto* part = P<unsigned long long>(ctx->scan_part);
    k_scan_partials<<<(unsigned)tiles, kScanThreads, 0, ctx->s>>>(n, cnt, part);
    LAUNCHED();
    k_scan_tops<<<1, kScanThreads, 0, ctx->s>>>(tiles, part);
    LAUNCHED();
    k_scan_apply<<<(unsigned)tiles, kScanThreads, 0, ctx->s>>>(n, cnt, part, off);
    LAUNCHED();
    return TL_OK;
}

// Segmented sort of every row of (off, adj) in place; tmp has >= off[n] slots
// (the big-row buckets index it by the row offsets).
tl_status sort_rows(tl_ctx* ctx, uint32_t n, uint64_t* off, const uint32_t* len, uint32_t* adj, uint32_t* tmp) {
    ENSURE(small, 128);
    ENSURE(lists, (size_t)std::max<uint32_t>(n, 1) * 4 * std::max(kClasses, (int)kSortClasses));
    auto* counts = static_cast<unsigned int*>(ctx->small.p);
    CK(cudaMemsetAsync(counts, 0, kSortClasses * sizeof(unsigned int), ctx->s));
    uint32_t* lists = P<uint32_t>(ctx->lists);
    SortLists L{};
    for (int c = 0; c < kSortClasses; ++c) L.rows[c] = lists + (uint64_t)c * n;
    L.counts = counts;
    CK(cudaEventRecord(ctx->sort_ev[0], ctx->s));
    k_sort_small<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(n, off, len, adj, L);
    LAUNCHED();
    CK(cudaEventRecord(ctx->sort_ev[1], ctx->s));
    unsigned int h[kSortClasses];
    CK(cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    const int end_bit = std::min(32, (int)(32 - __builtin_clz(std::max(n, 2u) - 1)) + 1);
    ctx->sort_run[0] = true;
    ctx->sort_run[1] = h[kSortW32] || h[kSortW64] || h[kSortW256];
    ctx->sort_run[2] = h[kSortB1K] || h[kSortB4K];
    ctx->sort_run[3] = h[kSortBig] != 0;
    CK(cudaEventRecord(ctx->sort_ev[2], ctx->s));
    if (h[kSortW32]) {
        k_sort_warp<2, 16><<<grid_for((uint64_t)h[kSortW32] * 16, 256, ctx->sms * 8), 256, 0, ctx->s>>>(
            off, len, adj, L.rows[kSortW32], counts + kSortW32);
        LAUNCHED();
    }
    if (h[kSortW64]) {
        k_sort_warp<2, 32><<<grid_for((uint64_t)h[kSortW64] * 32, 256, ctx->sms * 8), 256, 0, ctx->s>>>(
            off, len, adj, L.rows[kSortW64], counts + kSortW64);
        LAUNCHED();
    }
    if (h[kSortW256]) {
        k_sort_warp<8, 32><<<grid_for((uint64_t)h[kSortW256] * 32, 256, ctx->sms * 8), 256, 0, ctx->s>>>(
            off, len, adj, L.rows[kSortW256], counts + kSortW256);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->sort_ev[3], ctx->s));
    CK(cudaEventRecord(ctx->sort_ev[4], ctx->s));
    if (h[kSortB1K]) {
        k_sort_block<4><<<std::min<unsigned>(h[kSortB1K], ctx->sms * 8), kBlockSortThreads, 0, ctx->s>>>(
            off, len, adj, L.rows[kSortB1K], counts + kSortB1K, end_bit);
        LAUNCHED();
    }
    if (h[kSortB4K]) {
        k_sort_block<16><<<std::min<unsigned>(h[kSortB4K], ctx->sms * 8), kBlockSortThreads, 0, ctx->s>>>(
            off, len, adj, L.rows[kSortB4K], counts + kSortB4K, end_bit);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->sort_ev[5], ctx->s));
    CK(cudaEventRecord(ctx->sort_ev[6], ctx->s));
    if (h[kSortBig]) {
        const size_t smem = sizeof(BigSortSmem);
        CK(cudaFuncSetAttribute(k_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_sort_big<<<std::min<unsigned>(h[kSortBig], ctx->sms * 2), kBigThreads, smem, ctx->s>>>(
            n, off, len, adj, tmp, L.rows[kSortBig], counts + kSortBig);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->sort_ev[7], ctx->s));
    return TL_OK;
}

// Results of the last tl_list refer to the current view and pi; anything that
// replaces either drops them.
void drop_results(tl_ctx* ctx) {
    ctx->have_vcounts = false;
    ctx->have_tri = false;
    ctx->tri_count = 0;
}

tl_status orient_core(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* goff, const uint32_t* gadj,
                      const uint32_t* rank) {
    ctx->oriented = false;
    ctx->in_built = false;
    ctx->hv_built = false;
    ctx->view_normalized = false;
    drop_results(ctx);
    ctx->n = n;
    ctx->m = m;
    ENSURE(inv, (size_t)n * 4);
    ENSURE(radj, 2 * m * 4);
    ENSURE(outdeg, (size_t)n * 4);
    ENSURE(indeg, (size_t)n * 4);
    ENSURE(out_off, ((size_t)n + 1) * 8);
    ENSURE(lists, (size_t)n * 4 * kClasses);
    ENSURE(small, 128);
    auto* flags = static_cast<unsigned long long*>(ctx->small.p);  // [0] err, [4..] scratch
    const unsigned big = ctx->sms * 16;

    CK(cudaMemsetAsync(ctx->inv.p, 0xFF, (size_t)n * 4, ctx->s));
    CK(cudaMemsetAsync(flags, 0, 64, ctx->s));
    // rows of >= kLongDeg edges (one CTA each): list in the free part of
    // `lists` (the sort classes use its first 3n words), count + two queues
    uint32_t* long_rows = P<uint32_t>(ctx->lists) + 3 * (uint64_t)n;
    auto* long_cnt = reinterpret_cast<unsigned int*>(flags + 8);  // [0] count, [1] [2] queues
    CK(cudaMemsetAsync(long_cnt, 0, 16, ctx->s));
    if (n) {
        // pi and the offsets are validated before anything is indexed through them
        k_inverse<<<grid_for(n, 256, big), 256, 0, ctx->s>>>(n, rank, P<uint32_t>(ctx->inv), flags);
        LAUNCHED();
        k_check_offsets<<<grid_for((uint64_t)n + 1, 256, big), 256, 0, ctx->s>>>(n, 2 * m, goff, flags);
        LAUNCHED();
        unsigned long long pre = 0;
        CK(cudaMemcpyAsync(&pre, flags, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        if (pre & 3ull) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: ordering does not match graph (rank is not a permutation of [0, n))");
        if (pre & 8ull) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: offsets must start at 0, be non-decreasing and end at 2m");
        k_relabel_count<<<grid_for((uint64_t)n, 256, big * 2), 256, 0, ctx->s>>>(
            n, goff, gadj, rank, P<uint32_t>(ctx->radj), P<uint32_t>(ctx->outdeg), P<uint32_t>(ctx->indeg),
            long_rows, long_cnt, flags);
        LAUNCHED();
        k_relabel_long<<<ctx->sms * 2, kLongThreads, 0, ctx->s>>>(n, goff, gadj, rank, P<uint32_t>(ctx->radj),
                                                                  P<uint32_t>(ctx->outdeg), P<uint32_t>(ctx->indeg),
                                                                  long_rows, long_cnt, long_cnt + 1, flags);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->ev[PH_RELABEL], ctx->s));
    // out rows padded to quads: out_off holds the padded starts (multiples
    // of 4), outdeg the lengths; the pad slots hold kNone
    uint32_t* plen = P<uint32_t>(ctx->lists) + 4 * (uint64_t)n;
    if (n) {
        k_pad_len<<<grid_for(n, 256, big), 256, 0, ctx->s>>>(n, P<uint32_t>(ctx->outdeg), plen);
        LAUNCHED();
    }
    tl_status st = scan_offsets(ctx, n, plen, P<uint64_t>(ctx->out_off));
    if (st != TL_OK) return st;
    CK(cudaEventRecord(ctx->ev[PH_SCAN], ctx->s));
    unsigned long long errflag = 0, padded = 0;
    CK(cudaMemcpyAsync(&errflag, flags, 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaMemcpyAsync(&padded, P<uint64_t>(ctx->out_off) + n, 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    if (errflag & 3ull) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: ordering does not match graph (rank is not a permutation of [0, n))");
    if (errflag & 4ull) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: adjacency violates the Graph invariants (rows must be strictly increasing, in range, loop-free)");
    if (padded / 4 >= (1ull << 32)) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: graph too large (> 2^32 quads of out-rows)");
    ENSURE(out_adj, padded * 4 + 64);
    // radj becomes the big-row sort's temp row, indexed by the PADDED offsets
    // (up to m + 3n slots): grow it now, its contents are dead after k_scatter
    const size_t radj_need = std::max<size_t>(2 * m, padded + 64) * 4;
    if (n) {
        k_scatter<<<grid_for((uint64_t)n, 256, big * 2), 256, 0, ctx->s>>>(
            n, goff, P<uint32_t>(ctx->radj), rank, P<uint64_t>(ctx->out_off), P<uint32_t>(ctx->outdeg),
            P<uint32_t>(ctx->out_adj));
        LAUNCHED();
        k_scatter_long<<<ctx->sms * 2, kLongThreads, 0, ctx->s>>>(goff, P<uint32_t>(ctx->radj), rank,
                                                                  P<uint64_t>(ctx->out_off), P<uint32_t>(ctx->outdeg),
                                                                  P<uint32_t>(ctx->out_adj),
                                                                  long_rows, long_cnt, long_cnt + 2);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->ev[PH_SCATTER], ctx->s));
    if (ctx->radj.cap < radj_need) {
        CK(cudaStreamSynchronize(ctx->s));  // k_scatter still reads radj
        ENSURE(radj, radj_need);
    }
    st = sort_rows(ctx, n, P<uint64_t>(ctx->out_off), P<uint32_t>(ctx->outdeg), P<uint32_t>(ctx->out_adj),
                   P<uint32_t>(ctx->radj));
    if (st != TL_OK) return st;
    CK(cudaEventRecord(ctx->ev[PH_SORT], ctx->s));
    // costs + max out-degree
    CK(cudaMemsetAsync(flags + 2, 0, 6 * 8, ctx->s));
    if (n) {
        k_cost<<<grid_for(n, 256, ctx->sms * 4), 256, 0, ctx->s>>>(n, P<uint32_t>(ctx->outdeg), P<uint32_t>(ctx->indeg),
                                                                  flags + 2, flags + 7);
        LAUNCHED();
        k_maxdeg<<<grid_for(n, 256, ctx->sms * 4), 256, 0, ctx->s>>>(n, P<uint32_t>(ctx->outdeg),
                                                                    reinterpret_cast<unsigned int*>(flags + 6));
        LAUNCHED();
        k_hot_rank<<<1, 1, 0, ctx->s>>>(n, P<uint64_t>(ctx->out_off), kHotRowBytes / 4, flags + 10);
        LAUNCHED();
    }
    CK(cudaEventRecord(ctx->ev[PH_COST], ctx->s));
    unsigned long long res[6];
    CK(cudaMemcpyAsync(res, flags + 2, sizeof(res), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    if (res[5] != m)  // each undirected edge oriented once: only if every (u, v) has its (v, u) (graph.cpp:108)
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: adjacency is not symmetric (out-degrees do not sum to m)");
    std::memcpy(ctx->cost, res, sizeof(ctx->cost));
    ctx->max_out = static_cast<uint32_t>(res[4]);
    unsigned long long hot = n;
    if (n) {
        CK(cudaMemcpyAsync(&hot, flags + 10, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    }
    ctx->hot_rank = static_cast<uint32_t>(hot);
    ctx->phase_ms[PH_RELABEL] = ev_ms(ctx->ev[PH_H2D], ctx->ev[PH_RELABEL]);
    ctx->phase_ms[PH_SCAN] = ev_ms(ctx->ev[PH_RELABEL], ctx->ev[PH_SCAN]);
    ctx->phase_ms[PH_SCATTER] = ev_ms(ctx->ev[PH_SCAN], ctx->ev[PH_SCATTER]);
    ctx->phase_ms[PH_SORT] = ev_ms(ctx->ev[PH_SCATTER], ctx->ev[PH_SORT]);
    ctx->phase_ms[PH_COST] = ev_ms(ctx->ev[PH_SORT], ctx->ev[PH_COST]);
    ctx->orient_ms = ev_ms(ctx->ev[PH_H2D], ctx->ev[PH_COST]);
    for (int c = 0; c < 4; ++c)
        ctx->phase_ms[PH_SORT_SMALL + c] = ctx->sort_run[c] ? ev_ms(ctx->sort_ev[2 * c], ctx->sort_ev[2 * c + 1]) : 0.0;
    ctx->orient_launches = ctx->launches;
    ctx->oriented = true;
    return TL_OK;
}

// k_transpose: in-row s receives r for every successor s of r.
// Writes are bounded by the in-row's end (in_off[s + 1]): an asymmetric
// adjacency that slipped past the degree-sum check sets *err instead of
// writing past the row.
__global__ void k_transpose(uint32_t n, const uint64_t* __restrict__ out_off, const uint32_t* __restrict__ outdeg,
                            const uint32_t* __restrict__ out_adj, unsigned long long* __restrict__ cursor,
                            const uint64_t* __restrict__ in_off, uint32_t* __restrict__ in_adj,
                            unsigned long long* __restrict__ err) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t b = out_off[r], e = b + outdeg[r];
        for (uint64_t i = b + lane; i < e; i += 32) {
            const uint32_t s = out_adj[i];
            const unsigned long long pos = atomicAdd(&cursor[s], 1ull);
            if (pos < in_off[s + 1]) in_adj[pos] = static_cast<uint32_t>(r);
            else atomicOr(err, 16ull);
        }
    }
}

// In-CSR (predecessor rows) by transposing the out-CSR, then the same
// segmented sort. Built lazily: A+- never needs it.
tl_status ensure_in_csr(tl_ctx* ctx) {
    if (ctx->in_built) return TL_OK;
    const uint32_t n = ctx->n;
    const uint64_t m = ctx->m;
    ENSURE(in_off, ((size_t)n + 1) * 8);
    ENSURE(in_adj, m * 4);
    CK(cudaEventRecord(ctx->ev[PH_COUNT + 0], ctx->s));
    tl_status st = scan_offsets(ctx, n, P<uint32_t>(ctx->indeg), P<uint64_t>(ctx->in_off));
    if (st != TL_OK) return st;
    // cursor = copy of in_off; radj is free after orientation (it becomes the
    // cursor array here and the sort temp row afterwards)
    ENSURE(radj, std::max<size_t>(2 * m * 4, (size_t)n * 8));
    auto* cursor = P<unsigned long long>(ctx->radj);
    if (n) {
        CK(cudaMemcpyAsync(cursor, ctx->in_off.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->s));
        ENSURE(small, 128);
        auto* flags = static_cast<unsigned long long*>(ctx->small.p);
        CK(cudaMemsetAsync(flags, 0, 8, ctx->s));
        k_transpose<<<grid_for((uint64_t)n * 32, 256, ctx->sms * 32), 256, 0, ctx->s>>>(
            n, P<uint64_t>(ctx->out_off), P<uint32_t>(ctx->outdeg), P<uint32_t>(ctx->out_adj), cursor,
            P<uint64_t>(ctx->in_off), P<uint32_t>(ctx->in_adj), flags);
        LAUNCHED();
        unsigned long long err = 0;
        CK(cudaMemcpyAsync(&err, flags, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        if (err) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: adjacency is not symmetric (in-rows overflow)");
    }
    st = sort_rows(ctx, n, P<uint64_t>(ctx->in_off), nullptr, P<uint32_t>(ctx->in_adj), P<uint32_t>(ctx->radj));
    if (st != TL_OK) return st;
    CK(cudaEventRecord(ctx->ev[PH_COUNT + 1], ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    ctx->phase_ms[PH_IN_CSR] = ev_ms(ctx->ev[PH_COUNT + 0], ctx->ev[PH_COUNT + 1]);
    ctx->in_built = true;
    return TL_OK;
}

template <class K>
tl_status set_smem(tl_ctx* ctx, K kernel, size_t bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return TL_OK;
}

template <class K>
unsigned resident_grid(tl_ctx* ctx, K kernel, int threads, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1) {
        (void)cudaGetLastError();
        per_sm = 1;
    }
    return static_cast<unsigned>(per_sm * ctx->sms);
}

template <int ALGO, unsigned F, class CFG>
tl_status launch_cta(tl_ctx* ctx, ListParams p, uint32_t* list, unsigned count, unsigned int* queue) {
    p.seeds = list;
    p.nseeds = count;
    p.queue = queue;
    const size_t smem = smem_cta<F, CFG>();
    tl_status st = set_smem(ctx, k_list_cta<ALGO, F, CFG>, smem);
    if (st != TL_OK) return st;
    const unsigned grid = std::min<unsigned>(count, resident_grid(ctx, k_list_cta<ALGO, F, CFG>, CFG::kThreads, smem));
    k_list_cta<ALGO, F, CFG><<<grid, CFG::kThreads, smem, ctx->s>>>(p);
    LAUNCHED();
    return TL_OK;
}

template <int ALGO, unsigned F>
tl_status launch_classes(tl_ctx* ctx, ListParams base, uint32_t* const lists[kClasses],
                         const unsigned h[kClasses + 1], unsigned int* queues) {
    tl_status st;
    // class G first, on the side stream: a few long CTAs overlap the rest
    if (h[4]) {
        ListParams p = base;
        p.queue = queues + 4;
        p.seeds = lists[4];
        p.nseeds = h[4];
        const size_t smem = smem_giant<F>();
        if ((st = set_smem(ctx, k_list_giant<ALGO, F>, smem)) != TL_OK) return st;
#ifndef TRIGPU_G_GRID
#define TRIGPU_G_GRID 0  // CTAs for class G (0: one per SM)
#endif
        const unsigned grid = std::min<unsigned>(h[4], TRIGPU_G_GRID ? TRIGPU_G_GRID : (unsigned)ctx->sms);
        p.bitmap_words = ((uint64_t)ctx->n + 31) / 32 + 32;
        const size_t bm_bytes = (size_t)grid * p.bitmap_words * 4;
        if (ctx->bitmaps.cap < bm_bytes) {
            // fresh bitmaps start zeroed; every seed clears its own bits after use
            ENSURE(bitmaps, bm_bytes);
            CK(cudaMemsetAsync(ctx->bitmaps.p, 0, ctx->bitmaps.cap, ctx->s));
        }
        p.bitmaps = P<uint32_t>(ctx->bitmaps);
        CK(cudaEventRecord(ctx->fork, ctx->s));
        CK(cudaStreamWaitEvent(ctx->s2, ctx->fork, 0));
        CK(cudaEventRecord(ctx->cls_ev[8], ctx->s2));
        k_list_giant<ALGO, F><<<grid, kGThreads, smem, ctx->s2>>>(p);
        LAUNCHED();
        CK(cudaEventRecord(ctx->cls_ev[9], ctx->s2));
        CK(cudaEventRecord(ctx->join, ctx->s2));
        ctx->cls_run[4] = true;
    }
    if (h[0]) {
        ListParams p = base;
        p.seeds = lists[0];
        p.nseeds = h[0];
        p.queue = queues + 0;
        const size_t smem = smem_reg<F>();
        if ((st = set_smem(ctx, k_list_reg<ALGO, F>, smem)) != TL_OK) return st;
        const unsigned grid = std::min<unsigned>(grid_for((uint64_t)h[0] * 32, kRWarps * 32, ~0u),
                                                 resident_grid(ctx, k_list_reg<ALGO, F>, kRWarps * 32, smem));
        CK(cudaEventRecord(ctx->cls_ev[0], ctx->s));
        k_list_reg<ALGO, F><<<grid, kRWarps * 32, smem, ctx->s>>>(p);
        LAUNCHED();
        CK(cudaEventRecord(ctx->cls_ev[1], ctx->s));
        ctx->cls_run[0] = true;
    }
    if (h[kClasses]) {  // small class-H seeds of a large graph: warp per seed (back of lists[1])
        ListParams p = base;
        p.seeds = lists[1] + (ctx->n - h[kClasses]);
        p.nseeds = h[kClasses];
        p.queue = queues + 5;
        const size_t smem = smem_warp<F>();
        if ((st = set_smem(ctx, k_list_warp<ALGO, F>, smem)) != TL_OK) return st;
        const unsigned grid = std::min<unsigned>(grid_for((uint64_t)h[kClasses] * 32, kHWarps * 32, ~0u),
                                                 resident_grid(ctx, k_list_warp<ALGO, F>, kHWarps * 32, smem));
        CK(cudaEventRecord(ctx->cls_ev[2], ctx->s));
        k_list_warp<ALGO, F><<<grid, kHWarps * 32, smem, ctx->s>>>(p);
        LAUNCHED();
        CK(cudaEventRecord(ctx->cls_ev[3], ctx->s));
        ctx->cls_run[1] = true;
    }
    if (h[1]) {
        const bool first = !h[kClasses];  // the H time spans both launches
#if TRIGPU_H_CTA
        CK(cudaEventRecord(ctx->cls_ev[2], ctx->s));
        st = launch_cta<ALGO, F, CfgH>(ctx, base, lists[1], h[1], queues + 1);
        if (st != TL_OK) return st;
        CK(cudaEventRecord(ctx->cls_ev[3], ctx->s));
#else
      if (ctx->n > ctx->h_cta_min_n) {
        if (first) CK(cudaEventRecord(ctx->cls_ev[2], ctx->s));
        st = launch_cta<ALGO, F, CfgHWide>(ctx, base, lists[1], h[1], queues + 1);
        if (st != TL_OK) return st;
        CK(cudaEventRecord(ctx->cls_ev[3], ctx->s));
      } else {
        ListParams p = base;
        p.seeds = lists[1];
        p.nseeds = h[1];
        p.queue = queues + 1;
        const size_t smem = smem_warp<F>();
        if ((st = set_smem(ctx, k_list_warp<ALGO, F>, smem)) != TL_OK) return st;
        const unsigned grid = std::min<unsigned>(grid_for((uint64_t)h[1] * 32, kHWarps * 32, ~0u),
                                                 resident_grid(ctx, k_list_warp<ALGO, F>, kHWarps * 32, smem));
        CK(cudaEventRecord(ctx->cls_ev[2], ctx->s));
        k_list_warp<ALGO, F><<<grid, kHWarps * 32, smem, ctx->s>>>(p);
        LAUNCHED();
        CK(cudaEventRecord(ctx->cls_ev[3], ctx->s));
      }
#endif
        ctx->cls_run[1] = true;
    }
    if (h[2]) {
        CK(cudaEventRecord(ctx->cls_ev[4], ctx->s));
        st = ctx->n > ctx->wide_min_n ? launch_cta<ALGO, F, CfgC1Wide>(ctx, base, lists[2], h[2], queues + 2)
                                        : launch_cta<ALGO, F, CfgC1>(ctx, base, lists[2], h[2], queues + 2);
        if (st != TL_OK) return st;
        CK(cudaEventRecord(ctx->cls_ev[5], ctx->s));
        ctx->cls_run[2] = true;
    }
    if (h[3]) {
        CK(cudaEventRecord(ctx->cls_ev[6], ctx->s));
        st = launch_cta<ALGO, F, CfgC2>(ctx, base, lists[3], h[3], queues + 3);
        if (st != TL_OK) return st;
        CK(cudaEventRecord(ctx->cls_ev[7], ctx->s));
        ctx->cls_run[3] = true;
    }
    if (h[4]) CK(cudaStreamWaitEvent(ctx->s, ctx->join, 0));
    return TL_OK;
}

template <int ALGO>
tl_status launch_flags(tl_ctx* ctx, unsigned F, ListParams base, uint32_t* const lists[kClasses],
                       const unsigned h[kClasses + 1], unsigned int* queues) {
    switch (F & 7u) {
        case 0: return launch_classes<ALGO, 0>(ctx, base, lists, h, queues);
        case 1: return launch_classes<ALGO, 1>(ctx, base, lists, h, queues);
        case 2: return launch_classes<ALGO, 2>(ctx, base, lists, h, queues);
        case 3: return launch_classes<ALGO, 3>(ctx, base, lists, h, queues);
        case 4: return launch_classes<ALGO, 4>(ctx, base, lists, h, queues);
        case 5: return launch_classes<ALGO, 5>(ctx, base, lists, h, queues);
        case 6: return launch_classes<ALGO, 6>(ctx, base, lists, h, queues);
        default: return launch_classes<ALGO, 7>(ctx, base, lists, h, queues);
    }
}

}  // namespace

extern "C" {

TL_API int tl_version(void) { return 1; }

TL_API tl_status tl_create(tl_ctx** out, int device) {
    if (!out) return TL_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        (void)cudaGetLastError();
        g_create_error = std::string("tl_create: no CUDA device available (") +
                         (e != cudaSuccess ? cudaGetErrorString(e) : "device count 0") + ")";
        return TL_ERR_CUDA;
    }
    if (device < 0 || device >= count) {
        g_create_error = "tl_create: device index out of range";
        return TL_ERR_INVALID_ARGUMENT;
    }
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess || prop.major < 10) {
        g_create_error = e != cudaSuccess ? std::string("tl_create: ") + cudaGetErrorString(e)
                                          : "tl_create: this engine is built for sm_100a (B200) only";
        return TL_ERR_CUDA;
    }
    tl_ctx* ctx = new tl_ctx();
    ctx->device = device;
    ctx->sms = prop.multiProcessorCount;
    if ((e = cudaSetDevice(device)) != cudaSuccess || (e = cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->s2, cudaStreamNonBlocking)) != cudaSuccess) {
        g_create_error = std::string("tl_create: ") + cudaGetErrorString(e);
        delete ctx;
        return TL_ERR_CUDA;
    }
    for (auto& ev : ctx->ev) cudaEventCreate(&ev);
    for (auto& ev : ctx->cls_ev) cudaEventCreate(&ev);
    for (auto& ev : ctx->sort_ev) cudaEventCreate(&ev);
    cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming);
    *out = ctx;
    return TL_OK;
}

TL_API void tl_destroy(tl_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->s);
    cudaStreamSynchronize(ctx->s2);
    DevBuf* bufs[] = {&ctx->goff,   &ctx->gadj,   &ctx->rank,  &ctx->inv,    &ctx->radj,      &ctx->out_off,
                      &ctx->out_adj, &ctx->in_off, &ctx->in_adj, &ctx->outdeg, &ctx->indeg,     &ctx->lists,
                      &ctx->acc,    &ctx->vcount, &ctx->tri,   &ctx->scan_part, &ctx->bitmaps, &ctx->small,
                      &ctx->hv,     &ctx->sort_tmp, &ctx->labels, &ctx->holes, &ctx->segs};
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    for (auto& ev : ctx->ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->cls_ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->sort_ev) cudaEventDestroy(ev);
    if (ctx->timer0) cudaEventDestroy(ctx->timer0);
    if (ctx->timer1) cudaEventDestroy(ctx->timer1);
    cudaEventDestroy(ctx->fork);
    cudaEventDestroy(ctx->join);
    cudaStreamDestroy(ctx->s);
    cudaStreamDestroy(ctx->s2);
    delete ctx;
}

TL_API const char* tl_last_error(const tl_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

TL_API tl_status tl_check_sizes(uint32_t graph_n, uint32_t rank_n) {
    return graph_n == rank_n ? TL_OK : TL_ERR_INVALID_ARGUMENT;
}

static tl_status check_args(tl_ctx* ctx, uint32_t n, uint64_t m, const void* off, const void* adj, const void* rank,
                            bool need_rank = true) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    ctx->launches = 0;
    if ((n && (!off || (need_rank && !rank))) || (m && !adj))
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: null input pointer");
    if (n == 0xFFFFFFFFu) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: n must be < 2^32 - 1 (VertexId, common.hpp:11-13)");
    if (n > 0xFFF00000u)  // the listing pads partial quads with kNone, which must lie 2^20 above every rank
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: n > 2^32 - 2^20 is not supported by the listing engine");
    if (m > (uint64_t)n * (n ? n - 1 : 0) / 2) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: m exceeds n(n-1)/2");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    return TL_OK;
}

TL_API tl_status tl_orient(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                           const uint32_t* rank) {
    tl_status st = check_args(ctx, n, m, offsets, adj, rank);
    if (st != TL_OK) return st;
    if (n && offsets[0] != 0) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: offsets[0] must be 0");
    if (n && offsets[n] != 2 * m) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: offsets[n] must equal 2m");
    ctx->normalized = false;  // goff / gadj are overwritten
    ENSURE(goff, ((size_t)n + 1) * 8);
    ENSURE(gadj, 2 * m * 4);
    ENSURE(rank, (size_t)n * 4);
    CK(cudaEventRecord(ctx->ev[PH_COUNT + 2], ctx->s));
    CK(cudaMemcpyAsync(ctx->goff.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, ctx->s));
    if (m) CK(cudaMemcpyAsync(ctx->gadj.p, adj, 2 * m * 4, cudaMemcpyHostToDevice, ctx->s));
    if (n) CK(cudaMemcpyAsync(ctx->rank.p, rank, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->s));
    CK(cudaEventRecord(ctx->ev[PH_H2D], ctx->s));
    st = orient_core(ctx, n, m, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    ctx->h2d_ms = ctx->phase_ms[PH_H2D] = ev_ms(ctx->ev[PH_COUNT + 2], ctx->ev[PH_H2D]);
    return TL_OK;
}

// Degree / split order on the device into d_rank (device, n entries).
static tl_status order_core(tl_ctx* ctx, uint32_t n, const uint64_t* d_off, int method, uint32_t* d_rank) {
    if (method == TL_ORDER_CORE)
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "order: TL_ORDER_CORE needs the adjacency (tl_core_decompose)");
    if (method != TL_ORDER_DEGREE && method != TL_ORDER_SPLIT)
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "order: method must be TL_ORDER_DEGREE or TL_ORDER_SPLIT");
    if (!n) return TL_OK;
    // keys / values in and out: 4 x n words of `lists` (free outside tl_list)
    ENSURE(lists, (size_t)n * 4 * kClasses);
    uint32_t* L = P<uint32_t>(ctx->lists);
    uint32_t *k_in = L, *v_in = L + n, *k_out = L + 2 * (uint64_t)n, *v_out = L + 3 * (uint64_t)n;
    k_degree_keys<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(n, d_off, method == TL_ORDER_SPLIT, k_in,
                                                                        v_in);
    LAUNCHED();
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, v_out, (int)n, 0, 32, ctx->s));
    ENSURE(sort_tmp, tmp_bytes + 16);
    CK(cub::DeviceRadixSort::SortPairs(ctx->sort_tmp.p, tmp_bytes, k_in, k_out, v_in, v_out, (int)n, 0, 32, ctx->s));
    ctx->launches += 8;  // cub's onesweep passes (histogram + 4 x scan/sweep), approximate
    k_rank_from_sequence<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(n, v_out, method == TL_ORDER_SPLIT,
                                                                               d_rank);
    LAUNCHED();
    return TL_OK;
}

// core_decompose (ordering.cpp:141-188) on the device: coreness into `indeg`
// (n words), the degeneracy order's ranks into d_rank, level-synchronous
// peeling (core.cuh). d_off / d_adj: the Graph CSR on the device.
static tl_status core_order_core(tl_ctx* ctx, uint32_t n, const uint64_t* d_off, const uint32_t* d_adj,
                                 uint32_t* d_rank, uint32_t* degeneracy) {
    if (degeneracy) *degeneracy = 0;
    if (!n) return TL_OK;
    ENSURE(lists, (size_t)n * 4 * kClasses);
    ENSURE(outdeg, (size_t)n * 4 + 4);
    ENSURE(indeg, (size_t)n * 4 + 4);
    ENSURE(small, 128);
    uint32_t* L = P<uint32_t>(ctx->lists);
    uint32_t *alive = L, *kept = L + n, *f0 = L + 2 * (uint64_t)n, *f1 = L + 3 * (uint64_t)n;
    CoreState S{d_off, d_adj, P<uint32_t>(ctx->outdeg), L + 4 * (uint64_t)n, P<uint32_t>(ctx->indeg)};
    auto* acc = static_cast<unsigned int*>(ctx->small.p);  // [0] frontier, [1] kept, [2] min kept degree, [4..5] small-kernel state
    const unsigned big = ctx->sms * 16;
    k_core_init<<<grid_for(n, 256, big), 256, 0, ctx->s>>>(n, S, alive);
    LAUNCHED();
    uint32_t k = 0, r = 0, nalive = n, maxcore = 0;
    unsigned int h[8];
    while (nalive) {
        const unsigned int init[3] = {0u, 0u, kNone};
        CK(cudaMemcpyAsync(acc, init, sizeof init, cudaMemcpyHostToDevice, ctx->s));
        k_core_scan<<<grid_for(nalive, 256, big), 256, 0, ctx->s>>>(alive, nalive, S, k, r, f0, kept, acc);
        LAUNCHED();
        CK(cudaMemcpyAsync(h, acc, 12, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        std::swap(alive, kept);
        nalive = h[1];
        uint32_t count = h[0];
        if (!count) {  // empty level: jump to the smallest remaining degree
            if (nalive) k = h[2];
            continue;
        }
        maxcore = k;
        ++r;
        uint32_t *cur = f0, *nxt = f1;
        while (count) {
            if (count <= kCoreQ) {
                k_core_peel_small<<<1, 1024, 0, ctx->s>>>(cur, count, S, k, r, nxt, acc + 4);
                LAUNCHED();
                CK(cudaMemcpyAsync(h, acc + 4, 8, cudaMemcpyDeviceToHost, ctx->s));
                CK(cudaStreamSynchronize(ctx->s));
                r += h[0];
                count = h[1];
            } else {
                CK(cudaMemsetAsync(acc, 0, 4, ctx->s));
                k_core_peel<<<grid_for((uint64_t)count * 32, 256, big), 256, 0, ctx->s>>>(cur, count, S, k, r, nxt, acc);
                LAUNCHED();
                CK(cudaMemcpyAsync(h, acc, 4, cudaMemcpyDeviceToHost, ctx->s));
                CK(cudaStreamSynchronize(ctx->s));
                ++r;
                count = h[0];
            }
            std::swap(cur, nxt);
        }
        ++k;
    }
    if (degeneracy) *degeneracy = maxcore;
    // order = (removal round, id) ascending: one stable radix sort of the ids by round
    uint32_t *v_in = L, *k_out = L + n, *v_out = L + 2 * (uint64_t)n;
    k_core_iota<<<grid_for(n, 256, big), 256, 0, ctx->s>>>(n, v_in);
    LAUNCHED();
    int bits = 1;
    while (bits < 32 && (r >> bits)) ++bits;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, S.rnd, k_out, v_in, v_out, (int)n, 0, bits, ctx->s));
    ENSURE(sort_tmp, tmp_bytes + 16);
    CK(cub::DeviceRadixSort::SortPairs(ctx->sort_tmp.p, tmp_bytes, S.rnd, k_out, v_in, v_out, (int)n, 0, bits, ctx->s));
    ctx->launches += 2 * ((bits + 7) / 8);
    k_rank_from_sequence<<<grid_for(n, 256, big), 256, 0, ctx->s>>>(n, v_out, false, d_rank);
    LAUNCHED();
    return TL_OK;
}

TL_API tl_status tl_core_decompose_device(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* d_offsets,
                                          const uint32_t* d_adj, uint32_t* d_rank, uint32_t* d_coreness,
                                          uint32_t* degeneracy) {
    if (!ctx || (n && (!d_offsets || !d_rank)) || (m && !d_adj)) return TL_ERR_INVALID_ARGUMENT;
    if (n == 0xFFFFFFFFu) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "core_decompose: n must be < 2^32 - 1");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    ctx->oriented = false;  // outdeg / indeg / lists are reused
    drop_results(ctx);
    tl_status st = core_order_core(ctx, n, d_offsets, d_adj, d_rank, degeneracy);
    if (st != TL_OK) return st;
    if (n && d_coreness) CK(cudaMemcpyAsync(d_coreness, ctx->indeg.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_core_decompose(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                                   uint32_t* rank, uint32_t* coreness, uint32_t* degeneracy) {
    tl_status st = check_args(ctx, n, m, offsets, adj, nullptr, false);
    if (st != TL_OK) return st;
    if (n && offsets[0] != 0) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "core_decompose: offsets[0] must be 0");
    if (n && offsets[n] != 2 * m) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "core_decompose: offsets[n] must equal 2m");
    ctx->normalized = false;  // goff / gadj are overwritten
    ctx->oriented = false;
    drop_results(ctx);
    ENSURE(goff, ((size_t)n + 1) * 8);
    ENSURE(gadj, 2 * m * 4);
    ENSURE(rank, (size_t)n * 4 + 4);
    CK(cudaMemcpyAsync(ctx->goff.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, ctx->s));
    if (m) CK(cudaMemcpyAsync(ctx->gadj.p, adj, 2 * m * 4, cudaMemcpyHostToDevice, ctx->s));
    st = core_order_core(ctx, n, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank), degeneracy);
    if (st != TL_OK) return st;
    if (n && rank) CK(cudaMemcpyAsync(rank, ctx->rank.p, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->s));
    if (n && coreness) CK(cudaMemcpyAsync(coreness, ctx->indeg.p, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_order_device(tl_ctx* ctx, uint32_t n, const uint64_t* d_offsets, int method, uint32_t* d_rank) {
    if (!ctx || (n && (!d_offsets || !d_rank))) return TL_ERR_INVALID_ARGUMENT;
    if (n == 0xFFFFFFFFu) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "order: n must be < 2^32 - 1");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    tl_status st = order_core(ctx, n, d_offsets, method, d_rank);
    if (st != TL_OK) return st;
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_order(tl_ctx* ctx, uint32_t n, const uint64_t* offsets, int method, uint32_t* rank) {
    if (!ctx || (n && (!offsets || !rank))) return TL_ERR_INVALID_ARGUMENT;
    if (n == 0xFFFFFFFFu) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "order: n must be < 2^32 - 1");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    // goff and rank are overwritten: the view, its results and a normalized graph go
    ctx->normalized = false;
    ctx->oriented = false;
    drop_results(ctx);
    ENSURE(goff, ((size_t)n + 1) * 8);
    ENSURE(rank, (size_t)n * 4 + 4);
    CK(cudaMemcpyAsync(ctx->goff.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, ctx->s));
    tl_status st = order_core(ctx, n, P<uint64_t>(ctx->goff), method, P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    if (n) CK(cudaMemcpyAsync(rank, ctx->rank.p, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_orient_ordered(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                                   int method) {
    tl_status st = check_args(ctx, n, m, offsets, adj, nullptr, false);
    if (st != TL_OK) return st;
    if (n && offsets[0] != 0) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: offsets[0] must be 0");
    if (n && offsets[n] != 2 * m) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "orient: offsets[n] must equal 2m");
    ctx->normalized = false;  // goff / gadj are overwritten
    ENSURE(goff, ((size_t)n + 1) * 8);
    ENSURE(gadj, 2 * m * 4);
    ENSURE(rank, (size_t)n * 4 + 4);
    CK(cudaEventRecord(ctx->ev[PH_COUNT + 2], ctx->s));
    CK(cudaMemcpyAsync(ctx->goff.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, ctx->s));
    if (m) CK(cudaMemcpyAsync(ctx->gadj.p, adj, 2 * m * 4, cudaMemcpyHostToDevice, ctx->s));
    st = method == TL_ORDER_CORE
             ? core_order_core(ctx, n, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank), nullptr)
             : order_core(ctx, n, P<uint64_t>(ctx->goff), method, P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    CK(cudaEventRecord(ctx->ev[PH_H2D], ctx->s));
    st = orient_core(ctx, n, m, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    ctx->h2d_ms = ctx->phase_ms[PH_H2D] = ev_ms(ctx->ev[PH_COUNT + 2], ctx->ev[PH_H2D]);
    return TL_OK;
}

// ---- raw edge list -> Graph CSR on the device (normalize, graph.cpp:115-151) --
TL_API tl_status tl_normalize(tl_ctx* ctx, uint64_t k, const int64_t* edges, uint32_t* n_out, uint64_t* m_out,
                              uint64_t* loops_removed, uint64_t* duplicates_removed) {
    if (!ctx || (k && !edges) || !n_out || !m_out) return TL_ERR_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    ctx->normalized = false;
    ctx->oriented = false;  // goff / gadj / outdeg / radj are reused below
    drop_results(ctx);
    if (k > (1ull << 40)) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "normalize: more than 2^40 raw edges");
    // scratch: three regions of 16k bytes in radj (see normalize.cuh)
    const size_t R = std::max<size_t>(k * 16, 64);
    ENSURE(radj, 3 * R);
    ENSURE(small, 128);
    auto* flags = static_cast<unsigned long long*>(ctx->small.p);  // [0] loops, [2] / [3] selected counts
    CK(cudaMemsetAsync(flags, 0, 64, ctx->s));
    auto* base = static_cast<unsigned char*>(ctx->radj.p);
    long long* raw = reinterpret_cast<long long*>(base);
    unsigned char* r1 = base + R;
    unsigned char* r2 = base + 2 * R;
    auto* nsel = reinterpret_cast<long long*>(flags + 2);
    const unsigned big = ctx->sms * 16;
    if (k) CK(cudaMemcpyAsync(raw, edges, k * 16, cudaMemcpyHostToDevice, ctx->s));
    // cub scratch for the largest call of each kind
    size_t tmp_bytes = 0, tb = 0;
    const int64_t k2 = static_cast<int64_t>(2 * k);
    CK(cub::DeviceSelect::Flagged(nullptr, tb, raw, r2, reinterpret_cast<long long*>(r1), nsel, k2, ctx->s));
    tmp_bytes = std::max(tmp_bytes, tb);
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, reinterpret_cast<long long*>(r1), reinterpret_cast<long long*>(r2),
                                      k2, 0, 64, ctx->s));
    tmp_bytes = std::max(tmp_bytes, tb);
    CK(cub::DeviceSelect::Unique(nullptr, tb, reinterpret_cast<long long*>(r2), reinterpret_cast<long long*>(r1), nsel,
                                 k2, ctx->s));
    tmp_bytes = std::max(tmp_bytes, tb);
    ENSURE(sort_tmp, tmp_bytes + 64);
    // 1. labels: sorted distinct endpoints of the non-loop edges
    uint64_t e2 = 0;
    if (k) {
        k_loop_flags<<<grid_for(k, 256, big), 256, 0, ctx->s>>>(k, raw, r2, flags);
        LAUNCHED();
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceSelect::Flagged(ctx->sort_tmp.p, tb, raw, r2, reinterpret_cast<long long*>(r1), nsel, k2, ctx->s));
        long long e2_i = 0;
        CK(cudaMemcpyAsync(&e2_i, nsel, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        e2 = static_cast<uint64_t>(e2_i);
        ctx->launches += 3;
    }
    unsigned long long loops = 0;
    CK(cudaMemcpyAsync(&loops, flags, 8, cudaMemcpyDeviceToHost, ctx->s));
    uint64_t n64 = 0;
    if (e2) {
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceRadixSort::SortKeys(ctx->sort_tmp.p, tb, reinterpret_cast<long long*>(r1),
                                          reinterpret_cast<long long*>(r2), static_cast<int64_t>(e2), 0, 64, ctx->s));
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceSelect::Unique(ctx->sort_tmp.p, tb, reinterpret_cast<long long*>(r2),
                                     reinterpret_cast<long long*>(r1), nsel, static_cast<int64_t>(e2), ctx->s));
        ctx->launches += 10;
        long long n_i = 0;
        CK(cudaMemcpyAsync(&n_i, nsel, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        n64 = static_cast<uint64_t>(n_i);
    }
    CK(cudaStreamSynchronize(ctx->s));
    if (n64 > 0xFFF00000ull)  // the listing engine's limit (check_args)
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "normalize: more than 2^32 - 2^20 distinct labels");
    const uint32_t n = static_cast<uint32_t>(n64);
    ENSURE(labels, std::max<uint64_t>(n, 1) * 8);
    long long* lab = P<long long>(ctx->labels);
    if (n) CK(cudaMemcpyAsync(lab, r1, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->s));
    // 2-3. one key per raw edge, sorted and deduplicated: the kept edges
    const int hi_bits = 32 + std::max(1, 32 - __builtin_clz(std::max(n, 2u) - 1));
    auto* ekeys = reinterpret_cast<unsigned long long*>(r1);
    auto* esorted = reinterpret_cast<unsigned long long*>(r2);
    auto* edges_u = reinterpret_cast<unsigned long long*>(r1);
    uint64_t m = 0;
    if (e2) {
        k_edge_keys<<<grid_for(k, 256, big), 256, 0, ctx->s>>>(k, raw, lab, n, ekeys);
        LAUNCHED();
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceRadixSort::SortKeys(ctx->sort_tmp.p, tb, ekeys, esorted, static_cast<int64_t>(k), 0, hi_bits,
                                          ctx->s));
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceSelect::Unique(ctx->sort_tmp.p, tb, esorted, edges_u, nsel, static_cast<int64_t>(k), ctx->s));
        ctx->launches += 10;
        long long u_i = 0;
        CK(cudaMemcpyAsync(&u_i, nsel, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        m = static_cast<uint64_t>(u_i) - (loops ? 1 : 0);  // the loop key sorts last
    }
    // 4. CSR: directed pair keys, one sort -> rows sorted; degrees -> offsets
    ENSURE(goff, ((size_t)n + 1) * 8);
    ENSURE(gadj, std::max<uint64_t>(2 * m, 1) * 4);
    ENSURE(outdeg, (size_t)std::max<uint32_t>(n, 1) * 4);
    auto* dkeys = reinterpret_cast<unsigned long long*>(raw);  // 2m <= 2k words
    auto* dsorted = reinterpret_cast<unsigned long long*>(r2);
    if (n) CK(cudaMemsetAsync(ctx->outdeg.p, 0, (size_t)n * 4, ctx->s));
    if (m) {
        k_directed_keys<<<grid_for(m, 256, big), 256, 0, ctx->s>>>(m, edges_u, dkeys, P<uint32_t>(ctx->outdeg));
        LAUNCHED();
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, dkeys, dsorted, static_cast<int64_t>(2 * m), 0, hi_bits, ctx->s));
        if (tb > ctx->sort_tmp.cap) ENSURE(sort_tmp, tb + 64);
        tb = ctx->sort_tmp.cap;
        CK(cub::DeviceRadixSort::SortKeys(ctx->sort_tmp.p, tb, dkeys, dsorted, static_cast<int64_t>(2 * m), 0, hi_bits,
                                          ctx->s));
        ctx->launches += 8;
        k_low_words<<<grid_for(2 * m, 256, big), 256, 0, ctx->s>>>(2 * m, dsorted, P<uint32_t>(ctx->gadj));
        LAUNCHED();
    }
    tl_status st = scan_offsets(ctx, n, P<uint32_t>(ctx->outdeg), P<uint64_t>(ctx->goff));
    if (st != TL_OK) return st;
    CK(cudaStreamSynchronize(ctx->s));
    ctx->normalized = true;
    ctx->norm_n = n;
    ctx->norm_m = m;
    *n_out = n;
    *m_out = m;
    if (loops_removed) *loops_removed = loops;
    if (duplicates_removed) *duplicates_removed = k - loops - m;
    return TL_OK;
}

TL_API tl_status tl_fetch_graph(tl_ctx* ctx, uint64_t* offsets, uint32_t* adj, int64_t* labels) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->normalized) return ctx->fail(TL_ERR_STATE, "tl_fetch_graph: no normalized graph (call tl_normalize)");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    const uint32_t n = ctx->norm_n;
    const uint64_t m = ctx->norm_m;
    if (offsets) CK(cudaMemcpyAsync(offsets, ctx->goff.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, ctx->s));
    if (adj && m) CK(cudaMemcpyAsync(adj, ctx->gadj.p, 2 * m * 4, cudaMemcpyDeviceToHost, ctx->s));
    if (labels && n) CK(cudaMemcpyAsync(labels, ctx->labels.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

// Orient the device-resident normalized graph with a device ordering: the
// whole path raw edges -> listing without a host round trip.
TL_API tl_status tl_orient_normalized(tl_ctx* ctx, int method) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->normalized) return ctx->fail(TL_ERR_STATE, "tl_orient_normalized: no normalized graph (call tl_normalize)");
    const uint32_t n = ctx->norm_n;
    tl_status st = check_args(ctx, n, ctx->norm_m, ctx->goff.p, ctx->gadj.p, nullptr, false);
    if (st != TL_OK) return st;
    ENSURE(rank, (size_t)n * 4 + 4);
    st = method == TL_ORDER_CORE
             ? core_order_core(ctx, n, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank), nullptr)
             : order_core(ctx, n, P<uint64_t>(ctx->goff), method, P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    CK(cudaEventRecord(ctx->ev[PH_H2D], ctx->s));
    st = orient_core(ctx, n, ctx->norm_m, P<uint64_t>(ctx->goff), P<uint32_t>(ctx->gadj), P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    ctx->h2d_ms = ctx->phase_ms[PH_H2D] = 0;
    ctx->view_normalized = true;  // goff / gadj / labels untouched by orientation
    return TL_OK;
}

TL_API tl_status tl_fetch_ranks(tl_ctx* ctx, uint32_t* rank) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->oriented) return ctx->fail(TL_ERR_STATE, "tl_fetch_ranks: no oriented view");
    if (ctx->n && !rank) return TL_ERR_INVALID_ARGUMENT;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    if (ctx->n) CK(cudaMemcpyAsync(rank, ctx->rank.p, (size_t)ctx->n * 4, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_orient_device(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* d_offsets,
                                  const uint32_t* d_adj, const uint32_t* d_rank) {
    tl_status st = check_args(ctx, n, m, d_offsets, d_adj, d_rank);
    if (st != TL_OK) return st;
    // keep pi: exports map ranks back to dense ids after the call returns
    ENSURE(rank, (size_t)n * 4);
    CK(cudaEventRecord(ctx->ev[PH_H2D], ctx->s));
    if (n) CK(cudaMemcpyAsync(ctx->rank.p, d_rank, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->s));
    st = orient_core(ctx, n, m, d_offsets, d_adj, P<uint32_t>(ctx->rank));
    if (st != TL_OK) return st;
    ctx->h2d_ms = ctx->phase_ms[PH_H2D] = 0;
    return TL_OK;
}

TL_API tl_status tl_list(tl_ctx* ctx, int algo, unsigned out_flags, tl_stats* out) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    return tl_list_range(ctx, algo, out_flags, 0, ctx->n, out);
}

TL_API tl_status tl_list_range(tl_ctx* ctx, int algo, unsigned out_flags, uint32_t rank_begin, uint32_t rank_end,
                               tl_stats* out) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->oriented) return ctx->fail(TL_ERR_STATE, "tl_list: no oriented view (call tl_orient first)");
    if (algo != TL_ALGO_APP && algo != TL_ALGO_APM) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_list: algo must be TL_ALGO_APP or TL_ALGO_APM");
    if (out_flags & ~7u) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_list: unknown output flag");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    if ((uint64_t)ctx->max_out * 32 >= (1ull << 32))
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_list: out-degree >= 2^27 is not supported");
    const uint32_t n = ctx->n;
    if (rank_begin > rank_end || rank_end > n)
        return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_list_range: need rank_begin <= rank_end <= n");
    const bool full = rank_begin == 0 && rank_end == n;
    tl_status st;
    ctx->launches = 0;  // this call's kernels; the last orient's are in orient_launches
    if (algo == TL_ALGO_APP) {
        st = ensure_in_csr(ctx);
        if (st != TL_OK) return st;
    }
    ENSURE(acc, 8 * sizeof(unsigned long long));
    ENSURE(small, 128);
    auto* acc = P<unsigned long long>(ctx->acc);
    auto* counts = static_cast<unsigned int*>(ctx->small.p);  // [0..4] class sizes, [8..12] queues
    const bool want_vc = out_flags & TL_OUT_VERTEX_COUNTS;
    const bool want_list = out_flags & TL_OUT_LIST;
    if (want_vc) ENSURE(vcount, (size_t)n * 8);

    ListParams base{};
    base.n = n;
    base.set_off = algo == TL_ALGO_APM ? P<uint64_t>(ctx->out_off) : P<uint64_t>(ctx->in_off);
    base.set_len = algo == TL_ALGO_APM ? P<uint32_t>(ctx->outdeg) : P<uint32_t>(ctx->indeg);
    base.set_adj = algo == TL_ALGO_APM ? P<uint32_t>(ctx->out_adj) : P<uint32_t>(ctx->in_adj);
    base.out_off = P<uint64_t>(ctx->out_off);
    base.out_len = P<uint32_t>(ctx->outdeg);
    base.out_adj = P<uint32_t>(ctx->out_adj);
    base.inv = P<uint32_t>(ctx->inv);
    if ((out_flags & TL_OUT_CHECKSUM) && !ctx->hv_built) {
        // checksum sink: h(dense id) per rank, once per orientation
        ENSURE(hv, ((size_t)n + 1) * 8);
        {
            k_vertex_hash<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(n, P<uint32_t>(ctx->inv),
                                                                              P<unsigned long long>(ctx->hv));
            LAUNCHED();
        }
        ctx->hv_built = true;
    }
    base.hv = P<unsigned long long>(ctx->hv);
    base.acc = acc;
    base.vcount = want_vc ? P<unsigned long long>(ctx->vcount) : nullptr;
    base.variant = ctx->variant;
    base.hot_rank = ctx->hot_rank;
    base.r_search = ctx->max_out < kLongRow;  // no long rows anywhere: class R searches instead of probing a bitmap
    base.hist_base = n > kHist ? n - kHist : 0;
    base.bm_shrink = ctx->bm_shrink;

    CK(cudaEventRecord(ctx->ev[PH_COUNT + 3], ctx->s));
    CK(cudaMemsetAsync(counts, 0, 16 * sizeof(unsigned int), ctx->s));
    uint32_t* L = P<uint32_t>(ctx->lists);
    uint32_t* const lists[kClasses] = {L, L + n, L + 2 * (uint64_t)n, L + 3 * (uint64_t)n, L + 4 * (uint64_t)n};
    // class H in two lists (front / back of lists[1]) when the graph is large: seeds of
    // |S| <= h_split stay on the warp kernel, the others go CTA-wide
    const uint32_t h_small = n > ctx->h_cta_min_n ? ctx->h_split : 0u;
    SeedLists SL{{lists[0], lists[1], lists[2], lists[3], lists[4]}, counts, n, h_small};
    if (rank_end > rank_begin) {
        k_classify_seeds<<<grid_for(rank_end - rank_begin, 256, ctx->sms * 16), 256, 0, ctx->s>>>(
            rank_begin, rank_end, base.set_len, SL);
        LAUNCHED();
    }
    unsigned long long range_ops[2] = {0, 0};  // inner_ops, mark_ops of a partial range
    if (!full) {
        auto* rc = reinterpret_cast<unsigned long long*>(counts + 16);  // small[64..80)
        CK(cudaMemsetAsync(rc, 0, 16, ctx->s));
        if (rank_end > rank_begin) {
            k_range_cost<<<grid_for((uint64_t)(rank_end - rank_begin) * 32, 256, ctx->sms * 16), 256, 0, ctx->s>>>(
                rank_begin, rank_end, base.set_off, base.set_len, base.set_adj, base.out_len, rc);
            LAUNCHED();
        }
        CK(cudaMemcpyAsync(range_ops, rc, 16, cudaMemcpyDeviceToHost, ctx->s));
    }
    CK(cudaEventRecord(ctx->ev[PH_CLASSIFY], ctx->s));
    unsigned h[kClasses + 1];  // [kClasses] = small class-H seeds
    CK(cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    if (ctx->class_work) {  // per-class inner_ops (debug; outside the timed listing)
        auto* wk = reinterpret_cast<unsigned long long*>(counts + 20);  // small[80..120)
        CK(cudaMemsetAsync(wk, 0, kClasses * 8, ctx->s));
        for (int c = 0; c < kClasses; ++c)
            if (h[c]) {
                k_class_work<<<grid_for((uint64_t)h[c] * 32, 256, ctx->sms * 16), 256, 0, ctx->s>>>(
                    lists[c], h[c], base.set_off, base.set_len, base.set_adj, base.out_len, wk + c);
                LAUNCHED();
            }
        if (h[kClasses]) {
            k_class_work<<<grid_for((uint64_t)h[kClasses] * 32, 256, ctx->sms * 16), 256, 0, ctx->s>>>(
                lists[1] + (n - h[kClasses]), h[kClasses], base.set_off, base.set_len, base.set_adj, base.out_len,
                wk + 1);
            LAUNCHED();
        }
        unsigned long long w[kClasses];
        CK(cudaMemcpyAsync(w, wk, sizeof(w), cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        for (int c = 0; c < kClasses; ++c) ctx->phase_ms[PH_WORK_R + c] = static_cast<double>(w[c]);
    }

    CK(cudaEventRecord(ctx->ev[PH_COUNT + 4], ctx->s));  // listing kernels start
    auto run = [&](unsigned F) -> tl_status {
        for (bool& r : ctx->cls_run) r = false;
        CK(cudaMemsetAsync(acc, 0, 8 * sizeof(unsigned long long), ctx->s));  // counts, checksum, list cursors
        CK(cudaMemsetAsync(counts + 8, 0, 8 * sizeof(unsigned int), ctx->s));
        if (F & F_VCOUNT) CK(cudaMemsetAsync(ctx->vcount.p, 0, (size_t)n * 8, ctx->s));
        return algo == TL_ALGO_APM ? launch_flags<ALGO_APM>(ctx, F, base, lists, h, counts + 8)
                                   : launch_flags<ALGO_APP>(ctx, F, base, lists, h, counts + 8);
    };
    unsigned long long res[4] = {0, 0, 0, 0};
    constexpr unsigned kHolesCap = 1u << 17;  // >= every warp of every class launch
    if (want_list) {
        // One pass into the context's triangle buffer (grow-only, kept across
        // calls): warps claim kListChunk slots at a time, writes stop at
        // capacity. Only when the claims outgrow the buffer is it grown and
        // the pass repeated. First call: a quarter of the free device memory,
        // at most 2^31 triangles.
        if (ctx->tri.cap < 12 * 64) {
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
                (void)cudaGetLastError();
                free_b = 0;
            }
            const size_t want = std::min<size_t>(free_b / 4, (size_t{1} << 31) * 12);
            ENSURE(tri, std::max<size_t>(want / 12 * 12, 12 * 64));
        }
        ENSURE(holes, (size_t)kHolesCap * 16);
        base.tri = P<uint32_t>(ctx->tri);
        base.tri_cap = ctx->tri.cap / 12;
        base.holes = P<ulonglong2>(ctx->holes);
        base.holes_cap = kHolesCap;
    }
    st = run(out_flags);
    if (st != TL_OK) return st;
    CK(cudaMemcpyAsync(res, acc, sizeof(res), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    if (want_list && res[2] > base.tri_cap) {
        ENSURE(tri, (size_t)res[2] * 12 + (size_t)kListChunk * 12 * 4096);
        base.tri = P<uint32_t>(ctx->tri);
        base.tri_cap = ctx->tri.cap / 12;
        st = run(out_flags);
        if (st != TL_OK) return st;
        CK(cudaMemcpyAsync(res, acc, sizeof(res), cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        if (res[2] > base.tri_cap)
            return ctx->fail(TL_ERR_CUDA, "tl_list: list claims outgrew the regrown buffer");
    }
    if (want_list) {
        // Compaction: the chunks hold every triangle in [0, claimed) except
        // the recorded tails; move the triangles above the count into the
        // tails below it (at most one tail per warp).
        const unsigned long long T = res[0], claimed = res[2], nh = res[3];
        if (nh > kHolesCap) return ctx->fail(TL_ERR_CUDA, "tl_list: too many list chunk tails");
        std::vector<std::pair<unsigned long long, unsigned long long>> hs(nh);
        if (nh) {
            std::vector<ulonglong2> hv(nh);
            CK(cudaMemcpyAsync(hv.data(), ctx->holes.p, nh * 16, cudaMemcpyDeviceToHost, ctx->s));
            CK(cudaStreamSynchronize(ctx->s));
            for (size_t i = 0; i < nh; ++i) hs[i] = {hv[i].x, hv[i].y};
            std::sort(hs.begin(), hs.end());
        }
        unsigned long long hole_total = 0;
        for (auto& h : hs) hole_total += h.second;
        if (claimed - hole_total != T)
            return ctx->fail(TL_ERR_CUDA, "tl_list: list slots disagree with the triangle count");
        // destinations: tail parts below T; sources: the filled ranges in [T, claimed)
        std::vector<std::pair<unsigned long long, unsigned long long>> dst, src;
        unsigned long long pos = T;
        for (auto& h : hs) {
            if (h.first < T) dst.push_back({h.first, std::min(h.first + h.second, T) - h.first});
            const unsigned long long hb = std::max(h.first, T), he = h.first + h.second;
            if (he > T) {
                if (hb > pos) src.push_back({pos, hb - pos});
                pos = std::max(pos, he);
            }
        }
        if (claimed > pos) src.push_back({pos, claimed - pos});
        std::vector<ulonglong2> seg;
        std::vector<unsigned long long> seglen;
        size_t si = 0;
        unsigned long long soff = 0;
        for (auto& d : dst) {
            unsigned long long doff = 0;
            while (doff < d.second) {
                if (si >= src.size()) return ctx->fail(TL_ERR_CUDA, "tl_list: list compaction ran out of sources");
                const unsigned long long len = std::min(d.second - doff, src[si].second - soff);
                seg.push_back(make_ulonglong2(src[si].first + soff, d.first + doff));
                seglen.push_back(len);
                doff += len;
                soff += len;
                if (soff == src[si].second) {
                    ++si;
                    soff = 0;
                }
            }
        }
        if (!seg.empty()) {
            ENSURE(segs, seg.size() * 24);
            auto* d_seg = P<ulonglong2>(ctx->segs);
            auto* d_len = reinterpret_cast<unsigned long long*>(d_seg + seg.size());
            CK(cudaMemcpyAsync(d_seg, seg.data(), seg.size() * 16, cudaMemcpyHostToDevice, ctx->s));
            CK(cudaMemcpyAsync(d_len, seglen.data(), seg.size() * 8, cudaMemcpyHostToDevice, ctx->s));
            k_move_triangles<<<grid_for(seg.size(), 1, ctx->sms * 8), 256, 0, ctx->s>>>(d_seg, d_len, (unsigned)seg.size(),
                                                                                        P<uint32_t>(ctx->tri));
            LAUNCHED();
        }
        res[2] = T;
    }
    CK(cudaEventRecord(ctx->ev[PH_LIST], ctx->s));
    CK(cudaEventSynchronize(ctx->ev[PH_LIST]));
    ctx->phase_ms[PH_CLASSIFY] = ev_ms(ctx->ev[PH_COUNT + 3], ctx->ev[PH_CLASSIFY]);
    ctx->phase_ms[PH_LIST] = ev_ms(ctx->ev[PH_COUNT + 4], ctx->ev[PH_LIST]);
    for (int c = 0; c < kClasses; ++c)
        ctx->phase_ms[PH_LIST_R + c] = ctx->cls_run[c] ? ev_ms(ctx->cls_ev[2 * c], ctx->cls_ev[2 * c + 1]) : 0.0;
    ctx->have_vcounts = want_vc;
    ctx->have_tri = want_list;
    ctx->tri_count = want_list ? res[2] : 0;
    if (want_list && res[2] != res[0])
        return ctx->fail(TL_ERR_CUDA, "tl_list: the list cursor disagrees with the triangle count");
    if (out) {
        std::memset(out, 0, sizeof(*out));
        out->triangle_count = res[0];
        out->checksum = (out_flags & TL_OUT_CHECKSUM) ? res[1] : 0;
        out->c_pp = ctx->cost[0];
        out->c_pm = ctx->cost[1];
        out->c_mm = ctx->cost[2];
        out->sum_deg_sq = ctx->cost[3];
        out->inner_ops = !full ? range_ops[0] : algo == TL_ALGO_APM ? ctx->cost[1] : ctx->cost[0];
        out->mark_ops = !full ? range_ops[1] : 2 * ctx->m;
        out->orient_ms = ctx->orient_ms;
        out->list_ms = ev_ms(ctx->ev[PH_COUNT + 3], ctx->ev[PH_LIST]);
        out->h2d_ms = ctx->h2d_ms;
        out->kernel_launches = ctx->orient_launches + ctx->launches;
    }
    return TL_OK;
}

TL_API tl_status tl_fetch_triangles(tl_ctx* ctx, uint32_t* uvw, uint64_t cap, uint64_t* k) {
    if (!ctx || !k) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tri) return ctx->fail(TL_ERR_STATE, "tl_fetch_triangles: last tl_list did not use TL_OUT_LIST");
    *k = ctx->tri_count;
    if (cap < ctx->tri_count) return ctx->fail(TL_ERR_CAPACITY, "tl_fetch_triangles: buffer too small");
    if (ctx->tri_count) {
        if (!uvw) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_fetch_triangles: null buffer");
        CK(cudaMemcpyAsync(uvw, ctx->tri.p, ctx->tri_count * 12, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    }
    return TL_OK;
}

TL_API tl_status tl_fetch_triangles_range(tl_ctx* ctx, uint64_t first, uint64_t cap, uint32_t* uvw, uint64_t* k) {
    if (!ctx || !k) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tri) return ctx->fail(TL_ERR_STATE, "tl_fetch_triangles_range: last tl_list did not use TL_OUT_LIST");
    *k = first < ctx->tri_count ? std::min<uint64_t>(cap, ctx->tri_count - first) : 0;
    if (*k) {
        if (!uvw) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_fetch_triangles_range: null buffer");
        if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
        CK(cudaMemcpyAsync(uvw, P<uint32_t>(ctx->tri) + 3 * first, *k * 12, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    }
    return TL_OK;
}

TL_API tl_status tl_fetch_triangle_labels(tl_ctx* ctx, uint64_t first, uint64_t cap, const int64_t* labels,
                                          int64_t* out, uint64_t* k) {
    if (!ctx || !k) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tri) return ctx->fail(TL_ERR_STATE, "tl_fetch_triangle_labels: last tl_list did not use TL_OUT_LIST");
    if (!labels && !(ctx->normalized && ctx->view_normalized))
        return ctx->fail(TL_ERR_STATE, "tl_fetch_triangle_labels: no label table (pass one, or orient a tl_normalize graph)");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    *k = first < ctx->tri_count ? std::min<uint64_t>(cap, ctx->tri_count - first) : 0;
    if (!*k) return TL_OK;
    if (!out) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_fetch_triangle_labels: null buffer");
    const long long* lab = P<long long>(ctx->labels);
    if (labels) {  // caller's table: stage it after the normalize labels' slot
        ENSURE(sort_tmp, (size_t)ctx->n * 8 + 64);
        CK(cudaMemcpyAsync(ctx->sort_tmp.p, labels, (size_t)ctx->n * 8, cudaMemcpyHostToDevice, ctx->s));
        lab = P<long long>(ctx->sort_tmp);  // normalize's scratch; its graph and labels stay valid
    }
    ENSURE(scan_part, *k * 24);
    k_map_labels<<<grid_for(*k * 3, 256, ctx->sms * 16), 256, 0, ctx->s>>>(*k * 3, P<uint32_t>(ctx->tri) + 3 * first, lab,
                                                                          P<long long>(ctx->scan_part));
    LAUNCHED();
    CK(cudaMemcpyAsync(out, ctx->scan_part.p, *k * 24, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_fetch_vertex_counts(tl_ctx* ctx, uint64_t* counts) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->have_vcounts) return ctx->fail(TL_ERR_STATE, "tl_fetch_vertex_counts: last tl_list did not use TL_OUT_VERTEX_COUNTS");
    const uint32_t n = ctx->n;
    if (!n) return TL_OK;
    if (!counts) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_fetch_vertex_counts: null buffer");
    // dense[u] = vcount[rank[u]]; staged through radj (>= 8n bytes not guaranteed) -> scan_part
    ENSURE(scan_part, (size_t)n * 8);
    k_gather_u64<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(
        n, P<unsigned long long>(ctx->vcount), P<uint32_t>(ctx->rank), P<unsigned long long>(ctx->scan_part));
    LAUNCHED();
    CK(cudaMemcpyAsync(counts, ctx->scan_part.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return TL_OK;
}

TL_API tl_status tl_fetch_oriented(tl_ctx* ctx, uint64_t* succ_off, uint32_t* succ, uint64_t* pred_off,
                                   uint32_t* pred) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->oriented) return ctx->fail(TL_ERR_STATE, "tl_fetch_oriented: no oriented view");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx->cuda_fail("cudaSetDevice", cudaGetLastError());
    const uint32_t n = ctx->n;
    const uint64_t m = ctx->m;
    if (pred_off || pred) {
        tl_status st = ensure_in_csr(ctx);
        if (st != TL_OK) return st;
    }
    DevBuf doff, dadj, ddeg;
    auto cleanup = [&] {
        if (doff.p) cudaFree(doff.p);
        if (dadj.p) cudaFree(dadj.p);
        if (ddeg.p) cudaFree(ddeg.p);
    };
    for (int side = 0; side < 2; ++side) {
        uint64_t* ho = side == 0 ? succ_off : pred_off;
        uint32_t* ha = side == 0 ? succ : pred;
        if (!ho && !ha) continue;
        tl_status st;
        if ((st = ensure(ctx, doff, ((size_t)n + 1) * 8)) != TL_OK || (st = ensure(ctx, dadj, m * 4)) != TL_OK ||
            (st = ensure(ctx, ddeg, (size_t)n * 4 + 4)) != TL_OK) {
            cleanup();
            return st;
        }
        const uint32_t* deg = side == 0 ? P<uint32_t>(ctx->outdeg) : P<uint32_t>(ctx->indeg);
        const uint64_t* roff = side == 0 ? P<uint64_t>(ctx->out_off) : P<uint64_t>(ctx->in_off);
        const uint32_t* radj = side == 0 ? P<uint32_t>(ctx->out_adj) : P<uint32_t>(ctx->in_adj);
        if (n) {
            k_gather_u32<<<grid_for(n, 256, ctx->sms * 16), 256, 0, ctx->s>>>(n, deg, P<uint32_t>(ctx->rank),
                                                                            P<uint32_t>(ddeg));
            ++ctx->launches;
        }
        st = scan_offsets(ctx, n, P<uint32_t>(ddeg), P<uint64_t>(doff));
        if (st != TL_OK) {
            cleanup();
            return st;
        }
        if (n) {
            k_export_rows<<<grid_for((uint64_t)n * 32, 256, ctx->sms * 32), 256, 0, ctx->s>>>(
                n, P<uint32_t>(ctx->rank), P<uint32_t>(ctx->inv), roff, deg, radj, P<uint64_t>(doff), P<uint32_t>(dadj));
            ++ctx->launches;
        }
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess && ho) e = cudaMemcpyAsync(ho, doff.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, ctx->s);
        if (e == cudaSuccess && ha && m) e = cudaMemcpyAsync(ha, dadj.p, m * 4, cudaMemcpyDeviceToHost, ctx->s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->s);
        if (e != cudaSuccess) {
            cleanup();
            return ctx->cuda_fail("tl_fetch_oriented", e);
        }
    }
    cleanup();
    return TL_OK;
}

TL_API tl_status tl_cost_report(tl_ctx* ctx, uint64_t out[4]) {
    if (!ctx || !out) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->oriented) return ctx->fail(TL_ERR_STATE, "tl_cost_report: no oriented view");
    for (int i = 0; i < 4; ++i) out[i] = ctx->cost[i];
    return TL_OK;
}

TL_API tl_status tl_host_register(tl_ctx* ctx, void* ptr, size_t bytes) {
    if (!ctx || !ptr) return TL_ERR_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    CK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
    return TL_OK;
}

TL_API tl_status tl_host_unregister(tl_ctx* ctx, void* ptr) {
    if (!ctx || !ptr) return TL_ERR_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    CK(cudaHostUnregister(ptr));
    return TL_OK;
}

TL_API tl_status tl_timer_start(tl_ctx* ctx) {
    if (!ctx) return TL_ERR_INVALID_ARGUMENT;
    if (!ctx->timer0) {
        CK(cudaEventCreate(&ctx->timer0));
        CK(cudaEventCreate(&ctx->timer1));
    }
    CK(cudaEventRecord(ctx->timer0, ctx->s));
    return TL_OK;
}

TL_API tl_status tl_timer_stop(tl_ctx* ctx, double* ms) {
    if (!ctx || !ms || !ctx->timer0) return TL_ERR_INVALID_ARGUMENT;
    CK(cudaEventRecord(ctx->timer1, ctx->s));
    CK(cudaEventSynchronize(ctx->timer1));
    float f = 0;
    CK(cudaEventElapsedTime(&f, ctx->timer0, ctx->timer1));
    *ms = f;
    return TL_OK;
}

TL_API int tl_phase_times(const tl_ctx* ctx, double* ms, int cap) {
    if (!ctx || !ms) return 0;
    const int k = std::min<int>(cap, PH_COUNT);
    for (int i = 0; i < k; ++i) ms[i] = ctx->phase_ms[i];
    return k;
}

TL_API const char* tl_phase_name(int i) { return (i >= 0 && i < PH_COUNT) ? kPhaseNames[i] : ""; }

TL_API tl_status tl_debug_set(tl_ctx* ctx, int key, int value) {
    if (!ctx || value < 0) return TL_ERR_INVALID_ARGUMENT;
    if (key == TL_DEBUG_BM_SHRINK) {
        if (value > 16) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_debug_set: shrink must be <= 16");
        ctx->bm_shrink = static_cast<uint32_t>(value);
        return TL_OK;
    }
    if (key == TL_DEBUG_VARIANT) {
        ctx->variant = value;
        return TL_OK;
    }
    if (key == TL_DEBUG_CLASS_WORK) {
        ctx->class_work = value != 0;
        return TL_OK;
    }
    if (key == TL_DEBUG_H_WIDE_MIN_N) {
        ctx->h_cta_min_n = ctx->wide_min_n = static_cast<uint32_t>(value);
        return TL_OK;
    }
    if (key == TL_DEBUG_H_SPLIT) {
        if (value < 0 || value > 256) return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_debug_set: H split must be in [0, 256]");
        ctx->h_split = static_cast<uint32_t>(value);
        return TL_OK;
    }
    return ctx->fail(TL_ERR_INVALID_ARGUMENT, "tl_debug_set: unknown key");
}

}  // extern "C"
