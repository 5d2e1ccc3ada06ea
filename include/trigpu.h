/*
 * trigpu.h -- C-ABI of the B200 (sm_100a) triangle-listing engine.
 *
 * Drop-in boundary for the reference trilist listing path. The reference's
 * boundary is a C++ template API, not an ABI; each entry point below names the
 * reference interface it replaces (paths under /root/reference/proj):
 *
 *   tl_orient / tl_orient_device
 *       OrientedView::OrientedView(const Graph&, const Ordering&)
 *       core/include/trilist/oriented_view.hpp:19, core/src/oriented_view.cpp:7-47
 *   tl_list
 *       list_app / list_apm (view, sink)          core/include/trilist/listing.hpp:162-173
 *       list_app_parallel / list_apm_parallel     core/include/trilist/listing.hpp:187-199
 *       ListingStats                              core/include/trilist/listing.hpp:23-34
 *       (the GPU run is always "parallel": emission order is unspecified, as
 *        listing.hpp:185-186 states for the parallel variants)
 *   tl_fetch_triangles      CollectingSink::triangles   listing.hpp:46-56
 *   tl_fetch_vertex_counts  new per-vertex sink
 *   tl_fetch_oriented       OrientedView::successors / predecessors  oriented_view.hpp:24-29
 *   tl_cost_report          cost_report(const OrientedView&)  core/src/cost.cpp:27-38
 *
 * Conventions: plain pointers and sizes, int status codes, no exceptions cross
 * the ABI. Graph inputs are the reference Graph CSR (graph.hpp:59-60):
 * offsets uint64[n+1], adjacency uint32[2m], each row strictly increasing by
 * dense id; rank[v] = 0-based position of v (Ordering::ranks(),
 * ordering.hpp:30). Everything that leaves the library is in dense ids.
 * One context owns one CUDA stream and its device buffers; callers serialise
 * use of a context; contexts are independent.
 */
#ifndef TRIGPU_H
#define TRIGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TL_API __attribute__((visibility("default")))
#else
#define TL_API
#endif

typedef struct tl_ctx tl_ctx;

typedef enum {
    TL_OK = 0,
    TL_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference (oriented_view.cpp:8-9) */
    TL_ERR_CUDA = 2,             /* no device, launch failure, ... */
    TL_ERR_OUT_OF_MEMORY = 3,
    TL_ERR_STATE = 4,            /* e.g. tl_list before tl_orient */
    TL_ERR_CAPACITY = 5          /* caller buffer too small; *k holds the size needed */
} tl_status;

/* algorithm selection (trilist_cli.cpp:124-133, --algo {app,apm}) */
enum { TL_ALGO_APP = 0, TL_ALGO_APM = 1 };

/* output sinks, OR-able (the reference's --sink {count,collect}, extended) */
enum {
    TL_OUT_COUNT = 0,          /* CountingSink: triangle_count only */
    TL_OUT_CHECKSUM = 1,       /* order-independent 64-bit checksum */
    TL_OUT_VERTEX_COUNTS = 2,  /* per-vertex triangle counts, uint64[n] */
    TL_OUT_LIST = 4            /* CollectingSink: all (u,v,w) triples */
};

typedef struct {
    /* ListingStats (listing.hpp:23-34) */
    uint64_t triangle_count;
    uint64_t inner_ops; /* = c_pp (app) or c_pm (apm) */
    uint64_t mark_ops;  /* = 2m */
    /* extensions */
    uint64_t checksum;  /* sum mod 2^64 over triangles of h(a) h(b) h(c), h(v) = mix64(v) | 1, dense ids */
    uint64_t c_pp, c_pm, c_mm, sum_deg_sq; /* CostReport (cost.hpp:15-20) */
    double orient_ms;   /* device time of the last tl_orient (relabel+CSR+sort) */
    double list_ms;     /* device time of the listing kernels (ListingStats::wall_ms analogue) */
    double h2d_ms;      /* host->device copy time of the last tl_orient (0 for _device) */
    uint64_t kernel_launches; /* kernels launched by the last tl_orient + this tl_list */
} tl_stats;

TL_API int tl_version(void);
TL_API tl_status tl_create(tl_ctx** out, int device);
TL_API void tl_destroy(tl_ctx* ctx);
/* Last error text for ctx (or for a failed tl_create when ctx is NULL). */
TL_API const char* tl_last_error(const tl_ctx* ctx);

/* Build the oriented view on the device from HOST arrays (copied in). */
TL_API tl_status tl_orient(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets,
                           const uint32_t* adj, const uint32_t* rank);
/* Same from DEVICE arrays owned by the caller, valid for the duration of the
 * call (inputs already resident in HBM). */
TL_API tl_status tl_orient_device(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* d_offsets,
                                  const uint32_t* d_adj, const uint32_t* d_rank);
/* Orderings on the device: the reference's degree order
 * (ordering.cpp:66-96: counting sort by degree, ascending, ties by ascending
 * id) and split order (ordering.cpp:98-109: degree-descending sequence, even
 * positions fill the front, odd the back), bit-identical to the reference's
 * (tests/test_gpu_parity.py). degree(v) = offsets[v + 1] - offsets[v] of the
 * Graph CSR. tl_order: host arrays in and out; tl_order_device: device
 * arrays. Replaces degree_order / split_order (ordering.hpp) on the listing
 * path; the other orderings stay the reference's host code. */
enum { TL_ORDER_DEGREE = 0, TL_ORDER_SPLIT = 1, TL_ORDER_CORE = 2 };
TL_API tl_status tl_order(tl_ctx* ctx, uint32_t n, const uint64_t* offsets, int method, uint32_t* rank);
TL_API tl_status tl_order_device(tl_ctx* ctx, uint32_t n, const uint64_t* d_offsets, int method, uint32_t* d_rank);
/* k-core decomposition on the device: replaces
 * core_decompose / core_order (ordering.cpp:141-188; CoreDecomposition,
 * ordering.hpp:56-64). coreness[v] and the degeneracy equal the reference's
 * bit for bit. rank[v] is a degeneracy ordering with the reference order's
 * defining property (every vertex has at most coreness(v) successors, so
 * max d+ = degeneracy): vertices sorted by (removal round of the level-
 * synchronous peel, id). The reference's bucket queue removes one vertex at a
 * time and breaks ties by the history of its swaps; that sequence is not
 * reproduced (csrc/core.cuh says why), so rank differs from core_order(g)
 * among ties while every listing result is unchanged. rank / coreness may be
 * NULL. tl_core_decompose: host arrays; _device: device arrays. */
TL_API tl_status tl_core_decompose(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                                   uint32_t* rank, uint32_t* coreness, uint32_t* degeneracy);
TL_API tl_status tl_core_decompose_device(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* d_offsets,
                                          const uint32_t* d_adj, uint32_t* d_rank, uint32_t* d_coreness,
                                          uint32_t* degeneracy);
/* tl_orient with the ordering computed on the device by `method`
 * (TL_ORDER_DEGREE / TL_ORDER_SPLIT / TL_ORDER_CORE): the whole path from the
 * host Graph CSR, no host ordering. The ranks can be read back with
 * tl_fetch_ranks. */
TL_API tl_status tl_orient_ordered(tl_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* offsets,
                                   const uint32_t* adj, int method);
TL_API tl_status tl_fetch_ranks(tl_ctx* ctx, uint32_t* rank);

/* Raw labeled edge list -> the reference's Graph CSR, on the device
 * (SURVEY §8f): normalize (graph.cpp:115-151: loops dropped, endpoints
 * canonicalised, duplicates merged, labels = sorted distinct endpoints,
 * dense id = label rank) + Graph::from_dense_edges (graph.cpp:13-56: sorted
 * rows). edges = k (a, b) int64 label pairs (host). The graph stays on the
 * device: tl_fetch_graph copies out offsets (n+1), adj (2m) and labels (n);
 * tl_orient_normalized orients it with a device ordering (TL_ORDER_*).
 * 64-bit item counts (k up to 2^40, memory permitting: 48 bytes of device
 * scratch per raw edge); more than 2^32 - 2^20 distinct labels is
 * TL_ERR_INVALID_ARGUMENT. Text files: th_parse_edgelist (trihost.h). */
TL_API tl_status tl_normalize(tl_ctx* ctx, uint64_t k, const int64_t* edges, uint32_t* n, uint64_t* m,
                              uint64_t* loops_removed, uint64_t* duplicates_removed);
TL_API tl_status tl_fetch_graph(tl_ctx* ctx, uint64_t* offsets, uint32_t* adj, int64_t* labels);
TL_API tl_status tl_orient_normalized(tl_ctx* ctx, int method);
/* Mismatched sizes (rank length != n) are reported as in oriented_view.cpp:8-9. */
TL_API tl_status tl_check_sizes(uint32_t graph_n, uint32_t rank_n);

/* List every triangle once over G_pi with A++ (TL_ALGO_APP, listing.hpp:69-86)
 * or A+- (TL_ALGO_APM, listing.hpp:91-107). */
TL_API tl_status tl_list(tl_ctx* ctx, int algo, unsigned out_flags, tl_stats* out);
/* tl_list restricted to the seeds whose rank lies in [rank_begin, rank_end):
 * detail::run_app_range / run_apm_range (listing.hpp:69-107) over one rank
 * range, the unit run_parallel hands its lanes (listing.hpp:122-155).
 * inner_ops / mark_ops count that range's seeds only (c_pm / c_pp and 2m
 * over the full range); every sink is supported. */
TL_API tl_status tl_list_range(tl_ctx* ctx, int algo, unsigned out_flags, uint32_t rank_begin,
                               uint32_t rank_end, tl_stats* out);

/* Copy the triangles of the last TL_OUT_LIST run: 3*k dense ids, each triple
 * rank-ascending (u, v, w), triples in unspecified order. cap in triangles.
 * TL_ERR_CAPACITY (with *k set) when cap is too small. */
TL_API tl_status tl_fetch_triangles(tl_ctx* ctx, uint32_t* uvw, uint64_t cap, uint64_t* k);
/* Chunked reads of the same list, so a caller can stream
 * a list larger than its buffers to disk: triangles [first, first + k) with
 * k = min(cap, total - first), as dense ids, or mapped to the Graph's int64
 * labels (the CLI's --out writes labels, trilist_cli.cpp:212-220). labels =
 * the label table (int64[n], host), or NULL for the labels of the last
 * tl_normalize when the oriented graph is that graph. */
TL_API tl_status tl_fetch_triangles_range(tl_ctx* ctx, uint64_t first, uint64_t cap, uint32_t* uvw, uint64_t* k);
TL_API tl_status tl_fetch_triangle_labels(tl_ctx* ctx, uint64_t first, uint64_t cap, const int64_t* labels,
                                          int64_t* out, uint64_t* k);
/* Per-vertex triangle counts (dense ids) of the last TL_OUT_VERTEX_COUNTS run. */
TL_API tl_status tl_fetch_vertex_counts(tl_ctx* ctx, uint64_t* counts);
/* The oriented view in the reference layout (oriented_view.hpp:41-45):
 * succ_off/pred_off uint64[n+1] indexed by dense id, succ/pred uint32[m]
 * holding dense ids, each row rank-ascending. Any pointer may be NULL. */
TL_API tl_status tl_fetch_oriented(tl_ctx* ctx, uint64_t* succ_off, uint32_t* succ,
                                   uint64_t* pred_off, uint32_t* pred);
/* {c_pp, c_pm, c_mm, sum_deg_sq} of the current view. */
TL_API tl_status tl_cost_report(tl_ctx* ctx, uint64_t out[4]);

/* Page-lock / unlock caller host memory so tl_orient's copies run at full
 * PCIe rate (cudaHostRegister). */
TL_API tl_status tl_host_register(tl_ctx* ctx, void* ptr, size_t bytes);
TL_API tl_status tl_host_unregister(tl_ctx* ctx, void* ptr);

/* Device-time span on the context's stream: tl_timer_stop waits for the
 * stream and returns the CUDA-event elapsed time since tl_timer_start
 * (includes every kernel, copy and idle gap of the calls in between). */
TL_API tl_status tl_timer_start(tl_ctx* ctx);
TL_API tl_status tl_timer_stop(tl_ctx* ctx, double* ms);

/* Per-phase device times (ms) of the last orient + list, named by
 * tl_phase_name(i); returns the number of phases written (<= cap). */
TL_API int tl_phase_times(const tl_ctx* ctx, double* ms, int cap);
TL_API const char* tl_phase_name(int i);

/* Test-only knobs (not part of the reference interface; the product never
 * reads the environment):
 *   TL_DEBUG_BM_SHRINK  shrink every seed's shared-memory window and filter by
 *                       2^value so graphs small enough for the oracle take the
 *                       below-window (filter + exact verification) path;
 *   TL_DEBUG_VARIANT    probe variant of a -DTRIGPU_EXPERIMENTS build (2 = null
 *                       probe, timing only); ignored otherwise;
 *   TL_DEBUG_CLASS_WORK 1: each tl_list also reports the inner_ops of every
 *                       seed class through tl_phase_times ("work_*", counts);
 *   TL_DEBUG_H_WIDE_MIN_N  the graph-size thresholds above which class H is
 *                       split between the warp and the CTA kernel (default
 *                       2^21 vertices) and class C1 uses its 2^19-window
 *                       instance (default 2^25): both are set to this value,
 *                       so tests on small graphs force those paths with 0;
 *   TL_DEBUG_H_SPLIT    largest class-H |S| left on the warp-per-seed kernel
 *                       when class H is split (default 96; 0: all CTA, 256:
 *                       all warp).
 * Settings persist for the context. */
enum {
    TL_DEBUG_BM_SHRINK = 1,
    TL_DEBUG_VARIANT = 2,
    TL_DEBUG_CLASS_WORK = 3,
    TL_DEBUG_H_WIDE_MIN_N = 4,
    TL_DEBUG_H_SPLIT = 5
};
TL_API tl_status tl_debug_set(tl_ctx* ctx, int key, int value);

#ifdef __cplusplus
}
#endif

#endif
