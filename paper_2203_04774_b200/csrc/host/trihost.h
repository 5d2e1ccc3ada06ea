/*
 * trihost.h -- host-side input preparation for the GPU listing engine.
 *
 *  - Orderings and cost reports are the reference's own C++ (ordering.cpp,
 *    neigh.cpp, cost.cpp; compiled unchanged into libtrihost.so), reached
 *    through a trilist::Graph built with Graph::from_dense_edges
 *    (graph.cpp:13-56) so dense ids are preserved (SURVEY §7 "Hard parts").
 *  - Synthetic graphs C1-C5 (BASELINE.json configs): C1 is the reference's
 *    gen_gnm (graph.cpp:210-243); C2-C5 are this repo's counter-based,
 *    thread-parallel generators, bit-reproducible for a seed.
 *
 * Every graph handed out is the reference Graph's CSR layout: offsets
 * uint64[n+1], adjacency uint32[2m], rows strictly increasing, symmetric, no
 * loops, isolated vertices kept.
 */
#ifndef TRIHOST_H
#define TRIHOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t n;
    uint64_t m;        /* undirected edges */
    uint64_t* offsets; /* n+1 */
    uint32_t* adj;     /* 2m */
} th_csr;

const char* th_last_error(void);
int th_threads(void);

/* Generators. Each returns 0 and fills *out (free with th_csr_free). */
int th_gen_gnm(uint32_t n, uint64_t m, uint64_t seed, th_csr* out);
int th_gen_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed, th_csr* out);
/* The raw draws of th_gen_rmat (edge_factor << scale (u, v) pairs as int64,
 * loops and duplicates kept): normalize's input for the same graph. */
int th_gen_rmat_raw(uint32_t scale, uint32_t edge_factor, uint64_t seed, int64_t* out);
int th_gen_chung_lu(uint32_t n, uint64_t draws, double exponent, double wmin, double wmax,
                    uint64_t seed, th_csr* out);
int th_gen_ws(uint32_t n, uint32_t k, double p, uint64_t seed, th_csr* out);
/* CSR from an arbitrary list of pairs (loops dropped, both directions and
 * duplicates merged). */
int th_csr_from_pairs(uint32_t n, uint64_t npairs, const uint32_t* uv, th_csr* out);
void th_csr_free(th_csr* g);
/* 0 if the CSR satisfies the Graph invariants (graph.cpp:98-113). */
int th_csr_check(const th_csr* g);

/* Reference Graph handle (trilist::Graph built by from_dense_edges). */
void* th_graph_new(const th_csr* g);
void th_graph_free(void* graph);
/* The reference's text loader (load_edgelist_file, graph.cpp:164-192: one
 * "a b" label pair per line, lines whose first token starts with '#' skipped,
 * normalize()). The handle
 * works with th_order / th_cost; th_graph_to_csr copies its CSR out,
 * th_graph_labels its labels (int64[n], dense id -> original label). */
void* th_graph_load(const char* path, uint64_t* loops_removed, uint64_t* duplicates_removed);
int th_graph_to_csr(void* graph, th_csr* out);
/* Native multi-threaded reader of the same text format (mmap, one slice of
 * lines per thread; grammar and "line N: ..." errors of load_edgelist,
 * graph.cpp:164-186): *edges = k raw (a, b) int64 label pairs in file order,
 * loops and duplicates kept (normalize's input, graph.cpp:115); free with
 * th_free. Feed them to tl_normalize. 0 ok, -1 error (th_last_error). */
int th_parse_edgelist(const char* path, int64_t** edges, uint64_t* k);
void th_free(void* p);
void th_graph_labels(void* graph, int64_t* out);
/* Ordering by reference method name: identity random degree core split check
 * neigh (trilist_cli.cpp:47-64). rank_out[v] = 0-based position of v. */
int th_order(void* graph, const char* method, uint64_t seed, uint32_t* rank_out,
             double* order_ms);
/* cost_report(g, pi) (cost.cpp:7-25): {c_pp, c_pm, c_mm, sum_deg_sq}. */
int th_cost(void* graph, const uint32_t* rank, uint64_t out[4]);
/* One CSV row in the reference BenchRecord schema (bench.hpp:11-30). */
int th_bench_csv(const char* dataset, const char* algo, const char* ordering, const char* mode,
                 unsigned threads, uint64_t n, uint64_t m, uint64_t c_pp, uint64_t c_pm,
                 uint64_t inner_ops, uint64_t triangles, double load_ms, double order_ms,
                 double list_ms, char* buf, uint64_t cap);
const char* th_bench_csv_header(void);

#ifdef __cplusplus
}
#endif

#endif
