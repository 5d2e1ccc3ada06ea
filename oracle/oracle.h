/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference trilist listing path, used as the parity
 * checker for the GPU engine. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * Nothing on the product path (paper_2203_04774_b200/, libtrigpu.so) links or
 * calls it.
 *
 * Parity pinning: this restatement is checked against the reference itself
 * (oracle/_ref/libtrilist_ref.so, compiled from /root/reference/proj/core
 * sources by oracle/Makefile) and against the golden vectors in tests/golden/
 * that the reference's own tests assert (listing_test.cpp, cost_test.cpp,
 * graph_test.cpp, acceptance_main.cpp). See tests/test_oracle.py.
 */
#ifndef TRILIST_ORACLE_H
#define TRILIST_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_ALGO_APP = 0, OR_ALGO_APM = 1 };

typedef struct {
    uint64_t triangle_count; /* listing.hpp:24 */
    uint64_t inner_ops;      /* listing.hpp:25 */
    uint64_t mark_ops;       /* listing.hpp:26 */
    uint64_t checksum;       /* order-independent triangle checksum */
    double wall_ms;          /* loops only, as listing.hpp:113-116 */
} or_stats;

/* splitmix64 finaliser. */
uint64_t or_mix64(uint64_t z);
/* Vertex hash h(v) = mix64(v) | 1 (odd, so products never vanish). */
uint64_t or_vertex_hash(uint32_t v);
/* Hash of one triangle over DENSE ids: h(a) * h(b) * h(c) mod 2^64 --
 * symmetric, so no sort and no orientation dependence. The checksum is the
 * wrapping sum of this over all triangles. */
uint64_t or_triangle_hash(uint32_t a, uint32_t b, uint32_t c);

/* OrientedView(g, pi) (reference oriented_view.cpp:7-47): dense-id CSR with
 * each successor / predecessor row rank-ascending. Returns 0, or -1 when the
 * ordering is not a bijection of [0, n) (oriented_view.cpp:8-9 raises
 * std::invalid_argument). inverse[p] = vertex at position p. */
int or_orient(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
              const uint32_t* rank, uint64_t* succ_off, uint32_t* succ,
              uint64_t* pred_off, uint32_t* pred, uint32_t* inverse);

/* list_app / list_apm (listing.hpp:69-107, 122-155) over a rank range of
 * seeds [rank_begin, rank_end) with `threads` lanes pulling 1024-rank blocks.
 * Sinks (all optional): vcounts[n] += per-vertex triangle membership;
 * tri[3*k] receives (u, v, w) dense ids with rank(u)<rank(v)<rank(w) up to
 * tri_cap triangles (order unspecified when threads > 1). Returns the number
 * of triangles written to tri. */
uint64_t or_list(int algo, uint32_t n, const uint64_t* succ_off, const uint32_t* succ,
                 const uint64_t* pred_off, const uint32_t* pred, const uint32_t* inverse,
                 const uint32_t* rank, uint32_t rank_begin, uint32_t rank_end, int threads,
                 uint64_t* vcounts, uint32_t* tri, uint64_t tri_cap, or_stats* out);

/* cost_report(view) (reference cost.cpp:27-38): out = {c_pp, c_pm, c_mm, sum_deg_sq}. */
/* or_orient with `threads` lanes (bulk.cpp): identical output; for the
 * full-size parity tests. */
int or_orient_parallel(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                       const uint32_t* rank, uint64_t* succ_off, uint32_t* succ,
                       uint64_t* pred_off, uint32_t* pred, uint32_t* inverse, int threads);
/* CollectingSink::canonical (listing.hpp:57-62) in place over k triples
 * (sort inside each triple, then the triples), `threads` lanes (bulk.cpp). */
void or_sort_triples(uint32_t* tri, uint64_t k, int threads);
/* or_list over a sample of rank ranges [ranges[2i], ranges[2i+1]) in one
 * pulling pass (count + checksum only). */
int or_list_ranges(int algo, uint32_t n, const uint64_t* succ_off, const uint32_t* succ,
                   const uint64_t* pred_off, const uint32_t* pred, const uint32_t* inverse,
                   const uint32_t* ranges, uint64_t nranges, int threads, or_stats* out);
void or_cost(uint32_t n, const uint64_t* succ_off, const uint64_t* pred_off, uint64_t out[4]);

/* brute_triangles(g) (reference oracle.cpp:12-30) without the guard: sorted
 * (u<v<w) dense-id triples; returns the count (writes at most cap). */
uint64_t or_brute(uint32_t n, const uint64_t* offsets, const uint32_t* adj, uint32_t* tri,
                  uint64_t cap);

/* core_decompose (core/src/ordering.cpp:141-188): Batagelj-Zaversnik bucket
 * peeling, restated line for line - rank[v] = removal step of v (the
 * reference's core_order, swap for swap), coreness[v] = degree at removal;
 * returns the degeneracy. Checker for tl_core_decompose's coreness. */
uint32_t or_core_decompose(uint32_t n, const uint64_t* offsets, const uint32_t* adj, uint32_t* rank,
                           uint32_t* coreness);

/* Canonical form (listing.hpp:57-62): sort ids inside each triple, then sort
 * the triple list lexicographically. In place. */
void or_canonicalize(uint32_t* tri, uint64_t k);

#ifdef __cplusplus
}
#endif

#endif
