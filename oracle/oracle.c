/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference trilist listing path:
 *   or_orient  <- core/src/oriented_view.cpp:7-47
 *   or_list    <- core/include/trilist/listing.hpp:69-107 (loops),
 *                 :109-118 (run_single), :122-155 (run_parallel)
 *   or_cost    <- core/src/cost.cpp:27-38
 *   or_brute   <- core/src/oracle.cpp:12-30
 * plus the two sinks the reference does not have (per-vertex counts and the
 * order-independent checksum), defined identically in the
 * GPU engine (paper_2203_04774_b200/csrc/common.cuh).
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t or_vertex_hash(uint32_t v) { return or_mix64(v) | 1u; }

uint64_t or_triangle_hash(uint32_t a, uint32_t b, uint32_t c) {
    return or_vertex_hash(a) * or_vertex_hash(b) * or_vertex_hash(c);
}

/* oriented_view.cpp:7-47: count pass (:18-26), prefix sums (:27-30), then a
 * scatter visiting vertices by ascending rank so rows come out rank-ascending
 * (:34-46). */
int or_orient(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
              const uint32_t* rank, uint64_t* succ_off, uint32_t* succ,
              uint64_t* pred_off, uint32_t* pred, uint32_t* inverse) {
    (void)m;
    for (uint32_t p = 0; p < n; ++p) inverse[p] = 0xFFFFFFFFu;
    for (uint32_t v = 0; v < n; ++v) {
        if (rank[v] >= n || inverse[rank[v]] != 0xFFFFFFFFu) return -1;
        inverse[rank[v]] = v;
    }
    memset(succ_off, 0, sizeof(uint64_t) * ((size_t)n + 1));
    memset(pred_off, 0, sizeof(uint64_t) * ((size_t)n + 1));
    for (uint32_t u = 0; u < n; ++u) {
        const uint32_t ru = rank[u];
        for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
            if (ru < rank[adj[e]]) ++succ_off[u + 1];
            else ++pred_off[u + 1];
        }
    }
    for (uint32_t u = 0; u < n; ++u) {
        succ_off[u + 1] += succ_off[u];
        pred_off[u + 1] += pred_off[u];
    }
    uint64_t* sc = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    uint64_t* pc = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    memcpy(sc, succ_off, sizeof(uint64_t) * n);
    memcpy(pc, pred_off, sizeof(uint64_t) * n);
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t v = inverse[r];
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const uint32_t u = adj[e];
            if (rank[u] < r) succ[sc[u]++] = v; /* v is a successor of u */
            else pred[pc[u]++] = v;             /* v is a predecessor of u */
        }
    }
    free(sc);
    free(pc);
    return 0;
}

/* ---- listing ---------------------------------------------------------- */

typedef struct {
    int algo;
    uint32_t n;
    const uint64_t *succ_off, *pred_off;
    const uint32_t *succ, *pred, *inverse, *rank;
    uint32_t rank_begin, rank_end;
    uint64_t* vcounts;
    uint32_t* tri;
    uint64_t tri_cap;
    volatile uint64_t tri_cursor;
    volatile uint32_t next_block; /* listing.hpp:126 */
    const uint32_t* ranges;       /* optional sample: [ranges[2i], ranges[2i+1]) */
    uint64_t nranges;
    volatile uint64_t next_sub;   /* 1024-rank sub-block cursor over the sample */
    pthread_mutex_t lock;
    or_stats total;
} list_job;

typedef struct {
    uint64_t count, checksum, inner, mark;
} lane_acc;

static inline void emit(list_job* J, lane_acc* acc, uint32_t u, uint32_t v, uint32_t w) {
    acc->count++;
    acc->checksum += or_triangle_hash(u, v, w);
    if (J->vcounts) {
        __atomic_fetch_add(&J->vcounts[u], 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&J->vcounts[v], 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&J->vcounts[w], 1, __ATOMIC_RELAXED);
    }
    if (J->tri) {
        uint64_t k = __atomic_fetch_add(&J->tri_cursor, 1, __ATOMIC_RELAXED);
        if (k < J->tri_cap) {
            J->tri[3 * k] = u;
            J->tri[3 * k + 1] = v;
            J->tri[3 * k + 2] = w;
        }
    }
}

/* listing.hpp:69-86 (A++): seed w by rank, mark N^-(w), scan N^+(u) for
 * u in N^-(w). */
static void run_app_range(list_job* J, uint32_t rb, uint32_t re, uint8_t* table,
                          lane_acc* acc) {
    for (uint32_t r = rb; r < re; ++r) {
        const uint32_t w = J->inverse[r];
        const uint64_t pb = J->pred_off[w], pe = J->pred_off[w + 1];
        if (pb == pe) continue;
        for (uint64_t i = pb; i < pe; ++i) table[J->pred[i]] = 1;
        for (uint64_t i = pb; i < pe; ++i) {
            const uint32_t u = J->pred[i];
            const uint64_t sb = J->succ_off[u], se = J->succ_off[u + 1];
            acc->inner += se - sb;
            for (uint64_t k = sb; k < se; ++k) {
                const uint32_t v = J->succ[k];
                if (table[v]) emit(J, acc, u, v, w);
            }
        }
        for (uint64_t i = pb; i < pe; ++i) table[J->pred[i]] = 0;
        acc->mark += 2 * (pe - pb);
    }
}

/* listing.hpp:91-107 (A+-): seed u by rank, mark N^+(u), scan N^+(v) for
 * v in N^+(u). */
static void run_apm_range(list_job* J, uint32_t rb, uint32_t re, uint8_t* table,
                          lane_acc* acc) {
    for (uint32_t r = rb; r < re; ++r) {
        const uint32_t u = J->inverse[r];
        const uint64_t ub = J->succ_off[u], ue = J->succ_off[u + 1];
        if (ub == ue) continue;
        for (uint64_t i = ub; i < ue; ++i) table[J->succ[i]] = 1;
        for (uint64_t i = ub; i < ue; ++i) {
            const uint32_t v = J->succ[i];
            const uint64_t vb = J->succ_off[v], ve = J->succ_off[v + 1];
            acc->inner += ve - vb;
            for (uint64_t k = vb; k < ve; ++k) {
                const uint32_t w = J->succ[k];
                if (table[w]) emit(J, acc, u, v, w);
            }
        }
        for (uint64_t i = ub; i < ue; ++i) table[J->succ[i]] = 0;
        acc->mark += 2 * (ue - ub);
    }
}

static void* lane_main(void* arg) {
    list_job* J = (list_job*)arg;
    uint8_t* table = (uint8_t*)calloc(J->n ? J->n : 1, 1);
    lane_acc acc = {0, 0, 0, 0};
    while (J->ranges) {  /* sample mode: pull 1024-rank sub-blocks of the ranges */
        const uint64_t k = __atomic_fetch_add(&J->next_sub, 1u, __ATOMIC_RELAXED);
        uint64_t acc_blocks = 0, i = 0;
        uint32_t b = 0, e = 0;
        for (; i < J->nranges; ++i) {
            const uint32_t rb = J->ranges[2 * i];
            const uint32_t re = J->ranges[2 * i + 1] > J->n ? J->n : J->ranges[2 * i + 1];
            const uint64_t nb = re > rb ? (re - rb + 1023u) / 1024u : 0;
            if (k < acc_blocks + nb) {
                b = rb + (uint32_t)(k - acc_blocks) * 1024u;
                e = re - b > 1024u ? b + 1024u : re;
                break;
            }
            acc_blocks += nb;
        }
        if (i == J->nranges) break;
        if (J->algo == OR_ALGO_APP) run_app_range(J, b, e, table, &acc);
        else run_apm_range(J, b, e, table, &acc);
    }
    for (; !J->ranges;) {
        const uint32_t span = J->rank_end - J->rank_begin;
        const uint32_t off = __atomic_fetch_add(&J->next_block, 1024u, __ATOMIC_RELAXED);
        if (off >= span) break;
        const uint32_t b = J->rank_begin + off;
        const uint32_t e = (span - off > 1024u) ? b + 1024u : J->rank_end;
        if (J->algo == OR_ALGO_APP) run_app_range(J, b, e, table, &acc);
        else run_apm_range(J, b, e, table, &acc);
    }
    free(table);
    pthread_mutex_lock(&J->lock);
    J->total.triangle_count += acc.count;
    J->total.checksum += acc.checksum;
    J->total.inner_ops += acc.inner;
    J->total.mark_ops += acc.mark;
    pthread_mutex_unlock(&J->lock);
    return NULL;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

uint64_t or_list(int algo, uint32_t n, const uint64_t* succ_off, const uint32_t* succ,
                 const uint64_t* pred_off, const uint32_t* pred, const uint32_t* inverse,
                 const uint32_t* rank, uint32_t rank_begin, uint32_t rank_end, int threads,
                 uint64_t* vcounts, uint32_t* tri, uint64_t tri_cap, or_stats* out) {
    list_job J;
    memset(&J, 0, sizeof(J));
    J.algo = algo;
    J.n = n;
    J.succ_off = succ_off;
    J.succ = succ;
    J.pred_off = pred_off;
    J.pred = pred;
    J.inverse = inverse;
    J.rank = rank;
    J.rank_begin = rank_begin;
    J.rank_end = rank_end > n ? n : rank_end;
    if (J.rank_begin > J.rank_end) J.rank_begin = J.rank_end;
    J.vcounts = vcounts;
    J.tri = tri;
    J.tri_cap = tri ? tri_cap : 0;
    pthread_mutex_init(&J.lock, NULL);
    if (threads < 1) threads = 1;
    const double t0 = now_ms();
    if (threads == 1) {
        lane_main(&J);
    } else {
        pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
        for (int t = 0; t < threads; ++t) pthread_create(&pool[t], NULL, lane_main, &J);
        for (int t = 0; t < threads; ++t) pthread_join(pool[t], NULL);
        free(pool);
    }
    J.total.wall_ms = now_ms() - t0;
    pthread_mutex_destroy(&J.lock);
    if (out) *out = J.total;
    return J.tri_cursor < J.tri_cap ? J.tri_cursor : J.tri_cap;
}

/* Count + checksum over a sample of rank ranges (bench.py's cpu_baseline:
 * one pulling pass over all sampled blocks, tables allocated once per lane). */
int or_list_ranges(int algo, uint32_t n, const uint64_t* succ_off, const uint32_t* succ,
                   const uint64_t* pred_off, const uint32_t* pred, const uint32_t* inverse,
                   const uint32_t* ranges, uint64_t nranges, int threads, or_stats* out) {
    list_job J;
    memset(&J, 0, sizeof(J));
    J.algo = algo;
    J.n = n;
    J.succ_off = succ_off;
    J.succ = succ;
    J.pred_off = pred_off;
    J.pred = pred;
    J.inverse = inverse;
    J.ranges = ranges;
    J.nranges = nranges;
    pthread_mutex_init(&J.lock, NULL);
    if (threads < 1) threads = 1;
    const double t0 = now_ms();
    pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&pool[t], NULL, lane_main, &J);
    for (int t = 0; t < threads; ++t) pthread_join(pool[t], NULL);
    free(pool);
    J.total.wall_ms = now_ms() - t0;
    pthread_mutex_destroy(&J.lock);
    if (out) *out = J.total;
    return 0;
}

void or_cost(uint32_t n, const uint64_t* succ_off, const uint64_t* pred_off, uint64_t out[4]) {
    uint64_t pp = 0, pm = 0, mm = 0, dd = 0;
    for (uint32_t u = 0; u < n; ++u) {
        const uint64_t o = succ_off[u + 1] - succ_off[u];
        const uint64_t i = pred_off[u + 1] - pred_off[u];
        pp += o * o;
        pm += o * i;
        mm += i * i;
        dd += (o + i) * (o + i);
    }
    out[0] = pp;
    out[1] = pm;
    out[2] = mm;
    out[3] = dd;
}

static int has_edge(const uint64_t* offsets, const uint32_t* adj, uint32_t u, uint32_t v) {
    uint64_t lo = offsets[u], hi = offsets[u + 1];
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (adj[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo < offsets[u + 1] && adj[lo] == v;
}

uint64_t or_brute(uint32_t n, const uint64_t* offsets, const uint32_t* adj, uint32_t* tri,
                  uint64_t cap) {
    uint64_t k = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (uint64_t i = offsets[u]; i < offsets[u + 1]; ++i) {
            const uint32_t v = adj[i];
            if (v <= u) continue;
            for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
                const uint32_t w = adj[j];
                if (w <= v) continue;
                if (has_edge(offsets, adj, u, w)) {
                    if (tri && k < cap) {
                        tri[3 * k] = u;
                        tri[3 * k + 1] = v;
                        tri[3 * k + 2] = w;
                    }
                    ++k;
                }
            }
        }
    /* rows are ascending, so triples come out lexicographically sorted */
    return k;
}

static int cmp_triple(const void* a, const void* b) {
    const uint32_t* x = (const uint32_t*)a;
    const uint32_t* y = (const uint32_t*)b;
    for (int i = 0; i < 3; ++i)
        if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

void or_canonicalize(uint32_t* tri, uint64_t k) {
    for (uint64_t i = 0; i < k; ++i) {
        uint32_t* t = tri + 3 * i;
        uint32_t s;
        if (t[0] > t[1]) { s = t[0]; t[0] = t[1]; t[1] = s; }
        if (t[1] > t[2]) { s = t[1]; t[1] = t[2]; t[2] = s; }
        if (t[0] > t[1]) { s = t[0]; t[0] = t[1]; t[1] = s; }
    }
    qsort(tri, (size_t)k, 3 * sizeof(uint32_t), cmp_triple);
}

/* ---- core_decompose (ordering.cpp:141-188) ---------------------------------
 * vert holds the vertices sorted by current degree, pos their positions, bin
 * the first position of each degree bucket; a decrement of u swaps u with the
 * first vertex of its bucket and moves the bucket boundary past it
 * (ordering.cpp:170-181), so the removal sequence depends on the swap history
 * exactly as in the reference. */
uint32_t or_core_decompose(uint32_t n, const uint64_t* offsets, const uint32_t* adj, uint32_t* rank,
                           uint32_t* coreness) {
    if (n == 0) return 0;
    uint32_t max_deg = 0;
    uint32_t* deg = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* vert = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t v = 0; v < n; ++v) {
        deg[v] = (uint32_t)(offsets[v + 1] - offsets[v]);
        if (deg[v] > max_deg) max_deg = deg[v];
    }
    const size_t nb = (size_t)max_deg + 2;
    uint64_t* bin = (uint64_t*)calloc(nb, sizeof(uint64_t));
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * nb);
    for (uint32_t v = 0; v < n; ++v) ++bin[deg[v] + 1]; /* :150-153 */
    for (size_t d = 1; d < nb; ++d) bin[d] += bin[d - 1]; /* :154 */
    memcpy(cursor, bin, sizeof(uint64_t) * nb);
    for (uint32_t v = 0; v < n; ++v) { /* :156-160 */
        pos[v] = (uint32_t)cursor[deg[v]];
        vert[cursor[deg[v]]++] = v;
    }
    uint32_t degeneracy = 0;
    for (uint32_t step = 0; step < n; ++step) { /* :166-184 */
        const uint32_t v = vert[step];
        if (rank) rank[v] = step;
        if (coreness) coreness[v] = deg[v];
        if (deg[v] > degeneracy) degeneracy = deg[v];
        for (uint64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const uint32_t u = adj[e];
            if (deg[u] <= deg[v]) continue;
            const uint32_t du = deg[u];
            const uint32_t first_pos = (uint32_t)bin[du];
            const uint32_t first_vert = vert[first_pos];
            if (u != first_vert) {
                const uint32_t pu = pos[u];
                vert[pu] = first_vert;
                vert[first_pos] = u;
                pos[u] = first_pos;
                pos[first_vert] = pu;
            }
            ++bin[du];
            --deg[u];
        }
        ++bin[deg[v]];
    }
    free(deg);
    free(vert);
    free(pos);
    free(bin);
    free(cursor);
    return degeneracy;
}
