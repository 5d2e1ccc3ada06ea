// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the UNMODIFIED reference trilist core (compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libtrilist_ref.so). It is the checker the oracle restatement and
// the GPU engine are pinned against, and the "reference" CPU baseline that
// bench.py times. It calls the reference's own types and listing templates:
//   Graph::from_dense_edges  graph.cpp:13-56        gen_gnm      graph.cpp:210-243
//   orderings                ordering.cpp:50-188     neigh_order  neigh.cpp:200-208
//   cost_report              cost.cpp:7-25           OrientedView oriented_view.cpp:7-47
//   list_app / list_apm      listing.hpp:162-199     detail::run_*_range listing.hpp:69-107
//   brute_triangles          oracle.cpp:12-30
// The two sinks the reference lacks (checksum, per-vertex counts) are written
// against its sink concept (listing.hpp:36-38): default-constructible,
// operator()(u, v, w), merge(Sink&&).

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "trilist/cost.hpp"
#include "trilist/graph.hpp"
#include "trilist/listing.hpp"
#include "trilist/neigh.hpp"
#include "trilist/oracle.hpp"
#include "trilist/ordering.hpp"
#include "trilist/oriented_view.hpp"

using namespace trilist;

namespace {

thread_local std::string g_error;

std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// h(a) * h(b) * h(c) mod 2^64, h(v) = mix64(v) | 1 (symmetric: no sort)
std::uint64_t vertex_hash(VertexId v) { return mix64(v) | 1u; }

std::uint64_t triangle_hash(VertexId a, VertexId b, VertexId c) {
    return vertex_hash(a) * vertex_hash(b) * vertex_hash(c);
}

// Which outputs HarnessSink records; set once per ref_list call (the harness
// is not re-entrant, like the CLI it stands in for).
struct SinkConfig {
    bool vcounts = false;
    bool collect = false;
    VertexId n = 0;
};
SinkConfig g_cfg;

// Count + checksum + optional per-vertex counts + optional collection.
struct HarnessSink {
    std::uint64_t count = 0;
    std::uint64_t checksum = 0;
    std::vector<std::uint64_t> vcounts;
    std::vector<std::array<VertexId, 3>> triangles;

    void operator()(VertexId u, VertexId v, VertexId w) {
        ++count;
        checksum += triangle_hash(u, v, w);
        if (g_cfg.vcounts) {
            if (vcounts.empty()) vcounts.assign(g_cfg.n, 0);
            ++vcounts[u];
            ++vcounts[v];
            ++vcounts[w];
        }
        if (g_cfg.collect) triangles.push_back({u, v, w});
    }
    void merge(HarnessSink&& o) {
        count += o.count;
        checksum += o.checksum;
        if (!o.vcounts.empty()) {
            if (vcounts.empty()) vcounts.assign(g_cfg.n, 0);
            for (std::size_t i = 0; i < o.vcounts.size(); ++i) vcounts[i] += o.vcounts[i];
        }
        triangles.insert(triangles.end(), o.triangles.begin(), o.triangles.end());
    }
};

// run_parallel (listing.hpp:122-155) restricted to a rank sub-range: the same
// 1024-rank block pulling and per-lane table/sink/stats, so a bounded sample
// of seeds runs the reference's own inner loops unchanged.
template <typename Runner>
ListingStats ranged_parallel(const OrientedView& view, Runner runner, HarnessSink& sink,
                             unsigned threads, VertexId rb, VertexId re) {
    const VertexId n = view.vertex_count();
    constexpr VertexId kBlock = 1024;
    std::atomic<std::uint64_t> next{rb};
    std::mutex mu;
    ListingStats total;
    const auto t0 = std::chrono::steady_clock::now();
    auto worker = [&] {
        ListingStats local;
        HarnessSink local_sink;
        std::vector<std::uint8_t> table(n, 0);
        for (;;) {
            const std::uint64_t b = next.fetch_add(kBlock);
            if (b >= re) break;
            const VertexId e = static_cast<VertexId>(std::min<std::uint64_t>(re, b + kBlock));
            runner(view, static_cast<VertexId>(b), e, table, local_sink, local);
        }
        std::lock_guard<std::mutex> lock(mu);
        total.merge(local);
        sink.merge(std::move(local_sink));
    };
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < std::max(1u, threads); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    total.wall_ms = std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now() - t0).count();
    return total;
}

// The same pulling over an explicit list of rank sub-blocks (each <= 1024
// ranks): a bounded sample of the workload listed in ONE run_parallel-style
// call, so the per-call setup (a zeroed table(n) per lane, listing.hpp:134)
// is paid once per sample, as it is once per full listing.
template <typename Runner>
ListingStats blocks_parallel(const OrientedView& view, Runner runner, HarnessSink& sink, unsigned threads,
                             const std::vector<std::pair<VertexId, VertexId>>& blocks) {
    const VertexId n = view.vertex_count();
    std::atomic<std::size_t> next{0};
    std::mutex mu;
    ListingStats total;
    const auto t0 = std::chrono::steady_clock::now();
    auto worker = [&] {
        ListingStats local;
        HarnessSink local_sink;
        std::vector<std::uint8_t> table(n, 0);
        for (;;) {
            const std::size_t i = next.fetch_add(1);
            if (i >= blocks.size()) break;
            runner(view, blocks[i].first, blocks[i].second, table, local_sink, local);
        }
        std::lock_guard<std::mutex> lock(mu);
        total.merge(local);
        sink.merge(std::move(local_sink));
    };
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < std::max(1u, threads); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    total.wall_ms = std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now() - t0).count();
    return total;
}

}  // namespace

extern "C" {

struct ref_stats {
    std::uint64_t triangle_count, inner_ops, mark_ops, checksum;
    double wall_ms;
};

const char* ref_last_error() { return g_error.c_str(); }

void* ref_graph_from_csr(std::uint32_t n, const std::uint64_t* off, const std::uint32_t* adj) {
    try {
        std::vector<std::pair<VertexId, VertexId>> edges;
        edges.reserve(off[n] / 2);
        for (VertexId u = 0; u < n; ++u)
            for (std::uint64_t e = off[u]; e < off[u + 1]; ++e)
                if (u < adj[e]) edges.emplace_back(u, adj[e]);
        return new Graph(Graph::from_dense_edges(n, std::move(edges)));
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

void* ref_graph_from_edges(std::uint32_t n, std::uint64_t m, const std::uint32_t* uv) {
    try {
        std::vector<std::pair<VertexId, VertexId>> edges(m);
        for (std::uint64_t i = 0; i < m; ++i) edges[i] = {uv[2 * i], uv[2 * i + 1]};
        return new Graph(Graph::from_dense_edges(n, std::move(edges)));
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

// The reference's normalize (graph.cpp:115-151) on raw labeled pairs; labels
// of the result via ref_graph_labels.
void* ref_graph_normalize(std::uint64_t k, const std::int64_t* ab, std::uint64_t* loops, std::uint64_t* dups) {
    try {
        std::vector<LabeledEdge> raw(k);
        for (std::uint64_t i = 0; i < k; ++i) raw[i] = {ab[2 * i], ab[2 * i + 1]};
        NormalizeStats st;
        auto* g = new Graph(normalize(raw, &st));
        *loops = st.loops_removed;
        *dups = st.duplicates_removed;
        return g;
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

void ref_graph_labels(void* gp, std::int64_t* out) {
    const Graph& g = *static_cast<Graph*>(gp);
    for (VertexId u = 0; u < g.vertex_count(); ++u) out[u] = g.label_of(u);
}

void* ref_graph_gnm(std::uint32_t n, std::uint64_t m, std::uint64_t seed) {
    try {
        return new Graph(gen_gnm(n, m, seed));
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

// random_small_graph (acceptance_main.cpp:89-95) / testsupport::random_graph
// (test_support.hpp:26-32): n in [1, max_n], m uniform up to min(max_m, pairs),
// then gen_gnm with the next draw as its seed.
void* ref_graph_random_small(std::uint64_t seed, std::uint32_t max_n, std::uint64_t max_m) {
    try {
        std::mt19937_64 rng(seed);
        const VertexId n = static_cast<VertexId>(1 + bounded_rand(rng, max_n));
        const std::uint64_t pairs = static_cast<std::uint64_t>(n) * (n - 1) / 2;
        const std::uint64_t m = bounded_rand(rng, std::min(max_m, pairs) + 1);
        return new Graph(gen_gnm(n, m, rng()));
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }
std::uint32_t ref_graph_n(void* g) { return static_cast<Graph*>(g)->vertex_count(); }
std::uint64_t ref_graph_m(void* g) { return static_cast<Graph*>(g)->edge_count(); }

void ref_graph_csr(void* gp, std::uint64_t* off, std::uint32_t* adj) {
    const Graph& g = *static_cast<Graph*>(gp);
    std::uint64_t pos = 0;
    off[0] = 0;
    for (VertexId u = 0; u < g.vertex_count(); ++u) {
        for (VertexId v : g.neighbors(u)) adj[pos++] = v;
        off[u + 1] = pos;
    }
}

int ref_order(void* gp, const char* method, std::uint64_t seed, std::uint32_t* rank_out) {
    try {
        const Graph& g = *static_cast<Graph*>(gp);
        const std::string m = method;
        Ordering pi;
        if (m == "identity") pi = identity_order(g);
        else if (m == "random") pi = random_order(g, seed);
        else if (m == "degree") pi = degree_order(g);
        else if (m == "core") pi = core_order(g);
        else if (m == "split") pi = split_order(g);
        else if (m == "check") pi = check_order(g);
        else if (m == "neigh") pi = neigh_order(g);
        else {
            g_error = "unknown ordering method: " + m;
            return -1;
        }
        std::memcpy(rank_out, pi.ranks().data(), sizeof(VertexId) * pi.size());
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// core_decompose (ordering.cpp:141-188): ranks of the removal order, coreness; returns the
// degeneracy (-1 on error).
std::int64_t ref_core_decompose(void* gp, std::uint32_t* rank_out, std::uint32_t* coreness_out) {
    try {
        const Graph& g = *static_cast<Graph*>(gp);
        const CoreDecomposition cd = core_decompose(g);
        if (rank_out) std::memcpy(rank_out, cd.order.ranks().data(), sizeof(VertexId) * cd.order.size());
        if (coreness_out) std::memcpy(coreness_out, cd.coreness.data(), sizeof(VertexId) * cd.coreness.size());
        return cd.degeneracy;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

int ref_cost(void* gp, const std::uint32_t* rank, std::uint64_t out[4]) {
    try {
        const Graph& g = *static_cast<Graph*>(gp);
        const Ordering pi = Ordering::from_ranks(
            std::vector<VertexId>(rank, rank + g.vertex_count()));
        const CostReport r = cost_report(g, pi);
        out[0] = r.c_pp;
        out[1] = r.c_pm;
        out[2] = r.c_mm;
        out[3] = r.sum_deg_sq;
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// OrientedView from a rank array; rank length must equal n (pass n_rank to
// exercise the size-mismatch error, oriented_view.cpp:8-9).
void* ref_view(void* gp, const std::uint32_t* rank, std::uint32_t n_rank) {
    try {
        const Graph& g = *static_cast<Graph*>(gp);
        const Ordering pi =
            Ordering::from_ranks(std::vector<VertexId>(rank, rank + n_rank));
        return new OrientedView(g, pi);
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

void ref_view_free(void* v) { delete static_cast<OrientedView*>(v); }

void ref_view_csr(void* vp, std::uint64_t* so, std::uint32_t* s, std::uint64_t* po,
                  std::uint32_t* p) {
    const OrientedView& view = *static_cast<OrientedView*>(vp);
    std::uint64_t a = 0, b = 0;
    so[0] = po[0] = 0;
    for (VertexId u = 0; u < view.vertex_count(); ++u) {
        for (VertexId x : view.successors(u)) s[a++] = x;
        for (VertexId x : view.predecessors(u)) p[b++] = x;
        so[u + 1] = a;
        po[u + 1] = b;
    }
}

// Timed OrientedView construction (BM_Orient, listing_bench.cpp:61-68).
double ref_orient_ms(void* gp, const std::uint32_t* rank) {
    const Graph& g = *static_cast<Graph*>(gp);
    const Ordering pi =
        Ordering::from_ranks(std::vector<VertexId>(rank, rank + g.vertex_count()));
    const auto t0 = std::chrono::steady_clock::now();
    OrientedView view(g, pi);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    volatile auto sink = view.edge_count();
    (void)sink;
    return ms;
}

// algo 0 = app, 1 = apm. threads <= 1 and the full range go through the
// public single-threaded entry points (list_app / list_apm, whose emission
// order is deterministic); otherwise the parallel path.
int ref_list(void* vp, int algo, int threads, std::uint32_t rank_begin, std::uint32_t rank_end,
             std::uint64_t* vcounts, std::uint32_t* tri, std::uint64_t cap, std::uint64_t* k,
             ref_stats* out) {
    try {
        const OrientedView& view = *static_cast<OrientedView*>(vp);
        const VertexId n = view.vertex_count();
        g_cfg.vcounts = vcounts != nullptr;
        g_cfg.collect = tri != nullptr;
        g_cfg.n = n;
        HarnessSink sink;
        ListingStats st;
        const bool full = rank_begin == 0 && rank_end >= n;
        if (full && threads <= 1) {
            st = algo == 0 ? list_app(view, sink) : list_apm(view, sink);
        } else if (full) {
            st = algo == 0 ? list_app_parallel(view, sink, static_cast<unsigned>(threads))
                           : list_apm_parallel(view, sink, static_cast<unsigned>(threads));
        } else {
            const VertexId re = std::min<VertexId>(rank_end, n);
            if (algo == 0)
                st = ranged_parallel(
                    view, [](auto&&... a) { detail::run_app_range(std::forward<decltype(a)>(a)...); },
                    sink, static_cast<unsigned>(threads), rank_begin, re);
            else
                st = ranged_parallel(
                    view, [](auto&&... a) { detail::run_apm_range(std::forward<decltype(a)>(a)...); },
                    sink, static_cast<unsigned>(threads), rank_begin, re);
        }
        if (sink.count != st.triangle_count) {
            g_error = "sink count disagrees with ListingStats";
            return -1;
        }
        out->triangle_count = st.triangle_count;
        out->inner_ops = st.inner_ops;
        out->mark_ops = st.mark_ops;
        out->checksum = sink.checksum;
        out->wall_ms = st.wall_ms;
        if (vcounts && !sink.vcounts.empty())
            std::memcpy(vcounts, sink.vcounts.data(), sizeof(std::uint64_t) * n);
        else if (vcounts)
            std::memset(vcounts, 0, sizeof(std::uint64_t) * n);
        if (tri) {
            const std::uint64_t kk = std::min<std::uint64_t>(cap, sink.triangles.size());
            for (std::uint64_t i = 0; i < kk; ++i) {
                tri[3 * i] = sink.triangles[i][0];
                tri[3 * i + 1] = sink.triangles[i][1];
                tri[3 * i + 2] = sink.triangles[i][2];
            }
            *k = sink.triangles.size();
        }
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// Count + checksum over a sample of rank ranges ([ranges[2i], ranges[2i+1])),
// cut into 1024-rank blocks and pulled by `threads` lanes in one call.
int ref_list_ranges(void* vp, int algo, int threads, const std::uint32_t* ranges, std::uint64_t nranges,
                    ref_stats* out) {
    try {
        const OrientedView& view = *static_cast<OrientedView*>(vp);
        const VertexId n = view.vertex_count();
        g_cfg.vcounts = false;
        g_cfg.collect = false;
        g_cfg.n = n;
        std::vector<std::pair<VertexId, VertexId>> blocks;
        for (std::uint64_t i = 0; i < nranges; ++i) {
            const VertexId rb = ranges[2 * i], re = std::min<VertexId>(ranges[2 * i + 1], n);
            for (std::uint64_t b = rb; b < re; b += 1024)
                blocks.emplace_back(static_cast<VertexId>(b), static_cast<VertexId>(std::min<std::uint64_t>(re, b + 1024)));
        }
        HarnessSink sink;
        ListingStats st;
        if (algo == 0)
            st = blocks_parallel(
                view, [](auto&&... a) { detail::run_app_range(std::forward<decltype(a)>(a)...); }, sink,
                static_cast<unsigned>(threads), blocks);
        else
            st = blocks_parallel(
                view, [](auto&&... a) { detail::run_apm_range(std::forward<decltype(a)>(a)...); }, sink,
                static_cast<unsigned>(threads), blocks);
        out->triangle_count = st.triangle_count;
        out->inner_ops = st.inner_ops;
        out->mark_ops = st.mark_ops;
        out->checksum = sink.checksum;
        out->wall_ms = st.wall_ms;
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// brute_triangles (oracle.cpp:12-30) with an explicit guard.
std::int64_t ref_brute(void* gp, std::uint32_t guard, std::uint32_t* tri, std::uint64_t cap) {
    try {
        const auto t = brute_triangles(*static_cast<Graph*>(gp), guard);
        for (std::uint64_t i = 0; i < std::min<std::uint64_t>(cap, t.size()); ++i) {
            tri[3 * i] = t[i][0];
            tri[3 * i + 1] = t[i][1];
            tri[3 * i + 2] = t[i][2];
        }
        return static_cast<std::int64_t>(t.size());
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

}  // extern "C"
