// shim_test.cpp -- the reference's own listing checks, re-run through the
// trigpu C++ shim (include/trigpu.hpp) on the GPU. Built by `make
// build/shim_test` against the reference core sources (compiled in place) and
// libtrigpu.so; run by tests/test_gpu_parity.py::test_cpp_shim (GPU box).
//
// Mirrors: listing_test.cpp:14-118, graph_test.cpp:145-181, acceptance
// criteria 1-3 (acceptance_main.cpp:116-149) and 12 (:447-510). Ground truth is
// the reference itself (brute_triangles, cost_report, trilist::OrientedView,
// trilist::list_apm) linked into this binary.

#include <algorithm>
#include <array>
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "trigpu.hpp"
#include "trilist/cost.hpp"
#include "trilist/neigh.hpp"
#include "trilist/oracle.hpp"
#include "trilist/oriented_view.hpp"

using namespace trilist;

namespace {

int g_fail = 0;
std::uint64_t g_checks = 0;

void expect(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        if (g_fail < 20) std::printf("  FAIL: %s\n", what.c_str());
        ++g_fail;
    }
}

Graph random_small_graph(std::uint64_t seed, VertexId max_n, std::uint64_t max_m) {
    std::mt19937_64 rng(seed);
    const VertexId n = static_cast<VertexId>(1 + bounded_rand(rng, max_n));
    const std::uint64_t pairs = static_cast<std::uint64_t>(n) * (n - 1) / 2;
    const std::uint64_t m = bounded_rand(rng, std::min(max_m, pairs) + 1);
    return gen_gnm(n, m, rng());
}

std::vector<std::pair<std::string, Ordering>> all_orderings(const Graph& g, std::uint64_t seed) {
    return {{"identity", identity_order(g)}, {"random", random_order(g, seed)},
            {"degree", degree_order(g)},     {"core", core_order(g)},
            {"split", split_order(g)},       {"check", check_order(g)},
            {"neigh", neigh_order(g)}};
}

void section(const char* name, int before) {
    std::printf("%s [%s]\n", name, g_fail == before ? "PASS" : "FAIL");
}

}  // namespace

int main() {
    trigpu::Context& ctx = trigpu::default_context();
    (void)ctx;
    int f0;

    f0 = g_fail;  // listing_test.cpp:14-40
    {
        const Graph g = gen_gnm(3, 3, 0);
        const Ordering pi = identity_order(g);
        CountingSink count;
        const ListingStats app = trigpu::list_app(g, pi, count);
        expect(app.triangle_count == 1 && app.inner_ops == 5, "K3 app");
        const ListingStats apm = trigpu::list_apm(g, pi, count);
        expect(apm.triangle_count == 1 && apm.inner_ops == 1, "K3 apm");
        const Graph k4 = gen_gnm(4, 6, 0);
        expect(trigpu::list_app(k4, identity_order(k4), count).triangle_count == 4, "K4 app");
        expect(trigpu::list_apm(k4, identity_order(k4), count).triangle_count == 4, "K4 apm");
        const Graph e = gen_gnm(10, 0, 0);
        const ListingStats s = trigpu::list_apm(e, identity_order(e), count);
        expect(s.triangle_count == 0 && s.inner_ops == 0 && s.mark_ops == 0, "edgeless");
    }
    section("listing tiny graphs (listing_test.cpp:14-40)", f0);

    f0 = g_fail;  // listing_test.cpp:42-62
    {
        const Graph g = gen_gnm(25, 90, 3);
        const Ordering pi = random_order(g, 17);
        CollectingSink sink;
        trigpu::list_apm(g, pi, sink);
        std::set<std::array<VertexId, 3>> seen;
        for (const auto& [u, v, w] : sink.triangles) {
            expect(pi.rank_of(u) < pi.rank_of(v) && pi.rank_of(v) < pi.rank_of(w), "rank order");
            expect(g.has_edge(u, v) && g.has_edge(v, w) && g.has_edge(u, w), "edges exist");
            auto key = std::array{u, v, w};
            std::sort(key.begin(), key.end());
            expect(seen.insert(key).second, "duplicate-free");
        }
        CollectingSink ref_sink;
        trilist::list_apm(g, pi, ref_sink);
        expect(sink.canonical() == ref_sink.canonical(), "same set as reference");
    }
    section("emission respects ranks, duplicate-free (listing_test.cpp:42-62)", f0);

    f0 = g_fail;  // listing_test.cpp:64-78
    {
        const Graph g = gen_gnm(60, 400, 11);
        const auto expected = brute_triangles(g);
        for (const Ordering& pi : {identity_order(g), random_order(g, 1), degree_order(g), core_order(g),
                                   split_order(g), check_order(g)}) {
            CollectingSink a, b;
            trigpu::list_app(g, pi, a);
            trigpu::list_apm(g, pi, b);
            expect(a.canonical() == expected, "app vs brute");
            expect(b.canonical() == expected, "apm vs brute");
        }
    }
    section("both algorithms match brute force (listing_test.cpp:64-78)", f0);

    f0 = g_fail;  // listing_test.cpp:80-93
    for (std::uint64_t seed = 0; seed < 20; ++seed) {
        const Graph g = random_small_graph(seed, 40, 200);
        const Ordering pi = random_order(g, seed + 7);
        const CostReport report = cost_report(g, pi);
        CountingSink count;
        const ListingStats app = trigpu::list_app(g, pi, count);
        expect(app.inner_ops == report.c_pp && app.mark_ops == 2 * g.edge_count(), "app accounting");
        const ListingStats apm = trigpu::list_apm(g, pi, count);
        expect(apm.inner_ops == report.c_pm && apm.mark_ops == 2 * g.edge_count(), "apm accounting");
    }
    section("inner_ops == cost, mark_ops == 2m (listing_test.cpp:80-93)", f0);

    f0 = g_fail;  // listing_test.cpp:95-118
    {
        const Graph g = gen_gnm(300, 2500, 5);
        const Ordering pi = degree_order(g);
        const trilist::OrientedView rview(g, pi);
        CountingSink single;
        const ListingStats expected = trilist::list_apm(rview, single);
        CollectingSink reference;
        trilist::list_app(rview, reference);
        const trigpu::OrientedView view(g, pi);
        for (unsigned threads : {2u, 4u}) {
            CountingSink pc;
            const ListingStats st = trigpu::list_apm_parallel(view, pc, threads);
            expect(st.triangle_count == expected.triangle_count && st.inner_ops == expected.inner_ops &&
                       st.mark_ops == expected.mark_ops && pc.count == single.count,
                   "parallel totals");
            CollectingSink collected;
            trigpu::list_app_parallel(view, collected, threads);
            expect(collected.canonical() == reference.canonical(), "parallel canonical");
        }
    }
    section("parallel contract (listing_test.cpp:95-118)", f0);

    f0 = g_fail;  // graph_test.cpp:145-181 + exact rows vs trilist::OrientedView
    {
        const Graph g = gen_gnm(50, 200, 123);
        const Ordering pi = random_order(g, 5);
        const trigpu::OrientedView view(g, pi);
        const trilist::OrientedView rview(g, pi);
        std::uint64_t out_sum = 0, in_sum = 0;
        for (VertexId u = 0; u < 50; ++u) {
            out_sum += view.out_degree(u);
            in_sum += view.in_degree(u);
            expect(view.out_degree(u) + view.in_degree(u) == g.degree(u), "d+ + d- = d");
            const auto s = view.successors(u), rs = rview.successors(u);
            const auto p = view.predecessors(u), rp = rview.predecessors(u);
            expect(std::vector<VertexId>(s.begin(), s.end()) == std::vector<VertexId>(rs.begin(), rs.end()),
                   "successor row");
            expect(std::vector<VertexId>(p.begin(), p.end()) == std::vector<VertexId>(rp.begin(), rp.end()),
                   "predecessor row");
        }
        expect(out_sum == g.edge_count() && in_sum == g.edge_count(), "sum d+ = sum d- = m");
        bool threw = false;
        try {
            const Graph h = gen_gnm(5, 4, 1);
            trigpu::OrientedView bad(h, Ordering::identity(4));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "size mismatch throws std::invalid_argument");
    }
    section("orient partitions each neighborhood (graph_test.cpp:145-181)", f0);

    f0 = g_fail;  // device orderings == the reference's (ordering.cpp:66-109)
    {
        for (std::uint64_t seed = 0; seed < 40; ++seed) {
            const Graph g = random_small_graph(seed, 60, 400);
            expect(trigpu::degree_order(g).ranks().size() == g.vertex_count(), "degree order size");
            const auto a = trigpu::degree_order(g), b = degree_order(g);
            const auto c = trigpu::split_order(g), d = split_order(g);
            expect(std::equal(a.ranks().begin(), a.ranks().end(), b.ranks().begin()), "device degree order");
            expect(std::equal(c.ranks().begin(), c.ranks().end(), d.ranks().begin()), "device split order");
        }
        const Graph g = gen_gnm(100000, 1000000, 4242);
        const auto a = trigpu::degree_order(g), b = degree_order(g);
        expect(std::equal(a.ranks().begin(), a.ranks().end(), b.ranks().begin()), "device degree order, C1");
    }
    section("device degree / split orderings (ordering.cpp:66-109)", f0);

    f0 = g_fail;  // device k-core decomposition vs core_decompose (ordering.cpp:141-188)
    {
        auto check = [&](const Graph& g, const std::string& tag) {
            const CoreDecomposition a = trigpu::core_decompose(g), b = core_decompose(g);
            expect(a.coreness == b.coreness, "device coreness " + tag);
            expect(a.degeneracy == b.degeneracy, "device degeneracy " + tag);
            const OrientedView v(g, a.order);  // the reference's own view under the device order
            VertexId max_out = 0;
            bool ok = true;
            for (VertexId u = 0; u < g.vertex_count(); ++u) {
                max_out = std::max(max_out, v.out_degree(u));
                ok = ok && v.out_degree(u) <= b.coreness[u];
            }
            expect(ok, "d+ <= coreness under the device core order " + tag);
            expect(max_out <= b.degeneracy, "max d+ <= degeneracy " + tag);
        };
        for (std::uint64_t seed = 0; seed < 40; ++seed)
            check(random_small_graph(seed, 60, 400), "seed " + std::to_string(seed));
        check(gen_gnm(100000, 1000000, 4242), "C1");
    }
    section("device core decomposition (ordering.cpp:141-188)", f0);

    f0 = g_fail;  // acceptance criteria 1-3
    {
        const int c0 = g_fail;
        for (std::uint64_t seed = 0; seed < 200; ++seed) {
            const Graph g = random_small_graph(seed, 60, 400);
            const auto expected = brute_triangles(g);
            for (const auto& [name, pi] : all_orderings(g, seed)) {
                const CostReport report = cost_report(g, pi);
                const trigpu::OrientedView view(g, pi);
                CollectingSink a, b;
                const ListingStats app = trigpu::list_app(view, a);
                const ListingStats apm = trigpu::list_apm(view, b);
                const std::string tag = name + " seed " + std::to_string(seed);
                expect(a.canonical() == expected, "crit1 app " + tag);
                expect(b.canonical() == expected, "crit1 apm " + tag);
                expect(app.inner_ops == report.c_pp, "crit2 app " + tag);
                expect(apm.inner_ops == report.c_pm, "crit2 apm " + tag);
                expect(report.c_pp + 2 * report.c_pm + report.c_mm == report.sum_deg_sq, "crit3 " + tag);
            }
        }
        std::printf("  acceptance sweep: 200 graphs x 7 orderings x 2 algorithms, %d failures\n", g_fail - c0);
    }
    section("acceptance criteria 1-3 (acceptance_main.cpp:116-149)", f0);

    f0 = g_fail;  // acceptance criterion 12
    {
        const Graph g = gen_gnm(100000, 1000000, 4242);
        std::vector<std::pair<std::uint64_t, std::uint64_t>> rows;
        for (const auto& [name, pi] : all_orderings(g, 4242)) {
            const std::uint64_t c_pm = cost_report(g, pi).c_pm;
            const trigpu::OrientedView view(g, pi);
            trigpu::ChecksumSink sink;
            const ListingStats st = trigpu::list_apm(view, sink);
            expect(st.inner_ops == c_pm, "crit12 inner_ops == c_pm " + name);
            expect(st.triangle_count == 1338, "C1 triangle count " + name);
            rows.emplace_back(c_pm, st.inner_ops);
        }
        std::vector<std::size_t> a(rows.size()), b(rows.size());
        for (std::size_t i = 0; i < rows.size(); ++i) a[i] = b[i] = i;
        std::stable_sort(a.begin(), a.end(), [&](auto x, auto y) { return rows[x].first < rows[y].first; });
        std::stable_sort(b.begin(), b.end(), [&](auto x, auto y) { return rows[x].second < rows[y].second; });
        expect(a == b, "crit12 ranking by cost == ranking by work");
    }
    section("acceptance criterion 12 on C1 (acceptance_main.cpp:447-510)", f0);

    std::printf("%llu checks, %d failed\n", static_cast<unsigned long long>(g_checks), g_fail);
    return g_fail ? 1 : 0;
}
