// bulk.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h): multi-threaded checker
// helpers for the full-size (C2-C5) parity tests.
//
//   or_orient_parallel  the same OrientedView as or_orient / the reference
//                       (oriented_view.cpp:7-47): the reference fills every
//                       row in rank order (:32-46); here each row is filled
//                       from the vertex's own adjacency and sorted by rank,
//                       which gives the identical rank-ascending row (ranks
//                       are distinct). Pinned against or_orient in
//                       tests/test_oracle.py.
//   or_sort_triples     CollectingSink::canonical (listing.hpp:57-62): sort
//                       inside each triple, then the triples, lexicographic.
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "oracle.h"

namespace {

template <typename F>
void par_for(std::uint64_t count, int threads, F&& body) {  // body(begin, end)
    const int T = std::max(1, std::min<int>(threads, static_cast<int>(count / 1024 + 1)));
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
        const std::uint64_t b = count * t / T, e = count * (t + 1) / T;
        pool.emplace_back([&body, b, e] { body(b, e); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int or_orient_parallel(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj, const uint32_t* rank,
                       uint64_t* succ_off, uint32_t* succ, uint64_t* pred_off, uint32_t* pred, uint32_t* inverse,
                       int threads) {
    (void)m;
    for (uint32_t p = 0; p < n; ++p) inverse[p] = 0xFFFFFFFFu;
    for (uint32_t v = 0; v < n; ++v) {
        if (rank[v] >= n || inverse[rank[v]] != 0xFFFFFFFFu) return -1;
        inverse[rank[v]] = v;
    }
    succ_off[0] = pred_off[0] = 0;
    par_for(n, threads, [&](std::uint64_t b, std::uint64_t e) {
        for (std::uint64_t u = b; u < e; ++u) {
            std::uint64_t s = 0;
            const uint32_t ru = rank[u];
            for (std::uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) s += ru < rank[adj[k]];
            succ_off[u + 1] = s;
            pred_off[u + 1] = (offsets[u + 1] - offsets[u]) - s;
        }
    });
    for (uint32_t u = 0; u < n; ++u) {
        succ_off[u + 1] += succ_off[u];
        pred_off[u + 1] += pred_off[u];
    }
    par_for(n, threads, [&](std::uint64_t b, std::uint64_t e) {
        auto by_rank = [&](uint32_t x, uint32_t y) { return rank[x] < rank[y]; };
        for (std::uint64_t u = b; u < e; ++u) {
            const uint32_t ru = rank[u];
            std::uint64_t a = succ_off[u], c = pred_off[u];
            for (std::uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
                const uint32_t v = adj[k];
                if (ru < rank[v]) succ[a++] = v;
                else pred[c++] = v;
            }
            std::sort(succ + succ_off[u], succ + succ_off[u + 1], by_rank);
            std::sort(pred + pred_off[u], pred + pred_off[u + 1], by_rank);
        }
    });
    return 0;
}

void or_sort_triples(uint32_t* tri, uint64_t k, int threads) {
    using T3 = std::array<uint32_t, 3>;
    T3* t = reinterpret_cast<T3*>(tri);
    std::vector<uint32_t> tmax(std::max(1, threads) + 1, 0);
    {
        const int T = std::max(1, threads);
        std::vector<std::thread> pool;
        for (int th = 0; th < T; ++th)
            pool.emplace_back([&, th] {
                const std::uint64_t b = k * th / T, e = k * (th + 1) / T;
                uint32_t mx = 0;
                for (std::uint64_t i = b; i < e; ++i) {
                    std::sort(t[i].begin(), t[i].end());
                    mx = std::max(mx, t[i][0]);
                }
                tmax[th] = mx;
            });
        for (auto& p : pool) p.join();
    }
    uint32_t amax = 0;
    for (uint32_t x : tmax) amax = std::max(amax, x);
    // MSD bucket by the first id, then sort each bucket
    constexpr uint32_t B = 1u << 14;
    const uint64_t span = static_cast<uint64_t>(amax) + 1;
    auto bucket = [&](uint32_t a) { return static_cast<uint32_t>(static_cast<uint64_t>(a) * B / span); };
    const int T = std::max(1, threads);
    std::vector<std::vector<uint64_t>> cnt(T, std::vector<uint64_t>(B, 0));
    std::vector<std::thread> pool;
    for (int th = 0; th < T; ++th)
        pool.emplace_back([&, th] {
            const std::uint64_t b = k * th / T, e = k * (th + 1) / T;
            for (std::uint64_t i = b; i < e; ++i) ++cnt[th][bucket(t[i][0])];
        });
    for (auto& p : pool) p.join();
    pool.clear();
    std::vector<uint64_t> start(B + 1, 0);
    uint64_t acc = 0;
    for (uint32_t bk = 0; bk < B; ++bk) {
        start[bk] = acc;
        for (int th = 0; th < T; ++th) {
            const uint64_t c = cnt[th][bk];
            cnt[th][bk] = acc;
            acc += c;
        }
    }
    start[B] = acc;
    std::vector<T3> tmp(k);
    for (int th = 0; th < T; ++th)
        pool.emplace_back([&, th] {
            const std::uint64_t b = k * th / T, e = k * (th + 1) / T;
            for (std::uint64_t i = b; i < e; ++i) tmp[cnt[th][bucket(t[i][0])]++] = t[i];
        });
    for (auto& p : pool) p.join();
    pool.clear();
    std::atomic<uint32_t> next{0};
    for (int th = 0; th < T; ++th)
        pool.emplace_back([&] {
            for (;;) {
                const uint32_t bk = next.fetch_add(1);
                if (bk >= B) break;
                std::sort(tmp.begin() + static_cast<std::ptrdiff_t>(start[bk]),
                          tmp.begin() + static_cast<std::ptrdiff_t>(start[bk + 1]));
            }
        });
    for (auto& p : pool) p.join();
    std::memcpy(tri, tmp.data(), sizeof(T3) * k);
}

}  // extern "C"
