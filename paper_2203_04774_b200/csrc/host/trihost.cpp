// trihost.cpp -- see trihost.h.
//
// Generators are counter-based: draw(stream, i) = splitmix64 finaliser of a
// per-(seed, stream) base plus i * golden-gamma, so any thread can produce any
// draw and the output is independent of the thread count. Quadrant, rewiring
// and endpoint decisions use integer thresholds on the draws.
// Dedup is a thread-parallel LSD radix sort of directed (row << 32 | col) keys.

#include "trihost.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "trilist/bench.hpp"
#include "trilist/cost.hpp"
#include "trilist/graph.hpp"
#include "trilist/neigh.hpp"
#include "trilist/ordering.hpp"

namespace {

thread_local std::string g_err;

inline std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

struct Stream {
    std::uint64_t base;
    Stream(std::uint64_t seed, std::uint64_t stream) : base(mix64(seed + kGamma * (stream + 1))) {}
    std::uint64_t operator()(std::uint64_t i) const { return mix64(base + (i + 1) * kGamma); }
};

// Uniform in [0, n) from 32 random bits (multiply-high); deterministic.
inline std::uint32_t below(std::uint32_t r32, std::uint32_t n) {
    return static_cast<std::uint32_t>((static_cast<std::uint64_t>(r32) * n) >> 32);
}

unsigned nthreads() {
    if (const char* e = std::getenv("TRIHOST_THREADS")) {
        const int t = std::atoi(e);
        if (t > 0) return static_cast<unsigned>(t);
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? h : 1;
}

template <typename F>
void parallel_for(std::uint64_t count, F&& body) {  // body(tid, begin, end)
    const unsigned T = static_cast<unsigned>(std::min<std::uint64_t>(nthreads(), std::max<std::uint64_t>(1, count / 4096 + 1)));
    if (T <= 1) {
        body(0u, std::uint64_t{0}, count);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) {
        const std::uint64_t b = count * t / T, e = count * (t + 1) / T;
        pool.emplace_back([&body, t, b, e] { body(t, b, e); });
    }
    for (auto& th : pool) th.join();
}

// Stable LSD radix sort over `bits` low bits of the row half and col half.
void radix_sort_keys(std::vector<std::uint64_t>& keys, unsigned row_bits, unsigned col_bits) {
    constexpr unsigned D = 11;
    std::vector<std::pair<unsigned, unsigned>> passes;  // (shift, width)
    for (unsigned s = 0; s < col_bits; s += D) passes.push_back({s, std::min(D, col_bits - s)});
    for (unsigned s = 0; s < row_bits; s += D) passes.push_back({32 + s, std::min(D, row_bits - s)});
    std::vector<std::uint64_t> tmp(keys.size());
    const std::uint64_t N = keys.size();
    const unsigned T = static_cast<unsigned>(std::min<std::uint64_t>(nthreads(), std::max<std::uint64_t>(1, N / 65536 + 1)));
    std::vector<std::uint64_t> hist(static_cast<std::size_t>(T) << D);
    for (auto [shift, width] : passes) {
        const std::uint64_t mask = (1ULL << width) - 1;
        const std::size_t B = std::size_t{1} << width;
        std::fill(hist.begin(), hist.end(), 0);
        auto run = [&](auto&& f) {
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < T; ++t) pool.emplace_back([&, t] { f(t, N * t / T, N * (t + 1) / T); });
            for (auto& th : pool) th.join();
        };
        run([&](unsigned t, std::uint64_t b, std::uint64_t e) {
            std::uint64_t* h = hist.data() + (static_cast<std::size_t>(t) << D);
            for (std::uint64_t i = b; i < e; ++i) ++h[(keys[i] >> shift) & mask];
        });
        std::uint64_t acc = 0;
        for (std::size_t d = 0; d < B; ++d)
            for (unsigned t = 0; t < T; ++t) {
                std::uint64_t& h = hist[(static_cast<std::size_t>(t) << D) + d];
                const std::uint64_t c = h;
                h = acc;
                acc += c;
            }
        run([&](unsigned t, std::uint64_t b, std::uint64_t e) {
            std::uint64_t* h = hist.data() + (static_cast<std::size_t>(t) << D);
            for (std::uint64_t i = b; i < e; ++i) tmp[h[(keys[i] >> shift) & mask]++] = keys[i];
        });
        keys.swap(tmp);
    }
}

unsigned bits_for(std::uint64_t n) {
    unsigned b = 0;
    while ((1ULL << b) < n) ++b;
    return std::max(1u, b);
}

// keys: directed (row << 32 | col), both directions present, loops absent,
// duplicates allowed. Sorts, dedups, builds the CSR.
int csr_from_keys(std::uint32_t n, std::vector<std::uint64_t>& keys, th_csr* out) {
    const unsigned b = bits_for(n);
    radix_sort_keys(keys, b, b);
    // loop markers (~0) sort after every real key under the masked bit range
    // (a real key with both halves all-ones would be a loop)
    while (!keys.empty() && keys.back() == ~0ULL) keys.pop_back();
    // dedup (parallel: mark firsts, compact via per-thread counts)
    const std::uint64_t N = keys.size();
    const unsigned T = nthreads();
    std::vector<std::uint64_t> cnt(T + 1, 0);
    auto chunk = [&](unsigned t) { return std::make_pair(N * t / T, N * (t + 1) / T); };
    {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                auto [bb, ee] = chunk(t);
                std::uint64_t c = 0;
                for (std::uint64_t i = bb; i < ee; ++i) c += (i == 0 || keys[i] != keys[i - 1]);
                cnt[t + 1] = c;
            });
        for (auto& th : pool) th.join();
    }
    for (unsigned t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    const std::uint64_t U = cnt[T];
    if (U % 2 != 0) {
        g_err = "csr: asymmetric key set";
        return -1;
    }
    out->n = n;
    out->m = U / 2;
    out->offsets = static_cast<std::uint64_t*>(std::malloc(sizeof(std::uint64_t) * (static_cast<std::size_t>(n) + 1)));
    out->adj = static_cast<std::uint32_t*>(std::malloc(sizeof(std::uint32_t) * std::max<std::uint64_t>(U, 1)));
    if (!out->offsets || !out->adj) {
        g_err = "csr: out of host memory";
        return -1;
    }
    std::vector<std::atomic<std::uint32_t>> deg(n);
    for (auto& d : deg) d.store(0, std::memory_order_relaxed);
    {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                auto [bb, ee] = chunk(t);
                std::uint64_t pos = cnt[t];
                for (std::uint64_t i = bb; i < ee; ++i)
                    if (i == 0 || keys[i] != keys[i - 1]) {
                        out->adj[pos++] = static_cast<std::uint32_t>(keys[i]);
                        deg[keys[i] >> 32].fetch_add(1, std::memory_order_relaxed);
                    }
            });
        for (auto& th : pool) th.join();
    }
    out->offsets[0] = 0;
    for (std::uint32_t u = 0; u < n; ++u) out->offsets[u + 1] = out->offsets[u] + deg[u].load(std::memory_order_relaxed);
    return 0;
}

int csr_from_graph(const trilist::Graph& g, th_csr* out) {
    const std::uint32_t n = g.vertex_count();
    out->n = n;
    out->m = g.edge_count();
    out->offsets = static_cast<std::uint64_t*>(std::malloc(sizeof(std::uint64_t) * (static_cast<std::size_t>(n) + 1)));
    out->adj = static_cast<std::uint32_t*>(std::malloc(sizeof(std::uint32_t) * std::max<std::uint64_t>(2 * out->m, 1)));
    std::uint64_t pos = 0;
    out->offsets[0] = 0;
    for (std::uint32_t u = 0; u < n; ++u) {
        for (std::uint32_t v : g.neighbors(u)) out->adj[pos++] = v;
        out->offsets[u + 1] = pos;
    }
    return 0;
}

}  // namespace

extern "C" {

const char* th_last_error(void) { return g_err.c_str(); }
int th_threads(void) { return static_cast<int>(nthreads()); }

void th_csr_free(th_csr* g) {
    if (!g) return;
    std::free(g->offsets);
    std::free(g->adj);
    g->offsets = nullptr;
    g->adj = nullptr;
}

int th_gen_gnm(std::uint32_t n, std::uint64_t m, std::uint64_t seed, th_csr* out) {
    try {
        return csr_from_graph(trilist::gen_gnm(n, m, seed), out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// R-MAT (a,b,c,d) = (0.57, 0.19, 0.19, 0.05); per level one 32-bit half of a
// draw against integer thresholds round(x * 2^32). Draw i uses stream 1,
// indices i*ceil(scale/2) ... Symmetrised, deduplicated, loops dropped.
namespace {
// Draw i of the R-MAT recipe: `scale` quadrant picks, two per 64-bit draw.
struct RmatDraw {
    static constexpr std::uint32_t tA = 2448131359u;    // round(0.57 * 2^32)
    static constexpr std::uint32_t tAB = 3264175145u;   // round(0.76 * 2^32)
    static constexpr std::uint32_t tABC = 4080218931u;  // round(0.95 * 2^32)
    std::uint32_t scale, per;
    Stream rng;
    RmatDraw(std::uint32_t scale_, std::uint64_t seed) : scale(scale_), per((scale_ + 1) / 2), rng(seed, 1) {}
    void operator()(std::uint64_t i, std::uint32_t& u, std::uint32_t& v) const {
        u = 0;
        v = 0;
        for (std::uint32_t l = 0; l < scale; ++l) {
            const std::uint64_t r64 = rng(i * per + l / 2);
            const std::uint32_t r = (l & 1) ? static_cast<std::uint32_t>(r64) : static_cast<std::uint32_t>(r64 >> 32);
            const std::uint32_t bu = r >= tAB, bv = (r >= tA && r < tAB) || r >= tABC;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
    }
};
}  // namespace

int th_gen_rmat(std::uint32_t scale, std::uint32_t edge_factor, std::uint64_t seed, th_csr* out) {
    if (scale < 1 || scale > 31) {
        g_err = "rmat: scale must be in [1, 31]";
        return -1;
    }
    const std::uint32_t n = 1u << scale;
    const std::uint64_t draws = static_cast<std::uint64_t>(edge_factor) << scale;
    const RmatDraw draw(scale, seed);
    std::vector<std::uint64_t> keys(2 * draws);
    parallel_for(draws, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        for (std::uint64_t i = b; i < e; ++i) {
            std::uint32_t u, v;
            draw(i, u, v);
            if (u == v) {
                keys[2 * i] = keys[2 * i + 1] = ~0ULL;
            } else {
                keys[2 * i] = (static_cast<std::uint64_t>(u) << 32) | v;
                keys[2 * i + 1] = (static_cast<std::uint64_t>(v) << 32) | u;
            }
        }
    });
    // loop markers (~0) are dropped by csr_from_keys
    return csr_from_keys(n, keys, out);
}

int th_gen_rmat_raw(std::uint32_t scale, std::uint32_t edge_factor, std::uint64_t seed, std::int64_t* out) {
    if (scale < 1 || scale > 31) {
        g_err = "rmat: scale must be in [1, 31]";
        return -1;
    }
    const std::uint64_t draws = static_cast<std::uint64_t>(edge_factor) << scale;
    const RmatDraw draw(scale, seed);
    parallel_for(draws, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        for (std::uint64_t i = b; i < e; ++i) {
            std::uint32_t u, v;
            draw(i, u, v);
            out[2 * i] = u;
            out[2 * i + 1] = v;
        }
    });
    return 0;
}

// Chung-Lu: w_i = min(wmin * (1-U)^(-1/(exponent-1)), wmax) (Pareto tail
// exponent `exponent`, e.g. 2.1), `draws` endpoint pairs each drawn
// proportional to w through a Vose alias table with 53-bit integer coin
// thresholds. Loops dropped, duplicates merged.
int th_gen_chung_lu(std::uint32_t n, std::uint64_t draws, double exponent, double wmin,
                    double wmax, std::uint64_t seed, th_csr* out) {
    if (n < 2 || exponent <= 1.0) {
        g_err = "chung_lu: need n >= 2 and exponent > 1";
        return -1;
    }
    const Stream wr(seed, 2), er(seed, 3);
    std::vector<double> w(n);
    const double inv = -1.0 / (exponent - 1.0);
    double total = 0;
    for (std::uint32_t i = 0; i < n; ++i) {
        const double u = static_cast<double>(wr(i) >> 11) * (1.0 / 9007199254740992.0);
        w[i] = std::min(wmin * std::pow(1.0 - u, inv), wmax);
        total += w[i];
    }
    // Vose alias
    std::vector<double> q(n);
    std::vector<std::uint32_t> alias(n), small, large;
    for (std::uint32_t i = 0; i < n; ++i) {
        q[i] = w[i] * n / total;
        (q[i] < 1.0 ? small : large).push_back(i);
    }
    std::vector<std::uint64_t> thr(n);
    while (!small.empty() && !large.empty()) {
        const std::uint32_t s = small.back(), l = large.back();
        small.pop_back();
        thr[s] = static_cast<std::uint64_t>(q[s] * 9007199254740992.0);
        alias[s] = l;
        q[l] = (q[l] + q[s]) - 1.0;
        if (q[l] < 1.0) {
            large.pop_back();
            small.push_back(l);
        }
    }
    for (std::uint32_t i : large) thr[i] = 1ULL << 53, alias[i] = i;
    for (std::uint32_t i : small) thr[i] = 1ULL << 53, alias[i] = i;
    // endpoint j of pair i: slot from draw 4i+2j, coin (53 bits) from 4i+2j+1
    auto pick = [&](std::uint64_t d) {
        const std::uint32_t i = below(static_cast<std::uint32_t>(er(d) >> 32), n);
        return (er(d + 1) >> 11) < thr[i] ? i : alias[i];
    };
    std::vector<std::uint64_t> keys(2 * draws);
    std::atomic<std::uint64_t> loops{0};
    parallel_for(draws, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        std::uint64_t lp = 0;
        for (std::uint64_t i = b; i < e; ++i) {
            const std::uint32_t u = pick(4 * i), v = pick(4 * i + 2);
            if (u == v) {
                keys[2 * i] = keys[2 * i + 1] = ~0ULL;
                ++lp;
            } else {
                keys[2 * i] = (static_cast<std::uint64_t>(u) << 32) | v;
                keys[2 * i + 1] = (static_cast<std::uint64_t>(v) << 32) | u;
            }
        }
        loops += lp;
    });
    return csr_from_keys(n, keys, out);
}

// Watts-Strogatz: ring lattice, vertex i linked to i+1..i+k/2 (mod n); each
// lattice edge (i, i+j) rewires its far endpoint to a uniform vertex with
// probability p (integer threshold); loops dropped, duplicates merged.
int th_gen_ws(std::uint32_t n, std::uint32_t k, double p, std::uint64_t seed, th_csr* out) {
    if (k % 2 || k == 0 || k >= n) {
        g_err = "ws: k must be even, positive and < n";
        return -1;
    }
    const std::uint32_t half = k / 2;
    const std::uint64_t thr = static_cast<std::uint64_t>(std::llround(p * 4294967296.0));
    const Stream rng(seed, 4);
    const std::uint64_t E = static_cast<std::uint64_t>(n) * half;
    std::vector<std::uint64_t> keys(2 * E);
    std::atomic<std::uint64_t> loops{0};
    parallel_for(E, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        std::uint64_t lp = 0;
        for (std::uint64_t idx = b; idx < e; ++idx) {
            const std::uint32_t i = static_cast<std::uint32_t>(idx / half);
            const std::uint32_t j = static_cast<std::uint32_t>(idx % half) + 1;
            std::uint32_t t = static_cast<std::uint32_t>((static_cast<std::uint64_t>(i) + j) % n);
            const std::uint64_t r = rng(idx);
            if ((r >> 32) < thr) t = below(static_cast<std::uint32_t>(r), n);
            if (t == i) {
                keys[2 * idx] = keys[2 * idx + 1] = ~0ULL;
                ++lp;
            } else {
                keys[2 * idx] = (static_cast<std::uint64_t>(i) << 32) | t;
                keys[2 * idx + 1] = (static_cast<std::uint64_t>(t) << 32) | i;
            }
        }
        loops += lp;
    });
    return csr_from_keys(n, keys, out);
}

int th_csr_from_pairs(std::uint32_t n, std::uint64_t npairs, const std::uint32_t* uv, th_csr* out) {
    std::vector<std::uint64_t> keys;
    keys.reserve(2 * npairs);
    for (std::uint64_t i = 0; i < npairs; ++i) {
        const std::uint32_t u = uv[2 * i], v = uv[2 * i + 1];
        if (u >= n || v >= n) {
            g_err = "csr_from_pairs: vertex id out of range";
            return -1;
        }
        if (u == v) continue;
        keys.push_back((static_cast<std::uint64_t>(u) << 32) | v);
        keys.push_back((static_cast<std::uint64_t>(v) << 32) | u);
    }
    return csr_from_keys(n, keys, out);
}

int th_csr_check(const th_csr* g) {
    if (g->offsets[0] != 0 || g->offsets[g->n] != 2 * g->m) {
        g_err = "check: offsets do not span 2m";
        return -1;
    }
    for (std::uint32_t u = 0; u < g->n; ++u) {
        const std::uint64_t b = g->offsets[u], e = g->offsets[u + 1];
        if (e < b) {
            g_err = "check: offsets not monotone";
            return -1;
        }
        for (std::uint64_t i = b; i < e; ++i) {
            const std::uint32_t v = g->adj[i];
            if (v >= g->n || v == u || (i > b && g->adj[i - 1] >= v)) {
                g_err = "check: row not strictly increasing / loop / out of range";
                return -1;
            }
            const std::uint32_t* lo = g->adj + g->offsets[v];
            const std::uint32_t* hi = g->adj + g->offsets[v + 1];
            if (!std::binary_search(lo, hi, u)) {
                g_err = "check: asymmetric adjacency";
                return -1;
            }
        }
    }
    return 0;
}

void* th_graph_new(const th_csr* g) {
    try {
        std::vector<std::pair<trilist::VertexId, trilist::VertexId>> edges;
        edges.reserve(g->m);
        for (std::uint32_t u = 0; u < g->n; ++u)
            for (std::uint64_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e)
                if (u < g->adj[e]) edges.emplace_back(u, g->adj[e]);
        return new trilist::Graph(trilist::Graph::from_dense_edges(g->n, std::move(edges)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void th_graph_free(void* graph) { delete static_cast<trilist::Graph*>(graph); }

void* th_graph_load(const char* path, std::uint64_t* loops, std::uint64_t* dups) {
    try {
        trilist::NormalizeStats stats;
        auto* g = new trilist::Graph(trilist::load_edgelist_file(path, &stats));
        if (loops) *loops = stats.loops_removed;
        if (dups) *dups = stats.duplicates_removed;
        return g;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Native edge-list reader: the same line grammar as the reference's
// load_edgelist (graph.cpp:164-186) -- getline lines, one trailing '\r'
// dropped, tokens split on ' ' / '\t', empty lines and lines whose first token
// starts with '#' skipped, two std::from_chars int64 labels and nothing after
// them, else "line N: ..." (ParseError, common.hpp:16-20) for the FIRST bad
// line -- over an mmap of the file, one contiguous slice of lines per thread,
// slices concatenated in file order. The raw pairs (loops and duplicates
// kept) are what normalize() takes (graph.cpp:115), so the GPU normalize
// (tl_normalize) finishes the reference's load_edgelist_file.
int th_parse_edgelist(const char* path, std::int64_t** edges, std::uint64_t* k) {
    *edges = nullptr;
    *k = 0;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        g_err = std::string("cannot open edge list: ") + path;
        return -1;
    }
    struct stat sb {};
    if (::fstat(fd, &sb) != 0) {
        ::close(fd);
        g_err = std::string("cannot stat edge list: ") + path;
        return -1;
    }
    const std::size_t size = static_cast<std::size_t>(sb.st_size);
    const char* data = nullptr;
    if (size) {
        void* p = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
        if (p == MAP_FAILED) {
            ::close(fd);
            g_err = std::string("cannot map edge list: ") + path;
            return -1;
        }
        data = static_cast<const char*>(p);
    }
    ::close(fd);
    const unsigned T = static_cast<unsigned>(std::max<std::size_t>(1, std::min<std::size_t>(nthreads(), size / (1u << 20) + 1)));
    // slice t = the lines STARTING in [cut[t], cut[t+1])
    std::vector<std::size_t> cut(T + 1, size);
    cut[0] = 0;
    for (unsigned t = 1; t < T; ++t) {
        std::size_t c = size * t / T;
        const void* nl = c < size ? std::memchr(data + c, '\n', size - c) : nullptr;
        cut[t] = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - data) + 1 : size;
        cut[t] = std::max(cut[t], cut[t - 1]);
    }
    struct Slice {
        std::vector<std::int64_t> e;
        std::size_t bad = SIZE_MAX;  // byte offset of the first bad line
        std::string what;
    };
    std::vector<Slice> sl(T);
    auto is_sep = [](char c) { return c == ' ' || c == '\t'; };
    auto parse = [&](unsigned t) {
        Slice& s = sl[t];
        s.e.reserve((cut[t + 1] - cut[t]) / 8);
        std::size_t pos = cut[t];
        const std::size_t end = cut[t + 1];
        while (pos < end) {
            const char* nl = static_cast<const char*>(std::memchr(data + pos, '\n', size - pos));
            const std::size_t le = nl ? static_cast<std::size_t>(nl - data) : size;  // line [pos, le)
            std::size_t lend = le;
            if (lend > pos && data[lend - 1] == '\r') --lend;
            std::size_t i = pos;
            auto token = [&](std::size_t& b, std::size_t& e) {
                while (i < lend && is_sep(data[i])) ++i;
                b = i;
                while (i < lend && !is_sep(data[i])) ++i;
                e = i;
            };
            std::size_t ub, ue, vb, ve, tb, te;
            token(ub, ue);
            if (ue > ub && data[ub] != '#') {
                token(vb, ve);
                std::int64_t u = 0, v = 0;
                auto ok = [&](std::size_t b, std::size_t e, std::int64_t& out) {
                    const auto r = std::from_chars(data + b, data + e, out);
                    return r.ec == std::errc{} && r.ptr == data + e;
                };
                if (ve == vb || !ok(ub, ue, u) || !ok(vb, ve, v)) {
                    s.bad = pos;
                    s.what = "expected two integer labels, got \"" + std::string(data + pos, lend - pos) + "\"";
                    return;
                }
                token(tb, te);
                if (te > tb) {
                    s.bad = pos;
                    s.what = "trailing tokens after edge pair";
                    return;
                }
                s.e.push_back(u);
                s.e.push_back(v);
            }
            pos = le + 1;
        }
    };
    if (T == 1) {
        parse(0);
    } else {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t) pool.emplace_back(parse, t);
        for (auto& th : pool) th.join();
    }
    int rc = 0;
    std::uint64_t total = 0;
    for (unsigned t = 0; t < T && rc == 0; ++t) {
        if (sl[t].bad != SIZE_MAX) {  // the first bad line in file order
            const std::size_t line = 1 + static_cast<std::size_t>(std::count(data, data + sl[t].bad, '\n'));
            g_err = "line " + std::to_string(line) + ": " + sl[t].what;
            rc = -1;
        }
        total += sl[t].e.size();
    }
    if (rc == 0 && total) {
        auto* out = static_cast<std::int64_t*>(std::malloc(total * sizeof(std::int64_t)));
        if (!out) {
            g_err = "edge list: out of host memory";
            rc = -1;
        } else {
            std::uint64_t o = 0;
            for (auto& s : sl) {
                std::copy(s.e.begin(), s.e.end(), out + o);
                o += s.e.size();
            }
            *edges = out;
            *k = total / 2;
        }
    }
    if (data) ::munmap(const_cast<char*>(data), size);
    return rc;
}

void th_free(void* p) { std::free(p); }

int th_graph_to_csr(void* graph, th_csr* out) {
    return csr_from_graph(*static_cast<trilist::Graph*>(graph), out);
}

void th_graph_labels(void* graph, std::int64_t* out) {
    const auto& labels = static_cast<trilist::Graph*>(graph)->labels();
    std::copy(labels.begin(), labels.end(), out);
}

int th_order(void* graph, const char* method, std::uint64_t seed, std::uint32_t* rank_out,
             double* order_ms) {
    try {
        const trilist::Graph& g = *static_cast<trilist::Graph*>(graph);
        const std::string m = method;
        const auto t0 = std::chrono::steady_clock::now();
        trilist::Ordering pi;
        if (m == "identity") pi = trilist::identity_order(g);
        else if (m == "random") pi = trilist::random_order(g, seed);
        else if (m == "degree") pi = trilist::degree_order(g);
        else if (m == "core") pi = trilist::core_order(g);
        else if (m == "split") pi = trilist::split_order(g);
        else if (m == "check") pi = trilist::check_order(g);
        else if (m == "neigh") pi = trilist::neigh_order(g);
        else {
            g_err = "unknown ordering method: " + m;
            return -1;
        }
        if (order_ms)
            *order_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(rank_out, pi.ranks().data(), sizeof(std::uint32_t) * pi.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int th_cost(void* graph, const std::uint32_t* rank, std::uint64_t out[4]) {
    try {
        const trilist::Graph& g = *static_cast<trilist::Graph*>(graph);
        const auto pi = trilist::Ordering::from_ranks(
            std::vector<std::uint32_t>(rank, rank + g.vertex_count()));
        const auto r = trilist::cost_report(g, pi);
        out[0] = r.c_pp;
        out[1] = r.c_pm;
        out[2] = r.c_mm;
        out[3] = r.sum_deg_sq;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

const char* th_bench_csv_header(void) { return trilist::kBenchCsvHeader; }

int th_bench_csv(const char* dataset, const char* algo, const char* ordering, const char* mode,
                 unsigned threads, std::uint64_t n, std::uint64_t m, std::uint64_t c_pp,
                 std::uint64_t c_pm, std::uint64_t inner_ops, std::uint64_t triangles,
                 double load_ms, double order_ms, double list_ms, char* buf, std::uint64_t cap) {
    trilist::BenchRecord r;
    r.dataset = dataset;
    r.algo = algo;
    r.ordering = ordering;
    r.mode = mode;
    r.threads = threads;
    r.n = n;
    r.m = m;
    r.c_pp = c_pp;
    r.c_pm = c_pm;
    r.inner_ops = inner_ops;
    r.triangles = triangles;
    r.load_ms = load_ms;
    r.order_ms = order_ms;
    r.list_ms = list_ms;
    const std::string row = trilist::to_csv_row(r);
    if (row.size() + 1 > cap) return -1;
    std::memcpy(buf, row.c_str(), row.size() + 1);
    return 0;
}

}  // extern "C"
