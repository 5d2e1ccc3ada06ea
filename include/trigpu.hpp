// trigpu.hpp -- header-only C++ shim: the reference trilist listing API over
// the trigpu C-ABI (include/trigpu.h).
//
// A reference caller switches by replacing
//     #include "trilist/listing.hpp"        (core/include/trilist/listing.hpp)
//     trilist::OrientedView view(g, pi);    (oriented_view.hpp:19)
//     trilist::list_apm(view, sink);        (listing.hpp:168-173)
// with
//     #include "trigpu.hpp"
//     trigpu::OrientedView view(g, pi);
//     trigpu::list_apm(view, sink);
// Graph, Ordering, CountingSink, CollectingSink and ListingStats stay the
// reference's types. Semantics kept:
//   * std::invalid_argument("orient: ordering does not match graph") on a size
//     mismatch (oriented_view.cpp:8-9), std::runtime_error on device errors;
//   * ListingStats filled exactly: triangle_count, inner_ops = c_pp (app) /
//     c_pm (apm), mark_ops = 2m, wall_ms = listing kernel time;
//   * CountingSink / CollectingSink receive the same counts / triangle sets
//     (emission order unspecified, as for list_*_parallel, listing.hpp:185-186);
//   * any other sink gets the triangles replayed through operator()(u, v, w)
//     (slow path: the full list crosses PCIe).
// New sinks: trigpu::ChecksumSink and trigpu::VertexCountSink (fused on GPU).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "trigpu.h"
#include "trilist/graph.hpp"
#include "trilist/listing.hpp"
#include "trilist/ordering.hpp"

namespace trigpu {

using trilist::VertexId;

class Error : public std::runtime_error {
public:
    Error(tl_status st, const std::string& what) : std::runtime_error(what), status(st) {}
    tl_status status;
};

class Context {
public:
    explicit Context(int device = 0) {
        tl_ctx* p = nullptr;
        const tl_status st = tl_create(&p, device);
        if (st != TL_OK) throw Error(st, tl_last_error(nullptr));
        ctx_.reset(p);
    }
    tl_ctx* get() const { return ctx_.get(); }
    void check(tl_status st) const {
        if (st == TL_OK) return;
        const std::string msg = tl_last_error(ctx_.get());
        if (st == TL_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
        throw Error(st, msg);
    }

private:
    struct Del {
        void operator()(tl_ctx* p) const { tl_destroy(p); }
    };
    std::unique_ptr<tl_ctx, Del> ctx_;
};

inline Context& default_context() {
    static Context ctx(0);
    return ctx;
}

// degree_order / split_order (ordering.cpp:66-109) computed on the GPU;
// returns the reference's Ordering type with bit-identical ranks.
inline trilist::Ordering device_order(const trilist::Graph& g, int method, Context& ctx = default_context()) {
    const VertexId n = g.vertex_count();
    std::vector<std::uint64_t> off(static_cast<std::size_t>(n) + 1, 0);
    for (VertexId u = 0; u < n; ++u) off[u + 1] = off[u] + g.degree(u);
    std::vector<VertexId> rank(n);
    ctx.check(tl_order(ctx.get(), n, off.data(), method, rank.data()));
    return trilist::Ordering::from_ranks(std::move(rank));
}
inline trilist::Ordering degree_order(const trilist::Graph& g, Context& ctx = default_context()) {
    return device_order(g, TL_ORDER_DEGREE, ctx);
}
inline trilist::Ordering split_order(const trilist::Graph& g, Context& ctx = default_context()) {
    return device_order(g, TL_ORDER_SPLIT, ctx);
}

// core_decompose (ordering.cpp:141-188) on the GPU. coreness and degeneracy
// equal the reference's; `order` is a degeneracy ordering ((peel round, id)
// ascending, see trigpu.h), not the reference's swap-dependent sequence.
inline trilist::CoreDecomposition core_decompose(const trilist::Graph& g, Context& ctx = default_context()) {
    const VertexId n = g.vertex_count();
    std::vector<std::uint64_t> off(static_cast<std::size_t>(n) + 1, 0);
    std::vector<VertexId> adj;
    adj.reserve(2 * g.edge_count());
    for (VertexId u = 0; u < n; ++u) {
        off[u + 1] = off[u] + g.degree(u);
        for (VertexId v : g.neighbors(u)) adj.push_back(v);
    }
    std::vector<VertexId> rank(n);
    trilist::CoreDecomposition out;
    out.coreness.assign(n, 0);
    std::uint32_t dg = 0;
    ctx.check(tl_core_decompose(ctx.get(), n, g.edge_count(), off.data(), adj.data(), rank.data(),
                                out.coreness.data(), &dg));
    out.degeneracy = dg;
    out.order = trilist::Ordering::from_ranks(std::move(rank));
    return out;
}
inline trilist::Ordering core_order(const trilist::Graph& g, Context& ctx = default_context()) {
    return core_decompose(g, ctx).order;
}

// GPU-resident OrientedView (oriented_view.hpp:17-50). The device holds one
// view per Context; constructing another view in the same context replaces it
// (each listing call re-orients if needed).
class OrientedView {
public:
    OrientedView(const trilist::Graph& g, const trilist::Ordering& pi, Context& ctx = default_context())
        : ctx_(&ctx), g_(&g), n_(g.vertex_count()), m_(g.edge_count()), id_(next_id()) {
        if (pi.size() != g.vertex_count())
            throw std::invalid_argument("orient: ordering does not match graph");
        rank_.assign(pi.ranks().begin(), pi.ranks().end());
        inverse_.assign(pi.sequence().begin(), pi.sequence().end());
        offsets_.resize(static_cast<std::size_t>(n_) + 1);
        offsets_[0] = 0;
        for (VertexId u = 0; u < n_; ++u) offsets_[u + 1] = offsets_[u] + g.degree(u);
        upload();
    }

    VertexId vertex_count() const { return n_; }
    std::uint64_t edge_count() const { return m_; }
    VertexId rank_of(VertexId v) const { return rank_[v]; }
    VertexId vertex_at(VertexId p) const { return inverse_[p]; }

    std::span<const VertexId> successors(VertexId u) const {
        fetch();
        return {succ_.data() + succ_off_[u], succ_.data() + succ_off_[u + 1]};
    }
    std::span<const VertexId> predecessors(VertexId u) const {
        fetch();
        return {pred_.data() + pred_off_[u], pred_.data() + pred_off_[u + 1]};
    }
    VertexId out_degree(VertexId u) const {
        fetch();
        return static_cast<VertexId>(succ_off_[u + 1] - succ_off_[u]);
    }
    VertexId in_degree(VertexId u) const {
        fetch();
        return static_cast<VertexId>(pred_off_[u + 1] - pred_off_[u]);
    }

    Context& context() const { return *ctx_; }
    // (Re)build this view on the device if another view replaced it.
    void make_current() const {
        if (current_owner(ctx_) != id_) upload();
    }

private:
    static std::uint64_t next_id() {
        static std::uint64_t id = 0;
        return ++id;
    }
    // id of the view whose CSR the context currently holds
    static std::uint64_t& current_owner(Context* c) {
        static std::vector<std::pair<Context*, std::uint64_t>> owners;
        for (auto& [k, v] : owners)
            if (k == c) return v;
        owners.emplace_back(c, 0);
        return owners.back().second;
    }
    void upload() const {
        // contiguous adjacency_ (graph.hpp:60): neighbors(0) starts the array
        const VertexId* adj = m_ ? g_->neighbors(0).data() : nullptr;
        ctx_->check(tl_orient(ctx_->get(), n_, m_, offsets_.data(), adj, rank_.data()));
        current_owner(ctx_) = id_;
    }
    void fetch() const {
        if (fetched_) return;
        make_current();
        succ_off_.resize(static_cast<std::size_t>(n_) + 1);
        pred_off_.resize(static_cast<std::size_t>(n_) + 1);
        succ_.resize(m_);
        pred_.resize(m_);
        ctx_->check(tl_fetch_oriented(ctx_->get(), succ_off_.data(), succ_.data(), pred_off_.data(),
                                      pred_.data()));
        fetched_ = true;
    }

    Context* ctx_;
    const trilist::Graph* g_;
    VertexId n_;
    std::uint64_t m_;
    std::uint64_t id_;
    std::vector<VertexId> rank_, inverse_;
    std::vector<std::uint64_t> offsets_;
    mutable bool fetched_ = false;
    mutable std::vector<std::uint64_t> succ_off_, pred_off_;
    mutable std::vector<VertexId> succ_, pred_;
};

// Order-independent checksum sink, fused on the GPU.
struct ChecksumSink {
    std::uint64_t count = 0;
    std::uint64_t checksum = 0;
    void merge(ChecksumSink&& o) {
        count += o.count;
        checksum += o.checksum;
    }
};

// Per-vertex triangle counts, fused on the GPU.
struct VertexCountSink {
    std::uint64_t count = 0;
    std::vector<std::uint64_t> counts;
    void merge(VertexCountSink&& o) {
        count += o.count;
        if (counts.empty()) counts.assign(o.counts.size(), 0);
        for (std::size_t i = 0; i < o.counts.size(); ++i) counts[i] += o.counts[i];
    }
};

namespace detail {

template <class Sink>
trilist::ListingStats run(int algo, const OrientedView& view, Sink& sink) {
    using S = std::decay_t<Sink>;
    Context& ctx = view.context();
    view.make_current();
    unsigned flags = TL_OUT_COUNT;
    if constexpr (std::is_same_v<S, ChecksumSink>) flags = TL_OUT_CHECKSUM;
    else if constexpr (std::is_same_v<S, VertexCountSink>) flags = TL_OUT_VERTEX_COUNTS;
    else if constexpr (!std::is_same_v<S, trilist::CountingSink>) flags = TL_OUT_LIST;
    tl_stats st{};
    ctx.check(tl_list(ctx.get(), algo, flags, &st));
    trilist::ListingStats out;
    out.triangle_count = st.triangle_count;
    out.inner_ops = st.inner_ops;
    out.mark_ops = st.mark_ops;
    out.wall_ms = st.list_ms;
    if constexpr (std::is_same_v<S, trilist::CountingSink>) {
        sink.count += st.triangle_count;
    } else if constexpr (std::is_same_v<S, ChecksumSink>) {
        sink.count += st.triangle_count;
        sink.checksum += st.checksum;
    } else if constexpr (std::is_same_v<S, VertexCountSink>) {
        sink.count += st.triangle_count;
        std::vector<std::uint64_t> c(view.vertex_count());
        ctx.check(tl_fetch_vertex_counts(ctx.get(), c.data()));
        if (sink.counts.empty()) sink.counts.assign(c.size(), 0);
        for (std::size_t i = 0; i < c.size(); ++i) sink.counts[i] += c[i];
    } else {
        std::vector<VertexId> tri(3 * st.triangle_count);
        std::uint64_t k = 0;
        ctx.check(tl_fetch_triangles(ctx.get(), tri.data(), st.triangle_count, &k));
        if constexpr (std::is_same_v<S, trilist::CollectingSink>) {
            sink.triangles.reserve(sink.triangles.size() + k);
            for (std::uint64_t i = 0; i < k; ++i)
                sink.triangles.push_back({tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]});
        } else {
            for (std::uint64_t i = 0; i < k; ++i) sink(tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]);
        }
    }
    return out;
}

}  // namespace detail

// listing.hpp:162-166 / 168-173
template <typename Sink>
trilist::ListingStats list_app(const OrientedView& view, Sink&& sink) {
    return detail::run(TL_ALGO_APP, view, sink);
}
template <typename Sink>
trilist::ListingStats list_apm(const OrientedView& view, Sink&& sink) {
    return detail::run(TL_ALGO_APM, view, sink);
}
// listing.hpp:175-183
template <typename Sink>
trilist::ListingStats list_app(const trilist::Graph& g, const trilist::Ordering& pi, Sink&& sink) {
    return list_app(OrientedView(g, pi), sink);
}
template <typename Sink>
trilist::ListingStats list_apm(const trilist::Graph& g, const trilist::Ordering& pi, Sink&& sink) {
    return list_apm(OrientedView(g, pi), sink);
}
// listing.hpp:187-199: the device always runs every seed in parallel.
template <typename Sink>
trilist::ListingStats list_app_parallel(const OrientedView& view, Sink& sink, unsigned) {
    return list_app(view, sink);
}
template <typename Sink>
trilist::ListingStats list_apm_parallel(const OrientedView& view, Sink& sink, unsigned) {
    return list_apm(view, sink);
}

inline OrientedView orient(const trilist::Graph& g, const trilist::Ordering& pi) {
    return OrientedView(g, pi);
}

}  // namespace trigpu
