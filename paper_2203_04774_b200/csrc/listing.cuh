// listing.cuh -- degree-binned A+- / A++ listing kernels with fused sinks (K4-K6).
//
// Reference loops (core/include/trilist/listing.hpp):
//   A+- run_apm_range :91-107  seed u, mark N+(u), for v in N+(u) scan N+(v),
//                              emit (u, v, w) when w is marked
//   A++ run_app_range :69-86   seed w, mark N-(w), for u in N-(w) scan N+(u),
//                              emit (u, v, w) when v is marked
// Both are "seed s, probe set S = set-row(s), for x in S scan out-row(x), hit
// when y in S". All ids are ranks, rows ascending. The triangle is
// (s, x, y) for A+- and (x, y, s) for A++ - already rank-ascending.
//
// The reference's uint8 table[n] (listing.hpp:113) becomes a per-seed
// windowed bitmap in shared memory sized to the class of |S| (degree binning):
//   class R  2 <= |S| <= 32     warp per seed, 2^15-bit window per warp
//   class H  32 < |S| <= 256    warp per seed, 2^16-bit window per warp
//   class C1 256 < |S| <= 1024  CTA (8 warps) per seed, 2^18-bit window
//   class C2 1024 < |S| <= 4096 CTA (32 warps) per seed, 2^19-bit window
//   class G  |S| > 4096         CTA per seed, n-bit bitmap in global memory
// Every class reads the out-rows of the seed's set as 128-element chunks of
// 16-byte quads (one 512-byte warp load per chunk, four chunks in flight);
// rows shorter than kLongRow are walked as one flattened stream over 32 rows.
//
// Sinks are fused into the same pass (template flags): count, order-
// independent checksum over dense ids, per-vertex counts, and list output by
// warp-aggregated atomic append. inner_ops / mark_ops are not counted in the
// inner loop: they equal c_pm / c_pp and 2m (Property 1; listing_test.cpp:80-93)
// and come from the degree reduction k_cost.
#pragma once

#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace trigpu {

enum : unsigned { F_CHECKSUM = 1u, F_VCOUNT = 2u, F_LIST = 4u };
enum : int { ALGO_APP = 0, ALGO_APM = 1 };

struct ListParams {
    uint32_t n;
    const uint64_t* set_off;  // probe-set rows: out-CSR (A+-) or in-CSR (A++): start, length
    const uint32_t* set_len;
    const uint32_t* set_adj;
    const uint64_t* out_off;  // scanned rows: always the out-CSR, rows padded to quads (starts
    const uint32_t* out_len;  //   are multiples of 4, pad slots hold kNone)
    const uint32_t* out_adj;
    const uint32_t* inv;      // rank -> dense id
    const unsigned long long* hv;  // rank -> vertex_hash(dense id) (checksum sink)
    unsigned long long* acc;  // [0] triangles, [1] checksum, [2] list cursor
    unsigned long long* vcount;  // rank space
    uint32_t* tri;
    unsigned long long tri_cap;
    const uint32_t* seeds;    // class list
    unsigned int nseeds;
    unsigned int* queue;      // dynamic work counter
    uint32_t* bitmaps;        // class G only: one n-bit bitmap per CTA
    uint64_t bitmap_words;
    int variant;              // TL_DEBUG_VARIANT: 2 = null probe (experiments build, timing only)
    uint32_t bm_shrink;       // TL_DEBUG_BM_SHRINK: smaller windows (tests force the below-window path)
};

// Per-warp hit buffer (per-vertex-count and list sinks): hits (x, y) are
// compacted into shared memory by a ballot and emitted 32 at a time with
// every lane busy (dense-id gathers, atomics) instead of with the 1-3 lanes
// that hit in a batch.
constexpr int kHitBuf = 96;  // 31 pending + up to 2 batches of 32 before a drain

// ---- the probe: a windowed bitmap over the seed's set ----------------------
// S (sorted ranks s_0 < ... < s_{d-1}) is held in shared memory as
//   region A: an EXACT bitmap over the rank window [wb, wb + LA) - one bit per
//             rank, then one always-zero guard word;
//   region B: for the keys below the window (only when the set spans more
//             than LA ranks), a 2^KB-bit filter indexed by key mod 2^KB.
// wb = s_0 when the set fits the window (no region B), else
// wb = s_{d-1} + 1 - LA, so the window holds the set's TOP ranks: under
// degree order the scanned rows are made of hubs, so on R-MAT 100 % of the
// class H / C hits and >98 % of the probes fall in the window.
// A probe of y is ONE LDS.32 of the word of bit min(y - wb, LA) (offsets
// outside the window clamp onto the guard word). Rows are sorted, so the 32
// lanes of a chunk read few distinct words in distinct banks: ~1.3 shared
// wavefronts per 32 probes against ~9 for a 16-byte hash bucket.
// Elements below the window (rare; a chunk's are found by one compare per
// lane on its sorted quad) take region B; its candidates are verified exactly
// (V: binary search of the sorted set) on the spot and become ordinary hits,
// so the sinks only ever see exact hits.
template <bool kLow, class V>
struct WinProbe {
    static constexpr bool low = kLow;
    unsigned bm;     // shared address of region A
    unsigned bmb;    // shared address of region B
    uint32_t wb;     // window base
    uint32_t la;     // window length LA (a power of two)
    uint32_t maskb;  // 2^KB - 1
    V ver;
    // 0/1: y is in S (y inside the window) / 0 (y outside)
    __device__ __forceinline__ uint32_t bit(uint32_t y) const {
        const uint32_t o = min(y - wb, la);
        return (lds32(bm + ((o >> 5) << 2)) >> (o & 31u)) & 1u;
    }
    __device__ __forceinline__ bool below(uint32_t y) const { return y < wb; }
    // region-B candidate (call for y below the window only)
    __device__ __forceinline__ uint32_t cand(uint32_t y) const {
        const uint32_t o = y & maskb;
        return (lds32(bmb + ((o >> 5) << 2)) >> (o & 31u)) & 1u;
    }
    __device__ __forceinline__ bool verify(uint32_t y, bool act) const { return ver(y, act); }
    // the value padding a partial quad: never in the window, never below it
    // (tl_orient keeps n <= 2^32 - 2^20, so kNone - wb >= LA)
    __device__ __forceinline__ uint32_t sentinel() const { return kNone; }
};

// Bitmap geometry of one seed: window length, region-B mask, base.
struct WinGeom {
    uint32_t la, maskb, wb;
    bool low;
};
__device__ __forceinline__ WinGeom win_geom(uint32_t bits_a, uint32_t bits_b, uint32_t shrink, uint32_t s0,
                                            uint32_t top) {
    const uint32_t ka = bits_a > shrink + 5u ? bits_a - shrink : 5u;
    const uint32_t kb = bits_b > shrink + 5u ? bits_b - shrink : 5u;
    WinGeom g;
    g.la = 1u << ka;
    g.maskb = (1u << kb) - 1u;
    g.low = top - s0 >= g.la;
    g.wb = g.low ? top + 1u - g.la : s0;
    return g;
}
__device__ __forceinline__ void win_set(uint32_t* bma, uint32_t* bmb, const WinGeom& g, uint32_t key) {
    if (key >= g.wb) {
        const uint32_t o = key - g.wb;
        atomicOr(bma + (o >> 5), 1u << (o & 31u));
    } else {
        const uint32_t o = key & g.maskb;
        atomicOr(bmb + (o >> 5), 1u << (o & 31u));
    }
}
__device__ __forceinline__ void win_clear(uint32_t* bma, uint32_t* bmb, const WinGeom& g, uint32_t key) {
    if (key >= g.wb) bma[(key - g.wb) >> 5] = 0u;
    else bmb[(key & g.maskb) >> 5] = 0u;
}
constexpr size_t win_bytes(uint32_t bits_a, uint32_t bits_b) {
    return (size_t{1} << bits_a) / 8 + 16 + (size_t{1} << bits_b) / 8;  // A, guard (padded), B
}

// Exact membership for region-B candidates.
struct RegVerify {  // S sorted ascending, one key per lane, padded with kNone (warp-collective)
    uint32_t s;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        int pos = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, s, pos + step - 1);
            if (v < y) pos += step;
        }
        const uint32_t v = __shfl_sync(FULL, s, pos & 31);
        return act && pos < 32 && v == y && y != kNone;  // kNone pads the lanes past |S|
    }
};

struct RowVerify {  // branch-free binary search of the seed's sorted set row (L1-resident)
    const uint32_t* row;
    uint32_t d;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        uint32_t lo = 0, len = d;
        while (len > 1) {  // uniform trip count: log2(d) steps
            const uint32_t half = len >> 1;
            if (__ldg(row + lo + half) <= y) lo += half;
            len -= half;
        }
        return act && __ldg(row + lo) == y;
    }
};

// Class G: exact n-bit bitmap in global memory (L2-resident per CTA).
struct BitmapProbe {
    static constexpr bool low = false;
    const uint32_t* bm;
    uint32_t n;  // bits n .. are the always-zero slack words
    __device__ __forceinline__ uint32_t bit(uint32_t y) const {
        y = min(y, n);  // pad slots (kNone) read the zero slack
        return (__ldcg(bm + (y >> 5)) >> (y & 31)) & 1u;
    }
    __device__ __forceinline__ bool below(uint32_t) const { return false; }
    __device__ __forceinline__ uint32_t cand(uint32_t) const { return 0u; }
    __device__ __forceinline__ bool verify(uint32_t, bool act) const { return act; }
    __device__ __forceinline__ uint32_t sentinel() const { return n; }
};

// Timing-only probe (TL_DEBUG_VARIANT 2 in a -DTRIGPU_EXPERIMENTS build):
// touches every loaded element, never hits. Measures the row-streaming limit.
struct NullProbe {
    static constexpr bool low = false;
    __device__ __forceinline__ uint32_t bit(uint32_t y) const { return y == 0xFFFFFFFEu; }
    __device__ __forceinline__ bool below(uint32_t) const { return false; }
    __device__ __forceinline__ uint32_t cand(uint32_t) const { return 0u; }
    __device__ __forceinline__ bool verify(uint32_t, bool act) const { return act; }
    __device__ __forceinline__ uint32_t sentinel() const { return 0u; }
};

// Exact hit of one element, region-B candidates verified on the spot
// (warp-convergent: RegVerify shuffles).
template <class Probe>
__device__ __forceinline__ bool probe_one(const Probe& probe, uint32_t y, bool act) {
    bool hit = act && probe.bit(y);
    if constexpr (Probe::low) {
        const bool c = act && probe.below(y) && probe.cand(y);
        if (__any_sync(FULL, c)) hit |= probe.verify(y, c);
    }
    return hit;
}

// ---- sinks -------------------------------------------------------------------
// Count: hit bits are added in the stream. Checksum: sum over triangles
// (s, x, y) of h(s) h(x) h(y) (common.cuh), h from the per-rank table hv; with
// the count + checksum sinks nothing is buffered: a chunk's hits add their
// h(y) lane-locally and one multiply by h(s) h(x) folds them in (kFastSum).
// Per-vertex counts and lists go through the warp's hit buffer (emit).
template <int ALGO, unsigned F>
struct Sink {
    static constexpr bool kFastSum = (F & F_CHECKSUM) != 0u && (F & (F_VCOUNT | F_LIST)) == 0u;
    static constexpr bool kBuffered = (F & (F_VCOUNT | F_LIST)) != 0u;
    unsigned long long cnt = 0, sum = 0;
    unsigned long long hs = 0;    // h(seed)
    unsigned long long acc = 0;   // this seed's sum of h(x) h(y); times h(s) at end_unit
    unsigned seed_hits = 0;
    unsigned buf = 0;      // shared address of this warp's kHitBuf uint2 entries
    unsigned pending = 0;  // warp-uniform

    __device__ __forceinline__ void begin_unit(const ListParams& P, uint32_t seed) {
        if constexpr ((F & F_CHECKSUM) != 0u) hs = __ldg(P.hv + seed);
    }

    // One hit with its own x (short-row stream), kFastSum only.
    __device__ __forceinline__ void direct(const ListParams& P, bool hit, uint32_t x, uint32_t y) {
        if constexpr (kFastSum)
            if (hit) acc += __ldg(P.hv + x) * __ldg(P.hv + y);
    }

    // One 32-wide batch of hits (called convergently by the warp), kBuffered only.
    __device__ __forceinline__ void batch(bool hit, uint32_t x, uint32_t y) {
        if constexpr (kBuffered) {
            const unsigned b = __ballot_sync(FULL, hit);
            if (!b) return;
            if (hit) sts64(buf + 8u * (pending + __popc(b & lanemask_lt())), make_uint2(x, y));
            pending += __popc(b);
        }
    }

    // Handle n (<= 32) buffered hits, lane i taking entry i.
    __device__ __forceinline__ void emit(const ListParams& P, uint32_t seed, unsigned n, unsigned from) {
        const unsigned lane = lane_id();
        const bool hit = lane < n;
        const uint2 e = hit ? lds64(from + 8u * lane) : make_uint2(0, 0);
        const uint32_t x = e.x, y = e.y;
        if constexpr ((F & F_VCOUNT) != 0u) {
            // hubs recur within the 32 entries (same x for a chunk's hits,
            // the same hub y for many x): one atomic per distinct vertex
            const unsigned gx = __match_any_sync(FULL, hit ? x : kNone);
            const unsigned gy = __match_any_sync(FULL, hit ? y : kNone);
            if (hit && (gx & lanemask_lt()) == 0) atomicAdd(&P.vcount[x], (unsigned long long)__popc(gx));
            if (hit && (gy & lanemask_lt()) == 0) atomicAdd(&P.vcount[y], (unsigned long long)__popc(gy));
            seed_hits += hit;
        }
        if constexpr ((F & F_CHECKSUM) != 0u)
            if (hit) acc += __ldg(P.hv + x) * __ldg(P.hv + y);
        if constexpr ((F & F_LIST) != 0u) {
            const uint32_t ru = ALGO == ALGO_APM ? seed : x;
            const uint32_t rv = ALGO == ALGO_APM ? x : y;
            const uint32_t rw = ALGO == ALGO_APM ? y : seed;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&P.acc[2], (unsigned long long)n);
            base = __shfl_sync(FULL, base, 0);
            if (hit) {
                const unsigned long long k = base + lane;
                if (k < P.tri_cap) {
                    P.tri[3 * k] = __ldg(P.inv + ru);
                    P.tri[3 * k + 1] = __ldg(P.inv + rv);
                    P.tri[3 * k + 2] = __ldg(P.inv + rw);
                }
            }
        }
    }

    // Emit every full group of 32 buffered hits (call after <= 2 batches).
    __device__ __forceinline__ void drain(const ListParams& P, uint32_t seed) {
        if constexpr (kBuffered) {
            if (pending < 32) return;
            __syncwarp();
            unsigned done = 0;
            for (; pending - done >= 32; done += 32) emit(P, seed, 32, buf + 8u * done);
            __syncwarp();
            if (lane_id() < pending - done) sts64(buf + 8u * lane_id(), lds64(buf + 8u * (done + lane_id())));
            __syncwarp();
            pending -= done;
        }
    }

    // End of one seed's unit: drain the buffer, credit the seed's own count.
    __device__ __forceinline__ void end_unit(const ListParams& P, uint32_t seed) {
        if constexpr (kBuffered) {
            drain(P, seed);
            if (pending) {
                __syncwarp();
                emit(P, seed, pending, buf);
                __syncwarp();
                pending = 0;
            }
        }
        if constexpr ((F & F_VCOUNT) != 0u) {
            const unsigned long long h = warp_sum64(seed_hits);
            if (lane_id() == 0 && h) atomicAdd(&P.vcount[seed], h);
            seed_hits = 0;
        }
        if constexpr ((F & F_CHECKSUM) != 0u) {
            sum += hs * acc;
            acc = 0;
        }
    }

    __device__ __forceinline__ void flush(const ListParams& P) {
        const unsigned long long c = warp_sum64(cnt);
        if (lane_id() == 0 && c) atomicAdd(&P.acc[0], c);
        if constexpr ((F & F_CHECKSUM) != 0u) {
            const unsigned long long s = warp_sum64(sum);
            if (lane_id() == 0) atomicAdd(&P.acc[1], s);
        }
    }
};

// ---- row streaming -------------------------------------------------------------
// Out-rows are padded to whole 16-byte quads (pad slots hold kNone, which
// never hits), so long rows are read as 128-element CHUNKS of quads: lane l
// loads quad qb + l (ld.global.nc.v4: four elements), a warp load is 512
// contiguous bytes, and four chunks' loads are issued back to back in one asm
// block (ldg4q): a warp keeps 2 KB in flight. Lanes past the row's last quad
// are predicated off and their bits masked. The chunks come from a Cursor
// (rows held by the lanes, or a CTA's shared row table), four at a time; one
// batch may span several rows.
constexpr uint32_t kLongRow = 96;  // rows at least this long are read in quad chunks
constexpr int kQU = 4;             // chunks per batch

struct Chunk {
    uint32_t qb;  // first quad (global quad index into out_adj)
    uint32_t nq;  // quads of the row in this chunk (0 = no chunk)
    uint32_t x;   // row owner (sinks)
};

// chunks of a row of nqr quads
__device__ __forceinline__ uint32_t row_chunks(uint32_t nqr) { return (nqr + 31u) >> 5; }

template <int ALGO, unsigned F, bool kSparse, class Probe, class Cursor>
__device__ __forceinline__ void stream_quads(const ListParams& P, uint32_t seed, Cursor& cur, const Probe& probe,
                                             Sink<ALGO, F>& sink, unsigned& hits) {
    const unsigned lane = lane_id();
    const uint4* const quads = reinterpret_cast<const uint4*>(P.out_adj);
    // chunks per batch: 4 (2 KB in flight per warp); 2 for the buffered sinks,
    // whose batch / drain code would otherwise spill
    constexpr int QU = Sink<ALGO, F>::kBuffered ? 2 : kQU;
    uint4 y[QU];
#pragma unroll
    for (int i = 0; i < QU; ++i) y[i] = make_uint4(kNone, kNone, kNone, kNone);
    while (cur.more()) {
        Chunk ch[QU];
        cur.next(ch);
        const uint4* a[QU];
        bool pr[QU];
#pragma unroll
        for (int i = 0; i < QU; ++i) {
            pr[i] = lane < ch[i].nq;
            a[i] = quads + (ch[i].qb + lane);
        }
        ldgq<!kSparse>(a, pr, y);
        uint32_t hb[QU];
        bool any = false;
#pragma unroll
        for (int i = 0; i < QU; ++i) {
            hb[i] = probe.bit(y[i].x) | (probe.bit(y[i].y) << 1) | (probe.bit(y[i].z) << 2) | (probe.bit(y[i].w) << 3);
            hb[i] = pr[i] ? hb[i] : 0u;
            // a quad's first element is its smallest (rows sorted, pads last)
            if constexpr (Probe::low) any |= pr[i] && probe.below(y[i].x);
        }
        if constexpr (Probe::low) {
            // elements below the window: region-B candidates, verified here
            if (__any_sync(FULL, any)) {
#pragma unroll
                for (int i = 0; i < QU; ++i) {
                    if (!__any_sync(FULL, pr[i] && probe.below(y[i].x))) continue;
                    const uint32_t e[4] = {y[i].x, y[i].y, y[i].z, y[i].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool c = pr[i] && probe.below(e[k]) && probe.cand(e[k]);
                        if (__any_sync(FULL, c))
                            if (probe.verify(e[k], c)) hb[i] |= 1u << k;
                    }
                }
            }
        }
        uint32_t hm = 0;
#pragma unroll
        for (int i = 0; i < QU; ++i) hm |= hb[i] << (4 * i);
        hits += __popc(hm);
        if constexpr (Sink<ALGO, F>::kBuffered) {
            if (__any_sync(FULL, hm != 0)) {
#pragma unroll
                for (int i = 0; i < QU; ++i) {
                    if (__any_sync(FULL, hb[i] != 0)) {
                        sink.batch(hb[i] & 1u, ch[i].x, y[i].x);
                        sink.batch(hb[i] & 2u, ch[i].x, y[i].y);
                        sink.drain(P, seed);
                        sink.batch(hb[i] & 4u, ch[i].x, y[i].z);
                        sink.batch(hb[i] & 8u, ch[i].x, y[i].w);
                        sink.drain(P, seed);
                    }
                }
            }
        } else if constexpr (Sink<ALGO, F>::kFastSum) {
            // per chunk: sum over its hits y of h(y), then one multiply by
            // h(s) h(x). Straight-line predicated gathers (hub ranks: L1/L2
            // hits), all in flight before the first use.
            if (__any_sync(FULL, hm != 0)) {
                // hv base held in a register (else it is re-read from the
                // constant bank per predicated load); lanes without a hit
                // read hv[n] = 0, so the loads need no predicate
                const unsigned long long* hv;
                asm("mov.b64 %0, %1;" : "=l"(hv) : "l"(P.hv));
                const uint32_t zero = P.n;
                unsigned long long sy[QU];
#pragma unroll
                for (int i = 0; i < QU; ++i) {
                    const unsigned long long a0 = __ldg(hv + ((hb[i] & 1u) ? y[i].x : zero));
                    const unsigned long long a1 = __ldg(hv + ((hb[i] & 2u) ? y[i].y : zero));
                    const unsigned long long a2 = __ldg(hv + ((hb[i] & 4u) ? y[i].z : zero));
                    const unsigned long long a3 = __ldg(hv + ((hb[i] & 8u) ? y[i].w : zero));
                    sy[i] = (a0 + a1) + (a2 + a3);
                }
#pragma unroll
                for (int i = 0; i < QU; ++i)
                    if (hb[i]) sink.acc += sy[i] * __ldg(hv + ch[i].x);
            }
        }
    }
}

// Rows held by the lanes (lane j: row of x_j, first quad q0, nqr quads); the
// cursor visits the rows selected by `mask` in lane order, chunk by chunk.
// N chunks of one row are handed out at once when the row has them left.
struct LaneRowCursor {
    uint32_t q0l, nql, xl;  // this lane's row
    unsigned left;          // rows not started yet
    uint32_t q0, nqr, x, c, nch;  // current row (uniform)
    bool on;
    __device__ __forceinline__ LaneRowCursor(uint32_t q0_, uint32_t nq_, uint32_t x_, unsigned mask)
        : q0l(q0_), nql(nq_), xl(x_), left(mask), q0(0), nqr(0), x(0), c(0), nch(0), on(false) {
        advance();
    }
    __device__ __forceinline__ void advance() {
        on = left != 0;
        if (!on) return;
        const int j = __ffs(left) - 1;
        left &= left - 1;
        q0 = __shfl_sync(FULL, q0l, j);
        nqr = __shfl_sync(FULL, nql, j);
        x = __shfl_sync(FULL, xl, j);
        c = 0;
        nch = row_chunks(nqr);
    }
    __device__ __forceinline__ bool more() const { return on; }
    __device__ __forceinline__ Chunk at(uint32_t cc) const { return Chunk{q0 + 32u * cc, min(32u, nqr - 32u * cc), x}; }
    template <int N>
    __device__ __forceinline__ void next(Chunk (&ch)[N]) {
        if (c + N <= nch) {  // fast path: N chunks of the current row
#pragma unroll
            for (int i = 0; i < N; ++i) ch[i] = at(c + i);
            c += N;
            if (c == nch) advance();
            return;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (on) {
                ch[i] = at(c);
                if (++c == nch) advance();
            } else {
                ch[i] = Chunk{0, 0, 0};
            }
        }
    }
};

// A warp's contiguous range [g, ge) of a CTA seed's chunks (shared row table
// {first quad, quads, first chunk, x}), walked forward row by row.
struct CtaRowCursor {
    unsigned rows;
    uint32_t g, ge, i, rend;
    uint4 r;  // current row's entry
    __device__ __forceinline__ CtaRowCursor(unsigned rows_, uint32_t d, uint32_t gb, uint32_t ge_)
        : rows(rows_), g(gb), ge(ge_) {
        uint32_t lo = 0, hi = d - 1;
        while (lo < hi) {  // last row i with first_chunk(i) <= gb
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (lds32(rows + 16u * mid + 8u) <= gb) lo = mid;
            else hi = mid - 1;
        }
        i = lo;
        load();
    }
    __device__ __forceinline__ void load() {
        r = lds128(rows + 16u * i);
        rend = r.z + row_chunks(r.y);
    }
    __device__ __forceinline__ bool more() const { return g < ge; }
    __device__ __forceinline__ Chunk at(uint32_t gg) const {
        const uint32_t cc = gg - r.z;
        return Chunk{r.x + 32u * cc, min(32u, r.y - 32u * cc), r.w};
    }
    template <int N>
    __device__ __forceinline__ void next(Chunk (&ch)[N]) {
        if (g + N <= rend && g + N <= ge) {  // fast path: N chunks of the current row
#pragma unroll
            for (int k = 0; k < N; ++k) ch[k] = at(g + k);
            g += N;
            return;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (g < ge) {
                while (g >= rend) {
                    ++i;
                    load();
                }
                ch[k] = at(g);
                ++g;
            } else {
                ch[k] = Chunk{0, 0, 0};
            }
        }
    }
};

// Walk the out-rows of up to 32 x's (x valid on lanes with xvalid), probing
// every element y against the seed's set:
//   1. rows of >= kLongRow elements as quad chunks (stream_quads);
//   2. shorter rows as ONE flattened stream (lane f of a window reads
//      element f of the concatenated rows; the owning row of each lane comes
//      from an OR-reduction of the row starts), so short rows do not idle lanes.
template <int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void scan_rows(const ListParams& P, uint32_t seed, uint32_t x, bool xvalid,
                                          const Probe& probe, Sink<ALGO, F>& sink) {
    const unsigned lane = lane_id();
    uint64_t ro = 0;
    uint32_t rl = 0;
    if (xvalid) {
        ro = P.out_off[x];
        rl = P.out_len[x];
    }
    unsigned hits = 0;
    // ---- phase 1: long rows, quad chunks
    {
        LaneRowCursor cur(static_cast<uint32_t>(ro >> 2), (rl + 3u) >> 2, x, __ballot_sync(FULL, rl >= kLongRow));
        stream_quads<ALGO, F, true>(P, seed, cur, probe, sink, hits);
    }
    if (rl >= kLongRow) rl = 0;
    // ---- phase 2: short rows
    const unsigned ne = __ballot_sync(FULL, rl != 0);
    if (!ne) {
        sink.cnt += hits;
        return;
    }
    // compact non-empty rows to the low lanes
    const int cnt = __popc(ne);
    const int src = lane < (unsigned)cnt ? (int)__fns(ne, 0, lane + 1) : 0;
    const uint32_t cx = __shfl_sync(FULL, x, src);
    const uint64_t cro = shfl64(ro, src);
    uint32_t crl = __shfl_sync(FULL, rl, src);
    if (lane >= (unsigned)cnt) crl = 0;
    const uint32_t incl = warp_incl_scan(crl);
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    const uint32_t start = incl - crl;
    const uint64_t rbase = cro - start;  // element f of the stream lives at out_adj[rbase(row) + f]
    const unsigned le = lanemask_le();
    int before = 0;
    // two 32-wide windows per iteration: both loads are in flight before the
    // first probe
    for (uint32_t base = 0; base < total; base += 64) {
        const uint32_t rel = start - base;  // wraps when start < base: no bit
        const unsigned bitA = (crl != 0 && start >= base && rel < 32u) ? (1u << rel) : 0u;
        const unsigned bitB = (crl != 0 && start >= base && rel - 32u < 32u) ? (1u << (rel - 32u)) : 0u;
        const unsigned MA = __reduce_or_sync(FULL, bitA);
        const unsigned MB = __reduce_or_sync(FULL, bitB);
        const int ca = __popc(MA);
        int jA = before + __popc(MA & le) - 1;
        int jB = before + ca + __popc(MB & le) - 1;
        before += ca + __popc(MB);
        jA = jA > 31 ? 31 : jA;
        jB = jB > 31 ? 31 : jB;
        const uint32_t fA = base + lane, fB = fA + 32;
        const bool actA = fA < total, actB = fB < total;
        const uint64_t rbA = shfl64(rbase, jA);
        const uint64_t rbB = shfl64(rbase, jB);
        const uint32_t yA = actA ? __ldg(P.out_adj + rbA + fA) : kNone;
        const uint32_t yB = actB ? __ldg(P.out_adj + rbB + fB) : kNone;
        const bool hitA = probe_one(probe, yA, actA);
        const bool hitB = probe_one(probe, yB, actB);
        hits += (unsigned)hitA + (unsigned)hitB;
        if constexpr (Sink<ALGO, F>::kBuffered || Sink<ALGO, F>::kFastSum) {
            const uint32_t xA = __shfl_sync(FULL, cx, jA), xB = __shfl_sync(FULL, cx, jB);
            if constexpr (Sink<ALGO, F>::kBuffered) {
                sink.batch(hitA, xA, yA);
                sink.batch(hitB, xB, yB);
                sink.drain(P, seed);
            } else {
                sink.direct(P, hitA, xA, yA);
                sink.direct(P, hitB, xB, yB);
            }
        }
    }
    sink.cnt += hits;
}

// Chunks of 32 x's: set elements c, c + stride, ... below xe of the seed row at so.
template <int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void scan_x_range(const ListParams& P, uint32_t seed, uint64_t so, uint32_t cb,
                                             uint32_t xe, uint32_t stride, const Probe& probe, Sink<ALGO, F>& sink) {
    const unsigned lane = lane_id();
    for (uint32_t c = cb; c < xe; c += stride) {
        const bool xv = c + lane < xe;
        const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
        scan_rows<ALGO, F>(P, seed, x, xv, probe, sink);
    }
}

// Run body(probe) with the seed's bitmap: window only, or window + region B.
template <class V, class Body>
__device__ __forceinline__ void with_win_probe(const ListParams& P, unsigned bma, unsigned bmb, const WinGeom& g,
                                               const V& ver, Body&& body) {
#ifdef TRIGPU_EXPERIMENTS
    if (P.variant == 2) {
        body(NullProbe{});
        return;
    }
#endif
    if (!g.low) body(WinProbe<false, V>{bma, bmb, g.wb, g.la, g.maskb, ver});
    else body(WinProbe<true, V>{bma, bmb, g.wb, g.la, g.maskb, ver});
}

// ---- per-warp scratch in dynamic shared memory ------------------------------
// [warps x kHitBuf uint2 hit buffers (buffered sinks only)] followed by the
// kernel's bitmaps.
template <unsigned F>
__host__ __device__ constexpr size_t warp_scratch_bytes(int warps) {
    return (F & (F_VCOUNT | F_LIST)) ? static_cast<size_t>(warps) * kHitBuf * 8 : 0;
}

template <int ALGO, unsigned F>
__device__ __forceinline__ void attach_scratch(Sink<ALGO, F>& sink, unsigned char* base) {
    sink.buf = smem_addr(base + (threadIdx.x >> 5) * kHitBuf * 8);
}

// CTAs per SM of the warp-class kernels: 4 (64 registers) for count only; the
// sinks need more registers (3 CTAs, 80 registers) or they spill in the hot loop
#ifndef TRIGPU_WARP_MINB
#define TRIGPU_WARP_MINB 4
#endif
#ifndef TRIGPU_WARP_MINB_SINK
#define TRIGPU_WARP_MINB_SINK 3
#endif
#define WARP_MINB(F) ((F) == 0u ? TRIGPU_WARP_MINB : TRIGPU_WARP_MINB_SINK)

// ---- class R: |S| <= 32, warp per seed --------------------------------------
constexpr int kRWarps = 8;
#ifndef TRIGPU_R_BITS_A
#define TRIGPU_R_BITS_A 15
#endif
constexpr uint32_t kRBitsA = TRIGPU_R_BITS_A, kRBitsB = 11;  // 4 KB window + 256 B region B per warp
constexpr size_t kRBmBytes = win_bytes(kRBitsA, kRBitsB);

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kRWarps * 32, TRIGPU_WARP_MINB) k_list_reg(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t* bma = reinterpret_cast<uint32_t*>(dsm + warp_scratch_bytes<F>(kRWarps) + warp * kRBmBytes);
    uint32_t* bmb = bma + ((1u << kRBitsA) / 32 + 4);
    for (uint32_t i = lane; i < kRBmBytes / 4; i += 32) bma[i] = 0u;
    __syncwarp();
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        sink.begin_unit(P, seed);
        const uint64_t so = P.set_off[seed];
        const uint32_t d = P.set_len[seed];
        const uint32_t s = lane < d ? __ldg(P.set_adj + so + lane) : kNone;
        const WinGeom g = win_geom(kRBitsA, kRBitsB, P.bm_shrink, __shfl_sync(FULL, s, 0), __shfl_sync(FULL, s, d - 1));
        if (lane < d) win_set(bma, bmb, g, s);
        __syncwarp();
        with_win_probe(P, smem_addr(bma), smem_addr(bmb), g, RegVerify{s}, [&](const auto& probe) {
            scan_rows<ALGO, F>(P, seed, s, lane < d, probe, sink);
        });
        sink.end_unit(P, seed);
        __syncwarp();
        if (lane < d) win_clear(bma, bmb, g, s);
        __syncwarp();
    }
    sink.flush(P);
}

// ---- class H: 32 < |S| <= 256, warp per seed --------------------------------
constexpr int kHWarps = 8;
#ifndef TRIGPU_H_BITS_A
#define TRIGPU_H_BITS_A 16
#endif
constexpr uint32_t kHBitsA = TRIGPU_H_BITS_A, kHBitsB = 13;  // 8 KB window + 1 KB region B per warp
constexpr size_t kHBmBytes = win_bytes(kHBitsA, kHBitsB);

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kHWarps * 32, WARP_MINB(F)) k_list_warp(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t* bma = reinterpret_cast<uint32_t*>(dsm + warp_scratch_bytes<F>(kHWarps) + warp * kHBmBytes);
    uint32_t* bmb = bma + ((1u << kHBitsA) / 32 + 4);
    for (uint32_t i = lane; i < kHBmBytes / 4; i += 32) bma[i] = 0u;
    __syncwarp();
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        sink.begin_unit(P, seed);
        const uint64_t so = P.set_off[seed];
        const uint32_t d = P.set_len[seed];
        const uint32_t* row = P.set_adj + so;
        const WinGeom g = win_geom(kHBitsA, kHBitsB, P.bm_shrink, __ldg(row), __ldg(row + d - 1));
        for (uint32_t k = lane; k < d; k += 32) win_set(bma, bmb, g, __ldg(row + k));
        __syncwarp();
        with_win_probe(P, smem_addr(bma), smem_addr(bmb), g, RowVerify{row, d}, [&](const auto& probe) {
            scan_x_range<ALGO, F>(P, seed, so, 0, d, 32, probe, sink);
        });
        sink.end_unit(P, seed);
        __syncwarp();
        for (uint32_t k = lane; k < d; k += 32) win_clear(bma, bmb, g, __ldg(row + k));
        __syncwarp();
    }
    sink.flush(P);
}

// ---- class C: 256 < |S| <= 4096, CTA per seed ----------------------------------
// All warps of the CTA share the seed's bitmap. The seed's rows are cut into
// chunks (chunk prefix over the set in a shared row table) and split equally
// across the warps, so the CTA barrier at the end of a seed waits for
// balanced work. Two sizes: C1 (256 < |S| <= 1024) runs 8-warp CTAs, several
// per SM, so one CTA's seed barrier is hidden by the others; C2 (1024 < |S| <=
// 4096) runs one 32-warp CTA per SM.
template <int THREADS, uint32_t BITS_A, uint32_t BITS_B, uint32_t MAXD, int MINB>
struct CtaCfg {
    static constexpr int kThreads = THREADS;
    static constexpr int kWarps = THREADS / 32;
    static constexpr uint32_t kBitsA = BITS_A;  // window of 2^BITS_A ranks
    static constexpr uint32_t kBitsB = BITS_B;  // region B of 2^BITS_B bits
    static constexpr uint32_t kMaxD = MAXD;
    static constexpr int kMinBlocks = MINB;
};
using CfgC1 = CtaCfg<256, 18, 14, 1024, 3>;  // (2^17 window at 4 CTAs/SM: C4 -1 %, C5 +4 %)
using CfgC2 = CtaCfg<1024, 19, 15, 4096, 1>;  // (2 x 512-thread CTAs, 2^18 window: C5 5 % slower)
template <class CFG>
constexpr size_t cta_bitmap_bytes() { return win_bytes(CFG::kBitsA, CFG::kBitsB); }
template <class CFG>
constexpr size_t cta_row_bytes() { return CFG::kMaxD * 16; }  // uint4 {first quad, quads, first chunk, x}

template <int ALGO, unsigned F, class CFG>
__global__ void __launch_bounds__(CFG::kThreads, CFG::kMinBlocks) k_list_cta(ListParams P) {
    constexpr int kCThreads = CFG::kThreads;
    constexpr uint32_t kWords = cta_bitmap_bytes<CFG>() / 4;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned unit, total_chunks;
    using BS = cub::BlockScan<uint32_t, kCThreads>;
    __shared__ typename BS::TempStorage scan_tmp;
    uint32_t* bma = reinterpret_cast<uint32_t*>(dsm + warp_scratch_bytes<F>(CFG::kWarps));
    uint32_t* bmb = bma + ((1u << CFG::kBitsA) / 32 + 4);
    const unsigned rows = smem_addr(dsm + warp_scratch_bytes<F>(CFG::kWarps) + cta_bitmap_bytes<CFG>());
    for (uint32_t i = threadIdx.x; i < kWords; i += kCThreads) bma[i] = 0u;
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    constexpr int PER = CFG::kMaxD / kCThreads;  // set elements per thread
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) unit = atomicAdd(P.queue, 1u);
        __syncthreads();
        const unsigned u = unit;
        if (u >= P.nseeds) break;
        const uint32_t seed = P.seeds[u];
        sink.begin_unit(P, seed);
        const uint64_t so = P.set_off[seed];
        const uint32_t d = P.set_len[seed];
        const uint32_t* row = P.set_adj + so;
        const WinGeom g = win_geom(CFG::kBitsA, CFG::kBitsB, P.bm_shrink, __ldg(row), __ldg(row + d - 1));
        // bitmap + row table (blocked: thread t owns set elements PER*t ..)
        uint32_t nc[PER], q0[PER], nq[PER], xs[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = threadIdx.x * PER + k;
            nc[k] = 0;
            q0[k] = 0;
            nq[k] = 0;
            xs[k] = 0;
            if (i < d) {
                const uint32_t x = __ldg(row + i);
                win_set(bma, bmb, g, x);
                xs[k] = x;
                q0[k] = static_cast<uint32_t>(P.out_off[x] >> 2);
                nq[k] = (P.out_len[x] + 3u) >> 2;
                nc[k] = row_chunks(nq[k]);
            }
        }
        uint32_t agg;
        BS(scan_tmp).ExclusiveSum(nc, nc, agg);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = threadIdx.x * PER + k;
            if (i < d) sts128(rows + 16u * i, make_uint4(q0[k], nq[k], nc[k], xs[k]));
        }
        if (threadIdx.x == 0) total_chunks = agg;
        __syncthreads();
        const uint32_t nchunks = total_chunks;
        with_win_probe(P, smem_addr(bma), smem_addr(bmb), g, RowVerify{row, d}, [&](const auto& probe) {
            // equal, contiguous share of the seed's chunks per warp (measured
            // faster than claiming runs of 8 chunks from a shared counter)
            const unsigned warp = threadIdx.x >> 5;
            const uint32_t gb = static_cast<uint32_t>((static_cast<uint64_t>(nchunks) * warp) / CFG::kWarps);
            const uint32_t ge = static_cast<uint32_t>((static_cast<uint64_t>(nchunks) * (warp + 1)) / CFG::kWarps);
            if (gb < ge) {
                CtaRowCursor cur(rows, d, gb, ge);
                unsigned hits = 0;
                stream_quads<ALGO, F, false>(P, seed, cur, probe, sink, hits);
                sink.cnt += hits;
            }
        });
        sink.end_unit(P, seed);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < d; k += kCThreads) win_clear(bma, bmb, g, __ldg(row + k));
    }
    sink.flush(P);
}

// ---- class G: |S| > 4096, CTA per seed, global bitmap --------------------
constexpr int kGThreads = 512;
constexpr int kGWarps = kGThreads / 32;

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kGThreads) k_list_giant(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned unit;
    const unsigned warp = threadIdx.x >> 5;
    uint32_t* bm = P.bitmaps + (uint64_t)blockIdx.x * P.bitmap_words;
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) unit = atomicAdd(P.queue, 1u);
        __syncthreads();
        const unsigned u = unit;
        if (u >= P.nseeds) break;
        const uint32_t seed = P.seeds[u];
        sink.begin_unit(P, seed);
        const uint64_t so = P.set_off[seed];
        const uint32_t d = P.set_len[seed];
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(P.set_adj + so + k);
            atomicOr(bm + (v >> 5), 1u << (v & 31));
        }
        __syncthreads();
        const BitmapProbe probe{bm, P.n};
        scan_x_range<ALGO, F>(P, seed, so, warp * 32, d, kGWarps * 32, probe, sink);
        sink.end_unit(P, seed);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(P.set_adj + so + k);
            __stcg(bm + (v >> 5), 0u);
        }
    }
    sink.flush(P);
}

// dynamic shared memory per CTA of each class kernel
template <unsigned F> constexpr size_t smem_reg() { return warp_scratch_bytes<F>(kRWarps) + kRWarps * kRBmBytes; }
template <unsigned F> constexpr size_t smem_warp() { return warp_scratch_bytes<F>(kHWarps) + kHWarps * kHBmBytes; }
template <unsigned F, class CFG> constexpr size_t smem_cta() { return warp_scratch_bytes<F>(CFG::kWarps) + cta_bitmap_bytes<CFG>() + cta_row_bytes<CFG>(); }
template <unsigned F> constexpr size_t smem_giant() { return warp_scratch_bytes<F>(kGWarps); }

// ---- seed classification --------------------------------------------------
constexpr int kClasses = 5;  // R, H, C1, C2, G

struct SeedLists {
    uint32_t* lists[kClasses];
    unsigned int* counts;     // [kClasses]
};

__global__ void __launch_bounds__(256) k_classify_seeds(uint32_t n, const uint32_t* __restrict__ set_len,
                                                        SeedLists L) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t start = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t trips = (n + stride - 1) / stride;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t r = start + t * stride;
        uint64_t d = 0;
        if (r < n) d = set_len[r];
        int cls = -1;
        if (d >= 2) cls = d <= 32 ? 0 : d <= 256 ? 1 : d <= CfgC1::kMaxD ? 2 : d <= CfgC2::kMaxD ? 3 : 4;
#pragma unroll
        for (int c = 0; c < kClasses; ++c) {
            const unsigned b = __ballot_sync(FULL, cls == c);
            if (!b) continue;
            const unsigned leader = __ffs(b) - 1;
            unsigned base = 0;
            if (lane_id() == leader) base = atomicAdd(&L.counts[c], __popc(b));
            base = __shfl_sync(FULL, base, leader);
            if (cls == c) L.lists[c][base + __popc(b & lanemask_lt())] = (uint32_t)r;
        }
    }
}

}  // namespace trigpu
