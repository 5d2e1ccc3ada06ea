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
//   class H  32 < |S| <= 256    warp per seed, 2^16-bit window per warp; on graphs
//                               of more than 2^21 vertices only up to |S| = 96, the
//                               larger sets on a CTA (16 warps) per seed, 2^19 window
//   class C1 256 < |S| <= 1024  CTA (16 warps) per seed, 2^18-bit window (2^19 above
//                               2^25 vertices)
//   class C2 1024 < |S| <= 4096 CTA (32 warps) per seed, 2^19-bit window
//   class G  |S| > 4096         CTA per seed, 2^20-bit window + coarse filter in
//                               shared memory over an exact n-bit bitmap in global memory
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
    unsigned long long* acc;  // [0] triangles, [1] checksum, [2] list chunk cursor, [3] list holes
    unsigned long long* vcount;  // rank space
    uint32_t* tri;
    unsigned long long tri_cap;
    ulonglong2* holes;        // unused tails of the warps' last list chunks {start, length}
    unsigned holes_cap;
    const uint32_t* seeds;    // class list
    unsigned int nseeds;
    unsigned int* queue;      // dynamic work counter
    uint32_t* bitmaps;        // class G only: one n-bit bitmap per CTA
    uint64_t bitmap_words;
    uint32_t hot_rank;        // rows of ranks >= hot_rank (the most re-read ones) are loaded evict_last
    uint32_t hist_base;       // per-vertex counts of ranks >= hist_base are kept per CTA in shared memory
    int r_search;             // class R: shuffle search instead of the bitmap for sets wider than the window
                              //   (set when the graph has no long rows at all, see k_list_reg)
    int variant;              // TL_DEBUG_VARIANT: 2 = null probe (experiments build, timing only)
    uint32_t bm_shrink;       // TL_DEBUG_BM_SHRINK: smaller windows (tests force the below-window path)
};

// Per-warp hit buffer (per-vertex-count and list sinks): hits (x, y) are
// compacted into shared memory by a ballot and emitted 32 at a time with
// every lane busy (dense-id gathers, atomics) instead of with the 1-3 lanes
// that hit in a batch.
constexpr int kHitBuf = 96;  // 31 pending + up to 2 batches of 32 before a drain
constexpr unsigned kListChunk = 1024;  // list slots a warp claims per global atomic

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
        return (lds32(bit_word(bm, o)) >> (o & 31u)) & 1u;
    }
    __device__ __forceinline__ bool below(uint32_t y) const { return y < wb; }
    // region-B candidate (call for y below the window only)
    __device__ __forceinline__ uint32_t cand(uint32_t y) const {
        const uint32_t o = y & maskb;
        return (lds32(bit_word(bmb, o)) >> (o & 31u)) & 1u;
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

// Class R seeds whose set is wider than the window, on graphs without long rows
// (max d+ < kLongRow: lattice-like graphs): the 5-step shuffle search over S
// (one key per lane) answers every probe exactly, so the seed needs no bitmap
// at all - no set / clear and no filter + verification round, which on a
// Watts-Strogatz graph (sets spread over all ranks, a third of the probes
// hitting) ran for nearly every window: C3 count 12.8 -> 10.0 ms. On
// power-law graphs hits are rare, the filter almost never fires and the
// bitmap stays cheaper (C5 class R 320 vs 339 ms with the search), so the
// switch is per graph.
struct SearchProbe {
    static constexpr bool low = false;
    RegVerify ver;
    __device__ __forceinline__ uint32_t bit(uint32_t y) const { return ver(y, true); }
    __device__ __forceinline__ bool below(uint32_t) const { return false; }
    __device__ __forceinline__ uint32_t cand(uint32_t) const { return 0u; }
    __device__ __forceinline__ bool verify(uint32_t, bool act) const { return act; }
    __device__ __forceinline__ uint32_t sentinel() const { return kNone; }
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
    const uint32_t b = probe.bit(y);  // evaluated by every lane (SearchProbe shuffles)
    bool hit = act && b;
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
// Lists go through the warp's hit buffer (emit). Per-vertex counts are added
// where the hits are found: one atomic per chunk for its row owner x (all of
// a chunk's hits share x), one per hit for y, and one per seed; counts of the
// top kHist ranks (the hubs, which most hits land on under degree order) go
// to a per-CTA shared-memory histogram flushed once at the end of the kernel,
// the rest to global memory.
constexpr uint32_t kHist = 4096;
template <int ALGO, unsigned F>
struct Sink {
    static constexpr bool kFastSum = (F & F_CHECKSUM) != 0u && (F & F_LIST) == 0u;
    static constexpr bool kBuffered = (F & F_LIST) != 0u;
    unsigned long long cnt = 0, sum = 0;
    unsigned long long hs = 0;    // h(seed)
    unsigned long long acc = 0;   // this seed's sum of h(x) h(y); times h(s) at end_unit
    unsigned seed_hits = 0;
    unsigned buf = 0;      // shared address of this warp's kHitBuf uint2 entries
    unsigned pending = 0;  // warp-uniform
    unsigned long long lcur = 0, lend = 0;  // the warp's list chunk: next slot, end (warp-uniform)
    uint32_t* hist = nullptr;  // the CTA's kHist counters (F_VCOUNT)

    // c more triangles containing vertex v (rank)
    __device__ __forceinline__ void vc_add(const ListParams& P, uint32_t v, unsigned c) {
        if constexpr ((F & F_VCOUNT) != 0u) {
            if (v >= P.hist_base) atomicAdd(hist + (v - P.hist_base), c);
            else atomicAdd(&P.vcount[v], (unsigned long long)c);
        }
    }

    __device__ __forceinline__ void begin_unit(const ListParams& P, uint32_t seed) {
        if constexpr ((F & F_CHECKSUM) != 0u) hs = __ldg(P.hv + seed);
    }

    // One hit with its own x (short-row stream).
    __device__ __forceinline__ void direct(const ListParams& P, bool hit, uint32_t x, uint32_t y) {
        if constexpr (kFastSum)
            if (hit) acc += __ldg(P.hv + x) * __ldg(P.hv + y);
        if constexpr ((F & F_VCOUNT) != 0u) {
            if (hit) {
                vc_add(P, x, 1);
                vc_add(P, y, 1);
            }
            seed_hits += hit;
        }
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
        if constexpr ((F & F_CHECKSUM) != 0u)
            if (hit) acc += __ldg(P.hv + x) * __ldg(P.hv + y);
        if constexpr ((F & F_LIST) != 0u) {
            const uint32_t ru = ALGO == ALGO_APM ? seed : x;
            const uint32_t rv = ALGO == ALGO_APM ? x : y;
            const uint32_t rw = ALGO == ALGO_APM ? y : seed;
            // slots from the warp's own chunk of kListChunk, a new chunk (one
            // global atomic) when it runs out; a batch may straddle two chunks
            const unsigned long long base0 = lcur;
            const unsigned r = static_cast<unsigned>(min(lend - lcur, (unsigned long long)n));
            unsigned long long base1 = 0;
            if (r < n) {
                if (lane == 0) base1 = atomicAdd(&P.acc[2], (unsigned long long)kListChunk);
                base1 = __shfl_sync(FULL, base1, 0);
                lcur = base1 + (n - r);
                lend = base1 + kListChunk;
            } else {
                lcur += n;
            }
            if (hit) {
                const unsigned long long k = lane < r ? base0 + lane : base1 + (lane - r);
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
        if constexpr ((F & F_LIST) != 0u) {
            // the unused tail of the last chunk: recorded, filled after the
            // listing by moving triangles from the end (tl_list)
            if (lane_id() == 0 && lend > lcur) {
                const unsigned long long h = atomicAdd(&P.acc[3], 1ull);
                if (h < P.holes_cap) P.holes[h] = make_ulonglong2(lcur, lend - lcur);
            }
        }
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
#ifndef TRIGPU_L2HINT
#define TRIGPU_L2HINT 0
#endif
#ifndef TRIGPU_CKS
#define TRIGPU_CKS 0
#endif
constexpr uint32_t kLongRow = 96;  // rows at least this long are read in quad chunks
constexpr uint32_t kSlotBytes = 512;  // one chunk (32 quads) in a shared-memory stage
constexpr int kQU = 4;             // chunks per batch
#ifndef TRIGPU_SHORT_W
#define TRIGPU_SHORT_W 2  // (4: C3 -4 %, class R on C4 +3 %, per-vertex counts on C2 +8 %; 8: C3 +30 %)
#endif
constexpr int kShortW = TRIGPU_SHORT_W;  // 32-wide windows of the short-row stream per iteration

struct Chunk {
    uint32_t qb;  // first quad (global quad index into out_adj)
    uint32_t nq;  // quads of the row in this chunk (0 = no chunk)
    uint32_t x;   // row owner (sinks)
};

// chunks of a row of nqr quads
__device__ __forceinline__ uint32_t row_chunks(uint32_t nqr) { return (nqr + 31u) >> 5; }

// Probe QU quads (one per chunk, lane l holding quad l of each) against the
// seed's set and feed the hits to the sink. pr[i]: the lane's quad i is part
// of chunk i; ch[i].x owns chunk i.
template <int QU, int ALGO, unsigned F, class Probe, bool kStaged = false>
__device__ __forceinline__ void probe_quads(const ListParams& P, uint32_t seed, const Chunk (&ch)[QU], const bool (&pr)[QU],
                                            const uint4 (&y)[QU], const Probe& probe, Sink<ALGO, F>& sink,
                                            unsigned& hits, unsigned stage = 0) {
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
    if constexpr ((F & F_VCOUNT) != 0u) {
        sink.seed_hits += __popc(hm);
        if (__any_sync(FULL, hm != 0)) {
#pragma unroll
            for (int i = 0; i < QU; ++i) {  // x side: one atomic per chunk
                const unsigned c = __reduce_add_sync(FULL, __popc(hb[i]));
                if (lane_id() == 0 && c) sink.vc_add(P, ch[i].x, c);
            }
#pragma unroll
            for (int i = 0; i < QU; ++i) {  // y side: per hit
                if (hb[i] & 1u) sink.vc_add(P, y[i].x, 1);
                if (hb[i] & 2u) sink.vc_add(P, y[i].y, 1);
                if (hb[i] & 4u) sink.vc_add(P, y[i].z, 1);
                if (hb[i] & 8u) sink.vc_add(P, y[i].w, 1);
            }
        }
    }
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
    } else if constexpr (Sink<ALGO, F>::kFastSum && kStaged) {
        // the chunks sit in shared memory (the stage): walk each lane's hit
        // bits, reading the hit element back from the stage, so only hits
        // cost gathers (a warp iterates max over lanes of its hit count,
        // ~3, instead of once per element slot)
        if (__any_sync(FULL, hm != 0)) {
            const unsigned long long* hv;
            asm("mov.b64 %0, %1;" : "=l"(hv) : "l"(P.hv));
            unsigned long long hx[QU];
#pragma unroll
            for (int i = 0; i < QU; ++i) hx[i] = __ldg(hv + ch[i].x);
            unsigned long long a = 0;
            uint32_t b = hm;
            const unsigned lane16 = stage + 16u * lane_id();
            while (__any_sync(FULL, b != 0)) {
                if (b) {
                    const uint32_t bit = __ffs(b) - 1;
                    b &= b - 1;
                    const uint32_t i = bit >> 2;
                    const uint32_t yv = lds32(lane16 + i * kSlotBytes + 4u * (bit & 3u));
                    unsigned long long h = hx[0];
#pragma unroll
                    for (int j = 1; j < QU; ++j) h = i == (uint32_t)j ? hx[j] : h;
                    a += h * __ldg(hv + yv);
                }
            }
            sink.acc += a;
        }
    } else if constexpr (Sink<ALGO, F>::kFastSum) {
        // per chunk: sum over its hits y of h(y), then one multiply by
        // h(s) h(x). Straight-line gathers (hub ranks: L1/L2 hits), all in
        // flight before the first use.
        if (__any_sync(FULL, hm != 0)) {
            // hv base held in a register (else it is re-read from the
            // constant bank per predicated load)
            const unsigned long long* hv;
            asm("mov.b64 %0, %1;" : "=l"(hv) : "l"(P.hv));
            unsigned long long sy[QU];
#if TRIGPU_CKS == 1
            // conditional loads: only hit lanes generate memory requests
#pragma unroll
            for (int i = 0; i < QU; ++i) {
                unsigned long long a = 0;
                if (hb[i] & 1u) a += __ldg(hv + y[i].x);
                if (hb[i] & 2u) a += __ldg(hv + y[i].y);
                if (hb[i] & 4u) a += __ldg(hv + y[i].z);
                if (hb[i] & 8u) a += __ldg(hv + y[i].w);
                sy[i] = a;
            }
#pragma unroll
            for (int i = 0; i < QU; ++i)
                if (hb[i]) sink.acc += sy[i] * __ldg(hv + ch[i].x);
#else
            // lanes without a hit read hv[n] = 0, so the loads need no predicate
            const uint32_t zero = P.n;
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
#endif
        }
    }
}

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
#if TRIGPU_L2HINT
    const uint64_t pol_last = l2_policy_last(), pol_first = l2_policy_first();
#endif
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
#if TRIGPU_L2HINT
        uint64_t pol[QU];
#pragma unroll
        for (int i = 0; i < QU; ++i) pol[i] = ch[i].x >= P.hot_rank ? pol_last : pol_first;
        ldgq_pol<!kSparse>(a, pr, pol, y);
#else
        ldgq<!kSparse>(a, pr, y);
#endif
        probe_quads<QU>(P, seed, ch, pr, y, probe, sink, hits);
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

// Chunks [c, ce) of ONE row (a CTA's warps sharing a giant row).
struct RowRangeCursor {
    uint32_t q0, nqr, x, c, ce;
    __device__ __forceinline__ bool more() const { return c < ce; }
    template <int N>
    __device__ __forceinline__ void next(Chunk (&ch)[N]) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (c < ce) {
                ch[i] = Chunk{q0 + 32u * c, min(32u, nqr - 32u * c), x};
                ++c;
            } else {
                ch[i] = Chunk{0, 0, 0};
            }
        }
    }
};

// Rows a warp does not stream itself: the class G kernel collects the giant
// rows of a seed (>= kDeferQuads quads) in a shared list and its 32 warps
// stream each of them together afterwards - a single warp walking a
// million-element hub row is what the rest of the CTA waits for at the seed's
// barrier (ncu, C4 split order: barrier stall 10 per issue).
constexpr uint32_t kDeferQuads = 4096;  // 16 K elements: 128 chunks, one batch per warp
constexpr uint32_t kDeferCap = 1024;    // rows per seed; a full list falls back to the warp's own walk
struct NoDefer {
    static constexpr bool enabled = false;
    __device__ __forceinline__ bool push(uint32_t, uint32_t, uint32_t) const { return false; }
};
struct SharedRowList {
    static constexpr bool enabled = true;
    unsigned rows;        // shared address of kDeferCap uint4 {first quad, quads, x, -}
    unsigned int* count;  // shared counter
    __device__ __forceinline__ bool push(uint32_t q0, uint32_t nq, uint32_t x) const {
        const unsigned slot = atomicAdd(count, 1u);
        if (slot >= kDeferCap) return false;
        sts128(rows + 16u * slot, make_uint4(q0, nq, x, 0u));
        return true;
    }
};

// Walk the out-rows of up to 32 x's (x valid on lanes with xvalid), probing
// every element y against the seed's set:
//   1. rows of >= kLongRow elements as quad chunks (stream_quads);
//   2. shorter rows as ONE flattened stream (lane f of a window reads
//      element f of the concatenated rows; the owning row of each lane comes
//      from an OR-reduction of the row starts), so short rows do not idle lanes.
template <int ALGO, unsigned F, class Probe, class Defer = NoDefer>
__device__ __forceinline__ void scan_rows_at(const ListParams& P, uint32_t seed, uint32_t x, uint64_t ro, uint32_t rl,
                                             const Probe& probe, Sink<ALGO, F>& sink, const Defer& defer = Defer{}) {
    const unsigned lane = lane_id();
    unsigned hits = 0;
    // ---- phase 1: long rows, quad chunks
    {
        bool mine = rl >= kLongRow;
        if constexpr (Defer::enabled) {
            const uint32_t nq = (rl + 3u) >> 2;
            if (mine && nq >= kDeferQuads && defer.push(static_cast<uint32_t>(ro >> 2), nq, x)) mine = false;
        }
        LaneRowCursor cur(static_cast<uint32_t>(ro >> 2), (rl + 3u) >> 2, x, __ballot_sync(FULL, mine));
        stream_quads<ALGO, F, true>(P, seed, cur, probe, sink, hits);
    }
    if (rl >= kLongRow) rl = 0;
    // (A lane-per-row walk of the rows of <= 32 elements - each lane reading its own
    // row as quads - measured 35-50 % slower for class R on C2 / C3 / C4: 32
    // uncoalesced 16-byte loads per instruction cost more than the flattened
    // stream's index arithmetic.)
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
    // kShortW 32-wide windows per iteration: all their loads are in flight
    // before the first probe (a seed of short rows is latency-bound: the
    // number of dependent round trips per seed is what it costs)
    constexpr int W = Sink<ALGO, F>::kBuffered ? 2 : kShortW;
    for (uint32_t base = 0; base < total; base += 32u * W) {
        const uint32_t rel = start - base;  // wraps when start < base: no bit
        const bool own = crl != 0 && start >= base;
        int j[W];
        int acc = before;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t o = rel - 32u * w;
            const unsigned M = __reduce_or_sync(FULL, (own && o < 32u) ? (1u << o) : 0u);
            const int jj = acc + __popc(M & le) - 1;
            j[w] = jj > 31 ? 31 : jj;
            acc += __popc(M);
        }
        before = acc;
        uint32_t y[W];
        bool act[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t f = base + 32u * w + lane;
            act[w] = f < total;
            const uint64_t rb = shfl64(rbase, j[w]);
            y[w] = act[w] ? __ldg(P.out_adj + rb + f) : kNone;
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w >= 2 && base + 32u * w >= total) break;  // uniform: no element in this window
            const bool hit = probe_one(probe, y[w], act[w]);
            hits += (unsigned)hit;
            if constexpr (F != 0u) {
                const uint32_t xw = __shfl_sync(FULL, cx, j[w]);
                sink.direct(P, hit, xw, y[w]);
                if constexpr (Sink<ALGO, F>::kBuffered) {
                    sink.batch(hit, xw, y[w]);
                    if (w & 1) sink.drain(P, seed);
                }
            }
        }
    }
    sink.cnt += hits;
}

template <int ALGO, unsigned F, class Probe, class Defer = NoDefer>
__device__ __forceinline__ void scan_rows(const ListParams& P, uint32_t seed, uint32_t x, bool xvalid,
                                          const Probe& probe, Sink<ALGO, F>& sink, const Defer& defer = Defer{}) {
    uint64_t ro = 0;
    uint32_t rl = 0;
    if (xvalid) {
        ro = P.out_off[x];
        rl = P.out_len[x];
    }
    scan_rows_at<ALGO, F>(P, seed, x, ro, rl, probe, sink, defer);
}

// Chunks of 32 x's: set elements c, c + stride, ... below xe of the seed row at so.
// (Loading the next chunk's x's and row offsets ahead of the current chunk's
// streaming measured 2-3 % slower for class H on C4: the extra live registers
// cost more than the two round trips per 32 rows.)
template <int ALGO, unsigned F, class Probe, class Defer = NoDefer>
__device__ __forceinline__ void scan_x_range(const ListParams& P, uint32_t seed, uint64_t so, uint32_t cb,
                                             uint32_t xe, uint32_t stride, const Probe& probe, Sink<ALGO, F>& sink,
                                             const Defer& defer = Defer{}) {
    const unsigned lane = lane_id();
    for (uint32_t c = cb; c < xe; c += stride) {
        const bool xv = c + lane < xe;
        const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
        scan_rows<ALGO, F>(P, seed, x, xv, probe, sink, defer);
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
__host__ __device__ constexpr size_t hitbuf_bytes(int warps) {
    return (F & F_LIST) ? static_cast<size_t>(warps) * kHitBuf * 8 : 0;
}
template <unsigned F>
__host__ __device__ constexpr size_t warp_scratch_bytes(int warps) {
    return hitbuf_bytes<F>(warps) + ((F & F_VCOUNT) ? kHist * 4 : 0);
}

// Point the sink at its scratch and zero the CTA's count histogram (a CTA
// barrier: call before the work loop, from every thread).
template <int ALGO, unsigned F>
__device__ __forceinline__ void attach_scratch(Sink<ALGO, F>& sink, unsigned char* base) {
    sink.buf = smem_addr(base + (threadIdx.x >> 5) * kHitBuf * 8);
    if constexpr ((F & F_VCOUNT) != 0u) {
        sink.hist = reinterpret_cast<uint32_t*>(base + hitbuf_bytes<F>(blockDim.x >> 5));
        for (uint32_t i = threadIdx.x; i < kHist; i += blockDim.x) sink.hist[i] = 0u;
        __syncthreads();
    }
}

// After the work loop, from every thread: add the CTA's histogram to the
// global per-vertex counts.
template <int ALGO, unsigned F>
__device__ __forceinline__ void flush_hist(const ListParams& P, const Sink<ALGO, F>& sink) {
    if constexpr ((F & F_VCOUNT) != 0u) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < kHist; i += blockDim.x) {
            const uint32_t c = sink.hist[i];
            if (c) atomicAdd(&P.vcount[P.hist_base + i], (unsigned long long)c);
        }
    }
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
#ifndef TRIGPU_R_MINB_SINK
#define TRIGPU_R_MINB_SINK TRIGPU_WARP_MINB
#endif
#define R_MINB(F) ((F) == 0u ? TRIGPU_WARP_MINB : TRIGPU_R_MINB_SINK)

// ---- class R: |S| <= 32, warp per seed --------------------------------------
// The set of an R seed (<= 32 ranks) may span the whole rank range (e.g. on a
// Watts-Strogatz graph, where ranks are nearly unrelated to ring position), so
// a rank window would leave most of it to the filter + verification path. A
// per-warp open-addressing table of kRSlots keys (load <= 1/4, linear probing)
// answers every probe exactly with ~1 LDS, wherever the set lies.
constexpr uint32_t kRSlotBits = 7;
constexpr uint32_t kRSlots = 1u << kRSlotBits;
constexpr uint32_t kREmpty = 0xFFFFFFFEu;  // never a rank (and != kNone, the row pad)
__device__ __forceinline__ uint32_t r_slot(uint32_t y) { return (y * 0x9E3779B1u) >> (32 - kRSlotBits); }
struct HashProbe {
    static constexpr bool low = false;
    unsigned tab;  // shared address of the warp's kRSlots keys
    __device__ __forceinline__ uint32_t bit(uint32_t y) const {
        uint32_t h = r_slot(y);
        uint32_t k = lds32(tab + 4u * h);
        while (k != y && k != kREmpty) {
            h = (h + 1u) & (kRSlots - 1u);
            k = lds32(tab + 4u * h);
        }
        return k == y;
    }
    __device__ __forceinline__ bool below(uint32_t) const { return false; }
    __device__ __forceinline__ uint32_t cand(uint32_t) const { return 0u; }
    __device__ __forceinline__ bool verify(uint32_t, bool act) const { return act; }
    __device__ __forceinline__ uint32_t sentinel() const { return kNone; }
};
// insert key s (a rank) into the table; returns its slot
__device__ __forceinline__ uint32_t r_insert(uint32_t* tab, uint32_t s) {
    uint32_t h = r_slot(s);
    while (atomicCAS(tab + h, kREmpty, s) != kREmpty) h = (h + 1u) & (kRSlots - 1u);
    return h;
}
#ifndef TRIGPU_R_HASH
#define TRIGPU_R_HASH 0
#endif
#ifndef TRIGPU_R_SEARCH
#define TRIGPU_R_SEARCH 1  // wide sets of short rows: shuffle search instead of the bitmap
#endif
constexpr int kRWarps = 8;
#ifndef TRIGPU_R_BITS_A
#define TRIGPU_R_BITS_A 15
#endif
constexpr uint32_t kRBitsA = TRIGPU_R_BITS_A, kRBitsB = 11;  // 4 KB window + 256 B region B per warp
#if TRIGPU_R_HASH
constexpr size_t kRBmBytes = kRSlots * 4;
#else
constexpr size_t kRBmBytes = win_bytes(kRBitsA, kRBitsB);
#endif

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kRWarps * 32, R_MINB(F)) k_list_reg(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t* bma = reinterpret_cast<uint32_t*>(dsm + warp_scratch_bytes<F>(kRWarps) + warp * kRBmBytes);
    uint32_t* bmb = bma + ((1u << kRBitsA) / 32 + 4);
    for (uint32_t i = lane; i < kRBmBytes / 4; i += 32) bma[i] = TRIGPU_R_HASH ? kREmpty : 0u;
    __syncwarp();
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    // Seeds come in runs of 32 (one queue atomic); a run's seed ids, set rows
    // and sizes are loaded lane-parallel at once, and each seed's set (and
    // the offsets of its rows) is prefetched while the previous seed is
    // listed, so a seed waits on one dependent round trip (its rows) instead
    // of five. Tiny seeds are latency-bound, not bandwidth-bound.
    for (;;) {
        unsigned b = 0;
        if (lane == 0) b = atomicAdd(P.queue, 32u);
        b = __shfl_sync(FULL, b, 0);
        if (b >= P.nseeds) break;
        const unsigned cnt = min(32u, P.nseeds - b);
        uint32_t seed_l = 0, d_l = 0;
        uint64_t so_l = 0;
        if (lane < cnt) {
            seed_l = P.seeds[b + lane];
            so_l = P.set_off[seed_l];
            d_l = P.set_len[seed_l];
        }
        // seed 0's set and row offsets
        uint32_t d = __shfl_sync(FULL, d_l, 0);
        uint64_t so = shfl64(so_l, 0);
        uint32_t s = lane < d ? __ldg(P.set_adj + so + lane) : kNone;
        uint64_t ro = 0;
        uint32_t rl = 0;
        if (lane < d) {
            ro = P.out_off[s];
            rl = P.out_len[s];
        }
        for (unsigned k = 0; k < cnt; ++k) {
            const uint32_t seed = __shfl_sync(FULL, seed_l, k);
            // prefetch the next seed's set
            uint32_t d1 = 0, s1 = kNone;
            if (k + 1 < cnt) {
                d1 = __shfl_sync(FULL, d_l, k + 1);
                const uint64_t so1 = shfl64(so_l, k + 1);
                if (lane < d1) s1 = __ldg(P.set_adj + so1 + lane);
            }
            sink.begin_unit(P, seed);
#if TRIGPU_R_HASH
            uint32_t slot = 0;
            if (lane < d) slot = r_insert(bma, s);
            __syncwarp();
            scan_rows_at<ALGO, F>(P, seed, s, ro, rl, HashProbe{smem_addr(bma)}, sink);
            sink.end_unit(P, seed);
            __syncwarp();
            if (lane < d) bma[slot] = kREmpty;
            __syncwarp();
#else
            const WinGeom g =
                win_geom(kRBitsA, kRBitsB, P.bm_shrink, __shfl_sync(FULL, s, 0), __shfl_sync(FULL, s, d - 1));
#if TRIGPU_R_SEARCH
            if (P.r_search && g.low) {
                scan_rows_at<ALGO, F>(P, seed, s, ro, rl, SearchProbe{RegVerify{s}}, sink);
                sink.end_unit(P, seed);
            } else
#endif
            {
                if (lane < d) win_set(bma, bmb, g, s);
                __syncwarp();
                with_win_probe(P, smem_addr(bma), smem_addr(bmb), g, RegVerify{s}, [&](const auto& probe) {
                    scan_rows_at<ALGO, F>(P, seed, s, ro, rl, probe, sink);
                });
                sink.end_unit(P, seed);
                __syncwarp();
                if (lane < d) win_clear(bma, bmb, g, s);
                __syncwarp();
            }
#endif
            // the next seed's row offsets (its set has arrived by now)
            d = d1;
            s = s1;
            ro = 0;
            rl = 0;
            if (lane < d) {
                ro = P.out_off[s];
                rl = P.out_len[s];
            }
        }
    }
    sink.flush(P);
    flush_hist(P, sink);
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
    flush_hist(P, sink);
}

// ---- class C: 256 < |S| <= 4096, CTA per seed ----------------------------------
// All warps of the CTA share the seed's bitmap. The seed's rows are cut into
// chunks (chunk prefix over the set in a shared row table) and split equally
// across the warps, so the CTA barrier at the end of a seed waits for
// balanced work. Two sizes: C1 (256 < |S| <= 1024) runs 8-warp CTAs, several
// per SM, so one CTA's seed barrier is hidden by the others; C2 (1024 < |S| <=
// 4096) runs one 32-warp CTA per SM.
template <int THREADS, uint32_t BITS_A, uint32_t BITS_B, uint32_t MAXD, int MINB, int RING = 0>
struct CtaCfg {
    static constexpr int kThreads = THREADS;
    static constexpr int kWarps = THREADS / 32;
    static constexpr uint32_t kBitsA = BITS_A;  // window of 2^BITS_A ranks
    static constexpr uint32_t kBitsB = BITS_B;  // region B of 2^BITS_B bits
    static constexpr uint32_t kMaxD = MAXD;
    static constexpr int kMinBlocks = MINB;
    static constexpr int kRing = RING;  // 0: register loads; >0: per-warp ring of bulk-copied chunks
};
#ifndef TRIGPU_C1_RING
#define TRIGPU_C1_RING 0
#endif
#ifndef TRIGPU_C1_MINB
#define TRIGPU_C1_MINB 2
#endif
#ifndef TRIGPU_C2_RING
#define TRIGPU_C2_RING 0
#endif
#ifndef TRIGPU_C1_BITS_A
#define TRIGPU_C1_BITS_A 18
#endif
#ifndef TRIGPU_H_CTA
#define TRIGPU_H_CTA 0  // 1: class H as CTA-per-seed staged kernel (CfgH)
#endif
#ifndef TRIGPU_H_RING
#define TRIGPU_H_RING 2
#endif
#ifndef TRIGPU_H_MINB
#define TRIGPU_H_MINB 4
#endif
#ifndef TRIGPU_H_BITS_A_CTA
#define TRIGPU_H_BITS_A_CTA 17
#endif
#ifndef TRIGPU_HW_BITS_A
#define TRIGPU_HW_BITS_A 19
#endif
#ifndef TRIGPU_HW_MINB
#define TRIGPU_HW_MINB 2
#endif
#ifndef TRIGPU_C1_THREADS
#define TRIGPU_C1_THREADS 512
#endif
#ifndef TRIGPU_HW_THREADS
#define TRIGPU_HW_THREADS 512
#endif
// C1: 16-warp CTAs, 2 per SM at 64 registers. Measured (C5 / C4 class time, ms):
// 8 warps x 3 CTAs, 2^18 window 927 / 73.1; x 4 CTAs 1021 / 78.5; 16 warps x 2,
// 2^18 902 / 69.1; 16 warps x 2, 2^19 783 / 71.9; 32 warps x 1, 2^19 807 / 72.3.
// The 2^19 window is used above kWideMinN vertices (as for class H).
#ifndef TRIGPU_C1_MAXD
#define TRIGPU_C1_MAXD 1024
#endif
using CfgC1 = CtaCfg<TRIGPU_C1_THREADS, TRIGPU_C1_BITS_A, 14, TRIGPU_C1_MAXD, TRIGPU_C1_MINB, TRIGPU_C1_RING>;
using CfgC1Wide = CtaCfg<TRIGPU_C1_THREADS, TRIGPU_C1_BITS_A + 1, 14, TRIGPU_C1_MAXD, TRIGPU_C1_MINB, TRIGPU_C1_RING>;
#ifndef TRIGPU_C2_BITS_A
#define TRIGPU_C2_BITS_A 19
#endif
#ifndef TRIGPU_C2_THREADS
#define TRIGPU_C2_THREADS 1024
#endif
using CfgC2 = CtaCfg<TRIGPU_C2_THREADS, TRIGPU_C2_BITS_A, 15, 4096, 1, TRIGPU_C2_RING>;  // (2 x 512-thread CTAs, 2^18 window: C5 5 % slower)
using CfgH = CtaCfg<256, TRIGPU_H_BITS_A_CTA, 13, 256, TRIGPU_H_MINB, TRIGPU_H_RING>;
// Class H on graphs of more than 2^25 vertices: the set of an H seed spans so
// many ranks that the per-warp 2^16 window leaves many of its elements to the
// filter + verification path; a CTA per seed shares one wider window
// (measured on C5: warp kernel 1275 ms; CTA-wide, 8 warps x 3 CTAs/SM, 2^19
// window 1147 ms; 8 warps x 4, 2^18 1097 ms; 16 warps x 2, 2^19 1082 ms; 32
// warps x 1 1288 ms; on C4 the warp kernel stays faster).
using CfgHWide = CtaCfg<TRIGPU_HW_THREADS, TRIGPU_HW_BITS_A, 13, 256, TRIGPU_HW_MINB, 0>;
// Graph-size thresholds: above kHCtaMinN vertices class H is split - seeds of
// |S| <= kHSplit stay on the warp-per-seed kernel (cheap set-up, windows that
// still cover a small set), the larger sets go to the CTA kernel; above
// kWideMinN vertices C1 uses its 2^19-window instance. (C5 class H: all CTA
// 1087 ms, split at 64 / 96 / 128: 1074 / 1051 / 1050, all warp 1279; C4: all
// warp 74.2, split at 96: 69.1, all CTA 74.1; C2, 4 M vertices: count + checksum
// all warp 6.7, split 7.0; with per-vertex counts 15.3 vs 13.7.)
constexpr uint32_t kWideMinN = 1u << 25;
#ifndef TRIGPU_H_CTA_MIN_N
#define TRIGPU_H_CTA_MIN_N (1u << 21)
#endif
constexpr uint32_t kHCtaMinN = TRIGPU_H_CTA_MIN_N;
#ifndef TRIGPU_H_SPLIT
#define TRIGPU_H_SPLIT 96
#endif
constexpr uint32_t kHSplit = TRIGPU_H_SPLIT;
template <class CFG>
constexpr size_t cta_bitmap_bytes() { return win_bytes(CFG::kBitsA, CFG::kBitsB); }
template <class CFG>
constexpr size_t cta_row_bytes() { return CFG::kMaxD * 16; }  // uint4 {first quad, quads, first chunk, x}
// per warp: kRing stages of kStageChunks chunks (kSlotBytes each) + per stage
// an mbarrier (8 B, padded to 16) and kStageChunks {x, quads} records
constexpr int kStageChunks = 4;
constexpr uint32_t kStageBytes = kStageChunks * kSlotBytes;
template <class CFG>
constexpr size_t cta_ring_bytes() {
    return static_cast<size_t>(CFG::kWarps) * CFG::kRing * (kStageBytes + 16 + 8 * kStageChunks);
}

// A warp's contiguous chunk range [gb, ge) of the seed streamed through its
// ring of NS shared-memory stages of kStageChunks chunks: lane 0 bulk-copies
// (cp.async.bulk, the TMA engine) the chunks of stage j NS stages ahead of
// their use and arms the stage's mbarrier with their byte count; every lane
// waits on it, probes its quads (LDS.128) and, for the checksum, re-reads
// only its hit elements from the stage. The bytes in flight live in shared
// memory, not registers. `phases` (bit k = parity to wait for on stage k)
// persists across seeds.
template <int NS, int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void stream_ring(const ListParams& P, uint32_t seed, unsigned rows, uint32_t d,
                                            uint32_t gb, uint32_t ge, unsigned ring, unsigned bars, unsigned meta,
                                            uint32_t& phases, const Probe& probe, Sink<ALGO, F>& sink,
                                            unsigned& hits) {
    constexpr int K = kStageChunks;
    const unsigned lane = lane_id();
    const uint4* const quads = reinterpret_cast<const uint4*>(P.out_adj);
    CtaRowCursor prod(rows, d, gb, ge);
    const uint32_t nst = (ge - gb + K - 1) / K;  // stages of this range
    auto issue = [&](uint32_t k) {
        Chunk c[K];
        prod.next(c);
        if (lane == 0) {
            unsigned bytes = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) bytes += c[j].nq * 16u;
            sts128(meta + 8u * K * k, make_uint4(c[0].x, c[0].nq, c[1].x, c[1].nq));
            sts128(meta + 8u * K * k + 16u, make_uint4(c[2].x, c[2].nq, c[3].x, c[3].nq));
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bars + 16u * k, bytes);
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (c[j].nq) bulk_g2s(ring + kStageBytes * k + kSlotBytes * j, quads + c[j].qb, c[j].nq * 16u, bars + 16u * k);
        }
    };
    const uint32_t pro = nst < (uint32_t)NS ? nst : (uint32_t)NS;
    for (uint32_t k = 0; k < pro; ++k) issue(k);
    uint32_t k = 0;
    for (uint32_t i = 0; i < nst; ++i) {
        mbar_wait(bars + 16u * k, (phases >> k) & 1u);
        phases ^= 1u << k;
        const uint4 m0 = lds128(meta + 8u * K * k), m1 = lds128(meta + 8u * K * k + 16u);
        const Chunk ch[K] = {Chunk{0, m0.y, m0.x}, Chunk{0, m0.w, m0.z}, Chunk{0, m1.y, m1.x}, Chunk{0, m1.w, m1.z}};
        bool pr[K];
        uint4 y[K];
        const unsigned st = ring + kStageBytes * k;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            pr[j] = lane < ch[j].nq;
            y[j] = pr[j] ? lds128(st + kSlotBytes * j + 16u * lane) : make_uint4(kNone, kNone, kNone, kNone);
        }
        probe_quads<K, ALGO, F, Probe, true>(P, seed, ch, pr, y, probe, sink, hits, st);
        __syncwarp();
        if (i + NS < nst) issue(k);
        k = k + 1 == (uint32_t)NS ? 0 : k + 1;
    }
}

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
    // bulk-copy ring of this warp (kRing > 0): slots | barriers | {x, quads}
    const unsigned ring_base = rows + cta_row_bytes<CFG>();
    const unsigned wslot = ring_base + (threadIdx.x >> 5) * CFG::kRing * kStageBytes;
    const unsigned wbar = ring_base + CFG::kWarps * CFG::kRing * kStageBytes + (threadIdx.x >> 5) * CFG::kRing * 16u;
    const unsigned wmeta = ring_base + CFG::kWarps * CFG::kRing * (kStageBytes + 16u) +
                           (threadIdx.x >> 5) * CFG::kRing * 8u * kStageChunks;
    uint32_t phases = 0;
    if constexpr (CFG::kRing > 0) {
        if (lane_id() < (unsigned)CFG::kRing) mbar_init(wbar + 16u * lane_id(), 1);
        fence_mbar_init();
    }
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm);
    constexpr int PER = (CFG::kMaxD + kCThreads - 1) / kCThreads;  // set elements per thread
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
                unsigned hits = 0;
                if constexpr (CFG::kRing > 0) {
                    stream_ring<CFG::kRing>(P, seed, rows, d, gb, ge, wslot, wbar, wmeta, phases, probe, sink, hits);
                } else {
                    CtaRowCursor cur(rows, d, gb, ge);
                    stream_quads<ALGO, F, false>(P, seed, cur, probe, sink, hits);
                }
                sink.cnt += hits;
            }
        });
        sink.end_unit(P, seed);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < d; k += kCThreads) win_clear(bma, bmb, g, __ldg(row + k));
    }
    sink.flush(P);
    flush_hist(P, sink);
}

// (A barrier-free variant of k_list_cta - double-buffered bitmaps and row
// tables, a producer warp, mbarrier full / empty pairs so that a warp that
// finishes its share early runs ahead into the next seed - is in the history
// (commit "Run-ahead CTA kernel fixed ..."): correct, but for class H on C5 it
// measured 8 % slower than the barrier kernel.)

// ---- class G: |S| > 4096, CTA per seed ---------------------------------------
// A 2^20-rank shared-memory window over the set's top ranks (as the other
// classes), and for the set's elements below the window an exact n-bit
// bitmap in global memory (one per CTA, L2-resident slices): elements above
// the set's top rank cost one LDS of the guard word, elements in the window
// one LDS, only elements below the window touch the global bitmap (no
// verification needed: it is exact).
constexpr int kGThreads = 1024;
constexpr int kGWarps = kGThreads / 32;
#ifndef TRIGPU_G_BITS_A
#define TRIGPU_G_BITS_A 20
#endif
constexpr uint32_t kGBitsA = TRIGPU_G_BITS_A;
#ifndef TRIGPU_G_BITS_C
#define TRIGPU_G_BITS_C 18
#endif
constexpr uint32_t kGBitsC = TRIGPU_G_BITS_C;  // coarse filter below the window: 2^18 bits (32 KB)
constexpr size_t kGWinBytes = (size_t{1} << kGBitsA) / 8 + 16;
constexpr size_t kGCoarseBytes = (size_t{1} << kGBitsC) / 8;

// Below the window, a coarse shared-memory filter (bit i = some set element
// in ranks [i << cs, (i + 1) << cs)) answers most probes; only its positives
// read the exact global bitmap.
struct WinGlobalProbe {
    static constexpr bool low = true;
    unsigned bm;          // shared address of the window
    uint32_t wb, la;      // window base, length
    const uint32_t* gbm;  // exact global bitmap of the set's elements below wb
    unsigned bmc;         // shared address of the coarse filter
    uint32_t cs;          // coarse shift
    __device__ __forceinline__ uint32_t bit(uint32_t y) const {
        const uint32_t o = min(y - wb, la);
        return (lds32(bit_word(bm, o)) >> (o & 31u)) & 1u;
    }
    __device__ __forceinline__ bool below(uint32_t y) const { return y < wb; }
    __device__ __forceinline__ uint32_t cand(uint32_t y) const {
        const uint32_t c = y >> cs;
        if (!((lds32(bit_word(bmc, c)) >> (c & 31u)) & 1u)) return 0u;
        return (__ldcg(gbm + (y >> 5)) >> (y & 31u)) & 1u;
    }
    __device__ __forceinline__ bool verify(uint32_t, bool act) const { return act; }
    __device__ __forceinline__ uint32_t sentinel() const { return kNone; }
};

// (Cutting a giant seed into several CTA work items - interleaved slices of its
// x chunks - measured slower on C4 split A+- (G 168 -> 211 ms): every part
// rebuilds and clears the seed's bitmaps, O(|S|) global atomics.)
template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kGThreads) k_list_giant(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned unit;
    const unsigned warp = threadIdx.x >> 5;
    uint32_t* bm = P.bitmaps + (uint64_t)blockIdx.x * P.bitmap_words;
    uint32_t* win = reinterpret_cast<uint32_t*>(dsm + warp_scratch_bytes<F>(kGWarps));
    uint32_t* coarse = win + kGWinBytes / 4;
    constexpr uint32_t kWords = (kGWinBytes + kGCoarseBytes) / 4;
    for (uint32_t i = threadIdx.x; i < kWords; i += kGThreads) win[i] = 0u;
    __shared__ unsigned int giant_rows;  // rows of this seed left to the whole CTA
    const SharedRowList defer{smem_addr(dsm + warp_scratch_bytes<F>(kGWarps) + kGWinBytes + kGCoarseBytes), &giant_rows};
    if (threadIdx.x == 0) giant_rows = 0u;
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
        const uint32_t* row = P.set_adj + so;
        const uint32_t la = 1u << (kGBitsA > P.bm_shrink + 5u ? kGBitsA - P.bm_shrink : 5u);
        const uint32_t s0 = __ldg(row), top = __ldg(row + d - 1);
        const uint32_t wb = top - s0 >= la ? top + 1u - la : s0;
        // coarse shift: 2^kGBitsC bits cover the ranks below the window
        const uint32_t cs = wb > (1u << kGBitsC) ? 32u - __clz((wb - 1u) >> kGBitsC) : 0u;
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(row + k);
            if (v >= wb) {
                atomicOr(win + ((v - wb) >> 5), 1u << ((v - wb) & 31u));
            } else {
                atomicOr(bm + (v >> 5), 1u << (v & 31));
                atomicOr(coarse + ((v >> cs) >> 5), 1u << ((v >> cs) & 31u));
            }
        }
        __syncthreads();
        const WinGlobalProbe probe{smem_addr(win), wb, la, bm, smem_addr(coarse), cs};
        scan_x_range<ALGO, F>(P, seed, so, warp * 32, d, kGWarps * 32, probe, sink, defer);
        __syncthreads();
        {  // the seed's giant rows, every warp an equal share of each row's chunks
            const unsigned nrows = min(giant_rows, kDeferCap);
            unsigned hits = 0;
            for (unsigned i = 0; i < nrows; ++i) {
                const uint4 e = lds128(defer.rows + 16u * i);
                const uint32_t nch = row_chunks(e.y);
                RowRangeCursor cur{e.x, e.y, e.z, static_cast<uint32_t>((static_cast<uint64_t>(nch) * warp) / kGWarps),
                                   static_cast<uint32_t>((static_cast<uint64_t>(nch) * (warp + 1)) / kGWarps)};
                stream_quads<ALGO, F, true>(P, seed, cur, probe, sink, hits);
            }
            sink.cnt += hits;
        }
        sink.end_unit(P, seed);
        __syncthreads();
        if (threadIdx.x == 0) giant_rows = 0u;
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(row + k);
            if (v >= wb) {
                win[(v - wb) >> 5] = 0u;
            } else {
                __stcg(bm + (v >> 5), 0u);
                coarse[(v >> cs) >> 5] = 0u;
            }
        }
    }
    sink.flush(P);
    flush_hist(P, sink);
}

// dynamic shared memory per CTA of each class kernel
template <unsigned F> constexpr size_t smem_reg() { return warp_scratch_bytes<F>(kRWarps) + kRWarps * kRBmBytes; }
template <unsigned F> constexpr size_t smem_warp() { return warp_scratch_bytes<F>(kHWarps) + kHWarps * kHBmBytes; }
template <unsigned F, class CFG> constexpr size_t smem_cta() { return warp_scratch_bytes<F>(CFG::kWarps) + cta_bitmap_bytes<CFG>() + cta_row_bytes<CFG>() + cta_ring_bytes<CFG>(); }
template <unsigned F> constexpr size_t smem_giant() { return warp_scratch_bytes<F>(kGWarps) + kGWinBytes + kGCoarseBytes + kDeferCap * 16; }

// ---- seed classification --------------------------------------------------
constexpr int kClasses = 5;  // R, H, C1, C2, G

struct SeedLists {
    uint32_t* lists[kClasses];
    unsigned int* counts;     // [kClasses], then [kClasses] = the small class-H seeds
    uint32_t cap;             // entries per list
    uint32_t h_small;         // class-H seeds of |S| <= h_small go to the BACK of lists[1] (0: no split)
};

// Seeds with rank in [rb, re) and |S| >= 2 into their class lists.
__global__ void __launch_bounds__(256) k_classify_seeds(uint32_t rb, uint32_t re, const uint32_t* __restrict__ set_len,
                                                        SeedLists L) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t start = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t span = re - rb;
    const uint64_t trips = (span + stride - 1) / stride;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t r = rb + start + t * stride;
        uint64_t d = 0;
        if (r < re) d = set_len[r];
        int cls = -1;
        if (d >= 2) cls = d <= 32 ? 0 : d <= 256 ? 1 : d <= CfgC1::kMaxD ? 2 : d <= CfgC2::kMaxD ? 3 : 4;
        if (cls == 1 && d <= L.h_small) cls = kClasses;  // the two H lists share lists[1]: front and back
#pragma unroll
        for (int c = 0; c <= kClasses; ++c) {
            const unsigned b = __ballot_sync(FULL, cls == c);
            if (!b) continue;
            const unsigned leader = __ffs(b) - 1;
            unsigned base = 0;
            if (lane_id() == leader) base = atomicAdd(&L.counts[c], __popc(b));
            base = __shfl_sync(FULL, base, leader);
            const unsigned pos = base + __popc(b & lanemask_lt());
            if (cls == c) {
                if (c < kClasses) L.lists[c][pos] = (uint32_t)r;
                else L.lists[1][L.cap - 1u - pos] = (uint32_t)r;
            }
        }
    }
}

// List compaction: copy segment i's len triangles from src to dst (the
// triangles past the count fill the chunk tails left below it).
__global__ void k_move_triangles(const ulonglong2* __restrict__ seg_src_dst, const unsigned long long* __restrict__ seg_len,
                                 unsigned nseg, uint32_t* __restrict__ tri) {
    for (unsigned i = blockIdx.x; i < nseg; i += gridDim.x) {
        const unsigned long long src = seg_src_dst[i].x, dst = seg_src_dst[i].y, len = seg_len[i];
        for (unsigned long long k = threadIdx.x; k < 3 * len; k += blockDim.x) tri[3 * dst + k] = tri[3 * src + k];
    }
}

// Per-class inner_ops (TL_DEBUG_CLASS_WORK): work[c] += sum over x in set(s)
// of d+(x) for every seed s of class c. Warp per seed of one class list.
__global__ void __launch_bounds__(256) k_class_work(const uint32_t* __restrict__ seeds, unsigned nseeds,
                                                   const uint64_t* __restrict__ set_off,
                                                   const uint32_t* __restrict__ set_len,
                                                   const uint32_t* __restrict__ set_adj,
                                                   const uint32_t* __restrict__ out_len,
                                                   unsigned long long* __restrict__ work) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long w = 0;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nseeds; i += warps) {
        const uint32_t r = seeds[i];
        const uint64_t so = set_off[r];
        const uint32_t d = set_len[r];
        for (uint32_t k = lane; k < d; k += 32) w += out_len[set_adj[so + k]];
    }
    w = warp_sum64(w);
    if (lane == 0 && w) atomicAdd(work, w);
}

// inner_ops / mark_ops of the seeds in [rb, re) (tl_list_range): per seed s,
// inner += sum over x in set(s) of d+(x) (listing.hpp:80, 101), mark += 2|S|.
// Warp per seed.
__global__ void __launch_bounds__(256) k_range_cost(uint32_t rb, uint32_t re, const uint64_t* __restrict__ set_off,
                                                    const uint32_t* __restrict__ set_len,
                                                    const uint32_t* __restrict__ set_adj,
                                                    const uint32_t* __restrict__ out_len,
                                                    unsigned long long* __restrict__ acc) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long inner = 0, mark = 0;
    for (uint64_t r = rb + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5); r < re; r += warps) {
        const uint64_t so = set_off[r];
        const uint32_t d = set_len[r];
        if (lane == 0) mark += 2ull * d;
        for (uint32_t i = lane; i < d; i += 32) inner += out_len[set_adj[so + i]];
    }
    inner = warp_sum64(inner);
    mark = warp_sum64(mark);
    if (lane == 0) {
        atomicAdd(&acc[0], inner);
        atomicAdd(&acc[1], mark);
    }
}

}  // namespace trigpu
