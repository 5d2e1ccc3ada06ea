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
// The reference's uint8 table[n] becomes a per-seed probe structure sized to
// |S| (degree binning):
//   class R  2 <= |S| <= 32     warp per seed, S in registers (one id per lane),
//                               membership by a 5-step shuffle binary search
//   class H  32 < |S| <= 256    warp per seed, per-warp shared-memory hash
//   class C  256 < |S| <= 4096  CTA per (seed, x-slice), shared-memory hash
//   class G  |S| > 4096         CTA per seed, per-CTA global bitmap over ranks
// Every class walks the rows of 32 x's at a time as ONE flattened, coalesced
// stream (lane f of a batch reads element f of the concatenated rows; the row
// of each lane is found from a warp OR-reduction of row starts), so short
// rows do not idle lanes.
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
    const uint64_t* set_off;  // probe-set rows: out-CSR (A+-) or in-CSR (A++)
    const uint32_t* set_adj;
    const uint64_t* out_off;  // scanned rows: always the out-CSR
    const uint32_t* out_adj;
    const uint32_t* inv;      // rank -> dense id
    unsigned long long* acc;  // [0] triangles, [1] checksum, [2] list cursor
    unsigned long long* vcount;  // rank space
    uint32_t* tri;
    unsigned long long tri_cap;
    const uint32_t* seeds;    // class list
    unsigned int nseeds;
    unsigned int* queue;      // dynamic work counter
    uint32_t* bitmaps;        // class G only: one n-bit bitmap per CTA
    uint64_t bitmap_words;
    int variant;              // reserved for A/B probe experiments
    uint32_t win_bits;        // hub-window size (log2 ranks, capped per class); 0 = no window
};

// Per-warp hit buffer: hits (x, y) are compacted into shared memory by a
// ballot and emitted 32 at a time with every lane busy, instead of running
// the dense-id gathers / hash / atomics with the 1-3 lanes that hit in a batch.
constexpr int kHitBuf = 96;  // 31 pending + up to 2 batches of 32 before a drain
// 32-element blocks loaded per warp before probing (memory-level parallelism):
// the count-only sink keeps more in flight than the sinks that buffer hits
constexpr int kUnrollCount = 16;
constexpr int kUnrollSink = 8;
constexpr int kMetaBytes = 768;  // per warp: uint4[32] block table, u32[32] edge lanes, u32[32] x

// Emit n (<= 32) buffered hits, lane i taking entry i; returns this lane's
// checksum contribution. Out of line: it runs once per 32 triangles.
template <int ALGO, unsigned F>
__device__ __forceinline__ unsigned long long emit_hits(const ListParams& P, uint32_t seed, unsigned n,
                                                     unsigned from) {
    const unsigned lane = lane_id();
    const bool hit = lane < n;
    const uint2 e = hit ? lds64(from + 8u * lane) : make_uint2(0, 0);
    const uint32_t x = e.x, y = e.y;
    unsigned long long sum = 0;
    if constexpr ((F & F_VCOUNT) != 0u) {
        if (hit) {
            atomicAdd(&P.vcount[x], 1ull);
            atomicAdd(&P.vcount[y], 1ull);
        }
    }
    if constexpr ((F & (F_CHECKSUM | F_LIST)) != 0u) {
        const uint32_t ru = ALGO == ALGO_APM ? seed : x;
        const uint32_t rv = ALGO == ALGO_APM ? x : y;
        const uint32_t rw = ALGO == ALGO_APM ? y : seed;
        uint32_t du = 0, dv = 0, dw = 0;
        if (hit) {
            du = __ldg(P.inv + ru);
            dv = __ldg(P.inv + rv);
            dw = __ldg(P.inv + rw);
        }
        if constexpr ((F & F_CHECKSUM) != 0u)
            if (hit) sum = tri_hash(du, dv, dw);
        if constexpr ((F & F_LIST) != 0u) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&P.acc[2], (unsigned long long)n);
            base = __shfl_sync(FULL, base, 0);
            if (hit) {
                const unsigned long long k = base + lane;
                if (k < P.tri_cap) {
                    P.tri[3 * k] = du;
                    P.tri[3 * k + 1] = dv;
                    P.tri[3 * k + 2] = dw;
                }
            }
        }
    }
    return sum;
}

template <int ALGO, unsigned F>
struct Sink {
    unsigned long long cnt = 0, sum = 0;
    unsigned seed_hits = 0;
    unsigned buf = 0;      // shared address of this warp's kHitBuf uint2 entries
    unsigned meta = 0;     // (unused)
    unsigned ring = 0;     // shared address of this warp's cp.async ring (kRing x 128 B)
    unsigned pending = 0;  // warp-uniform

    // One 32-wide batch (called convergently by the whole warp).
    __device__ __forceinline__ void batch(bool hit, uint32_t x, uint32_t y) {
        if constexpr (F != 0u) {
            const unsigned b = __ballot_sync(FULL, hit);
            if (!b) return;
            if constexpr ((F & F_VCOUNT) != 0u) seed_hits += hit;
            if (hit) sts64(buf + 8u * (pending + __popc(b & lanemask_lt())), make_uint2(x, y));
            pending += __popc(b);
        }
    }

    // Same, with x read (broadcast) from shared memory only if some lane hit.
    __device__ __forceinline__ void batch_lazy(bool hit, unsigned xaddr, uint32_t y) {
        if constexpr (F != 0u) {
            const unsigned b = __ballot_sync(FULL, hit);
            if (!b) return;
            const uint32_t x = lds32(xaddr);
            if constexpr ((F & F_VCOUNT) != 0u) seed_hits += hit;
            if (hit) sts64(buf + 8u * (pending + __popc(b & lanemask_lt())), make_uint2(x, y));
            pending += __popc(b);
        }
    }

    // Emit every full group of 32 buffered hits (call after <= 2 batches).
    __device__ __forceinline__ void drain(const ListParams& P, uint32_t seed) {
        if constexpr (F != 0u) {
            if (pending < 32) return;
            __syncwarp();
            unsigned done = 0;
            for (; pending - done >= 32; done += 32) sum += emit_hits<ALGO, F>(P, seed, 32, buf + 8u * done);
            __syncwarp();
            if (lane_id() < pending - done) sts64(buf + 8u * lane_id(), lds64(buf + 8u * (done + lane_id())));
            __syncwarp();
            pending -= done;
        }
    }

    // End of one seed's unit: drain the buffer, credit the seed's own count.
    __device__ __forceinline__ void end_unit(const ListParams& P, uint32_t seed) {
        if constexpr (F != 0u) {
            drain(P, seed);
            if (pending) {
                __syncwarp();
                sum += emit_hits<ALGO, F>(P, seed, pending, buf);
                __syncwarp();
                pending = 0;
            }
        }
        if constexpr ((F & F_VCOUNT) != 0u) {
            const unsigned long long h = warp_sum64(seed_hits);
            if (lane_id() == 0 && h) atomicAdd(&P.vcount[seed], h);
            seed_hits = 0;
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

// Probe the elements of blocks [kb, ke) of one row (base rp, len elements;
// block k = elements 32k .. 32k+31, lane l takes element 32k + l): four
// blocks' loads issued back to back, then probed; the row end is predicated.
#ifndef TRIGPU_STREAM_U
#define TRIGPU_STREAM_U 4
#endif
__device__ __forceinline__ void ldg_batch(const uint32_t* const (&a)[4], uint32_t (&y)[4]) { ldg4(a, y); }
__device__ __forceinline__ void ldg_batch(const uint32_t* const (&a)[8], uint32_t (&y)[8]) { ldg8(a, y); }

template <int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void stream_blocks(const ListParams& P, uint32_t seed, const uint32_t* rp, uint32_t len,
                                              uint32_t kb, uint32_t ke, uint32_t x, const Probe& probe,
                                              Sink<ALGO, F>& sink, unsigned& hits) {
    constexpr int U = TRIGPU_STREAM_U;
    const unsigned lane = lane_id();
    const uint32_t* p = rp + 32u * kb + lane;
    uint32_t pos = 32u * kb + lane;
    for (uint32_t k = kb; k < ke; k += U) {
        const uint32_t* a[U];
        uint32_t y[U];
        bool ok[U], h[U];
#pragma unroll
        for (int i = 0; i < U; ++i) {
            ok[i] = k + i < ke && pos + 32u * i < len;
            a[i] = ok[i] ? p + 32 * i : rp;
        }
        ldg_batch(a, y);
        probe_batch(probe, y, ok, h);
        bool any = false;
#pragma unroll
        for (int i = 0; i < U; ++i) {
            hits += h[i];
            any |= h[i];
        }
        if constexpr (F != 0u) {
            if (__any_sync(FULL, any)) {
#pragma unroll
                for (int i = 0; i < U; ++i) {
                    sink.batch(h[i], x, y[i]);
                    if (i % 2 == 1) sink.drain(P, seed);
                }
            }
        }
        p += 32 * U;
        pos += 32 * U;
    }
}

// Walk the out-rows of up to 32 x's (x valid on lanes with xvalid), probing
// every element y against the seed's set. Two phases:
//   1. rows of >= 32 elements, as 128-byte-ALIGNED blocks of 32 elements
//      (partial first / last block predicated), flattened over all blocks of
//      all such rows: block g belongs to row j = #rows whose blocks end at or
//      before g (one vote); the row's block offset and edge lanes come from a
//      per-warp shared-memory table read with a broadcast LDS; lane l reads
//      element l of the block (one fully coalesced 128 B line). Software-
//      pipelined: the next four blocks' loads are issued before the current
//      four are probed (up to eight loads in flight per lane);
//   2. rows of < 32 elements as ONE flattened stream (lane f of a window
//      reads element f of the concatenated rows; the owning row of each lane
//      comes from an OR-reduction of the row starts), so short rows do not
//      idle lanes.
template <int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void scan_rows(const ListParams& P, uint32_t seed, uint32_t x, bool xvalid,
                                          const Probe& probe, Sink<ALGO, F>& sink) {
    const unsigned lane = lane_id();
    uint64_t ro = 0;
    uint32_t rl = 0;
    if (xvalid) {
        ro = P.out_off[x];
        rl = static_cast<uint32_t>(P.out_off[x + 1] - ro);
    }
    unsigned hits = 0;
    // ---- phase 1: rows of >= 32 elements, one at a time, whole warp per row
    unsigned longm = __ballot_sync(FULL, rl >= 32u);
    while (longm) {
        const int j = __ffs(longm) - 1;
        longm &= longm - 1;
        const uint32_t len = __shfl_sync(FULL, rl, j);
        const uint32_t* rp = P.out_adj + shfl64(ro, j);
        stream_blocks<ALGO, F>(P, seed, rp, len, 0, (len + 31u) >> 5, __shfl_sync(FULL, x, j), probe, sink, hits);
    }
    if (rl >= 32u) rl = 0;
    // ---- phase 2: tails
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
        const bool hitA = probe(yA, actA);
        const bool hitB = probe(yB, actB);
        hits += (unsigned)hitA + (unsigned)hitB;
        if constexpr (F != 0u) {
            sink.batch(hitA, __shfl_sync(FULL, cx, jA), yA);
            sink.batch(hitB, __shfl_sync(FULL, cx, jB), yB);
            sink.drain(P, seed);
        }
    }
    sink.cnt += hits;
}

// Chunks of 32 x's: set elements c, c + stride, ... below xe of the seed row at so.
template <int ALGO, unsigned F, class Probe>
__device__ __forceinline__ void scan_x_range(const ListParams& P, uint32_t seed, uint64_t so, uint32_t cb,
                                             uint32_t xe, uint32_t stride, Probe probe, Sink<ALGO, F>& sink) {
    const unsigned lane = lane_id();
    for (uint32_t c = cb; c < xe; c += stride) {
        const bool xv = c + lane < xe;
        const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
        scan_rows<ALGO, F>(P, seed, x, xv, probe, sink);
    }
}

// ---- probes --------------------------------------------------------------

struct RegProbe {  // S sorted ascending, one element per lane, padded with kNone
    uint32_t s;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        int pos = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, s, pos + step - 1);
            if (v < y) pos += step;
        }
        const uint32_t v = __shfl_sync(FULL, s, pos & 31);
        return act && pos < 32 && v == y;
    }
};

// Probe structure of classes H and C: a direct bitmap over the top window
// [wbase, n) of the rank space plus a bucketised hash table for the rest.
//
// Under degree ordering on power-law graphs the scanned rows N+(x) are made
// of hubs, i.e. the top ranks: on R-MAT, 90 % of all probes hit the top
// 0.2 % of ranks (scale 22). A sorted row's 32-element block therefore falls
// in a handful of bitmap words, so the window probe is one LDS.32 that the
// lanes of a warp mostly share (broadcast, no bank conflicts) and it is exact.
// Other probes go to the hash table: nb (power of two) buckets of four u32
// slots, one 16-byte LDS.128 per probe, slots filled in order (slot 3 used
// <=> bucket full), overflow keys in a small stash scanned only for full
// buckets. If even the stash overflows the seed falls back to a binary
// search of its sorted row in global memory, so the result stays exact.
constexpr uint32_t kStash = 32;

struct BucketTable {
    uint32_t* slots;      // 4 * nb u32, shared memory
    uint32_t* stash;      // kStash u32, shared memory
    unsigned* nstash;     // shared counter (> kStash: overflowed)
    uint32_t* win;        // window bitmap, shared memory
    uint32_t wbase;       // first rank of the window
};

__device__ __forceinline__ uint32_t bucket_shift(uint32_t d, uint32_t max_bits) {
    // nb = smallest power of two >= 2d (<= 1/2 key per slot-quad on average), >= 16
    uint32_t bits = 32 - __clz(max(2u * d - 1u, 15u));
    bits = bits > max_bits ? max_bits : bits;
    return 32 - bits;
}

__device__ __forceinline__ void bucket_insert(const BucketTable& T, uint32_t shift, uint32_t key) {
#ifdef TRIGPU_HUB_WINDOW
    if (key >= T.wbase) {
        const uint32_t o = key - T.wbase;
        atomicOr(T.win + (o >> 5), 1u << (o & 31));
        return;
    }
#endif
    uint32_t* b = T.slots + 4u * ((key * 0x9E3779B1u) >> shift);
#pragma unroll
    for (int s = 0; s < 4; ++s)
        if (atomicCAS(&b[s], kNone, key) == kNone) return;
    const unsigned i = atomicAdd(T.nstash, 1u);
    if (i < kStash) T.stash[i] = key;
}

__device__ __forceinline__ void bucket_clear(const BucketTable& T, uint32_t shift, uint32_t key) {
#ifdef TRIGPU_HUB_WINDOW
    if (key >= T.wbase) {
        T.win[(key - T.wbase) >> 5] = 0u;
        return;
    }
#endif
    uint4* b = reinterpret_cast<uint4*>(T.slots) + ((key * 0x9E3779B1u) >> shift);
    *b = make_uint4(kNone, kNone, kNone, kNone);
}

template <bool kStashed>
struct BucketProbe {
    unsigned win;     // shared address of the window bitmap
    uint32_t wbase;
    unsigned slots;   // shared address of the bucket array
    unsigned stash;   // shared address of the stash
    uint32_t shift;
    uint32_t nstash;  // kStashed == false <=> nstash == 0 (the common case)
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
#ifdef TRIGPU_HUB_WINDOW
        if (!act) return false;
        if (y >= wbase) {
            const uint32_t o = y - wbase;
            return (lds32(win + 4u * (o >> 5)) >> (o & 31)) & 1u;
        }
#endif
        const uint4 v = lds128(slots + 16u * ((y * 0x9E3779B1u) >> shift));
        bool hit = (v.x == y) | (v.y == y) | (v.z == y) | (v.w == y);
        if constexpr (kStashed) {
            if (act && !hit && v.w != kNone)
                for (uint32_t i = 0; i < nstash; ++i) hit |= lds32(stash + 4u * i) == y;
        }
        return act && hit;
    }
    // N probes at once: window words as predicated LDS.32 (no branches), the
    // hash path only if some lane of the warp has a below-window element.
    template <int N>
    __device__ __forceinline__ void batch(const uint32_t (&y)[N], const bool (&ok)[N], bool (&h)[N]) const {
#ifndef TRIGPU_HUB_WINDOW
#pragma unroll
        for (int k = 0; k < N; ++k) h[k] = (*this)(y[k], ok[k]);
        return;
#endif
        bool need = false;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const bool inw = ok[k] && y[k] >= wbase;
            const uint32_t o = y[k] - wbase;
            const uint32_t w = lds32_if(win + 4u * (o >> 5), inw);
            h[k] = (w >> (o & 31)) & 1u;
            need |= ok[k] && !inw;
        }
        if (__any_sync(FULL, need)) {
#pragma unroll
            for (int k = 0; k < N; ++k)
                if (ok[k] && y[k] < wbase) h[k] = (*this)(y[k], true);
        }
    }
};

// Default batched probe: N scalar probes.
template <class Probe, int N>
__device__ __forceinline__ void probe_batch(const Probe& p, const uint32_t (&y)[N], const bool (&ok)[N],
                                            bool (&h)[N]) {
#pragma unroll
    for (int k = 0; k < N; ++k) h[k] = p(y[k], ok[k]);
}
template <bool S, int N>
__device__ __forceinline__ void probe_batch(const BucketProbe<S>& p, const uint32_t (&y)[N], const bool (&ok)[N],
                                            bool (&h)[N]) {
    p.batch(y, ok, h);
}

// Exact fallback: binary search of the seed's sorted set row (global).
struct SearchProbe {
    const uint32_t* row;
    uint32_t d;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        if (!act) return false;
        uint32_t lo = 0, hi = d;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(row + mid) < y) lo = mid + 1;
            else hi = mid;
        }
        return lo < d && __ldg(row + lo) == y;
    }
};

// Timing-only probe (TRIGPU_VARIANT=2): touches every loaded element, never
// hits. Measures the row-streaming limit of a kernel without the probe cost.
struct NullProbe {
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const { return act && y == 0xFFFFFFFEu; }
};

// Dispatch on the table state of the current seed (uniform per unit).
template <class Body>
__device__ __forceinline__ void dispatch_probe(const BucketTable& T, uint32_t shift, unsigned ns,
                                               const uint32_t* row, uint32_t d, int variant, Body&& body) {
#ifdef TRIGPU_EXPERIMENTS
    if (variant == 2) {
        body(NullProbe{});
        return;
    }
#endif
    if (ns == 0)
        body(BucketProbe<false>{smem_addr(T.win), T.wbase, smem_addr(T.slots), 0, shift, 0});
    else if (ns <= kStash)
        body(BucketProbe<true>{smem_addr(T.win), T.wbase, smem_addr(T.slots), smem_addr(T.stash), shift, ns});
    else
        body(SearchProbe{row, d});
}

struct BitmapProbe {
    const uint32_t* bm;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        if (!act) return false;
        return (__ldcg(bm + (y >> 5)) >> (y & 31)) & 1u;
    }
};

// ---- per-warp scratch in dynamic shared memory ------------------------------
// [warps x kMetaBytes row tables][warps x kHitBuf uint2 hit buffers, F != 0]
// followed by the kernel's probe tables.
#ifndef TRIGPU_RING
#define TRIGPU_RING 0
#endif
constexpr uint32_t kRing = 8;  // blocks in flight per warp (power of two)
constexpr size_t kRingBytes = TRIGPU_RING ? kRing * 128 : 0;

template <unsigned F>
__host__ __device__ constexpr size_t warp_scratch_bytes(int warps) {
    return static_cast<size_t>(warps) * ((F ? kHitBuf * 8 : 0) + kRingBytes);
}

template <int ALGO, unsigned F>
__device__ __forceinline__ void attach_scratch(Sink<ALGO, F>& sink, unsigned char* base, int warps) {
    const unsigned w = threadIdx.x >> 5;
    if constexpr (F != 0u) sink.buf = smem_addr(base + w * kHitBuf * 8);
    sink.ring = smem_addr(base + warps * (F ? kHitBuf * 8 : 0) + w * kRingBytes);
}

// ---- class R: |S| <= 32, warp per seed, S in registers -------------------
constexpr int kRWarps = 8;

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kRWarps * 32) k_list_reg(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = lane_id();
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm, kRWarps);
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        const uint32_t s = lane < d ? __ldg(P.set_adj + so + lane) : kNone;
#ifdef TRIGPU_EXPERIMENTS
        if (P.variant == 2) {
            scan_rows<ALGO, F>(P, seed, s, lane < d, NullProbe{}, sink);
            sink.end_unit(P, seed);
            continue;
        }
#endif
        scan_rows<ALGO, F>(P, seed, s, lane < d, RegProbe{s}, sink);
        sink.end_unit(P, seed);
    }
    sink.flush(P);
}

// ---- class H: 32 < |S| <= 256, warp per seed, per-warp probe table ------
constexpr int kHWarps = 8;
constexpr uint32_t kHMaxBits = 8;     // 256 buckets = 4 KB per warp
constexpr uint32_t kHWinBits = 13;    // 8192-rank window = 1 KB per warp
constexpr size_t kHTableBytes = (16u << kHMaxBits) + (1u << kHWinBits) / 8 + kStash * 4 + 16;

// wbase for a window of 2^win_bits top ranks; win_bits == 0 disables it.
__device__ __forceinline__ uint32_t window_base(uint32_t n, uint32_t win_bits) {
    if (win_bits == 0) return 0xFFFFFFFFu;
    return n > (1u << win_bits) ? n - (1u << win_bits) : 0u;
}

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kHWarps * 32) k_list_hash_warp(ListParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned char* tbase = dsm + warp_scratch_bytes<F>(kHWarps) + warp * kHTableBytes;
    constexpr uint32_t kSlotBytes = 16u << kHMaxBits, kWinBytes = (1u << kHWinBits) / 8;
    BucketTable T{reinterpret_cast<uint32_t*>(tbase), reinterpret_cast<uint32_t*>(tbase + kSlotBytes + kWinBytes),
                  reinterpret_cast<unsigned*>(tbase + kSlotBytes + kWinBytes + kStash * 4),
                  reinterpret_cast<uint32_t*>(tbase + kSlotBytes),
                  window_base(P.n, min(P.win_bits, kHWinBits))};
    for (uint32_t i = lane; i < (4u << kHMaxBits); i += 32) T.slots[i] = kNone;
    for (uint32_t i = lane; i < kWinBytes / 4; i += 32) T.win[i] = 0u;
    if (lane == 0) *T.nstash = 0;
    __syncwarp();
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm, kHWarps);
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        const uint32_t shift = bucket_shift(d, kHMaxBits);
        for (uint32_t k = lane; k < d; k += 32) bucket_insert(T, shift, __ldg(P.set_adj + so + k));
        __syncwarp();
        dispatch_probe(T, shift, *T.nstash, P.set_adj + so, d, P.variant, [&](const auto& probe) {
            scan_x_range<ALGO, F>(P, seed, so, 0, d, 32, probe, sink);
        });
        sink.end_unit(P, seed);
        __syncwarp();
        for (uint32_t k = lane; k < d; k += 32) bucket_clear(T, shift, __ldg(P.set_adj + so + k));
        if (lane == 0) *T.nstash = 0;
        __syncwarp();
    }
    sink.flush(P);
}

// ---- class C: 256 < |S| <= 4096, CTA per seed, bucket table -------------
// All 32 warps of the CTA share the seed's table. The seed's rows are cut
// into 32-element blocks (block prefix over the set in shared memory) and
// warps pull batches of kCBatch blocks from a shared counter, so the CTA
// barrier at the end of a seed waits for at most one batch per warp.
// Two sizes: C1 (256 < |S| <= 1024) runs 8-warp CTAs, several per SM, so one
// CTA's seed barrier is hidden by the others; C2 (1024 < |S| <= 4096) needs
// the 64 KB table and runs one 32-warp CTA per SM.
template <int THREADS, uint32_t MAXBITS, uint32_t MAXD, int MINB>
struct CtaCfg {
    static constexpr int kThreads = THREADS;
    static constexpr int kWarps = THREADS / 32;
    static constexpr uint32_t kMaxBits = MAXBITS;  // 2^MAXBITS buckets
    static constexpr uint32_t kMaxD = MAXD;
    static constexpr int kMinBlocks = MINB;
};
using CfgC1 = CtaCfg<256, 11, 1024, 4>;
using CfgC2 = CtaCfg<1024, 12, 4096, 1>;
constexpr uint32_t kCBatch = 4;
constexpr uint32_t kCWinBits = 18;  // 262144-rank window = 32 KB
#ifdef TRIGPU_HUB_WINDOW
constexpr uint32_t kCWinBytes = (1u << kCWinBits) / 8;
#else
constexpr uint32_t kCWinBytes = 16;
#endif
template <class CFG>
constexpr size_t cta_table_bytes() { return (16u << CFG::kMaxBits) + kCWinBytes + kStash * 4 + 16; }
template <class CFG>
constexpr size_t cta_row_bytes() { return CFG::kMaxD * 16; }  // uint4 {ro lo, ro hi, len, first block}

template <int ALGO, unsigned F, class CFG, class Probe>
__device__ __forceinline__ void cta_blocks(const ListParams& P, uint32_t seed, uint64_t so, uint32_t d,
                                           unsigned rows, uint32_t nblocks, const Probe& probe,
                                           Sink<ALGO, F>& sink) {
    const unsigned warp = threadIdx.x >> 5;
    // equal share of the seed's blocks per warp (equal work), contiguous so
    // the owning rows are found once and then walked forward
    const uint32_t gb = static_cast<uint32_t>((static_cast<uint64_t>(nblocks) * warp) / CFG::kWarps);
    const uint32_t ge = static_cast<uint32_t>((static_cast<uint64_t>(nblocks) * (warp + 1)) / CFG::kWarps);
    if (gb >= ge) return;
    uint32_t lo = 0, hi = d - 1;
    while (lo < hi) {  // last row i with first_block(i) <= gb
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (lds32(rows + 16u * mid + 12u) <= gb) lo = mid;
        else hi = mid - 1;
    }
    unsigned hits = 0;
#if TRIGPU_RING
    // kRing blocks in flight per warp through cp.async into a shared-memory
    // ring (lane l copies and later reads only its own word of each slot),
    // so the depth costs no registers. Two cursors walk the rows: one issues
    // block g + kRing while the other consumes block g.
    const unsigned ring = sink.ring;
    const unsigned lane = lane_id();
    uint32_t ii = lo, ci = lo;
    uint4 ir = lds128(rows + 16u * lo), cr = ir;
    uint32_t inext = lo + 1 < d ? lds32(rows + 16u * (lo + 1) + 12u) : 0xFFFFFFFFu, cnext = inext;
    uint32_t gi = gb;
    auto issue = [&](uint32_t slot) {
        if (gi < ge) {
            while (inext <= gi) {
                ++ii;
                ir = lds128(rows + 16u * ii);
                inext = ii + 1 < d ? lds32(rows + 16u * (ii + 1) + 12u) : 0xFFFFFFFFu;
            }
            const uint32_t pos = 32u * (gi - ir.w) + lane;
            if (pos < ir.z)
                cp_async4(ring + 128u * slot + 4u * lane,
                          P.out_adj + ((static_cast<uint64_t>(ir.y) << 32) | ir.x) + pos);
        }
        cp_async_commit();
        ++gi;
    };
#pragma unroll
    for (uint32_t s = 0; s < kRing; ++s) issue(s);
    for (uint32_t g = gb; g < ge; ++g) {
        cp_async_wait<kRing - 1>();
        const uint32_t slot = (g - gb) & (kRing - 1);
        while (cnext <= g) {
            ++ci;
            cr = lds128(rows + 16u * ci);
            cnext = ci + 1 < d ? lds32(rows + 16u * (ci + 1) + 12u) : 0xFFFFFFFFu;
        }
        const bool ok = 32u * (g - cr.w) + lane < cr.z;
        const uint32_t y = ok ? lds32(ring + 128u * slot + 4u * lane) : kNone;
        const bool h = probe(y, ok);
        hits += h;
        if constexpr (F != 0u) {
            if (__any_sync(FULL, h)) sink.batch(h, __ldg(P.set_adj + so + ci), y);
            if (((g - gb) & 1u) == 1u) sink.drain(P, seed);
        }
        issue(slot);
    }
    cp_async_wait<0>();
#else
    for (uint32_t i = lo, g = gb; g < ge && i < d; ++i) {
        const uint4 r = lds128(rows + 16u * i);  // {ro lo, ro hi, len, first block}
        const uint32_t nb = (r.z + 31u) >> 5;
        if (r.w + nb <= g) continue;  // empty row (or already covered)
        const uint32_t kb = g - r.w, ke = min(ge - r.w, nb);
        const uint32_t x = F ? __ldg(P.set_adj + so + i) : 0u;
        stream_blocks<ALGO, F>(P, seed, P.out_adj + ((static_cast<uint64_t>(r.y) << 32) | r.x), r.z, kb, ke, x,
                               probe, sink, hits);
        g = r.w + ke;
    }
#endif
    sink.cnt += hits;
}

template <int ALGO, unsigned F, class CFG>
__global__ void __launch_bounds__(CFG::kThreads, CFG::kMinBlocks) k_list_hash_cta(ListParams P) {
    constexpr int kCThreads = CFG::kThreads;
    constexpr int kCWarps = CFG::kWarps;
    constexpr uint32_t kCMaxBits = CFG::kMaxBits;
    constexpr uint32_t kCMaxD = CFG::kMaxD;
    constexpr size_t kCTableBytes = cta_table_bytes<CFG>();
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned unit, next_block, total_blocks;
    using BS = cub::BlockScan<uint32_t, kCThreads>;
    __shared__ typename BS::TempStorage scan_tmp;
    unsigned char* tbase = dsm + warp_scratch_bytes<F>(kCWarps);
    constexpr uint32_t kSlotBytes = 16u << kCMaxBits, kWinBytes = kCWinBytes;
    BucketTable T{reinterpret_cast<uint32_t*>(tbase), reinterpret_cast<uint32_t*>(tbase + kSlotBytes + kWinBytes),
                  reinterpret_cast<unsigned*>(tbase + kSlotBytes + kWinBytes + kStash * 4),
                  reinterpret_cast<uint32_t*>(tbase + kSlotBytes),
                  window_base(P.n, min(P.win_bits, kCWinBits))};
    const unsigned rows = smem_addr(tbase + kCTableBytes);
    for (uint32_t i = threadIdx.x; i < (4u << kCMaxBits); i += kCThreads) T.slots[i] = kNone;
    for (uint32_t i = threadIdx.x; i < kWinBytes / 4; i += kCThreads) T.win[i] = 0u;
    if (threadIdx.x == 0) *T.nstash = 0;
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm, kCWarps);
    constexpr int PER = kCMaxD / kCThreads;  // set elements per thread
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unit = atomicAdd(P.queue, 1u);
            next_block = 0;
        }
        __syncthreads();
        const unsigned u = unit;
        if (u >= P.nseeds) break;
        const uint32_t seed = P.seeds[u];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        const uint32_t shift = bucket_shift(d, kCMaxBits);
        // table + row info (blocked: thread t owns set elements PER*t ..)
        uint32_t nb[PER];
        uint64_t ro[PER];
        uint32_t len[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = threadIdx.x * PER + k;
            nb[k] = 0;
            ro[k] = 0;
            len[k] = 0;
            if (i < d) {
                const uint32_t x = __ldg(P.set_adj + so + i);
                bucket_insert(T, shift, x);
                ro[k] = P.out_off[x];
                len[k] = static_cast<uint32_t>(P.out_off[x + 1] - ro[k]);
                nb[k] = (len[k] + 31u) >> 5;
            }
        }
        uint32_t agg;
        BS(scan_tmp).ExclusiveSum(nb, nb, agg);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = threadIdx.x * PER + k;
            if (i < d)
                sts128(rows + 16u * i, make_uint4(static_cast<uint32_t>(ro[k]), static_cast<uint32_t>(ro[k] >> 32),
                                                  len[k], nb[k]));
        }
        if (threadIdx.x == 0) total_blocks = agg;
        __syncthreads();
        const uint32_t nblocks = total_blocks;
        dispatch_probe(T, shift, *T.nstash, P.set_adj + so, d, P.variant, [&](const auto& probe) {
            cta_blocks<ALGO, F, CFG>(P, seed, so, d, rows, nblocks, probe, sink);
        });
        sink.end_unit(P, seed);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < d; k += kCThreads) bucket_clear(T, shift, __ldg(P.set_adj + so + k));
        if (threadIdx.x == 0) *T.nstash = 0;
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
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t* bm = P.bitmaps + (uint64_t)blockIdx.x * P.bitmap_words;
    Sink<ALGO, F> sink;
    attach_scratch(sink, dsm, kGWarps);
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) unit = atomicAdd(P.queue, 1u);
        __syncthreads();
        const unsigned u = unit;
        if (u >= P.nseeds) break;
        const uint32_t seed = P.seeds[u];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(P.set_adj + so + k);
            atomicOr(bm + (v >> 5), 1u << (v & 31));
        }
        __syncthreads();
        BitmapProbe probe{bm};
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
template <unsigned F> constexpr size_t smem_reg() { return warp_scratch_bytes<F>(kRWarps); }
template <unsigned F> constexpr size_t smem_hash_warp() { return warp_scratch_bytes<F>(kHWarps) + kHWarps * kHTableBytes; }
template <unsigned F, class CFG> constexpr size_t smem_hash_cta() { return warp_scratch_bytes<F>(CFG::kWarps) + cta_table_bytes<CFG>() + cta_row_bytes<CFG>(); }
template <unsigned F> constexpr size_t smem_giant() { return warp_scratch_bytes<F>(kGWarps); }

// ---- seed classification --------------------------------------------------
constexpr int kClasses = 5;  // R, H, C1, C2, G

struct SeedLists {
    uint32_t* lists[kClasses];
    unsigned int* counts;     // [kClasses]
};

__global__ void __launch_bounds__(256) k_classify_seeds(uint32_t n, const uint64_t* __restrict__ set_off,
                                                        SeedLists L) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t start = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t trips = (n + stride - 1) / stride;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t r = start + t * stride;
        uint64_t d = 0;
        if (r < n) d = set_off[r + 1] - set_off[r];
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
