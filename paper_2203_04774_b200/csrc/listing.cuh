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
};

template <int ALGO, unsigned F>
struct Sink {
    unsigned long long cnt = 0, sum = 0;
    unsigned long long seed_hits = 0;

    // Called convergently by the whole warp once per 32-wide batch.
    __device__ __forceinline__ void batch(const ListParams& P, bool hit, uint32_t seed, uint32_t x,
                                          uint32_t y) {
        cnt += hit;
        if constexpr (F == 0u) return;
        if constexpr ((F & F_VCOUNT) != 0u) {
            if (hit) {
                atomicAdd(&P.vcount[x], 1ull);
                atomicAdd(&P.vcount[y], 1ull);
                ++seed_hits;
            }
        }
        if constexpr ((F & (F_CHECKSUM | F_LIST)) != 0u) {
            const uint32_t ru = ALGO == ALGO_APM ? seed : x;
            const uint32_t rv = ALGO == ALGO_APM ? x : y;
            const uint32_t rw = ALGO == ALGO_APM ? y : seed;
            uint32_t du = 0, dv = 0, dw = 0;
            if (hit) {
                du = P.inv[ru];
                dv = P.inv[rv];
                dw = P.inv[rw];
            }
            if constexpr ((F & F_CHECKSUM) != 0u)
                if (hit) sum += tri_hash(du, dv, dw);
            if constexpr ((F & F_LIST) != 0u) {
                const unsigned b = __ballot_sync(FULL, hit);
                if (b) {
                    const unsigned leader = __ffs(b) - 1;
                    unsigned long long base = 0;
                    if (lane_id() == leader) base = atomicAdd(&P.acc[2], (unsigned long long)__popc(b));
                    base = __shfl_sync(FULL, base, leader);
                    if (hit) {
                        const unsigned long long k = base + __popc(b & lanemask_lt());
                        if (k < P.tri_cap) {
                            P.tri[3 * k] = du;
                            P.tri[3 * k + 1] = dv;
                            P.tri[3 * k + 2] = dw;
                        }
                    }
                }
            }
        }
    }

    // End of one seed's unit: credit the seed's own per-vertex count.
    __device__ __forceinline__ void end_unit(const ListParams& P, uint32_t seed) {
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

// Walk the out-rows of up to 32 x's (x valid on lanes with xvalid) as one
// flattened stream, probing every element y against the seed's set.
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
    const unsigned ne = __ballot_sync(FULL, rl != 0);
    if (!ne) return;
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
    for (uint32_t base = 0; base < total; base += 32) {
        const unsigned bit = (crl != 0 && start >= base && start - base < 32u) ? (1u << (start - base)) : 0u;
        const unsigned M = __reduce_or_sync(FULL, bit);
        int j = before + __popc(M & le) - 1;
        before += __popc(M);
        j = j > 31 ? 31 : j;
        const uint32_t f = base + lane;
        const bool act = f < total;
        const uint64_t rb = shfl64(rbase, j);
        const uint32_t y = act ? __ldg(P.out_adj + rb + f) : kNone;
        const bool hit = probe(y, act);
        if constexpr (F == 0u) {
            sink.cnt += hit;
        } else {
            const uint32_t xx = __shfl_sync(FULL, cx, j);
            sink.batch(P, hit, seed, xx, y);
        }
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

struct HashProbe {  // open addressing, linear probing, kNone = empty
    const uint32_t* tab;
    uint32_t mask, shift;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        if (!act) return false;
        uint32_t h = slot_hash(y, shift);
        for (;;) {
            const uint32_t t = tab[h];
            if (t == y) return true;
            if (t == kNone) return false;
            h = (h + 1) & mask;
        }
    }
};

struct BitmapProbe {
    const uint32_t* bm;
    __device__ __forceinline__ bool operator()(uint32_t y, bool act) const {
        if (!act) return false;
        return (__ldcg(bm + (y >> 5)) >> (y & 31)) & 1u;
    }
};

__device__ __forceinline__ uint32_t table_bits(uint32_t d, uint32_t max_bits) {
    // smallest power of two >= 4d (load factor <= 1/4), at least 64 slots
    uint32_t bits = 32 - __clz(max(4u * d - 1u, 63u));
    return bits > max_bits ? max_bits : bits;
}

__device__ __forceinline__ void hash_insert(uint32_t* tab, uint32_t mask, uint32_t shift, uint32_t key) {
    uint32_t h = slot_hash(key, shift);
    while (atomicCAS(&tab[h], kNone, key) != kNone) h = (h + 1) & mask;
}

// ---- class R: |S| <= 32, warp per seed, S in registers -------------------
template <int ALGO, unsigned F>
__global__ void __launch_bounds__(256) k_list_reg(ListParams P) {
    const unsigned lane = lane_id();
    Sink<ALGO, F> sink;
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        const uint32_t s = lane < d ? __ldg(P.set_adj + so + lane) : kNone;
        RegProbe probe{s};
        scan_rows<ALGO, F>(P, seed, s, lane < d, probe, sink);
        sink.end_unit(P, seed);
    }
    sink.flush(P);
}

// ---- class H: 32 < |S| <= 256, warp per seed, per-warp smem hash --------
constexpr int kHWarps = 8;
constexpr uint32_t kHMaxBits = 10;  // 1024 slots per warp

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kHWarps * 32) k_list_hash_warp(ListParams P) {
    __shared__ uint32_t tabs[kHWarps][1u << kHMaxBits];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t* tab = tabs[warp];
    for (uint32_t i = lane; i < (1u << kHMaxBits); i += 32) tab[i] = kNone;
    __syncwarp();
    Sink<ALGO, F> sink;
    for (;;) {
        unsigned i = 0;
        if (lane == 0) i = atomicAdd(P.queue, 1u);
        i = __shfl_sync(FULL, i, 0);
        if (i >= P.nseeds) break;
        const uint32_t seed = P.seeds[i];
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        const uint32_t bits = table_bits(d, kHMaxBits);
        const uint32_t mask = (1u << bits) - 1, shift = 32 - bits;
        for (uint32_t k = lane; k < d; k += 32) hash_insert(tab, mask, shift, __ldg(P.set_adj + so + k));
        __syncwarp();
        HashProbe probe{tab, mask, shift};
        for (uint32_t c = 0; c < d; c += 32) {
            const bool xv = c + lane < d;
            const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
            scan_rows<ALGO, F>(P, seed, x, xv, probe, sink);
        }
        sink.end_unit(P, seed);
        __syncwarp();
        for (uint32_t k = lane; k <= mask; k += 32) tab[k] = kNone;
        __syncwarp();
    }
    sink.flush(P);
}

// ---- class C: 256 < |S| <= 4096, CTA per (seed, x-slice), smem hash ------
constexpr int kCThreads = 512;
constexpr uint32_t kCMaxBits = 14;  // 16384 slots = 64 KB
constexpr uint32_t kCSlice = 1024;  // x's per unit
constexpr uint32_t kCMaxSlices = 4096 / kCSlice;

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kCThreads) k_list_hash_cta(ListParams P) {
    extern __shared__ __align__(16) uint32_t ctab[];
    __shared__ unsigned unit;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    constexpr unsigned W = kCThreads / 32;
    for (uint32_t i = threadIdx.x; i < (1u << kCMaxBits); i += kCThreads) ctab[i] = kNone;
    Sink<ALGO, F> sink;
    uint32_t cur_seed = kNone, cur_mask = 0, cur_shift = 0;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) unit = atomicAdd(P.queue, 1u);
        __syncthreads();
        const unsigned u = unit;
        if (u >= P.nseeds * kCMaxSlices) break;
        const uint32_t seed = P.seeds[u / kCMaxSlices];
        const uint32_t slice = u % kCMaxSlices;
        const uint64_t so = P.set_off[seed];
        const uint32_t d = static_cast<uint32_t>(P.set_off[seed + 1] - so);
        if (slice * kCSlice >= d) continue;  // uniform across the CTA
        if (seed != cur_seed) {
            if (cur_seed != kNone)
                for (uint32_t k = threadIdx.x; k <= cur_mask; k += kCThreads) ctab[k] = kNone;
            __syncthreads();
            const uint32_t bits = table_bits(d, kCMaxBits);
            cur_mask = (1u << bits) - 1;
            cur_shift = 32 - bits;
            for (uint32_t k = threadIdx.x; k < d; k += kCThreads)
                hash_insert(ctab, cur_mask, cur_shift, __ldg(P.set_adj + so + k));
            cur_seed = seed;
            __syncthreads();
        }
        HashProbe probe{ctab, cur_mask, cur_shift};
        const uint32_t xb = slice * kCSlice, xe = min(d, xb + kCSlice);
        for (uint32_t c = xb + warp * 32; c < xe; c += W * 32) {
            const bool xv = c + lane < xe;
            const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
            scan_rows<ALGO, F>(P, seed, x, xv, probe, sink);
        }
        sink.end_unit(P, seed);
    }
    sink.flush(P);
}

// ---- class G: |S| > 4096, CTA per seed, global bitmap --------------------
constexpr int kGThreads = 1024;

template <int ALGO, unsigned F>
__global__ void __launch_bounds__(kGThreads) k_list_giant(ListParams P) {
    __shared__ unsigned unit;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    constexpr unsigned W = kGThreads / 32;
    uint32_t* bm = P.bitmaps + (uint64_t)blockIdx.x * P.bitmap_words;
    Sink<ALGO, F> sink;
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
        for (uint32_t c = warp * 32; c < d; c += W * 32) {
            const bool xv = c + lane < d;
            const uint32_t x = xv ? __ldg(P.set_adj + so + c + lane) : kNone;
            scan_rows<ALGO, F>(P, seed, x, xv, probe, sink);
        }
        sink.end_unit(P, seed);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < d; k += kGThreads) {
            const uint32_t v = __ldg(P.set_adj + so + k);
            __stcg(bm + (v >> 5), 0u);
        }
    }
    sink.flush(P);
}

// ---- seed classification --------------------------------------------------
struct SeedLists {
    uint32_t* lists[4];       // R, H, C, G
    unsigned int* counts;     // [4]
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
        if (d >= 2) cls = d <= 32 ? 0 : d <= 256 ? 1 : d <= 4096 ? 2 : 3;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
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
