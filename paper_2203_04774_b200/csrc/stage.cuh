// stage.cuh -- bulk-copy (TMA engine) staging of out-rows into shared memory.
//
// The listing inner loop streams the rows N+(x) of every x in a seed's set and
// probes each element. Issued as ordinary loads, a warp can only keep a few
// 128 B lines in flight, far below what HBM needs (~40+ KB per SM). Here each
// warp owns a ring of kNS shared-memory stages; a stage is filled by one
// cp.async.bulk (global -> shared, completion on an mbarrier) per row piece,
// issued lane-parallel, and the warp probes stage s while stages s+1..s+kNS-1
// are in flight. Rows are packed into a stage back to back at 16-byte
// granularity (the bulk-copy alignment); the lead / trail words outside a row
// are overwritten with kNone after arrival, so the probe loop is a plain
// 32-wide sweep of the stage with no per-element row bookkeeping.
#pragma once

#include "common.cuh"

namespace trigpu {

constexpr int kNS = 4;                          // stages per warp
constexpr int kStageSlots = 256;                // u32 slots per stage (1 KB)
constexpr int kStageBytes = kStageSlots * 4;
// per-warp area: stages | piece tables (uint4[32] per stage) | mbarriers
constexpr int kStageAreaBytes = kNS * kStageBytes + kNS * 512 + kNS * 8;  // 5152 B

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One warp's staging pipeline over the rows of set elements [xb, xe) of one
// seed (x = set_adj[so + i]).
struct Stager {
    unsigned area;        // shared address of this warp's kStageAreaBytes
    unsigned phases = 0;  // parity bit per stage (warp-uniform)
    // row source: lane l holds the row of x = set_adj[so + c + l]
    const uint32_t* xs = nullptr;  // set_adj + so
    uint32_t c = 0, xe = 0;
    uint32_t x = kNone;
    uint64_t ro = 0;
    uint32_t rl = 0;
    uint32_t r0 = 0, off0 = 0;  // cursor: next element is row r0 at offset off0
    bool done = false;

    __device__ __forceinline__ unsigned buf(int s) const { return area + s * kStageBytes; }
    __device__ __forceinline__ unsigned tab(int s) const { return area + kNS * kStageBytes + s * 512; }
    __device__ __forceinline__ unsigned bar(int s) const { return area + kNS * kStageBytes + kNS * 512 + s * 8; }

    __device__ __forceinline__ void init_barriers() {
        if (lane_id() == 0)
            for (int s = 0; s < kNS; ++s) mbar_init(bar(s), 1);
        mbar_fence_init();
        __syncwarp();
    }

    __device__ __forceinline__ void load_chunk(const uint64_t* out_off) {
        const uint32_t i = c + lane_id();
        x = kNone;
        ro = 0;
        rl = 0;
        if (i < xe) {
            x = __ldg(xs + i);
            ro = out_off[x];
            rl = static_cast<uint32_t>(out_off[x + 1] - ro);
        }
        r0 = 0;
        off0 = 0;
    }

    __device__ __forceinline__ void start(const uint32_t* set_row, uint32_t xb, uint32_t xend,
                                          const uint64_t* out_off) {
        xs = set_row;
        c = xb;
        xe = xend;
        done = xb >= xend;
        if (!done) load_chunk(out_off);
    }

    // Fill stage s with the next pieces of work; false when none is left.
    __device__ __forceinline__ bool issue(int s, const uint64_t* out_off, const uint32_t* out_adj) {
        const unsigned lane = lane_id();
        uint32_t rem;
        for (;;) {
            if (done) return false;
            rem = lane < r0 ? 0u : (lane == r0 ? rl - off0 : rl);
            if (__any_sync(FULL, rem != 0)) break;
            c += 32;
            if (c >= xe) {
                done = true;
                return false;
            }
            load_chunk(out_off);
        }
        const uint64_t st = ro + (lane == r0 ? off0 : 0u);
        const uint32_t lead = static_cast<uint32_t>(st) & 3u;  // words before st in its 16 B
        const uint32_t need = rem ? ((lead + rem + 3u) & ~3u) : 0u;
        const uint32_t incl = warp_incl_scan(need);
        const bool fits = rem != 0 && incl <= (uint32_t)kStageSlots;
        const unsigned nf = __ballot_sync(FULL, rem != 0 && !fits);
        const int q = nf ? __ffs(nf) - 1 : 32;
        // partial piece of row q in the room left
        uint32_t plen = fits ? rem : 0u;
        uint32_t pslot = incl - need;
        if (q < 32) {
            const uint32_t before = __shfl_sync(FULL, incl - need, q);
            const uint32_t lq = __shfl_sync(FULL, lead, q);
            const uint32_t remq = __shfl_sync(FULL, rem, q);
            const int room = (int)(((uint32_t)kStageSlots - before) & ~3u) - (int)lq;
            const uint32_t part = room > 0 ? min((uint32_t)room, remq) : 0u;
            if (lane == (unsigned)q) {
                plen = part;
                pslot = before;
            }
            // advance the cursor to (q, offset + part)
            const uint32_t base_off = (q == (int)r0) ? off0 : 0u;
            r0 = q;
            off0 = base_off + part;
        } else {
            r0 = 32;
            off0 = 0;
        }
        const uint32_t pwords = plen ? ((lead + plen + 3u) & ~3u) : 0u;
        const uint32_t bytes = __reduce_add_sync(FULL, pwords * 4u);
        // piece table: lane -> {first valid slot, length, x, padded words}
        sts128(tab(s) + 16u * lane, make_uint4(pslot + lead, plen, x, pwords));
        if (lane == 0) mbar_arrive_expect_tx(bar(s), bytes);
        __syncwarp();
        if (plen) {
            fence_proxy_async();
            bulk_g2s(buf(s) + 4u * pslot, out_adj + (st - lead), pwords * 4u, bar(s));
        }
        return true;
    }

    // Wait for stage s, blank its padding; returns the number of slots used.
    __device__ __forceinline__ uint32_t arrive(int s) {
        const unsigned lane = lane_id();
        mbar_wait(bar(s), (phases >> s) & 1u);
        phases ^= 1u << s;
        const uint4 e = lds128(tab(s) + 16u * lane);  // {first, len, x, words}
        if (e.y) {
            const uint32_t p0 = e.x & ~3u;  // piece start slot (16 B aligned)
            for (uint32_t k = p0; k < e.x; ++k) sts32(buf(s) + 4u * k, kNone);
            for (uint32_t k = e.x + e.y; k < p0 + e.w; ++k) sts32(buf(s) + 4u * k, kNone);
        }
        const uint32_t end = e.y ? (e.x & ~3u) + e.w : 0u;
        const uint32_t used = __reduce_max_sync(FULL, end);
        __syncwarp();
        return used;
    }

    // x owning slot f of stage s: the last piece whose first slot is <= f.
    // Piece lanes are contiguous; lanes before them read as 0, after as ~0,
    // so `first` is non-decreasing across lanes.
    __device__ __forceinline__ uint32_t owner_x(int s, uint32_t f) const {
        const unsigned lane = lane_id();
        const uint4 e = lds128(tab(s) + 16u * lane);
        const unsigned pm = __ballot_sync(FULL, e.y != 0);
        const unsigned lo_lane = pm ? __ffs(pm) - 1 : 0;
        const uint32_t first = e.y ? e.x : (lane < lo_lane ? 0u : 0xFFFFFFFFu);
        int k = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, first, k + step);
            if (v <= f) k += step;
        }
        return __shfl_sync(FULL, e.z, k);
    }
};

}  // namespace trigpu
