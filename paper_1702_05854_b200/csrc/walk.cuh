// Device-side primitives of one HSAW walk step: the xorshift64* stream, the start-node draw, the
// node-record load and the live in-edge pick with one-load verification. Shared by the encode
// kernel (K1) and the decode kernel (K2) so that generation and replay cannot disagree.
#pragma once

#include "common.cuh"

namespace hsawgpu {

// xorshift64* step, proj/include/hsaw/prng.hpp:41-48. Returns the scrambled output.
__device__ __forceinline__ uint64_t prg_next(uint64_t& s) {
    uint64_t x = s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    s = x;
    return x * 0x2545F4914F6CDD1DULL;
}

// One draw as the 53-bit integer k with u01 = k * 2^-53 (prng.hpp:51-53).
__device__ __forceinline__ uint64_t draw53(uint64_t& s) { return prg_next(s) >> 11; }

// splitmix step + zero skip, prng.hpp:29-38,65-72.
__device__ __forceinline__ uint64_t seed_from_worker(uint64_t worker_id) {
    uint64_t st = worker_id;
    for (;;) {
        uint64_t z = st + 0x9E3779B97F4A7C15ULL;
        uint64_t o = z;
        o ^= o >> 30;
        o *= 0xBF58476D1CE4E5B9ULL;
        o ^= o >> 27;
        o *= 0x94D049BB133111EBULL;
        o ^= o >> 31;
        if (o != 0) return o;
        st = z;
    }
}

// ---- draw sources of the walk kernels ------------------------------------------------------------
// XorRng is the reference's stream (xorshift64* chained through a batch): the bit-exact mode.
// PhiloxRng is the throughput mode of north_star item 2: a counter-based Philox4x32-10 substream
// per WALK INDEX (counter = walk id | draw-pair index, fixed key), so every attempt is an
// independent work item and a finished lane refills at once instead of carrying a 10-attempt
// chain. Its walks follow the same law but are not the reference's walks: statistical parity only.
struct XorRng {
    uint64_t s;
    __device__ __forceinline__ void start(uint64_t worker_id) {
        s = seed_from_worker(worker_id);  // sampler.cpp:272
#pragma unroll
        for (int i = 0; i < 8; ++i) (void)prg_next(s);  // burn-in, sampler.cpp:273
    }
    __device__ __forceinline__ uint64_t snapshot() const { return s; }
    __device__ __forceinline__ void restore(uint64_t snap) { s = snap; }
    __device__ __forceinline__ bool valid() const { return s != 0; }
    __device__ __forceinline__ uint64_t draw() { return draw53(s); }
    __device__ __forceinline__ void skip() { (void)prg_next(s); }
};

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                             uint32_t k0, uint32_t k1) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
}

struct PhiloxRng {
    uint64_t id;     // walk index: the encoded "seed" of the walk
    uint64_t spare;  // second 64-bit half of the last block
    uint32_t ctr;    // next draw-pair index
    uint32_t have;
    __device__ __forceinline__ void start(uint64_t walk_id) { restore(walk_id); }
    __device__ __forceinline__ uint64_t snapshot() const { return id; }
    __device__ __forceinline__ void restore(uint64_t snap) {
        id = snap;
        ctr = 0;
        have = 0;
    }
    __device__ __forceinline__ bool valid() const { return true; }
    __device__ __forceinline__ uint64_t draw() {
        if (have) {
            have = 0;
            return spare >> 11;
        }
        uint32_t c0 = (uint32_t)id, c1 = (uint32_t)(id >> 32), c2 = ctr++, c3 = 0x48534157u;  // "HSAW"
        uint32_t k0 = 0xA4093822u, k1 = 0x299F31D0u;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            philox_round(c0, c1, c2, c3, k0, k1);
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        spare = (uint64_t)c2 | ((uint64_t)c3 << 32);
        have = 1;
        return ((uint64_t)c0 | ((uint64_t)c1 << 32)) >> 11;
    }
    __device__ __forceinline__ void skip() { (void)draw(); }
};

// pick_uniform_node, prng.hpp:57-61: floor(fl(u01 * (double)n)) clamped to n-1. The product is a
// single IEEE round-to-nearest FP64 multiply on both sides (no FMA contraction possible).
__device__ __forceinline__ uint32_t start_node(uint64_t k, uint32_t n) {
    double r = __dmul_rn(__ull2double_rn(k), 0x1.0p-53);  // exact: k < 2^53
    uint32_t v = __double2uint_rz(__dmul_rn(r, __uint2double_rn(n)));
    return v < n ? v : n - 1;
}

// 256-bit read-only load of one node record (LDG.E.256 on sm_100a): one sector, one request.
__device__ __forceinline__ NodeRec load_node(const NodeRec* __restrict__ nodes, uint32_t v) {
    uint64_t a, b, c, d;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(nodes + v));
    NodeRec r;
    r.lo = (uint32_t)a;
    r.deg = (uint32_t)(a >> 32);
    r.tot_thr = b;
    r.acc_thr = c;
    r.scale = d;
    return r;
}

__device__ __forceinline__ EdgeRec load_edge(const EdgeRec* __restrict__ edges, uint64_t e) {
    uint64_t a, b, c, d;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(edges + e));
    EdgeRec r;
    r.thr = a;
    r.src = (uint32_t)b;
    r.prev_hi = (uint32_t)(b >> 32);
    r.src_lo = (uint32_t)c;
    r.src_deg = (uint32_t)(c >> 32);
    r.src_deficit = (uint32_t)d;
    r.flags = (uint32_t)(d >> 32);
    return r;
}

__device__ __forceinline__ uint32_t ceil_log2(uint32_t d) {  // d >= 1
    return d <= 1 ? 0u : 32u - __clz(d - 1);
}

// pick_live_in_edge (proj/include/hsaw/graph.hpp:61-80) for a draw k that already passed the
// "no edge" test (deg > 0 and k < tot_thr). Returns the slot index within the row: the first i
// with k < thr[lo+i] — identical to both the linear scan (:67-70) and the binary search (:72-78)
// of the reference because rows are non-decreasing. Fast path: one record load at the
// interpolation guess, verified against thr[g] and the packed top bits of thr[g-1]; anything the
// single load cannot prove falls back to a binary search over the row.
__device__ __forceinline__ uint32_t pick_slot(const EdgeRec* __restrict__ edges, uint32_t lo,
                                              uint32_t deg, uint64_t scale, uint64_t k,
                                              EdgeRec& rec_out) {
    uint64_t gq = __umul64hi(k << 11, scale) >> 31;
    uint32_t g = gq >= deg ? deg - 1 : (uint32_t)gq;
    EdgeRec rec = load_edge(edges, (uint64_t)lo + g);
    bool below = k < rec.thr;
    bool above_prev = g == 0 || (uint32_t)(k >> 21) > rec.prev_hi;
    if (below && above_prev) {
        rec_out = rec;
        return g;
    }
    // slow path: exact first index with k < thr, restricted to the side the probe ruled in
    // invariant: answer in [a, b] and k < thr[b] is known (thr[deg-1] == tot_thr > k)
    uint32_t a, b;
    if (below) {
        a = 0;
        b = g;
    } else {
        a = g + 1;
        b = deg - 1;
        if (a > b) a = b;  // unreachable for k < tot_thr; keeps the final load inside the row
    }
    while (a < b) {
        uint32_t mid = a + (b - a) / 2;
        EdgeRec pr = load_edge(edges, (uint64_t)lo + mid);
        if (k < pr.thr)
            b = mid;
        else
            a = mid + 1;
    }
    rec_out = load_edge(edges, (uint64_t)lo + a);
    return a;
}

// Row header of the picked edge's source node, when the edge record carries a usable one.
// Returns false when the node record must be read instead (suspect source or non-simple row).
__device__ __forceinline__ bool header_from_edge(const EdgeRec& rec, uint32_t& lo, uint32_t& deg,
                                                 uint64_t& tot, uint64_t& scale) {
    if ((rec.flags & (kEdgeSimple | kEdgeSuspect)) != kEdgeSimple) return false;
    lo = rec.src_lo;
    deg = rec.src_deg;
    tot = deg ? (1ull << 53) - rec.src_deficit : 0;
    scale = (uint64_t)deg << 31;  // guess hint for a row whose weights sum to ~1
    return true;
}

// ---- compact layout ------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t hdr_deg(uint32_t w) { return w & kHdrDegMask; }
__device__ __forceinline__ uint32_t hdr_mb(uint32_t w) { return (w >> kHdrDegBits) & 63u; }
__device__ __forceinline__ bool hdr_suspect(uint32_t w) { return (w >> 31) != 0; }

// (lo, w, acceptance code, 0): one 16-byte gather per arrival
__device__ __forceinline__ uint4 load_hdr(const uint4* __restrict__ hdr, uint32_t v) {
    uint4 h;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(h.x), "=r"(h.y), "=r"(h.z), "=r"(h.w)
                 : "l"(hdr + v));
    return h;
}

// in_src[e] of the compact layout: one gather, whatever the form (DeviceGraph::src_bits).
// BITS is a compile-time constant in the production kernel and s.bits elsewhere.
template <int BITS>
__device__ __forceinline__ uint32_t load_src_as(const uint32_t* __restrict__ p, uint64_t e,
                                                bool& dead) {
    if (BITS == 21) {  // three 21-bit entries per 64-bit word; e < 2^32
        const uint32_t q = __umulhi((uint32_t)e, 0xAAAAAAABu) >> 1;  // e / 3
        const uint32_t r = (uint32_t)e - 3 * q;
        uint64_t w;
        asm volatile("ld.global.nc.u64 %0, [%1];"
                     : "=l"(w)
                     : "l"(reinterpret_cast<const uint64_t*>(p) + q));
        const uint32_t v = (uint32_t)(w >> (21 * r)) & 0x1FFFFFu;
        dead = (v >> 20) != 0;
        return v & 0xFFFFFu;
    }
    uint32_t u;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(u) : "l"(p + e));
    if (BITS == 32) {
        dead = (u >> 31) != 0;
        return u & 0x7FFFFFFFu;
    }
    dead = false;
    return u;
}

__device__ __forceinline__ uint32_t load_src(const SrcRef& s, uint64_t e, bool& dead) {
    if (s.bits == 21) return load_src_as<21>(s.p, e, dead);
    if (s.bits == 32) return load_src_as<32>(s.p, e, dead);
    return load_src_as<0>(s.p, e, dead);
}

// Live-edge pick on an arithmetic row without touching the thresholds: slot = (k * deg) >> 53.
// Returns true when the draw is provably live and the slot exact, i.e. the fractional part of
// k * deg / 2^53 keeps the row's margin 2^mb clear of both slot boundaries (graph.cu,
// build_compact: the margin covers the distance of every threshold, the total-weight threshold
// included, from the ideal grid). deg < 2^25, k < 2^53: the product needs 78 bits.
__device__ __forceinline__ bool pick_arith(uint32_t w, uint64_t k, uint32_t& slot) {
    const uint32_t deg = hdr_deg(w);
    const uint64_t plo = k * deg, phi = __umul64hi(k, (uint64_t)deg);
    slot = (uint32_t)((plo >> 53) | (phi << 11));
    // margin test on the top 32 bits of the 53-bit fraction: fh >= mh and fh <= ~mh imply
    // 2^mb <= frac <= 2^53 - 2^mb (mh = 2^max(mb - 21, 0)); the few draws this rounds into the
    // margin take the exact path like the others. mb > 52 (kHdrSlow): never satisfied.
    const uint32_t mb = hdr_mb(w);
    const uint32_t mh = mb > 52 ? 0xFFFFFFFFu : (1u << (mb > 21 ? mb - 21 : 0));
    const uint32_t fh = (uint32_t)(plo >> 21);
    return fh >= mh && fh <= ~mh;
}

// Exact path of the compact layout: pick_live_in_edge (graph.hpp:61-80) from the node record and
// the threshold array. Returns -1 for "no edge", else the first slot i with k < thr[lo + i].
// Everything is passed and returned by value so that callers keep their walk state in registers.
static __device__ __noinline__ int64_t pick_exact_slot(const NodeRec* __restrict__ nodes,
                                                const uint64_t* __restrict__ thr, uint32_t v,
                                                uint64_t k) {
    NodeRec r = load_node(nodes, v);
    if (r.deg == 0 || k >= r.tot_thr) return -1;
    uint32_t a = 0, b = r.deg - 1;  // answer in [a, b]; k < thr[b] holds (thr[deg-1] == tot_thr)
    while (a < b) {
        uint32_t mid = a + (b - a) / 2;
        if (k < __ldg(thr + (uint64_t)r.lo + mid))
            b = mid;
        else
            a = mid + 1;
    }
    return (int64_t)a;
}

// Same, also reporting the row's true degree (the header field saturates at 2^25 - 1).
__device__ __forceinline__ bool pick_exact(const NodeRec* __restrict__ nodes,
                                           const uint64_t* __restrict__ thr, uint32_t v, uint64_t k,
                                           uint32_t& deg, uint32_t& slot) {
    int64_t r = pick_exact_slot(nodes, thr, v, k);
    deg = load_node(nodes, v).deg;
    if (r < 0) return false;
    slot = (uint32_t)r;
    return true;
}

// Algorithmic bytes of one pick in the reference layout:
// empty row 16; r >= total 24; success 28 + 8*ceil(log2 d). p_of (8) is added when resolve runs.
__device__ __forceinline__ uint32_t pick_alg_bytes(uint32_t deg, bool success) {
    if (deg == 0) return 16;
    if (!success) return 24;
    return 28 + 8 * ceil_log2(deg);
}

}  // namespace hsawgpu
