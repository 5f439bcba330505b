// Sampler kernels for sm_100a:
//   K1  encode_kernel         thread_sample for a range of batches (proj/src/sampler.cpp:267-290)
//   K2  decode_kernel         DecodeContext::decode replay (proj/src/sampler.cpp:295-338)
//   K2b distinct_kernel(s)    the exact visited-set verdict of decode, on the materialised nodes
//
// Execution model: one lane owns one batch (K1) or one walk (K2) at a time — the
// xorshift64* chain inside a batch is strictly sequential — and the warp runs ONE flattened loop
// whose body is "one draw + at most one edge-record load + one node-record load" for every lane,
// whatever phase of its walk the lane is in. Lanes that finish refill from a global cursor with a
// warp-aggregated atomicAdd, so a warp never waits for its longest attempt.
#include <algorithm>
#include <cstdlib>

#include "sampler.cuh"
#include "walk.cuh"

namespace hsawgpu {

namespace {

constexpr int kThreads = 256;
constexpr int kDefaultEncodeBlocksPerSM = 5;  // 48 registers, no spills (ptxas -v)
constexpr int kDefaultRecordBlocksPerSM = 4;  // recording: 4 x 32 KB staging, measured best

struct EncodeParams {
    const NodeRec* nodes;
    const EdgeRec* edges;
    const uint4* hdr;      // compact layout (DeviceGraph)
    SrcRef src;
    const uint64_t* thr;
    uint32_t n;
    uint32_t l;       // attempts per batch
    uint32_t window;  // runtime width for the generic kernel
    uint64_t first_worker;
    uint64_t nbatches;
    uint64_t* out_seed;
    uint32_t* out_len;
    uint32_t* out_count;
    uint64_t* stats;   // u64[8]
    uint64_t* cursor;  // next batch index of this launch
    // recording variant (REC): accepted walks are logged as (node, edge id) pairs while they are
    // generated, so the replay kernel is only needed for the few walks that outgrow their chunk
    uint2* arena;            // pair log, carved into kLogChunk-pair chunks by atomicAdd
    uint32_t arena_cap;      // pairs
    uint32_t* arena_cursor;  // next free chunk (pairs)
    uint32_t* out_log;       // per (batch, seq) slot: first pair of the walk, or kLogOverflow
    uint32_t grow_mode;      // experiment, see grow_log (0 = off)
    // restricted variant (RESTR): start nodes drawn from `domain`, walks that move onto a node
    // outside `allowed` are aborted and counted per batch (sampler.cpp:24-31,196-199,528)
    const uint32_t* domain;
    uint32_t ndomain;
    const uint8_t* allowed;
    uint32_t* out_cross;
};

constexpr uint32_t kLogChunk = 4096;    // pairs per chunk (32 KB)
constexpr uint32_t kLogReserve = 1024;  // a new attempt starts only with this much room left
constexpr uint32_t kLogOverflow = 0xFFFFFFFFu;
constexpr uint32_t kStage = 16;         // pairs staged per thread in shared memory (128 bytes)

// 256-bit store of one full 32-byte sector (four pairs).
template <bool STREAMING>
__device__ __forceinline__ void store_sector(uint2* dst, uint2 a, uint2 b, uint2 c, uint2 d) {
    uint64_t x0 = (uint64_t)a.x | ((uint64_t)a.y << 32), x1 = (uint64_t)b.x | ((uint64_t)b.y << 32);
    uint64_t x2 = (uint64_t)c.x | ((uint64_t)c.y << 32), x3 = (uint64_t)d.x | ((uint64_t)d.y << 32);
    if (STREAMING)  // evict-first: the log is written once and read once, keep it out of L2's way
        asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "l"(x0), "l"(x1),
                     "l"(x2), "l"(x3));
    else
        asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "l"(x0), "l"(x1),
                     "l"(x2), "l"(x3));
}

// WindowFilter (proj/src/sampler.cpp:65-86) as a shift register of the last W pushed nodes: the
// ring buffer's content is exactly that set, and contains() only asks for membership.
template <int W>
struct Window {
    uint32_t r[W > 0 ? W : 1];
    __device__ __forceinline__ void reset(uint32_t, uint32_t v0) {
#pragma unroll
        for (int i = 0; i < W; ++i) r[i] = kInvalidNode;
        push(v0);
    }
    __device__ __forceinline__ bool contains(uint32_t u) const {
        bool c = false;
#pragma unroll
        for (int i = 0; i < W; ++i) c |= r[i] == u;
        return c;
    }
    __device__ __forceinline__ void push(uint32_t u) {
        if (W == 0) return;
#pragma unroll
        for (int i = W - 1; i > 0; --i) r[i] = r[i - 1];
        r[0] = u;
    }
};

// Runtime width 0..8 (any SamplerConfig::window, clamped to 8 as sampler.cpp:71 does).
template <>
struct Window<-1> {
    uint32_t r[8];
    uint32_t size;
    __device__ __forceinline__ void reset(uint32_t w, uint32_t v0) {
        size = w > 8 ? 8 : w;
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = kInvalidNode;
        push(v0);
    }
    __device__ __forceinline__ bool contains(uint32_t u) const {
        bool c = false;
#pragma unroll
        for (int i = 0; i < 8; ++i) c |= (i < (int)size) && r[i] == u;
        return c;
    }
    __device__ __forceinline__ void push(uint32_t u) {
        if (size == 0) return;
#pragma unroll
        for (int i = 7; i > 0; --i)
            if (i < (int)size) r[i] = r[i - 1];
        r[0] = u;
    }
};

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
    return v;
}

// Warp-aggregated claim of work items from a global cursor. Returns true and sets `mine` for
// lanes that wanted and got an item; sets `drained` (warp-uniform) once the cursor passed total.
__device__ __forceinline__ bool claim(uint64_t* cursor, uint64_t total, bool want, uint32_t lane,
                                      uint64_t& mine, bool& drained) {
    unsigned need = __ballot_sync(kFullMask, want);
    if (!need) return false;
    int leader = __ffs(need) - 1;
    uint64_t base = 0;
    if ((int)lane == leader)
        base = atomicAdd(reinterpret_cast<unsigned long long*>(cursor),
                         (unsigned long long)__popc(need));
    base = __shfl_sync(kFullMask, base, leader);
    if (base + __popc(need) >= total) drained = true;
    if (!want) return false;
    mine = base + __popc(need & ((1u << lane) - 1));
    return mine < total;
}

// FloydState::check's tortoise move (proj/src/sampler.cpp:121-137): the second cursor replays the
// attempt's own draw stream, so its pick is the one the hare made at that position (always live)
// and its resolve is never a hit; only the draws have to be consumed again. The cursor is kept as
// (generator state, node): the row comes from the node record and the exact pick of the layout,
// a non-default correctness path that costs three dependent reads per move. Returns the node the
// tortoise arrives at.
template <int LAYOUT, class RNG>
static __device__ __noinline__ uint32_t tortoise_step(const NodeRec* __restrict__ nodes,
                                                      const EdgeRec* __restrict__ edges,
                                                      const uint64_t* __restrict__ thr, SrcRef src,
                                                      RNG& t_rng, uint32_t t_node) {
    const NodeRec r = load_node(nodes, t_node);
    const uint64_t k = t_rng.draw();  // advance_edge, sampler.cpp:45
    uint32_t u;
    if (LAYOUT == kLayoutCompact) {
        const int64_t slot = pick_exact_slot(nodes, thr, t_node, k);
        bool dead;
        u = load_src(src, (uint64_t)r.lo + (uint32_t)(slot < 0 ? 0 : slot), dead);
    } else {
        EdgeRec e;
        (void)pick_slot(edges, r.lo, r.deg, r.scale, k, e);
        u = e.src;
    }
    if (load_node(nodes, u).acc_thr != 0) t_rng.skip();  // resolve(): a suspect costs one draw
    return u;
}

// ---- K1 ----------------------------------------------------------------------------------------
// HEUR: 0 Brent, 1 Floyd, 2 None (CycleHeuristic, proj/include/hsaw/sampler.hpp:46). WIN: window
// width or -1 for the runtime-width variant.
// REC: 0 plain encode, 1 record walks (default stores), 2 record with streaming (.cs) stores.
// STATS: per-lane work counters (draws, picks, algorithmic bytes) for instrumentation runs.
// LAYOUT: kLayoutFat (32-byte edge records) or kLayoutCompact (in_src + 8-byte row headers).
// Opt-in (HSAW_LOG_GROW=1; off by default, measured at the very end of round 2): a walk that fills
// its log chunk moves to a fresh run of chunks twice its length instead of being replayed by K2 -
// the pairs logged so far ([from, from + have): whole staged lines, all flushed) are copied by the
// lane itself with plain 8-byte volatile accesses and the walk goes on recording there; when the
// arena has no room the walk is replayed as before. At C4 this removes the replay (~80 walks per
// 2^20 batches, 1.5 ms of single-lane latency beside K2b's main pass): 22.07 -> 21.94 ms per step
// with a first version whose vectorised copy (ld.global.cg.v4 + the st.global.cs.v4.u64 asm of
// store_sector) turned out to lose the copied prefix when many lanes of a warp moved at once
// (ring tests); this plain copy passes them (tests/test_gpu_sampler.py::test_log_growth_opt_in).
__device__ __noinline__ uint32_t grow_log(uint2* arena, uint32_t* cursor, uint32_t cap,
                                          uint32_t from, uint32_t have, uint32_t need) {
    const uint32_t base = atomicAdd(cursor, need);
    if ((uint64_t)base + need > cap) return kLogOverflow;
    volatile unsigned long long* src = reinterpret_cast<volatile unsigned long long*>(arena + from);
    volatile unsigned long long* dst = reinterpret_cast<volatile unsigned long long*>(arena + base);
    for (uint32_t i = 0; i < have; i += 8) {  // `have` is a multiple of kStage; 8 loads in flight
        unsigned long long t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = src[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[i + q] = t[q];
    }
    return base;
}

template <int HEUR, int WIN, int MINB, int REC, bool STATS, int LAYOUT, bool RESTR = false,
          class RNG = XorRng>
__global__ void __launch_bounds__(kThreads, MINB) encode_kernel(EncodeParams p) {
    // REC: every thread stages kStage pairs (128 bytes) in shared memory, slot-major so the
    // 8-byte accesses are conflict-free, and flushes whole 128-byte lines: short failed attempts
    // never reach global memory and the log stream stays burst-friendly for HBM.
    __shared__ uint2 stage[REC ? kStage : 1][REC ? kThreads : 1];
    uint32_t lpos = 0, lend = 0, astart = 0;  // log write position / chunk end / attempt start
    bool rec_ok = false, arena_dead = false;
    // writes the staged pairs of line `base` (kStage-aligned), sectors [0, nsect)
    auto flush = [&](uint32_t base, uint32_t nsect) {
#pragma unroll
        for (uint32_t q = 0; q < kStage / 4; ++q)
            if (q < nsect)
                store_sector<REC == 2>(p.arena + base + 4 * q, stage[4 * q][threadIdx.x],
                                       stage[4 * q + 1][threadIdx.x], stage[4 * q + 2][threadIdx.x],
                                       stage[4 * q + 3][threadIdx.x]);
    };
    auto log_pair = [&](uint32_t node, uint32_t edge) {
        if (!REC || !rec_ok) return;
        if (lpos == lend) {  // the walk outgrew its chunk: it will be replayed instead
            const uint32_t have = lpos - astart;
            const uint32_t need = (2 * have + kLogChunk - 1) / kLogChunk * kLogChunk;
            const uint32_t moved = (arena_dead || p.grow_mode == 0)
                                       ? kLogOverflow
                                       : grow_log(p.arena, p.arena_cursor, p.arena_cap, astart, have, need);
            if (moved == kLogOverflow) {
                rec_ok = false;
                arena_dead = arena_dead || p.grow_mode != 0;
                return;
            }
            astart = moved;
            lpos = moved + have;
            lend = moved + need;
        }
        stage[lpos & (kStage - 1)][threadIdx.x] = make_uint2(node, edge);
        if ((lpos & (kStage - 1)) == kStage - 1) flush(lpos & ~(kStage - 1), kStage / 4);
        ++lpos;
    };
    const uint32_t lane = threadIdx.x & 31;
    const NodeRec* __restrict__ nodes = p.nodes;
    const EdgeRec* __restrict__ edges = p.edges;

    RNG rng{};
    uint64_t snapshot = 0;
    uint32_t bidx = 0;  // batch index within the launch (launches hold < 2^32 batches)
    uint32_t lo = 0, deg = 0;
    uint64_t tot = 0, scale = 0;  // fat layout: total-weight threshold and guess scale of the row
    uint32_t hw = 0, cur = 0;     // compact layout: header word and id of the current node
    uint32_t nedges = 0, att = 0, cnt = 0, ncross = 0;
    bool have = false, fresh = true, drained = false;
    Window<WIN> win;
    uint32_t b_anchor = kInvalidNode, b_power = 1, b_lam = 0;
    RNG t_rng{};                     // Floyd: the tortoise cursor (generator state, node)
    uint32_t t_node = kInvalidNode;
    // per-lane work counters; 32 bits suffice for one launch's share of one lane, except bytes
    uint32_t st_draws = 0, st_steps = 0, st_att = 0, st_acc = 0;
    uint64_t st_bytes = 0, st_pairs = 0;

    for (;;) {
        if (!drained) {
            uint64_t mine = 0;
            if (claim(p.cursor, p.nbatches, !have, lane, mine, drained)) {
                bidx = (uint32_t)mine;
                rng.start(p.first_worker + mine);  // seed + burn-in, sampler.cpp:272-273
                att = 0;
                cnt = 0;
                ncross = 0;
                fresh = true;
                have = true;
            }
        }
        if (!__any_sync(kFullMask, have)) break;
        if (!have) continue;

        // ---- one step of this lane's current attempt (run_walk_attempt, sampler.cpp:147-204)
        uint32_t u = 0;
        bool walking, from_edge = false;
        EdgeRec erec;
        if (fresh) {
            snapshot = rng.snapshot();  // Seed_h, sampler.cpp:155,277
            uint64_t k = rng.draw();
            u = RESTR ? __ldg(p.domain + start_node(k, p.ndomain))  // sampler.cpp:26-31
                      : start_node(k, p.n);                         // sampler.cpp:24
            nedges = 0;
            walking = true;
            if (STATS) st_draws += 1;
            if (STATS) st_att += 1;
            if (REC) {
                lpos = (lpos + kStage - 1) & ~(kStage - 1);  // walks start on a 128-byte line
                if (lend - lpos < kLogReserve && !arena_dead) {
                    uint32_t base = atomicAdd(p.arena_cursor, kLogChunk);
                    if (base <= p.arena_cap - kLogChunk) {
                        lpos = base;
                        lend = base + kLogChunk;
                    } else {
                        arena_dead = true;  // arena exhausted: remaining walks are replayed
                        lpos = lend = 0;
                    }
                }
                astart = lpos;
                rec_ok = lend - lpos >= kLogReserve;
                log_pair(u, kInvalidNode);
            }
        } else {
            walking = false;
            if (nedges < p.n) {  // len_cap = g.n, sampler.cpp:43,281
                uint64_t k = rng.draw();
                if (STATS) st_draws += 1;
                if (STATS) st_steps += 1;
                bool live;
                uint32_t slot_in_row = 0;
                if (LAYOUT == kLayoutCompact) {
                    uint32_t true_deg = deg;
                    if (deg == 0)
                        live = false;
                    else if (pick_arith(hw, k, slot_in_row))
                        live = true;
                    else  // draw inside the row's margin, or not an arithmetic row: exact path
                        live = pick_exact(nodes, p.thr, cur, k, true_deg, slot_in_row);
                    if (STATS) st_bytes += pick_alg_bytes(true_deg, live);
                    bool dead_end;
                    if (live) u = load_src(p.src, (uint64_t)lo + slot_in_row, dead_end);
                } else {
                    live = deg != 0 && k < tot;  // graph.hpp:66
                    if (STATS) st_bytes += pick_alg_bytes(deg, live);
                    if (live) {
                        slot_in_row = pick_slot(edges, lo, deg, scale, k, erec);
                        u = erec.src;
                        from_edge = true;
                    }
                }
                if (live) {
                    bool cyc = win.contains(u);  // sampler.cpp:180
                    if (HEUR == 0 && !cyc) {     // BrentState::check, sampler.cpp:100-108
                        if (u == b_anchor) {
                            cyc = true;
                        } else if (++b_lam == b_power) {
                            b_anchor = u;
                            b_power <<= 1;
                            b_lam = 0;
                        }
                    }
                    // FloydState::check, sampler.cpp:121-137: hare_pos counts the hare's steps that
                    // reached the check (= nedges + 1 here); every second one moves the tortoise
                    if (HEUR == 1 && !cyc && ((nedges + 1) & 1u) == 0) {
                        t_node = tortoise_step<LAYOUT>(nodes, edges, p.thr, p.src, t_rng, t_node);
                        cyc = t_node == u;
                    }
                    if (!cyc) {
                        ++nedges;  // resolve(), sampler.cpp:54
                        walking = true;
                        log_pair(u, lo + slot_in_row);
                    }
                }
            }
        }

        bool attempt_done = true;
        if (walking) {
            if (STATS) st_bytes += 8;  // p_of[u]
            NodeRec rec;
            uint32_t new_hw = 0;
            bool accepted = false;
            if (LAYOUT == kLayoutCompact) {
                // 8-byte row header of u; the node record is only read for suspects
                const uint4 h = load_hdr(p.hdr, u);
                rec.lo = h.x;
                rec.deg = hdr_deg(h.y);
                new_hw = h.y;
                if (hdr_suspect(h.y)) {  // is_suspect, sampler.cpp:32,55
                    const NodeRec full = load_node(nodes, u);
                    uint64_t k2 = rng.draw();
                    if (STATS) st_draws += 1;
                    accepted = k2 < full.acc_thr;  // r <= p_of[u], sampler.cpp:34,57
                }
            } else if (from_edge &&
                       header_from_edge(erec, rec.lo, rec.deg, rec.tot_thr, rec.scale)) {
                // Common case: u is not a suspect (no acceptance draw) and the edge record already
                // holds u's row header, so the walk continues without touching u's node record.
                rec.acc_thr = 0;
            } else {
                rec = load_node(nodes, u);
                if (rec.acc_thr != 0) {  // is_suspect, sampler.cpp:32,55
                    uint64_t k2 = rng.draw();
                    if (STATS) st_draws += 1;
                    accepted = k2 < rec.acc_thr;  // r <= p_of[u], sampler.cpp:34,57
                }
            }
            if (accepted) {
                uint64_t slot = (uint64_t)bidx * p.l + cnt;  // seq = index among accepted, :283
                p.out_seed[slot] = snapshot;
                p.out_len[slot] = nedges;
                if (REC) {
                    if (rec_ok) {
                        if (lpos & (kStage - 1))  // last, partially filled line
                            flush(lpos & ~(kStage - 1), ((lpos & (kStage - 1)) + 3) / 4);
                        p.out_log[slot] = astart;
                        astart = lpos;                    // keep the walk: later rewinds stop here
                    } else {
                        p.out_log[slot] = kLogOverflow;
                    }
                }
                ++cnt;
                if (STATS) st_acc += 1;
                if (STATS) st_pairs += nedges + 1;  // items of the accepted walk (8 B each logged)
            } else if (RESTR && !fresh && __ldg(p.allowed + u) == 0) {
                // continuing would need u's adjacency, which this part does not hold: the attempt
                // is aborted without another draw and counted as a crossing (sampler.cpp:196-199)
                ++ncross;
            } else {
                lo = rec.lo;
                deg = rec.deg;
                if (LAYOUT == kLayoutCompact) {
                    hw = new_hw;
                    cur = u;
                } else {
                    tot = rec.tot_thr;
                    scale = rec.scale;
                }
                if (fresh) {
                    win.reset(p.window, u);  // sampler.cpp:166-169
                    b_anchor = u;
                    b_power = 1;
                    b_lam = 0;
                    if (HEUR == 1) {  // FloydState::reset, sampler.cpp:116-122: the tortoise has
                        t_rng = rng;  // replayed the start draw and its resolve, like the hare
                        t_node = u;
                    }
                } else {
                    win.push(u);  // sampler.cpp:200
                }
                attempt_done = false;
                if (deg == 0) {
                    // The next pick is certain to fail after exactly one draw (empty row), unless
                    // the length cap stops it before drawing: settle it now, saving an iteration.
                    if (nedges < p.n) {
                        rng.skip();
                        if (STATS) st_draws += 1;
                        if (STATS) st_steps += 1;
                        if (STATS) st_bytes += 16;
                    }
                    attempt_done = true;
                }
            }
        }
        if (attempt_done) {
            fresh = true;
            if (REC) lpos = astart;  // failed attempt: reuse its log space (no-op after accept)
            if (++att == p.l) {
                p.out_count[bidx] = cnt;
                if (RESTR) p.out_cross[bidx] = ncross;
                have = false;
            }
        } else {
            fresh = false;
        }
    }

    if (!STATS) return;
    const uint64_t w_draws = warp_sum(st_draws), w_steps = warp_sum(st_steps);
    const uint64_t w_bytes = warp_sum(st_bytes), w_att = warp_sum(st_att);
    const uint64_t w_acc = warp_sum(st_acc);
    if (lane == 0 && p.stats) {
        auto* st = reinterpret_cast<unsigned long long*>(p.stats);
        atomicAdd(st + ST_ATTEMPTS, (unsigned long long)w_att);
        atomicAdd(st + ST_DRAWS, (unsigned long long)w_draws);
        atomicAdd(st + ST_STEPS, (unsigned long long)w_steps);
        atomicAdd(st + ST_BYTES, (unsigned long long)w_bytes);
        atomicAdd(st + ST_ACCEPTED, (unsigned long long)w_acc);
    }
    const uint64_t w_pairs = warp_sum(st_pairs);
    if (lane == 0 && p.stats)
        atomicAdd(reinterpret_cast<unsigned long long*>(p.stats) + ST_SPARE,
                  (unsigned long long)w_pairs);
}

// ---- K1, production variant ----------------------------------------------------------------------
// The default sampler configuration (Brent + window 2, recording) on the compact layout. Same
// stream, same outputs as encode_kernel; organised around the measured limits of the generic
// kernel once the graph is L2 resident (profiles/README.md): instruction issue, and memory waits
// taken by a single lane while the rest of the warp idles.
//  * one draw per iteration for every lane, hoisted out of the start / step branches;
//  * per step two dependent L2 gathers (in_src[e], then the 16-byte header of the source) and
//    nothing else: suspects are settled from the 32-bit acceptance code in the header, the node
//    record is read only for the 2^-32 ambiguous draws;
//  * the pair log is staged per thread in shared memory (rotated so that the per-step stores of a
//    warp and the line read-back are both conflict free) and full 128-byte lines are written out
//    by the whole warp at the end of the iteration instead of 45 instructions run by one lane.
constexpr int kFastBlocksPerSM = 5;

// STAGE: pairs staged per thread (one line of STAGE * 8 bytes per write-out).
// SRC_BITS: form of the source array (DeviceGraph::src_bits), a compile-time constant here.
template <int MINB, int STAGE, int SRC_BITS>
__global__ void __launch_bounds__(kThreads, MINB) encode_compact_kernel(EncodeParams p) {
    __shared__ __align__(16) uint2 stage[kThreads * STAGE];  // [thread][(pos + 2 lane) % STAGE]
    __shared__ uint64_t snap[kThreads];         // Seed_h of the running attempt
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const NodeRec* __restrict__ nodes = p.nodes;

    uint64_t s = 0;
    uint32_t bidx = 0, att = 0, cnt = 0;
    uint32_t lo = 0, hw = 0;                   // row start and header word of the current node
    uint32_t r0 = kInvalidNode, r1 = kInvalidNode;  // window(2): r0 is the current node
    uint32_t b_anchor = kInvalidNode, b_power = 1, b_lam = 0;
    uint32_t nedges = 0;
    uint32_t lpos = 0, lend = 0, astart = 0;
    bool have = false, fresh = true, drained = false, rec_ok = false, arena_dead = false;

    for (;;) {
        if (!drained) {
            uint64_t mine = 0;
            if (claim(p.cursor, p.nbatches, !have, lane, mine, drained)) {
                bidx = (uint32_t)mine;
                s = seed_from_worker(p.first_worker + mine);  // sampler.cpp:272
#pragma unroll
                for (int i = 0; i < 8; ++i) (void)prg_next(s);  // burn-in, sampler.cpp:273
                att = 0;
                cnt = 0;
                fresh = true;
                have = true;
            }
        }
        if (!__any_sync(kFullMask, have)) break;

        uint32_t flush_n = 0, flush_base = 0;  // pairs of a staged line to write out below
        bool arrive = false;
        uint32_t u = 0, edge = kInvalidNode;
        if (have) {
            const uint64_t s_before = s;
            const uint64_t k = draw53(s);  // start draw or pick draw
            if (fresh) {
                snap[tid] = s_before;     // Seed_h, sampler.cpp:155,277
                u = start_node(k, p.n);  // sampler.cpp:24
                nedges = 0;
                lpos = (lpos + STAGE - 1) & ~(STAGE - 1);  // walks start on a 128-byte line
                if (lend - lpos < kLogReserve && !arena_dead) {
                    uint32_t base = atomicAdd(p.arena_cursor, kLogChunk);
                    if (base <= p.arena_cap - kLogChunk) {
                        lpos = base;
                        lend = base + kLogChunk;
                    } else {
                        arena_dead = true;  // arena exhausted: remaining walks are replayed
                        lpos = lend = 0;
                    }
                }
                astart = lpos;
                rec_ok = lend - lpos >= kLogReserve;
                arrive = true;
            } else if (nedges >= p.n) {
                s = s_before;  // len_cap = g.n stops before drawing, sampler.cpp:43,281
            } else {
                // rows with deg == 0 never get here: they are settled on arrival (below)
                uint32_t slot = 0;
                bool live = pick_arith(hw, k, slot);
                if (!live) {  // draw inside the row's margin, or not an arithmetic row
                    const int64_t ex = pick_exact_slot(nodes, p.thr, r0, k);
                    live = ex >= 0;
                    slot = (uint32_t)ex;
                }
                if (live) {
                    bool dead_end;
                    u = load_src_as<SRC_BITS>(p.src.p, (uint64_t)lo + slot, dead_end);
                    bool cyc = (u == r0) | (u == r1);  // sampler.cpp:180
                    if (!cyc) {                        // BrentState::check, sampler.cpp:100-108
                        if (u == b_anchor) {
                            cyc = true;
                        } else if (++b_lam == b_power) {
                            b_anchor = u;
                            b_power <<= 1;
                            b_lam = 0;
                        }
                    }
                    if (!cyc) {
                        ++nedges;  // resolve(), sampler.cpp:54
                        if (dead_end) {
                            // u is no suspect (no acceptance draw) and has no in-edges: the next
                            // pick fails after exactly one draw unless the length cap stops it
                            // before drawing. Settled here, without reading u's header.
                            if (nedges < p.n) (void)prg_next(s);
                        } else {
                            edge = lo + slot;
                            arrive = true;
                        }
                    }
                }
            }
        }
        __syncwarp();  // starting and stepping lanes arrive together: one header read per iteration

        bool done = true;
        if (arrive) {
            const uint4 h = load_hdr(p.hdr, u);
            const uint32_t a32 = h.z;
            if (rec_ok) {
                if (lpos == lend) {  // the walk outgrew its chunk: it will be replayed
                    rec_ok = false;
                } else {
                    stage[tid * STAGE + ((lpos + 2 * lane) & (STAGE - 1))] = make_uint2(u, edge);
                    ++lpos;
                    if ((lpos & (STAGE - 1)) == 0) {
                        flush_n = STAGE;
                        flush_base = lpos - STAGE;
                    }
                }
            }
            bool accepted = false;
            if (a32 != 0) {  // is_suspect, sampler.cpp:32,55
                const uint64_t k2 = draw53(s);
                const uint32_t k2h = (uint32_t)(k2 >> 21);
                if (a32 != 0xFFFFFFFFu && k2h != a32 - 1)
                    accepted = k2h < a32 - 1;
                else  // r <= p_of[u] against the exact threshold, sampler.cpp:34,57
                    accepted = k2 < load_node(nodes, u).acc_thr;
            }
            if (accepted) {
                const uint64_t out = (uint64_t)bidx * p.l + cnt;  // seq, sampler.cpp:283
                p.out_seed[out] = snap[tid];
                p.out_len[out] = nedges;
                if (rec_ok) {
                    if (lpos & (STAGE - 1)) {  // last, partially filled line: whole sectors
                        flush_n = ((lpos & (STAGE - 1)) + 3) & ~3u;
                        flush_base = lpos & ~(STAGE - 1);
                    }
                    p.out_log[out] = astart;
                    astart = lpos;  // keep the walk: later rewinds stop here
                } else {
                    p.out_log[out] = kLogOverflow;
                }
                ++cnt;
            } else {
                lo = h.x;
                hw = h.y;
                if (fresh) {  // win.reset / brent.reset, sampler.cpp:166-169
                    r1 = kInvalidNode;
                    b_anchor = u;
                    b_power = 1;
                    b_lam = 0;
                } else {
                    r1 = r0;  // win.push, sampler.cpp:200
                }
                r0 = u;
                done = false;
                if (hdr_deg(hw) == 0) {
                    // the next pick fails after exactly one draw (empty row) unless the
                    // length cap stops it before drawing: settle it now
                    if (nedges < p.n) (void)prg_next(s);
                    done = true;
                }
            }
        }
        if (have) {
            if (done) {
                fresh = true;
                lpos = astart;  // failed attempt: reuse its log space (no-op after an accept)
                if (++att == p.l) {
                    p.out_count[bidx] = cnt;
                    have = false;
                }
            } else {
                fresh = false;
            }
        }

        // write-out of the staged line that filled up in this iteration (or of the last, partial
        // line of an accepted walk, whole sectors): every such lane copies its own 64 bytes with
        // 128-bit shared loads and 256-bit streaming stores; the lanes that have nothing to write
        // just sit the few instructions out
        if (flush_n != 0) {
            uint2* dst = p.arena + flush_base;
#pragma unroll
            for (uint32_t q = 0; q < STAGE / 4; ++q) {
                if (4 * q < flush_n) {
                    const uint4 a = *reinterpret_cast<const uint4*>(
                        &stage[tid * STAGE + ((4 * q + 2 * lane) & (STAGE - 1))]);
                    const uint4 b = *reinterpret_cast<const uint4*>(
                        &stage[tid * STAGE + ((4 * q + 2 + 2 * lane) & (STAGE - 1))]);
                    asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(
                                     dst + 4 * q),
                                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y),
                                 "r"(b.z), "r"(b.w));
                }
            }
        }
    }
}

// ---- K2 ----------------------------------------------------------------------------------------
struct DecodeParams {
    const NodeRec* nodes;
    const EdgeRec* edges;
    const uint4* hdr;  // compact layout (DeviceGraph)
    SrcRef src;
    const uint64_t* thr;
    uint32_t n;
    uint64_t nwalks;
    const uint64_t* seed;
    const uint32_t* len;
    const uint64_t* edge_off;
    uint32_t* out_nodes;
    uint32_t* out_edges;
    uint8_t* status;
    uint32_t* nnodes;  // nullable: nodes written per walk (only needed for foreign encodings)
    uint64_t* stats;
    uint64_t* cursor;
    // PAIRS mode (replay of walks whose log overflowed): work item i is walk sel[i] and its
    // (node, edge id) pairs go to pair_dst[sel[i]]
    const uint32_t* sel;
    uint2* const* pair_dst;
    // restricted replay (decode_restricted, sampler.cpp:299-338): the start node comes from the domain
    const uint32_t* domain;
    uint32_t ndomain;
};

template <bool PAIRS, int LAYOUT, class RNG = XorRng>
__global__ void __launch_bounds__(kThreads) decode_kernel(DecodeParams p) {
    const uint32_t lane = threadIdx.x & 31;
    const NodeRec* __restrict__ nodes = p.nodes;
    const EdgeRec* __restrict__ edges = p.edges;

    RNG rng{};
    uint64_t w = 0, base = 0;
    uint2* pairs = nullptr;
    uint32_t lo = 0, deg = 0, len = 0, nedges = 0;
    uint64_t tot = 0, scale = 0;
    uint32_t hw = 0, cur = 0;  // compact layout: header word and id of the current node
    bool have = false, fresh = true, drained = false;
    uint64_t st_steps = 0;

    for (;;) {
        if (!drained) {
            uint64_t mine = 0;
            if (claim(p.cursor, p.nwalks, !have, lane, mine, drained)) {
                w = PAIRS ? p.sel[mine] : mine;
                rng.restore(p.seed[w]);
                len = p.len[w];
                if (PAIRS)
                    pairs = p.pair_dst[w];
                else
                    base = p.edge_off[w];
                fresh = true;
                have = true;
            }
        }
        if (!__any_sync(kFullMask, have)) break;
        if (!have) continue;

        uint32_t verdict = 0;  // 0 keep walking, 1 decoded, 2 mismatch
        uint32_t u = 0;
        bool arrived = false, from_edge = false;
        EdgeRec erec;
        if (fresh) {
            if (!rng.valid()) {
                verdict = 2;  // "decode: zero seed state", sampler.cpp:306
                nedges = 0;
                if (p.nnodes) p.nnodes[w] = 0;
            } else {
                uint64_t k = rng.draw();
                u = p.domain ? __ldg(p.domain + start_node(k, p.ndomain)) : start_node(k, p.n);
                nedges = 0;
                if (PAIRS)
                    pairs[0] = make_uint2(u, kInvalidNode);
                else
                    p.out_nodes[base + w] = u;
                arrived = true;
            }
        } else {
            // advance_edge with len_cap = n (sampler.cpp:322-324): any stop here is a mismatch
            if (nedges >= p.n) {
                verdict = 2;
            } else {
                uint64_t k = rng.draw();
                st_steps += 1;
                bool live;
                uint32_t slot = 0;
                if (LAYOUT == kLayoutCompact) {
                    uint32_t true_deg = deg;
                    if (deg == 0)
                        live = false;
                    else if (pick_arith(hw, k, slot))
                        live = true;
                    else
                        live = pick_exact(nodes, p.thr, cur, k, true_deg, slot);
                    bool dead_end;
                    if (live) u = load_src(p.src, (uint64_t)lo + slot, dead_end);
                } else {
                    live = deg != 0 && k < tot;
                    if (live) {
                        slot = pick_slot(edges, lo, deg, scale, k, erec);
                        u = erec.src;
                        from_edge = true;
                    }
                }
                if (!live) {
                    verdict = 2;
                } else {
                    if (PAIRS) {
                        ++nedges;
                        pairs[nedges] = make_uint2(u, lo + slot);
                    } else {
                        p.out_edges[base + nedges] = lo + slot;
                        ++nedges;
                        p.out_nodes[base + w + nedges] = u;
                    }
                    arrived = true;
                }
            }
        }
        if (arrived) {
            NodeRec rec;
            uint32_t new_hw = 0;
            bool hit = false;
            if (LAYOUT == kLayoutCompact) {
                const uint4 h = load_hdr(p.hdr, u);
                rec.lo = h.x;
                rec.deg = hdr_deg(h.y);
                new_hw = h.y;
                if (hdr_suspect(h.y)) hit = rng.draw() < load_node(nodes, u).acc_thr;
            } else if (from_edge &&
                       header_from_edge(erec, rec.lo, rec.deg, rec.tot_thr, rec.scale)) {
                rec.acc_thr = 0;
            } else {
                rec = load_node(nodes, u);
                if (rec.acc_thr != 0) hit = rng.draw() < rec.acc_thr;
            }
            if (hit) {
                verdict = nedges == len ? 1 : 2;  // sampler.cpp:311-314, 329-332
            } else if (nedges >= len) {
                verdict = 2;  // sampler.cpp:316-317, 334-335
            } else {
                lo = rec.lo;
                deg = rec.deg;
                if (LAYOUT == kLayoutCompact) {
                    hw = new_hw;
                    cur = u;
                } else {
                    tot = rec.tot_thr;
                    scale = rec.scale;
                }
                fresh = false;
            }
        }
        if (verdict != 0) {
            p.status[w] = (uint8_t)verdict;
            if (p.nnodes && !(fresh && !rng.valid())) p.nnodes[w] = nedges + 1;
            have = false;
        }
    }
    st_steps = warp_sum(st_steps);
    if (lane == 0 && p.stats)
        atomicAdd(reinterpret_cast<unsigned long long*>(p.stats) + ST_DECODE_STEPS,
                  (unsigned long long)st_steps);
}

// ---- K2b ---------------------------------------------------------------------------------------
// Verdict to reproduce (sampler.cpp:318-337): the walk is dropped iff its replayed nodes are not
// pairwise distinct. One warp per walk; <= 32 nodes: one __match_any_sync; <= kSmemNodes: an
// open-addressing hash set in shared memory; longer walks are queued for distinct_long_kernel.
// Two table sizes: the main pass keeps 48 warps per SM resident (six blocks: launch_distinct_check) with 4 KB tables (walks of up to
// 512 nodes); the few longer walks are queued for a second pass with 16 KB tables, and walks beyond
// that for the block-per-walk kernel.
#ifndef HSAW_K2B_LOAD
#define HSAW_K2B_LOAD 4
#endif
constexpr uint32_t kTableLoad = HSAW_K2B_LOAD;  // slots per node before rounding up to a power of two
#ifndef HSAW_K2B_BITMAP
#define HSAW_K2B_BITMAP 1
#endif
constexpr bool kBitmapProof = HSAW_K2B_BITMAP != 0;  // compile-time A/B of the bit-map fast path
constexpr int kCheckWarps = 8, kMidWarps = 4;
constexpr int kCheckMinBlocks = 6;  // register budget of the main pass (blocks per SM), see launch_distinct_check
constexpr uint32_t kTableSize = 1024, kMidTableSize = 4096;  // u32 slots per warp
constexpr uint32_t kSmemNodes = kMidTableSize / 2;           // largest walk handled in shared memory

struct CheckParams {
    uint64_t nwalks;
    const uint64_t* edge_off;
    const uint32_t* nodes;
    const uint32_t* nnodes;  // nullable: default len + 1
    // pair-log source (fused path): walk w = pair_src[w][0 .. lens[w]] (.x = node)
    const uint2* const* pair_src;
    const uint32_t* lens;
    uint8_t* status;
    uint32_t* long_list;   // (walk id, node count) pairs needing the long path
    uint32_t* long_count;  // [0] long walks queued, [1] walks dropped (status 1 -> 0), [2] mid queued
    uint32_t long_cap;
    uint32_t* mid_list;    // walk ids queued for the 16 KB-table pass
    uint32_t mid_cap;
    const uint32_t* sel;   // non-null: the work items are sel[0 .. nwalks)
};

__device__ __forceinline__ uint32_t node_hash(uint32_t v, uint32_t bits) {
    return (v * 2654435761u) >> (32 - bits);
}

template <bool PAIRS>
__device__ __forceinline__ uint32_t walk_node(const CheckParams& p, uint64_t w, uint64_t base,
                                              uint32_t i) {
    if (PAIRS) return p.pair_src[w][i].x;
    return p.nodes[base + i];
}

// Work is dealt in groups of 32 consecutive walks per warp: lane j reads the metadata of walk j of
// the group (coalesced), the walks are then processed one by one with their metadata broadcast by
// shuffles, and every lane has up to four node reads in flight before the first insert, so a walk
// costs one exposed memory latency per 128 nodes instead of one per 32.
// GROUP: walks dealt to a warp at a time (32 for the bulk pass; 1 for the short queues of long
// walks, where 32 serial long walks per warp would leave most of the GPU idle).
// MINB: resident blocks per SM the register budget is held to (the main pass: 6 x 32 KB of tables
// fill the shared memory of an SM; without the bound the kernel takes 52 registers, four blocks).
template <bool PAIRS, uint32_t TABLE, int WARPS, uint32_t GROUP, int MINB = 1>
__global__ void __launch_bounds__(WARPS * 32, MINB) distinct_kernel(CheckParams p) {
    extern __shared__ __align__(16) uint32_t tables[];  // WARPS x TABLE
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    uint32_t* tab = tables + wib * TABLE;
    const uint64_t warp = (uint64_t)blockIdx.x * WARPS + wib;
    const uint64_t nwarps = (uint64_t)gridDim.x * WARPS;
    const uint64_t ngroups = (p.nwalks + GROUP - 1) / GROUP;
    uint32_t dropped = 0;
    for (uint64_t grp = warp; grp < ngroups; grp += nwarps) {
        const uint64_t item = grp * GROUP + lane;
        uint64_t my_w = 0, my_src = 0;  // walk id; pair-log pointer or offset into p.nodes
        uint32_t my_nn = 0;
        uint8_t my_st = 0;
        if (lane < GROUP && item < p.nwalks) {
            my_w = p.sel ? p.sel[item] : item;
            my_st = p.status[my_w];
            if (my_st != 0) {
                if (PAIRS) {
                    my_nn = p.lens[my_w] + 1;
                    my_src = reinterpret_cast<uint64_t>(p.pair_src[my_w]);
                } else {
                    my_nn = p.nnodes ? p.nnodes[my_w]
                                     : (uint32_t)(p.edge_off[my_w + 1] - p.edge_off[my_w]) + 1;
                    my_src = p.edge_off[my_w] + my_w;
                }
            }
        }
        unsigned todo = __ballot_sync(kFullMask, my_nn > 1);  // a single node cannot repeat
        auto node_of = [&](uint64_t srcv, uint32_t i) -> uint32_t {
            if (PAIRS) return __ldg(&reinterpret_cast<const uint2*>(srcv)[i].x);
            return __ldg(p.nodes + srcv + i);
        };
        // The first 128 nodes of the NEXT walk of the group are requested before the current
        // walk's inserts start, so the load latency of a walk hides behind the table work of its
        // predecessor instead of being paid once per walk (the walks of a warp run back to back).
        uint32_t pre[4];
        uint32_t pre_nn = 0;
        uint64_t pre_src = 0;
        auto prefetch = [&](unsigned rest) {
            if (!rest) return;
            const int jn = __ffs(rest) - 1;
            pre_nn = __shfl_sync(kFullMask, my_nn, jn);
            pre_src = __shfl_sync(kFullMask, my_src, jn);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t i = q * 32 + lane;
                pre[q] = i < pre_nn ? node_of(pre_src, i) : kInvalidNode;
            }
        };
        prefetch(todo);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t nn = pre_nn;
            const uint64_t srcv = pre_src;
            uint32_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = pre[q];
            prefetch(todo);
            auto node_at = [&](uint32_t i) -> uint32_t { return node_of(srcv, i); };
            bool dup = false;
            if (nn <= 32) {
                unsigned valid = nn == 32 ? kFullMask : ((1u << nn) - 1);
                unsigned same = __match_any_sync(kFullMask, v[0]) & valid & ~(1u << lane);
                dup = __any_sync(kFullMask, lane < nn && same != 0);
            } else if (nn <= TABLE / 2) {
                // table of >= 4*nn slots where the warp's share allows it, else >= 2*nn: lanes
                // probe in lockstep, so the longest probe sequence of the 32 sets the pace
                // HSAW_K2B_LOAD (compile-time A/B): table of >= 4*nn slots; 2*nn was measured slower (C4: K2b 2.7 -> 3.5 ms per step: the lanes probe in lockstep, the longest probe sets the pace)
                uint32_t bits = 32 - __clz(kTableLoad * nn - 1);
                if ((1u << bits) > TABLE) --bits;
                const uint32_t size = 1u << bits;
                bool mydup = false;
                // Fast proof of distinctness first: every node sets two hashed bits of a
                // 32*TABLE-bit map (the same shared memory); a node that finds one of its bits
                // clear differs from every node before it, so if that holds for all of them the
                // walk is done - two atomicOr per node, no probing, no lockstep tails. Only walks
                // in which some node finds both bits set (a true repeat, or chance) go through
                // the exact hash set below.
                bool exact_needed = true;
                // (worth it while false alarms stay rare: with two bits per node about
                // nn^3 / (3 * (16 TABLE)^2) of the walks, 8 % at 400 nodes in the main pass)
                if (kBitmapProof && (uint64_t)nn * nn * nn <= 24ull * TABLE * TABLE * 16 / 6) {
                    constexpr uint32_t kMapBits = 5 + (TABLE == 1024 ? 10 : TABLE == 4096 ? 12 : 0);
                    static_assert(TABLE == 1024 || TABLE == 4096, "bit-map width follows the table size");
                    for (uint32_t i = lane; i < TABLE / 4; i += 32)  // 128-bit stores
                        reinterpret_cast<uint4*>(tab)[i] = make_uint4(0u, 0u, 0u, 0u);
                    __syncwarp();
                    uint32_t coll = 0;
                    uint32_t first[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) first[q] = v[q];
                    for (uint32_t c = 0; c < nn; c += 128) {
                        uint32_t x[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t i = c + q * 32 + lane;
                            x[q] = c == 0 ? first[q] : (i < nn ? node_at(i) : kInvalidNode);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (c + q * 32 + lane >= nn) continue;
                            // two bits per node: a node equal to an earlier one finds BOTH set;
                            // finding either clear proves it new (0.4 % false alarms at 131
                            // nodes, against 23 % with one bit)
                            const uint32_t r1 = (x[q] * 0x85EBCA6Bu) >> (32 - kMapBits);
                            const uint32_t r2 = (x[q] * 0xC2B2AE35u) >> (32 - kMapBits);
                            const uint32_t o1 = atomicOr(&tab[r1 >> 5], 1u << (r1 & 31)) >> (r1 & 31);
                            const uint32_t o2 = atomicOr(&tab[r2 >> 5], 1u << (r2 & 31)) >> (r2 & 31);
                            coll |= o1 & o2;
                        }
                    }
                    exact_needed = __any_sync(kFullMask, coll & 1u);
                    __syncwarp();
                }
                for (uint32_t c = 0; exact_needed && c < nn; c += 128) {
                    if (c != 0) {  // (the first 128 were requested one walk ahead)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t i = c + q * 32 + lane;
                            v[q] = i < nn ? node_at(i) : kInvalidNode;
                        }
                    }
                    if (c == 0) {  // the clears overlap the reads in flight
                        // (nn > 32 here, so size >= 128 words: whole 128-bit stores per lane)
                        for (uint32_t i = lane; i < size / 4; i += 32)
                            reinterpret_cast<uint4*>(tab)[i] =
                                make_uint4(kInvalidNode, kInvalidNode, kInvalidNode, kInvalidNode);
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (c + q * 32 + lane >= nn) continue;
                        uint32_t h = node_hash(v[q], bits);
                        for (;;) {
                            uint32_t old = atomicCAS(&tab[h], kInvalidNode, v[q]);
                            if (old == kInvalidNode) break;
                            if (old == v[q]) {
                                mydup = true;
                                break;
                            }
                            h = (h + 1) & (size - 1);
                        }
                    }
                }
                dup = __any_sync(kFullMask, mydup);
                __syncwarp();
            } else {
                const uint32_t w32 = (uint32_t)__shfl_sync(kFullMask, my_w, j);
                if (lane == 0) {
                    if (nn <= kSmemNodes) {  // too long for this pass's table: the mid pass
                        uint32_t at = atomicAdd(p.long_count + 2, 1u);
                        if (at < p.mid_cap) p.mid_list[at] = w32;
                    } else {
                        uint32_t at = atomicAdd(p.long_count, 1u);
                        if (at < p.long_cap) {
                            p.long_list[2 * at] = w32;
                            p.long_list[2 * at + 1] = nn;
                        }
                    }
                }
                continue;
            }
            if (dup && (int)lane == j) {  // the lane that owns the walk's metadata records the verdict
                p.status[my_w] = 0;
                if (my_st == 1) ++dropped;
            }
        }
    }
    if (dropped) atomicAdd(p.long_count + 1, dropped);
}

// Long walks (> kSmemNodes nodes): one block per walk, hash set in global scratch.
template <bool PAIRS>
__global__ void __launch_bounds__(256) distinct_long_kernel(CheckParams p, uint32_t nlong,
                                                            const uint64_t* table_off,
                                                            uint32_t* tables) {
    uint32_t i = blockIdx.x;
    if (i >= nlong) return;
    uint32_t w = p.long_list[2 * i];
    uint64_t base = PAIRS ? 0 : p.edge_off[w] + w;
    uint32_t nn = p.long_list[2 * i + 1];
    uint32_t* tab = tables + table_off[i];
    uint64_t size = table_off[i + 1] - table_off[i];  // power of two >= 2*nn
    uint32_t bits = 63 - __clzll((long long)size);
    for (uint64_t j = threadIdx.x; j < size; j += blockDim.x) tab[j] = kInvalidNode;
    __syncthreads();
    bool mydup = false;
    for (uint32_t j = threadIdx.x; j < nn; j += blockDim.x) {
        uint32_t v = walk_node<PAIRS>(p, w, base, j);
        uint64_t h = node_hash(v, bits);
        for (;;) {
            uint32_t old = atomicCAS(&tab[h], kInvalidNode, v);
            if (old == kInvalidNode) break;
            if (old == v) {
                mydup = true;
                break;
            }
            h = (h + 1) & (size - 1);
        }
    }
    if (__syncthreads_or(mydup) && threadIdx.x == 0) {
        if (p.status[w] == 1) atomicAdd(p.long_count + 1, 1u);
        p.status[w] = 0;
    }
}

template <class K>
int persistent_blocks(hsaw_gpu_ctx* ctx, K kernel, uint64_t items) {
    int per_sm = 0;
    HSAW_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
    if (per_sm < 1) per_sm = 1;
    uint64_t want = (items + kThreads - 1) / kThreads;
    uint64_t full = (uint64_t)ctx->sm_count * per_sm;  // one resident wave: 148 x blocks/SM
    return (int)(want < full ? (want ? want : 1) : full);
}

}  // namespace

void validate_cfg(const hsaw_sampler_cfg& cfg) {
    if (cfg.heuristic < 0 || cfg.heuristic > 2) fail(HSAW_EINVAL, "sampler: unknown heuristic");
    if (cfg.batch_size == 0) fail(HSAW_EINVAL, "sampler: batch_size must be positive");
    if (cfg.rng_mode > 1) fail(HSAW_EINVAL, "sampler: unknown rng_mode");
    if (cfg.rng_mode == 1 && (cfg.heuristic != 0 || cfg.window != 2))
        fail(HSAW_EINVAL, "sampler: the Philox per-walk mode is built for Brent + window 2 only");
}

// rec == nullptr: plain encode. Otherwise accepted walks are logged into rec->arena.
void launch_encode(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg& cfg, uint64_t first_worker,
                   uint64_t nbatches, uint64_t* d_seed, uint32_t* d_len, uint32_t* d_count,
                   uint64_t* d_stats, uint64_t* d_cursor, const EncodeRecord* rec,
                   bool with_stats) {
    if (nbatches == 0) return;
    if (nbatches > 0xFFFFFFFFull) fail(HSAW_EINVAL, "encode: more than 2^32 batches per launch");
    // a chunk sampled ahead of its predecessor's post-processing runs on the context's second
    // stream (stream.cu sample_range); everything else on the context stream
    cudaStream_t st = ctx->k1_stream ? ctx->k1_stream : ctx->stream;
    EncodeParams p{ctx->g.nodes, ctx->g.edges, ctx->g.hdr, src_ref(ctx->g), ctx->g.thr,
                   ctx->g.n, cfg.batch_size, cfg.window, first_worker, nbatches, d_seed, d_len, d_count,
                   d_stats, d_cursor, nullptr, 0, nullptr, nullptr, 0, nullptr, 0, nullptr, nullptr};
    if (const char* env = std::getenv("HSAW_LOG_GROW")) p.grow_mode = (uint32_t)std::atoi(env);
    const bool compact = ctx->g.layout == kLayoutCompact;
    if (cfg.rng_mode == 1) {
        // Philox per-walk mode: the caller passes one work item per ATTEMPT (batch_size 1), so a
        // lane that finishes its attempt refills at once; recording as in the default path
        if (ctx->restr.domain) fail(HSAW_EINVAL, "encode: the Philox mode does not combine with a restriction");
        if (cfg.batch_size != 1) fail(HSAW_EINVAL, "encode: Philox launches carry one attempt per item");
        if (rec) {
            if (rec->arena_cap < kLogChunk) fail(HSAW_EINVAL, "encode: record arena too small");
            p.arena = rec->arena;
            p.arena_cap = rec->arena_cap;
            p.arena_cursor = rec->arena_cursor;
            p.out_log = rec->out_log;
            HSAW_CUDA_CHECK(cudaMemsetAsync(rec->arena_cursor, 0, 4, st));
        }
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, st));
        auto go_p = [&](auto kernel) {
            int blocks = persistent_blocks(ctx, kernel, nbatches);
            StageScope timer(ctx, HSAW_STAGE_ENCODE, st);
            kernel<<<blocks, kThreads, 0, st>>>(p);
            check_launch(ctx, "encode_kernel(philox)");
        };
        if (rec)
            compact ? go_p(encode_kernel<0, 2, 4, 2, false, kLayoutCompact, false, PhiloxRng>)
                    : go_p(encode_kernel<0, 2, 4, 2, false, kLayoutFat, false, PhiloxRng>);
        else
            compact ? go_p(encode_kernel<0, 2, 4, 0, true, kLayoutCompact, false, PhiloxRng>)
                    : go_p(encode_kernel<0, 2, 4, 0, true, kLayoutFat, false, PhiloxRng>);
        return;
    }
    if (ctx->restr.domain) {  // partitioned sampling: the restricted instantiations, never recording
        if (rec) fail(HSAW_EINVAL, "encode: restricted sampling does not record");
        if (!ctx->restr.allowed || !ctx->restr.out_cross || ctx->restr.ndomain == 0)
            fail(HSAW_EINVAL, "encode: incomplete restriction");
        p.domain = ctx->restr.domain;
        p.ndomain = ctx->restr.ndomain;
        p.allowed = ctx->restr.allowed;
        p.out_cross = ctx->restr.out_cross;
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, st));
        auto go_r = [&](auto kernel) {
            int blocks = persistent_blocks(ctx, kernel, nbatches);
            StageScope timer(ctx, HSAW_STAGE_ENCODE, st);
            kernel<<<blocks, kThreads, 0, st>>>(p);
            check_launch(ctx, "encode_kernel(restricted)");
        };
#define HSAW_GO_R(H, W)                                                              \
    (compact ? go_r(encode_kernel<H, W, 4, 0, true, kLayoutCompact, true>)           \
             : go_r(encode_kernel<H, W, 4, 0, true, kLayoutFat, true>))
        const bool br = cfg.heuristic == 0;
        if (cfg.heuristic == 1)  // Floyd: one runtime-window instantiation
            HSAW_GO_R(1, -1);
        else if (cfg.window == 2)
            br ? HSAW_GO_R(0, 2) : HSAW_GO_R(2, 2);
        else if (cfg.window == 0)
            br ? HSAW_GO_R(0, 0) : HSAW_GO_R(2, 0);
        else
            br ? HSAW_GO_R(0, -1) : HSAW_GO_R(2, -1);
#undef HSAW_GO_R
        return;
    }
// one instantiation per graph layout
#define HSAW_GO(H, W, B, R, S)                                                   \
    (compact ? go(encode_kernel<H, W, B, R, S, kLayoutCompact>)                  \
             : go(encode_kernel<H, W, B, R, S, kLayoutFat>))
    if (rec) {
        if (rec->arena_cap < kLogChunk) fail(HSAW_EINVAL, "encode: record arena too small");
        p.arena = rec->arena;
        p.arena_cap = rec->arena_cap;
        p.arena_cursor = rec->arena_cursor;
        p.out_log = rec->out_log;
        HSAW_CUDA_CHECK(cudaMemsetAsync(rec->arena_cursor, 0, 4, st));
    }
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, st));
    auto go = [&](auto kernel) {
        int blocks = persistent_blocks(ctx, kernel, nbatches);
        // Resident blocks per SM. Once the edge records outgrow the TLB's reach (8 GB and more:
        // the 36 G gathers/s plateau of tools/tlb_probe.cu) the recording kernel is bound by
        // HBM's random-gather rate, not by lanes in flight: 3 blocks per SM run 1-2.5 % FASTER
        // than the 4 its registers allow (Twitter shape, 47 GB of records, per 2^20 batches:
        // 18.6 / 18.8 ms, 2 blocks: 21.0) and leave a quarter of every SM to whatever runs
        // beside K1 (stream.cu sample_range). Below that (LiveJournal shape, 2.2 GB: 9.76 ms with
        // 3 blocks, 9.66 with 4) every lane still counts.
        // HSAW_K1_GRID_BLOCKS_PER_SM: A/B knob (0 = whatever fits).
        int per_sm = (rec && !compact && (uint64_t)ctx->g.m * sizeof(EdgeRec) > (8ull << 30)) ? 3 : 0;
        if (const char* env = std::getenv("HSAW_K1_GRID_BLOCKS_PER_SM")) per_sm = std::atoi(env);
        if (per_sm > 0) blocks = std::min(blocks, per_sm * ctx->sm_count);
        StageScope timer(ctx, HSAW_STAGE_ENCODE, st);
        kernel<<<blocks, kThreads, 0, st>>>(p);
        check_launch(ctx, "encode_kernel");
    };
    const bool brent = cfg.heuristic == 0;
    static const bool fast_off = [] {  // A/B knob: HSAW_K1_GENERIC=1 keeps the generic kernel
        const char* env = std::getenv("HSAW_K1_GENERIC");
        return env && std::atoi(env) != 0;
    }();
    if (cfg.window == 2 && brent && compact && rec && !with_stats && !fast_off) {
        // Resident blocks per SM are capped explicitly and the shared-memory carve-out is sized
        // for exactly that many blocks: what is left of the 228 KB stays L1, which serves the
        // hub rows (HSAW_K1_FAST_BLOCKS: A/B knob).
        static const int fast_blocks = [] {
            const char* env = std::getenv("HSAW_K1_FAST_BLOCKS");
            int b = env ? std::atoi(env) : kFastBlocksPerSM;
            return b < 1 ? 1 : (b > 8 ? 8 : b);
        }();
        static const int fast_stage = [] {  // A/B knob: pairs staged per thread (8 or 16)
            const char* env = std::getenv("HSAW_K1_FAST_STAGE");
            return env ? std::atoi(env) : 8;
        }();
        auto run = [&](auto kernel) {
            cudaFuncAttributes fa{};
            HSAW_CUDA_CHECK(cudaFuncGetAttributes(&fa, kernel));
            const int smem_kb = (int)((fa.sharedSizeBytes + 1024 + 1023) / 1024) * fast_blocks;
            int carve = (smem_kb * 100 + 227) / 228;
            HSAW_CUDA_CHECK(cudaFuncSetAttribute(
                kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve > 100 ? 100 : carve));
            int blocks = persistent_blocks(ctx, kernel, nbatches);
            blocks = std::min(blocks, fast_blocks * ctx->sm_count);
            StageScope timer(ctx, HSAW_STAGE_ENCODE, st);
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(blocks);
            lc.blockDim = dim3(kThreads);
            lc.stream = st;
            cudaLaunchAttribute attr{};
            if (ctx->k1_window_on) {  // keep the graph's L2 lines through the kernel's log stream
                attr.id = cudaLaunchAttributeAccessPolicyWindow;
                attr.val.accessPolicyWindow = ctx->k1_window;
                lc.attrs = &attr;
                lc.numAttrs = 1;
            }
            HSAW_CUDA_CHECK(cudaLaunchKernelEx(&lc, kernel, p));
            check_launch(ctx, "encode_compact_kernel");
        };
        const uint32_t sb = ctx->g.src_bits;
        if (fast_stage == 16) {
            sb == 21 ? run(encode_compact_kernel<4, 16, 21>)
                     : sb == 32 ? run(encode_compact_kernel<4, 16, 32>)
                                : run(encode_compact_kernel<4, 16, 0>);
        } else if (fast_blocks >= 6 && sb == 21) {
            run(encode_compact_kernel<6, 8, 21>);  // 40 registers (A/B)
        } else {
            sb == 21 ? run(encode_compact_kernel<4, 8, 21>)
                     : sb == 32 ? run(encode_compact_kernel<4, 8, 32>)
                                : run(encode_compact_kernel<4, 8, 0>);
        }
    } else if (cfg.window == 2 && brent) {
        // The default configuration gets the tuned variants: resident blocks per SM (register
        // budget), recording mode and instrumentation are compile-time parameters.
        static const int occ_env = [] {
            const char* env = std::getenv("HSAW_K1_BLOCKS_PER_SM");
            return env ? std::atoi(env) : 0;
        }();
        static const int store_mode = [] {  // 1 default stores, 2 streaming (.cs) stores
            const char* env = std::getenv("HSAW_LOG_STORE");
            return env && std::atoi(env) == 1 ? 1 : 2;
        }();
        const int mode = rec ? store_mode : 0;
        const bool five = (occ_env ? occ_env : (rec ? kDefaultRecordBlocksPerSM
                                                    : kDefaultEncodeBlocksPerSM)) >= 5;
        const int key = mode * 4 + (five ? 2 : 0) + (with_stats ? 1 : 0);
        switch (key) {
            case 0: HSAW_GO(0, 2, 4, 0, false); break;
            case 1: HSAW_GO(0, 2, 4, 0, true); break;
            case 2: HSAW_GO(0, 2, 5, 0, false); break;
            case 3: HSAW_GO(0, 2, 5, 0, true); break;
            case 4: HSAW_GO(0, 2, 4, 1, false); break;
            case 5: HSAW_GO(0, 2, 4, 1, true); break;
            case 6: HSAW_GO(0, 2, 5, 1, false); break;
            case 7: HSAW_GO(0, 2, 5, 1, true); break;
            case 8: HSAW_GO(0, 2, 4, 2, false); break;
            case 9: HSAW_GO(0, 2, 4, 2, true); break;
            case 10: HSAW_GO(0, 2, 5, 2, false); break;
            default: HSAW_GO(0, 2, 5, 2, true); break;
        }
    } else {
        // other SamplerConfig values: correctness paths, instrumented, never recording
        if (rec) fail(HSAW_EINVAL, "encode: recording is only built for the default sampler config");
        if (cfg.heuristic == 1)  // Floyd: one runtime-window instantiation
            HSAW_GO(1, -1, 4, 0, true);
        else if (cfg.window == 2)
            HSAW_GO(2, 2, 4, 0, true);
        else if (cfg.window == 0)
            brent ? HSAW_GO(0, 0, 4, 0, true) : HSAW_GO(2, 0, 4, 0, true);
        else
            brent ? HSAW_GO(0, -1, 4, 0, true) : HSAW_GO(2, -1, 4, 0, true);
    }
#undef HSAW_GO
}

bool record_supported(const hsaw_sampler_cfg& cfg) { return cfg.heuristic == 0 && cfg.window == 2; }

uint32_t record_chunk_pairs() { return kLogChunk; }
uint32_t record_overflow_marker() { return kLogOverflow; }

// Lanes of one resident wave of the default recording kernel (each may hold one open chunk).
uint64_t record_resident_lanes(hsaw_gpu_ctx* ctx) {
    int a = persistent_blocks(ctx, encode_kernel<0, 2, 4, 2, false, kLayoutFat>, ~0ull >> 8);
    int b = 6 * ctx->sm_count;  // upper bound of encode_compact_kernel's resident blocks
    return (uint64_t)std::max(a, b) * kThreads;
}

static void launch_decode_impl(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* d_seed,
                               const uint32_t* d_len, const uint64_t* d_edge_off,
                               uint32_t* d_nodes, uint32_t* d_edges, uint8_t* d_status,
                               uint32_t* d_nnodes, uint64_t* d_stats, uint64_t* d_cursor) {
    if (nwalks == 0) return;
    DecodeParams p{ctx->g.nodes, ctx->g.edges, ctx->g.hdr, src_ref(ctx->g), ctx->g.thr, ctx->g.n,
                   nwalks,       d_seed,       d_len,      d_edge_off, d_nodes,    d_edges,
                   d_status,     d_nnodes,     d_stats,    d_cursor,   nullptr,    nullptr,
                   ctx->restr.domain, ctx->restr.ndomain};
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, ctx->stream));
    auto go = [&](auto kernel) {
        int blocks = persistent_blocks(ctx, kernel, nwalks);
        StageScope timer(ctx, HSAW_STAGE_DECODE);
        kernel<<<blocks, kThreads, 0, ctx->stream>>>(p);
        check_launch(ctx, "decode_kernel");
    };
    if (ctx->rng_mode == 1)
        ctx->g.layout == kLayoutCompact ? go(decode_kernel<false, kLayoutCompact, PhiloxRng>)
                                        : go(decode_kernel<false, kLayoutFat, PhiloxRng>);
    else if (ctx->g.layout == kLayoutCompact)
        go(decode_kernel<false, kLayoutCompact>);
    else
        go(decode_kernel<false, kLayoutFat>);
}

void launch_decode(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* d_seed,
                   const uint32_t* d_len, const uint64_t* d_edge_off, uint32_t* d_nodes,
                   uint32_t* d_edges, uint8_t* d_status, uint64_t* d_stats, uint64_t* d_cursor) {
    launch_decode_impl(ctx, nwalks, d_seed, d_len, d_edge_off, d_nodes, d_edges, d_status,
                       nullptr, d_stats, d_cursor);
}

// Replay of the `nsel` walks listed in d_sel (indices into the encoded arrays) as pair logs.
// walks with more nodes than this are only queued by K2b's main pass (the mid / long passes read
// them): the edge count from which a replay may overlap that pass
uint32_t distinct_check_defers_walks_longer_than() { return kTableSize / 2; }

// Makes the context stream wait for a replay that was launched on the side stream.
void join_side_stream(hsaw_gpu_ctx* ctx) {
    if (!ctx->side_pending) return;
    HSAW_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->side_done, 0));
    ctx->side_pending = false;
}

// on_side: run on the context's side stream, after everything queued on the context stream so
// far; join_side_stream orders the context stream behind it again.
void launch_decode_pairs(hsaw_gpu_ctx* ctx, uint64_t nsel, const uint32_t* d_sel,
                         const uint64_t* d_seed, const uint32_t* d_len, uint2* const* d_pair_dst,
                         uint8_t* d_status, uint64_t* d_stats, uint64_t* d_cursor, bool on_side) {
    if (nsel == 0) return;
    DecodeParams p{ctx->g.nodes, ctx->g.edges, ctx->g.hdr, src_ref(ctx->g), ctx->g.thr, ctx->g.n,
                   nsel,         d_seed,       d_len,      nullptr,    nullptr,    nullptr,
                   d_status,     nullptr,      d_stats,    d_cursor,   d_sel,      d_pair_dst};
    cudaStream_t run = ctx->stream;
    if (on_side) {
        if (!ctx->side) {
            HSAW_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
            HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->side_go, cudaEventDisableTiming));
            HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->side_done, cudaEventDisableTiming));
        }
        HSAW_CUDA_CHECK(cudaEventRecord(ctx->side_go, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamWaitEvent(ctx->side, ctx->side_go, 0));
        run = ctx->side;
    }
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, run));
    auto go = [&](auto kernel) {
        int blocks = persistent_blocks(ctx, kernel, nsel);
        StageScope timer(ctx, HSAW_STAGE_DECODE, run);
        kernel<<<blocks, kThreads, 0, run>>>(p);
        check_launch(ctx, "decode_kernel<pairs>");
    };
    if (ctx->rng_mode == 1)
        ctx->g.layout == kLayoutCompact ? go(decode_kernel<true, kLayoutCompact, PhiloxRng>)
                                        : go(decode_kernel<true, kLayoutFat, PhiloxRng>);
    else if (ctx->g.layout == kLayoutCompact)
        go(decode_kernel<true, kLayoutCompact>);
    else
        go(decode_kernel<true, kLayoutFat>);
    if (on_side) {
        HSAW_CUDA_CHECK(cudaEventRecord(ctx->side_done, ctx->side));
        ctx->side_pending = true;
    }
}

// Exact recheck on either node source. Classic: d_edge_off/d_nodes(/d_nnodes). Pair logs:
// d_pair_src + d_lens.
template <bool PAIRS>
static uint32_t distinct_check_impl(hsaw_gpu_ctx* ctx, uint64_t nwalks,
                                    const uint64_t* d_edge_off, const uint32_t* d_nodes,
                                    const uint32_t* d_nnodes, const uint2* const* d_pair_src,
                                    const uint32_t* d_lens, uint8_t* d_status) {
    if (nwalks == 0) return 0;
    if (nwalks > 0xFFFFFFFFull) fail(HSAW_EINVAL, "distinct check: more than 2^32 walks per call");
    const uint32_t long_cap = 1u << 16;
    const uint32_t mid_cap = (uint32_t)std::min<uint64_t>(nwalks, 1u << 22);
    ctx->chk_list.ensure_scratch(2ull * long_cap);
    ctx->chk_mid.ensure_scratch(mid_cap);
    ctx->chk_counters.ensure_scratch(4);
    uint32_t* counters = ctx->chk_counters.p;
    HSAW_CUDA_CHECK(cudaMemsetAsync(counters, 0, 16, ctx->stream));
    CheckParams p{nwalks,   d_edge_off,      d_nodes,  d_nnodes, d_pair_src,      d_lens,
                  d_status, ctx->chk_list.p, counters, long_cap, ctx->chk_mid.p, mid_cap,
                  nullptr};
    auto mid_kernel = distinct_kernel<PAIRS, kMidTableSize, kMidWarps, 1>;
    const int smem_main = kCheckWarps * kTableSize * 4, smem_mid = kMidWarps * kMidTableSize * 4;
    static bool attr_set = false;
    if (!attr_set) {
        HSAW_CUDA_CHECK(cudaFuncSetAttribute(mid_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem_mid));
        attr_set = true;
    }
    uint32_t* h = reinterpret_cast<uint32_t*>(ctx->h_scalars + 32);
    {
        // Register budget and grid of the main pass (C4, ms per 2^20-batch step; until the end of
        // round 2 it ran with 52 registers = 4 resident blocks and a grid of 7 per SM: 1.88). Six
        // blocks per SM (40 registers, 40 bytes of spills; 6 x 32 KB of tables fill the shared
        // memory) with a grid of eight waves: 1.63. The waves matter as much as the occupancy:
        // walks differ in length by orders of magnitude, a single resident wave with a static
        // stride leaves SMs idle behind the slowest warps (2.53 with 4 blocks, 2.15 with 6),
        // later blocks fill the gaps. HSAW_K2B_MINB (1 / 5 / 6), HSAW_K2B_GRID_PER_SM: A/B knobs.
        static const int minb = [] {
            const char* env = std::getenv("HSAW_K2B_MINB");
            return env ? std::atoi(env) : kCheckMinBlocks;
        }();
        auto go = [&](auto main_kernel) {
            HSAW_CUDA_CHECK(cudaFuncSetAttribute(main_kernel,
                                                 cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 cudaSharedmemCarveoutMaxShared));
            int per_sm = 0;
            HSAW_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, main_kernel, kCheckWarps * 32, smem_main));
            per_sm = std::max(per_sm, 1) * 8;
            if (const char* env = std::getenv("HSAW_K2B_GRID_PER_SM")) per_sm = std::max(1, std::atoi(env));
            uint64_t want = ((nwalks + 31) / 32 + kCheckWarps - 1) / kCheckWarps;  // 32 walks per warp
            uint64_t full = (uint64_t)ctx->sm_count * per_sm;
            int blocks = (int)(want < full ? want : full);
            StageScope timer(ctx, HSAW_STAGE_DISTINCT);
            main_kernel<<<blocks, kCheckWarps * 32, smem_main, ctx->stream>>>(p);
            check_launch(ctx, "distinct_kernel");
        };
        if (minb >= 6)
            go(distinct_kernel<PAIRS, kTableSize, kCheckWarps, 32, 6>);
        else if (minb == 5)
            go(distinct_kernel<PAIRS, kTableSize, kCheckWarps, 32, 5>);
        else
            go(distinct_kernel<PAIRS, kTableSize, kCheckWarps, 32, 1>);
    }
    HSAW_CUDA_CHECK(cudaMemcpyAsync(h, counters, 16, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (h[2] > mid_cap) fail(HSAW_ECUDA, "distinct check: mid-size walk queue overflow");
    join_side_stream(ctx);  // a replay running beside the main pass: its walks are read from here on
    if (h[2]) {  // walks of 513..2048 nodes: second pass with 16 KB tables over the queued ids
        CheckParams q = p;
        q.nwalks = h[2];
        q.sel = ctx->chk_mid.p;
        uint64_t want = ((uint64_t)h[2] + kMidWarps - 1) / kMidWarps;
        uint64_t full = (uint64_t)ctx->sm_count * 3;
        int blocks = (int)(want < full ? want : full);
        {
            StageScope timer(ctx, HSAW_STAGE_DISTINCT);
            mid_kernel<<<blocks, kMidWarps * 32, smem_mid, ctx->stream>>>(q);
            check_launch(ctx, "distinct_kernel<mid>");
        }
        HSAW_CUDA_CHECK(cudaMemcpyAsync(h, counters, 16, cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    uint32_t nlong = h[0];
    if (nlong > long_cap) fail(HSAW_ECUDA, "distinct check: too many long walks in one round");
    if (nlong) {
        // rare path: size one global hash table per long walk, run one block per walk
        std::vector<uint32_t> pairs(2ull * nlong);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(pairs.data(), ctx->chk_list.p, 8ull * nlong,
                                        cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        std::vector<uint64_t> toff(nlong + 1, 0);
        for (uint32_t i = 0; i < nlong; ++i) {
            uint64_t nn = pairs[2 * i + 1];
            uint64_t size = 1;
            while (size < 2 * nn) size <<= 1;
            toff[i + 1] = toff[i] + size;
        }
        DevVec<uint32_t> tables;
        DevVec<uint64_t> d_toff;
        tables.ensure_scratch(toff[nlong]);
        d_toff.ensure_scratch(nlong + 1);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(d_toff.p, toff.data(), 8ull * (nlong + 1),
                                        cudaMemcpyHostToDevice, ctx->stream));
        {
            StageScope timer(ctx, HSAW_STAGE_DISTINCT);
            distinct_long_kernel<PAIRS><<<nlong, 256, 0, ctx->stream>>>(p, nlong, d_toff.p,
                                                                        tables.p);
            check_launch(ctx, "distinct_long_kernel");
        }
        HSAW_CUDA_CHECK(cudaMemcpyAsync(h, counters, 8, cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    return h[1];
}

uint32_t launch_distinct_check(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* d_edge_off,
                               const uint32_t* d_nodes, uint8_t* d_status) {
    return distinct_check_impl<false>(ctx, nwalks, d_edge_off, d_nodes, nullptr, nullptr, nullptr,
                                      d_status);
}

uint32_t launch_distinct_check_pairs(hsaw_gpu_ctx* ctx, uint64_t nwalks,
                                     const uint2* const* d_pair_src, const uint32_t* d_lens,
                                     uint8_t* d_status) {
    return distinct_check_impl<true>(ctx, nwalks, nullptr, nullptr, nullptr, d_pair_src, d_lens,
                                     d_status);
}

}  // namespace hsawgpu

using namespace hsawgpu;

extern "C" {

int hsaw_gpu_encode_batches(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg* cfg,
                            uint64_t first_worker_id, uint64_t nbatches, uint64_t* out_seed,
                            uint32_t* out_len, uint32_t* out_count, uint64_t* stats) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!cfg || !out_seed || !out_len || !out_count) fail(HSAW_EINVAL, "encode: null argument");
        if (!ctx->g.nodes) fail(HSAW_EINVAL, "encode: no graph uploaded");
        validate_cfg(*cfg);
        if (nbatches == 0) return;
        uint64_t slots = nbatches * cfg->batch_size;
        DevVec<uint64_t> d_seed, d_stats;
        DevVec<uint32_t> d_len, d_count;
        d_seed.ensure_scratch(slots);
        d_len.ensure_scratch(slots);
        d_count.ensure_scratch(nbatches);
        d_stats.ensure_scratch(9);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_stats.p, 0, 72, ctx->stream));
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_seed.p, 0, slots * 8, ctx->stream));
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_len.p, 0, slots * 4, ctx->stream));
        launch_encode(ctx, *cfg, first_worker_id, nbatches, d_seed.p, d_len.p, d_count.p,
                      d_stats.p, d_stats.p + 8, nullptr, true);
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(out_seed, d_seed.p, slots * 8, cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(out_len, d_len.p, slots * 4, cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(out_count, d_count.p, nbatches * 4, cudaMemcpyDeviceToHost,
                                        ctx->stream));
        if (stats)
            HSAW_CUDA_CHECK(
                cudaMemcpyAsync(stats, d_stats.p, 64, cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int hsaw_gpu_encode_stats(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg* cfg, uint64_t first_worker_id,
                          uint64_t nbatches, uint64_t* stats) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!cfg || !stats) fail(HSAW_EINVAL, "encode_stats: null argument");
        if (!ctx->g.nodes) fail(HSAW_EINVAL, "encode_stats: no graph uploaded");
        validate_cfg(*cfg);
        for (int i = 0; i < 8; ++i) stats[i] = 0;
        if (nbatches == 0) return;
        const uint64_t kChunk = 1ull << 22;
        DevVec<uint64_t> d_seed, d_stats;
        DevVec<uint32_t> d_len, d_count;
        uint64_t per = std::min(nbatches, kChunk);
        d_seed.ensure_scratch(per * cfg->batch_size);
        d_len.ensure_scratch(per * cfg->batch_size);
        d_count.ensure_scratch(per);
        d_stats.ensure_scratch(9);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_stats.p, 0, 72, ctx->stream));
        for (uint64_t done = 0; done < nbatches; done += per) {
            uint64_t nb = std::min(per, nbatches - done);
            launch_encode(ctx, *cfg, first_worker_id + done, nb, d_seed.p, d_len.p, d_count.p,
                          d_stats.p, d_stats.p + 8, nullptr, true);
        }
        HSAW_CUDA_CHECK(cudaMemcpyAsync(ctx->h_scalars, d_stats.p, 64, cudaMemcpyDeviceToHost,
                                        ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < 8; ++i) stats[i] = ctx->h_scalars[i];
    });
}

int hsaw_gpu_decode_walks(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* seeds,
                          const uint32_t* lens, const uint64_t* edge_off, uint32_t* out_nodes,
                          uint32_t* out_edges, uint8_t* out_status) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->g.nodes) fail(HSAW_EINVAL, "decode: no graph uploaded");
        if (nwalks == 0) return;
        if (!seeds || !lens || !edge_off || !out_nodes || !out_edges || !out_status)
            fail(HSAW_EINVAL, "decode: null argument");
        uint64_t total = 0;
        for (uint64_t w = 0; w < nwalks; ++w) {
            if (edge_off[w] != total) fail(HSAW_EINVAL, "decode: edge_off is not the prefix sum of lens");
            total += lens[w];
        }
        if (edge_off[nwalks] != total) fail(HSAW_EINVAL, "decode: edge_off is not the prefix sum of lens");
        DevVec<uint64_t> d_seed, d_off, d_scal;
        DevVec<uint32_t> d_len, d_nodes, d_edges, d_nn;
        DevVec<uint8_t> d_status;
        d_seed.ensure_scratch(nwalks);
        d_len.ensure_scratch(nwalks);
        d_off.ensure_scratch(nwalks + 1);
        d_nodes.ensure_scratch(total + nwalks);
        d_edges.ensure_scratch(total + 1);
        d_nn.ensure_scratch(nwalks);
        d_status.ensure_scratch(nwalks);
        d_scal.ensure_scratch(9);
        cudaStream_t st = ctx->stream;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(d_seed.p, seeds, nwalks * 8, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(d_len.p, lens, nwalks * 4, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(d_off.p, edge_off, (nwalks + 1) * 8, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_scal.p, 0, 72, st));
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_nodes.p, 0xFF, (total + nwalks) * 4, st));
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_edges.p, 0xFF, (total + 1) * 4, st));
        launch_decode_impl(ctx, nwalks, d_seed.p, d_len.p, d_off.p, d_nodes.p, d_edges.p,
                           d_status.p, d_nn.p, d_scal.p, d_scal.p + 8);
        (void)distinct_check_impl<false>(ctx, nwalks, d_off.p, d_nodes.p, d_nn.p, nullptr, nullptr,
                                         d_status.p);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(out_nodes, d_nodes.p, (total + nwalks) * 4,
                                        cudaMemcpyDeviceToHost, st));
        if (total)
            HSAW_CUDA_CHECK(
                cudaMemcpyAsync(out_edges, d_edges.p, total * 4, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(out_status, d_status.p, nwalks, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
