// Context lifetime and graph upload: the reference's CSR arrays are copied to the device once and
// re-laid out by two kernels into the node/edge records the walk kernels read.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "hostcheck.h"
#include "walk.cuh"

using namespace hsawgpu;

namespace {

// ceil(c * 2^53) as an exact integer, saturated to 2^53 (any threshold >= 2^53 never excludes a
// 53-bit draw). c * 2^53 is exact (power-of-two scaling); the conversion rounds toward +inf.
__device__ __forceinline__ uint64_t ge_threshold(double c) {
    if (!(c > 0.0)) return 0;  // also NaN
    if (c >= 1.0) return 1ull << 53;
    return __double2ull_ru(c * 0x1.0p53);
}

// floor(p * 2^53) + 1 for suspects (r <= p  <=>  k < floor(p*2^53)+1), 0 for non-suspects
// (is_suspect is p > 0, proj/include/hsaw/graph.hpp:91).
__device__ __forceinline__ uint64_t accept_threshold(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return (1ull << 53) + 1;
    return __double2ull_rd(p * 0x1.0p53) + 1;
}

__global__ void build_node_records(uint32_t n, const uint64_t* __restrict__ off,
                                   const double* __restrict__ cum, const double* __restrict__ p_of,
                                   NodeRec* __restrict__ out) {
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint64_t lo = off[v], hi = off[v + 1];
    NodeRec r;
    r.lo = (uint32_t)lo;
    r.deg = (uint32_t)(hi - lo);
    r.tot_thr = 0;
    r.scale = 0;
    if (hi > lo) {
        double total = cum[hi - 1];
        r.tot_thr = ge_threshold(total);
        double sc = total > 0.0 ? (double)r.deg / total * 2147483648.0 : 0.0;
        r.scale = sc >= 1.8e19 ? ~0ull : (uint64_t)(sc + 0.5);
    }
    r.acc_thr = accept_threshold(p_of[v]);
    out[v] = r;
}

__global__ void update_accept_thresholds(uint32_t n, const double* __restrict__ p_of,
                                         NodeRec* __restrict__ out) {
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    out[v].acc_thr = accept_threshold(p_of[v]);
}

// Row header of node u as the edge records carry it: simple iff the total-weight threshold is
// within 2^32 draw units of 2^53 (always the case for 1/d rows) or the row is empty. Read from
// u's node record (built first): ONE 32-byte gather per edge. The first version went back to the
// CSR (offset pair -> last cumulative weight of the row, plus p_of): three dependent DRAM lines
// per edge, 76 ms for the 1.47 G edges of the Twitter shape.
__device__ __forceinline__ void source_header(const NodeRec* __restrict__ nodes, uint32_t u,
                                              EdgeRec& r) {
    const NodeRec s = load_node(nodes, u);
    r.src_lo = s.lo;
    r.src_deg = s.deg;
    r.src_deficit = 0;
    r.flags = s.acc_thr != 0 ? kEdgeSuspect : 0u;  // acc_thr != 0 <=> p_of[u] > 0
    if (s.deg == 0) {
        r.flags |= kEdgeSimple;
    } else {
        uint64_t deficit = (1ull << 53) - s.tot_thr;  // tot_thr = ge_threshold(cum[hi - 1]) <= 2^53
        if (deficit <= 0xFFFFFFFFull) {
            r.src_deficit = (uint32_t)deficit;
            r.flags |= kEdgeSimple;
        }
    }
}

// Edge records of the slots first, first + stride, ... of row v.
__device__ __forceinline__ void edge_row_slice(uint32_t v, uint32_t n, uint64_t lo, uint64_t hi,
                                               uint32_t first, uint32_t stride,
                                               const uint64_t* __restrict__ off,
                                               const uint32_t* __restrict__ src,
                                               const double* __restrict__ cum,
                                               const NodeRec* __restrict__ nodes,
                                               EdgeRec* __restrict__ out,
                                               uint32_t* __restrict__ bad_row) {
    for (uint64_t e = lo + first; e < hi; e += stride) {
        double c = cum[e];
        EdgeRec r;
        r.thr = ge_threshold(c);
        r.src = src[e];
        uint64_t prev = 0;
        if (e > lo) {
            double cp = cum[e - 1];
            prev = ge_threshold(cp);
            if (!(c >= cp)) atomicMin(bad_row, v);  // decreasing or NaN cumulative weights
        }
        uint64_t ph = prev >> 21;
        r.prev_hi = ph > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)ph;
        if (r.src >= n) {
            atomicMin(bad_row + 1, v);  // source id out of range
            r.src_lo = r.src_deg = r.src_deficit = r.flags = 0;
        } else {
            source_header(nodes, r.src, r);
        }
        out[e] = r;
    }
}

// One warp per row, lanes stride the row's slots; rows longer than 2048 slots are queued for
// build_edge_records_big (one block per row) so that hub rows are not a single warp's tail.
__global__ void build_edge_records(uint32_t n, const uint64_t* __restrict__ off,
                                   const uint32_t* __restrict__ src, const double* __restrict__ cum,
                                   const NodeRec* __restrict__ nodes, EdgeRec* __restrict__ out,
                                   uint32_t* __restrict__ bad_row, uint32_t* __restrict__ big_rows,
                                   uint32_t* __restrict__ big_count, uint32_t big_cap) {
    uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < n; v += nwarps) {
        uint64_t lo = off[v], hi = off[v + 1];
        if (hi - lo > 2048) {
            uint32_t at = 0;
            if (lane == 0) at = atomicAdd(big_count, 1u);
            at = __shfl_sync(kFullMask, at, 0);
            if (at < big_cap) {
                if (lane == 0) big_rows[at] = v;
                continue;
            }
        }
        edge_row_slice(v, n, lo, hi, lane, 32, off, src, cum, nodes, out, bad_row);
    }
}

__global__ void __launch_bounds__(256) build_edge_records_big(
    uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ src,
    const double* __restrict__ cum, const NodeRec* __restrict__ nodes, EdgeRec* __restrict__ out,
    uint32_t* __restrict__ bad_row, const uint32_t* __restrict__ big_rows,
    const uint32_t* __restrict__ big_count, uint32_t big_cap) {
    const uint32_t count = min(*big_count, big_cap);
    for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
        const uint32_t v = big_rows[i];
        edge_row_slice(v, n, off[v], off[v + 1], threadIdx.x, blockDim.x, off, src, cum, nodes, out,
                       bad_row);
    }
}


// Compact layout: thresholds (exact path only), validation, and per row the margin inside which the
// arithmetic pick (k * deg) >> 53 may disagree with the thresholds. With err_i the distance of
// threshold i from the ideal grid in units of 1/deg, err_i = |thr[i] * deg - (i+1) * 2^53|, every
// draw whose guess differs from the threshold-defined slot has frac(k * deg / 2^53) < max err or
// > 2^53 - max err (walk.cuh, pick_arith). The last threshold is the total-weight one, so "no live
// edge" draws (k >= thr[deg-1]) fall inside the margin as well. One warp per row.
// Top 32 bits of the acceptance threshold, biased by one so that 0 means "not a suspect": with
// A = acc32 - 1 and h = k >> 21, h < A accepts and h > A rejects; h == A (2^-32 of the draws) and
// the saturated code 0xFFFFFFFF are settled against the exact threshold in the node record.
__device__ __forceinline__ uint32_t accept_code(double p) {
    uint64_t t = accept_threshold(p);
    if (t == 0) return 0;
    uint64_t a = (t >> 21) + 1;
    return a >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)a;
}

// Row slice [first, first + stride, ...) of row v: thresholds, validation, largest grid error.
__device__ __forceinline__ uint64_t compact_row_slice(uint32_t v, uint32_t n, uint64_t lo,
                                                      uint64_t hi, uint32_t first, uint32_t stride,
                                                      const uint32_t* __restrict__ src,
                                                      const double* __restrict__ cum,
                                                      uint64_t* __restrict__ thr,
                                                      uint32_t* __restrict__ bad_row) {
    const uint64_t kSat = 1ull << 62;
    const uint64_t d = hi - lo;
    uint64_t maxerr = 0;
    for (uint64_t e = lo + first; e < hi; e += stride) {
        double c = cum[e];
        uint64_t t = ge_threshold(c);
        thr[e] = t;
        if (e > lo && !(c >= cum[e - 1])) atomicMin(bad_row, v);  // decreasing or NaN
        if (src[e] >= n) atomicMin(bad_row + 1, v);               // source id out of range
        unsigned __int128 a = (unsigned __int128)t * d;
        unsigned __int128 b = (unsigned __int128)(e - lo + 1) << 53;
        unsigned __int128 diff = a > b ? a - b : b - a;
        uint64_t err = diff >= kSat ? kSat : (uint64_t)diff;
        maxerr = err > maxerr ? err : maxerr;
    }
    return maxerr;
}

__device__ __forceinline__ void write_header(uint32_t v, uint64_t lo, uint64_t d, uint64_t maxerr,
                                             const double* __restrict__ p_of,
                                             uint4* __restrict__ hdr, int force_exact) {
    uint64_t need = maxerr + d + 1;               // margin in units of 1/deg, with slack
    uint32_t mb = 64 - __clzll((long long)need);  // 2^mb > need
    if (mb > 52 || d > kHdrDegMask || force_exact) mb = kHdrSlow;
    uint32_t w = (uint32_t)(d > kHdrDegMask ? kHdrDegMask : d) | (mb << kHdrDegBits) |
                 (p_of[v] > 0.0 ? 0x80000000u : 0u);
    hdr[v] = make_uint4((uint32_t)lo, w, accept_code(p_of[v]), 0u);
}

// One warp per row; rows longer than kBigRow are queued for build_compact_big (a single warp
// walking a 38 k-edge hub row was the whole kernel's tail: 1.5 ms for 16 M edges).
constexpr uint64_t kBigRow = 2048;

__global__ void build_compact(uint32_t n, const uint64_t* __restrict__ off,
                              const uint32_t* __restrict__ src, const double* __restrict__ cum,
                              const double* __restrict__ p_of, uint64_t* __restrict__ thr,
                              uint4* __restrict__ hdr, uint32_t* __restrict__ bad_row,
                              int force_exact, uint32_t* __restrict__ big_rows,
                              uint32_t* __restrict__ big_count, uint32_t big_cap) {
    uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < n; v += nwarps) {
        uint64_t lo = off[v], hi = off[v + 1];
        if (hi - lo > kBigRow) {
            uint32_t at = 0;
            if (lane == 0) at = atomicAdd(big_count, 1u);
            at = __shfl_sync(kFullMask, at, 0);
            if (at < big_cap) {
                if (lane == 0) big_rows[at] = v;
                continue;
            }  // queue full: fall through and do it here
        }
        uint64_t maxerr = compact_row_slice(v, n, lo, hi, lane, 32, src, cum, thr, bad_row);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t other = __shfl_xor_sync(kFullMask, maxerr, o);
            maxerr = other > maxerr ? other : maxerr;
        }
        if (lane == 0) write_header(v, lo, hi - lo, maxerr, p_of, hdr, force_exact);
    }
}

// One block per queued row.
__global__ void __launch_bounds__(256) build_compact_big(
    uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ src,
    const double* __restrict__ cum, const double* __restrict__ p_of, uint64_t* __restrict__ thr,
    uint4* __restrict__ hdr, uint32_t* __restrict__ bad_row, int force_exact,
    const uint32_t* __restrict__ big_rows, const uint32_t* __restrict__ big_count,
    uint32_t big_cap) {
    __shared__ uint64_t smax[8];
    const uint32_t count = min(*big_count, big_cap);
    for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
        const uint32_t v = big_rows[i];
        const uint64_t lo = off[v], hi = off[v + 1];
        uint64_t maxerr =
            compact_row_slice(v, n, lo, hi, threadIdx.x, blockDim.x, src, cum, thr, bad_row);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t other = __shfl_xor_sync(kFullMask, maxerr, o);
            maxerr = other > maxerr ? other : maxerr;
        }
        if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = maxerr;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) maxerr = smax[w] > maxerr ? smax[w] : maxerr;
            write_header(v, lo, hi - lo, maxerr, p_of, hdr, force_exact);
        }
        __syncthreads();
    }
}

// Sources of the compact layout with their dead-end flags (DeviceGraph::src_bits): one thread per
// 64-bit word of three 21-bit entries, or per 32-bit entry.
__device__ __forceinline__ bool dead_end(uint32_t u, uint32_t n, const uint64_t* __restrict__ off,
                                         const double* __restrict__ p_of) {
    return u < n && off[u + 1] == off[u] && !(p_of[u] > 0.0);
}

__global__ void pack_sources21(uint64_t m, uint32_t n, const uint32_t* __restrict__ src,
                               const uint64_t* __restrict__ off, const double* __restrict__ p_of,
                               uint64_t* __restrict__ out) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (3 * q >= m) return;
    uint64_t w = 0;
    for (uint32_t r = 0; r < 3; ++r) {
        const uint64_t e = 3 * q + r;
        if (e >= m) break;
        const uint32_t u = src[e];
        uint64_t v = u & 0xFFFFFu;
        if (dead_end(u, n, off, p_of)) v |= 1u << 20;
        w |= v << (21 * r);
    }
    out[q] = w;
}

__global__ void flag_sources32(uint64_t m, uint32_t n, const uint32_t* __restrict__ src,
                               const uint64_t* __restrict__ off, const double* __restrict__ p_of,
                               uint32_t* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const uint32_t u = src[e];
    out[e] = dead_end(u, n, off, p_of) ? (u | 0x80000000u) : u;
}

// New suspect set on the same graph: recompute the dead-end flags in place (the in-degree comes
// from the row headers).
__global__ void reflag_sources(uint64_t m, const uint4* __restrict__ hdr,
                               const double* __restrict__ p_of, uint32_t bits,
                               uint32_t* __restrict__ src) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto dead = [&](uint32_t u) { return (hdr[u].y & kHdrDegMask) == 0 && !(p_of[u] > 0.0); };
    if (bits == 21) {
        if (3 * q >= m) return;
        uint64_t* words = reinterpret_cast<uint64_t*>(src);
        const uint64_t in = words[q];
        uint64_t w = 0;
        for (uint32_t r = 0; r < 3 && 3 * q + r < m; ++r) {
            const uint32_t u = (uint32_t)(in >> (21 * r)) & 0xFFFFFu;
            w |= ((uint64_t)u | (dead(u) ? 1u << 20 : 0u)) << (21 * r);
        }
        words[q] = w;
    } else {
        if (q >= m) return;
        const uint32_t u = src[q] & 0x7FFFFFFFu;
        src[q] = dead(u) ? (u | 0x80000000u) : u;
    }
}

__global__ void update_hdr_suspect_flags(uint32_t n, const double* __restrict__ p_of,
                                         uint4* __restrict__ hdr) {
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint32_t w = hdr[v].y & 0x7FFFFFFFu;
    if (p_of[v] > 0.0) w |= 0x80000000u;
    hdr[v].y = w;
    hdr[v].z = accept_code(p_of[v]);
}

// New suspect set on the same graph: refresh the suspect bit the edge records carry.
__global__ void update_edge_suspect_flags(uint32_t m, const double* __restrict__ p_of,
                                          EdgeRec* __restrict__ edges) {
    uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    uint32_t f = edges[e].flags & ~kEdgeSuspect;
    if (p_of[edges[e].src] > 0.0) f |= kEdgeSuspect;
    edges[e].flags = f;
}

// ---- per-device facts, queried once (cudaGetDeviceProperties costs milliseconds) -----------------
struct DeviceInfo {
    int sm_count = 0, l2_bytes = 0;
    size_t max_persist = 0, max_window = 0;
};
const DeviceInfo& device_info(int device) {
    static std::mutex mu;
    static std::map<int, DeviceInfo> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    DeviceInfo d;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess) d.sm_count = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device) == cudaSuccess) d.l2_bytes = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess)
        d.max_persist = (size_t)v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, device) == cudaSuccess)
        d.max_window = (size_t)v;
    cudaGetLastError();
    // keep freed pool memory cached instead of returning it to the driver at every sync
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t never = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &never);
    }
    cudaGetLastError();
    return cache.emplace(device, d).first->second;
}

// ---- host -> device copies of pageable arrays ---------------------------------------------------
// The reference hands over plain std::vector storage. A single cudaMemcpy from pageable memory
// runs at ~10 GB/s (one driver thread staging through pinned buffers); here a few host threads
// stage 4 MB chunks into a process-wide ring of pinned buffers and issue the DMA themselves, so
// the copy runs at host-memory speed. The consumer stream waits on the copiers' last events.
class StagedCopier {
public:
    using Job = hsawgpu::CopyJob;
    static constexpr int kMaxThreads = 16, kMaxSlots = 4;
    static size_t chunk_bytes() {  // HSAW_UPLOAD_CHUNK_MB: A/B knob
        static const size_t v = [] {
            const char* env = std::getenv("HSAW_UPLOAD_CHUNK_MB");
            int mb = env ? std::atoi(env) : 4;
            return (size_t)std::max(1, std::min(mb, 64)) << 20;
        }();
        return v;
    }
    static int slots_per_thread() {  // HSAW_UPLOAD_SLOTS: A/B knob
        static const int v = [] {
            const char* env = std::getenv("HSAW_UPLOAD_SLOTS");
            int k = env ? std::atoi(env) : 2;
            return std::max(2, std::min(k, kMaxSlots));
        }();
        return v;
    }

    // Copies all jobs; returns false (nothing copied) when the ring cannot be set up.
    // to_device: pageable host -> device; otherwise device -> pageable host (the call returns
    // once the host arrays are complete).
    // piece_bytes (0 = a whole ring slot): smaller pieces keep the part of the ring in use inside
    // the last-level cache, which pays when other host threads stream through memory at the same
    // time (the in_cum check of graph_upload: 2 MB pieces 250 ms per call, 4 MB 295 ms; alone,
    // 4 MB pieces copy faster: 51 vs 43 GB/s)
    static bool run(int device, cudaStream_t consumer, const std::vector<Job>& jobs,
                    bool to_device = true, size_t piece_bytes = 0) {
        static std::mutex mu;  // one staged copy at a time per process
        std::lock_guard<std::mutex> lock(mu);
        State& st = state(device);
        if (!st.ok) return false;
        struct Piece {
            char* dst;
            const char* src;
            size_t bytes;
        };
        const size_t kChunk = piece_bytes && piece_bytes < chunk_bytes() ? piece_bytes : chunk_bytes();
        const int kSlotsPerThread = slots_per_thread();
        std::vector<Piece> pieces;
        for (const Job& j : jobs)
            for (size_t o = 0; o < j.bytes; o += kChunk)
                pieces.push_back({(char*)j.dst + o, (const char*)j.src + o,
                                  std::min(kChunk, j.bytes - o)});
        if (pieces.empty()) return true;
        const int nthreads = (int)std::min<size_t>(st.nthreads, pieces.size());
        // the copies must not overtake earlier work on the consumer stream that uses the targets
        cudaEventRecord(st.gate, consumer);
        std::vector<cudaError_t> errs(nthreads, cudaSuccess);
        auto work = [&](int t) {
            cudaSetDevice(device);
            cudaStream_t s = st.streams[t];
            cudaStreamWaitEvent(s, st.gate, 0);
            int turn = 0;
            if (to_device) {
                for (size_t i = t; i < pieces.size(); i += nthreads, ++turn) {
                    const int slot = t * kSlotsPerThread + (turn % kSlotsPerThread);
                    if (turn >= kSlotsPerThread) cudaEventSynchronize(st.slot_done[slot]);
                    staging_copy(st.pinned[slot], pieces[i].src, pieces[i].bytes);  // hostcheck.cpp
                    cudaError_t e = cudaMemcpyAsync(pieces[i].dst, st.pinned[slot],
                                                    pieces[i].bytes, cudaMemcpyHostToDevice, s);
                    if (e != cudaSuccess) errs[t] = e;
                    cudaEventRecord(st.slot_done[slot], s);
                }
            } else {
                // device -> pinned slot (DMA), then pinned -> pageable by this thread, one chunk
                // behind so the DMA of chunk i+1 overlaps the host copy of chunk i
                size_t prev = pieces.size();
                int prev_slot = 0;
                for (size_t i = t; i < pieces.size(); i += nthreads, ++turn) {
                    const int slot = t * kSlotsPerThread + (turn % kSlotsPerThread);
                    cudaError_t e = cudaMemcpyAsync(st.pinned[slot], pieces[i].src, pieces[i].bytes,
                                                    cudaMemcpyDeviceToHost, s);
                    if (e != cudaSuccess) errs[t] = e;
                    cudaEventRecord(st.slot_done[slot], s);
                    if (prev != pieces.size()) {
                        cudaEventSynchronize(st.slot_done[prev_slot]);
                        std::memcpy(pieces[prev].dst, st.pinned[prev_slot], pieces[prev].bytes);
                    }
                    prev = i;
                    prev_slot = slot;
                }
                if (prev != pieces.size()) {
                    cudaEventSynchronize(st.slot_done[prev_slot]);
                    std::memcpy(pieces[prev].dst, st.pinned[prev_slot], pieces[prev].bytes);
                }
            }
            cudaEventRecord(st.thread_done[t], s);
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        for (int t = 0; t < nthreads; ++t) {
            cudaStreamWaitEvent(consumer, st.thread_done[t], 0);
            if (errs[t] != cudaSuccess) HSAW_CUDA_CHECK(errs[t]);
        }
        // the pinned ring is reused by the next call: its DMA reads must have finished by then
        for (int t = 0; t < nthreads; ++t) cudaEventSynchronize(st.thread_done[t]);
        return true;
    }

private:
    struct State {
        bool ok = false;
        int nthreads = 0;
        void* pinned[kMaxThreads * kMaxSlots] = {};
        cudaEvent_t slot_done[kMaxThreads * kMaxSlots] = {};
        cudaEvent_t thread_done[kMaxThreads] = {};
        cudaStream_t streams[kMaxThreads] = {};
        cudaEvent_t gate = nullptr;
    };
    static State& state(int device) {
        static std::map<int, State> per_device;
        State& st = per_device[device];
        if (st.nthreads) return st;
        // 8 copier threads reach the pinned-DMA rate of a Gen5 x16 link from pageable memory
        // (tools/upload_probe.cu on the B200 box: 4 threads 47 GB/s, 8 threads 51, pinned 55.6)
        int want = 8;
        if (const char* env = std::getenv("HSAW_UPLOAD_THREADS")) want = std::atoi(env);
        unsigned hw = std::thread::hardware_concurrency();
        if (hw && (unsigned)want > hw) want = (int)hw;
        st.nthreads = std::max(1, std::min(want, kMaxThreads));
        bool ok = want > 0;
        for (int i = 0; ok && i < st.nthreads * slots_per_thread(); ++i) {
            ok = cudaHostAlloc(&st.pinned[i], chunk_bytes(), cudaHostAllocDefault) == cudaSuccess &&
                 cudaEventCreateWithFlags(&st.slot_done[i], cudaEventDisableTiming) == cudaSuccess;
        }
        for (int t = 0; ok && t < st.nthreads; ++t) {
            ok = cudaStreamCreateWithFlags(&st.streams[t], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&st.thread_done[t], cudaEventDisableTiming) == cudaSuccess;
        }
        if (ok) ok = cudaEventCreateWithFlags(&st.gate, cudaEventDisableTiming) == cudaSuccess;
        if (!ok) cudaGetLastError();
        st.ok = ok;
        return st;
    }
};

// Every walk step reads one node record and one edge record. The node records are the smaller,
// reused half (32 n bytes: 32 MB at 1 M nodes, hubs are hot at any size), so they get the
// persisting share of the 126 MB L2 through an access-policy window on the context stream, while
// everything else (edge records, walk logs) streams through the rest. HSAW_L2_PERSIST=0 disables.
void pin_in_l2(hsaw_gpu_ctx* ctx, const void* base, size_t bytes);

void pin_node_records_in_l2(hsaw_gpu_ctx* ctx) {
    pin_in_l2(ctx, ctx->g.nodes, (size_t)ctx->g.n * sizeof(NodeRec));
}

// Compact layout: the headers and sources (one allocation) are the hot, reused data; the walk
// logs, slot arrays and pool writes stream through. While they fit the persisting share of L2
// (B200: 79 MB) a window over them is attached to the K1 launches (sampler.cu), marking these
// lines persisting so that K1's own 3 GB log stream cannot evict them: K1 5.51 -> 5.15 ms on C2.
// The compaction kernels that follow lose a little (0.60 -> 0.71 ms: 60 MB of the cache stay
// persisting; resetting them after K1 with cudaCtxResetPersistingL2Cache costs more than it
// returns), the step gains 3 %. HSAW_L2_PERSIST=0 disables.
void pin_compact_graph_in_l2(hsaw_gpu_ctx* ctx) {
    ctx->k1_window_on = false;
    if (const char* env = std::getenv("HSAW_L2_PERSIST"))
        if (std::atoi(env) == 0) return;
    const DeviceInfo& di = device_info(ctx->device);
    const size_t src_bytes = ctx->g.src_bits == 21 ? 8 * (((size_t)ctx->g.m + 2) / 3)
                                                   : (size_t)ctx->g.m * 4;
    const size_t bytes = (size_t)ctx->g.n * 16 + src_bytes;
    if (bytes == 0 || bytes > di.max_persist || bytes > di.max_window) return;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    ctx->k1_window.base_ptr = ctx->g.hdr;
    ctx->k1_window.num_bytes = bytes;
    ctx->k1_window.hitRatio = 1.0f;
    ctx->k1_window.hitProp = cudaAccessPropertyPersisting;
    ctx->k1_window.missProp = cudaAccessPropertyNormal;
    ctx->k1_window_on = true;
}

void pin_in_l2(hsaw_gpu_ctx* ctx, const void* base, size_t bytes) {
    if (const char* env = std::getenv("HSAW_L2_PERSIST"))
        if (std::atoi(env) == 0) return;
    const DeviceInfo& di = device_info(ctx->device);
    size_t max_persist = di.max_persist;
    size_t max_window = di.max_window;
    if (max_persist == 0 || max_window == 0) return;
    size_t carve = std::min(bytes, max_persist);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = std::min(bytes, max_window);
    attr.accessPolicyWindow.hitRatio =
        (float)std::min(1.0, (double)carve / (double)attr.accessPolicyWindow.num_bytes);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &attr) !=
        cudaSuccess)
        cudaGetLastError();
}

// Layout choice: the compact arrays while the 16-byte row headers fit well inside L2
// (the header gather then stays an L2 hit even when the sources spill to HBM), else fat edge
// records (one HBM line per step) while they fit the TLB's reach, else compact again. HSAW_LAYOUT=compact|fat
// overrides.
int choose_layout(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m) {
    if (const char* env = std::getenv("HSAW_LAYOUT")) {
        if (env[0] == 'c') return kLayoutCompact;
        if (env[0] == 'f') return kLayoutFat;
    }
    const uint64_t l2 = (uint64_t)device_info(ctx->device).l2_bytes;
    // (crossover measured at ~3 M nodes once the fat layout lost its stream-wide L2 window: R-MAT
    // scale 21 compact 177 vs fat 159 M HSAW/s, 3 M nodes 137 vs 137, LiveJournal shape 4.85 M
    // nodes 138 vs 148, scale 23 134 vs 159 - the headers must fit the share of L2 that one
    // partition keeps, not all of it)
    if (16ull * n <= l2 * 3 / 8) return kLayoutCompact;
    // One gather per step beats two only while the edge records stay inside the TLB's reach:
    // dependent random 32-byte gathers run at 36 G/s from tables of up to 64 GB and at 14 / 10 / 9
    // G/s from 96 / 120 / 150 GB, whatever the allocation API (tools/tlb_probe.cu,
    // profiles/r02e_tlb_probe.txt: 2 MB pages everywhere). The Friendster shape (3.78 G edges,
    // 121 GB of records) samples 1.6x faster from 15 GB of sources + 1 GB of headers.
    return 32ull * m <= (64ull << 30) ? kLayoutFat : kLayoutCompact;
}

void free_graph(hsaw_gpu_ctx* ctx) {  // the backing stores keep their capacity for the next upload
    ctx->k1_window_on = false;
    ctx->g = DeviceGraph{};
    ctx->graph_bytes = 0;
}

// Per-device parking lot for the device buffers of destroyed contexts (see swap_buffers).
struct Parked {
    std::mutex mu;
    std::map<int, hsaw_gpu_ctx*> by_device;
    ~Parked() {
        // process teardown: the CUDA context may already be gone, so the buffers are abandoned
        for (auto& kv : by_device) {
            kv.second->for_each_buffer([](auto& v) {
                v.p = nullptr;
                v.cap = v.size = 0;
            });
            kv.second->pool_cache.nodes.abandon();
            kv.second->pool_cache.edges.abandon();
        }
    }
};
Parked& parked() {
    static Parked p;
    return p;
}

// Allocation failure (common.cuh, run_oom_hook): the walk-pool buffers of finished streams are idle
// by construction (a live stream owns its arrays; they come back here when it is destroyed).
void release_idle_caches(hsaw_gpu_ctx* ctx) { ctx->pool_cache.release(); }
const bool oom_hook_registered = [] {
    oom_hook() = &release_idle_caches;
    return true;
}();

void adopt_parked_buffers(hsaw_gpu_ctx* ctx) {
    Parked& pk = parked();
    std::lock_guard<std::mutex> lock(pk.mu);
    auto it = pk.by_device.find(ctx->device);
    if (it == pk.by_device.end()) return;
    ctx->swap_buffers(*it->second);
    ctx->for_each_buffer([&](auto& v) { v.owner = ctx->stream; });
    ctx->pool_cache.nodes.rebind(ctx->stream);
    ctx->pool_cache.edges.rebind(ctx->stream);
    std::swap(ctx->d_scalars, it->second->d_scalars);  // scalar scratch (device + pinned mirror)
    std::swap(ctx->h_scalars, it->second->h_scalars);
}

void park_buffers(hsaw_gpu_ctx* ctx) {
    Parked& pk = parked();
    std::lock_guard<std::mutex> lock(pk.mu);
    hsaw_gpu_ctx*& slot = pk.by_device[ctx->device];
    if (!slot) slot = new hsaw_gpu_ctx;  // holder object: only its buffers are used
    slot->for_each_buffer([](auto& v) {   // drop whatever an earlier context left (no stream: sync free)
        if (v.p) cudaFree(v.p);
        v.p = nullptr;
        v.cap = v.size = 0;
    });
    slot->pool_cache.nodes.release();
    slot->pool_cache.edges.release();
    slot->swap_buffers(*ctx);
    slot->for_each_buffer([](auto& v) { v.owner = nullptr; });
    slot->pool_cache.nodes.rebind(nullptr);
    slot->pool_cache.edges.rebind(nullptr);
    if (!slot->d_scalars) std::swap(slot->d_scalars, ctx->d_scalars);
    if (!slot->h_scalars) std::swap(slot->h_scalars, ctx->h_scalars);
}

}  // namespace

namespace hsawgpu {

template <class InIt, class OutT>
static void exclusive_sum_impl(hsaw_gpu_ctx* ctx, InIt in, OutT* out, uint64_t count) {
    if (count == 0) return;
    size_t bytes = 0;
    HSAW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, ctx->stream));
    ctx->cub_tmp.ensure_scratch(bytes ? bytes : 1);
    HSAW_CUDA_CHECK(
        cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, bytes, in, out, count, ctx->stream));
    ++ctx->launches;
}

struct WidenU32 {
    const uint32_t* p;
    using value_type = uint64_t;
    using difference_type = int64_t;
    using pointer = const uint64_t*;
    using reference = uint64_t;
    using iterator_category = std::random_access_iterator_tag;
    __host__ __device__ uint64_t operator[](int64_t i) const { return p[i]; }
    __host__ __device__ uint64_t operator*() const { return *p; }
    __host__ __device__ WidenU32 operator+(int64_t i) const { return WidenU32{p + i}; }
};
struct WidenU8 {
    const uint8_t* p;
    using value_type = uint32_t;
    using difference_type = int64_t;
    using pointer = const uint32_t*;
    using reference = uint32_t;
    using iterator_category = std::random_access_iterator_tag;
    __host__ __device__ uint32_t operator[](int64_t i) const { return p[i]; }
    __host__ __device__ uint32_t operator*() const { return *p; }
    __host__ __device__ WidenU8 operator+(int64_t i) const { return WidenU8{p + i}; }
};

void exclusive_sum_u32_to_u64(hsaw_gpu_ctx* ctx, const uint32_t* in, uint64_t* out,
                              uint64_t count) {
    exclusive_sum_impl(ctx, WidenU32{in}, out, count);
}
void exclusive_sum_u32(hsaw_gpu_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t count) {
    exclusive_sum_impl(ctx, in, out, count);
}
void exclusive_sum_u8_to_u32(hsaw_gpu_ctx* ctx, const uint8_t* in, uint32_t* out, uint64_t count) {
    exclusive_sum_impl(ctx, WidenU8{in}, out, count);
}

}  // namespace hsawgpu

namespace hsawgpu {

// Large transfers: multi-threaded staging through pinned memory; small ones (and the fallback when
// the ring cannot be set up) go through plain pageable copies on the context stream.
void copy_to_device(hsaw_gpu_ctx* ctx, const std::vector<CopyJob>& jobs, size_t piece_bytes) {
    uint64_t total = 0;
    for (const auto& j : jobs) total += j.bytes;
    if (total >= (16u << 20) && StagedCopier::run(ctx->device, ctx->stream, jobs, true, piece_bytes))
        return;
    for (const auto& j : jobs)
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(j.dst, j.src, j.bytes, cudaMemcpyHostToDevice, ctx->stream));
}

// Device -> host; returns with the host arrays complete.
void copy_to_host(hsaw_gpu_ctx* ctx, const std::vector<CopyJob>& jobs) {
    uint64_t total = 0;
    for (const auto& j : jobs) total += j.bytes;
    if (total >= (16u << 20) && StagedCopier::run(ctx->device, ctx->stream, jobs, false)) return;
    for (const auto& j : jobs)
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(j.dst, j.src, j.bytes, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

// Chooses the layout for an (n, m) graph and points ctx->g at (re)allocated stores. Returns true
// for the compact layout.
bool prepare_layout(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m) {
    // what an earlier solve left behind (adopted from a parked context, or this context's own) is
    // sized for another graph: it goes back to the pool before the new stores are allocated
    ctx->release_solve_scratch();
    const int layout = choose_layout(ctx, n, m);
    const bool compact = layout == kLayoutCompact;
    ctx->g_nodes_store.ensure_scratch(n);
    ctx->g.nodes = ctx->g_nodes_store.p;
    ctx->g.layout = layout;
    if (compact) {
        // sources with dead-end flags: 21-bit entries (three per 64-bit word) while ids fit in 20
        // bits, else 32-bit entries; HSAW_PACK=0 keeps plain sources without flags (A/B runs)
        uint32_t bits = n <= (1u << 20) ? 21 : (n <= (1u << 31) ? 32 : 0);
        if (const char* env = std::getenv("HSAW_PACK")) {
            const int v = std::atoi(env);
            if (v == 0) bits = 0;
            if (v == 32 && bits == 21) bits = 32;
        }
        ctx->g.src_bits = bits;
        const uint64_t src_words = bits == 21 ? 2 * (((uint64_t)m + 2) / 3) + 2 : (m ? m : 1);
        // header words first (16-byte aligned), then the sources
        ctx->g_compact_store.ensure_scratch(4ull * n + src_words);
        ctx->g_thr_store.ensure_scratch(m ? m : 1);
        ctx->g.hdr = reinterpret_cast<uint4*>(ctx->g_compact_store.p);
        ctx->g.src = ctx->g_compact_store.p + 4ull * n;
        ctx->g.thr = ctx->g_thr_store.p;
    } else {
        ctx->g_edges_store.ensure_scratch(m ? m : 1);
        ctx->g.edges = ctx->g_edges_store.p;
    }
    return compact;
}

// WeightMode::InDegree rows as build_graph sums them (proj/src/graph.cpp:172-178): 1.0 / d added d
// times, left to right. One thread per row: the sum is a dependent chain by definition. Used by
// hsaw_gpu_graph_upload when the host arrays were verified to hold exactly these sums.
__global__ void indegree_row_cum(uint32_t n, const uint64_t* __restrict__ off,
                                 double* __restrict__ in_cum) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint64_t lo = off[v], hi = off[v + 1];
    if (hi <= lo) return;
    const double wd = 1.0 / (double)(hi - lo);
    double cum = 0.0;
    for (uint64_t i = lo; i < hi; ++i) {
        cum = __dadd_rn(cum, wd);
        in_cum[i] = cum;
    }
}

// Re-lays a device-resident CSR (the reference's arrays) out into the walk kernels' records.
// Synchronises; throws HSAW_EDATA on bad rows.
void install_graph(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const uint64_t* d_off,
                   const uint32_t* d_src, const double* d_cum, const double* d_p) {
    cudaStream_t st = ctx->stream;
    const bool compact = ctx->g.layout == kLayoutCompact;
    uint32_t* d_bad = reinterpret_cast<uint32_t*>(ctx->d_scalars + 60);
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_bad, 0xFF, 8, st));
    {
        StageScope timer(ctx, HSAW_STAGE_UPLOAD);
        build_node_records<<<(n + 255) / 256, 256, 0, st>>>(n, d_off, d_cum, d_p, ctx->g.nodes);
        check_launch(ctx, "build_node_records");
        int blocks = ctx->sm_count * 8;
        const uint32_t big_cap = 1u << 16;
        ctx->chk_list.ensure_scratch(big_cap + 1);  // [0] = count, then the queued row ids
        uint32_t* big_count = ctx->chk_list.p;
        uint32_t* big_rows = ctx->chk_list.p + 1;
        HSAW_CUDA_CHECK(cudaMemsetAsync(big_count, 0, 4, st));
        if (compact) {
            const char* env = std::getenv("HSAW_FORCE_EXACT");  // test hook: exact picks only
            const int force = env && std::atoi(env) != 0;
            build_compact<<<blocks, 256, 0, st>>>(n, d_off, d_src, d_cum, d_p, ctx->g.thr,
                                                  ctx->g.hdr, d_bad, force, big_rows, big_count,
                                                  big_cap);
            check_launch(ctx, "build_compact");
            build_compact_big<<<ctx->sm_count * 2, 256, 0, st>>>(n, d_off, d_src, d_cum, d_p,
                                                                 ctx->g.thr, ctx->g.hdr, d_bad,
                                                                 force, big_rows, big_count, big_cap);
            check_launch(ctx, "build_compact_big");
            if (m && ctx->g.src_bits == 21) {
                const uint64_t words = ((uint64_t)m + 2) / 3;
                pack_sources21<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(
                    m, n, d_src, d_off, d_p, reinterpret_cast<uint64_t*>(ctx->g.src));
                check_launch(ctx, "pack_sources21");
            } else if (m && ctx->g.src_bits == 32) {
                flag_sources32<<<(unsigned)(((uint64_t)m + 255) / 256), 256, 0, st>>>(
                    m, n, d_src, d_off, d_p, ctx->g.src);
                check_launch(ctx, "flag_sources32");
            } else if (m) {
                HSAW_CUDA_CHECK(cudaMemcpyAsync(ctx->g.src, d_src, (uint64_t)m * 4,
                                                cudaMemcpyDeviceToDevice, st));
            }
        } else if (m) {
            build_edge_records<<<blocks, 256, 0, st>>>(n, d_off, d_src, d_cum, ctx->g.nodes, ctx->g.edges,
                                                       d_bad, big_rows, big_count, big_cap);
            check_launch(ctx, "build_edge_records");
            build_edge_records_big<<<ctx->sm_count * 8, 256, 0, st>>>(
                n, d_off, d_src, d_cum, ctx->g.nodes, ctx->g.edges, d_bad, big_rows, big_count, big_cap);
            check_launch(ctx, "build_edge_records_big");
        }
    }
    uint32_t both[2] = {0, 0};
    HSAW_CUDA_CHECK(cudaMemcpyAsync(both, d_bad, 8, cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    if (both[1] != 0xFFFFFFFFu)
        fail(HSAW_EDATA,
             "graph: source id out of range in the row of node " + std::to_string(both[1]));
    if (both[0] != 0xFFFFFFFFu)
        fail(HSAW_EDATA,
             "graph: cumulative weights not increasing at node " + std::to_string(both[0]));
    ctx->g.n = n;
    ctx->g.m = m;
    if (compact) {
        const uint64_t src_bytes =
            ctx->g.src_bits == 21 ? 8 * (((uint64_t)m + 2) / 3) : (uint64_t)m * 4;
        ctx->graph_bytes = (uint64_t)n * (sizeof(NodeRec) + 16) + (uint64_t)m * 8 + src_bytes;
        pin_compact_graph_in_l2(ctx);
    } else {
        ctx->graph_bytes = (uint64_t)n * sizeof(NodeRec) + (uint64_t)m * sizeof(EdgeRec);
        // Round 1 put a stream-wide access-policy window over the node records here (persisting
        // hits, STREAMING misses). On the shapes that take this layout it buys K1 nothing (start
        // nodes are uniform, the records are read for suspects only) and it marks every other
        // access of every kernel on the stream evict-first: the greedy counters, the compaction
        // and the membership filters lost their L2 residency to it (Twitter shape: K1 20.1 ->
        // 18.8 ms, compaction 2.97 -> 1.2 ms per step, index stage 1.43 -> 1.03 s per solve once
        // it was gone). HSAW_L2_PIN_NODES=1 brings it back for A/B runs.
        if (const char* env = std::getenv("HSAW_L2_PIN_NODES"))
            if (std::atoi(env) != 0) pin_node_records_in_l2(ctx);
    }
}

void release_graph(hsaw_gpu_ctx* ctx) { free_graph(ctx); }

}  // namespace hsawgpu

extern "C" {

int hsaw_gpu_ctx_create(int device, void* cuda_stream, hsaw_gpu_ctx** out) {
    if (!out) return HSAW_EINVAL;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return HSAW_ECUDA;  // no CPU fallback: the path needs a CUDA device
    }
    auto* ctx = new hsaw_gpu_ctx;
    ctx->device = device;
    int rc = guarded(ctx, [&] {
        ctx->sm_count = device_info(device).sm_count;
        if (ctx->sm_count <= 0) fail(HSAW_ECUDA, "cannot query the device");
        if (cuda_stream) {
            ctx->stream = static_cast<cudaStream_t>(cuda_stream);
        } else {
            HSAW_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
        adopt_parked_buffers(ctx);
        if (!ctx->d_scalars) HSAW_CUDA_CHECK(cudaMalloc(&ctx->d_scalars, 64 * sizeof(uint64_t)));
        if (!ctx->h_scalars)
            HSAW_CUDA_CHECK(cudaMallocHost(&ctx->h_scalars, 64 * sizeof(uint64_t)));
    });
    if (rc != HSAW_OK) {
        hsaw_gpu_ctx_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return HSAW_OK;
}

void hsaw_gpu_ctx_destroy(hsaw_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    collect_timings(ctx);
    for (cudaEvent_t e : ctx->free_events) cudaEventDestroy(e);
    free_graph(ctx);
    drop_held_csr(ctx);
    park_buffers(ctx);       // keep the device buffers for the next context on this device
    if (ctx->d_scalars) cudaFree(ctx->d_scalars);
    if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
    ctx->release_scratch();  // (now empty) stream-ordered frees precede the stream's destruction
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
        cudaEventDestroy(ctx->side_go);
        cudaEventDestroy(ctx->side_done);
    }
    if (ctx->ahead[0]) {
        for (cudaStream_t a : ctx->ahead) {
            cudaStreamSynchronize(a);
            cudaStreamDestroy(a);
        }
        cudaEventDestroy(ctx->ahead_go);
        for (cudaEvent_t e : ctx->ahead_done) cudaEventDestroy(e);
    }
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* hsaw_gpu_last_error(const hsaw_gpu_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : "no context (CUDA device unavailable?)";
}

void* hsaw_gpu_ctx_cuda_stream(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int hsaw_gpu_ctx_sync(hsaw_gpu_ctx* ctx) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] { HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

uint64_t hsaw_gpu_graph_bytes(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->graph_bytes : 0; }
int hsaw_gpu_graph_layout(const hsaw_gpu_ctx* ctx) {
    if (!ctx || !ctx->g.nodes) return -1;
    return ctx->g.layout == kLayoutCompact ? (int)ctx->g.src_bits : 0;
}
int hsaw_gpu_graph_upload_mode(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->upload_mode : 0; }
uint64_t hsaw_gpu_graph_upload_bytes(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->upload_bytes : 0; }
uint64_t hsaw_gpu_launch_count(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

void hsaw_gpu_debug_counters(double* out3) {
    const AllocStats& a = alloc_stats();
    out3[0] = a.seconds;
    out3[1] = (double)a.calls;
    out3[2] = (double)a.bytes;
}

int hsaw_gpu_stage_times(hsaw_gpu_ctx* ctx, double* ms, uint64_t* count, int reset) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        collect_timings(ctx);
        for (int i = 0; i < HSAW_STAGE_COUNT; ++i) {
            if (ms) ms[i] = ctx->stage_ms[i];
            if (count) count[i] = ctx->stage_launches[i];
            if (reset) {
                ctx->stage_ms[i] = 0;
                ctx->stage_launches[i] = 0;
            }
        }
    });
}

int hsaw_gpu_graph_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const uint64_t* in_offsets,
                          const uint32_t* in_src, const double* in_cum, const double* p_of) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (n == 0) fail(HSAW_EDATA, "graph: no nodes");
        if (!in_offsets || !p_of || (m && (!in_src || !in_cum)))
            fail(HSAW_EINVAL, "graph_upload: null array");
        // HSAW_UPLOAD_TIMING=1: phase times of this call on stderr (host clock, stream synchronised)
        static const bool timing = [] {
            const char* env = std::getenv("HSAW_UPLOAD_TIMING");
            return env && std::atoi(env) != 0;
        }();
        auto t_last = std::chrono::steady_clock::now();
        if (in_offsets[0] != 0 || in_offsets[n] != m)
            fail(HSAW_EDATA, "graph: offsets do not cover edge range");
        {   // 41.6 M offsets at the Twitter shape: 40 ms on one core, shared out over eight
            const unsigned parts = n > (1u << 22) ? 8u : 1u;
            std::vector<uint8_t> bad(parts, 0);
            auto scan = [&](unsigned t) {
                const uint64_t a = (uint64_t)n * t / parts, b = (uint64_t)n * (t + 1) / parts;
                uint8_t any = 0;
                for (uint64_t v = a; v < b; ++v) any |= in_offsets[v + 1] < in_offsets[v];
                bad[t] = any;
            };
            std::vector<std::thread> pool;
            for (unsigned t = 1; t < parts; ++t) pool.emplace_back(scan, t);
            scan(0);
            for (auto& th : pool) th.join();
            for (uint8_t x : bad)
                if (x) fail(HSAW_EDATA, "graph: offsets not monotone");
        }
        auto lap = [&](const char* what) {
            if (!timing) return;
            cudaStreamSynchronize(ctx->stream);
            auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[hsaw upload] %-10s %8.2f ms\n", what,
                         std::chrono::duration<double, std::milli>(t - t_last).count());
            t_last = t;
        };
        lap("checks");
        free_graph(ctx);
        cudaStream_t st = ctx->stream;
        uint64_t* d_off = nullptr;
        uint32_t* d_src = nullptr;
        double *d_cum = nullptr, *d_p = nullptr;
        auto cleanup = [&] {
            if (d_off) cudaFreeAsync(d_off, st);
            if (d_src) cudaFreeAsync(d_src, st);
            if (d_cum) cudaFreeAsync(d_cum, st);
            if (d_p) cudaFreeAsync(d_p, st);
        };
        try {
            prepare_layout(ctx, n, m);
            d_off = static_cast<uint64_t*>(pool_alloc(((uint64_t)n + 1) * 8, st));
            d_src = static_cast<uint32_t*>(pool_alloc((uint64_t)(m ? m : 1) * 4, st));
            d_cum = static_cast<double*>(pool_alloc((uint64_t)(m ? m : 1) * 8, st));
            d_p = static_cast<double*>(pool_alloc((uint64_t)n * 8, st));
            // in_cum is two thirds of the bytes (8 of 12 per edge) and, under the standard LT
            // weighting (WeightMode::InDegree, graph.cpp:172-178), a pure function of the offsets.
            // For large graphs spare host threads check that claim bit for bit while the other
            // arrays are on the wire; if it holds, the sums are regenerated on the device instead
            // of crossing PCIe (Twitter shape: 18.3 -> 6.5 GB per upload). Any other weights, or a
            // single differing bit, take the plain copy. HSAW_UPLOAD_REGEN=0 disables.
            const unsigned hw = std::thread::hardware_concurrency();
            bool try_regen = m >= (1u << 23) && hw >= 12;  // (C2, 16 M edges: 16.3 -> 14.7 ms per call)
            if (const char* env = std::getenv("HSAW_UPLOAD_REGEN")) {
                const int v = std::atoi(env);
                try_regen = v >= 2 ? m > 0 : (v != 0 && try_regen);  // 2, 3 force the attempt (tests)
            }
            // The check and the wire share in_cum through one work list (RowCheck, hostcheck.cpp):
            // the check workers verify chunks from the front while the other arrays are copied;
            // when those are through, this thread copies chunks from the back until the two meet.
            // On an idle 16-core box the workers get through nearly all of it; when the host cores
            // are busy the link takes the tail, so the call never falls behind the plain copy by
            // more than the small part verified in vain. (A fixed split and a rate threshold were
            // both tried: the first cannot know the box's state, the second misfires on start-up.
            // So was building the fat layout's edge records per segment of sources on the side
            // stream while the next segment is on the wire: the build's random gathers slow the
            // incoming DMA by as much as they save - copy 176 -> 211 ms, call 253 vs 255 ms at
            // the Twitter shape, 29 -> 44 ms at C3.)
            std::vector<CopyJob> first, rest;
            first.push_back({d_off, in_offsets, ((uint64_t)n + 1) * 8});
            if (m) rest.push_back({d_src, in_src, (uint64_t)m * 4});
            if (m && !try_regen) rest.push_back({d_cum, in_cum, (uint64_t)m * 8});
            rest.push_back({d_p, p_of, (uint64_t)n * 8});
            uint64_t sent = 0;
            for (const CopyJob& j : first) sent += j.bytes;
            for (const CopyJob& j : rest) sent += j.bytes;
            lap("alloc");
            uint64_t chunk_edges = 1u << 21;  // 16 MB of in_cum per chunk
            if (const char* env = std::getenv("HSAW_UPLOAD_CHUNK_EDGES"))  // tests: many small chunks
                chunk_edges = (uint64_t)std::max(1ll, std::atoll(env));
            std::unique_ptr<RowCheck> check;
            std::thread checker;
            if (try_regen) {
                check.reset(new RowCheck(n, in_offsets, in_cum, chunk_edges));
                checker = std::thread([&] {
                    // beside the 8 copier threads (B200 box, 16 cores: 8 / 12 / 16 workers ->
                    // 258 / 226 / 226 ms for 11.7 GB, against 230 ms more on the wire)
                    unsigned workers = hw >= 16 ? 12u : 4u;
                    if (const char* env = std::getenv("HSAW_UPLOAD_CHECK_THREADS"))
                        workers = (unsigned)std::max(1, std::atoi(env));
                    check->run(workers);
                });
            }
            uint64_t copied_edges = 0;
            try {
                copy_to_device(ctx, first);
                if (try_regen) {
                    // the sums are regenerated on the side stream as soon as the offsets are
                    // there, beside the remaining copies (13 ms at the Twitter shape); chunks that
                    // are copied instead, or everything if the check fails, overwrite them
                    if (!ctx->side) {
                        HSAW_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
                        HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->side_go, cudaEventDisableTiming));
                        HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->side_done, cudaEventDisableTiming));
                    }
                    HSAW_CUDA_CHECK(cudaEventRecord(ctx->side_go, st));
                    HSAW_CUDA_CHECK(cudaStreamWaitEvent(ctx->side, ctx->side_go, 0));
                    indegree_row_cum<<<(n + 255) / 256, 256, 0, ctx->side>>>(n, d_off, d_cum);
                    check_launch(ctx, "indegree_row_cum");
                    HSAW_CUDA_CHECK(cudaEventRecord(ctx->side_done, ctx->side));
                }
                const size_t piece = try_regen ? (size_t)(2u << 20) : 0;
                copy_to_device(ctx, rest, piece);
                if (try_regen) {
                    HSAW_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->side_done, 0));  // join the side stream
                    lap("copy");
                    // HSAW_UPLOAD_REGEN=2 (tests): the whole array goes through the check (3: shared)
                    const char* env = std::getenv("HSAW_UPLOAD_REGEN");
                    const bool share = !(env && std::atoi(env) == 2);
                    uint64_t e0 = 0, e1 = 0;
                    while (share && !check->differs() && check->claim_back(16, &e0, &e1)) {
                        if (e1 == e0) continue;
                        copy_to_device(ctx, {CopyJob{d_cum + e0, in_cum + e0, (e1 - e0) * 8}}, piece);
                        copied_edges += e1 - e0;
                    }
                }
            } catch (...) {
                if (checker.joinable()) checker.join();
                throw;
            }
            if (checker.joinable()) checker.join();
            bool regen_ok = false;
            if (try_regen) {
                lap("check+tail");
                regen_ok = !check->differs();
                if (!regen_ok && m) {
                    copy_to_device(ctx, {CopyJob{d_cum, in_cum, (uint64_t)m * 8}});
                    copied_edges = m;
                    lap("cum");
                }
                sent += copied_edges * 8;
            } else {
                lap("copy");
            }
            install_graph(ctx, n, m, d_off, d_src, d_cum, d_p);
            lap("install");
            ctx->upload_mode = try_regen && regen_ok && copied_edges < m ? 1 : 0;
            ctx->upload_bytes = sent;
        } catch (...) {
            cleanup();
            free_graph(ctx);
            throw;
        }
        cleanup();
    });
}

int hsaw_gpu_suspects_upload(hsaw_gpu_ctx* ctx, const double* p_of) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->g.nodes) fail(HSAW_EINVAL, "suspects_upload: no graph uploaded");
        if (!p_of) fail(HSAW_EINVAL, "suspects_upload: null array");
        uint32_t n = ctx->g.n;
        double* d_p = nullptr;
        d_p = static_cast<double*>(pool_alloc((uint64_t)n * 8, ctx->stream));
        cudaError_t e =
            cudaMemcpyAsync(d_p, p_of, (uint64_t)n * 8, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) {
            update_accept_thresholds<<<(n + 255) / 256, 256, 0, ctx->stream>>>(n, d_p,
                                                                               ctx->g.nodes);
            ++ctx->launches;
            if (ctx->g.layout == kLayoutCompact) {
                update_hdr_suspect_flags<<<(n + 255) / 256, 256, 0, ctx->stream>>>(
                    n, d_p, ctx->g.hdr);
                ++ctx->launches;
                if (ctx->g.m && ctx->g.src_bits) {
                    const uint64_t items =
                        ctx->g.src_bits == 21 ? ((uint64_t)ctx->g.m + 2) / 3 : (uint64_t)ctx->g.m;
                    reflag_sources<<<(unsigned)((items + 255) / 256), 256, 0, ctx->stream>>>(
                        ctx->g.m, ctx->g.hdr, d_p, ctx->g.src_bits, ctx->g.src);
                    ++ctx->launches;
                }
            } else if (ctx->g.m) {
                update_edge_suspect_flags<<<(ctx->g.m + 255) / 256, 256, 0, ctx->stream>>>(
                    ctx->g.m, d_p, ctx->g.edges);
                ++ctx->launches;
            }
            e = cudaStreamSynchronize(ctx->stream);
        }
        cudaFreeAsync(d_p, ctx->stream);
        HSAW_CUDA_CHECK(e);
    });
}

}  // extern "C"
