// Shared host/device plumbing for libhsaw_gpu: error handling, device vectors, the context object
// and the device-side graph layout. Product code — never includes anything from oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <type_traits>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/hsaw_gpu.h"

namespace hsawgpu {

constexpr uint32_t kInvalidNode = 0xFFFFFFFFu;  // proj/include/hsaw/types.hpp:12
constexpr unsigned kFullMask = 0xFFFFFFFFu;

// ---- device-side graph layout ---------------------------------------------------
// One 32-byte sector per node: everything a walk needs on arrival at the node (acceptance
// threshold) and for the next live-edge pick (row start, degree, total-weight threshold, guess
// scale). Thresholds are exact integer images of the reference's doubles: with k = draw >> 11,
// u01 = k * 2^-53 (proj/include/hsaw/prng.hpp:51-53), so
//   r >= c   <=>  k >= ceil(c * 2^53)          ("no edge", graph.hpp:66; "cum > r", :67-78)
//   r <= p   <=>  k <  floor(p * 2^53) + 1      (acceptance, proj/src/sampler.cpp:34,57)
struct __align__(32) NodeRec {
    uint32_t lo;       // first in-edge slot (edge id of the row start); m < 2^32
    uint32_t deg;      // in-degree
    uint64_t tot_thr;  // ceil(in_cum[hi-1] * 2^53); 0 for an empty row
    uint64_t acc_thr;  // 0 = not a suspect; else floor(p_of * 2^53) + 1
    uint64_t scale;    // round(deg / total * 2^31): interpolation guess = (k * scale) >> 84
};
static_assert(sizeof(NodeRec) == 32, "node record must be one 32-byte sector");

// One 32-byte sector per in-edge, in CSR (edge id) order. Besides the pick threshold it carries the
// row header of the edge's SOURCE node, so that in the common case (source is not a suspect and its
// total in-weight is within 2^32 draw units of 1) the walk continues from the edge record alone:
// one dependent sector read per step instead of two. Anything else (suspect source, rows whose
// weights sum well below 1) falls back to the node record — same results, one more load.
struct __align__(32) EdgeRec {
    uint64_t thr;          // ceil(in_cum[e] * 2^53): slot e is picked iff thr[e-1] <= k < thr[e]
    uint32_t src;          // in_src[e]
    uint32_t prev_hi;      // thr[e-1] >> 21 (0 for the first slot of a row): one-load verification
    uint32_t src_lo;       // NodeRec(src).lo
    uint32_t src_deg;      // NodeRec(src).deg
    uint32_t src_deficit;  // 2^53 - NodeRec(src).tot_thr when kEdgeSimple is set
    uint32_t flags;        // kEdgeSuspect: src is a suspect; kEdgeSimple: header fields are usable
};
static_assert(sizeof(EdgeRec) == 32, "edge record must be one 32-byte sector");
constexpr uint32_t kEdgeSuspect = 1u, kEdgeSimple = 2u;

// Compact layout: when 4 m + 8 n bytes fit in L2, a step reads in_src[e] (4 bytes)
// and the 8-byte row header of the source instead of a 32-byte edge record, and both arrays stay
// L2 resident (the headers are 16 bytes: row start, w, and the top 32 bits of the acceptance
// threshold, so one gather settles an arrival). w = deg (25 bits) | margin exponent mb (6 bits) |
// suspect (1 bit).
// A row is "arithmetic" when its thresholds sit within a margin of the ideal (i+1) * 2^53 / deg
// grid (always the case for 1/d rows): then slot = (k * deg) >> 53 is exact for every draw whose
// fractional part keeps 2^mb clear of a slot boundary, and the thresholds are never read. Draws
// inside the margin and rows with mb == kHdrSlow take the exact path (node record + binary search
// over thr[]), so arbitrary weights stay bit-exact, only slower.
constexpr uint32_t kHdrDegBits = 25, kHdrDegMask = (1u << kHdrDegBits) - 1, kHdrSlow = 63;
constexpr int kLayoutFat = 0, kLayoutCompact = 1;

struct DeviceGraph {
    uint32_t n = 0, m = 0;
    int layout = kLayoutFat;
    NodeRec* nodes = nullptr;
    EdgeRec* edges = nullptr;         // fat layout only
    uint4* hdr = nullptr;             // compact layout: (lo, w, acceptance code, 0) per node;
                                      // code 0 = not a suspect, else (acc_thr >> 21) + 1
    // compact layout: in_src with a "dead end" flag per entry (the source has an empty in-row and
    // is not a suspect: the walk ends there and its header is never read). src_bits selects the
    // form: 21 = three entries per 64-bit word (20-bit node id + flag; n <= 2^20: 2.67 bytes per
    // edge, the hot set of C2 drops from 80 to 59 MB), 32 = one u32 per entry with the flag in
    // bit 31 (n <= 2^31), 0 = plain u32 without flags (HSAW_PACK=0, A/B runs).
    uint32_t* src = nullptr;
    uint32_t src_bits = 0;
    uint64_t* thr = nullptr;          // compact layout: ceil(in_cum * 2^53), exact path only
};

// ---- errors ------------------------------------------------------------------------------------
struct Error {
    int status;
    std::string msg;
};

#define HSAW_CUDA_CHECK(expr)                                                                  \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            throw ::hsawgpu::Error{HSAW_ECUDA, std::string(#expr) + ": " +                     \
                                                   cudaGetErrorString(_e)};                    \
    } while (0)

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error{status, msg}; }

// ---- device memory: stream-ordered pool allocations ---------------------------------------------
// All device buffers come from the device's default cudaMallocAsync pool (release threshold set to
// "never" at context creation), ordered on the context stream: growing a scratch buffer or the
// walk pool costs no device synchronisation and freed memory is reused by the next request.
// The stream in effect is the one of the C-ABI call being served (set by guarded()).
inline cudaStream_t& current_stream() {
    static thread_local cudaStream_t st = nullptr;
    return st;
}

// Host-side cost of pool allocations (debug counters, read through hsaw_gpu_debug_counters).
struct AllocStats {
    double seconds = 0;
    uint64_t calls = 0, bytes = 0;
};
inline AllocStats& alloc_stats() {
    static AllocStats s;
    return s;
}

// Allocation sizes are rounded up to 1/8-octave classes (<= 12.5 % slack) so that buffers freed
// by one round / stream are exact-fit candidates for the next and the pool does not fragment.
// Beyond 1 GiB (graph stores, sort buffers of the C4 / C5 shapes) the classes are 64 MiB steps: a
// 47 GB edge-record store must not carry gigabytes of slack.
inline uint64_t size_class(uint64_t bytes) {
    if (bytes <= (1ull << 16)) return 1ull << 16;
    if (bytes > (1ull << 30)) return (bytes + (1ull << 26) - 1) & ~((1ull << 26) - 1);
    int top = 63 - __builtin_clzll(bytes);
    uint64_t step = 1ull << (top - 3);
    return (bytes + step - 1) & ~(step - 1);
}

// The context whose C-ABI call this thread is serving (set by guarded()), and the last resort of a
// failing allocation: a hook that drops that context's IDLE caches (the recycled walk-pool buffers
// of finished streams: tens of gigabytes of mapped virtual memory at the Twitter shape, which no
// pool trim can reach). Registered by graph.cu.
inline hsaw_gpu_ctx*& current_ctx() {
    static thread_local hsaw_gpu_ctx* c = nullptr;
    return c;
}
using OomHook = void (*)(hsaw_gpu_ctx*);
inline OomHook& oom_hook() {
    static OomHook h = nullptr;
    return h;
}
inline void run_oom_hook() {
    if (oom_hook() && current_ctx()) oom_hook()(current_ctx());
}

// cudaMallocAsync with one retry after dropping idle caches and handing the pool's cached blocks
// back to the driver (the pool never releases memory on its own: release threshold "never").
inline void* pool_alloc(uint64_t bytes, cudaStream_t st) {
    void* np = nullptr;
    cudaError_t e = cudaMallocAsync(&np, bytes, st);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        cudaStreamSynchronize(st);
        run_oom_hook();
        int dev = 0;
        cudaMemPool_t pool = nullptr;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
            cudaMemPoolTrimTo(pool, 0);
        e = cudaMallocAsync(&np, bytes, st);
    }
    if (e != cudaSuccess)
        throw ::hsawgpu::Error{HSAW_ECUDA, "device allocation of " + std::to_string(bytes) +
                                               " bytes: " + cudaGetErrorString(e)};
    return np;
}

template <class T>
struct DevVec {
    T* p = nullptr;
    uint64_t size = 0, cap = 0;
    cudaStream_t owner = nullptr;  // stream the buffer was allocated on

    DevVec() = default;
    DevVec(const DevVec&) = delete;
    DevVec& operator=(const DevVec&) = delete;
    DevVec(DevVec&& o) noexcept { swap(o); }
    DevVec& operator=(DevVec&& o) noexcept {
        if (this != &o) {
            release();
            swap(o);
        }
        return *this;
    }
    ~DevVec() { release(); }

    void release() {
        if (p) cudaFreeAsync(p, owner);
        p = nullptr;
        size = cap = 0;
    }
    void swap(DevVec& o) {
        std::swap(p, o.p);
        std::swap(size, o.size);
        std::swap(cap, o.cap);
        std::swap(owner, o.owner);
    }
    // `count` is rounded up in place to the size class actually allocated.
    static T* alloc(uint64_t& count, cudaStream_t st) {
        T* np = nullptr;
        uint64_t bytes = size_class(count * sizeof(T));
        count = bytes / sizeof(T);
        auto t0 = std::chrono::steady_clock::now();
        np = static_cast<T*>(pool_alloc(bytes, st));
        AllocStats& a = alloc_stats();
        a.seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        a.calls += 1;
        a.bytes += bytes;
        return np;
    }
    void ensure_exact(uint64_t want) {  // no headroom (large one-off buffers)
        if (want <= cap) return;
        cudaStream_t st = current_stream();
        if (p) cudaFreeAsync(p, owner);
        p = nullptr;
        cap = 0;
        uint64_t ncap = want;
        p = alloc(ncap, st);
        cap = ncap;
        owner = st;
    }
    // Grows capacity (doubling) preserving the first `size` elements; stream-ordered, no sync.
    void reserve(uint64_t want, cudaStream_t st) {
        if (want <= cap) return;
        uint64_t ncap = cap * 2;
        if (ncap < want) ncap = want;
        if (ncap < 1024) ncap = 1024;
        T* np = alloc(ncap, st);
        if (p && size) {
            cudaError_t e = cudaMemcpyAsync(np, p, size * sizeof(T), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) {
                cudaFreeAsync(np, st);
                HSAW_CUDA_CHECK(e);
            }
        }
        if (p) cudaFreeAsync(p, st);
        p = np;
        cap = ncap;
        owner = st;
    }
    // Scratch use: capacity only, contents undefined. Small buffers get 50 % headroom so that a
    // slightly larger request of the next round still fits; buffers past 1 GiB are sized exactly.
    void ensure_scratch(uint64_t want) {
        if (want <= cap) return;
        cudaStream_t st = current_stream();
        if (p) cudaFreeAsync(p, owner);
        p = nullptr;
        cap = 0;
        uint64_t ncap = want * sizeof(T) > (1ull << 30) ? want : want + want / 2;
        p = alloc(ncap, st);
        cap = ncap;
        owner = st;
    }
};


// ---- growable device arrays on CUDA virtual memory ------------------------------------------------
// The walk pool of a stream is the one structure whose final size is not known in advance (the
// doubling loop decides) and that reaches tens of gigabytes at the Twitter shape. A DevVec grows by
// allocate-copy-free, which needs old + new at once (3x the payload while doubling); a GrowVec
// reserves virtual address space for the whole device once and maps physical chunks behind the
// data as it grows: the array never moves, nothing is copied and the peak is the payload itself.
// The driver entry points are resolved through the runtime (no link-time libcuda dependency, so
// the library still loads on a machine without a driver); without them a GrowVec behaves like a
// DevVec.
struct VmmApi {
    CUresult (*address_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*address_free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                       unsigned long long) = nullptr;
    CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    bool ok = false;

    static const VmmApi& get() {
        static const VmmApi api = [] {
            VmmApi a;
            auto load = [](const char* name, auto& fn) {
                void* ptr = nullptr;
                cudaDriverEntryPointQueryResult q{};
                if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) != cudaSuccess ||
                    q != cudaDriverEntryPointSuccess || !ptr) {
                    cudaGetLastError();
                    return false;
                }
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(ptr);
                return true;
            };
            const char* off = std::getenv("HSAW_VMM");  // A/B knob: HSAW_VMM=0 -> plain DevVec growth
            a.ok = !(off && std::atoi(off) == 0) &&
                   load("cuMemAddressReserve", a.address_reserve) &&
                   load("cuMemAddressFree", a.address_free) && load("cuMemCreate", a.create) &&
                   load("cuMemRelease", a.release) && load("cuMemMap", a.map) &&
                   load("cuMemUnmap", a.unmap) && load("cuMemSetAccess", a.set_access) &&
                   load("cuMemGetAllocationGranularity", a.granularity);
            return a;
        }();
        return api;
    }
};

template <class T>
struct GrowVec {
    T* p = nullptr;
    uint64_t size = 0, cap = 0;  // elements; cap = mapped capacity
    cudaStream_t owner = nullptr;

    GrowVec() = default;
    GrowVec(const GrowVec&) = delete;
    GrowVec& operator=(const GrowVec&) = delete;
    GrowVec(GrowVec&& o) noexcept { swap(o); }
    GrowVec& operator=(GrowVec&& o) noexcept {
        if (this != &o) {
            release();
            swap(o);
        }
        return *this;
    }
    ~GrowVec() { release(); }

    void swap(GrowVec& o) {
        std::swap(p, o.p);
        std::swap(size, o.size);
        std::swap(cap, o.cap);
        std::swap(owner, o.owner);
        std::swap(base_, o.base_);
        std::swap(va_bytes_, o.va_bytes_);
        std::swap(mapped_, o.mapped_);
        std::swap(device_, o.device_);
        chunks_.swap(o.chunks_);
        plain_.swap(o.plain_);
    }

    // Grows in place (contents preserved, pointer stable once mapped) to hold `want` elements.
    void reserve(uint64_t want, cudaStream_t st) {
        if (want <= cap) return;
        const VmmApi& api = VmmApi::get();
        if (!api.ok) {  // no virtual memory management: allocate-copy-free
            plain_.size = size;
            plain_.reserve(want, st);
            p = plain_.p;
            cap = plain_.cap;
            owner = st;
            return;
        }
        owner = st;
        CUmemAllocationProp prop{};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        if (!base_) {
            HSAW_CUDA_CHECK(cudaGetDevice(&device_));
            prop.location.id = device_;
            size_t gran = 0;
            if (api.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran)
                gran = 2u << 20;
            gran_ = gran;
            size_t free_b = 0, total_b = 0;
            HSAW_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
            va_bytes_ = round_up(total_b, gran_);
            if (api.address_reserve(&base_, va_bytes_, 0, 0, 0) != CUDA_SUCCESS)
                throw ::hsawgpu::Error{HSAW_ECUDA, "cuMemAddressReserve failed"};
        }
        prop.location.id = device_;
        const uint64_t need = round_up(want * sizeof(T), gran_);
        if (need > va_bytes_)
            throw ::hsawgpu::Error{HSAW_ECUDA, "device allocation of " + std::to_string(need) +
                                                   " bytes: out of memory"};
        // map at least a quarter more than is already there (bounded), so a pool that grows chunk
        // by chunk needs a few dozen driver calls over its life, not one per chunk
        uint64_t grow = need - mapped_;
        const uint64_t floor_b = std::min<uint64_t>(std::max<uint64_t>(mapped_ / 4, 32ull << 20), 2ull << 30);
        if (grow < floor_b) grow = std::min<uint64_t>(round_up(floor_b, gran_), va_bytes_ - mapped_);
        CUmemGenericAllocationHandle h{};
        CUresult rc = api.create(&h, grow, &prop, 0);
        if (rc == CUDA_ERROR_OUT_OF_MEMORY) {
            // physical memory may sit in the stream-ordered pool's cache or in the idle walk-pool
            // buffers of finished streams: hand it back and retry with the exact need
            cudaStreamSynchronize(st);
            run_oom_hook();
            cudaMemPool_t pool = nullptr;
            if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
            grow = need - mapped_;
            rc = api.create(&h, grow, &prop, 0);
        }
        if (rc != CUDA_SUCCESS)
            throw ::hsawgpu::Error{HSAW_ECUDA, "device allocation of " + std::to_string(grow) +
                                                   " bytes: out of memory"};
        CUmemAccessDesc acc{};
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (api.map(base_ + mapped_, grow, 0, h, 0) != CUDA_SUCCESS ||
            api.set_access(base_ + mapped_, grow, &acc, 1) != CUDA_SUCCESS) {
            api.release(h);
            throw ::hsawgpu::Error{HSAW_ECUDA, "cuMemMap failed"};
        }
        chunks_.push_back({h, grow});
        mapped_ += grow;
        p = reinterpret_cast<T*>(base_);
        cap = mapped_ / sizeof(T);
        AllocStats& a = alloc_stats();
        a.calls += 1;
        a.bytes += grow;
    }

    // Unmaps and frees everything. Work that touches the array must have finished: the owning
    // stream is synchronised first.
    void release() {
        if (base_) {
            const VmmApi& api = VmmApi::get();
            if (owner) cudaStreamSynchronize(owner);
            uint64_t at = 0;
            for (auto& c : chunks_) {
                api.unmap(base_ + at, c.second);
                api.release(c.first);
                at += c.second;
            }
            api.address_free(base_, va_bytes_);
        }
        chunks_.clear();
        plain_.release();
        base_ = 0;
        va_bytes_ = mapped_ = 0;
        p = nullptr;
        size = cap = 0;
    }
    // process teardown after the CUDA context is gone: forget without calling the driver
    void abandon() {
        chunks_.clear();
        plain_.p = nullptr;
        plain_.cap = plain_.size = 0;
        base_ = 0;
        va_bytes_ = mapped_ = 0;
        p = nullptr;
        size = cap = 0;
    }
    void rebind(cudaStream_t st) {
        owner = st;
        plain_.owner = st;
    }

private:
    static uint64_t round_up(uint64_t x, uint64_t g) { return (x + g - 1) / g * g; }
    CUdeviceptr base_ = 0;
    uint64_t va_bytes_ = 0, mapped_ = 0, gran_ = 2u << 20;
    int device_ = 0;
    std::vector<std::pair<CUmemGenericAllocationHandle, uint64_t>> chunks_;
    DevVec<T> plain_;  // fallback storage when the driver entry points are unavailable
};

// Per-chunk scratch of the sample stream (stream.cu). Lives in the context so that consecutive
// streams on one graph (the doubling loop is re-run per esia() call) reuse it without allocating.
struct SamplerScratch {
    DevVec<uint64_t> slot_seed, enc_seed, tmp_off, voff, enc_batch;
    DevVec<uint32_t> slot_len, count, first, enc_len, enc_seq, tmp_nodes, tmp_edges, vidx;
    DevVec<uint8_t> status;
    // fused path: pair-log arena written by K1, per-slot log offsets, per-walk log pointers,
    // replay space + selection list for walks whose log overflowed
    DevVec<uint2> arena, replay;
    DevVec<uint32_t> slot_log, ovf_pairs, sel;
    DevVec<uint64_t> enc_src;
    DevVec<uint64_t> k1_words;  // [0] K1's work cursor, [1] its arena cursor (fused path)
    void release() {
        k1_words.release();
        arena.release(); replay.release(); slot_log.release(); ovf_pairs.release();
        sel.release(); enc_src.release();
        slot_seed.release(); enc_seed.release(); tmp_off.release(); voff.release();
        enc_batch.release(); slot_len.release(); count.release(); first.release();
        enc_len.release(); enc_seq.release(); tmp_nodes.release(); tmp_edges.release();
        vidx.release(); status.release();
    }
};

// A device-resident CSR in the reference's own arrays (in_offsets / in_src / in_cum), held by the
// context between a device-side build (rmat.cu) and its installation / download.
struct HeldCsr {
    DevVec<uint64_t> off;
    DevVec<uint32_t> src;
    DevVec<double> cum;
    uint32_t n = 0;
    uint64_t m = 0;
    bool valid = false;
};

// Partitioned sampling (proj/src/partition.cpp:153-279, sampler.cpp:510-539): while a restricted
// stream samples a chunk, the sampler launches read the restriction from the context.
struct Restriction {
    const uint32_t* domain = nullptr;  // device: start nodes (a part's base list)
    uint32_t ndomain = 0;
    const uint8_t* allowed = nullptr;  // device: byte mask over nodes (the part's h-hop extension)
    uint32_t* out_cross = nullptr;     // device: crossings per batch of the launch
};

// Walk-pool buffers handed back by a destroyed stream, taken over by the next one.
// Buffers of the dense reduced greedy instance (greedy.cu, build_dense): kept on the context like
// the other greedy scratch, so a solve's six greedy calls do not churn gigabytes through the pool.
struct DenseScratch {
    DevVec<uint32_t> bits, pc, base, bloom, ids, cnt, items, pw, pr, sw, flag;
    DevVec<uint64_t> map, start;
    template <class F>
    void for_each(F&& f) {
        f(bits); f(pc); f(base); f(bloom); f(ids); f(cnt); f(items); f(pw); f(pr); f(sw); f(flag);
        f(map); f(start);
    }
    void release() {
        for_each([](auto& v) { v.release(); });
    }
    void swap(DenseScratch& o) {
        bits.swap(o.bits); pc.swap(o.pc); base.swap(o.base); bloom.swap(o.bloom); ids.swap(o.ids);
        cnt.swap(o.cnt); items.swap(o.items); pw.swap(o.pw); pr.swap(o.pr); sw.swap(o.sw);
        flag.swap(o.flag); map.swap(o.map); start.swap(o.start);
    }
};

struct PoolCache {
    DevVec<uint64_t> edge_off, tag_batch, accepted_after_batch;
    DevVec<uint32_t> tag_seq;
    GrowVec<uint32_t> nodes, edges;  // the two big ones: grown in place (virtual memory)
    void release() {
        edge_off.release(); tag_batch.release(); accepted_after_batch.release();
        nodes.release(); edges.release(); tag_seq.release();
    }
};

}  // namespace hsawgpu

// ---- the context (opaque to C callers) ---------------------------------------------------------
struct hsaw_gpu_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    hsawgpu::DeviceGraph g;
    uint64_t graph_bytes = 0;
    int upload_mode = 0;  // in_cum of the last graph_upload: 0 copied, 1 (partly) regenerated on the device
    uint64_t upload_bytes = 0;  // bytes the last graph_upload copied host -> device
    // side stream for work that may run beside the context stream (the replay of walks that
    // outgrew their log chunk, sampler.cu launch_decode_pairs / join_side_stream)
    cudaStream_t side = nullptr;
    cudaEvent_t side_go = nullptr, side_done = nullptr;
    bool side_pending = false;
    // second stream for the chunk that is sampled AHEAD (stream.cu sample_range): K1 of chunk
    // i + 1 runs on it beside the recheck / compaction of chunk i on the context stream.
    // k1_stream is non-null only while such a launch is being queued.
    // (two of them, used alternately: consecutive K1 launches overlap each other's tails, the
    // last lanes of a launch chase the longest walks for a millisecond or more)
    cudaStream_t ahead[2] = {nullptr, nullptr};
    cudaEvent_t ahead_go = nullptr, ahead_done[2] = {nullptr, nullptr};
    cudaStream_t k1_stream = nullptr;
    // L2 access-policy window over the compact graph (headers + sources), attached to the K1
    // launches only: those lines are marked persisting, so the walk-log stream of the same kernel
    // cannot evict them, while every other kernel on the stream keeps normal caching.
    cudaAccessPolicyWindow k1_window{};
    bool k1_window_on = false;
    uint64_t launches = 0;
    uint64_t greedy_full_index_reruns = 0;  // thresholded index was too optimistic (diagnostic)
    uint64_t last_greedy_min_gain = 0;      // smallest per-round gain of the last hsaw_gpu_greedy
    std::string last_error;
    // reusable scratch
    hsawgpu::DevVec<unsigned char> cub_tmp;
    hsawgpu::DevVec<hsawgpu::NodeRec> g_nodes_store;  // backing store of g.nodes / g.edges
    hsawgpu::DevVec<hsawgpu::EdgeRec> g_edges_store;
    hsawgpu::DevVec<uint32_t> g_compact_store;  // compact layout: 4 n header words, then m sources
    hsawgpu::DevVec<uint64_t> g_thr_store;      // compact layout: pick thresholds (exact path)
    hsawgpu::DevVec<uint32_t> chk_list, chk_mid, chk_counters;  // distinctness-check scratch
    hsawgpu::SamplerScratch samp;                        // per-chunk sampler scratch
    hsawgpu::SamplerScratch samp2;  // K1 outputs of the chunk sampled ahead (slot arrays, counts, arena)
    hsawgpu::PoolCache pool_cache;                       // recycled walk-pool buffers
    hsawgpu::HeldCsr held;                               // device-built CSR awaiting install / fetch
    hsawgpu::Restriction restr;                          // set only while a restricted chunk runs
    uint32_t rng_mode = 0;  // draw source of the sampler launches of the running chunk (cfg.rng_mode)
    // greedy / coverage scratch (greedy.cu), reused across the doubling iterations
    hsawgpu::DevVec<uint32_t> g_cand_bits, g_cnt, g_fill, g_inv, g_covered, g_solution, g_query_bits;
    hsawgpu::DevVec<uint32_t> g_indexed_bits;  // items that own an inverted list
    hsawgpu::DevVec<uint32_t> g_filter;        // hashed membership pre-filter (greedy.cu BitFilter)
    hsawgpu::DevVec<uint32_t> g_hist_prefix, g_hist_seg;  // histogram cache (greedy.cu HistCache)
    hsawgpu::DevVec<uint32_t> g_sorted;  // radix-partitioned copy of the items (large id spaces)
    hsawgpu::DenseScratch g_dense;       // dense reduced instance (large id spaces)
    hsawgpu::DevVec<uint64_t> g_pos, g_partial, g_gains, g_blkmax;
    uint64_t* d_scalars = nullptr;  // 64 u64 of device scratch for counters / cursors
    uint64_t* h_scalars = nullptr;  // pinned mirror
    // per-stage device time, measured with CUDA events on `stream` around the kernels themselves
    struct Pending {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<cudaEvent_t> free_events;
    std::vector<Pending> pending;
    double stage_ms[HSAW_STAGE_COUNT] = {};
    uint64_t stage_launches[HSAW_STAGE_COUNT] = {};

    // Swaps every reusable device buffer with `o` (used to park the buffers of a dying context in
    // a per-device cache and to hand them to the next context: a fresh DeviceGraph per call — the
    // host-buffer e2e path — then allocates nothing in steady state).
    void swap_buffers(hsaw_gpu_ctx& o) {
        g_nodes_store.swap(o.g_nodes_store);
        g_edges_store.swap(o.g_edges_store);
        g_compact_store.swap(o.g_compact_store);
        g_thr_store.swap(o.g_thr_store);
        cub_tmp.swap(o.cub_tmp);
        chk_list.swap(o.chk_list);
        chk_mid.swap(o.chk_mid);
        chk_counters.swap(o.chk_counters);
        std::swap(samp, o.samp);
        std::swap(samp2, o.samp2);
        std::swap(pool_cache, o.pool_cache);
        g_cand_bits.swap(o.g_cand_bits);
        g_cnt.swap(o.g_cnt);
        g_fill.swap(o.g_fill);
        g_inv.swap(o.g_inv);
        g_covered.swap(o.g_covered);
        g_solution.swap(o.g_solution);
        g_query_bits.swap(o.g_query_bits);
        g_pos.swap(o.g_pos);
        g_partial.swap(o.g_partial);
        g_gains.swap(o.g_gains);
        g_blkmax.swap(o.g_blkmax);
        g_sorted.swap(o.g_sorted);
        g_indexed_bits.swap(o.g_indexed_bits);
        g_filter.swap(o.g_filter);
        g_hist_prefix.swap(o.g_hist_prefix);
        g_hist_seg.swap(o.g_hist_seg);
        g_dense.swap(o.g_dense);
    }
    template <class F>
    void for_each_buffer(F&& f) {
        f(g_nodes_store); f(g_edges_store); f(g_compact_store); f(g_thr_store); f(cub_tmp); f(chk_list); f(chk_mid); f(chk_counters);
        f(samp.slot_seed); f(samp.enc_seed); f(samp.tmp_off); f(samp.voff); f(samp.enc_batch);
        f(samp.slot_len); f(samp.count); f(samp.first); f(samp.enc_len); f(samp.enc_seq);
        f(samp.tmp_nodes); f(samp.tmp_edges); f(samp.vidx); f(samp.status); f(samp.arena);
        f(samp.replay); f(samp.slot_log); f(samp.ovf_pairs); f(samp.sel); f(samp.enc_src);
        f(samp.k1_words);
        f(samp2.slot_seed); f(samp2.slot_len); f(samp2.slot_log); f(samp2.count); f(samp2.first);
        f(samp2.arena); f(samp2.k1_words);
        f(pool_cache.edge_off); f(pool_cache.tag_batch); f(pool_cache.accepted_after_batch);
        f(pool_cache.tag_seq);  // pool_cache.nodes / .edges are GrowVecs: handled by the callers
        f(g_cand_bits); f(g_cnt); f(g_fill); f(g_inv); f(g_covered); f(g_solution);
        f(g_query_bits); f(g_pos); f(g_partial); f(g_gains); f(g_blkmax); f(g_sorted);
        f(g_indexed_bits); f(g_filter); f(g_hist_prefix); f(g_hist_seg);
        g_dense.for_each(f);
    }

    // The buffers a solve leaves behind (greedy index, histogram cache, partition copy): tens of
    // gigabytes at the Twitter shape, worthless once another graph is installed. Back to the pool.
    void release_solve_scratch() {
        g_cand_bits.release(); g_cnt.release(); g_fill.release(); g_inv.release();
        g_covered.release(); g_solution.release(); g_query_bits.release(); g_pos.release();
        g_partial.release(); g_gains.release(); g_blkmax.release(); g_sorted.release();
        g_indexed_bits.release(); g_filter.release(); g_hist_prefix.release(); g_hist_seg.release();
        g_dense.release();
    }

    void release_scratch() {
        g_nodes_store.release();
        g_edges_store.release();
        g_compact_store.release();
        g_thr_store.release();
        samp.release();
        samp2.release();
        pool_cache.release();
        cub_tmp.release();
        chk_list.release();
        chk_mid.release();
        chk_counters.release();
        g_cand_bits.release();
        g_cnt.release();
        g_fill.release();
        g_inv.release();
        g_covered.release();
        g_solution.release();
        g_query_bits.release();
        g_pos.release();
        g_partial.release();
        g_gains.release();
        g_blkmax.release();
        g_sorted.release();
        g_indexed_bits.release();
        g_filter.release();
        g_hist_prefix.release();
        g_hist_seg.release();
        g_dense.release();
    }
};

namespace hsawgpu {

// Runs `f`, mapping exceptions to status codes and recording the message on the context.
template <class F>
int guarded(hsaw_gpu_ctx* ctx, F&& f) {
    try {
        if (ctx) {
            HSAW_CUDA_CHECK(cudaSetDevice(ctx->device));
            current_stream() = ctx->stream;
            current_ctx() = ctx;
        }
        f();
        return HSAW_OK;
    } catch (const Error& e) {
        if (ctx) ctx->last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->last_error = "host allocation failed";
        return HSAW_ECUDA;
    } catch (const std::exception& e) {
        if (ctx) ctx->last_error = e.what();
        return HSAW_ECUDA;
    }
}

inline void check_launch(hsaw_gpu_ctx* ctx, const char* what) {
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(HSAW_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- stage timing: tic/toc bracket kernels with events; collect() after a stream sync ----------
struct StageScope {
    hsaw_gpu_ctx* ctx;
    int stage;
    cudaEvent_t a = nullptr, b = nullptr;
    static cudaEvent_t get(hsaw_gpu_ctx* c) {
        if (!c->free_events.empty()) {
            cudaEvent_t e = c->free_events.back();
            c->free_events.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        HSAW_CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    cudaStream_t on = nullptr;
    StageScope(hsaw_gpu_ctx* c, int s, cudaStream_t stream = nullptr)
        : ctx(c), stage(s), on(stream ? stream : c->stream) {
        a = get(c);
        b = get(c);
        cudaEventRecord(a, on);
    }
    ~StageScope() {
        cudaEventRecord(b, on);
        ctx->pending.push_back({stage, a, b});
        ++ctx->stage_launches[stage];
    }
};

// Folds finished event pairs into ctx->stage_ms. Call after the stream has been synchronised.
inline void collect_timings(hsaw_gpu_ctx* ctx) {
    size_t kept = 0;
    for (auto& p : ctx->pending) {
        // a pair recorded on the second stream (a chunk sampled ahead) may still be running
        if (cudaEventQuery(p.b) == cudaErrorNotReady) {
            ctx->pending[kept++] = p;
            continue;
        }
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) ctx->stage_ms[p.stage] += ms;
        ctx->free_events.push_back(p.a);
        ctx->free_events.push_back(p.b);
    }
    ctx->pending.resize(kept);
    cudaGetLastError();
}

// ---- graph installation (graph.cu), shared with the device CSR builder (build.cu) ----------------
struct CopyJob {
    void* dst;
    const void* src;
    size_t bytes;
};
void copy_to_device(hsaw_gpu_ctx* ctx, const std::vector<CopyJob>& jobs, size_t piece_bytes = 0);
void copy_to_host(hsaw_gpu_ctx* ctx, const std::vector<CopyJob>& jobs);
bool prepare_layout(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m);
// Kernel-side view of DeviceGraph::src (passed by value in the kernel parameter structs).
struct SrcRef {
    const uint32_t* p;
    uint32_t bits;
};
inline SrcRef src_ref(const DeviceGraph& g) { return SrcRef{g.src, g.src_bits}; }
void install_graph(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const uint64_t* d_off,
                   const uint32_t* d_src, const double* d_cum, const double* d_p);
void release_graph(hsaw_gpu_ctx* ctx);
void drop_held_csr(hsaw_gpu_ctx* ctx);  // rmat.cu
// Device CSR builder (build.cu): edge list -> resident graph in the chosen layout. on_device: the
// edge arrays are device pointers (the text parser's output) instead of host arrays.
void build_and_install(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                       const uint32_t* edge_v, const double* edge_w, int weight_mode,
                       const double* host_p_of, bool on_device);

// exclusive prefix sums (CUB) on the context stream; out may have a wider type than in
void exclusive_sum_u32_to_u64(hsaw_gpu_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t count);
void exclusive_sum_u32(hsaw_gpu_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t count);
void exclusive_sum_u8_to_u32(hsaw_gpu_ctx* ctx, const uint8_t* in, uint32_t* out, uint64_t count);

}  // namespace hsawgpu
