// Greedy max-cover on device-resident walks (kernels K3-K6):
//   K3  item_histogram     marginal-gain counts = occurrences of each candidate item in R_t
//   K3b scatter_inverted   item -> walks inverted index (counting sort: histogram, scan, scatter)
//   K4  block_maxima / select_lazy   lazily maintained block maxima of (count desc, id asc) keys
//   K5  cover_winner       final argmax + mark the winner's walks covered + decrement the counts
//                          of every other item in those walks
//   K6  count_covered      CoverageIndex::coverage_of
// Semantics follow proj/src/coverage.cpp:91-166: each round selects the candidate with the largest
// number of still-uncovered walks containing it, ties to the smallest id; rounds whose best gain
// is zero are padded with the smallest unselected candidate ids (host side).
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "stream.cuh"

using namespace hsawgpu;


namespace {
struct WalkView;
}

namespace {

// Walks [w0, w0 + cnt) of either source. Walk w occupies items[off[w] + add*w, off[w+1] + add*(w+1)).
struct WalkView {
    const uint64_t* off;
    const uint32_t* items;
    uint64_t w0, cnt;
    uint32_t add;  // 1 for the node arrays of a stream (len + 1 nodes per walk), else 0
    uint32_t limit;
};

__device__ __forceinline__ void walk_extent(const WalkView& v, uint64_t w, uint64_t& b, uint64_t& e) {
    b = v.off[w] + v.add * w;
    e = v.off[w + 1] + v.add * (w + 1);
}

__device__ __forceinline__ bool is_cand(const uint32_t* __restrict__ cand_bits, uint32_t item) {
    return cand_bits == nullptr || ((cand_bits[item >> 5] >> (item & 31)) & 1u);
}

// Membership pre-filter for bitmaps that do not fit L2 (m / 8 bytes = 183 MB at the Twitter shape):
// one hashed bit per member in a table small enough to stay cached (64 KB..16 MB). A clear bit
// proves non-membership, so the random DRAM read of the real bitmap is only paid for members and
// the few false positives; answers are unchanged. log2 == 0 disables the filter.
struct BitFilter {
    const uint32_t* bits;
    uint32_t log2;  // table size in bits = 2^log2
};
__device__ __forceinline__ uint32_t filter_slot(uint32_t item, uint32_t log2) {
    return (item * 0x9E3779B1u) >> (32 - log2);
}
__device__ __forceinline__ bool filter_pass(const BitFilter& f, uint32_t item) {
    if (f.log2 == 0) return true;
    const uint32_t h = filter_slot(item, f.log2);
    return (__ldg(f.bits + (h >> 5)) >> (h & 31)) & 1u;
}
__global__ void set_filter_bits(const uint32_t* __restrict__ ids, uint64_t n, uint32_t log2,
                                uint32_t* __restrict__ filter) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t h = filter_slot(ids[i], log2);
    atomicOr(&filter[h >> 5], 1u << (h & 31));
}

__global__ void set_bits(const uint32_t* __restrict__ ids, uint64_t n, uint32_t* __restrict__ bits) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicOr(&bits[ids[i] >> 5], 1u << (ids[i] & 31));
}

__global__ void clear_bits(const uint32_t* __restrict__ ids, uint64_t n,
                           uint32_t* __restrict__ bits) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) bits[ids[i] >> 5] = 0;
}

// K3: flat, coalesced pass over the item range of the walks.
__global__ void item_histogram(WalkView v, uint64_t p0, uint64_t p1,
                               const uint32_t* __restrict__ cand_bits, uint32_t* __restrict__ cnt) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = p0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += stride) {
        uint32_t item = v.items[p];
        if (item < v.limit && is_cand(cand_bits, item)) atomicAdd(&cnt[item], 1u);
    }
}

// K3 on a plain key array (the radix-partitioned copy of the items, see partitioned_histogram).
__global__ void key_histogram(const uint32_t* __restrict__ keys, uint64_t n, uint32_t limit,
                              const uint32_t* __restrict__ cand_bits, uint32_t* __restrict__ cnt) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        uint32_t item = __ldcs(keys + p);  // read once: must not push the counters out of L2
        if (item < limit && is_cand(cand_bits, item)) atomicAdd(&cnt[item], 1u);
    }
}

// K3 for large id spaces, shared-memory form. Random counter updates in global memory run at
// ~40 G/s on this device whatever the window they fall into (L2 misses when the window is wide,
// same-sector serialisation when it is narrow: measured with 8..20 partition bits). So the keys
// are sorted on their top bits down to windows of 2^wbits ids (<= 128 KB of counters), one CTA
// takes a window, counts its keys with shared-memory atomics and adds the window to the global
// array with plain coalesced read-modify-writes (it is the only writer of that range).
// starts[b] = first position of window b's keys in the sorted slice (starts[nbuckets] = end of the
// in-range keys). Four keys per thread (128-bit loads), the left neighbour comes by shuffle.
__global__ void __launch_bounds__(256) bucket_starts(const uint32_t* __restrict__ keys, uint64_t n,
                                                     uint32_t wbits, uint32_t nbuckets,
                                                     uint64_t* __restrict__ starts) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // quad index
    const uint64_t i0 = q * 4;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t b[4] = {nbuckets, nbuckets, nbuckets, nbuckets};
    if (i0 + 3 < n) {
        const uint4 k4 = __ldcs(reinterpret_cast<const uint4*>(keys) + q);
        b[0] = min(k4.x >> wbits, nbuckets);  // ids >= limit: past the last window
        b[1] = min(k4.y >> wbits, nbuckets);
        b[2] = min(k4.z >> wbits, nbuckets);
        b[3] = min(k4.w >> wbits, nbuckets);
    } else {
        for (int j = 0; j < 4; ++j)
            if (i0 + j < n) b[j] = min(keys[i0 + j] >> wbits, nbuckets);
    }
    uint32_t left = __shfl_up_sync(kFullMask, b[3], 1);
    if (i0 >= n) return;
    if (lane == 0 && i0 > 0) left = min(keys[i0 - 1] >> wbits, nbuckets);
    for (int j = 0; j < 4 && i0 + j < n; ++j) {
        const uint64_t i = i0 + j;
        const uint32_t prev = j ? b[j - 1] : left;
        for (uint32_t x = i ? prev + 1 : 0u; x <= b[j]; ++x) starts[x] = i;
        if (i == n - 1)
            for (uint32_t x = b[j] + 1; x <= nbuckets; ++x) starts[x] = n;
    }
}

// One CTA per window: zero, count (eight key loads in flight per thread), then add the window to
// the global counters with all of a thread's 32 read-modify-writes issued together (the loads of
// the non-zero slots first, then the stores) instead of one dependent round trip per slot.
__global__ void __launch_bounds__(1024) window_histogram(const uint32_t* __restrict__ keys,
                                                         const uint64_t* __restrict__ starts,
                                                         uint32_t wbits, uint32_t limit,
                                                         const uint32_t* __restrict__ cand_bits,
                                                         uint32_t* __restrict__ cnt) {
    extern __shared__ uint32_t win[];
    const uint32_t W = 1u << wbits;
    const uint64_t a = starts[blockIdx.x], b = starts[blockIdx.x + 1];
    if (a == b) return;
    for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) win[i] = 0;
    __syncthreads();
    uint64_t p = a + threadIdx.x;
    for (; p + 7 * 1024ull < b; p += 8 * 1024ull) {
        uint32_t k[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) k[j] = __ldcs(keys + p + j * 1024ull);
#pragma unroll
        for (int j = 0; j < 8; ++j) atomicAdd(&win[k[j] & (W - 1)], 1u);
    }
    for (; p < b; p += 1024) atomicAdd(&win[__ldcs(keys + p) & (W - 1)], 1u);
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x << wbits;
    for (uint32_t i0 = threadIdx.x; i0 < W; i0 += 8 * 1024) {
        uint32_t c[8], g[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t i = i0 + j * 1024;
            const uint64_t id = base + i;
            c[j] = i < W ? win[i] : 0u;
            if (c[j] && (id >= limit || !is_cand(cand_bits, (uint32_t)id))) c[j] = 0;
            g[j] = c[j] ? cnt[id] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (c[j]) cnt[base + i0 + j * 1024] = g[j] + c[j];
    }
}

// K3b: one warp per walk; slot order inside an item's list is irrelevant (set semantics).
// One bit per item: is it indexed (candidate with count >= min_count)? The bitmap (limit / 8
// bytes) stays in L2, so the scatter pass needs no random HBM read per item to find that out.
__global__ void mark_indexed(const uint32_t* __restrict__ cnt, uint32_t limit, uint32_t min_count,
                             uint32_t* __restrict__ bits, uint32_t* __restrict__ filter,
                             uint32_t filter_log2) {
    uint64_t word = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t base = word * 32;
    if (base >= limit) return;
    uint32_t w = 0;
#pragma unroll 8
    for (uint32_t j = 0; j < 32; ++j) {
        uint64_t id = base + j;
        // count > 0 already implies "candidate": the histogram only counts candidates
        if (id < limit && cnt[id] >= min_count && cnt[id] != 0) {
            w |= 1u << j;
            if (filter_log2) {
                const uint32_t h = filter_slot((uint32_t)id, filter_log2);
                atomicOr(&filter[h >> 5], 1u << (h & 31));
            }
        }
    }
    bits[word] = w;
}

__global__ void scatter_inverted(WalkView v, const uint32_t* __restrict__ indexed_bits,
                                 BitFilter filter, const uint64_t* __restrict__ pos,
                                 uint32_t* __restrict__ fill, uint32_t* __restrict__ inv) {
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < v.cnt; i += nwarps) {
        uint64_t w = v.w0 + i;
        uint64_t b, e;
        walk_extent(v, w, b, e);
        for (uint64_t p = b + lane; p < e; p += 32) {
            uint32_t item = v.items[p];
            // only items that can still win a round are indexed (min_count, see hsaw_gpu_greedy);
            // a dense reduced instance holds nothing else (indexed_bits == nullptr)
            if (item < v.limit && (indexed_bits == nullptr ||
                                   (filter_pass(filter, item) &&
                                    ((indexed_bits[item >> 5] >> (item & 31)) & 1u)))) {
                uint32_t slot = atomicAdd(&fill[item], 1u);
                inv[pos[item] + slot] = (uint32_t)i;
            }
        }
    }
}

// Occurrences per count value (counts >= kCountBins - 1 share the last bin): lets the host pick the
// smallest count worth indexing. occ_bins[c] += c * (#items with count c).
// A streaming pass over the counters (5.9 GB at the Twitter shape, where the mean count is ~7): the
// bins are per-warp 32-bit ITEM counters in shared memory (native atomics whose conflicts stay
// inside one warp), multiplied out once per block; 128-bit loads. The first version hammered one
// 64-bit shared-memory bin per count with CAS loops: 1.2 TB/s.
constexpr uint32_t kCountBins = 1024;
constexpr uint32_t kCocWarps = 8;
__global__ void __launch_bounds__(kCocWarps * 32) count_of_counts(const uint32_t* __restrict__ cnt,
                                                                   uint32_t limit,
                                                                   unsigned long long* __restrict__ occ_bins) {
    __shared__ uint32_t bins[kCocWarps][kCountBins];
    __shared__ unsigned long long big;  // sum of the counts >= kCountBins - 1 (rare)
    for (uint32_t i = threadIdx.x; i < kCocWarps * kCountBins; i += blockDim.x) (&bins[0][0])[i] = 0;
    if (threadIdx.x == 0) big = 0;
    __syncthreads();
    uint32_t* mine = bins[threadIdx.x >> 5];
    auto add = [&](uint32_t c) {
        if (c == 0) return;
        if (c < kCountBins - 1)
            atomicAdd(&mine[c], 1u);
        else
            atomicAdd(&big, (unsigned long long)c);
    };
    // 128-bit loads over the 16-byte aligned middle (pool allocations are aligned; a caller's
    // device pointer need not be), scalar loads for the few counters before and after it
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t head = min((uint64_t)((16u - (reinterpret_cast<uintptr_t>(cnt) & 15u)) & 15u) / 4,
                              (uint64_t)limit);
    const uint64_t quads = (limit - head) / 4;
    const uint4* cnt4 = reinterpret_cast<const uint4*>(cnt + head);
    for (uint64_t i = tid; i < quads; i += stride) {
        const uint4 c = __ldcs(cnt4 + i);
        add(c.x);
        add(c.y);
        add(c.z);
        add(c.w);
    }
    if (tid < head) add(cnt[tid]);
    const uint64_t tail0 = head + quads * 4;
    if (tid < limit - tail0) add(cnt[tail0 + tid]);
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < kCountBins - 1; c += blockDim.x) {
        unsigned long long n = 0;
#pragma unroll
        for (uint32_t w = 0; w < kCocWarps; ++w) n += bins[w][c];
        if (n) atomicAdd(&occ_bins[c], n * c);
    }
    if (threadIdx.x == 0 && big) atomicAdd(&occ_bins[kCountBins - 1], big);
}

// pos input: counts below the threshold take no inverted-list space
__global__ void threshold_counts(const uint32_t* __restrict__ cnt, uint64_t n, uint32_t min_count,
                                 uint32_t* __restrict__ out) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = cnt[i] >= min_count ? cnt[i] : 0;
}

// ---- dense reduced instance of a large id space ---------------------------------------------------
// With 1.47 G edge ids (Twitter shape) every per-item array of the greedy run is 6..12 GB and every
// access to it a DRAM round trip: the histogram, the inverted-list scatter (one bitmap line, one
// fill counter and one list slot per indexed occurrence), and each of the ~130 count decrements per
// covered walk in the rounds. Only the items at or above the indexing threshold can be selected
// (see hsaw_gpu_greedy), a few per cent of the ids. build_dense renames them 0..D-1 in id order
// (so the smallest-id tie-break is unchanged) and copies the walks restricted to them, in one
// streaming pass, into a (start, length) view whose items are the new names: everything after it
// (pos / fill / counts / block maxima / the rounds) works on D-sized arrays that live in L2 and on
// walks an eighth as long. Gains, selections and the "winner below the threshold" protocol are
// those of the full instance: the reduced walks hold every occurrence of every indexed item.

// Word-blocked two-bit Bloom filter in front of the rank map (367 MB at the Twitter shape: one DRAM
// line per lookup): a clear bit proves "not indexed" from a table that stays cached.
struct Bloom2 {
    const uint32_t* words;
    uint32_t log2w;  // table size in 32-bit words = 2^log2w
};
__device__ __forceinline__ void bloom2_slot(uint32_t item, uint32_t log2w, uint32_t& word, uint32_t& mask) {
    word = (item * 0x9E3779B1u) >> (32 - log2w);
    const uint32_t h2 = item * 0x85EBCA6Bu;
    mask = (1u << (h2 >> 27)) | (1u << ((h2 >> 22) & 31u));
}
__device__ __forceinline__ bool bloom2_pass(const Bloom2& f, uint32_t item) {
    uint32_t word, mask;
    bloom2_slot(item, f.log2w, word, mask);
    return (__ldg(f.words + word) & mask) == mask;
}

// One warp per 32 words (1024 ids): coalesced count reads, the ballot of "indexed" IS the word.
__global__ void __launch_bounds__(256) dense_mark(const uint32_t* __restrict__ cnt, uint32_t limit,
                                                  uint32_t min_count, uint32_t* __restrict__ bits,
                                                  uint32_t* __restrict__ pc, uint32_t* __restrict__ bloom,
                                                  uint32_t log2w) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t words = ((uint64_t)limit + 31) / 32;
    const uint64_t w0 = warp * 32;
    if (w0 >= words) return;
    uint32_t my = 0;
#pragma unroll 4
    for (uint32_t j = 0; j < 32; ++j) {
        const uint64_t id = (w0 + j) * 32 + lane;
        const uint32_t c = id < limit ? cnt[id] : 0u;
        const bool in = c != 0 && c >= min_count;
        const uint32_t m = __ballot_sync(kFullMask, in);
        if (lane == j) my = m;
        if (in) {
            uint32_t word, mask;
            bloom2_slot((uint32_t)id, log2w, word, mask);
            atomicOr(&bloom[word], mask);
        }
    }
    if (w0 + lane < words) {
        bits[w0 + lane] = my;
        pc[w0 + lane] = __popc(my);
    }
}

// rmap[word] = (indexed bits of the word, rank of its first indexed id); ids / counts by rank.
__global__ void __launch_bounds__(256) dense_emit(const uint32_t* __restrict__ cnt, uint32_t limit,
                                                  const uint32_t* __restrict__ bits,
                                                  const uint32_t* __restrict__ base,
                                                  uint2* __restrict__ rmap, uint32_t* __restrict__ rids,
                                                  uint32_t* __restrict__ rcnt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t words = ((uint64_t)limit + 31) / 32;
    const uint64_t w0 = warp * 32;
    if (w0 >= words) return;
    uint32_t my_bits = 0, my_base = 0;
    if (w0 + lane < words) {
        my_bits = bits[w0 + lane];
        my_base = base[w0 + lane];
        rmap[w0 + lane] = make_uint2(my_bits, my_base);
    }
    uint32_t any = __ballot_sync(kFullMask, my_bits != 0);
    while (any) {
        const int j = __ffs(any) - 1;
        any &= any - 1;
        const uint32_t b = __shfl_sync(kFullMask, my_bits, j);
        const uint32_t r0 = __shfl_sync(kFullMask, my_base, j);
        if ((b >> lane) & 1u) {
            const uint32_t id = (uint32_t)((w0 + j) * 32 + lane);
            const uint32_t r = r0 + __popc(b & ((1u << lane) - 1u));
            rids[r] = id;
            rcnt[r] = cnt[id];
        }
    }
}

// (Measured and dropped: the filter copied to shared memory - 64 KB copies changed nothing, 128 KB
// ones leave one block per SM: 42 -> 51 ms per C4 solve - and 128-bit item loads with one vote per
// four items: 42 -> 55 ms. At the largest R_t the pass runs at 1.9 TB/s with 67 % of the issue
// slots busy: per-item filter arithmetic, not memory.)
// The walks' indexed items as (walk, new name) pairs: a flat, coalesced pass over the item range
// (the walk structure does not matter to a membership test); only for the few items that pass the
// filter and the map is the owning walk looked up (binary search over the extents) and the pair
// appended through a warp-aggregated cursor. The first version went walk by walk (one warp per
// walk, block-wide allocation): 0.6 TB/s on the 39 GB of the largest R_t.
__global__ void __launch_bounds__(256) dense_pairs(WalkView v, uint64_t p0, uint64_t p1, Bloom2 bloom,
                                                   const uint2* __restrict__ rmap,
                                                   unsigned long long* __restrict__ cursor,
                                                   uint32_t* __restrict__ pair_walk,
                                                   uint32_t* __restrict__ pair_rank) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int kInFlight = 4;
    // (the loop bound is warp-uniform: the ballots below need all 32 lanes)
    for (uint64_t wbase = p0 + (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wbase < p1;
         wbase += kInFlight * stride) {
        const uint64_t base = wbase + lane;
        uint32_t it[kInFlight];
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) {
            const uint64_t p = base + j * stride;
            it[j] = p < p1 ? __ldcs(v.items + p) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) {
            const uint64_t p = base + j * stride;
            uint32_t rank = 0;
            bool keep = it[j] < v.limit && bloom2_pass(bloom, it[j]);
            if (keep) {
                const uint2 m = __ldg(rmap + (it[j] >> 5));
                keep = (m.x >> (it[j] & 31)) & 1u;
                rank = m.y + __popc(m.x & ((1u << (it[j] & 31)) - 1u));
            }
            const uint32_t mask = __ballot_sync(kFullMask, keep);
            if (!mask) continue;
            uint64_t wi = 0;
            if (keep) {  // largest walk index whose first item position is <= p
                uint64_t lo = 0, hi = v.cnt - 1;
                while (lo < hi) {
                    const uint64_t mid = lo + (hi - lo + 1) / 2;
                    const uint64_t w = v.w0 + mid;
                    if (v.off[w] + v.add * w <= p)
                        lo = mid;
                    else
                        hi = mid - 1;
                }
                wi = lo;
            }
            unsigned long long at = 0;
            const int leader = __ffs(mask) - 1;
            if ((int)lane == leader) at = atomicAdd(cursor, (unsigned long long)__popc(mask));
            at = __shfl_sync(kFullMask, at, leader) + __popc(mask & ((1u << lane) - 1u));
            if (keep) {
                pair_walk[at] = (uint32_t)wi;
                pair_rank[at] = rank;
            }
        }
    }
}

// pairs sorted by walk -> heads of the runs (flag[n] = 0 closes the scan) and the run starts
__global__ void pair_heads(const uint32_t* __restrict__ sw, uint64_t n, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= n) flag[i] = i < n && (i == 0 || sw[i] != sw[i - 1]) ? 1u : 0u;
}
__global__ void pair_starts(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ widx,
                            uint64_t n, uint64_t* __restrict__ start) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) start[widx[i]] = i;
    if (i == n) start[widx[n]] = n;
}

// solution slots hold ranks of the dense instance: back to ids (markers pass through)
__global__ void dense_solution_ids(uint32_t* __restrict__ sol, uint32_t n, uint32_t limit,
                                   const uint32_t* __restrict__ rids) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && sol[i] < limit) sol[i] = rids[sol[i]];
}

__device__ __forceinline__ uint64_t block_max_u64(uint64_t v, uint64_t* smem) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t other = __shfl_xor_sync(kFullMask, v, o);
        v = other > v ? other : v;
    }
    uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    uint32_t nw = blockDim.x >> 5;
    v = threadIdx.x < nw ? smem[threadIdx.x] : 0;
    if (wid == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t other = __shfl_xor_sync(kFullMask, v, o);
            v = other > v ? other : v;
        }
        if (lane == 0) smem[0] = v;
    }
    __syncthreads();
    v = smem[0];
    __syncthreads();
    return v;
}

// ---- lazy block maxima (CELF at block granularity) ---------------------------------------------
// Counts only ever decrease during a greedy run, so a block maximum computed earlier is an upper
// bound of the block's true maximum. Each round re-tightens only the block holding the largest
// bound until that bound is exact — then it is the global argmax — instead of scanning all
// `limit` counters (16 M for C2 edges, 1.47 G at the Twitter shape) every round. Keys are
// count << 32 | ~id, unique per item, so the (largest gain, smallest id) order is preserved.
// Block size: 2^bshift items, at least 2048, and large enough for the bounds of all blocks to fit
// the tail kernel's shared memory (1.47 G edge ids at the Twitter shape -> 65536-item blocks,
// 22 k bounds; a grid-wide round over 717 k 2048-item blocks cost 0.33 ms there).
constexpr uint32_t kMinBlockShift = 11;
constexpr uint32_t kTailMaxBlocks = 24000;  // x 8 bytes + exact bits <= 200 KB of shared memory
inline uint32_t block_shift_for(uint64_t limit) {
    uint32_t sh = kMinBlockShift;
    if (const char* env = std::getenv("HSAW_GREEDY_BLOCK_SHIFT")) {  // test hook: force large blocks
        const int v = std::atoi(env);
        if (v >= (int)kMinBlockShift && v <= 20) sh = (uint32_t)v;
    }
    while (((limit + (1ull << sh) - 1) >> sh) > kTailMaxBlocks && sh < 31) ++sh;
    return sh;
}
constexpr uint32_t kUnindexed = 0xFFFFFFFEu;  // round marker: winner below the index threshold

__device__ __forceinline__ uint64_t gain_key(uint32_t count, uint32_t id) {
    return count ? ((uint64_t)count << 32) | (0xFFFFFFFFu - id) : 0;
}

// blkmax[b] = exact max key of items [b * 2048, (b + 1) * 2048)
__global__ void __launch_bounds__(256) block_maxima(const uint32_t* __restrict__ cnt,
                                                    uint32_t limit, uint64_t* __restrict__ blkmax,
                                                    uint32_t bshift) {
    __shared__ uint64_t smem[32];
    const uint32_t kMaxBlockItems = 1u << bshift;
    const uint64_t base = (uint64_t)blockIdx.x * kMaxBlockItems;
    uint64_t best = 0;
    for (uint32_t i = threadIdx.x; i < kMaxBlockItems; i += blockDim.x) {
        uint64_t id = base + i;
        if (id < limit) {
            uint64_t k = gain_key(cnt[id], (uint32_t)id);
            best = k > best ? k : best;
        }
    }
    best = block_max_u64(best, smem);
    if (threadIdx.x == 0) blkmax[blockIdx.x] = best;
}

// One CTA: repeat { take the block with the largest bound; recompute it exactly } until the
// largest bound is exact. Writes the winner key to out[0] (0 = no positive gain left).
__global__ void __launch_bounds__(1024) select_lazy(const uint32_t* __restrict__ cnt,
                                                    uint32_t limit, uint64_t* __restrict__ blkmax,
                                                    uint32_t nblk, uint64_t* __restrict__ out,
                                                    uint32_t bshift) {
    __shared__ uint64_t smem[32];
    __shared__ uint32_t s_blk;
    const uint32_t kMaxBlockItems = 1u << bshift;
    // The block of the previous round's winner holds the stalest bound there is (the winner's own
    // key, now covered): tighten it up front instead of spending a whole scan to find that out.
    // (Whatever out[0] holds, recomputing a valid block's maximum exactly is always sound.)
    const uint64_t prev = out[0];
    const uint32_t hint = (0xFFFFFFFFu - (uint32_t)prev) / kMaxBlockItems;
    if (prev != 0 && hint < nblk) {
        const uint32_t blk = hint;
        const uint64_t base = (uint64_t)blk * kMaxBlockItems;
        uint64_t exact = 0;
        for (uint32_t i = threadIdx.x; i < kMaxBlockItems; i += blockDim.x) {
            uint64_t id = base + i;
            if (id < limit) {
                uint64_t k = gain_key(cnt[id], (uint32_t)id);
                exact = k > exact ? k : exact;
            }
        }
        exact = block_max_u64(exact, smem);
        if (threadIdx.x == 0) blkmax[blk] = exact;
        __syncthreads();
    }
    for (;;) {
        uint64_t best = 0;
        uint32_t best_b = 0;
        for (uint32_t b = threadIdx.x; b < nblk; b += blockDim.x) {
            uint64_t k = blkmax[b];
            if (k > best) {
                best = k;
                best_b = b;
            }
        }
        const uint64_t top = block_max_u64(best, smem);
        if (top == 0) {
            if (threadIdx.x == 0) out[0] = 0;
            return;
        }
        if (best == top) s_blk = best_b;  // keys are unique: exactly one thread holds the top
        __syncthreads();
        const uint32_t blk = s_blk;
        const uint64_t base = (uint64_t)blk * kMaxBlockItems;
        uint64_t exact = 0;
        for (uint32_t i = threadIdx.x; i < kMaxBlockItems; i += blockDim.x) {
            uint64_t id = base + i;
            if (id < limit) {
                uint64_t k = gain_key(cnt[id], (uint32_t)id);
                exact = k > exact ? k : exact;
            }
        }
        exact = block_max_u64(exact, smem);
        if (exact == top) {  // the bound was exact: every other block is bounded below it
            if (threadIdx.x == 0) out[0] = top;
            return;
        }
        if (threadIdx.x == 0) blkmax[blk] = exact;  // tighten and look again
        __syncthreads();
    }
}

// K5: every block re-reduces the partial maxima (identical result), then the blocks share the
// winner's inverted list: one warp per listed walk, claimed through an atomicOr on the covered
// bitmap, decrementing the counts of the walk's candidate items.
__global__ void __launch_bounds__(256) cover_winner(WalkView v, const uint64_t* __restrict__ partial,
                                                    uint32_t npartial,
                                                    const uint32_t* __restrict__ cand_bits,
                                                    const uint64_t* __restrict__ pos,
                                                    const uint32_t* __restrict__ inv,
                                                    uint32_t* __restrict__ cnt,
                                                    uint32_t* __restrict__ covered,
                                                    uint32_t round, uint32_t* __restrict__ solution,
                                                    uint64_t* __restrict__ gains,
                                                    uint32_t min_indexed) {
    __shared__ uint64_t smem[32];
    uint64_t best = 0;
    for (uint32_t i = threadIdx.x; i < npartial; i += blockDim.x) {
        uint64_t k = partial[i];
        best = k > best ? k : best;
    }
    best = block_max_u64(best, smem);
    uint32_t gain = (uint32_t)(best >> 32);
    uint32_t item = 0xFFFFFFFFu - (uint32_t)best;
    // A winner below the indexing threshold has no inverted list: report it (kUnindexed) and
    // stop; the host rebuilds the full index. Items above the threshold are always indexed
    // because counts only decrease.
    const bool unindexed = gain != 0 && gain < min_indexed;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        solution[round] = unindexed ? kUnindexed : (gain ? item : 0xFFFFFFFFu);
        gains[round] = gain;
    }
    if (gain == 0 || unindexed) return;
    uint64_t lb = pos[item], le = pos[item + 1];
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = lb + warp; i < le; i += nwarps) {
        uint32_t lw = inv[i];
        uint32_t old = 0;
        if (lane == 0) old = atomicOr(&covered[lw >> 5], 1u << (lw & 31));
        old = __shfl_sync(kFullMask, old, 0);
        if (old & (1u << (lw & 31))) continue;  // already covered (earlier round or duplicate item)
        uint64_t w = v.w0 + lw;
        uint64_t b, e;
        walk_extent(v, w, b, e);
        for (uint64_t p = b + lane; p < e; p += 32) {
            uint32_t it = v.items[p];
            if (it < v.limit && is_cand(cand_bits, it)) atomicSub(&cnt[it], 1u);
        }
    }
}

// ---- the tail of a greedy run in one CTA ---------------------------------------------------------
// Selected gains never increase from one round to the next (submodularity), and once the winner's
// inverted list is a few thousand walks a whole grid is wasted on it: a round is then ~15 us of
// launch and reduction latency around ~1 us of work. This kernel runs rounds [first, k) back to
// back in ONE block of 1024 threads: the lazy block maxima live in shared memory (nblk * 8 bytes),
// selection is select_lazy's, the cover is cover_winner's with the block's 32 warps, and nothing
// leaves the SM between rounds except the count atomics (read back with ld.global.cg).
// It stops — reporting how many rounds it completed in done_out — at a zero gain, at a winner
// below the indexing threshold, or at a winner whose list is longer than max_list (the host then
// runs that round with the grid-wide kernels and comes back).
__global__ void __launch_bounds__(1024) greedy_tail_kernel(
    WalkView v, const uint32_t* __restrict__ cand_bits, const uint64_t* __restrict__ pos,
    const uint32_t* __restrict__ inv, uint32_t* cnt, uint32_t* covered, uint64_t* blkmax,
    uint32_t nblk, uint32_t first, uint32_t k, uint32_t* __restrict__ solution,
    uint64_t* __restrict__ gains, uint32_t min_indexed, uint32_t max_list,
    uint32_t* __restrict__ done_out, int bounds_exact, uint32_t bshift) {
    const uint32_t kMaxBlockItems = 1u << bshift;
    // s_max[b]: upper bound of block b's maximum key; s_exact bit b: the bound IS the maximum.
    // A bound is made exact by recomputing the block and stays exact until the item that attains
    // it is decremented (decrements of other items cannot change a maximum), which the cover
    // phase detects by comparing ids — so a block that surfaces as the top again usually needs no
    // recomputation at all.
    extern __shared__ uint64_t s_max[];
    uint32_t* s_exact = reinterpret_cast<uint32_t*>(s_max + nblk);
    __shared__ uint64_t smem[32];
    __shared__ uint32_t s_blk;
    const uint32_t limit = v.limit;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (uint32_t b = threadIdx.x; b < nblk; b += blockDim.x) s_max[b] = blkmax[b];
    // bounds_exact: blkmax comes straight from block_maxima (no grid-wide round has decremented
    // anything since), so every bound already is its block's maximum
    for (uint32_t b = threadIdx.x; b < (nblk + 31) / 32; b += blockDim.x)
        s_exact[b] = bounds_exact ? 0xFFFFFFFFu : 0u;
    __syncthreads();
    uint32_t r = first;
    for (; r < k; ++r) {
        // ---- selection: the block holding the largest bound, tightened until that bound is exact
        uint64_t top;
        for (;;) {
            uint64_t best = 0;
            uint32_t best_b = 0;
            for (uint32_t b = threadIdx.x; b < nblk; b += blockDim.x) {
                uint64_t key = s_max[b];
                if (key > best) {
                    best = key;
                    best_b = b;
                }
            }
            top = block_max_u64(best, smem);
            if (top == 0) break;
            if (best == top) s_blk = best_b;  // keys are unique
            __syncthreads();
            const uint32_t blk = s_blk;
            if ((s_exact[blk >> 5] >> (blk & 31)) & 1u) break;  // known exact: the global argmax
            const uint64_t base = (uint64_t)blk * kMaxBlockItems;
            uint64_t exact = 0;
            for (uint32_t i = threadIdx.x; i < kMaxBlockItems; i += blockDim.x) {
                uint64_t id = base + i;
                if (id < limit) {
                    uint64_t key = gain_key(__ldcg(cnt + id), (uint32_t)id);
                    exact = key > exact ? key : exact;
                }
            }
            exact = block_max_u64(exact, smem);
            if (threadIdx.x == 0) {
                s_max[blk] = exact;
                s_exact[blk >> 5] |= 1u << (blk & 31);
            }
            __syncthreads();
            if (exact == top) break;
        }
        // Every thread must have taken its exit from the selection loop (which reads s_exact)
        // before any warp starts covering (which clears s_exact bits): without this barrier a slow
        // warp could see the top block's bit already cleared by a fast one and go on recomputing
        // alone - found by compute-sanitizer racecheck as barrier-mismatch hazards.
        __syncthreads();
        const uint32_t gain = (uint32_t)(top >> 32);
        const uint32_t item = 0xFFFFFFFFu - (uint32_t)top;
        const bool unindexed = gain != 0 && gain < min_indexed;
        uint64_t lb = 0, le = 0;
        if (gain != 0 && !unindexed) {
            lb = pos[item];
            le = pos[item + 1];
        }
        const bool too_long = le - lb > max_list;
        if (gain == 0 || unindexed) {  // report the round like cover_winner does, then stop
            if (threadIdx.x == 0) {
                solution[r] = unindexed ? kUnindexed : 0xFFFFFFFFu;
                gains[r] = gain;
            }
            ++r;
            break;
        }
        if (too_long) break;  // round r is left to the grid-wide kernels
        if (threadIdx.x == 0) {
            solution[r] = item;
            gains[r] = gain;
        }
        // ---- cover: the block's warps share the winner's inverted list, one walk per warp at a
        // time (lane-parallel claiming and a shared-memory queue of claimed walks were both
        // measured slower: the round is a chain of ~7 dependent memory round trips either way)
        // two walks per warp and iteration: their list entries, claims (lanes 0 and 1), extents
        // and items are fetched side by side, so each trip of the dependent chain
        // inv -> {claim, extent} -> items serves two walks. A walk listed twice (an item that
        // occurs twice in it) is claimed by exactly one of the two atomics, as before.
        for (uint64_t i = lb + warp; i < le; i += 2 * nwarps) {
            const uint64_t i2 = i + nwarps;
            const bool has2 = i2 < le;
            const uint32_t lw1 = inv[i];
            const uint32_t lw2 = has2 ? inv[i2] : 0u;
            uint32_t old = 0;
            if (lane == 0) old = atomicOr(&covered[lw1 >> 5], 1u << (lw1 & 31));
            if (lane == 1 && has2) old = atomicOr(&covered[lw2 >> 5], 1u << (lw2 & 31));
            // the extents are fetched while the claims are in flight: one round trip less on the
            // round's dependent chain (a claim that fails wastes two loads)
            const uint64_t w1 = v.w0 + lw1, w2 = v.w0 + lw2;
            uint64_t b1, e1, b2 = 0, e2 = 0;
            walk_extent(v, w1, b1, e1);
            if (has2) walk_extent(v, w2, b2, e2);
            const uint32_t old1 = __shfl_sync(kFullMask, old, 0);
            const uint32_t old2 = __shfl_sync(kFullMask, old, 1);
            const uint64_t len1 = (old1 & (1u << (lw1 & 31))) ? 0 : e1 - b1;  // 0: already covered
            const uint64_t len2 = (!has2 || (old2 & (1u << (lw2 & 31)))) ? 0 : e2 - b2;
            const uint64_t longest = len1 > len2 ? len1 : len2;
            for (uint64_t q = lane; q < longest; q += 32) {
                uint32_t it1 = 0xFFFFFFFFu, it2 = 0xFFFFFFFFu;
                if (q < len1) it1 = v.items[b1 + q];
                if (q < len2) it2 = v.items[b2 + q];
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const uint32_t it = s2 ? it2 : it1;
                    if (it < limit && is_cand(cand_bits, it)) {
                        atomicSub(&cnt[it], 1u);
                        const uint32_t blk = it / kMaxBlockItems;
                        if ((uint32_t)s_max[blk] == 0xFFFFFFFFu - it)  // the item attaining the bound
                            atomicAnd(&s_exact[blk >> 5], ~(1u << (blk & 31)));
                    }
                }
            }
        }
        // One CTA owns the counts for the whole launch: the barrier alone orders this round's
        // count atomics before the next round's ld.global.cg reads (CTA-scope visibility is all
        // that is needed; a device-scope fence here cost a full round trip and an L1 flush per
        // round). The kernel boundary publishes everything to the grid-wide kernels.
        __syncthreads();
        // The winner's count just dropped, so its block's bound is stale by construction and - being
        // the largest key of the last round - would surface first in the next selection only to
        // be recomputed there and make that selection start over. Tighten it now instead.
        {
            const uint32_t wb = item / kMaxBlockItems;
            const uint64_t base = (uint64_t)wb * kMaxBlockItems;
            uint64_t exact = 0;
            for (uint32_t i = threadIdx.x; i < kMaxBlockItems; i += blockDim.x) {
                uint64_t id = base + i;
                if (id < limit) {
                    uint64_t key = gain_key(__ldcg(cnt + id), (uint32_t)id);
                    exact = key > exact ? key : exact;
                }
            }
            exact = block_max_u64(exact, smem);
            if (threadIdx.x == 0) {
                s_max[wb] = exact;
                s_exact[wb >> 5] |= 1u << (wb & 31);
            }
            __syncthreads();
        }
    }
    // hand the bounds back to the grid-wide kernels and report progress
    for (uint32_t b = threadIdx.x; b < nblk; b += blockDim.x) blkmax[b] = s_max[b];
    if (threadIdx.x == 0) *done_out = r;
}

// K6: one warp per walk; a walk counts once if any of its items is in the query bitmap.
__global__ void __launch_bounds__(256) count_covered(WalkView v,
                                                     const uint32_t* __restrict__ query_bits,
                                                     BitFilter filter,
                                                     unsigned long long* __restrict__ out) {
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t mine = 0;
    for (uint64_t i = warp; i < v.cnt; i += nwarps) {
        uint64_t w = v.w0 + i;
        uint64_t b = v.off[w] + v.add * w, e = v.off[w + 1] + v.add * (w + 1);
        bool hit = false;
        for (uint64_t p = b + lane; p < e && !hit; p += 32) {
            uint32_t it = v.items[p];
            hit = it < v.limit && filter_pass(filter, it) &&
                  ((query_bits[it >> 5] >> (it & 31)) & 1u);
        }
        if (__any_sync(kFullMask, hit) && lane == 0) ++mine;
    }
    if (lane == 0 && mine) atomicAdd(out, (unsigned long long)mine);
}

// K6, flat form: a coalesced pass over the item range; the walk of an item only matters for the
// few items that are in the query set (binary search over the extents, then one bit per walk so
// that a walk counts once). The walk-by-walk form above streams at ~1.9 TB/s on 130-item walks.
__global__ void __launch_bounds__(256) count_covered_flat(WalkView v, uint64_t p0, uint64_t p1,
                                                          const uint32_t* __restrict__ query_bits,
                                                          BitFilter filter,
                                                          uint32_t* __restrict__ walk_bits,
                                                          unsigned long long* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int kInFlight = 4;
    uint32_t mine = 0;
    for (uint64_t base = p0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < p1;
         base += kInFlight * stride) {
        uint32_t it[kInFlight];
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) {
            const uint64_t p = base + j * stride;
            it[j] = p < p1 ? __ldcs(v.items + p) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) {
            if (!(it[j] < v.limit && filter_pass(filter, it[j]) &&
                  ((query_bits[it[j] >> 5] >> (it[j] & 31)) & 1u)))
                continue;
            const uint64_t p = base + j * stride;
            uint64_t lo = 0, hi = v.cnt - 1;  // largest walk index whose first item is at or before p
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo + 1) / 2;
                const uint64_t w = v.w0 + mid;
                if (v.off[w] + v.add * w <= p)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const uint32_t bit = 1u << (lo & 31);
            if (!(atomicOr(&walk_bits[lo >> 5], bit) & bit)) ++mine;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFullMask, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, (unsigned long long)mine);
}

// ---- stepwise session (sharded solves): the same round split into host-visible steps -----------
// select_final: reduce the partial maxima to the winner (item, gain) for the host.
__global__ void __launch_bounds__(256) select_final(const uint64_t* __restrict__ partial,
                                                    uint32_t npartial, uint64_t* __restrict__ out) {
    __shared__ uint64_t smem[32];
    uint64_t best = 0;
    for (uint32_t i = threadIdx.x; i < npartial; i += blockDim.x) {
        uint64_t k = partial[i];
        best = k > best ? k : best;
    }
    best = block_max_u64(best, smem);
    if (threadIdx.x == 0) {
        out[0] = best >> 32;                                 // gain
        out[1] = best ? 0xFFFFFFFFu - (uint32_t)best : 0xFFFFFFFFu;  // item
    }
}

// cover_item: like cover_winner for a host-chosen item, and every decrement is also appended to
// `list` (warp-aggregated) so that peer ranks can replay it on their replica of the counts.
__global__ void __launch_bounds__(256) cover_item(WalkView v, uint32_t item,
                                                  const uint32_t* __restrict__ cand_bits,
                                                  const uint64_t* __restrict__ pos,
                                                  const uint32_t* __restrict__ inv,
                                                  uint32_t* __restrict__ cnt,
                                                  uint32_t* __restrict__ covered,
                                                  uint32_t* __restrict__ list, uint64_t list_cap,
                                                  unsigned long long* __restrict__ list_count) {
    uint64_t lb = pos[item], le = pos[item + 1];
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = lb + warp; i < le; i += nwarps) {
        uint32_t lw = inv[i];
        uint32_t old = 0;
        if (lane == 0) old = atomicOr(&covered[lw >> 5], 1u << (lw & 31));
        old = __shfl_sync(kFullMask, old, 0);
        if (old & (1u << (lw & 31))) continue;
        uint64_t w = v.w0 + lw;
        uint64_t b = v.off[w] + v.add * w, e = v.off[w + 1] + v.add * (w + 1);
        for (uint64_t p0 = b; p0 < e; p0 += 32) {
            uint64_t p = p0 + lane;
            uint32_t it = p < e ? v.items[p] : 0xFFFFFFFFu;
            bool dec = p < e && it < v.limit && is_cand(cand_bits, it);
            if (dec) atomicSub(&cnt[it], 1u);
            unsigned m = __ballot_sync(kFullMask, dec);
            if (m) {
                unsigned long long base = 0;
                if (lane == (uint32_t)(__ffs(m) - 1)) base = atomicAdd(list_count, (unsigned long long)__popc(m));
                base = __shfl_sync(kFullMask, base, __ffs(m) - 1);
                uint64_t slot = base + __popc(m & ((1u << lane) - 1));
                if (dec && slot < list_cap) list[slot] = it;
            }
        }
    }
}

__global__ void apply_decrements(const uint32_t* __restrict__ items, uint64_t n, uint32_t limit,
                                 uint32_t* __restrict__ cnt) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && items[i] < limit) atomicSub(&cnt[items[i]], 1u);
}

WalkView make_view(const hsaw_gpu_stream* s, const hsaw_gpu_walkset* ws, int kind, uint64_t off,
                   uint64_t cnt) {
    if ((s != nullptr) == (ws != nullptr))
        fail(HSAW_EINVAL, "exactly one of stream / walkset must be given");
    WalkView v{};
    if (s) {
        if (kind != HSAW_KIND_EDGE && kind != HSAW_KIND_NODE) fail(HSAW_EINVAL, "unknown item kind");
        if (off + cnt > s->accepted)
            fail(HSAW_ERANGE, "sample stream prefix not materialized");
        if (kind == HSAW_KIND_EDGE ? !s->keep_edges : !s->keep_nodes)
            fail(HSAW_EINVAL, "this stream does not keep the item array of that kind (stream_keep)");
        v.off = s->edge_off.p;
        v.items = kind == HSAW_KIND_EDGE ? s->edges.p : s->nodes.p;
        v.add = kind == HSAW_KIND_EDGE ? 0u : 1u;
        v.limit = kind == HSAW_KIND_EDGE ? s->ctx->g.m : s->ctx->g.n;
    } else {
        if (off + cnt > ws->nsets) fail(HSAW_ERANGE, "walk set range out of bounds");
        v.off = ws->off.p;
        v.items = ws->items.p;
        v.add = 0;
        v.limit = ws->limit;
    }
    v.w0 = off;
    v.cnt = cnt;
    return v;
}

uint64_t read_u64(hsaw_gpu_ctx* ctx, const uint64_t* d) {
    HSAW_CUDA_CHECK(cudaMemcpyAsync(ctx->h_scalars, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return ctx->h_scalars[0];
}
uint32_t read_u32(hsaw_gpu_ctx* ctx, const uint32_t* d) {
    HSAW_CUDA_CHECK(cudaMemcpyAsync(ctx->h_scalars, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return *reinterpret_cast<uint32_t*>(ctx->h_scalars);
}

// first/last item position of the view (two 8-byte reads)
void view_span(hsaw_gpu_ctx* ctx, const WalkView& v, uint64_t* p0, uint64_t* p1) {
    uint64_t a = 0, b = 0;
    HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[0], v.off + v.w0, 8, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[1], v.off + v.w0 + v.cnt, 8,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    a = ctx->h_scalars[0];
    b = ctx->h_scalars[1];
    *p0 = a + (uint64_t)v.add * v.w0;
    *p1 = b + (uint64_t)v.add * (v.w0 + v.cnt);
}

// Sorted, de-duplicated candidate ids (host) + device bitmap. Returns the candidate count.
uint64_t prepare_candidates(hsaw_gpu_ctx* ctx, uint32_t limit, const uint32_t* cand_ids,
                            uint64_t ncand, std::vector<uint32_t>& sorted,
                            DevVec<uint32_t>& bits) {
    if (!cand_ids) return limit;  // CandidateSet::all
    sorted.assign(cand_ids, cand_ids + ncand);
    for (uint32_t id : sorted)
        if (id >= limit)  // candidate_mask, proj/src/coverage.cpp:18-20
            fail(HSAW_EDATA, "candidate id out of range: " + std::to_string(id));
    std::sort(sorted.begin(), sorted.end());
    sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
    uint64_t words = ((uint64_t)limit + 31) / 32 + 1;
    bits.ensure_scratch(words);
    HSAW_CUDA_CHECK(cudaMemsetAsync(bits.p, 0, words * 4, ctx->stream));
    if (!sorted.empty()) {
        DevVec<uint32_t> d_ids;
        d_ids.ensure_scratch(sorted.size());
        HSAW_CUDA_CHECK(cudaMemcpyAsync(d_ids.p, sorted.data(), sorted.size() * 4,
                                        cudaMemcpyHostToDevice, ctx->stream));
        set_bits<<<(unsigned)((sorted.size() + 255) / 256), 256, 0, ctx->stream>>>(
            d_ids.p, sorted.size(), bits.p);
        check_launch(ctx, "set_bits");
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    return sorted.size();
}

}  // namespace

// A zeroed filter table for `members` entries of an id space of `limit` items, or {nullptr, 0} when
// the exact bitmap (limit / 8 bytes) is small enough to stay in L2 by itself. Sized for <= ~0.4 %
// false positives, between 64 KB and 32 MB.
static BitFilter prepare_filter(hsaw_gpu_ctx* ctx, uint64_t limit, uint64_t members) {
    if (limit / 8 <= (24ull << 20)) return BitFilter{nullptr, 0};
    uint32_t log2 = 19;
    while ((1ull << log2) < members * 256 && log2 < 28) ++log2;
    const uint64_t words = (1ull << log2) / 32;
    ctx->g_filter.ensure_scratch(words);
    HSAW_CUDA_CHECK(cudaMemsetAsync(ctx->g_filter.p, 0, words * 4, ctx->stream));
    return BitFilter{ctx->g_filter.p, log2};
}

// K3: occurrences of every candidate item in the walks' item range [p0, p1) -> cnt[item] (cnt is
// zeroed by the caller). When the counters do not fit L2, random atomics go to
// HBM one 32-byte sector at a time; one 8-bit radix pass on the items' top bits first
// makes consecutive items fall into one ~1/256 window of the counters, which L2 holds.
static void histogram_counts(hsaw_gpu_ctx* ctx, const WalkView& v, uint64_t p0, uint64_t p1,
                             const uint32_t* d_cand, uint32_t* d_cnt) {
    cudaStream_t st = ctx->stream;
    const uint32_t limit = v.limit;
    const int wide = ctx->sm_count * 8;
    if (p1 > p0) {
        StageScope timer(ctx, HSAW_STAGE_INDEX);
        const uint64_t nitems = p1 - p0;
        int hb = (int)std::min<uint64_t>((nitems + 255) / 256, (uint64_t)wide);
        const bool partition = (uint64_t)limit * 4 > (48ull << 20) && nitems > (1ull << 22);
        if (partition) {
            // in slices: the partitioned copy and the sort's scratch stay bounded however large
            // the pool is (5 G items per half at the Twitter shape). Every slice sweeps the whole
            // counter array once (read + write back through L2), so slices are as large as free
            // memory allows: an eighth of it per buffer, between 2^27 and 2^31 items.
            uint64_t slice = 1ull << 28;
            if (nitems > slice) {  // (cudaMemGetInfo is a slow call: only asked when it matters)
                size_t free_b = 0, total_b = 0;
                HSAW_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
                while (slice < (1ull << 31) && slice * 2 * 4 <= (free_b + ctx->g_sorted.cap * 4) / 8)
                    slice *= 2;
            }
            const uint64_t kSlice = slice;
            DevVec<uint32_t>& d_sorted = ctx->g_sorted;
            d_sorted.ensure_scratch(std::min(nitems, kSlice));
            int top = 32 - __builtin_clz(limit - 1);
            // HSAW_HIST_BITS: radix bits of the partition (A/B knob). 0 = the shared-memory form:
            // windows of at most 2^15 ids (128 KB of counters per CTA), two radix passes at the
            // Twitter shape. Anything else: that many top bits, counted with global atomics.
            static const int part_bits = [] {
                const char* env = std::getenv("HSAW_HIST_BITS");
                const int v = env ? std::atoi(env) : 0;
                return v < 0 ? 0 : (v > 32 ? 32 : v);
            }();
            const bool windows = part_bits == 0;
            const int wbits = std::min(15, top);
            int begin_bit = windows ? wbits : std::max(0, top - part_bits);
            const uint32_t nbuckets = (uint32_t)(((uint64_t)limit + (1ull << wbits) - 1) >> wbits);
            DevVec<uint64_t> starts;
            if (windows) {
                starts.ensure_scratch((uint64_t)nbuckets + 2);
                HSAW_CUDA_CHECK(cudaFuncSetAttribute(window_histogram,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)(4u << wbits)));
            }
            for (uint64_t at = 0; at < nitems; at += kSlice) {
                const uint64_t len = std::min(kSlice, nitems - at);
                size_t bytes = 0;
                HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(
                    nullptr, bytes, v.items + p0 + at, d_sorted.p, (int64_t)len, begin_bit, top, st));
                ctx->cub_tmp.ensure_scratch(bytes ? bytes : 1);
                HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(
                    ctx->cub_tmp.p, bytes, v.items + p0 + at, d_sorted.p, (int64_t)len, begin_bit,
                    top, st));
                ++ctx->launches;
                if (windows) {
                    bucket_starts<<<(unsigned)((len + 1023) / 1024), 256, 0, st>>>(
                        d_sorted.p, len, (uint32_t)wbits, nbuckets, starts.p);
                    check_launch(ctx, "bucket_starts");
                    window_histogram<<<nbuckets, 1024, (size_t)4 << wbits, st>>>(
                        d_sorted.p, starts.p, (uint32_t)wbits, limit, d_cand, d_cnt);
                    check_launch(ctx, "window_histogram");
                } else {
                    int sb = (int)std::min<uint64_t>((len + 255) / 256, (uint64_t)wide);
                    key_histogram<<<sb, 256, 0, st>>>(d_sorted.p, len, limit, d_cand, d_cnt);
                    check_launch(ctx, "key_histogram");
                }
            }
        } else {
            item_histogram<<<hb, 256, 0, st>>>(v, p0, p1, d_cand, d_cnt);
            check_launch(ctx, "item_histogram");
        }
    }
}

// ---- per-context histogram cache of a stream's walks -------------------------------------------------
// The doubling loop (proj/src/interdiction.cpp:36-47) asks, iteration after iteration, for the
// counts of R'_t = walks [s, 2s) (the upper bound) and of R_t = walks [0, s) (greedy). R_{t+1} is
// R_t u R'_t, so with the counts of the prefix kept and each new segment folded into it, every
// walk item is histogrammed exactly ONCE per solve instead of once per iteration that contains it
// (at the Twitter shape: 20 G instead of 37 G random counter updates). Only for "all candidates".
struct HistCache {
    uint64_t stream_uid = 0;
    int kind = -1;
    uint64_t prefix_end = 0;              // prefix[] = counts of walks [0, prefix_end)
    uint64_t seg_begin = 0, seg_end = 0;  // seg[] = counts of walks [seg_begin, seg_end), if seg_ok
    bool seg_ok = false;
    const uint32_t *prefix_buf = nullptr, *seg_buf = nullptr;  // the buffers the state describes
};
static HistCache& hist_cache(hsaw_gpu_ctx* ctx) {
    static std::mutex mu;
    static std::map<hsaw_gpu_ctx*, HistCache> caches;  // contexts are few and long-lived
    std::lock_guard<std::mutex> lock(mu);
    return caches[ctx];
}

// (128-bit accesses when both arrays are 16-byte aligned: 17.6 GB per fold at the Twitter shape)
__global__ void add_counts(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t done = 0;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        const uint64_t quads = n / 4;
        for (uint64_t i = tid; i < quads; i += stride) {
            uint4 a = d4[i];
            const uint4 b = __ldcs(s4 + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
            d4[i] = a;
        }
        done = quads * 4;
    }
    for (uint64_t i = done + tid; i < n; i += stride) dst[i] += src[i];
}

__global__ void offsets_to_lens(const uint64_t* __restrict__ off, uint64_t n, uint32_t* __restrict__ lens) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) lens[i] = (uint32_t)(off[i + 1] - off[i]);
}

static bool hist_cache_usable(const hsaw_gpu_stream* stream, const uint32_t* cand_ids) {
    static const bool off = [] {
        const char* env = std::getenv("HSAW_HIST_CACHE");  // A/B knob
        return env && std::atoi(env) == 0;
    }();
    return stream != nullptr && cand_ids == nullptr && !off;
}

// accumulates the counts of the stream's walks [a, b) into cnt (not zeroed here)
static void hist_accumulate(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind, uint64_t a,
                            uint64_t b, uint32_t* cnt) {
    if (b <= a) return;
    WalkView v = make_view(stream, nullptr, kind, a, b - a);
    uint64_t p0 = 0, p1 = 0;
    view_span(ctx, v, &p0, &p1);
    histogram_counts(ctx, v, p0, p1, nullptr, cnt);
}

static HistCache& hist_bind(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind,
                            uint64_t limit) {
    HistCache& hc = hist_cache(ctx);
    ctx->g_hist_prefix.ensure_scratch(limit + 4);
    ctx->g_hist_seg.ensure_scratch(limit + 4);
    // (the buffers are scratch of the context: a graph install or an allocation failure may have
    // released them since the state was recorded)
    if (hc.stream_uid != stream->uid || hc.kind != kind || hc.prefix_buf != ctx->g_hist_prefix.p ||
        hc.seg_buf != ctx->g_hist_seg.p) {
        hc = HistCache{};
        hc.stream_uid = stream->uid;
        hc.kind = kind;
        hc.prefix_buf = ctx->g_hist_prefix.p;
        hc.seg_buf = ctx->g_hist_seg.p;
    }
    if (hc.prefix_end == 0)
        HSAW_CUDA_CHECK(cudaMemsetAsync(ctx->g_hist_prefix.p, 0, (limit + 4) * 4, ctx->stream));
    return hc;
}

// folds the cached segment into the prefix when it starts at or after the prefix's end (the gap,
// if any, is histogrammed now): afterwards prefix = [0, seg_end)
static void hist_fold(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind, uint64_t limit,
                      HistCache& hc) {
    if (!hc.seg_ok || hc.seg_begin < hc.prefix_end) return;
    hist_accumulate(ctx, stream, kind, hc.prefix_end, hc.seg_begin, ctx->g_hist_prefix.p);
    {
        StageScope timer(ctx, HSAW_STAGE_INDEX);
        add_counts<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(ctx->g_hist_prefix.p,
                                                               ctx->g_hist_seg.p, limit);
        check_launch(ctx, "add_counts");
    }
    hc.prefix_end = hc.seg_end;
    hc.seg_ok = false;
}

// counts of the stream's walks [a, b), device resident, valid until the next cache call
static const uint32_t* hist_segment(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind,
                                    uint64_t limit, uint64_t a, uint64_t b) {
    HistCache& hc = hist_bind(ctx, stream, kind, limit);
    if (hc.seg_ok && hc.seg_begin == a && hc.seg_end == b) return ctx->g_hist_seg.p;
    if (a == 0) {  // a prefix request in disguise
        hist_fold(ctx, stream, kind, limit, hc);
        hc.seg_ok = false;
    } else {
        hist_fold(ctx, stream, kind, limit, hc);
    }
    HSAW_CUDA_CHECK(cudaMemsetAsync(ctx->g_hist_seg.p, 0, (limit + 4) * 4, ctx->stream));
    hist_accumulate(ctx, stream, kind, a, b, ctx->g_hist_seg.p);
    hc.seg_begin = a;
    hc.seg_end = b;
    hc.seg_ok = true;
    return ctx->g_hist_seg.p;
}

// counts of the stream's walks [0, x)
static const uint32_t* hist_prefix(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind,
                                   uint64_t limit, uint64_t x) {
    HistCache& hc = hist_bind(ctx, stream, kind, limit);
    if (hc.seg_ok && hc.seg_begin >= hc.prefix_end && hc.seg_end <= x)
        hist_fold(ctx, stream, kind, limit, hc);
    if (hc.prefix_end > x) {  // cannot shrink: start over
        HSAW_CUDA_CHECK(cudaMemsetAsync(ctx->g_hist_prefix.p, 0, (limit + 4) * 4, ctx->stream));
        hc.prefix_end = 0;
    }
    hist_accumulate(ctx, stream, kind, hc.prefix_end, x, ctx->g_hist_prefix.p);
    hc.prefix_end = x;
    return ctx->g_hist_prefix.p;
}

extern "C" {

int hsaw_gpu_walkset_import(hsaw_gpu_ctx* ctx, uint32_t limit, uint64_t nsets,
                            const uint64_t* set_off, const uint32_t* items,
                            hsaw_gpu_walkset** out) {
    if (!ctx || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        if (!set_off) fail(HSAW_EINVAL, "walkset_import: null offsets");
        if (nsets > 0xFFFFFFFFull) fail(HSAW_EINVAL, "walkset_import: more than 2^32 sets");
        if (set_off[0] != 0) fail(HSAW_EINVAL, "walkset_import: offsets must start at 0");
        for (uint64_t i = 0; i < nsets; ++i)
            if (set_off[i + 1] < set_off[i]) fail(HSAW_EINVAL, "walkset_import: offsets decrease");
        uint64_t nitems = set_off[nsets];
        if (nitems && !items) fail(HSAW_EINVAL, "walkset_import: null items");
        auto* w = new hsaw_gpu_walkset;
        w->ctx = ctx;
        w->limit = limit;
        w->nsets = nsets;
        w->nitems = nitems;
        try {
            w->off.ensure_scratch(nsets + 1);
            w->items.ensure_scratch(nitems + 1);
            HSAW_CUDA_CHECK(cudaMemcpyAsync(w->off.p, set_off, (nsets + 1) * 8,
                                            cudaMemcpyHostToDevice, ctx->stream));
            if (nitems)
                HSAW_CUDA_CHECK(cudaMemcpyAsync(w->items.p, items, nitems * 4,
                                                cudaMemcpyHostToDevice, ctx->stream));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete w;
            throw;
        }
        *out = w;
    });
}

void hsaw_gpu_walkset_destroy(hsaw_gpu_walkset* w) {
    if (!w) return;
    cudaSetDevice(w->ctx->device);
    delete w;
}

int hsaw_gpu_greedy(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                    const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                    const uint32_t* cand_ids, uint64_t ncand, uint32_t k, uint32_t* solution,
                    uint64_t* coverage) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!solution || !coverage) fail(HSAW_EINVAL, "greedy: null output");
        WalkView v = make_view(stream, walkset, kind, off, cnt);
        if (cnt > 0xFFFFFFFFull) fail(HSAW_EINVAL, "greedy: more than 2^32 walks");  // coverage.hpp:41
        cudaStream_t st = ctx->stream;
        const uint32_t limit = v.limit;
        std::vector<uint32_t> cand_sorted;
        DevVec<uint32_t>& cand_bits = ctx->g_cand_bits;
        uint64_t ncands = prepare_candidates(ctx, limit, cand_ids, ncand, cand_sorted, cand_bits);
        const uint32_t* d_cand = cand_ids ? cand_bits.p : nullptr;
        if (k > ncands)  // proj/src/coverage.cpp:93-94
            fail(HSAW_EINVAL, "budget k exceeds candidate count");
        *coverage = 0;
        if (k == 0) return;

        // ---- one greedy run with inverted lists for items whose count is >= min_count
        // (0 = choose from the count distribution). Returns false when a round's winner fell below
        // the threshold, i.e. the run must be repeated with the full index (min_count 1).
        DevVec<uint32_t>& d_cnt = ctx->g_cnt;
        DevVec<uint32_t>& d_fill = ctx->g_fill;
        DevVec<uint64_t>& d_pos = ctx->g_pos;
        DevVec<uint32_t>& d_inv = ctx->g_inv;
        DevVec<uint32_t>& d_cov = ctx->g_covered;
        DevVec<uint64_t>& d_partial = ctx->g_partial;  // [0] = winner key of the round
        DevVec<uint64_t>& d_blkmax = ctx->g_blkmax;
        DevVec<uint32_t>& d_sol = ctx->g_solution;
        DevVec<uint64_t>& d_gain = ctx->g_gains;
        d_partial.ensure_scratch(kCountBins + 4);
        d_sol.ensure_scratch(k);
        d_gain.ensure_scratch(k);
        uint64_t cov_words = (cnt + 31) / 32 + 1;
        d_cov.ensure_scratch(cov_words);
        std::vector<uint32_t> h_sol(k, 0xFFFFFFFFu);
        std::vector<uint64_t> h_gain(k, 0);
        uint64_t p0 = 0, p1 = 0;
        if (cnt) view_span(ctx, v, &p0, &p1);
        const int wide = ctx->sm_count * 8;
        const int cover_blocks = ctx->sm_count * 2;
        uint32_t done = 0;
        // Id spaces from 4 M items run on a dense reduced instance (build_dense above; C2's 16 M
        // edges: eSIA k=1000 0.083 -> 0.056 s, the Twitter shape: see DESIGN.md). HSAW_DENSE_MIN_BYTES:
        // size of the per-item counter array from which it applies (0 forces it everywhere: tests);
        // HSAW_INDEX_MASS_DIV: the indexed items hold at most 1/div of all occurrences.
        const uint64_t dense_min_bytes = [] {  // (read per call: the tests flip it)
            const char* env = std::getenv("HSAW_DENSE_MIN_BYTES");
            return env ? std::strtoull(env, nullptr, 10) : (16ull << 20);
        }();
        const uint64_t mass_div = [] {
            const char* env = std::getenv("HSAW_INDEX_MASS_DIV");
            const uint64_t d = env ? std::strtoull(env, nullptr, 10) : 8;
            return d ? d : 8;
        }();
        const bool dense_forced = dense_min_bytes == 0;
        const bool dense_possible = cand_ids == nullptr && p1 > p0 &&
                                    (dense_forced || ((uint64_t)limit * 4 > dense_min_bytes &&
                                                      p1 - p0 > (1ull << 20)));

        // min_count 0: choose the indexing threshold from the count distribution: the mass rule
        // (at most 1/mass_div of all occurrences indexed), raised to ck_percent % of the k-th
        // largest count when ck_percent is set. A winner's gain never exceeds its initial count
        // and the gains of a run never increase, so items whose count is below the LAST round's
        // gain can never be selected: a threshold near that gain keeps a few thousand items
        // instead of millions. It is a guess that the protocol verifies (a round whose winner
        // falls below the threshold fails the run), so a wrong guess costs one cheap attempt.
        std::vector<uint32_t> failed_thresholds;
        // counts of the view's items (limit + zero pad entries) and their distribution: computed
        // once, again only after an attempt that decremented them in place (the non-dense form on
        // counts that did not come from the histogram cache)
        const uint32_t* full_cnt = nullptr;
        const bool from_cache = hist_cache_usable(stream, cand_ids) && off == 0;
        bool counts_valid = false;
        std::vector<uint64_t> bins;
        // ---- K3: marginal-gain counts (a stream prefix comes from the histogram cache) and their
        // distribution; idempotent until an attempt invalidates the counts
        auto prepare = [&](bool want_bins) {
            if (!counts_valid) {
                if (from_cache) {
                    full_cnt = hist_prefix(ctx, stream, kind, limit, cnt);
                } else {
                    d_cnt.ensure_scratch((uint64_t)limit + 4);
                    HSAW_CUDA_CHECK(cudaMemsetAsync(d_cnt.p, 0, ((uint64_t)limit + 4) * 4, st));
                    histogram_counts(ctx, v, p0, p1, d_cand, d_cnt.p);
                    full_cnt = d_cnt.p;
                }
                counts_valid = true;
                bins.clear();
            }
            if (want_bins && bins.empty()) {
                auto* d_bins = reinterpret_cast<unsigned long long*>(d_partial.p + 4);
                HSAW_CUDA_CHECK(cudaMemsetAsync(d_bins, 0, kCountBins * 8, st));
                {
                    StageScope timer(ctx, HSAW_STAGE_INDEX);
                    count_of_counts<<<wide, kCocWarps * 32, 0, st>>>(full_cnt, limit, d_bins);
                    check_launch(ctx, "count_of_counts");
                }
                bins.resize(kCountBins);
                HSAW_CUDA_CHECK(cudaMemcpyAsync(bins.data(), d_bins, kCountBins * 8,
                                                cudaMemcpyDeviceToHost, st));
                HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            }
        };
        auto run = [&](uint32_t min_count, uint32_t ck_percent) -> bool {
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_cov.p, 0, cov_words * 4, st));
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_partial.p, 0, 8, st));  // no previous winner yet
            prepare(min_count == 0 || dense_possible);
            uint64_t total = 0;  // occurrences of all (candidate) items in the view
            for (uint64_t b : bins) total += b;
            if (min_count == 0) {
                // Index only what can win: the smallest count whose items (and everything above)
                // make up at most 1/8 of all occurrences. Small inputs index everything.
                min_count = 1;
                if (total > (1ull << 20)) {
                    uint64_t above = 0;
                    min_count = kCountBins - 1;
                    for (uint32_t c = kCountBins - 1; c >= 1; --c) {
                        if (above + bins[c] > total / mass_div) break;
                        above += bins[c];
                        min_count = c;
                    }
                }
                if (ck_percent) {
                    // k-th largest count (the pooled top bin is counted as if all its items sat at
                    // its lower edge: more items than there are, i.e. a bolder guess at worst)
                    uint64_t items = 0;
                    uint32_t ck = 0;
                    for (uint32_t c = kCountBins - 1; c >= 1 && ck == 0; --c) {
                        items += (bins[c] + c - 1) / c;
                        if (items >= k) ck = c;
                    }
                    min_count = std::max<uint32_t>(min_count, (uint32_t)((uint64_t)ck * ck_percent / 100));
                }
                for (uint32_t t : failed_thresholds)
                    if (min_count >= t) return false;  // already known to be too high
            }
            // ---- the instance the rounds run on: the view itself, or its dense reduction
            // (the full index too takes the dense form while the view holds fewer items than the
            // id space has ids: every per-item array then has one entry per PRESENT item - nSIA at
            // the Twitter shape: 4.7 M node occurrences against 41.6 M nodes)
            const bool dense = dense_possible && (dense_forced || min_count > 1 || total < limit);
            WalkView rv = v;
            uint32_t rlimit = limit;
            uint32_t* rcnt = nullptr;
            DenseScratch& dx = ctx->g_dense;
            DevVec<uint32_t>&x_bits = dx.bits, &x_pc = dx.pc, &x_base = dx.base, &x_bloom = dx.bloom,
                             &x_ids = dx.ids, &x_cnt = dx.cnt, &x_items = dx.items, &x_pw = dx.pw,
                             &x_pr = dx.pr, &x_sw = dx.sw, &x_flag = dx.flag;
            DevVec<uint64_t>&x_map = dx.map, &x_start = dx.start;
            if (dense) {
                uint64_t occ = 0, d_est = 0;  // occurrences / distinct ids at or above min_count
                for (uint32_t c = std::max(min_count, 1u); c < kCountBins; ++c) {
                    occ += bins[c];
                    d_est += c < kCountBins - 1 ? bins[c] / c : (bins[c] + kCountBins - 2) / (kCountBins - 1);
                }
                const uint64_t words = ((uint64_t)limit + 31) / 32;
                uint32_t log2w = 14;  // 32 filter bits per indexed id where a cached table allows it
                while ((1ull << log2w) < d_est && log2w < 23) ++log2w;
                x_bits.ensure_scratch(words + 1);
                x_pc.ensure_scratch(words + 1);
                x_base.ensure_scratch(words + 1);
                x_bloom.ensure_scratch(1ull << log2w);
                HSAW_CUDA_CHECK(cudaMemsetAsync(x_bloom.p, 0, (1ull << log2w) * 4, st));
                HSAW_CUDA_CHECK(cudaMemsetAsync(x_pc.p + words, 0, 4, st));
                const unsigned mark_blocks = (unsigned)((words + 255) / 256);  // 8 warps x 32 words
                {
                    StageScope timer(ctx, HSAW_STAGE_INDEX);
                    dense_mark<<<mark_blocks, 256, 0, st>>>(full_cnt, limit, std::max(min_count, 1u),
                                                            x_bits.p, x_pc.p, x_bloom.p, log2w);
                    check_launch(ctx, "dense_mark");
                    exclusive_sum_u32(ctx, x_pc.p, x_base.p, words + 1);
                }
                const uint64_t D = read_u32(ctx, x_base.p + words);
                if (D == 0) {
                    // nothing at or above the threshold (the mass rule can land one above a flat
                    // distribution's only count): the full-id form would report an unindexed
                    // winner at once; with threshold 1 there is simply nothing to select
                    if (min_count > 1) {
                        failed_thresholds.push_back(min_count);
                        return false;
                    }
                    done = 0;
                    return true;
                }
                x_map.ensure_scratch(words + 1);
                x_ids.ensure_scratch(D + 1);
                x_cnt.ensure_scratch(D + 4);
                const uint64_t P = occ;  // every occurrence of an indexed item becomes one pair
                if (const char* env = std::getenv("HSAW_GREEDY_DEBUG"))
                    if (std::atoi(env))
                        std::fprintf(stderr,
                                     "[hsaw greedy] walks %llu items %llu k %u: threshold %u (%u %% of "
                                     "c_k) -> D %llu ids, %llu pairs, filter 2^%u words\n",
                                     (unsigned long long)cnt, (unsigned long long)(p1 - p0), k,
                                     min_count, ck_percent, (unsigned long long)D,
                                     (unsigned long long)P, log2w);
                x_pw.ensure_scratch(P + 2);
                x_pr.ensure_scratch(P + 2);
                x_sw.ensure_scratch(P + 2);
                x_items.ensure_scratch(P + 2);
                x_flag.ensure_scratch(P + 2);
                auto* d_cursor = reinterpret_cast<unsigned long long*>(ctx->d_scalars + 12);
                HSAW_CUDA_CHECK(cudaMemsetAsync(d_cursor, 0, 8, st));
                HSAW_CUDA_CHECK(cudaMemsetAsync(x_cnt.p, 0, (D + 4) * 4, st));
                {
                    StageScope timer(ctx, HSAW_STAGE_INDEX);
                    dense_emit<<<mark_blocks, 256, 0, st>>>(full_cnt, limit, x_bits.p, x_base.p,
                                                            reinterpret_cast<uint2*>(x_map.p), x_ids.p,
                                                            x_cnt.p);
                    check_launch(ctx, "dense_emit");
                    const int eb = (int)std::min<uint64_t>((p1 - p0 + 1023) / 1024, (uint64_t)wide * 2);
                    dense_pairs<<<eb, 256, 0, st>>>(v, p0, p1, Bloom2{x_bloom.p, log2w},
                                                    reinterpret_cast<const uint2*>(x_map.p), d_cursor,
                                                    x_pw.p, x_pr.p);
                    check_launch(ctx, "dense_pairs");
                }
                if (read_u64(ctx, reinterpret_cast<uint64_t*>(d_cursor)) != P)
                    fail(HSAW_ECUDA, "greedy: dense instance does not match the counts (internal error)");
                uint64_t nw = 0;
                if (P) {
                    StageScope timer(ctx, HSAW_STAGE_INDEX);
                    int wbits = 1;
                    while (wbits < 32 && (1ull << wbits) < cnt) ++wbits;
                    size_t bytes = 0;
                    HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(
                        nullptr, bytes, x_pw.p, x_sw.p, x_pr.p, x_items.p, (int64_t)P, 0, wbits, st));
                    ctx->cub_tmp.ensure_scratch(bytes ? bytes : 1);
                    HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(
                        ctx->cub_tmp.p, bytes, x_pw.p, x_sw.p, x_pr.p, x_items.p, (int64_t)P, 0, wbits,
                        st));
                    ++ctx->launches;
                    pair_heads<<<(unsigned)((P + 256) / 256), 256, 0, st>>>(x_sw.p, P, x_flag.p);
                    check_launch(ctx, "pair_heads");
                    exclusive_sum_u32(ctx, x_flag.p, x_pw.p, P + 1);  // x_pw: walk rank of each pair
                }
                if (P) nw = read_u32(ctx, x_pw.p + P);
                x_start.ensure_scratch(nw + 2);
                if (P) {
                    StageScope timer(ctx, HSAW_STAGE_INDEX);
                    pair_starts<<<(unsigned)((P + 256) / 256), 256, 0, st>>>(x_flag.p, x_pw.p, P,
                                                                             x_start.p);
                    check_launch(ctx, "pair_starts");
                } else {
                    HSAW_CUDA_CHECK(cudaMemsetAsync(x_start.p, 0, 8, st));
                }
                rv = WalkView{x_start.p, x_items.p, 0, nw, 0, (uint32_t)D};
                rlimit = (uint32_t)D;
                rcnt = x_cnt.p;
            } else {
                d_cnt.ensure_scratch((uint64_t)limit + 4);
                if (from_cache) {
                    HSAW_CUDA_CHECK(cudaMemsetAsync(d_cnt.p + limit, 0, 16, st));
                    HSAW_CUDA_CHECK(cudaMemcpyAsync(d_cnt.p, full_cnt, (uint64_t)limit * 4,
                                                    cudaMemcpyDeviceToDevice, st));
                }
                rcnt = d_cnt.p;
                if (!from_cache) counts_valid = false;  // the rounds decrement d_cnt in place
            }
            const uint32_t index_min = dense ? 1u : min_count;  // a dense instance holds indexed items only
            const uint32_t bshift = block_shift_for(rlimit);
            const uint32_t nblk = (uint32_t)(((uint64_t)rlimit + (1ull << bshift) - 1) >> bshift);
            d_blkmax.ensure_scratch(nblk + 1);
            d_fill.ensure_scratch((uint64_t)rlimit + 4);
            d_pos.ensure_scratch((uint64_t)rlimit + 2);
            // ---- K3b: inverted lists (counting sort) of the items at or above min_count
            uint32_t* d_thr = d_fill.p;  // reused as the scan input, re-zeroed below
            {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                uint64_t n1 = (uint64_t)rlimit + 1;
                threshold_counts<<<(unsigned)((n1 + 255) / 256), 256, 0, st>>>(rcnt, n1, index_min, d_thr);
                check_launch(ctx, "threshold_counts");
                exclusive_sum_u32_to_u64(ctx, d_thr, d_pos.p, n1);
                HSAW_CUDA_CHECK(cudaMemsetAsync(d_fill.p, 0, ((uint64_t)rlimit + 4) * 4, st));
            }
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[0], d_pos.p + rlimit, 8,
                                            cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            const uint64_t indexed = ctx->h_scalars[0];
            d_inv.ensure_scratch(indexed + 1);
            if (indexed) {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                int sb = (int)std::min<uint64_t>((cnt + 7) / 8, (uint64_t)wide);
                if (dense) {
                    scatter_inverted<<<sb, 256, 0, st>>>(rv, nullptr, BitFilter{nullptr, 0}, d_pos.p,
                                                         d_fill.p, d_inv.p);
                } else {
                    DevVec<uint32_t>& d_ibits = ctx->g_indexed_bits;
                    uint64_t words = ((uint64_t)limit + 31) / 32;
                    d_ibits.ensure_scratch(words + 1);
                    const BitFilter filt = prepare_filter(ctx, limit, indexed);
                    mark_indexed<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(
                        rcnt, limit, min_count, d_ibits.p, const_cast<uint32_t*>(filt.bits), filt.log2);
                    check_launch(ctx, "mark_indexed");
                    scatter_inverted<<<sb, 256, 0, st>>>(rv, d_ibits.p, filt, d_pos.p, d_fill.p, d_inv.p);
                }
                check_launch(ctx, "scatter_inverted");
            }
            // ---- rounds
            if (p1 > p0) {
                StageScope timer(ctx, HSAW_STAGE_ROUNDS);
                block_maxima<<<nblk, 256, 0, st>>>(rcnt, rlimit, d_blkmax.p, bshift);
                check_launch(ctx, "block_maxima");
            }
            done = 0;
            bool exhausted = p1 == p0;
            bool blkmax_fresh = p1 > p0;  // block_maxima just ran: the bounds are exact maxima
            // Rounds with long lists go to the grid-wide kernel pair, a few at a time; as soon as
            // the lists are short the single-CTA tail kernel takes all remaining rounds in one
            // launch (it hands a round back if its list is too long after all).
            static const bool tail_off = [] {
                const char* env = std::getenv("HSAW_GREEDY_TAIL");  // A/B knob
                return env && std::atoi(env) == 0;
            }();
            const uint32_t kMaxTailList = 4096;
            const size_t tail_smem = (size_t)nblk * 8 + ((size_t)nblk + 31) / 32 * 4;
            const bool tail_ok = !tail_off && tail_smem <= (200u << 10);
            // the opt-in is a per-device function attribute: set before every use (it is a
            // host-side table write, nothing next to a launch)
            if (tail_ok && tail_smem > (48u << 10))
                HSAW_CUDA_CHECK(cudaFuncSetAttribute(greedy_tail_kernel,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)tail_smem));
            uint32_t* d_done = reinterpret_cast<uint32_t*>(d_partial.p + 2);
            bool try_tail = tail_ok;
            while (done < k && !exhausted) {
                uint32_t upto;
                if (try_tail) {
                    HSAW_CUDA_CHECK(cudaMemsetAsync(d_done, 0, 4, st));
                    {
                        StageScope timer(ctx, HSAW_STAGE_ROUNDS);
                        greedy_tail_kernel<<<1, 1024, tail_smem, st>>>(
                            rv, d_cand, d_pos.p, d_inv.p, rcnt, d_cov.p, d_blkmax.p, nblk, done,
                            k, d_sol.p, d_gain.p, min_count, kMaxTailList, d_done,
                            blkmax_fresh ? 1 : 0, bshift);
                        blkmax_fresh = false;  // the tail's own rounds decrement counts
                        check_launch(ctx, "greedy_tail_kernel");
                    }
                    uint32_t h_done = 0;
                    HSAW_CUDA_CHECK(
                        cudaMemcpyAsync(&h_done, d_done, 4, cudaMemcpyDeviceToHost, st));
                    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
                    upto = h_done;
                    try_tail = false;  // if rounds are left, the next one has a long list
                } else {
                    blkmax_fresh = false;
                    uint32_t group = std::min<uint32_t>(k - done, tail_ok ? 4 : 64);
                    StageScope timer(ctx, HSAW_STAGE_ROUNDS);
                    for (uint32_t r = done; r < done + group; ++r) {
                        select_lazy<<<1, 1024, 0, st>>>(rcnt, rlimit, d_blkmax.p, nblk,
                                                        d_partial.p, bshift);
                        check_launch(ctx, "select_lazy");
                        cover_winner<<<cover_blocks, 256, 0, st>>>(
                            rv, d_partial.p, 1, d_cand, d_pos.p, d_inv.p, rcnt, d_cov.p, r,
                            d_sol.p, d_gain.p, min_count);
                        check_launch(ctx, "cover_winner");
                    }
                    upto = done + group;
                    try_tail = tail_ok;
                }
                if (upto > done) {
                    HSAW_CUDA_CHECK(cudaMemcpyAsync(h_sol.data() + done, d_sol.p + done,
                                                    (upto - done) * 4ull, cudaMemcpyDeviceToHost,
                                                    st));
                    HSAW_CUDA_CHECK(cudaMemcpyAsync(h_gain.data() + done, d_gain.p + done,
                                                    (upto - done) * 8ull, cudaMemcpyDeviceToHost,
                                                    st));
                    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
                }
                uint32_t r = done;
                for (; r < upto; ++r) {
                    if (h_sol[r] == kUnindexed) {  // needs a lower threshold / the full index
                        failed_thresholds.push_back(min_count);
                        return false;
                    }
                    if (h_gain[r] == 0) {
                        // A dense instance holds the indexed items only: running out of gain there
                        // says nothing about the items below the threshold, which still have
                        // their (smaller) counts - the full-id form would have reported one of
                        // them as an unindexed winner.
                        if (dense && min_count > 1) {
                            bool below = false;
                            for (uint32_t c = 1; c < min_count && c < kCountBins && !below; ++c)
                                below = bins[c] != 0;
                            if (below) {
                                failed_thresholds.push_back(min_count);
                                return false;
                            }
                        }
                        exhausted = true;
                        break;
                    }
                }
                done = r;
            }
            if (dense && done) {  // the rounds selected ranks of the dense instance: back to ids
                dense_solution_ids<<<(done + 255) / 256, 256, 0, st>>>(d_sol.p, done, rlimit, x_ids.p);
                check_launch(ctx, "dense_solution_ids");
                HSAW_CUDA_CHECK(cudaMemcpyAsync(h_sol.data(), d_sol.p, done * 4ull,
                                                cudaMemcpyDeviceToHost, st));
                HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            }
            return true;
        };
        bool ok = false;
        // Thresholds only pay while the rounds' gains stay near the initial counts. When the k
        // largest counts alone add up to a good part of the walks (node candidates next to the
        // suspects: a few hundred picks cover almost everything), coverage saturates, the late
        // gains collapse towards 1 and every thresholded attempt is bound to fail: go straight to
        // the full index then.
        bool saturating = false;
        if (dense_possible) {
            prepare(true);
            uint64_t top = bins[kCountBins - 1], left = k;
            for (uint32_t c = kCountBins - 2; c >= 1 && left > 0; --c) {
                const uint64_t take = std::min<uint64_t>(bins[c] / c, left);
                top += take * c;
                left -= take;
            }
            saturating = top >= cnt / 2;
        }
        if (dense_possible && !saturating)  // optimistic thresholds: a dense attempt is cheap
            for (uint32_t pct : {60u, 30u})
                if ((ok = run(0, pct))) break;
        if (!ok && !saturating) ok = run(0, 0);
        if (!ok) {
            ++ctx->greedy_full_index_reruns;
            if (!run(1, 0)) fail(HSAW_ECUDA, "greedy: full index run reported an unindexed winner");
        }
        collect_timings(ctx);
        // ---- zero-gain padding: smallest unselected candidates in ascending order
        // (proj/src/coverage.cpp:101-106,155; pinned by tests/test_coverage.cpp:58-64)
        uint64_t cov = 0;
        // smallest gain of this run's rounds (0 when fewer than k rounds had a positive gain):
        // what a caller that fed a thresholded instance needs to know (sharded solve)
        ctx->last_greedy_min_gain = done < k ? 0 : ~0ull;
        for (uint32_t r = 0; r < done; ++r) {
            solution[r] = h_sol[r];
            cov += h_gain[r];
            ctx->last_greedy_min_gain = std::min<uint64_t>(ctx->last_greedy_min_gain, h_gain[r]);
        }
        if (done < k) {
            std::vector<uint32_t> chosen(solution, solution + done);
            std::sort(chosen.begin(), chosen.end());
            uint64_t ci = 0;  // index into the ascending candidate sequence
            size_t sj = 0;
            for (uint32_t r = done; r < k; ++r) {
                for (;;) {
                    uint32_t c = cand_ids ? cand_sorted[ci] : (uint32_t)ci;
                    while (sj < chosen.size() && chosen[sj] < c) ++sj;
                    if (sj < chosen.size() && chosen[sj] == c) {
                        ++ci;
                        continue;
                    }
                    solution[r] = c;
                    ++ci;
                    break;
                }
            }
        }
        *coverage = cov;
    });
}

// ---- stepwise greedy session -------------------------------------------------------------------
struct hsaw_gpu_rounds {
    hsaw_gpu_ctx* ctx = nullptr;
    WalkView v{};
    uint32_t limit = 0;
    uint32_t* d_counts = nullptr;  // caller-owned: global marginal-gain counts after all-reduce
    bool has_cand = false;
    DevVec<uint32_t> cand_bits, fill, inv, covered, indexed_bits;
    DevVec<uint64_t> pos, partial, scalars;
    uint64_t occurrences = 0;
    uint32_t npartial = 0;
    uint32_t bshift = 11;
    bool maxima_ready = false;
};

int hsaw_gpu_rounds_begin(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                          const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                          const uint32_t* cand_ids, uint64_t ncand, uint32_t* d_counts,
                          hsaw_gpu_rounds** out) {
    if (!ctx || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        if (!d_counts) fail(HSAW_EINVAL, "greedy_begin: null counts buffer");
        WalkView v = make_view(stream, walkset, kind, off, cnt);
        if (cnt > 0xFFFFFFFFull) fail(HSAW_EINVAL, "greedy_begin: more than 2^32 walks");
        auto* g = new hsaw_gpu_rounds;
        try {
            g->ctx = ctx;
            g->v = v;
            g->limit = v.limit;
            g->d_counts = d_counts;
            g->has_cand = cand_ids != nullptr;
            cudaStream_t st = ctx->stream;
            std::vector<uint32_t> sorted;
            (void)prepare_candidates(ctx, v.limit, cand_ids, ncand, sorted, g->cand_bits);
            const uint32_t* d_cand = g->has_cand ? g->cand_bits.p : nullptr;
            const uint64_t limit = v.limit;
            g->fill.ensure_scratch(limit + 4);
            g->pos.ensure_scratch(limit + 2);
            g->scalars.ensure_scratch(8);
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, (limit + 4) * 4, st));
            HSAW_CUDA_CHECK(cudaMemsetAsync(g->fill.p, 0, (limit + 4) * 4, st));
            uint64_t p0 = 0, p1 = 0;
            if (cnt) view_span(ctx, v, &p0, &p1);
            const int wide = ctx->sm_count * 8;
            {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                if (p1 > p0) {
                    int hb = (int)std::min<uint64_t>((p1 - p0 + 255) / 256, (uint64_t)wide);
                    item_histogram<<<hb, 256, 0, st>>>(v, p0, p1, d_cand, d_counts);
                    check_launch(ctx, "item_histogram");
                }
                exclusive_sum_u32_to_u64(ctx, d_counts, g->pos.p, limit + 1);
            }
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[0], g->pos.p + limit, 8,
                                            cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            g->occurrences = ctx->h_scalars[0];
            g->inv.ensure_scratch(g->occurrences + 1);
            if (g->occurrences) {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                int sb = (int)std::min<uint64_t>((cnt + 7) / 8, (uint64_t)wide);
                uint64_t words = (limit + 31) / 32;
                g->indexed_bits.ensure_scratch(words + 1);
                mark_indexed<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(
                    d_counts, (uint32_t)limit, 1u, g->indexed_bits.p, nullptr, 0);
                check_launch(ctx, "mark_indexed");
                scatter_inverted<<<sb, 256, 0, st>>>(v, g->indexed_bits.p, BitFilter{nullptr, 0},
                                                     g->pos.p, g->fill.p, g->inv.p);
                check_launch(ctx, "scatter_inverted");
            }
            uint64_t cov_words = (cnt + 31) / 32 + 1;
            g->covered.ensure_scratch(cov_words);
            HSAW_CUDA_CHECK(cudaMemsetAsync(g->covered.p, 0, cov_words * 4, st));
            g->bshift = block_shift_for(limit);
            g->npartial = (uint32_t)(((uint64_t)limit + (1ull << g->bshift) - 1) >> g->bshift);  // blocks
            g->partial.ensure_scratch(g->npartial + 1);  // block maxima, built at the first select
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            collect_timings(ctx);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

uint64_t hsaw_gpu_rounds_occurrences(const hsaw_gpu_rounds* g) { return g ? g->occurrences : 0; }

int hsaw_gpu_rounds_select(hsaw_gpu_rounds* g, uint32_t* item, uint64_t* gain) {
    if (!g || !item || !gain) return HSAW_EINVAL;
    hsaw_gpu_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        cudaStream_t st = ctx->stream;
        {
            StageScope timer(ctx, HSAW_STAGE_ROUNDS);
            if (!g->maxima_ready) {  // after the caller's all-reduce of the counts
                block_maxima<<<g->npartial, 256, 0, st>>>(g->d_counts, g->limit, g->partial.p, g->bshift);
                check_launch(ctx, "block_maxima");
                g->maxima_ready = true;
            }
            select_lazy<<<1, 1024, 0, st>>>(g->d_counts, g->limit, g->partial.p, g->npartial,
                                            g->scalars.p + 3, g->bshift);
            check_launch(ctx, "select_lazy");
            select_final<<<1, 256, 0, st>>>(g->scalars.p + 3, 1, g->scalars.p);
            check_launch(ctx, "select_final");
        }
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[0], g->scalars.p, 16,
                                        cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        collect_timings(ctx);
        *gain = ctx->h_scalars[0];
        *item = (uint32_t)ctx->h_scalars[1];
    });
}

int hsaw_gpu_rounds_cover(hsaw_gpu_rounds* g, uint32_t item, uint32_t* d_list, uint64_t list_cap,
                          uint64_t* n_out) {
    if (!g || !n_out) return HSAW_EINVAL;
    hsaw_gpu_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        if (item >= g->limit) fail(HSAW_EINVAL, "greedy_cover: item out of range");
        if (list_cap && !d_list) fail(HSAW_EINVAL, "greedy_cover: null list buffer");
        cudaStream_t st = ctx->stream;
        auto* d_count = reinterpret_cast<unsigned long long*>(g->scalars.p + 2);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_count, 0, 8, st));
        if (g->occurrences) {
            StageScope timer(ctx, HSAW_STAGE_ROUNDS);
            cover_item<<<ctx->sm_count * 2, 256, 0, st>>>(
                g->v, item, g->has_cand ? g->cand_bits.p : nullptr, g->pos.p, g->inv.p,
                g->d_counts, g->covered.p, d_list, list_cap, d_count);
            check_launch(ctx, "cover_item");
        }
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(&ctx->h_scalars[0], d_count, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        collect_timings(ctx);
        *n_out = ctx->h_scalars[0];
        if (*n_out > list_cap) fail(HSAW_EINVAL, "greedy_cover: decrement list buffer too small");
    });
}

int hsaw_gpu_rounds_apply(hsaw_gpu_rounds* g, const uint32_t* d_items, uint64_t n) {
    if (!g) return HSAW_EINVAL;
    hsaw_gpu_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        if (n == 0) return;
        if (!d_items) fail(HSAW_EINVAL, "greedy_apply: null items");
        StageScope timer(ctx, HSAW_STAGE_ROUNDS);
        apply_decrements<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(d_items, n, g->limit,
                                                                              g->d_counts);
        check_launch(ctx, "apply_decrements");
    });
}

void hsaw_gpu_rounds_end(hsaw_gpu_rounds* g) {
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    current_stream() = g->ctx->stream;
    cudaStreamSynchronize(g->ctx->stream);
    delete g;
}

int hsaw_gpu_coverage_upper_bound(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                                  const hsaw_gpu_walkset* walkset, int kind, uint64_t off,
                                  uint64_t cnt, const uint32_t* cand_ids, uint64_t ncand,
                                  uint32_t k, uint64_t* bound) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!bound) fail(HSAW_EINVAL, "coverage_upper_bound: null output");
        WalkView v = make_view(stream, walkset, kind, off, cnt);
        *bound = 0;
        if (cnt == 0 || k == 0) return;
        cudaStream_t st = ctx->stream;
        const uint32_t limit = v.limit;
        std::vector<uint32_t> cand_sorted;
        DevVec<uint32_t>& cand_bits = ctx->g_cand_bits;
        (void)prepare_candidates(ctx, limit, cand_ids, ncand, cand_sorted, cand_bits);
        const uint32_t* d_cand = cand_ids ? cand_bits.p : nullptr;
        DevVec<uint32_t>& d_cnt = ctx->g_cnt;
        DevVec<uint64_t>& d_partial = ctx->g_partial;
        d_partial.ensure_scratch(kCountBins + 4);
        uint64_t p0 = 0, p1 = 0;
        view_span(ctx, v, &p0, &p1);
        if (p1 == p0) return;
        const uint32_t* counts = nullptr;
        if (hist_cache_usable(stream, cand_ids)) {
            counts = hist_segment(ctx, stream, kind, limit, off, off + cnt);
        } else {
            d_cnt.ensure_scratch((uint64_t)limit + 4);
            counts = d_cnt.p;
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_cnt.p, 0, ((uint64_t)limit + 4) * 4, st));
            histogram_counts(ctx, v, p0, p1, d_cand, d_cnt.p);
        }
        auto* d_bins = reinterpret_cast<unsigned long long*>(d_partial.p + 4);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_bins, 0, kCountBins * 8, st));
        {
            StageScope timer(ctx, HSAW_STAGE_INDEX);
            count_of_counts<<<ctx->sm_count * 8, kCocWarps * 32, 0, st>>>(counts, limit, d_bins);
            check_launch(ctx, "count_of_counts");
        }
        std::vector<uint64_t> bins(kCountBins);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(bins.data(), d_bins, kCountBins * 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        collect_timings(ctx);
        // bins[c] = c * (#items occurring c times); the last bin sums every count >= kCountBins-1
        // and is taken whole without using up any of the k slots, so the result stays a bound
        uint64_t total = bins[kCountBins - 1], left = k;
        for (uint32_t c = kCountBins - 2; c >= 1 && left > 0; --c) {
            uint64_t items = bins[c] / c;
            uint64_t take = std::min(items, left);
            total += take * c;
            left -= take;
        }
        *bound = std::min<uint64_t>(total, cnt);
    });
}

int hsaw_gpu_coverage_of(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                         const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                         const uint32_t* cand_ids, uint64_t ncand, const uint32_t* items,
                         uint64_t nitems, uint64_t* coverage) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!coverage) fail(HSAW_EINVAL, "coverage_of: null output");
        if (nitems && !items) fail(HSAW_EINVAL, "coverage_of: null items");
        WalkView v = make_view(stream, walkset, kind, off, cnt);
        *coverage = 0;
        if (cnt == 0 || nitems == 0) return;
        cudaStream_t st = ctx->stream;
        // only candidate items are indexed (CoverageIndex::insert, proj/src/coverage.cpp:31-35)
        std::vector<uint32_t> q;
        q.reserve(nitems);
        std::vector<uint32_t> cand_sorted;
        if (cand_ids) {
            cand_sorted.assign(cand_ids, cand_ids + ncand);
            std::sort(cand_sorted.begin(), cand_sorted.end());
        }
        for (uint64_t i = 0; i < nitems; ++i) {
            uint32_t it = items[i];
            if (it >= v.limit) continue;
            if (cand_ids && !std::binary_search(cand_sorted.begin(), cand_sorted.end(), it)) continue;
            q.push_back(it);
        }
        if (q.empty()) return;
        DevVec<uint32_t>& bits = ctx->g_query_bits;
        uint64_t words = ((uint64_t)v.limit + 31) / 32 + 1;
        if (bits.cap < words) {
            bits.ensure_scratch(words);
            HSAW_CUDA_CHECK(cudaMemsetAsync(bits.p, 0, bits.cap * 4, st));  // kept all-zero between calls
        }
        DevVec<uint32_t>& d_q = ctx->g_solution;
        d_q.ensure_scratch(q.size());
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(d_q.p, q.data(), q.size() * 4, cudaMemcpyHostToDevice, st));
        unsigned qb = (unsigned)((q.size() + 255) / 256);
        set_bits<<<qb, 256, 0, st>>>(d_q.p, q.size(), bits.p);
        check_launch(ctx, "set_bits");
        unsigned long long* d_out = reinterpret_cast<unsigned long long*>(ctx->d_scalars + 8);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 8, st));
        {
            StageScope timer(ctx, HSAW_STAGE_COVERAGE);
            int blocks = (int)std::min<uint64_t>((cnt + 7) / 8, (uint64_t)ctx->sm_count * 8);
            BitFilter filt = prepare_filter(ctx, v.limit, q.size());
            if (filt.log2) {
                set_filter_bits<<<qb, 256, 0, st>>>(d_q.p, q.size(), filt.log2,
                                                    const_cast<uint32_t*>(filt.bits));
                check_launch(ctx, "set_filter_bits");
            }
            // HSAW_COVERAGE_FLAT: 0 keeps the walk-by-walk kernel, 2 forces the flat one (tests);
            // default: flat from 2^20 items (read per call)
            const char* fenv = std::getenv("HSAW_COVERAGE_FLAT");
            const int fmode = fenv ? std::atoi(fenv) : 1;
            uint64_t p0 = 0, p1 = 0;
            view_span(ctx, v, &p0, &p1);
            if (p1 > p0 && (fmode == 2 || (fmode == 1 && p1 - p0 > (1ull << 20)))) {
                DevVec<uint32_t>& wb = ctx->g_covered;
                const uint64_t wwords = (cnt + 31) / 32 + 1;
                wb.ensure_scratch(wwords);
                HSAW_CUDA_CHECK(cudaMemsetAsync(wb.p, 0, wwords * 4, st));
                const int fb = (int)std::min<uint64_t>((p1 - p0 + 1023) / 1024,
                                                       (uint64_t)ctx->sm_count * 16);
                count_covered_flat<<<fb, 256, 0, st>>>(v, p0, p1, bits.p, filt, wb.p, d_out);
                check_launch(ctx, "count_covered_flat");
            } else {
                count_covered<<<blocks, 256, 0, st>>>(v, bits.p, filt, d_out);
                check_launch(ctx, "count_covered");
            }
            clear_bits<<<qb, 256, 0, st>>>(d_q.p, q.size(), bits.p);
            check_launch(ctx, "clear_bits");
        }
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(&ctx->h_scalars[0], d_out, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        collect_timings(ctx);
        *coverage = ctx->h_scalars[0];
    });
}

}  // extern "C"

// ---- building blocks of the sharded solve (paper_1702_05854_b200/sharded.py) -------------------------
// Walks are sharded over ranks; counts are combined with an all-reduce by the caller (NCCL over
// NVLink through torch.distributed, or libnccl directly). After the all-reduce every rank knows the
// global marginal-gain vector, extracts from its LOCAL walks only the items that can still win
// (global count >= the indexing threshold — the same rule the single-GPU greedy uses), the ranks
// all-gather those reduced walks, and each runs the single-GPU greedy (tail kernel included) on
// the gathered set redundantly: identical selections everywhere, rounds stay ~8 us, and what
// crosses NVLink is at most an eighth of the items once per greedy call instead of two collectives
// per round.

// one warp per walk: how many of its items are indexed
__global__ void reduced_count(WalkView v, const uint32_t* __restrict__ indexed_bits, BitFilter filter,
                              uint32_t* __restrict__ wcount) {
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < v.cnt; i += nwarps) {
        uint64_t w = v.w0 + i;
        uint64_t b = v.off[w] + v.add * w, e = v.off[w + 1] + v.add * (w + 1);
        uint32_t c = 0;
        for (uint64_t p = b + lane; p < e; p += 32) {
            uint32_t it = v.items[p];
            c += it < v.limit && filter_pass(filter, it) &&
                 ((indexed_bits[it >> 5] >> (it & 31)) & 1u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFullMask, c, o);
        if (lane == 0) wcount[i] = c;
    }
}

__global__ void reduced_flags(const uint32_t* __restrict__ wcount, uint64_t n,
                              uint32_t* __restrict__ flag) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= n) flag[i] = i < n && wcount[i] ? 1u : 0u;
}

// kept walks (>= 1 indexed item) in order; item order inside a walk is irrelevant (set semantics
// with multiplicity), so lanes place their items by ballot ranks
__global__ void reduced_write(WalkView v, const uint32_t* __restrict__ indexed_bits, BitFilter filter,
                              const uint32_t* __restrict__ wcount, const uint32_t* __restrict__ widx,
                              const uint64_t* __restrict__ ioff, uint32_t* __restrict__ out_lens,
                              uint32_t* __restrict__ out_items) {
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < v.cnt; i += nwarps) {
        if (!wcount[i]) continue;
        uint64_t w = v.w0 + i;
        uint64_t b = v.off[w] + v.add * w, e = v.off[w + 1] + v.add * (w + 1);
        if (lane == 0) out_lens[widx[i]] = wcount[i];
        uint64_t at = ioff[i];
        for (uint64_t p0 = b; p0 < e; p0 += 32) {
            uint64_t p = p0 + lane;
            uint32_t it = p < e ? v.items[p] : 0xFFFFFFFFu;
            bool keep = p < e && it < v.limit && filter_pass(filter, it) &&
                        ((indexed_bits[it >> 5] >> (it & 31)) & 1u);
            unsigned m = __ballot_sync(kFullMask, keep);
            if (keep) out_items[at + __popc(m & ((1u << lane) - 1))] = it;
            at += __popc(m);
        }
    }
}

static uint64_t scan_total_u32(hsaw_gpu_ctx* ctx, const uint32_t* d_in, uint64_t* d_out, uint64_t n) {
    exclusive_sum_u32_to_u64(ctx, d_in, d_out, n + 1);
    uint64_t total = 0;
    HSAW_CUDA_CHECK(cudaMemcpyAsync(&total, d_out + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return total;
}

extern "C" {

int hsaw_gpu_stream_histogram(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind,
                              uint64_t off, uint64_t cnt, const uint32_t* cand_ids, uint64_t ncand,
                              uint32_t* d_counts) {
    if (!ctx || !stream || !d_counts) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        WalkView v = make_view(stream, nullptr, kind, off, cnt);
        std::vector<uint32_t> cand_sorted;
        (void)prepare_candidates(ctx, v.limit, cand_ids, ncand, cand_sorted, ctx->g_cand_bits);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, (uint64_t)v.limit * 4, ctx->stream));
        if (cnt) {
            uint64_t p0 = 0, p1 = 0;
            view_span(ctx, v, &p0, &p1);
            histogram_counts(ctx, v, p0, p1, cand_ids ? ctx->g_cand_bits.p : nullptr, d_counts);
        }
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        collect_timings(ctx);
    });
}

// bins[c] = c * (#items with count c), counts >= kCountBins - 1 pooled in the last bin
static std::vector<uint64_t> count_bins(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit) {
    ctx->g_partial.ensure_scratch(kCountBins + 4);
    auto* d_bins = reinterpret_cast<unsigned long long*>(ctx->g_partial.p + 4);
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_bins, 0, kCountBins * 8, ctx->stream));
    {
        StageScope timer(ctx, HSAW_STAGE_INDEX);
        count_of_counts<<<ctx->sm_count * 8, kCocWarps * 32, 0, ctx->stream>>>(d_counts, limit, d_bins);
        check_launch(ctx, "count_of_counts");
    }
    std::vector<uint64_t> bins(kCountBins);
    HSAW_CUDA_CHECK(cudaMemcpyAsync(bins.data(), d_bins, kCountBins * 8, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    collect_timings(ctx);
    return bins;
}

int hsaw_gpu_counts_bound(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit, uint32_t k,
                          uint64_t cap, uint64_t* bound) {
    if (!ctx || !d_counts || !bound) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        const std::vector<uint64_t> bins = count_bins(ctx, d_counts, limit);
        uint64_t total = bins[kCountBins - 1], left = k;  // as hsaw_gpu_coverage_upper_bound
        for (uint32_t c = kCountBins - 2; c >= 1 && left > 0; --c) {
            uint64_t items = bins[c] / c;
            uint64_t take = std::min(items, left);
            total += take * c;
            left -= take;
        }
        *bound = std::min<uint64_t>(total, cap);
    });
}

int hsaw_gpu_counts_threshold(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit,
                              uint32_t* min_count) {
    if (!ctx || !d_counts || !min_count) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        const std::vector<uint64_t> bins = count_bins(ctx, d_counts, limit);
        uint64_t total = 0;
        for (uint64_t b : bins) total += b;
        uint32_t mc = 1;  // the rule of hsaw_gpu_greedy: index at most 1/8 of all occurrences
        if (total > (1ull << 20)) {
            uint64_t above = 0;
            mc = kCountBins - 1;
            for (uint32_t c = kCountBins - 1; c >= 1; --c) {
                if (above + bins[c] > total / 8) break;
                above += bins[c];
                mc = c;
            }
        }
        *min_count = mc;
    });
}

// The mass rule of hsaw_gpu_counts_threshold raised to ck_percent % of the k-th largest count: the
// optimistic rungs of hsaw_gpu_greedy's threshold ladder for callers that gather reduced walks
// (a run whose smallest gain stays at or above the threshold proves it was enough).
int hsaw_gpu_counts_threshold_for(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit,
                                  uint32_t k, uint32_t ck_percent, uint32_t* min_count) {
    if (!ctx || !d_counts || !min_count) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        const std::vector<uint64_t> bins = count_bins(ctx, d_counts, limit);
        uint64_t total = 0;
        for (uint64_t b : bins) total += b;
        uint32_t mc = 1;
        if (total > (1ull << 20)) {
            uint64_t above = 0;
            mc = kCountBins - 1;
            for (uint32_t c = kCountBins - 1; c >= 1; --c) {
                if (above + bins[c] > total / 8) break;
                above += bins[c];
                mc = c;
            }
        }
        if (ck_percent && k) {
            uint64_t items = 0;
            uint32_t ck = 0;
            for (uint32_t c = kCountBins - 1; c >= 1 && ck == 0; --c) {
                items += (bins[c] + c - 1) / c;
                if (items >= k) ck = c;
            }
            mc = std::max<uint32_t>(mc, (uint32_t)((uint64_t)ck * ck_percent / 100));
        }
        *min_count = mc;
    });
}

int hsaw_gpu_reduced_walks(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind, uint64_t off,
                           uint64_t cnt, const uint32_t* d_counts, uint32_t min_count,
                           hsaw_gpu_walkset** out, uint64_t* nsets, uint64_t* nitems) {
    if (!ctx || !stream || !d_counts || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        WalkView v = make_view(stream, nullptr, kind, off, cnt);
        cudaStream_t st = ctx->stream;
        const uint32_t limit = v.limit;
        auto w = std::make_unique<hsaw_gpu_walkset>();
        w->ctx = ctx;
        w->limit = limit;
        DevVec<uint32_t> wcount, flag, widx32;
        DevVec<uint64_t> ioff, widx;
        wcount.ensure_scratch(cnt + 1);
        flag.ensure_scratch(cnt + 1);
        ioff.ensure_scratch(cnt + 2);
        widx.ensure_scratch(cnt + 2);
        widx32.ensure_scratch(cnt + 1);
        uint64_t kept = 0, total = 0;
        if (cnt) {
            DevVec<uint32_t>& d_ibits = ctx->g_indexed_bits;
            const uint64_t words = ((uint64_t)limit + 31) / 32;
            d_ibits.ensure_scratch(words + 1);
            const BitFilter filt = prepare_filter(ctx, limit, (uint64_t)1 << 24);
            const int wide = ctx->sm_count * 8;
            const int sb = (int)std::min<uint64_t>((cnt + 7) / 8, (uint64_t)wide);
            {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                mark_indexed<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(
                    d_counts, limit, min_count ? min_count : 1u, d_ibits.p,
                    const_cast<uint32_t*>(filt.bits), filt.log2);
                check_launch(ctx, "mark_indexed");
                HSAW_CUDA_CHECK(cudaMemsetAsync(wcount.p + cnt, 0, 4, st));
                reduced_count<<<sb, 256, 0, st>>>(v, d_ibits.p, filt, wcount.p);
                check_launch(ctx, "reduced_count");
                reduced_flags<<<(unsigned)((cnt + 256) / 256), 256, 0, st>>>(wcount.p, cnt, flag.p);
                check_launch(ctx, "reduced_flags");
            }
            total = scan_total_u32(ctx, wcount.p, ioff.p, cnt);
            kept = scan_total_u32(ctx, flag.p, widx.p, cnt);
            // 32-bit copy of the walk ranks for the write kernel (kept < 2^32: walk ids are u32)
            w->off.ensure_scratch(kept + 1);
            w->items.ensure_scratch(total + 1);
            DevVec<uint32_t> lens;
            lens.ensure_scratch(kept + 1);
            exclusive_sum_u32(ctx, flag.p, widx32.p, cnt + 1);
            {
                StageScope timer(ctx, HSAW_STAGE_INDEX);
                reduced_write<<<sb, 256, 0, st>>>(v, d_ibits.p, filt, wcount.p, widx32.p, ioff.p,
                                                  lens.p, w->items.p);
                check_launch(ctx, "reduced_write");
            }
            HSAW_CUDA_CHECK(cudaMemsetAsync(lens.p + kept, 0, 4, st));
            exclusive_sum_u32_to_u64(ctx, lens.p, w->off.p, kept + 1);
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        } else {
            w->off.ensure_scratch(1);
            HSAW_CUDA_CHECK(cudaMemsetAsync(w->off.p, 0, 8, st));
            w->items.ensure_scratch(1);
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        }
        collect_timings(ctx);
        w->nsets = kept;
        w->nitems = total;
        if (nsets) *nsets = kept;
        if (nitems) *nitems = total;
        *out = w.release();
    });
}

// device-to-device: per-set lengths (u32[nsets]) and the items of a walk set into caller buffers
int hsaw_gpu_walkset_copy_device(const hsaw_gpu_walkset* w, uint32_t* d_lens, uint32_t* d_items) {
    if (!w) return HSAW_EINVAL;
    return guarded(w->ctx, [&] {
        cudaStream_t st = w->ctx->stream;
        if (d_lens && w->nsets) {
            offsets_to_lens<<<(unsigned)((w->nsets + 255) / 256), 256, 0, st>>>(w->off.p, w->nsets, d_lens);
            check_launch(w->ctx, "offsets_to_lens");
        }
        if (d_items && w->nitems)
            HSAW_CUDA_CHECK(cudaMemcpyAsync(d_items, w->items.p, w->nitems * 4,
                                            cudaMemcpyDeviceToDevice, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

// a walk set from device-resident per-set lengths and concatenated items (the all-gathered pieces)
int hsaw_gpu_walkset_from_device(hsaw_gpu_ctx* ctx, uint32_t limit, uint64_t nsets,
                                 const uint32_t* d_lens, const uint32_t* d_items, uint64_t nitems,
                                 hsaw_gpu_walkset** out) {
    if (!ctx || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        if (nsets > 0xFFFFFFFFull) fail(HSAW_EINVAL, "walkset_from_device: more than 2^32 sets");
        if ((nsets && !d_lens) || (nitems && !d_items)) fail(HSAW_EINVAL, "walkset_from_device: null array");
        auto w = std::make_unique<hsaw_gpu_walkset>();
        w->ctx = ctx;
        w->limit = limit;
        w->nsets = nsets;
        w->nitems = nitems;
        w->off.ensure_scratch(nsets + 1);
        w->items.ensure_scratch(nitems + 1);
        cudaStream_t st = ctx->stream;
        if (nsets) {
            DevVec<uint32_t> lens;
            lens.ensure_scratch(nsets + 1);
            HSAW_CUDA_CHECK(cudaMemcpyAsync(lens.p, d_lens, nsets * 4, cudaMemcpyDeviceToDevice, st));
            HSAW_CUDA_CHECK(cudaMemsetAsync(lens.p + nsets, 0, 4, st));
            exclusive_sum_u32_to_u64(ctx, lens.p, w->off.p, nsets + 1);
            uint64_t total = 0;
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&total, w->off.p + nsets, 8, cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            if (total != nitems) fail(HSAW_EINVAL, "walkset_from_device: lengths do not add up to nitems");
        } else {
            HSAW_CUDA_CHECK(cudaMemsetAsync(w->off.p, 0, 8, st));
        }
        if (nitems)
            HSAW_CUDA_CHECK(cudaMemcpyAsync(w->items.p, d_items, nitems * 4, cudaMemcpyDeviceToDevice, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        *out = w.release();
    });
}

uint64_t hsaw_gpu_last_greedy_min_gain(const hsaw_gpu_ctx* ctx) { return ctx ? ctx->last_greedy_min_gain : 0; }

// Plumbing for a host that drives several contexts from one process without its own CUDA code
// (host/multi.cpp): device buffers, copies between any two device pointers (unified addressing;
// across devices the driver goes peer-to-peer or through the host) and the element-wise sum the
// in-process all-reduce is made of. With distinct devices the host layer uses NCCL instead.
int hsaw_gpu_device_alloc(hsaw_gpu_ctx* ctx, uint64_t bytes, void** out) {
    if (!ctx || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        *out = pool_alloc(bytes ? bytes : 1, ctx->stream);
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}
void hsaw_gpu_device_free(hsaw_gpu_ctx* ctx, void* p) {
    if (!ctx || !p) return;
    guarded(ctx, [&] { cudaFreeAsync(p, ctx->stream); });
}
int hsaw_gpu_device_copy(hsaw_gpu_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (bytes) HSAW_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}
int hsaw_gpu_counts_add(hsaw_gpu_ctx* ctx, uint32_t* d_dst, const uint32_t* d_src, uint64_t n) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (n) {
            add_counts<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(d_dst, d_src, n);
            check_launch(ctx, "add_counts");
        }
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
