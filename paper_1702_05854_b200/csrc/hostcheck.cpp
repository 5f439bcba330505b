// Host-side check behind hsaw_gpu_graph_upload's "regenerate in_cum on the device" path
// (graph.cu): do the caller's cumulative weights equal, bit for bit, the sequential 1/in-degree
// sums of WeightMode::InDegree (proj/src/graph.cpp:172-178: w = 1.0 / d, cum += w, left to right)?
// Each element is compared with its left neighbour plus w (cum[lo] with w itself), which states
// the same thing by induction and has no dependent chain, so the scan runs at memory speed:
// AVX2 where the CPU has it (4 doubles per compare), scalar otherwise. Plain g++ translation unit:
// the intrinsics stay out of nvcc's front end.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "hostcheck.h"

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace hsawgpu {

namespace {

// 1.0 / d for the short rows that make up most of a power-law graph (a division per row costs
// as much as checking a dozen elements)
constexpr uint64_t kRecipTable = 2048;
const double* recip_table() {
    static const std::vector<double> t = [] {
        std::vector<double> r(kRecipTable, 0.0);
        for (uint64_t d = 1; d < kRecipTable; ++d) r[d] = 1.0 / (double)d;
        return r;
    }();
    return t.data();
}

// mismatches in one row (any non-zero value = "differs"); c = cum + lo, d = row length >= 1
inline uint64_t row_scalar(const double* c, uint64_t d, double w) {
    uint64_t bad = c[0] != w;  // 0.0 + w
    for (uint64_t i = 1; i < d; ++i) bad += c[i] != c[i - 1] + w;
    return bad;
}

#if defined(__x86_64__)
__attribute__((target("avx2"))) uint64_t rows_avx2(const uint64_t* off, const double* cum,
                                                   uint64_t va, uint64_t vb,
                                                   const std::atomic<bool>& stop) {
    uint64_t bad = 0;
    const double* recip = recip_table();
    for (uint64_t v = va; v < vb; ++v) {
        if ((v & 1023) == 0 && (bad || stop.load(std::memory_order_relaxed))) break;
        const uint64_t lo = off[v], hi = off[v + 1];
        if (hi <= lo) continue;
        const uint64_t d = hi - lo;
        const double w = d < kRecipTable ? recip[d] : 1.0 / (double)d;
        const double* c = cum + lo;
        bad += c[0] != w;
        const __m256d wv = _mm256_set1_pd(w);
        __m256d acc = _mm256_setzero_pd();
        uint64_t i = 1;
        for (; i + 4 <= d; i += 4) {
            const __m256d a = _mm256_loadu_pd(c + i);
            const __m256d s = _mm256_add_pd(_mm256_loadu_pd(c + i - 1), wv);
            acc = _mm256_or_pd(acc, _mm256_cmp_pd(a, s, _CMP_NEQ_UQ));  // NaN counts as different
        }
        bad += (uint64_t)_mm256_movemask_pd(acc);
        for (; i < d; ++i) bad += c[i] != c[i - 1] + w;
    }
    return bad;
}
#endif

uint64_t rows_plain(const uint64_t* off, const double* cum, uint64_t va, uint64_t vb,
                    const std::atomic<bool>& stop) {
    uint64_t bad = 0;
    for (uint64_t v = va; v < vb; ++v) {
        if ((v & 1023) == 0 && (bad || stop.load(std::memory_order_relaxed))) break;
        const uint64_t lo = off[v], hi = off[v + 1];
        if (hi > lo) bad += row_scalar(cum + lo, hi - lo, 1.0 / (double)(hi - lo));
    }
    return bad;
}

// first row whose first edge is at or after edge position e
uint64_t row_at(const uint64_t* off, uint64_t n, uint64_t e) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (off[mid] < e)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

}  // namespace

#if defined(__x86_64__)
namespace {
__attribute__((target("avx2"))) void copy_nt_avx2(char* dst, const char* src, size_t bytes) {
    size_t i = 0;
    for (; i + 128 <= bytes; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    _mm_sfence();
    if (i < bytes) std::memcpy(dst + i, src + i, bytes - i);
}
}  // namespace
#endif

// Pageable -> pinned staging copy of the upload path: memcpy, or (A/B knob) non-temporal stores,
// which save the read-for-ownership of the slot's lines but bypass the cache the DMA could read
// the slot from.
void staging_copy(void* dst, const void* src, size_t bytes) {
#if defined(__x86_64__)
    static const bool avx2 = [] {
        // HSAW_UPLOAD_NT=1 turns the non-temporal form on. Measured beside the in_cum check at
        // the Twitter shape (ms per upload call, 2 / 4 MB ring slots): plain memcpy 253 / 295,
        // non-temporal 276 / 283 - with 2 MB slots the ring stays in the last-level cache and
        // the DMA reads it from there, which the cache-bypassing stores defeat. Off by default.
        const char* env = std::getenv("HSAW_UPLOAD_NT");
        return env && std::atoi(env) != 0 && __builtin_cpu_supports("avx2");
    }();
    if (avx2 && (reinterpret_cast<uintptr_t>(dst) & 31u) == 0 && bytes >= 4096) {
        copy_nt_avx2(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
        return;
    }
#endif
    std::memcpy(dst, src, bytes);
}

// off: n + 1 non-decreasing offsets (checked by the caller), cum: off[n] doubles.
//
// The array is cut into row-aligned chunks of ~edges_per_chunk elements on one work list with two
// ends: check workers claim chunks from the front, the uploader - once the other arrays are on
// the wire - claims runs of chunks from the back and simply copies them. So the split between
// "verified, regenerated on the device" and "copied" follows whatever the host cores and the link
// manage at that moment (an idle 16-core box verifies everything beside the other copies; a busy
// one leaves the tail to PCIe), and no rate has to be guessed in advance.
RowCheck::RowCheck(uint32_t n, const uint64_t* off, const double* cum, uint64_t edges_per_chunk)
    : n_(n), off_(off), cum_(cum) {
    const uint64_t m = off[n];
    const uint64_t per = std::max<uint64_t>(edges_per_chunk, 1);
    const uint64_t chunks = std::max<uint64_t>(1, std::min<uint64_t>((m + per - 1) / per, 1u << 20));
    rows_.resize(chunks + 1);
    for (uint64_t c = 0; c < chunks; ++c) rows_[c] = c == 0 ? 0 : row_at(off, n, m / chunks * c);
    rows_[chunks] = n;
    ends_.store(chunks);  // front 0 (high half), back = chunks (low half)
#if defined(__x86_64__)
    avx2_ = __builtin_cpu_supports("avx2");
#endif
}

bool RowCheck::claim_front(uint64_t* c) {
    uint64_t e = ends_.load(std::memory_order_relaxed);
    for (;;) {
        const uint64_t front = e >> 32, back = e & 0xFFFFFFFFu;
        if (front >= back) return false;
        if (ends_.compare_exchange_weak(e, ((front + 1) << 32) | back, std::memory_order_acq_rel)) {
            *c = front;
            return true;
        }
    }
}

bool RowCheck::claim_back(uint32_t max_chunks, uint64_t* e0, uint64_t* e1) {
    uint64_t e = ends_.load(std::memory_order_relaxed);
    for (;;) {
        const uint64_t front = e >> 32, back = e & 0xFFFFFFFFu;
        if (front >= back || max_chunks == 0) return false;
        // near the end leave the workers something to do: at most half of what is left
        const uint64_t take = std::max<uint64_t>(1, std::min<uint64_t>(max_chunks, (back - front + 1) / 2));
        if (ends_.compare_exchange_weak(e, (front << 32) | (back - take), std::memory_order_acq_rel)) {
            *e0 = off_[rows_[back - take]];
            *e1 = off_[rows_[back]];
            return true;
        }
    }
}

void RowCheck::work() {
    uint64_t c;
    while (!differs_.load(std::memory_order_relaxed) && claim_front(&c)) {
        const uint64_t va = rows_[c], vb = rows_[c + 1];
#if defined(__x86_64__)
        const uint64_t bad = avx2_ ? rows_avx2(off_, cum_, va, vb, differs_)
                                   : rows_plain(off_, cum_, va, vb, differs_);
#else
        const uint64_t bad = rows_plain(off_, cum_, va, vb, differs_);
#endif
        if (bad) differs_.store(true, std::memory_order_relaxed);
        checked_.fetch_add(off_[vb] - off_[va], std::memory_order_relaxed);
    }
}

void RowCheck::run(unsigned threads) {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back([this] { work(); });
    work();
    for (auto& th : pool) th.join();
}

// The whole array through the check (tests, tools).
bool rows_are_indegree_sums(uint32_t n, const uint64_t* off, const double* cum, unsigned threads) {
    RowCheck check(n, off, cum, 1u << 21);
    check.run(threads ? threads : 1);
    return !check.differs();
}

}  // namespace hsawgpu
