// Edge-list text ingest on the device: the parsing and id-remap half of
// load_edge_list (proj/src/graph.cpp:29-59 parse_line, :201-241). The file goes up as bytes; one
// thread per line tokenises it the way `std::istringstream >> token` does (C-locale whitespace),
// reads the two ids and validates / converts the optional weight; raw ids are sorted, uniqued and
// replaced by their rank (the reference's "dense, ascending by raw id" map).
//
// The device parser implements the *plain* grammar only: unsigned decimal ids of at most 19 digits
// and weights of the form digits[.digits][(e|E)[+-]digits] with at most 19 significant digits in
// a safely normal range, converted with the Eisel-Lemire algorithm (correctly rounded, i.e. the
// double strtod / std::stod returns) or handed back when that algorithm cannot decide. Anything
// else a line may legally or illegally contain (signs, hex floats, inf/nan, overlong numbers,
// malformed lines, a missing weight in given-weight mode) is NOT guessed at: the first such line is
// reported and the host layer re-reads the file with its own reference-equivalent parser, which
// also words the errors. Results are therefore identical by construction on the plain grammar and
// by delegation elsewhere.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace hsawgpu {
namespace {

constexpr uint8_t kBlank = 0, kEdge = 1, kHost = 2;
constexpr uint64_t kNoLine = ~0ull;

struct Pow5 {
    uint64_t hi, lo;
};
__device__ const Pow5 kPow5[] = {
#include "pow5_table.inc"
};
constexpr int kSmallestPow5 = -342;

__device__ __forceinline__ bool is_space(unsigned char c) {  // isspace, "C" locale
    return c == ' ' || (c >= '\t' && c <= '\r');
}
__device__ __forceinline__ bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// Eisel-Lemire: w * 10^q (w != 0 exact, q the decimal exponent) -> correctly rounded binary64.
// Returns false when the value is outside the normal range handled here or the 128-bit product
// cannot decide the rounding; the caller then defers to the host's strtod.
__device__ bool decimal_to_double(uint64_t w, int q, double& out) {
    if (q < -300 || q > 280) return false;
    const int lz = __clzll((long long)w);
    w <<= lz;
    const Pow5 p = kPow5[q - kSmallestPow5];
    uint64_t lo = w * p.hi, hi = __umul64hi(w, p.hi);
    if ((hi & 0x1FFull) == 0x1FFull) {  // 64 - (52 + 3) low bits all set: refine with the low word
        const uint64_t second_hi = __umul64hi(w, p.lo);
        lo += second_hi;
        if (second_hi > lo) ++hi;
    }
    if (lo == ~0ull && (q < -27 || q > 55)) return false;
    const int upperbit = (int)(hi >> 63);
    const int shift = upperbit + 64 - 52 - 3;
    uint64_t mant = hi >> shift;
    int power2 = ((((152170 + 65536) * q) >> 16) + 63) + upperbit - lz + 1023;
    if (power2 <= 0) return false;  // subnormal: host
    if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 && (mant << shift) == hi)
        mant &= ~1ull;  // exactly half way with an even significand below: round down
    mant += mant & 1;
    mant >>= 1;
    if (mant >= (2ull << 52)) {
        mant = 1ull << 52;
        ++power2;
    }
    mant &= ~(1ull << 52);
    if (power2 >= 0x7FF) return false;
    out = __longlong_as_double((long long)(mant | ((uint64_t)power2 << 52)));
    return true;
}

// std::stoull on a plain token: all digits, at most 19 of them (always < 2^64).
__device__ bool parse_id(const char* t, uint32_t len, uint64_t& x) {
    if (len == 0 || len > 19) return false;
    uint64_t v = 0;
    for (uint32_t i = 0; i < len; ++i) {
        if (!is_digit(t[i])) return false;
        v = v * 10 + (uint64_t)(t[i] - '0');
    }
    x = v;
    return true;
}

// std::stod on a plain token. value_needed = false: only decide that stod would accept it.
__device__ bool parse_weight(const char* t, uint32_t len, bool value_needed, double& x) {
    uint64_t sig = 0;
    int nsig = 0, frac = 0;
    uint32_t i = 0;
    bool any = false, seen_dot = false;
    for (; i < len; ++i) {
        const unsigned char c = t[i];
        if (c == '.') {
            if (seen_dot) return false;
            seen_dot = true;
            continue;
        }
        if (!is_digit(c)) break;
        any = true;
        if (seen_dot) ++frac;
        if (sig == 0 && c == '0') continue;  // leading zeros carry no precision
        if (nsig == 19) return false;        // more significant digits than a u64 holds exactly
        sig = sig * 10 + (uint64_t)(c - '0');
        ++nsig;
    }
    if (!any) return false;
    int e10 = 0;
    if (i < len) {
        if (t[i] != 'e' && t[i] != 'E') return false;
        ++i;
        bool neg = false;
        if (i < len && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
        if (i >= len) return false;  // "1e": stod would stop before the 'e' -> trailing characters
        for (; i < len; ++i) {
            if (!is_digit(t[i])) return false;
            e10 = e10 * 10 + (t[i] - '0');
            if (e10 > 100000) return false;
        }
        if (neg) e10 = -e10;
    }
    if (sig == 0) {  // an exact zero of any spelling
        x = 0.0;
        return true;
    }
    const int q = e10 - frac;
    // |value| in [10^(q + nsig - 1), 10^(q + nsig)): keep well inside the normal range, where stod
    // neither overflows nor reports ERANGE for a subnormal result
    if (q + nsig < -290 || q + nsig > 290) return false;
    if (!value_needed) {
        x = 0.0;
        return true;
    }
    return decimal_to_double(sig, q, x);
}

struct LineStart {
    const char* text;
    __device__ bool operator()(uint64_t p) const { return p == 0 || text[p - 1] == '\n'; }
};

// parse_line (graph.cpp:29-59) for line i = [start[i], end) where end is the next line's start
// minus the newline, or the end of the text.
__global__ void parse_lines(const char* __restrict__ text, uint64_t bytes,
                            const uint64_t* __restrict__ start, uint64_t nlines,
                            int weight_required, int value_needed, uint8_t* __restrict__ kind,
                            uint64_t* __restrict__ eu, uint64_t* __restrict__ ev,
                            double* __restrict__ ew, unsigned long long* first_host_line) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nlines) return;
    const uint64_t s = start[i];
    uint64_t e = i + 1 < nlines ? start[i + 1] - 1 : bytes;
    if (i + 1 == nlines && e > s && text[e - 1] == '\n') --e;  // trailing newline of the file
    const char* t = text + s;
    const uint64_t len = e - s;
    uint64_t p = 0;
    uint64_t tok_at[4];
    uint32_t tok_len[4];
    int ntok = 0;
    bool too_many = false;
    while (p < len) {
        while (p < len && is_space(t[p])) ++p;
        if (p >= len) break;
        if (ntok == 0 && t[p] == '#') {  // comment line (first non-space character)
            kind[i] = kBlank;
            return;
        }
        const uint64_t b = p;
        while (p < len && !is_space(t[p])) ++p;
        if (ntok == 3 || p - b > 400) {
            too_many = true;
            break;
        }
        tok_at[ntok] = b;
        tok_len[ntok] = (uint32_t)(p - b);
        ++ntok;
    }
    if (ntok == 0 && !too_many) {
        kind[i] = kBlank;
        return;
    }
    uint64_t u = 0, v = 0;
    double w = 0.0;
    bool ok = !too_many && ntok >= 2;
    ok = ok && parse_id(t + tok_at[0], tok_len[0], u) && parse_id(t + tok_at[1], tok_len[1], v);
    if (ok && ntok == 3) ok = parse_weight(t + tok_at[2], tok_len[2], value_needed != 0, w);
    if (ok && ntok == 2 && weight_required) ok = false;  // the host words this error
    if (!ok) {
        kind[i] = kHost;
        atomicMin(first_host_line, (unsigned long long)i);
        return;
    }
    kind[i] = kEdge;
    eu[i] = u;
    ev[i] = v;
    ew[i] = w;
}

__global__ void count_newlines(const char* __restrict__ text, uint64_t bytes,
                               unsigned long long* total) {
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes;
         i += (uint64_t)gridDim.x * blockDim.x)
        c += text[i] == '\n';
    c = __reduce_add_sync(kFullMask, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

__global__ void edge_flags(const uint8_t* __restrict__ kind, uint64_t nlines, uint8_t* flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nlines) flag[i] = kind[i] == kEdge;
}

// edges in file order + the 2E raw ids for the remap
__global__ void gather_edges(const uint8_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                             uint64_t nlines, const uint64_t* __restrict__ lu,
                             const uint64_t* __restrict__ lv, const double* __restrict__ lw,
                             uint64_t ne, uint64_t* __restrict__ ids, double* __restrict__ w) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nlines || !flag[i]) return;
    const uint32_t k = pos[i];
    ids[k] = lu[i];
    ids[ne + k] = lv[i];
    w[k] = lw[i];
}

// rank of each raw id among the sorted distinct ids (graph.cpp:232-241)
__global__ void dense_ids(const uint64_t* __restrict__ ids, uint64_t count,
                          const uint64_t* __restrict__ sorted, uint64_t nids,
                          uint32_t* __restrict__ dense) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t x = ids[i];
    uint64_t a = 0, b = nids;
    while (a < b) {
        const uint64_t mid = a + (b - a) / 2;
        if (sorted[mid] < x)
            a = mid + 1;
        else
            b = mid;
    }
    dense[i] = (uint32_t)a;
}

}  // namespace
}  // namespace hsawgpu

using namespace hsawgpu;

// Parsed edge list resident on the device, handed to the caller by the fetch call.
struct hsaw_gpu_edge_text {
    hsaw_gpu_ctx* ctx = nullptr;
    uint64_t ne = 0, nids = 0;
    DevVec<uint32_t> dense;   // 2 * ne: dense u, then dense v
    DevVec<double> w;         // ne
    DevVec<uint64_t> sorted;  // nids raw ids ascending
};

extern "C" {

int hsaw_gpu_edge_text_parse(hsaw_gpu_ctx* ctx, const char* text, uint64_t bytes,
                             int weight_required, int weight_values, hsaw_gpu_edge_text** out,
                             uint64_t* nedges, uint64_t* nids, int* identity,
                             uint64_t* host_line) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!out || !nedges || !nids || !identity || !host_line)
            fail(HSAW_EINVAL, "edge_text_parse: null output");
        if (bytes && !text) fail(HSAW_EINVAL, "edge_text_parse: null text");
        *out = nullptr;
        *nedges = *nids = 0;
        *identity = 0;
        *host_line = 0;
        if (bytes == 0) return;
        cudaStream_t st = ctx->stream;
        DevVec<char> d_text;
        d_text.ensure_scratch(bytes + 1);
        copy_to_device(ctx, {{d_text.p, text, bytes}});

        // line starts
        DevVec<uint64_t> start;
        uint64_t* d_n = ctx->d_scalars + 24;
        {
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_n, 0, 8, st));
            const unsigned grid = (unsigned)std::min<uint64_t>((bytes + 255) / 256,
                                                               (uint64_t)ctx->sm_count * 16);
            count_newlines<<<grid, 256, 0, st>>>(d_text.p, bytes,
                                                 reinterpret_cast<unsigned long long*>(d_n));
            check_launch(ctx, "count_newlines");
            uint64_t newlines = 0;
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&newlines, d_n, 8, cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            start.ensure_scratch(newlines + 1);
        }
        thrust::counting_iterator<uint64_t> positions(0);
        LineStart pred{d_text.p};
        size_t tmp = 0;
        HSAW_CUDA_CHECK(cub::DeviceSelect::If(nullptr, tmp, positions, start.p, d_n, (int64_t)bytes,
                                              pred, st));
        ctx->cub_tmp.ensure_scratch(tmp ? tmp : 1);
        {
            StageScope timer(ctx, HSAW_STAGE_UPLOAD);
            HSAW_CUDA_CHECK(cub::DeviceSelect::If(ctx->cub_tmp.p, tmp, positions, start.p, d_n,
                                                  (int64_t)bytes, pred, st));
            ++ctx->launches;
        }
        uint64_t nlines = 0;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&nlines, d_n, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        if (nlines > 0xFFFFFFF0ull) fail(HSAW_EINVAL, "edge_text_parse: more than 2^32 lines");

        // per-line parse
        DevVec<uint8_t> kind, flag;
        DevVec<uint64_t> lu, lv;
        DevVec<double> lw;
        DevVec<uint32_t> pos;
        kind.ensure_scratch(nlines);
        flag.ensure_scratch(nlines);
        lu.ensure_scratch(nlines);
        lv.ensure_scratch(nlines);
        lw.ensure_scratch(nlines);
        pos.ensure_scratch(nlines);
        unsigned long long* d_first = reinterpret_cast<unsigned long long*>(ctx->d_scalars + 25);
        HSAW_CUDA_CHECK(cudaMemsetAsync(d_first, 0xFF, 8, st));
        const unsigned lb = (unsigned)((nlines + 127) / 128);
        {
            StageScope timer(ctx, HSAW_STAGE_UPLOAD);
            parse_lines<<<lb, 128, 0, st>>>(d_text.p, bytes, start.p, nlines, weight_required,
                                            weight_values, kind.p, lu.p, lv.p, lw.p, d_first);
            check_launch(ctx, "parse_lines");
            edge_flags<<<(unsigned)((nlines + 255) / 256), 256, 0, st>>>(kind.p, nlines, flag.p);
            check_launch(ctx, "edge_flags");
        }
        exclusive_sum_u8_to_u32(ctx, flag.p, pos.p, nlines);
        uint64_t first = kNoLine;
        uint32_t last_pos = 0;
        uint8_t last_flag = 0;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&last_pos, pos.p + (nlines - 1), 4, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&last_flag, flag.p + (nlines - 1), 1, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        if (first != kNoLine) {  // a line outside the plain grammar: the host parser takes over
            *host_line = first + 1;
            collect_timings(ctx);
            return;
        }
        const uint64_t ne = (uint64_t)last_pos + last_flag;
        *nedges = ne;
        if (ne == 0) {
            collect_timings(ctx);
            return;
        }

        // raw ids -> dense ids
        auto* el = new hsaw_gpu_edge_text;
        try {
            el->ctx = ctx;
            el->ne = ne;
            DevVec<uint64_t> ids, ids_sorted;
            ids.ensure_scratch(2 * ne);
            ids_sorted.ensure_scratch(2 * ne);
            el->w.ensure_scratch(ne);
            el->dense.ensure_scratch(2 * ne);
            el->sorted.ensure_scratch(2 * ne);
            StageScope timer(ctx, HSAW_STAGE_UPLOAD);
            gather_edges<<<(unsigned)((nlines + 255) / 256), 256, 0, st>>>(
                flag.p, pos.p, nlines, lu.p, lv.p, lw.p, ne, ids.p, el->w.p);
            check_launch(ctx, "gather_edges");
            size_t t1 = 0, t2 = 0;
            HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, t1, ids.p, ids_sorted.p,
                                                           (int64_t)(2 * ne), 0, 64, st));
            HSAW_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, t2, ids_sorted.p, el->sorted.p, d_n,
                                                      (int64_t)(2 * ne), st));
            ctx->cub_tmp.ensure_scratch(std::max(t1, t2) + 1);
            HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ctx->cub_tmp.p, t1, ids.p, ids_sorted.p,
                                                           (int64_t)(2 * ne), 0, 64, st));
            HSAW_CUDA_CHECK(cub::DeviceSelect::Unique(ctx->cub_tmp.p, t2, ids_sorted.p,
                                                      el->sorted.p, d_n, (int64_t)(2 * ne), st));
            ctx->launches += 2;
            uint64_t n_ids = 0;
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&n_ids, d_n, 8, cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            el->nids = n_ids;
            uint64_t largest = 0;
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&largest, el->sorted.p + (n_ids - 1), 8,
                                            cudaMemcpyDeviceToHost, st));
            dense_ids<<<(unsigned)((2 * ne + 255) / 256), 256, 0, st>>>(ids.p, 2 * ne, el->sorted.p,
                                                                        n_ids, el->dense.p);
            check_launch(ctx, "dense_ids");
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
            *nids = n_ids;
            *identity = largest == n_ids - 1;  // graph.cpp:236
        } catch (...) {
            delete el;
            throw;
        }
        collect_timings(ctx);
        *out = el;
    });
}

int hsaw_gpu_edge_text_fetch(hsaw_gpu_edge_text* el, uint32_t* edge_u, uint32_t* edge_v,
                             double* edge_w, uint64_t* raw_ids) {
    if (!el) return HSAW_EINVAL;
    return guarded(el->ctx, [&] {
        std::vector<CopyJob> jobs;
        if (edge_u) jobs.push_back({edge_u, el->dense.p, el->ne * 4});
        if (edge_v) jobs.push_back({edge_v, el->dense.p + el->ne, el->ne * 4});
        if (edge_w) jobs.push_back({edge_w, el->w.p, el->ne * 8});
        if (raw_ids) jobs.push_back({raw_ids, el->sorted.p, el->nids * 8});
        if (!jobs.empty()) copy_to_host(el->ctx, jobs);
    });
}

int hsaw_gpu_edge_text_install(hsaw_gpu_edge_text* el, int weight_mode, const double* p_of) {
    if (!el) return HSAW_EINVAL;
    return guarded(el->ctx, [&] {
        if (el->nids > 0xFFFFFFFEull) fail(HSAW_EINVAL, "edge_text_install: node ids are 32-bit");
        build_and_install(el->ctx, (uint32_t)el->nids, el->ne, el->dense.p, el->dense.p + el->ne,
                          weight_mode == 0 ? el->w.p : nullptr, weight_mode, p_of, true);
    });
}

void hsaw_gpu_edge_text_free(hsaw_gpu_edge_text* el) {
    if (!el) return;
    cudaSetDevice(el->ctx->device);
    current_stream() = el->ctx->stream;
    delete el;
}

}  // extern "C"
