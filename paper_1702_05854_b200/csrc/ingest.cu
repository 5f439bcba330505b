// Binary ingest on the device: the body of an HSAW1 cache file
// (save_cache / load_cache, proj/src/graph.cpp:383-430) is uploaded as it lies on disk and decoded
// by kernels: little-endian u64 offsets, u64-widened sources, weight bit patterns; then the
// per-row sequential cumulative sums and edge_dst of load_cache (:417-424) and the checks of
// ProbGraph::validate() (:70-104), one thread per row. The host only parses the 21-byte header.
//
// Errors: the kernels find the FIRST offending row; the host copies that one row back and replays
// validate()'s checks on it in the reference's order, so the DataError message is the reference's.
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"

namespace hsawgpu {
namespace {

constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr double kInSumTolerance = 1e-12;  // proj/include/hsaw/graph.hpp (validate, :100)

// body: (n + 1) offsets, m sources (u64 each), m weights (f64 bit patterns), all little endian.
__global__ void decode_cache(const uint64_t* __restrict__ body, uint32_t n, uint32_t m,
                             uint64_t* __restrict__ off, uint32_t* __restrict__ src,
                             double* __restrict__ weight) {
    const uint64_t total = (uint64_t)n + 1 + 2ull * m;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = body[i];
        if (i <= n)
            off[i] = x;
        else if (i <= (uint64_t)n + m)
            src[i - n - 1] = (uint32_t)x;  // static_cast<NodeId>(get_u64(f)), graph.cpp:411
        else
            weight[i - n - 1 - m] = __longlong_as_double((long long)x);
    }
}

// One thread per row: cum += weight (graph.cpp:419-423), edge_dst, and whether validate() would
// object to anything in the row. err[0] = first row with unusable offsets, err[1] = first row
// failing a check of validate().
__global__ void cache_rows(uint32_t n, uint32_t m, const uint64_t* __restrict__ off,
                           const uint32_t* __restrict__ src, const double* __restrict__ weight,
                           double* __restrict__ in_cum, uint32_t* __restrict__ edge_dst,
                           uint32_t* __restrict__ err) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint64_t lo = off[v], hi = off[v + 1];
    if (hi < lo || hi > m) {
        atomicMin(err + 0, v);
        return;
    }
    double cum = 0.0;
    bool bad = false;
    uint32_t prev_u = 0;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint32_t u = src[i];
        const double w = weight[i];
        const double next = cum + w;
        bad |= u >= n || u == v || (i > lo && u <= prev_u);
        bad |= !(w > 0.0) || w > 1.0;
        bad |= !(next > cum);
        prev_u = u;
        cum = next;
        in_cum[i] = cum;
        if (edge_dst) edge_dst[i] = v;
    }
    bad |= hi > lo && cum > 1.0 + kInSumTolerance;
    if (bad) atomicMin(err + 1, v);
}

std::string d2s(double x) { return std::to_string(x); }  // "%f", as the reference's messages

struct DecodedCache {
    DevVec<uint64_t> body, off;
    DevVec<uint32_t> src, dst;
    DevVec<double> weight, cum;
};

// validate() on one row, in the reference's order (graph.cpp:79-103); throws on the first failure.
void replay_row(uint32_t v, uint32_t n, uint64_t lo, const std::vector<uint32_t>& src,
                const std::vector<double>& weight) {
    double prev_cum = 0.0;
    for (size_t k = 0; k < src.size(); ++k) {
        const uint32_t u = src[k];
        if (u >= n) fail(HSAW_EDATA, "graph: source id out of range");
        if (u == v) fail(HSAW_EDATA, "graph: self-loop on node " + std::to_string(v));
        if (k > 0 && src[k] <= src[k - 1])
            fail(HSAW_EDATA,
                 "graph: in-adjacency not sorted / duplicate edge into " + std::to_string(v));
        const double w = weight[k];
        if (!(w > 0.0) || w > 1.0)
            fail(HSAW_EDATA, "graph: weight out of (0,1] on edge " + std::to_string(lo + k));
        const double cum = prev_cum + w;
        if (!(cum > prev_cum))
            fail(HSAW_EDATA, "graph: cumulative weights not increasing at node " + std::to_string(v));
        prev_cum = cum;
    }
    if (!src.empty() && prev_cum > 1.0 + kInSumTolerance)
        fail(HSAW_EDATA,
             "graph: in-weight sum " + d2s(prev_cum) + " > 1 at node " + std::to_string(v));
}

void decode_on_device(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const void* body, bool want_dst,
                      DecodedCache& c) {
    if (n == 0) fail(HSAW_EDATA, "graph: offsets do not cover edge range");
    if (!body) fail(HSAW_EINVAL, "cache: null body");
    cudaStream_t st = ctx->stream;
    const uint64_t words = (uint64_t)n + 1 + 2ull * m;
    c.body.ensure_scratch(words);
    c.off.ensure_scratch((uint64_t)n + 1);
    c.src.ensure_scratch(std::max<uint32_t>(m, 1));
    c.weight.ensure_scratch(std::max<uint32_t>(m, 1));
    c.cum.ensure_scratch(std::max<uint32_t>(m, 1));
    if (want_dst) c.dst.ensure_scratch(std::max<uint32_t>(m, 1));
    copy_to_device(ctx, {{c.body.p, body, words * 8}});
    uint32_t* d_err = reinterpret_cast<uint32_t*>(ctx->d_scalars + 16);
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_err, 0xFF, 8, st));
    {
        StageScope timer(ctx, HSAW_STAGE_UPLOAD);
        const unsigned grid = (unsigned)std::min<uint64_t>((words + 255) / 256,
                                                           (uint64_t)ctx->sm_count * 16);
        decode_cache<<<grid, 256, 0, st>>>(c.body.p, n, m, c.off.p, c.src.p, c.weight.p);
        check_launch(ctx, "decode_cache");
        cache_rows<<<(n + 127) / 128, 128, 0, st>>>(n, m, c.off.p, c.src.p, c.weight.p, c.cum.p,
                                                    want_dst ? c.dst.p : nullptr, d_err);
        check_launch(ctx, "cache_rows");
    }
    uint32_t err[2];
    uint64_t ends[2];
    HSAW_CUDA_CHECK(cudaMemcpyAsync(err, d_err, 8, cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaMemcpyAsync(&ends[0], c.off.p, 8, cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaMemcpyAsync(&ends[1], c.off.p + n, 8, cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    // validate()'s order (graph.cpp:76-103): coverage of the edge range first, then the rows in
    // ascending order, where a row whose offsets run backwards (or past m: the reference's loader
    // would have read out of bounds there) is "not monotone" and any other defect is replayed on
    // the host to get the reference's wording - whichever row comes first
    if (ends[0] != 0 || ends[1] != m) fail(HSAW_EDATA, "graph: offsets do not cover edge range");
    if (err[0] != kNoRow && (err[1] == kNoRow || err[0] <= err[1]))
        fail(HSAW_EDATA, "graph: offsets not monotone");
    if (err[1] != kNoRow) {
        const uint32_t v = err[1];
        uint64_t lohi[2];
        HSAW_CUDA_CHECK(cudaMemcpyAsync(lohi, c.off.p + v, 16, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        const uint64_t d = lohi[1] - lohi[0];
        std::vector<uint32_t> rs(d);
        std::vector<double> rw(d);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(rs.data(), c.src.p + lohi[0], d * 4, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(rw.data(), c.weight.p + lohi[0], d * 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        replay_row(v, n, lohi[0], rs, rw);
        fail(HSAW_EDATA, "graph: row " + std::to_string(v) + " rejected by the device check only");
    }
}

}  // namespace
}  // namespace hsawgpu

using namespace hsawgpu;

extern "C" {

int hsaw_gpu_cache_decode(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const void* body,
                          uint64_t* out_in_offsets, uint32_t* out_in_src, double* out_in_cum,
                          double* out_weight, uint32_t* out_edge_dst) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!out_in_offsets || (m && (!out_in_src || !out_in_cum)))
            fail(HSAW_EINVAL, "cache_decode: null output array");
        DecodedCache c;
        decode_on_device(ctx, n, m, body, out_edge_dst != nullptr, c);
        std::vector<CopyJob> jobs{{out_in_offsets, c.off.p, ((uint64_t)n + 1) * 8}};
        if (m) {
            jobs.push_back({out_in_src, c.src.p, (uint64_t)m * 4});
            jobs.push_back({out_in_cum, c.cum.p, (uint64_t)m * 8});
            if (out_weight) jobs.push_back({out_weight, c.weight.p, (uint64_t)m * 8});
            if (out_edge_dst) jobs.push_back({out_edge_dst, c.dst.p, (uint64_t)m * 4});
        }
        copy_to_host(ctx, jobs);
        collect_timings(ctx);
    });
}

int hsaw_gpu_graph_cache_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const void* body,
                                const double* p_of) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        release_graph(ctx);
        cudaStream_t st = ctx->stream;
        double* d_p = nullptr;
        try {
            if (n == 0) fail(HSAW_EDATA, "graph: offsets do not cover edge range");
            prepare_layout(ctx, n, m);
            DecodedCache c;
            decode_on_device(ctx, n, m, body, false, c);
            d_p = static_cast<double*>(pool_alloc((uint64_t)n * 8, st));
            if (p_of)
                HSAW_CUDA_CHECK(cudaMemcpyAsync(d_p, p_of, (uint64_t)n * 8, cudaMemcpyHostToDevice, st));
            else
                HSAW_CUDA_CHECK(cudaMemsetAsync(d_p, 0, (uint64_t)n * 8, st));
            install_graph(ctx, n, m, c.off.p, c.src.p, c.cum.p, d_p);
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));  // c's buffers are released on return
        } catch (...) {
            if (d_p) cudaFreeAsync(d_p, st);
            release_graph(ctx);
            throw;
        }
        cudaFreeAsync(d_p, st);
        collect_timings(ctx);
    });
}

}  // extern "C"
