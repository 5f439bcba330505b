// Device build of the in-CSR from an edge list: the step before the sampling path (SURVEY.md §8f,
// row 1). Replaces build_graph (proj/src/graph.cpp:112-199) for WeightMode::Given and ::InDegree:
// canonical order by (target, source), edge id = CSR position, per-row SEQUENTIAL FP64 cumulative
// sums (so in_cum is bit-identical to the reference's), and the reference's data errors with its
// own messages. WeightMode::RandomNormalized draws one global xorshift stream over all edges in
// row order and stays on the host.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

using namespace hsawgpu;

namespace {

constexpr double kInSumTolerance = 1e-12;  // proj/src/graph.cpp:19
constexpr uint32_t kNone = 0xFFFFFFFFu;

// error slots (u32, atomicMin): first offending input edge / sorted position / node
enum { E_INPUT = 0, E_DUP = 1, E_SUM = 2, E_MONO = 3, E_COUNT = 4 };

// (target << 32 | source) keys, input index as payload, and the per-edge input checks of
// proj/src/graph.cpp:115-123 (endpoint range, self-loop, Given weight in (0,1]).
__global__ void edge_keys(uint64_t ne, uint32_t n, const uint32_t* __restrict__ u,
                          const uint32_t* __restrict__ v, const double* __restrict__ w,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                          uint32_t* __restrict__ err) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    uint32_t a = u[i], b = v[i];
    bool bad = a >= n || b >= n || a == b;
    if (w) {
        double x = w[i];
        bad = bad || !(x > 0.0) || x > 1.0;
    }
    if (bad) atomicMin(err + E_INPUT, (uint32_t)i);
    keys[i] = ((uint64_t)b << 32) | a;
    vals[i] = (uint32_t)i;
}

// Sorted keys -> in_src / edge_dst, duplicate detection (graph.cpp:129-134) and row offsets: the
// edge at a row boundary writes the offsets of its own row and of the empty rows before it.
__global__ void split_sorted(uint64_t ne, uint32_t n, const uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ in_src, uint32_t* __restrict__ edge_dst,
                             uint64_t* __restrict__ off, uint32_t* __restrict__ err) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    uint64_t k = keys[i];
    uint32_t dst = (uint32_t)(k >> 32);
    in_src[i] = (uint32_t)k;
    if (edge_dst) edge_dst[i] = dst;
    if (dst >= n) return;  // out-of-range input: reported from E_INPUT, keep the writes in bounds
    if (i == 0) {
        for (uint32_t x = 0; x <= dst; ++x) off[x] = 0;
    } else {
        uint64_t kp = keys[i - 1];
        if (kp == k) atomicMin(err + E_DUP, (uint32_t)i);
        uint32_t pd = (uint32_t)(kp >> 32);
        for (uint32_t x = pd + 1; x <= dst; ++x) off[x] = i;
    }
    if (i == ne - 1)
        for (uint64_t x = (uint64_t)dst + 1; x <= n; ++x) off[x] = ne;
}

__global__ void fill_offsets(uint64_t count, uint64_t value, uint64_t* __restrict__ off) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) off[i] = value;
}

// One thread per row: weights and the sequential cumulative sum, exactly the loops of
// graph.cpp:153-179 (Given: weight of the sorted edge; InDegree: 1.0 / d added d times), plus the
// row checks of build_graph (Given: sum > 1 + 1e-12) and validate() (:93, :100-102).
__global__ void row_weights(uint32_t n, const uint64_t* __restrict__ off,
                            const uint32_t* __restrict__ vals, const double* __restrict__ w_in,
                            double* __restrict__ in_cum, double* __restrict__ weight,
                            uint32_t* __restrict__ err) {
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint64_t lo = off[v], hi = off[v + 1];
    if (hi <= lo) return;
    const double wd = 1.0 / (double)(hi - lo);
    double cum = 0.0;
    bool mono = true;
    for (uint64_t i = lo; i < hi; ++i) {
        const double w = w_in ? w_in[vals[i]] : wd;
        const double next = cum + w;
        if (!(next > cum)) mono = false;  // validate(): "cumulative weights not increasing"
        cum = next;
        in_cum[i] = cum;
        if (weight) weight[i] = w;
    }
    if (cum > 1.0 + kInSumTolerance) atomicMin(err + E_SUM, v);
    if (!mono) atomicMin(err + E_MONO, v);
}

std::string d2s(double x) { return std::to_string(x); }  // "%f", as the reference's messages

}  // namespace

namespace hsawgpu {

struct DeviceCsr {
    DevVec<uint64_t> off;
    DevVec<uint32_t> src, dst, vals;
    DevVec<double> cum, weight, w_in;
};

// Builds the CSR on the device. want_aux: also produce weight[] and edge_dst[]. When `src_out` is
// given the sorted sources are written there (the compact layout's own array) instead of csr.src.
// Throws HSAW_EDATA with the reference's message on bad input.
// on_device: edge_u / edge_v / edge_w are device arrays already (the text parser's output); they are
// used in place and single elements are copied back only to word an error.
void build_device_csr(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                      const uint32_t* edge_v, const double* edge_w, int weight_mode, bool want_aux,
                      uint32_t* src_out, DeviceCsr& csr, bool on_device = false) {
    if (n == 0) fail(HSAW_EDATA, "graph: no nodes");
    if (ne > 0xFFFFFFFEull) fail(HSAW_EINVAL, "build: edge ids are 32-bit (types.hpp:10)");
    if (weight_mode != 0 && weight_mode != 1)
        fail(HSAW_EINVAL, "build: only WeightMode::Given (0) and ::InDegree (1) are built on the device");
    if (ne && (!edge_u || !edge_v)) fail(HSAW_EINVAL, "build: null edge array");
    const bool given = weight_mode == 0;
    if (given && ne && !edge_w) fail(HSAW_EINVAL, "build: WeightMode::Given needs edge weights");
    cudaStream_t st = ctx->stream;
    const uint64_t cap = ne ? ne : 1;

    DevVec<uint32_t> d_u, d_v;
    DevVec<uint64_t> keys_in, keys_out;
    DevVec<uint32_t> vals_in;
    if (!on_device) {
        d_u.ensure_scratch(cap);
        d_v.ensure_scratch(cap);
    }
    keys_in.ensure_scratch(cap);
    keys_out.ensure_scratch(cap);
    vals_in.ensure_scratch(cap);
    csr.vals.ensure_scratch(cap);
    csr.off.ensure_scratch((uint64_t)n + 1);
    csr.cum.ensure_scratch(cap);
    if (!src_out) csr.src.ensure_scratch(cap);
    if (want_aux) {
        csr.weight.ensure_scratch(cap);
        csr.dst.ensure_scratch(cap);
    }
    if (given && !on_device) csr.w_in.ensure_scratch(cap);
    uint32_t* d_err = reinterpret_cast<uint32_t*>(ctx->d_scalars + 56);
    HSAW_CUDA_CHECK(cudaMemsetAsync(d_err, 0xFF, E_COUNT * 4, st));

    if (ne == 0) {
        fill_offsets<<<(unsigned)(((uint64_t)n + 1 + 255) / 256), 256, 0, st>>>((uint64_t)n + 1, 0,
                                                                                csr.off.p);
        check_launch(ctx, "fill_offsets");
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        return;
    }

    const uint32_t* in_u = edge_u;
    const uint32_t* in_v = edge_v;
    const double* in_w = given ? edge_w : nullptr;
    if (!on_device) {
        std::vector<CopyJob> jobs{{d_u.p, edge_u, ne * 4}, {d_v.p, edge_v, ne * 4}};
        if (given) jobs.push_back({csr.w_in.p, edge_w, ne * 8});
        copy_to_device(ctx, jobs);
        in_u = d_u.p;
        in_v = d_v.p;
        in_w = given ? csr.w_in.p : nullptr;
    }
    {
        StageScope timer(ctx, HSAW_STAGE_UPLOAD);
        const unsigned eb = (unsigned)((ne + 255) / 256);
        edge_keys<<<eb, 256, 0, st>>>(ne, n, in_u, in_v, in_w, keys_in.p, vals_in.p, d_err);
        check_launch(ctx, "edge_keys");
        int node_bits = 32 - __builtin_clz(n > 1 ? n - 1 : 1);
        int end_bit = std::min(64, 32 + node_bits);
        size_t bytes = 0;
        HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in.p, keys_out.p,
                                                        vals_in.p, csr.vals.p, (int64_t)ne, 0,
                                                        end_bit, st));
        ctx->cub_tmp.ensure_scratch(bytes ? bytes : 1);
        HSAW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, bytes, keys_in.p,
                                                        keys_out.p, vals_in.p, csr.vals.p,
                                                        (int64_t)ne, 0, end_bit, st));
        ++ctx->launches;
        split_sorted<<<eb, 256, 0, st>>>(ne, n, keys_out.p, src_out ? src_out : csr.src.p,
                                         want_aux ? csr.dst.p : nullptr, csr.off.p, d_err);
        check_launch(ctx, "split_sorted");
    }
    // input errors first (build_graph checks them before sorting); rows are only summed for
    // well-formed input, so the offsets are valid when row_weights runs
    uint32_t err[E_COUNT];
    HSAW_CUDA_CHECK(cudaMemcpyAsync(err, d_err, sizeof(err), cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    if (err[E_INPUT] != kNone) {
        const uint64_t i = err[E_INPUT];
        uint32_t a = 0, b = 0;
        double wi = 0.0;
        if (on_device) {
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&a, in_u + i, 4, cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaMemcpyAsync(&b, in_v + i, 4, cudaMemcpyDeviceToHost, st));
            if (in_w) HSAW_CUDA_CHECK(cudaMemcpyAsync(&wi, in_w + i, 8, cudaMemcpyDeviceToHost, st));
            HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        } else {
            a = edge_u[i];
            b = edge_v[i];
            if (given) wi = edge_w[i];
        }
        if (a >= n || b >= n) fail(HSAW_EDATA, "edge endpoint out of range");
        if (a == b)
            fail(HSAW_EDATA, "self-loop " + std::to_string(a) + " -> " + std::to_string(b));
        fail(HSAW_EDATA, "weight " + d2s(wi) + " out of (0,1] on edge " +
                             std::to_string(a) + " -> " + std::to_string(b));
    }
    if (err[E_DUP] != kNone) {
        uint64_t key = 0;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&key, keys_out.p + err[E_DUP], 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        fail(HSAW_EDATA, "duplicate edge " + std::to_string((uint32_t)key) + " -> " +
                             std::to_string((uint32_t)(key >> 32)));
    }
    {
        StageScope timer(ctx, HSAW_STAGE_UPLOAD);
        row_weights<<<(n + 127) / 128, 128, 0, st>>>(n, csr.off.p, csr.vals.p,
                                                     in_w, csr.cum.p,
                                                     want_aux ? csr.weight.p : nullptr, d_err);
        check_launch(ctx, "row_weights");
    }
    HSAW_CUDA_CHECK(cudaMemcpyAsync(err, d_err, sizeof(err), cudaMemcpyDeviceToHost, st));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    auto row_total = [&](uint32_t v) {
        uint64_t hi = 0;
        double tot = 0.0;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&hi, csr.off.p + v + 1, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&tot, csr.cum.p + hi - 1, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        return tot;
    };
    if (given) {
        // build_graph's own check runs over all rows before validate() (graph.cpp:163-165)
        if (err[E_SUM] != kNone)
            fail(HSAW_EDATA, "in-weight sum " + d2s(row_total(err[E_SUM])) + " > 1 at node " +
                                 std::to_string(err[E_SUM]));
        if (err[E_MONO] != kNone)
            fail(HSAW_EDATA, "graph: cumulative weights not increasing at node " +
                                 std::to_string(err[E_MONO]));
    } else {
        // validate() walks the rows in order: within a row the per-edge check precedes the sum
        const uint32_t first = std::min(err[E_SUM], err[E_MONO]);
        if (first != kNone) {
            if (err[E_MONO] == first)
                fail(HSAW_EDATA, "graph: cumulative weights not increasing at node " +
                                     std::to_string(first));
            fail(HSAW_EDATA, "graph: in-weight sum " + d2s(row_total(first)) + " > 1 at node " +
                                 std::to_string(first));
        }
    }
}

void build_and_install(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                       const uint32_t* edge_v, const double* edge_w, int weight_mode,
                       const double* host_p_of, bool on_device) {
    release_graph(ctx);
    cudaStream_t st = ctx->stream;
    double* d_p = nullptr;
    try {
        if (n == 0) fail(HSAW_EDATA, "graph: no nodes");
        if (ne > 0xFFFFFFFEull) fail(HSAW_EINVAL, "build: edge ids are 32-bit (types.hpp:10)");
        prepare_layout(ctx, n, (uint32_t)ne);
        DeviceCsr csr;
        build_device_csr(ctx, n, ne, edge_u, edge_v, edge_w, weight_mode, false, nullptr, csr,
                         on_device);
        d_p = static_cast<double*>(pool_alloc((uint64_t)n * 8, st));
        if (host_p_of)
            HSAW_CUDA_CHECK(
                cudaMemcpyAsync(d_p, host_p_of, (uint64_t)n * 8, cudaMemcpyHostToDevice, st));
        else
            HSAW_CUDA_CHECK(cudaMemsetAsync(d_p, 0, (uint64_t)n * 8, st));
        install_graph(ctx, n, (uint32_t)ne, csr.off.p, csr.src.p, csr.cum.p, d_p);
    } catch (...) {
        if (d_p) cudaFreeAsync(d_p, st);
        release_graph(ctx);
        throw;
    }
    cudaFreeAsync(d_p, st);
    collect_timings(ctx);
}

}  // namespace hsawgpu

extern "C" {

int hsaw_gpu_csr_build(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                       const uint32_t* edge_v, const double* edge_w, int weight_mode,
                       uint64_t* out_in_offsets, uint32_t* out_in_src, double* out_in_cum,
                       double* out_weight, uint32_t* out_edge_dst) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!out_in_offsets || (ne && (!out_in_src || !out_in_cum)))
            fail(HSAW_EINVAL, "csr_build: null output array");
        DeviceCsr csr;
        const bool aux = out_weight || out_edge_dst;
        build_device_csr(ctx, n, ne, edge_u, edge_v, edge_w, weight_mode, aux, nullptr, csr);
        std::vector<CopyJob> jobs{{out_in_offsets, csr.off.p, ((uint64_t)n + 1) * 8}};
        if (ne) {
            jobs.push_back({out_in_src, csr.src.p, ne * 4});
            jobs.push_back({out_in_cum, csr.cum.p, ne * 8});
            if (out_weight) jobs.push_back({out_weight, csr.weight.p, ne * 8});
            if (out_edge_dst) jobs.push_back({out_edge_dst, csr.dst.p, ne * 4});
        }
        copy_to_host(ctx, jobs);
        collect_timings(ctx);
    });
}

int hsaw_gpu_graph_build_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                                const uint32_t* edge_v, const double* edge_w, int weight_mode,
                                const double* p_of) {
    if (!ctx) return HSAW_EINVAL;
    return guarded(ctx, [&] {
        if (!p_of) fail(HSAW_EINVAL, "graph_build_upload: null suspect array");
        build_and_install(ctx, n, ne, edge_u, edge_v, edge_w, weight_mode, p_of, false);
    });
}

}  // extern "C"
