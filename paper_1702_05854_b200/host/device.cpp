// Device-backed halves of the reference interface: everything here forwards to the C-ABI of
// include/hsaw_gpu.h and rethrows its status codes as the exception types the reference uses
// (std::invalid_argument / DataError / SamplingError / std::out_of_range), so callers and the CLI
// keep the reference's error behaviour (proj/src/cli.cpp:520-538).
#include <chrono>
#include <cstdio>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <fstream>

#include "hsaw_b200.hpp"
#include "hsaw_gpu.h"

namespace hsaw {

namespace {

void raise(int status, hsaw_gpu_ctx* ctx, const char* where) {
    if (status == HSAW_OK) return;
    std::string msg = std::string(where) + ": " + hsaw_gpu_last_error(ctx);
    switch (status) {
        case HSAW_EINVAL: throw std::invalid_argument(msg);
        case HSAW_EDATA: throw DataError(msg);
        case HSAW_EBUDGET: throw SamplingError(msg);
        case HSAW_ERANGE: throw std::out_of_range(msg);
        default: throw DeviceError(msg);
    }
}

hsaw_sampler_cfg to_c(const SamplerConfig& cfg) {
    hsaw_sampler_cfg c{};
    c.heuristic = cfg.heuristic == CycleHeuristic::Brent   ? 0
                  : cfg.heuristic == CycleHeuristic::Floyd ? 1
                                                           : 2;
    c.window = cfg.window;
    c.batch_size = cfg.batch_size;
    c.max_attempts = cfg.max_attempts;
    c.rng_mode = cfg.rng == WalkRng::PhiloxPerWalk ? 1u : 0u;
    return c;
}

// flat export -> vector<HsawSample>
std::vector<HsawSample> unpack(std::uint64_t count, const std::vector<std::uint64_t>& edge_off,
                               const std::vector<std::uint32_t>& nodes,
                               const std::vector<std::uint32_t>& edges) {
    std::vector<HsawSample> out(count);
    for (std::uint64_t w = 0; w < count; ++w) {
        const std::uint64_t a = edge_off[w], b = edge_off[w + 1];
        out[w].nodes.assign(nodes.begin() + a + w, nodes.begin() + b + w + 1);
        out[w].edge_ids.assign(edges.begin() + a, edges.begin() + b);
    }
    return out;
}

}  // namespace

// ---- build_graph on the device -------------------------------------------------------------------
ProbGraph build_graph_device(NodeId n, std::uint64_t nedges, const NodeId* u, const NodeId* v,
                             const double* w, WeightMode mode, int device) {
    if (mode == WeightMode::RandomNormalized)
        throw std::invalid_argument("build_graph_device: RandomNormalized is built on the host");
    hsaw_gpu_ctx* ctx = nullptr;
    if (hsaw_gpu_ctx_create(device, nullptr, &ctx) != HSAW_OK)
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    ProbGraph g;
    g.n = n;
    g.m = static_cast<EdgeId>(nedges);
    g.in_offsets.resize(static_cast<std::size_t>(n) + 1);
    g.in_src.resize(nedges);
    g.in_cum.resize(nedges);
    g.weight.resize(nedges);
    g.edge_dst.resize(nedges);
    int rc = hsaw_gpu_csr_build(ctx, n, nedges, u, v, w, mode == WeightMode::Given ? 0 : 1,
                                g.in_offsets.data(), g.in_src.data(), g.in_cum.data(),
                                g.weight.data(), g.edge_dst.data());
    std::string msg = rc == HSAW_OK ? std::string() : std::string(hsaw_gpu_last_error(ctx));
    hsaw_gpu_ctx_destroy(ctx);
    if (rc == HSAW_EDATA) throw DataError(msg);  // the reference's own messages, unprefixed
    if (rc == HSAW_EINVAL) throw std::invalid_argument(msg);
    if (rc != HSAW_OK) throw DeviceError(msg);
    return g;
}

ProbGraph build_graph_device(NodeId n, const std::vector<std::tuple<NodeId, NodeId, double>>& edges,
                             WeightMode mode, std::uint64_t seed, int device) {
    if (mode == WeightMode::RandomNormalized) return build_graph(n, edges, mode, seed);
    std::vector<NodeId> u(edges.size()), v(edges.size());
    std::vector<double> w(mode == WeightMode::Given ? edges.size() : 0);
    for (std::size_t i = 0; i < edges.size(); ++i) {
        u[i] = std::get<0>(edges[i]);
        v[i] = std::get<1>(edges[i]);
        if (mode == WeightMode::Given) w[i] = std::get<2>(edges[i]);
    }
    return build_graph_device(n, edges.size(), u.data(), v.data(),
                              mode == WeightMode::Given ? w.data() : nullptr, mode, device);
}

// ---- R-MAT bench graphs on the device --------------------------------------------------------------
namespace {

// Fetches the CSR held by `ctx` into g (n, m set by the caller). lean: in_offsets / in_src / in_cum only.
void fetch_held_csr(hsaw_gpu_ctx* ctx, ProbGraph& g, bool lean) {
    g.in_offsets.resize(static_cast<std::size_t>(g.n) + 1);
    g.in_src.resize(g.m);
    g.in_cum.resize(g.m);
    raise(hsaw_gpu_held_csr_fetch(ctx, g.in_offsets.data(), g.in_src.data(), g.in_cum.data()), ctx,
          "rmat_graph_device");
    if (lean) return;
    g.weight.resize(g.m);
    g.edge_dst.resize(g.m);
    for (NodeId v = 0; v < g.n; ++v) {
        const std::uint64_t lo = g.in_offsets[v], hi = g.in_offsets[v + 1];
        if (hi == lo) continue;
        const double share = 1.0 / static_cast<double>(hi - lo);  // rmat_graph_n's weight
        for (std::uint64_t e = lo; e < hi; ++e) {
            g.weight[e] = share;
            g.edge_dst[e] = v;
        }
    }
}

}  // namespace

ProbGraph rmat_graph_device(NodeId n, std::uint64_t raw_edges, std::uint64_t seed, double a,
                            double b, double c, int device, bool lean) {
    RmatLabels lab = rmat_labels(n, seed);
    hsaw_gpu_ctx* ctx = nullptr;
    if (hsaw_gpu_ctx_create(device, nullptr, &ctx) != HSAW_OK)
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    ProbGraph g;
    try {
        std::uint64_t m = 0;
        raise(hsaw_gpu_rmat_build(ctx, n, raw_edges, lab.label.data(), lab.state.state, a, b, c, &m),
              ctx, "rmat_graph_device");
        g.n = n;
        g.m = static_cast<EdgeId>(m);
        fetch_held_csr(ctx, g, lean);
    } catch (...) {
        hsaw_gpu_ctx_destroy(ctx);
        throw;
    }
    hsaw_gpu_ctx_destroy(ctx);
    return g;
}

std::unique_ptr<DeviceGraph> DeviceGraph::from_rmat(NodeId n, std::uint64_t raw_edges,
                                                    std::uint64_t seed, const SuspectSet* vi,
                                                    double a, double b, double c, int device,
                                                    void* cuda_stream, ProbGraph* host_copy) {
    if (vi && vi->p_of.size() != n) throw std::invalid_argument("suspect set does not match graph");
    RmatLabels lab = rmat_labels(n, seed);
    std::unique_ptr<DeviceGraph> dg(new DeviceGraph());
    if (hsaw_gpu_ctx_create(device, cuda_stream, &dg->ctx_) != HSAW_OK) {
        dg->ctx_ = nullptr;
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    }
    std::uint64_t m = 0;
    raise(hsaw_gpu_rmat_build(dg->ctx_, n, raw_edges, lab.label.data(), lab.state.state, a, b, c, &m),
          dg->ctx_, "DeviceGraph::from_rmat");
    lab.label = {};
    dg->n_ = n;
    dg->m_ = static_cast<EdgeId>(m);
    if (host_copy) {
        host_copy->n = n;
        host_copy->m = dg->m_;
        host_copy->weight.clear();
        host_copy->edge_dst.clear();
        fetch_held_csr(dg->ctx_, *host_copy, true);
    }
    raise(hsaw_gpu_held_csr_install(dg->ctx_, vi ? vi->p_of.data() : nullptr, 0), dg->ctx_,
          "DeviceGraph::from_rmat");
    return dg;
}

// ---- binary ingest on the device -------------------------------------------------------------------
namespace {

// The HSAW1 file mapped read-only; header checks with load_cache's own messages
// (proj/src/graph.cpp:398-416: "cannot open cache", "bad cache magic in", "truncated cache").
struct MappedCache {
    void* base = MAP_FAILED;
    std::size_t bytes = 0;
    NodeId n = 0;
    EdgeId m = 0;
    const unsigned char* body = nullptr;

    explicit MappedCache(const std::string& path) {
        int fd = ::open(path.c_str(), O_RDONLY);
        if (fd < 0) throw DataError("cannot open cache: " + path);
        struct stat st {};
        if (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
            ::close(fd);
            throw DataError("cannot open cache: " + path);
        }
        bytes = static_cast<std::size_t>(st.st_size);
        if (bytes) base = ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0);
        ::close(fd);
        const auto* b = static_cast<const unsigned char*>(base);
        if (base == MAP_FAILED || bytes < 5 || std::memcmp(b, "HSAW1", 5) != 0) {
            unmap();
            throw DataError("bad cache magic in " + path);
        }
        auto le64 = [&](std::size_t at) {
            std::uint64_t x = 0;
            for (int i = 0; i < 8; ++i)
                x |= static_cast<std::uint64_t>(at + i < bytes ? b[at + i] : 0xFF) << (8 * i);
            return x;
        };
        n = static_cast<NodeId>(le64(5));   // static_cast<NodeId>(get_u64(f)), graph.cpp:403
        m = static_cast<EdgeId>(le64(13));
        const std::uint64_t need = 21 + 8 * (static_cast<std::uint64_t>(n) + 1 + 2ull * m);
        if (bytes < need) {
            unmap();
            throw DataError("truncated cache: " + path);
        }
        ::madvise(base, bytes, MADV_SEQUENTIAL);
        body = b + 21;
    }
    void unmap() {
        if (base != MAP_FAILED) ::munmap(base, bytes);
        base = MAP_FAILED;
    }
    ~MappedCache() { unmap(); }
    MappedCache(const MappedCache&) = delete;
    MappedCache& operator=(const MappedCache&) = delete;
};

}  // namespace

// ---- text ingest on the device --------------------------------------------------------------------
ProbGraph load_edge_list_device(const std::string& path, WeightMode mode, std::uint64_t seed,
                                const LoadOptions& opts, int device) {
    if (opts.symmetrize) return load_edge_list(path, mode, seed, opts);  // host dedupe of tuples
    int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) throw DataError("cannot open edge list: " + path);
    struct stat st {};
    if (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
        ::close(fd);
        return load_edge_list(path, mode, seed, opts);  // pipes etc.: stream through the host parser
    }
    const std::size_t bytes = static_cast<std::size_t>(st.st_size);
    void* base = bytes ? ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0) : nullptr;
    ::close(fd);
    if (bytes && base == MAP_FAILED) return load_edge_list(path, mode, seed, opts);
    struct Unmap {
        void* p;
        std::size_t n;
        ~Unmap() {
            if (p && n) ::munmap(p, n);
        }
    } unmap{base, bytes};
    if (bytes) ::madvise(base, bytes, MADV_SEQUENTIAL);

    hsaw_gpu_ctx* ctx = nullptr;
    if (hsaw_gpu_ctx_create(device, nullptr, &ctx) != HSAW_OK)
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    struct CtxGuard {
        hsaw_gpu_ctx* c;
        ~CtxGuard() { hsaw_gpu_ctx_destroy(c); }
    } guard{ctx};

    hsaw_gpu_edge_text* el = nullptr;
    std::uint64_t ne = 0, nids = 0, host_line = 0;
    int identity = 0;
    const bool given = mode == WeightMode::Given;
    int rc = hsaw_gpu_edge_text_parse(ctx, static_cast<const char*>(base), bytes, given ? 1 : 0,
                                      given ? 1 : 0, &el, &ne, &nids, &identity, &host_line);
    if (rc != HSAW_OK) raise(rc, ctx, "load_edge_list");
    // a line the device does not parse: the host parser decides what it is and words the error
    if (host_line != 0) return load_edge_list(path, mode, seed, opts);
    if (ne == 0) throw DataError(path + ": no edges");  // graph.cpp:231
    struct ElGuard {
        hsaw_gpu_edge_text* e;
        ~ElGuard() { hsaw_gpu_edge_text_free(e); }
    } el_guard{el};

    std::vector<NodeId> u(ne), v(ne);
    std::vector<double> w(given ? ne : 0);
    const bool write_map = !identity || !opts.mapping_out.empty();  // graph.cpp:254
    std::vector<std::uint64_t> raw_ids(write_map ? nids : 0);
    rc = hsaw_gpu_edge_text_fetch(el, u.data(), v.data(), given ? w.data() : nullptr,
                                  write_map ? raw_ids.data() : nullptr);
    if (rc != HSAW_OK) raise(rc, ctx, "load_edge_list");
    if (write_map) {
        const std::string map_path = opts.mapping_out.empty() ? path + ".nodemap" : opts.mapping_out;
        std::ofstream mf(map_path);
        if (!mf) throw DataError("cannot write node map: " + map_path);
        for (std::size_t i = 0; i < raw_ids.size(); ++i) mf << raw_ids[i] << ' ' << i << '\n';
    }
    const NodeId n = static_cast<NodeId>(nids);
    if (mode == WeightMode::RandomNormalized) {  // one global draw stream over the rows: host
        std::vector<std::tuple<NodeId, NodeId, double>> edges(ne);
        for (std::size_t i = 0; i < ne; ++i) edges[i] = {u[i], v[i], 0.0};
        return build_graph(n, std::move(edges), mode, seed);
    }
    return build_graph_device(n, ne, u.data(), v.data(), given ? w.data() : nullptr, mode, device);
}

ProbGraph load_cache_device(const std::string& path, int device) {
    MappedCache file(path);
    if (file.n == 0) {
        // the reference accepts an empty cache (load_cache reads the single offset, sums no rows,
        // validate() passes iff that offset is 0 and m is 0, proj/src/graph.cpp:76-77); nothing
        // for a device to do
        std::uint64_t first = 0;
        std::memcpy(&first, file.body, 8);
        if (first != 0 || file.m != 0) throw DataError("graph: offsets do not cover edge range");
        ProbGraph empty;
        empty.in_offsets.assign(1, 0);
        return empty;
    }
    hsaw_gpu_ctx* ctx = nullptr;
    if (hsaw_gpu_ctx_create(device, nullptr, &ctx) != HSAW_OK)
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    ProbGraph g;
    g.n = file.n;
    g.m = file.m;
    g.in_offsets.resize(static_cast<std::size_t>(g.n) + 1);
    g.in_src.resize(g.m);
    g.in_cum.resize(g.m);
    g.weight.resize(g.m);
    g.edge_dst.resize(g.m);
    int rc = hsaw_gpu_cache_decode(ctx, g.n, g.m, file.body, g.in_offsets.data(), g.in_src.data(),
                                   g.in_cum.data(), g.weight.data(), g.edge_dst.data());
    std::string msg = rc == HSAW_OK ? std::string() : std::string(hsaw_gpu_last_error(ctx));
    hsaw_gpu_ctx_destroy(ctx);
    if (rc == HSAW_EDATA) throw DataError(msg);  // validate()'s own messages, unprefixed
    if (rc == HSAW_EINVAL) throw std::invalid_argument(msg);
    if (rc != HSAW_OK) throw DeviceError(msg);
    return g;
}

std::unique_ptr<DeviceGraph> DeviceGraph::from_cache(const std::string& path, int device,
                                                     void* cuda_stream) {
    MappedCache file(path);
    std::unique_ptr<DeviceGraph> dg(new DeviceGraph());
    if (hsaw_gpu_ctx_create(device, cuda_stream, &dg->ctx_) != HSAW_OK) {
        dg->ctx_ = nullptr;
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    }
    dg->n_ = file.n;
    dg->m_ = file.m;
    int rc = hsaw_gpu_graph_cache_upload(dg->ctx_, file.n, file.m, file.body, nullptr);
    if (rc != HSAW_OK) {
        std::string msg = hsaw_gpu_last_error(dg->ctx_);
        if (rc == HSAW_EDATA) throw DataError(msg);
        if (rc == HSAW_EINVAL) throw std::invalid_argument(msg);
        throw DeviceError(msg);
    }
    return dg;
}

std::unique_ptr<DeviceGraph> DeviceGraph::from_edge_list(const std::string& path, WeightMode mode,
                                                         int device, void* cuda_stream) {
    if (mode == WeightMode::RandomNormalized) return nullptr;  // host draw stream
    int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) throw DataError("cannot open edge list: " + path);
    struct stat st {};
    if (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode) || st.st_size == 0) {
        ::close(fd);
        return nullptr;
    }
    const std::size_t bytes = static_cast<std::size_t>(st.st_size);
    void* base = ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0);
    ::close(fd);
    if (base == MAP_FAILED) return nullptr;
    struct Unmap {
        void* p;
        std::size_t n;
        ~Unmap() { ::munmap(p, n); }
    } unmap{base, bytes};
    ::madvise(base, bytes, MADV_SEQUENTIAL);

    std::unique_ptr<DeviceGraph> dg(new DeviceGraph());
    if (hsaw_gpu_ctx_create(device, cuda_stream, &dg->ctx_) != HSAW_OK) {
        dg->ctx_ = nullptr;
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    }
    hsaw_gpu_edge_text* el = nullptr;
    std::uint64_t ne = 0, nids = 0, host_line = 0;
    int identity = 0;
    const int given = mode == WeightMode::Given ? 1 : 0;
    int rc = hsaw_gpu_edge_text_parse(dg->ctx_, static_cast<const char*>(base), bytes, given, given,
                                      &el, &ne, &nids, &identity, &host_line);
    if (rc != HSAW_OK) raise(rc, dg->ctx_, "from_edge_list");
    if (host_line != 0 || el == nullptr) return nullptr;  // host loader's business (incl. "no edges")
    struct ElGuard {
        hsaw_gpu_edge_text* e;
        ~ElGuard() { hsaw_gpu_edge_text_free(e); }
    } el_guard{el};
    rc = hsaw_gpu_edge_text_install(el, given ? 0 : 1, nullptr);
    if (rc != HSAW_OK) {
        std::string msg = hsaw_gpu_last_error(dg->ctx_);
        if (rc == HSAW_EDATA) throw DataError(msg);  // build_graph's / validate()'s own messages
        if (rc == HSAW_EINVAL) throw std::invalid_argument(msg);
        throw DeviceError(msg);
    }
    dg->n_ = static_cast<NodeId>(nids);
    dg->m_ = static_cast<EdgeId>(ne);
    return dg;
}

// ---- DeviceGraph --------------------------------------------------------------------------------
DeviceGraph::DeviceGraph(const ProbGraph& g, const SuspectSet& vi, int device, void* cuda_stream)
    : n_(g.n), m_(g.m) {
    if (vi.p_of.size() != g.n) throw std::invalid_argument("suspect set does not match graph");
    const char* tenv = std::getenv("HSAW_UPLOAD_TIMING");
    const bool timing = tenv && std::atoi(tenv) != 0;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = hsaw_gpu_ctx_create(device, cuda_stream, &ctx_);
    if (rc != HSAW_OK)
        throw DeviceError("no usable CUDA device: the HSAW path has no CPU fallback");
    const auto t1 = std::chrono::steady_clock::now();
    rc = hsaw_gpu_graph_upload(ctx_, g.n, g.m, g.in_offsets.data(), g.in_src.data(),
                               g.in_cum.data(), vi.p_of.data());
    if (timing) {
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[hsaw upload] ctx_create %.2f ms, graph_upload %.2f ms\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    if (rc != HSAW_OK) {
        std::string msg = hsaw_gpu_last_error(ctx_);
        hsaw_gpu_ctx_destroy(ctx_);
        ctx_ = nullptr;
        if (rc == HSAW_EDATA) throw DataError(msg);
        if (rc == HSAW_EINVAL) throw std::invalid_argument(msg);
        throw DeviceError(msg);
    }
}

DeviceGraph::~DeviceGraph() { hsaw_gpu_ctx_destroy(ctx_); }

void DeviceGraph::set_suspects(const SuspectSet& vi) {
    if (vi.p_of.size() != n_) throw std::invalid_argument("suspect set does not match graph");
    raise(hsaw_gpu_suspects_upload(ctx_, vi.p_of.data()), ctx_, "set_suspects");
}

std::uint64_t DeviceGraph::device_bytes() const { return hsaw_gpu_graph_bytes(ctx_); }
std::uint64_t DeviceGraph::launches() const { return hsaw_gpu_launch_count(ctx_); }

std::vector<double> DeviceGraph::stage_ms(bool reset) const {
    std::vector<double> ms(HSAW_STAGE_COUNT, 0.0);
    raise(hsaw_gpu_stage_times(ctx_, ms.data(), nullptr, reset ? 1 : 0), ctx_, "stage_times");
    return ms;
}

// ---- thread_sample / decode ---------------------------------------------------------------------
std::vector<EncodedWalk> thread_sample(const DeviceGraph& dg, std::uint64_t worker_id,
                                       std::uint32_t l, const SamplerConfig& cfg) {
    SamplerConfig one = cfg;
    one.batch_size = l;  // the batch length is the call's l, as in the reference signature
    hsaw_sampler_cfg c = to_c(one);
    std::vector<EncodedWalk> out;
    if (l == 0) return out;
    std::vector<std::uint64_t> seeds(l);
    std::vector<std::uint32_t> lens(l);
    std::uint32_t count = 0;
    raise(hsaw_gpu_encode_batches(dg.ctx(), &c, worker_id, 1, seeds.data(), lens.data(), &count,
                                  nullptr),
          dg.ctx(), "thread_sample");
    out.reserve(count);
    for (std::uint32_t i = 0; i < count; ++i)
        out.push_back(EncodedWalk{PrgState{seeds[i]}, lens[i], worker_id, i});
    return out;
}

std::vector<EncodedWalk> thread_sample(const ProbGraph& g, const SuspectSet& vi,
                                       std::uint64_t worker_id, std::uint32_t l,
                                       const SamplerConfig& cfg) {
    DeviceGraph dg(g, vi);
    return thread_sample(dg, worker_id, l, cfg);
}

std::vector<std::optional<HsawSample>> DecodeContext::decode(std::span<const EncodedWalk> walks) {
    const std::uint64_t nw = walks.size();
    std::vector<std::optional<HsawSample>> out(nw);
    if (nw == 0) return out;
    std::vector<std::uint64_t> seeds(nw), edge_off(nw + 1, 0);
    std::vector<std::uint32_t> lens(nw);
    for (std::uint64_t w = 0; w < nw; ++w) {
        seeds[w] = walks[w].seed.state;
        lens[w] = walks[w].len;
        edge_off[w + 1] = edge_off[w] + lens[w];
    }
    std::vector<std::uint32_t> nodes(edge_off[nw] + nw), edges(edge_off[nw] + 1);
    std::vector<std::uint8_t> status(nw);
    raise(hsaw_gpu_decode_walks(dg_.ctx(), nw, seeds.data(), lens.data(), edge_off.data(),
                                nodes.data(), edges.data(), status.data()),
          dg_.ctx(), "decode");
    for (std::uint64_t w = 0; w < nw; ++w) {
        if (status[w] == 2)  // proj/src/sampler.cpp:306-335
            throw DataError("decode: replay disagrees with the encoded walk");
        if (status[w] == 0) continue;  // cycle the generation heuristic missed
        HsawSample s;
        s.nodes.assign(nodes.begin() + edge_off[w] + w, nodes.begin() + edge_off[w + 1] + w + 1);
        s.edge_ids.assign(edges.begin() + edge_off[w], edges.begin() + edge_off[w + 1]);
        out[w] = std::move(s);
    }
    return out;
}

std::optional<HsawSample> DecodeContext::decode(const EncodedWalk& ew) {
    return std::move(decode(std::span<const EncodedWalk>(&ew, 1))[0]);
}

// ---- SampleStream -------------------------------------------------------------------------------
SampleStream::SampleStream(const DeviceGraph& dg, std::uint64_t seed, SamplerConfig cfg,
                           Items items)
    : dg_(dg) {
    hsaw_sampler_cfg c = to_c(cfg);
    raise(hsaw_gpu_stream_create(dg.ctx(), seed, &c, &s_), dg.ctx(), "SampleStream");
    if (items != Items::Both) {
        const int rc = hsaw_gpu_stream_keep(s_, items == Items::NodesOnly, items == Items::EdgesOnly);
        if (rc != HSAW_OK) {
            hsaw_gpu_stream_destroy(s_);
            s_ = nullptr;
            raise(rc, dg.ctx(), "SampleStream");
        }
    }
}

SampleStream::~SampleStream() { hsaw_gpu_stream_destroy(s_); }

void SampleStream::ensure(std::uint64_t min_accepted) {
    raise(hsaw_gpu_stream_ensure(s_, min_accepted), dg_.ctx(), "ensure");
}

void SampleStream::restrict(std::span<const NodeId> start_domain, const std::uint8_t* allowed) {
    raise(hsaw_gpu_stream_restrict(s_, start_domain.data(), start_domain.size(), allowed), dg_.ctx(),
          "restrict");
}

std::uint64_t SampleStream::crossings_for(std::uint64_t min_accepted) const {
    std::uint64_t c = 0;
    raise(hsaw_gpu_stream_crossings(s_, min_accepted, &c), dg_.ctx(), "crossings_for");
    return c;
}

std::uint64_t SampleStream::materialized() const {
    std::uint64_t acc = 0;
    raise(hsaw_gpu_stream_size(s_, &acc, nullptr, nullptr), dg_.ctx(), "stream_size");
    return acc;
}

std::vector<std::uint64_t> SampleStream::stats() const {
    std::vector<std::uint64_t> st(8, 0);
    raise(hsaw_gpu_stream_stats(s_, st.data()), dg_.ctx(), "stream_stats");
    return st;
}

std::vector<HsawSample> SampleStream::prefix(std::uint64_t offset, std::uint64_t count) const {
    std::uint64_t total_edges = 0;
    raise(hsaw_gpu_stream_slice_edges(s_, offset, count, &total_edges), dg_.ctx(), "prefix");
    std::vector<std::uint64_t> edge_off(count + 1);
    std::vector<std::uint32_t> nodes(total_edges + count + 1), edges(total_edges + 1);
    raise(hsaw_gpu_stream_export(s_, offset, count, edge_off.data(), nodes.data(), edges.data(),
                                 nullptr, nullptr),
          dg_.ctx(), "prefix");
    return unpack(count, edge_off, nodes, edges);
}

SampleStream::Counters SampleStream::counters_for(std::uint64_t min_accepted) const {
    Counters c;
    raise(hsaw_gpu_stream_counters(s_, min_accepted, &c.attempts, &c.accepted), dg_.ctx(),
          "counters_for");
    return c;
}

SamplePool SampleStream::to_pool(std::uint64_t min_accepted) const {
    Counters c = counters_for(min_accepted);
    SamplePool pool;
    pool.attempts = c.attempts;
    std::uint64_t total_edges = 0;
    raise(hsaw_gpu_stream_slice_edges(s_, 0, c.accepted, &total_edges), dg_.ctx(), "to_pool");
    std::vector<std::uint64_t> edge_off(c.accepted + 1), workers(c.accepted + 1);
    std::vector<std::uint32_t> nodes(total_edges + c.accepted + 1), edges(total_edges + 1),
        seqs(c.accepted + 1);
    raise(hsaw_gpu_stream_export(s_, 0, c.accepted, edge_off.data(), nodes.data(), edges.data(),
                                 workers.data(), seqs.data()),
          dg_.ctx(), "to_pool");
    pool.samples = unpack(c.accepted, edge_off, nodes, edges);
    pool.tags.resize(c.accepted);
    for (std::uint64_t w = 0; w < c.accepted; ++w) pool.tags[w] = WalkTag{workers[w], seqs[w]};
    return pool;
}

SamplePool stream_samples(const DeviceGraph& dg, std::uint64_t target, std::uint64_t seed,
                          const SamplerConfig& cfg) {
    SampleStream stream(dg, seed, cfg);
    stream.ensure(target);
    return stream.to_pool(target);
}

SamplePool stream_samples(const ProbGraph& g, const SuspectSet& vi, std::uint32_t /*workers*/,
                          std::uint64_t target, std::uint64_t seed, const SamplerConfig& cfg) {
    DeviceGraph dg(g, vi);
    return stream_samples(dg, target, seed, cfg);
}

double estimate_influence(const SamplePool& pool, NodeId n) {  // proj/src/sampler.cpp:503-508
    if (pool.attempts == 0) throw std::invalid_argument("estimate_influence: no attempts");
    return static_cast<double>(n) * static_cast<double>(pool.accepted()) /
           static_cast<double>(pool.attempts);
}

void dump_walks(const SamplePool& pool, std::ostream& out) {  // "worker seq len v1 .. vl"
    for (std::size_t i = 0; i < pool.samples.size(); ++i) {
        out << pool.tags[i].worker_id << ' ' << pool.tags[i].seq << ' '
            << pool.samples[i].edge_ids.size();
        for (NodeId v : pool.samples[i].nodes) out << ' ' << v;
        out << '\n';
    }
}

// ---- CoverageIndex / greedy ---------------------------------------------------------------------
namespace {

std::uint64_t count_candidates(const CandidateSet& cand, std::uint32_t limit) {
    if (!cand.ids) return limit;
    std::vector<std::uint32_t> ids = *cand.ids;
    for (std::uint32_t id : ids)
        if (id >= limit)  // candidate_mask, proj/src/coverage.cpp:18-20
            throw DataError("candidate id out of range: " + std::to_string(id));
    std::sort(ids.begin(), ids.end());
    return static_cast<std::uint64_t>(std::unique(ids.begin(), ids.end()) - ids.begin());
}

}  // namespace

CoverageIndex::CoverageIndex(ItemKind kind, const SampleStream& stream, std::uint64_t offset,
                             std::uint64_t count, const CandidateSet& cand, const ProbGraph& g)
    : kind_(kind), ctx_(stream.device().ctx()), stream_(stream.handle()), offset_(offset),
      count_(count), cand_(cand.ids) {
    if (cand.kind != kind)  // proj/src/coverage.cpp:41-42
        throw std::invalid_argument("candidate kind does not match index kind");
    if (offset + count > stream.materialized())
        throw std::out_of_range("sample stream prefix not materialized");
    ncand_ = count_candidates(cand, kind == ItemKind::Edge ? g.m : g.n);
}

CoverageIndex::CoverageIndex(const DeviceGraph& dg,
                             std::span<const std::vector<std::uint32_t>> item_sets,
                             const CandidateSet& cand, const ProbGraph& g)
    : kind_(cand.kind), ctx_(dg.ctx()), count_(item_sets.size()), cand_(cand.ids) {
    const std::uint32_t limit = kind_ == ItemKind::Edge ? g.m : g.n;
    ncand_ = count_candidates(cand, limit);
    std::vector<std::uint64_t> off(item_sets.size() + 1, 0);
    for (std::size_t i = 0; i < item_sets.size(); ++i) off[i + 1] = off[i] + item_sets[i].size();
    std::vector<std::uint32_t> flat;
    flat.reserve(off.back() + 1);
    for (const auto& s : item_sets) flat.insert(flat.end(), s.begin(), s.end());
    raise(hsaw_gpu_walkset_import(ctx_, limit, item_sets.size(), off.data(), flat.data(),
                                  &walkset_),
          ctx_, "CoverageIndex");
}

CoverageIndex::CoverageIndex(const DeviceGraph& dg, hsaw_gpu_walkset* adopted, std::uint64_t nsets,
                             const CandidateSet& cand, const ProbGraph& g)
    : kind_(cand.kind), ctx_(dg.ctx()), walkset_(adopted), count_(nsets), cand_(cand.ids) {
    ncand_ = count_candidates(cand, kind_ == ItemKind::Edge ? g.m : g.n);
}

CoverageIndex::~CoverageIndex() { hsaw_gpu_walkset_destroy(walkset_); }

std::uint64_t CoverageIndex::coverage_upper_bound(std::uint32_t k) const {
    std::uint64_t ub = 0;
    raise(hsaw_gpu_coverage_upper_bound(ctx_, stream_, walkset_,
                                        kind_ == ItemKind::Edge ? HSAW_KIND_EDGE : HSAW_KIND_NODE,
                                        offset_, count_, cand_ ? cand_->data() : nullptr,
                                        cand_ ? cand_->size() : 0, k, &ub),
          ctx_, "coverage_upper_bound");
    return ub;
}

std::uint64_t CoverageIndex::coverage_of(std::span<const std::uint32_t> items) const {
    std::uint64_t cov = 0;
    raise(hsaw_gpu_coverage_of(ctx_, stream_, walkset_,
                               kind_ == ItemKind::Edge ? HSAW_KIND_EDGE : HSAW_KIND_NODE, offset_,
                               count_, cand_ ? cand_->data() : nullptr, cand_ ? cand_->size() : 0,
                               items.data(), items.size(), &cov),
          ctx_, "coverage_of");
    return cov;
}

struct GreedyAccess {
    static GreedyResult run(const CoverageIndex& idx, std::uint32_t k) {
        if (k > idx.ncand_)  // proj/src/coverage.cpp:93-94
            throw std::invalid_argument("budget k exceeds candidate count");
        GreedyResult res;
        if (k == 0) return res;
        res.solution.assign(k, 0);
        // an explicit but empty candidate list must stay distinguishable from "all"
        static const std::uint32_t none = 0;
        const std::uint32_t* cand = idx.cand_ ? (idx.cand_->empty() ? &none : idx.cand_->data())
                                              : nullptr;
        raise(hsaw_gpu_greedy(idx.ctx_, idx.stream_, idx.walkset_,
                              idx.kind_ == ItemKind::Edge ? HSAW_KIND_EDGE : HSAW_KIND_NODE,
                              idx.offset_, idx.count_, cand, idx.cand_ ? idx.cand_->size() : 0, k,
                              res.solution.data(), &res.coverage),
              idx.ctx_, "greedy_max_cover");
        return res;
    }
};

GreedyResult greedy_max_cover(const CoverageIndex& idx, std::uint32_t k) {
    return GreedyAccess::run(idx, k);
}

}  // namespace hsaw

// ---- evaluation: paired forward simulation (proj/src/evaluation.cpp:195-242) ---------------------
namespace hsaw {

namespace {
void raise_eval(int status, hsaw_gpu_ctx* ctx) {  // the reference's own messages, unprefixed
    if (status == HSAW_OK) return;
    std::string msg = hsaw_gpu_last_error(ctx);
    switch (status) {
        case HSAW_EINVAL: throw std::invalid_argument(msg);
        case HSAW_EDATA: throw DataError(msg);
        default: throw DeviceError(msg);
    }
}
int kind_code(ItemKind k) { return k == ItemKind::Edge ? HSAW_KIND_EDGE : HSAW_KIND_NODE; }
}  // namespace

void RemovalSet::validate(const ProbGraph& g) const {
    std::uint32_t limit = kind == ItemKind::Edge ? g.m : g.n;
    for (std::uint32_t id : ids)
        if (id >= limit) throw DataError("removal id out of range: " + std::to_string(id));
}

std::uint32_t lt_forward_simulate(const DeviceGraph& dg, PrgState& s) {
    std::uint32_t full = 0;
    raise_eval(hsaw_gpu_paired_runs(dg.ctx(), -1, nullptr, 0, &s.state, 1, &full, nullptr), dg.ctx());
    return full;
}

std::uint32_t lt_forward_simulate(const ProbGraph& g, const SuspectSet& vi, PrgState& s) {
    DeviceGraph dg(g, vi);
    return lt_forward_simulate(dg, s);
}

PairedRuns paired_runs(const DeviceGraph& dg, const RemovalSet& removal, std::uint64_t runs,
                       PrgState& s) {
    PairedRuns out;
    out.full.resize(runs);
    out.residual.resize(runs);
    raise_eval(hsaw_gpu_paired_runs(dg.ctx(), kind_code(removal.kind), removal.ids.data(),
                                    removal.ids.size(), &s.state, runs, out.full.data(),
                                    out.residual.data()),
               dg.ctx());
    return out;
}

SuspensionEstimate estimate_suspension(const DeviceGraph& dg, const RemovalSet& removal,
                                       double epsilon, double delta, PrgState& s) {
    SuspensionEstimate e;
    int capped = 0;
    raise_eval(hsaw_gpu_estimate_suspension(dg.ctx(), kind_code(removal.kind), removal.ids.data(),
                                            removal.ids.size(), epsilon, delta, &s.state, &e.value,
                                            &capped, &e.runs),
               dg.ctx());
    e.capped = capped != 0;
    return e;
}

SuspensionEstimate estimate_suspension(const ProbGraph& g, const SuspectSet& vi,
                                       const RemovalSet& removal, double epsilon, double delta,
                                       PrgState& s) {
    // argument checks before any device work, in the reference's order (evaluation.cpp:214-218)
    if (!(epsilon > 0.0) || epsilon >= 1.0) throw std::invalid_argument("epsilon must be in (0,1)");
    if (!(delta > 0.0) || delta >= 1.0) throw std::invalid_argument("delta must be in (0,1)");
    removal.validate(g);
    if (removal.ids.empty()) return {0.0, false, 0};
    DeviceGraph dg(g, vi);
    return estimate_suspension(dg, removal, epsilon, delta, s);
}

}  // namespace hsaw
