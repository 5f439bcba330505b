// C wrappers over the C++ host layer (include/hsaw_host.h): handle marshalling and the
// exception -> status mapping, nothing else.
#include "hsaw_host.h"

#include <cstring>
#include <string>

#include "hsaw_b200.hpp"

using namespace hsaw;

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return 1;
    } catch (const DataError& e) {
        g_error = e.what();
        return 2;
    } catch (const SamplingError& e) {
        g_error = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_error = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 5;
    }
}

const ProbGraph& G(const void* g) { return *static_cast<const ProbGraph*>(g); }

SuspectSet dense_suspects(const ProbGraph& g, const double* p_of) {
    std::vector<std::pair<NodeId, double>> mem;
    for (NodeId v = 0; v < g.n; ++v)
        if (p_of[v] != 0.0) mem.emplace_back(v, p_of[v]);
    return SuspectSet::from_members(std::move(mem), g);
}

}  // namespace

extern "C" {

const char* hsawh_last_error(void) { return g_error.c_str(); }

int hsawh_graph_load_edge_list(const char* path, int weight_mode, uint64_t seed, int symmetrize,
                               const char* mapping_out, void** out) {
    return guarded([&] {
        LoadOptions opts;
        opts.symmetrize = symmetrize != 0;
        if (mapping_out) opts.mapping_out = mapping_out;
        *out = new ProbGraph(load_edge_list(path, static_cast<WeightMode>(weight_mode), seed, opts));
    });
}

int hsawh_graph_build(uint32_t n, uint64_t nedges, const uint32_t* u, const uint32_t* v,
                      const double* w, int weight_mode, uint64_t seed, void** out) {
    return guarded([&] {
        std::vector<std::tuple<NodeId, NodeId, double>> edges;
        edges.reserve(nedges);
        for (uint64_t i = 0; i < nedges; ++i) edges.emplace_back(u[i], v[i], w ? w[i] : 0.0);
        *out = new ProbGraph(
            build_graph(n, std::move(edges), static_cast<WeightMode>(weight_mode), seed));
    });
}

int hsawh_graph_build_device(uint32_t n, uint64_t nedges, const uint32_t* u, const uint32_t* v,
                             const double* w, int weight_mode, int device, void** out) {
    return guarded([&] {
        *out = new ProbGraph(build_graph_device(n, nedges, u, v, w,
                                                static_cast<WeightMode>(weight_mode), device));
    });
}

int hsawh_graph_synth(uint32_t n, uint32_t density, uint64_t seed, void** out) {
    return guarded([&] { *out = new ProbGraph(synth_graph(n, density, seed)); });
}

int hsawh_graph_rmat(uint32_t scale, double edge_factor, uint64_t seed, void** out) {
    return guarded([&] { *out = new ProbGraph(rmat_graph(scale, edge_factor, seed)); });
}

int hsawh_graph_rmat_n(uint32_t n, uint64_t raw_edges, uint64_t seed, void** out) {
    return guarded([&] { *out = new ProbGraph(rmat_graph_n(n, raw_edges, seed)); });
}

int hsawh_graph_rmat_device(uint32_t n, uint64_t raw_edges, uint64_t seed, int device, int lean,
                            void** out) {
    return guarded([&] {
        *out = new ProbGraph(rmat_graph_device(n, raw_edges, seed, 0.57, 0.19, 0.19, device, lean != 0));
    });
}

int hsawh_graph_shell(uint32_t n, uint32_t m, void** out) {
    return guarded([&] {
        auto* g = new ProbGraph;
        g->n = n;
        g->m = m;
        *out = g;
    });
}

void hsawh_graph_ptrs(const void* gp, const uint64_t** in_offsets, const uint32_t** in_src,
                      const double** in_cum) {
    const ProbGraph& g = G(gp);
    *in_offsets = g.in_offsets.data();
    *in_src = g.in_src.data();
    *in_cum = g.in_cum.data();
}

int hsawh_suspects_random_n(uint32_t n, uint32_t count, uint64_t seed, double* p_of) {
    return guarded([&] {
        SuspectSet vi = random_suspects(n, count, seed);
        std::memcpy(p_of, vi.p_of.data(), 8 * vi.p_of.size());
    });
}

int hsawh_device_from_rmat(uint32_t n, uint64_t raw_edges, uint64_t seed, const double* p_of,
                           int device, void* cuda_stream, int want_host, void** dg_out,
                           void** g_out) {
    return guarded([&] {
        std::unique_ptr<SuspectSet> vi;
        if (p_of) {
            std::vector<std::pair<NodeId, double>> mem;
            for (NodeId v = 0; v < n; ++v)
                if (p_of[v] != 0.0) mem.emplace_back(v, p_of[v]);
            vi = std::make_unique<SuspectSet>(SuspectSet::from_members(std::move(mem), n));
        }
        auto host = std::make_unique<ProbGraph>();
        auto dg = DeviceGraph::from_rmat(n, raw_edges, seed, vi.get(), 0.57, 0.19, 0.19, device,
                                         cuda_stream, want_host ? host.get() : nullptr);
        if (!want_host) {  // a shell: node and edge counts only
            host->n = dg->n();
            host->m = dg->m();
        }
        *dg_out = dg.release();
        *g_out = host.release();
    });
}

int hsawh_graph_from_csr(uint32_t n, uint32_t m, const uint64_t* in_offsets,
                         const uint32_t* in_src, const double* in_cum, void** out) {
    return guarded([&] { *out = new ProbGraph(graph_from_csr(n, m, in_offsets, in_src, in_cum)); });
}

int hsawh_graph_save_cache(const void* g, const char* path) {
    return guarded([&] { save_cache(G(g), path); });
}
int hsawh_graph_load_cache(const char* path, void** out) {
    return guarded([&] { *out = new ProbGraph(load_cache(path)); });
}
int hsawh_graph_save_edge_list(const void* g, const char* path) {
    return guarded([&] { save_edge_list(G(g), path); });
}
int hsawh_graph_validate(const void* g) {
    return guarded([&] { G(g).validate(); });
}

void hsawh_graph_dims(const void* g, uint32_t* n, uint32_t* m) {
    *n = G(g).n;
    *m = G(g).m;
}

void hsawh_graph_copy(const void* gp, uint64_t* in_offsets, uint32_t* in_src, double* in_cum,
                      double* weight, uint32_t* edge_dst) {
    const ProbGraph& g = G(gp);
    if (in_offsets) std::memcpy(in_offsets, g.in_offsets.data(), 8 * g.in_offsets.size());
    if (in_src) std::memcpy(in_src, g.in_src.data(), 4 * g.in_src.size());
    if (in_cum) std::memcpy(in_cum, g.in_cum.data(), 8 * g.in_cum.size());
    if (weight) std::memcpy(weight, g.weight.data(), 8 * g.weight.size());
    if (edge_dst) std::memcpy(edge_dst, g.edge_dst.data(), 4 * g.edge_dst.size());
}

void hsawh_graph_free(void* g) { delete static_cast<ProbGraph*>(g); }

int hsawh_suspects_random(const void* g, uint32_t count, uint64_t seed, double* p_of) {
    return guarded([&] {
        SuspectSet vi = random_suspects(G(g), count, seed);
        std::memcpy(p_of, vi.p_of.data(), 8 * vi.p_of.size());
    });
}

int hsawh_suspects_load(const char* path, const void* g, double* p_of) {
    return guarded([&] {
        SuspectSet vi = load_suspects(path, G(g));
        std::memcpy(p_of, vi.p_of.data(), 8 * vi.p_of.size());
    });
}

int hsawh_schedule(uint64_t M, uint32_t k, double eps, double delta, double* out4,
                   uint32_t* t_max) {
    return guarded([&] {
        Schedule s = compute_schedule_m(M, k, eps, delta);
        out4[0] = s.n_max;
        out4[1] = s.lambda;
        out4[2] = s.lambda1;
        out4[3] = static_cast<double>(s.lambda_samples());
        *t_max = s.t_max;
    });
}

int hsawh_check(double cov_r, double cov_rp, double n_rp, uint64_t M, uint32_t k, double eps,
                double delta, uint32_t t, int* pass, double* eps_t) {
    return guarded([&] {
        CheckResult c = check_counts(cov_r, cov_rp, n_rp, compute_schedule_m(M, k, eps, delta), t);
        *pass = c.pass ? 1 : 0;
        *eps_t = c.eps_t;
    });
}

int hsawh_device_create(const void* g, const double* p_of, int device, void* cuda_stream,
                        void** out) {
    return guarded([&] {
        SuspectSet vi = dense_suspects(G(g), p_of);
        *out = new DeviceGraph(G(g), vi, device, cuda_stream);
    });
}

/* A prebuilt hsaw::SuspectSet (what a C++ caller of DeviceGraph(g, vi) holds already): built once
 * from the dense p_of array, so repeated device_create calls do not rebuild it. */
int hsawh_suspects_create(const void* g, const double* p_of, void** out) {
    return guarded([&] { *out = new SuspectSet(dense_suspects(G(g), p_of)); });
}
void hsawh_suspects_free(void* vi) { delete static_cast<SuspectSet*>(vi); }

int hsawh_device_create_vi(const void* g, const void* vi, int device, void* cuda_stream,
                           void** out) {
    return guarded([&] {
        *out = new DeviceGraph(G(g), *static_cast<const SuspectSet*>(vi), device, cuda_stream);
    });
}

void hsawh_device_free(void* dg) { delete static_cast<DeviceGraph*>(dg); }

void* hsawh_device_ctx(const void* dg) { return static_cast<const DeviceGraph*>(dg)->ctx(); }

int hsawh_interdict(const void* dg, const void* g, const double* p_of, int kind,
                    const uint32_t* cand, uint64_t ncand, uint32_t k, double eps, double delta,
                    uint64_t seed, uint32_t batch_size, uint64_t max_attempts, int device,
                    hsawh_result* out, uint32_t* solution, char* json, uint64_t json_cap) {
    return hsawh_interdict_rng(dg, g, p_of, kind, cand, ncand, k, eps, delta, seed, batch_size,
                               max_attempts, device, 0, out, solution, json, json_cap);
}

int hsawh_interdict_rng(const void* dg, const void* g, const double* p_of, int kind,
                        const uint32_t* cand, uint64_t ncand, uint32_t k, double eps, double delta,
                        uint64_t seed, uint32_t batch_size, uint64_t max_attempts, int device,
                        int rng_mode, hsawh_result* out, uint32_t* solution, char* json,
                        uint64_t json_cap) {
    return guarded([&] {
        const ItemKind ik = kind == 0 ? ItemKind::Edge : ItemKind::Node;
        CandidateSet cs = cand ? CandidateSet::of(ik, std::vector<std::uint32_t>(cand, cand + ncand))
                               : CandidateSet::all(ik);
        InterdictionOptions opts;
        opts.seed = seed;
        opts.sampler.batch_size = batch_size;
        opts.sampler.max_attempts = max_attempts;
        opts.sampler.rng = rng_mode == 1 ? WalkRng::PhiloxPerWalk : WalkRng::Reference;
        opts.device = device;
        InterdictionResult r;
        if (dg) {
            const auto& d = *static_cast<const DeviceGraph*>(dg);
            r = kind == 0 ? esia(d, G(g), cs, k, eps, delta, opts)
                          : nsia(d, G(g), cs, k, eps, delta, opts);
        } else {
            SuspectSet vi = dense_suspects(G(g), p_of);
            r = kind == 0 ? esia(G(g), vi, cs, k, eps, delta, opts)
                          : nsia(G(g), vi, cs, k, eps, delta, opts);
        }
        out->k = r.k;
        out->iterations = r.iterations;
        out->coverage = r.coverage;
        out->samples_used = r.samples_used;
        out->attempts = r.attempts;
        out->est_suspension = r.est_suspension;
        out->wall_time_s = r.wall_time_s;
        out->sample_s = r.sample_s;
        out->greedy_s = r.greedy_s;
        out->check_s = r.check_s;
        out->passed_check = r.passed_check ? 1 : 0;
        std::memcpy(solution, r.solution.data(), 4 * r.solution.size());
        if (json && json_cap) {
            std::string j = to_json(r, false);
            std::strncpy(json, j.c_str(), json_cap - 1);
            json[json_cap - 1] = 0;
        }
    });
}

int hsawh_sample(const void* dg, uint64_t target, uint64_t seed, uint64_t max_attempts,
                 uint64_t* attempts, uint64_t* accepted) {
    return guarded([&] {
        SamplerConfig cfg;
        cfg.max_attempts = max_attempts;
        SampleStream stream(*static_cast<const DeviceGraph*>(dg), seed, cfg);
        stream.ensure(target);
        auto c = stream.counters_for(target);
        *attempts = c.attempts;
        *accepted = c.accepted;
    });
}

int hsawh_stream_samples(const void* g, const double* p_of, uint64_t target, uint64_t seed,
                         uint32_t batch_size, uint64_t max_attempts, void** pool_out) {
    return guarded([&] {
        SuspectSet vi = dense_suspects(G(g), p_of);
        SamplerConfig cfg;
        cfg.batch_size = batch_size;
        cfg.max_attempts = max_attempts;
        *pool_out = new SamplePool(stream_samples(G(g), vi, 1, target, seed, cfg));
    });
}

void hsawh_pool_stats(const void* pool, uint64_t* nsamples, uint64_t* attempts,
                      uint64_t* total_edges) {
    const auto& p = *static_cast<const SamplePool*>(pool);
    *nsamples = p.samples.size();
    *attempts = p.attempts;
    uint64_t t = 0;
    for (const auto& s : p.samples) t += s.edge_ids.size();
    *total_edges = t;
}

void hsawh_pool_copy(const void* pool, uint64_t* edge_off, uint32_t* nodes, uint32_t* edges,
                     uint64_t* tag_worker, uint32_t* tag_seq) {
    const auto& p = *static_cast<const SamplePool*>(pool);
    uint64_t eo = 0;
    for (std::size_t w = 0; w < p.samples.size(); ++w) {
        const auto& s = p.samples[w];
        edge_off[w] = eo;
        std::memcpy(nodes + eo + w, s.nodes.data(), 4 * s.nodes.size());
        std::memcpy(edges + eo, s.edge_ids.data(), 4 * s.edge_ids.size());
        eo += s.edge_ids.size();
        if (tag_worker) tag_worker[w] = p.tags[w].worker_id;
        if (tag_seq) tag_seq[w] = p.tags[w].seq;
    }
    edge_off[p.samples.size()] = eo;
}

void hsawh_pool_free(void* pool) { delete static_cast<SamplePool*>(pool); }

int hsawh_graph_load_edge_list_device(const char* path, int weight_mode, uint64_t seed,
                                      int symmetrize, const char* mapping_out, int device,
                                      void** out) {
    return guarded([&] {
        LoadOptions opts;
        opts.symmetrize = symmetrize != 0;
        if (mapping_out) opts.mapping_out = mapping_out;
        *out = new ProbGraph(load_edge_list_device(path, static_cast<WeightMode>(weight_mode), seed,
                                                   opts, device));
    });
}

int hsawh_graph_load_cache_device(const char* path, int device, void** out) {
    return guarded([&] { *out = new ProbGraph(load_cache_device(path, device)); });
}

int hsawh_device_from_cache(const char* path, int device, void* cuda_stream, void** out) {
    return guarded([&] { *out = DeviceGraph::from_cache(path, device, cuda_stream).release(); });
}

int hsawh_device_from_edge_list(const char* path, int weight_mode, int device, void* cuda_stream,
                                void** out) {
    return guarded([&] {
        *out = DeviceGraph::from_edge_list(path, static_cast<WeightMode>(weight_mode), device,
                                           cuda_stream)
                   .release();
    });
}

int hsawh_device_set_suspects(void* dg, const void* g, const double* p_of) {
    return guarded([&] {
        SuspectSet vi = dense_suspects(G(g), p_of);
        static_cast<DeviceGraph*>(dg)->set_suspects(vi);
    });
}

int hsawh_lt_forward_simulate(const void* dg, const void* g, const double* p_of, uint64_t* state,
                              uint32_t* infected) {
    return guarded([&] {
        PrgState s{*state};
        if (dg) {
            *infected = lt_forward_simulate(*static_cast<const DeviceGraph*>(dg), s);
        } else {
            SuspectSet vi = dense_suspects(G(g), p_of);
            *infected = lt_forward_simulate(G(g), vi, s);
        }
        *state = s.state;
    });
}

int hsawh_estimate_suspension(const void* dg, const void* g, const double* p_of, int kind,
                              const uint32_t* ids, uint64_t nids, double eps, double delta,
                              uint64_t* state, double* value, int* capped, uint64_t* runs) {
    return guarded([&] {
        RemovalSet r;
        r.kind = kind == 0 ? ItemKind::Edge : ItemKind::Node;
        r.ids.assign(ids, ids + nids);
        PrgState s{*state};
        SuspensionEstimate e;
        if (dg) {
            e = estimate_suspension(*static_cast<const DeviceGraph*>(dg), r, eps, delta, s);
        } else {
            SuspectSet vi = dense_suspects(G(g), p_of);
            e = estimate_suspension(G(g), vi, r, eps, delta, s);
        }
        *state = s.state;
        *value = e.value;
        *capped = e.capped ? 1 : 0;
        *runs = e.runs;
    });
}

int hsawh_partition(const void* g, uint32_t p, int method, uint64_t seed, const char* part_file,
                    uint32_t hops, uint32_t* assign_out, uint8_t* extended_out) {
    return guarded([&] {
        const ProbGraph& gr = G(g);
        Partitioning part = extend_partition(
            gr, partition_graph(gr, p, static_cast<PartitionMethod>(method), seed,
                                part_file ? part_file : ""), hops);
        if (assign_out) std::memcpy(assign_out, part.assign.data(), 4 * part.assign.size());
        if (extended_out)
            for (std::uint32_t i = 0; i < part.p; ++i)
                std::memcpy(extended_out + static_cast<std::size_t>(i) * gr.n,
                            part.extended[i].data(), gr.n);
    });
}

int hsawh_distributed_sample(const void* dg, uint32_t n, uint32_t p, uint32_t hops,
                             const uint32_t* assign, const uint8_t* extended,
                             uint64_t total_target, uint64_t seed, uint32_t batch_size,
                             uint64_t max_attempts, void** pool_out, uint64_t* crossings,
                             uint64_t* attempts, double* crossing_fraction, uint64_t* targets) {
    return guarded([&] {
        Partitioning part;
        part.p = p;
        part.hops = hops;
        part.assign.assign(assign, assign + n);
        part.base.assign(p, {});
        for (NodeId v = 0; v < n; ++v) {
            if (assign[v] >= p) throw DataError("part id out of range");
            part.base[assign[v]].push_back(v);
        }
        part.extended.resize(p);
        for (std::uint32_t i = 0; i < p; ++i)
            part.extended[i].assign(extended + static_cast<std::size_t>(i) * n,
                                    extended + static_cast<std::size_t>(i + 1) * n);
        SamplerConfig cfg;
        cfg.batch_size = batch_size;
        cfg.max_attempts = max_attempts;
        DistributedResult r = distributed_sample(*static_cast<const DeviceGraph*>(dg), part,
                                                 total_target, seed, cfg);
        *pool_out = new SamplePool(std::move(r.pool));
        *crossings = r.crossings;
        *attempts = r.attempts;
        *crossing_fraction = r.crossing_fraction;
        for (std::uint32_t i = 0; i < p; ++i) targets[i] = r.targets[i];
    });
}

int hsawh_baseline(const void* dg, const void* g, const double* p_of, int kind, int mode,
                   uint32_t k, uint64_t* state, uint32_t infmax_samples, uint32_t* ids_out) {
    return guarded([&] {
        SuspectSet vi = dense_suspects(G(g), p_of);
        PrgState s{*state};
        const auto bk = static_cast<BaselineKind>(kind);
        const ItemKind ik = mode == 0 ? ItemKind::Edge : ItemKind::Node;
        RemovalSet r = dg ? baseline(*static_cast<const DeviceGraph*>(dg), G(g), vi, bk, ik, k, s,
                                     infmax_samples)
                          : baseline(G(g), vi, bk, ik, k, s, infmax_samples);
        *state = s.state;
        std::memcpy(ids_out, r.ids.data(), 4 * r.ids.size());
    });
}

int hsawh_rr_node_sets(const void* dg, uint64_t* state, uint32_t count, uint64_t* set_off,
                       uint32_t* items, uint64_t items_cap, uint64_t* total) {
    return guarded([&] {
        PrgState s{*state};
        auto sets = rr_node_sets(*static_cast<const DeviceGraph*>(dg), s, count);
        uint64_t at = 0;
        set_off[0] = 0;
        for (uint32_t i = 0; i < count; ++i) {
            if (at + sets[i].size() <= items_cap)
                std::memcpy(items + at, sets[i].data(), 4 * sets[i].size());
            at += sets[i].size();
            set_off[i + 1] = at;
        }
        *total = at;
        *state = s.state;
    });
}

int hsawh_interdict_devices(const void* g, const double* p_of, int kind, const uint32_t* cand,
                            uint64_t ncand, uint32_t k, double eps, double delta, uint64_t seed,
                            uint64_t max_attempts, const int* devices, uint32_t ndevices,
                            hsawh_result* out, uint32_t* solution) {
    return guarded([&] {
        const ItemKind ik = kind == 0 ? ItemKind::Edge : ItemKind::Node;
        CandidateSet cs = cand ? CandidateSet::of(ik, std::vector<std::uint32_t>(cand, cand + ncand))
                               : CandidateSet::all(ik);
        InterdictionOptions opts;
        opts.seed = seed;
        opts.sampler.max_attempts = max_attempts;
        opts.devices.assign(devices, devices + ndevices);
        SuspectSet vi = dense_suspects(G(g), p_of);
        InterdictionResult r = kind == 0 ? esia(G(g), vi, cs, k, eps, delta, opts)
                                         : nsia(G(g), vi, cs, k, eps, delta, opts);
        out->k = r.k;
        out->iterations = r.iterations;
        out->coverage = r.coverage;
        out->samples_used = r.samples_used;
        out->attempts = r.attempts;
        out->est_suspension = r.est_suspension;
        out->wall_time_s = r.wall_time_s;
        out->sample_s = r.sample_s;
        out->greedy_s = r.greedy_s;
        out->check_s = r.check_s;
        out->passed_check = r.passed_check ? 1 : 0;
        std::memcpy(solution, r.solution.data(), 4 * r.solution.size());
    });
}

void hsawh_multi_transport(const int* devices, uint32_t ndevices, char* out, uint64_t cap) {
    const std::string s = multi_device_transport(std::vector<int>(devices, devices + ndevices));
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
}

void hsawh_json_number(double x, char* out, uint64_t cap) {
    const std::string s = json_number(x);
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
}

int hsawh_run_cli(int argc, const char** argv) {
    return run_cli(std::vector<std::string>(argv, argv + argc));
}

}  // extern "C"
