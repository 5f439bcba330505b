// TEST INFRASTRUCTURE ONLY — not part of the product path.
//
// C-ABI shim over the UNMODIFIED reference library. The reference sources are
// compiled where they lie (/root/reference/proj/src/*.cpp, see oracle/Makefile)
// and linked with this file into oracle/_ref/libhsaw_ref.so. Nothing from the
// reference is copied: this file only *calls* the public functions declared in
// /root/reference/proj/include/hsaw/*.hpp so that tests/, bench.py's CPU
// baseline leg and the golden-vector generator can drive the real reference
// through ctypes.
//
// Status codes mirror the CLI exit codes of the reference (proj/src/cli.cpp:520-538):
//   0 ok, 1 std::invalid_argument, 2 hsaw::DataError, 3 any other runtime
//   error (SamplingError included), 4 std::out_of_range.

#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "hsaw/coverage.hpp"
#include "hsaw/evaluation.hpp"
#include "hsaw/graph.hpp"
#include "hsaw/interdiction.hpp"
#include "hsaw/partition.hpp"
#include "hsaw/prng.hpp"
#include "hsaw/sampler.hpp"

using namespace hsaw;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

SamplerConfig make_cfg(int heuristic, std::uint32_t window,
                       std::uint32_t batch_size, std::uint64_t max_attempts) {
    SamplerConfig cfg;
    cfg.heuristic = heuristic == 0   ? CycleHeuristic::Brent
                    : heuristic == 1 ? CycleHeuristic::Floyd
                                     : CycleHeuristic::None;
    cfg.window = window;
    cfg.batch_size = batch_size;
    cfg.max_attempts = max_attempts;
    return cfg;
}

CandidateSet make_cand(int kind, const std::uint32_t* ids, std::uint64_t nids,
                       int has_ids) {
    ItemKind k = kind == 0 ? ItemKind::Edge : ItemKind::Node;
    if (!has_ids) return CandidateSet::all(k);
    return CandidateSet::of(k, std::vector<std::uint32_t>(ids, ids + nids));
}

std::vector<std::vector<std::uint32_t>> make_sets(std::uint64_t nsets,
                                                  const std::uint64_t* off,
                                                  const std::uint32_t* items) {
    std::vector<std::vector<std::uint32_t>> sets(nsets);
    for (std::uint64_t i = 0; i < nsets; ++i)
        sets[i].assign(items + off[i], items + off[i + 1]);
    return sets;
}

// id-space-only graph for the raw item-set CoverageIndex constructor
// (proj/src/coverage.cpp:60-74 reads g.m / g.n and nothing else).
ProbGraph id_space(std::uint32_t limit) {
    ProbGraph g;
    g.n = limit;
    g.m = limit;
    return g;
}

struct Pool {
    SamplePool pool;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- prng (proj/include/hsaw/prng.hpp) -------------------------------------
void ref_splitmix_next(std::uint64_t state, std::uint64_t* out_state,
                       std::uint64_t* out_output) {
    auto r = splitmix_next(state);
    *out_state = r.state;
    *out_output = r.output;
}
std::uint64_t ref_prg_next(std::uint64_t* state) {
    PrgState s{*state};
    std::uint64_t o = prg_next(s);
    *state = s.state;
    return o;
}
double ref_u01(std::uint64_t output) { return u01(output); }
std::uint64_t ref_seed_from_worker(std::uint64_t worker_id) {
    return seed_from_worker(worker_id).state;
}
std::uint32_t ref_pick_uniform_node(std::uint64_t* state, std::uint32_t n) {
    PrgState s{*state};
    NodeId v = pick_uniform_node(s, n);
    *state = s.state;
    return v;
}

// ---- graphs -----------------------------------------------------------------
// Direct CSR fill, no validate(): the survey (§0) shows validate() rejects
// InDegree rows with d >= 36217, so bench graphs enter both sides this way.
void* ref_graph_from_csr(std::uint32_t n, std::uint32_t m,
                         const std::uint64_t* in_offsets,
                         const std::uint32_t* in_src, const double* in_cum) {
    auto* g = new ProbGraph;
    g->n = n;
    g->m = m;
    g->in_offsets.assign(in_offsets, in_offsets + n + 1);
    g->in_src.assign(in_src, in_src + m);
    g->in_cum.assign(in_cum, in_cum + m);
    g->weight.resize(m);
    g->edge_dst.resize(m);
    for (std::uint32_t v = 0; v < n; ++v) {
        double prev = 0.0;
        for (std::uint64_t i = in_offsets[v]; i < in_offsets[v + 1]; ++i) {
            g->weight[i] = in_cum[i] - prev;
            prev = in_cum[i];
            g->edge_dst[i] = v;
        }
    }
    return g;
}

// Sampler-only variant for the 10^9-edge bench shapes: weight / edge_dst stay
// empty (run_walk_attempt and decode read in_offsets / in_src / in_cum only,
// proj/src/sampler.cpp:16-62, graph.hpp:61-80), 12 instead of 24 bytes per edge.
void* ref_graph_from_csr_lean(std::uint32_t n, std::uint32_t m,
                              const std::uint64_t* in_offsets,
                              const std::uint32_t* in_src,
                              const double* in_cum) {
    auto* g = new ProbGraph;
    g->n = n;
    g->m = m;
    g->in_offsets.assign(in_offsets, in_offsets + n + 1);
    g->in_src.assign(in_src, in_src + m);
    g->in_cum.assign(in_cum, in_cum + m);
    return g;
}

int ref_graph_build(std::uint32_t n, std::uint64_t ne, const std::uint32_t* u,
                    const std::uint32_t* v, const double* w, int mode,
                    std::uint64_t seed, void** out) {
    return guarded([&] {
        std::vector<std::tuple<NodeId, NodeId, double>> edges;
        edges.reserve(ne);
        for (std::uint64_t i = 0; i < ne; ++i)
            edges.emplace_back(u[i], v[i], w ? w[i] : 0.0);
        *out = new ProbGraph(build_graph(
            n, std::move(edges), static_cast<WeightMode>(mode), seed));
    });
}

int ref_graph_load_edge_list(const char* path, int mode, std::uint64_t seed,
                             int symmetrize, const char* mapping_out,
                             void** out) {
    return guarded([&] {
        LoadOptions opts;
        opts.symmetrize = symmetrize != 0;
        if (mapping_out) opts.mapping_out = mapping_out;
        *out = new ProbGraph(
            load_edge_list(path, static_cast<WeightMode>(mode), seed, opts));
    });
}

int ref_graph_synth(std::uint32_t n, std::uint32_t density, std::uint64_t seed,
                    void** out) {
    return guarded(
        [&] { *out = new ProbGraph(synth_graph(n, density, seed)); });
}

int ref_graph_save_cache(void* g, const char* path) {
    return guarded([&] { save_cache(*static_cast<ProbGraph*>(g), path); });
}
int ref_graph_load_cache(const char* path, void** out) {
    return guarded([&] { *out = new ProbGraph(load_cache(path)); });
}
int ref_graph_save_edge_list(void* g, const char* path) {
    return guarded([&] { save_edge_list(*static_cast<ProbGraph*>(g), path); });
}
int ref_graph_validate(void* g) {
    return guarded([&] { static_cast<ProbGraph*>(g)->validate(); });
}

void ref_graph_dims(void* gp, std::uint32_t* n, std::uint32_t* m) {
    auto* g = static_cast<ProbGraph*>(gp);
    *n = g->n;
    *m = g->m;
}

void ref_graph_copy(void* gp, std::uint64_t* in_offsets, std::uint32_t* in_src,
                    double* in_cum, double* weight, std::uint32_t* edge_dst) {
    auto* g = static_cast<ProbGraph*>(gp);
    if (in_offsets)
        std::memcpy(in_offsets, g->in_offsets.data(), 8 * g->in_offsets.size());
    if (in_src) std::memcpy(in_src, g->in_src.data(), 4 * g->in_src.size());
    if (in_cum) std::memcpy(in_cum, g->in_cum.data(), 8 * g->in_cum.size());
    if (weight) std::memcpy(weight, g->weight.data(), 8 * g->weight.size());
    if (edge_dst)
        std::memcpy(edge_dst, g->edge_dst.data(), 4 * g->edge_dst.size());
}

void ref_graph_free(void* g) { delete static_cast<ProbGraph*>(g); }

// ---- suspects ---------------------------------------------------------------
// Dense p_of (0 = not a suspect) -> SuspectSet through from_members.
int ref_suspects_from_p(void* gp, const double* p_of, void** out) {
    return guarded([&] {
        auto* g = static_cast<ProbGraph*>(gp);
        std::vector<std::pair<NodeId, double>> mem;
        for (NodeId v = 0; v < g->n; ++v)
            if (p_of[v] != 0.0) mem.emplace_back(v, p_of[v]);
        *out = new SuspectSet(SuspectSet::from_members(std::move(mem), *g));
    });
}
int ref_suspects_random(void* gp, std::uint32_t count, std::uint64_t seed,
                        void** out) {
    return guarded([&] {
        *out = new SuspectSet(
            random_suspects(*static_cast<ProbGraph*>(gp), count, seed));
    });
}
int ref_suspects_load(const char* path, void* gp, void** out) {
    return guarded([&] {
        *out = new SuspectSet(load_suspects(path, *static_cast<ProbGraph*>(gp)));
    });
}
void ref_suspects_copy_p(void* vip, double* p_of) {
    auto* vi = static_cast<SuspectSet*>(vip);
    std::memcpy(p_of, vi->p_of.data(), 8 * vi->p_of.size());
}
std::uint64_t ref_suspects_size(void* vip) {
    return static_cast<SuspectSet*>(vip)->size();
}
void ref_suspects_free(void* vi) { delete static_cast<SuspectSet*>(vi); }

// ---- sampler ----------------------------------------------------------------
// thread_sample (proj/src/sampler.cpp:267-290): returns the number of encoded
// walks; seeds/lens must hold l entries.
std::int64_t ref_thread_sample(void* gp, void* vip, std::uint64_t worker_id,
                               std::uint32_t l, int heuristic,
                               std::uint32_t window, std::uint64_t* seeds,
                               std::uint32_t* lens) {
    std::int64_t count = -1;
    int rc = guarded([&] {
        SamplerConfig cfg = make_cfg(heuristic, window, 10, 100'000'000);
        auto walks = thread_sample(*static_cast<ProbGraph*>(gp),
                                   *static_cast<SuspectSet*>(vip), worker_id, l,
                                   cfg);
        for (std::size_t i = 0; i < walks.size(); ++i) {
            seeds[i] = walks[i].seed.state;
            lens[i] = walks[i].len;
        }
        count = static_cast<std::int64_t>(walks.size());
    });
    return rc == 0 ? count : -rc;
}

// DecodeContext::decode (proj/src/sampler.cpp:295-338): 1 decoded, 0 dropped
// (missed cycle), negative = -status. nodes holds len+1, edges holds len.
int ref_decode(void* gp, void* vip, std::uint64_t seed, std::uint32_t len,
               std::uint32_t* nodes, std::uint32_t* edges) {
    int result = 0;
    int rc = guarded([&] {
        EncodedWalk ew{PrgState{seed}, len, 0, 0};
        auto s = decode_walk(*static_cast<ProbGraph*>(gp),
                             *static_cast<SuspectSet*>(vip), ew);
        if (!s) {
            result = 0;
            return;
        }
        std::memcpy(nodes, s->nodes.data(), 4 * s->nodes.size());
        std::memcpy(edges, s->edge_ids.data(), 4 * s->edge_ids.size());
        result = 1;
    });
    return rc == 0 ? result : -rc;
}

int ref_stream_samples(void* gp, void* vip, std::uint32_t workers,
                       std::uint64_t target, std::uint64_t seed, int heuristic,
                       std::uint32_t window, std::uint32_t batch_size,
                       std::uint64_t max_attempts, void** out) {
    return guarded([&] {
        SamplerConfig cfg = make_cfg(heuristic, window, batch_size, max_attempts);
        auto* p = new Pool;
        try {
            p->pool = stream_samples(*static_cast<ProbGraph*>(gp),
                                     *static_cast<SuspectSet*>(vip), workers,
                                     target, seed, cfg);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

void ref_pool_stats(void* pp, std::uint64_t* nsamples, std::uint64_t* attempts,
                    std::uint64_t* total_edges) {
    auto* p = static_cast<Pool*>(pp);
    *nsamples = p->pool.samples.size();
    *attempts = p->pool.attempts;
    std::uint64_t t = 0;
    for (const auto& s : p->pool.samples) t += s.edge_ids.size();
    *total_edges = t;
}

// edge_off has nsamples+1 entries; walk w has edges [edge_off[w], edge_off[w+1])
// and nodes [edge_off[w]+w, edge_off[w+1]+w+1).
void ref_pool_copy(void* pp, std::uint64_t* edge_off, std::uint32_t* nodes,
                   std::uint32_t* edges, std::uint64_t* tag_worker,
                   std::uint32_t* tag_seq) {
    auto* p = static_cast<Pool*>(pp);
    std::uint64_t eo = 0;
    for (std::size_t w = 0; w < p->pool.samples.size(); ++w) {
        const auto& s = p->pool.samples[w];
        edge_off[w] = eo;
        std::memcpy(nodes + eo + w, s.nodes.data(), 4 * s.nodes.size());
        std::memcpy(edges + eo, s.edge_ids.data(), 4 * s.edge_ids.size());
        eo += s.edge_ids.size();
        if (tag_worker) tag_worker[w] = p->pool.tags[w].worker_id;
        if (tag_seq) tag_seq[w] = p->pool.tags[w].seq;
    }
    edge_off[p->pool.samples.size()] = eo;
}

void ref_pool_free(void* p) { delete static_cast<Pool*>(p); }

// ---- ranking baselines (proj/include/hsaw/evaluation.hpp:45-50) ---------------
// kind: 0 Pagerank, 1 MaxDegree, 2 Randomized, 3 InfMaxV, 4 InfMaxVI; ids_out holds k ids
int ref_baseline(void* gp, void* vip, int kind, int mode, std::uint32_t k,
                 std::uint64_t* state, std::uint32_t infmax_samples,
                 std::uint32_t* ids_out) {
    return guarded([&] {
        PrgState s{*state};
        RemovalSet r = baseline(*static_cast<ProbGraph*>(gp), *static_cast<SuspectSet*>(vip),
                                static_cast<BaselineKind>(kind),
                                mode == 0 ? ItemKind::Edge : ItemKind::Node, k, s,
                                infmax_samples);
        *state = s.state;
        std::memcpy(ids_out, r.ids.data(), 4 * r.ids.size());
    });
}

// ---- partitioned sampling (proj/include/hsaw/partition.hpp) -------------------
// method: 0 Hash, 1 LabelProp, 2 = the given assignment (what ExternalFile reads,
// built without the file: assign + rebuild_base + extend_partition(.., 0)).
int ref_partition_graph(void* gp, std::uint32_t p, int method, std::uint64_t seed,
                        const std::uint32_t* assign, void** out) {
    return guarded([&] {
        auto& g = *static_cast<ProbGraph*>(gp);
        if (method == 2) {
            if (p < 1 || p > g.n) throw DataError("part count must be in [1, n]");
            Partitioning part;
            part.p = p;
            part.assign.assign(assign, assign + g.n);
            part.base.assign(p, {});
            for (NodeId v = 0; v < g.n; ++v) {
                if (part.assign[v] >= p) throw DataError("part id out of range");
                part.base[part.assign[v]].push_back(v);
            }
            *out = new Partitioning(extend_partition(g, std::move(part), 0));
        } else {
            *out = new Partitioning(partition_graph(
                g, p, method == 0 ? PartitionMethod::Hash : PartitionMethod::LabelProp, seed));
        }
    });
}
int ref_extend_partition(void* gp, void* partp, std::uint32_t h, void** out) {
    return guarded([&] {
        *out = new Partitioning(extend_partition(*static_cast<ProbGraph*>(gp),
                                                 *static_cast<Partitioning*>(partp), h));
    });
}
// assign u32[n]; extended u8[p * n] (part-major); either may be null
void ref_partition_copy(void* partp, std::uint32_t* assign, std::uint8_t* extended) {
    auto& part = *static_cast<Partitioning*>(partp);
    if (assign) std::memcpy(assign, part.assign.data(), 4 * part.assign.size());
    if (extended)
        for (std::uint32_t i = 0; i < part.p; ++i)
            std::memcpy(extended + static_cast<std::size_t>(i) * part.assign.size(),
                        part.extended[i].data(), part.extended[i].size());
}
void ref_partition_free(void* partp) { delete static_cast<Partitioning*>(partp); }

// distributed_sample: pool handle (ref_pool_*), crossings, attempts, targets u64[p]
int ref_distributed_sample(void* gp, void* vip, void* partp, std::uint64_t total_target,
                           std::uint64_t seed, std::uint32_t workers, int heuristic,
                           std::uint32_t window, std::uint32_t batch_size,
                           std::uint64_t max_attempts, void** pool_out,
                           std::uint64_t* crossings, std::uint64_t* attempts,
                           double* crossing_fraction, std::uint64_t* targets) {
    return guarded([&] {
        SamplerConfig cfg = make_cfg(heuristic, window, batch_size, max_attempts);
        auto& part = *static_cast<Partitioning*>(partp);
        DistributedResult r = distributed_sample(*static_cast<ProbGraph*>(gp),
                                                 *static_cast<SuspectSet*>(vip), part,
                                                 total_target, seed, workers, cfg);
        auto* p = new Pool;
        p->pool = std::move(r.pool);
        *pool_out = p;
        *crossings = r.crossings;
        *attempts = r.attempts;
        *crossing_fraction = r.crossing_fraction;
        for (std::uint32_t i = 0; i < part.p; ++i) targets[i] = r.targets[i];
    });
}

// ---- coverage / greedy on raw item sets (fixed-walk-set mode) ---------------
int ref_greedy(int kind, std::uint32_t limit, std::uint64_t nsets,
               const std::uint64_t* set_off, const std::uint32_t* items,
               const std::uint32_t* cand_ids, std::uint64_t ncand, int has_cand,
               std::uint32_t k, int naive, std::uint32_t* solution,
               std::uint64_t* coverage) {
    return guarded([&] {
        ProbGraph g = id_space(limit);
        auto sets = make_sets(nsets, set_off, items);
        CandidateSet cand = make_cand(kind, cand_ids, ncand, has_cand);
        CoverageIndex idx(sets, cand, g);
        GreedyResult r =
            naive ? greedy_max_cover_naive(idx, k) : greedy_max_cover(idx, k);
        std::memcpy(solution, r.solution.data(), 4 * r.solution.size());
        *coverage = r.coverage;
    });
}

int ref_coverage_of(int kind, std::uint32_t limit, std::uint64_t nsets,
                    const std::uint64_t* set_off, const std::uint32_t* items,
                    const std::uint32_t* cand_ids, std::uint64_t ncand,
                    int has_cand, const std::uint32_t* query,
                    std::uint64_t nquery, std::uint64_t* coverage) {
    return guarded([&] {
        ProbGraph g = id_space(limit);
        auto sets = make_sets(nsets, set_off, items);
        CandidateSet cand = make_cand(kind, cand_ids, ncand, has_cand);
        CoverageIndex idx(sets, cand, g);
        *coverage = idx.coverage_of({query, nquery});
    });
}

// out4 = {n_max, lambda, lambda1, (double)lambda_samples}
int ref_schedule(std::uint64_t M, std::uint32_t k, double eps, double delta,
                 double* out4, std::uint32_t* t_max) {
    return guarded([&] {
        Schedule s = compute_schedule_m(M, k, eps, delta);
        out4[0] = s.n_max;
        out4[1] = s.lambda;
        out4[2] = s.lambda1;
        out4[3] = static_cast<double>(s.lambda_samples());
        *t_max = s.t_max;
    });
}

double ref_ln_choose(std::uint64_t M, std::uint64_t k) { return ln_choose(M, k); }

int ref_check_solution(int kind, std::uint32_t limit, std::uint64_t nsets_r,
                       const std::uint64_t* off_r, const std::uint32_t* items_r,
                       std::uint64_t nsets_rp, const std::uint64_t* off_rp,
                       const std::uint32_t* items_rp,
                       const std::uint32_t* cand_ids, std::uint64_t ncand,
                       int has_cand, const std::uint32_t* solution,
                       std::uint64_t nsol, std::uint64_t M, std::uint32_t k,
                       double eps, double delta, std::uint32_t t, int* pass,
                       double* eps_t) {
    return guarded([&] {
        ProbGraph g = id_space(limit);
        CandidateSet cand = make_cand(kind, cand_ids, ncand, has_cand);
        auto sr = make_sets(nsets_r, off_r, items_r);
        auto srp = make_sets(nsets_rp, off_rp, items_rp);
        CoverageIndex r(sr, cand, g), rp(srp, cand, g);
        Schedule sched = compute_schedule_m(M, k, eps, delta);
        CheckResult c = check_solution({solution, nsol}, r, rp, sched, t);
        *pass = c.pass ? 1 : 0;
        *eps_t = c.eps_t;
    });
}

// ---- interdiction -----------------------------------------------------------
struct RefResult {
    std::uint32_t k;
    std::uint32_t iterations;
    std::uint64_t coverage;
    std::uint64_t samples_used;
    std::uint64_t attempts;
    double est_suspension;
    double wall_time_s;
    int passed_check;
};

int ref_interdict(void* gp, void* vip, int kind, const std::uint32_t* cand_ids,
                  std::uint64_t ncand, int has_cand, std::uint32_t k, double eps,
                  double delta, std::uint32_t workers, std::uint64_t seed,
                  std::uint32_t batch_size, std::uint64_t max_attempts,
                  RefResult* out, std::uint32_t* solution, char* json,
                  std::uint64_t json_cap) {
    return guarded([&] {
        InterdictionOptions opts;
        opts.workers = workers;
        opts.seed = seed;
        opts.sampler.batch_size = batch_size;
        opts.sampler.max_attempts = max_attempts;
        CandidateSet cand = make_cand(kind, cand_ids, ncand, has_cand);
        auto& g = *static_cast<ProbGraph*>(gp);
        auto& vi = *static_cast<SuspectSet*>(vip);
        InterdictionResult r = kind == 0 ? esia(g, vi, cand, k, eps, delta, opts)
                                         : nsia(g, vi, cand, k, eps, delta, opts);
        out->k = r.k;
        out->iterations = r.iterations;
        out->coverage = r.coverage;
        out->samples_used = r.samples_used;
        out->attempts = r.attempts;
        out->est_suspension = r.est_suspension;
        out->wall_time_s = r.wall_time_s;
        out->passed_check = r.passed_check ? 1 : 0;
        std::memcpy(solution, r.solution.data(), 4 * r.solution.size());
        if (json && json_cap) {
            std::string j = to_json(r, false);
            std::strncpy(json, j.c_str(), json_cap - 1);
            json[json_cap - 1] = 0;
        }
    });
}

// ---- paired LT forward simulation (proj/include/hsaw/evaluation.hpp:16-39) ----
int ref_lt_forward_simulate(void* gp, void* vip, std::uint64_t* state,
                            std::uint32_t* infected) {
    return guarded([&] {
        PrgState s{*state};
        *infected = lt_forward_simulate(*static_cast<ProbGraph*>(gp),
                                        *static_cast<SuspectSet*>(vip), s);
        *state = s.state;
    });
}
int ref_estimate_suspension(void* gp, void* vip, int kind,
                            const std::uint32_t* ids, std::uint64_t nids,
                            double epsilon, double delta, std::uint64_t* state,
                            double* value, int* capped, std::uint64_t* runs) {
    return guarded([&] {
        RemovalSet r;
        r.kind = kind == 0 ? ItemKind::Edge : ItemKind::Node;
        r.ids.assign(ids, ids + nids);
        PrgState s{*state};
        SuspensionEstimate e = estimate_suspension(
            *static_cast<ProbGraph*>(gp), *static_cast<SuspectSet*>(vip), r,
            epsilon, delta, s);
        *state = s.state;
        *value = e.value;
        *capped = e.capped ? 1 : 0;
        *runs = e.runs;
    });
}

}  // extern "C"
