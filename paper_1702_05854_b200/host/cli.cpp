// `hsaw` command line on the device path: the subcommands and flags of the reference CLI that sit
// on the hot path (interdict, sample, bench, synth, estimate — /root/reference/proj/src/cli.cpp:400-485), the
// same JSON documents and the same exit codes (0 ok, 1 usage, 2 data, 3 runtime; cli.cpp:520-538).
// The reference parses with CLI11 (not available here); this is a small flag parser with the same
// spelling: `--name value` or `--name=value`. `--workers` is accepted and ignored (the GPU is the
// worker pool); `--device N` is new. baseline / partition are outside the ported path.
#include <charconv>
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>

#include "hsaw_b200.hpp"

namespace hsaw {

namespace {

struct UsageError : std::runtime_error {
    explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};

struct Flags {
    std::map<std::string, std::string> values;
    std::set<std::string> switches;

    bool has(const std::string& name) const { return values.count(name) != 0; }
    std::string str(const std::string& name, const std::string& dflt = "") const {
        auto it = values.find(name);
        return it == values.end() ? dflt : it->second;
    }
    std::uint64_t u64(const std::string& name, std::uint64_t dflt) const {
        if (!has(name)) return dflt;
        const std::string& v = values.at(name);
        try {
            std::size_t used = 0;
            if (!v.empty() && v[0] == '-') throw UsageError("");
            std::uint64_t x = std::stoull(v, &used);
            if (used != v.size()) throw UsageError("");
            return x;
        } catch (...) {
            throw UsageError("--" + name + ": expected a non-negative integer, got '" + v + "'");
        }
    }
    double real(const std::string& name, double dflt) const {
        if (!has(name)) return dflt;
        const std::string& v = values.at(name);
        try {
            std::size_t used = 0;
            double x = std::stod(v, &used);
            if (used != v.size()) throw UsageError("");
            return x;
        } catch (...) {
            throw UsageError("--" + name + ": expected a number, got '" + v + "'");
        }
    }
    void require(const std::string& name) const {
        if (!has(name)) throw UsageError("--" + name + " is required");
    }
};

Flags parse_flags(const std::vector<std::string>& args, std::size_t from,
                  const std::set<std::string>& valued, const std::set<std::string>& boolean) {
    Flags f;
    for (std::size_t i = from; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
        std::string name = a.substr(2), value;
        bool inline_value = false;
        if (auto eq = name.find('='); eq != std::string::npos) {
            value = name.substr(eq + 1);
            name = name.substr(0, eq);
            inline_value = true;
        }
        if (boolean.count(name)) {
            f.switches.insert(name);
            continue;
        }
        if (!valued.count(name)) throw UsageError("unknown option --" + name);
        if (!inline_value) {
            if (i + 1 >= args.size()) throw UsageError("--" + name + " needs a value");
            value = args[++i];
        }
        f.values[name] = value;
    }
    return f;
}

WeightMode weight_mode(const std::string& w) {
    if (w == "given") return WeightMode::Given;
    if (w == "indegree") return WeightMode::InDegree;
    if (w == "random-normalized") return WeightMode::RandomNormalized;
    throw UsageError("--weights: expected given|indegree|random-normalized");
}

// GraphArgs::load, cli.cpp:38-48: binary caches load directly, else the edge list.
// on_host: the command itself never touches the device (`partition` without --target), so the
// host loaders are used (same ProbGraph, same errors).
ProbGraph load_graph(const Flags& f, std::uint64_t seed, bool on_host = false) {
    const std::string path = f.str("graph");
    {
        std::ifstream probe(path, std::ios::binary);
        char magic[5] = {};
        // binary caches are decoded, summed and validated on the device (same ProbGraph, same errors)
        if (probe.read(magic, 5) && std::string(magic, 5) == "HSAW1")
            return on_host ? load_cache(path)
                           : load_cache_device(path, static_cast<int>(f.u64("device", 0)));
    }
    LoadOptions opts;
    opts.symmetrize = f.switches.count("symmetrize") != 0;
    if (on_host) return load_edge_list(path, weight_mode(f.str("weights", "indegree")), 0, opts);
    // text edge lists are parsed, re-ranked, sorted and summed on the device; anything outside the
    // device parser's plain grammar goes through the host parser inside this call
    // the reference's GraphArgs::seed is never bound to --seed (proj/src/cli.cpp:28,47,410): the
    // graph is always loaded with seed 0, --seed drives suspects and sampling only
    (void)seed;
    return load_edge_list_device(path, weight_mode(f.str("weights", "indegree")), 0, opts,
                                 static_cast<int>(f.u64("device", 0)));
}

SuspectSet load_suspect_args(const Flags& f, const ProbGraph& g, std::uint64_t seed) {
    if (f.has("suspects")) return load_suspects(f.str("suspects"), g);
    const std::uint64_t count = f.u64("random-suspects", 0);
    if (count > 0) return random_suspects(g, static_cast<NodeId>(count), seed);
    throw UsageError("one of --suspects or --random-suspects is required");
}

void emit(const std::string& text, const std::string& output) {
    if (output.empty()) {
        std::cout << text << '\n';
        return;
    }
    std::ofstream f(output);
    if (!f) throw DataError("cannot write output: " + output);
    f << text << '\n';
}

// read_item_file, cli.cpp:95-136: one id per line, or "u v" naming an edge by its endpoints.
std::vector<std::uint32_t> read_item_file(const std::string& path, ItemKind kind,
                                          const ProbGraph& g) {
    std::ifstream in(path);
    if (!in) throw DataError("cannot open item file: " + path);
    std::map<std::pair<NodeId, NodeId>, EdgeId> by_endpoints;
    if (kind == ItemKind::Edge)
        for (EdgeId e = 0; e < g.m; ++e) by_endpoints[g.endpoints(e)] = e;
    std::vector<std::uint32_t> ids;
    std::string line;
    for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
        std::istringstream row(line);
        std::vector<std::uint64_t> nums;
        for (std::uint64_t x; row >> x;) nums.push_back(x);
        if (nums.empty()) continue;
        if (nums.size() == 1) {
            ids.push_back(static_cast<std::uint32_t>(nums[0]));
        } else if (nums.size() == 2 && kind == ItemKind::Edge) {
            auto it = by_endpoints.find({static_cast<NodeId>(nums[0]), static_cast<NodeId>(nums[1])});
            if (it == by_endpoints.end())
                throw DataError(path + ":" + std::to_string(lineno) + ": unknown edge " +
                                std::to_string(nums[0]) + " -> " + std::to_string(nums[1]));
            ids.push_back(it->second);
        } else {
            throw DataError(path + ":" + std::to_string(lineno) + ": malformed line");
        }
    }
    return ids;
}

std::string json_real(double x) {
    std::ostringstream s;
    s.precision(17);
    s << x;
    return s.str();
}

// nlohmann's number form (json_number, solver.cpp)
std::string json_shortest(double x) { return json_number(x); }

const std::set<std::string> kGraphFlags = {"graph", "weights", "suspects", "random-suspects"};

std::set<std::string> with(std::set<std::string> base, std::initializer_list<const char*> more) {
    for (const char* m : more) base.insert(m);
    return base;
}

int cmd_interdict(const Flags& f) {  // cli.cpp:138-160
    f.require("graph");
    f.require("k");
    const std::uint64_t k = f.u64("k", 1);
    if (k < 1) {
        std::cerr << "error: --k must be at least 1\n";
        return 1;
    }
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = load_graph(f, seed);
    SuspectSet vi = load_suspect_args(f, g, seed);
    const std::string mode = f.str("mode", "edge");
    if (mode != "edge" && mode != "node") throw UsageError("--mode: expected edge|node");
    const ItemKind kind = mode == "edge" ? ItemKind::Edge : ItemKind::Node;
    CandidateSet cand = CandidateSet::all(kind);
    const std::string cand_path = f.str("candidates", "all");
    if (!cand_path.empty() && cand_path != "all")
        cand = CandidateSet::of(kind, read_item_file(cand_path, kind, g));
    InterdictionOptions opts;
    opts.workers = static_cast<std::uint32_t>(f.u64("workers", 1));
    opts.seed = seed;
    opts.sampler.max_attempts = f.u64("max-attempts", 100'000'000);
    opts.device = static_cast<int>(f.u64("device", 0));
    // --gpus N: devices 0..N-1 (graph replicated, walks sharded, NCCL); --devices a,b,c: an explicit
    // list (a repeated id runs the same path over the in-process exchange: one-GPU boxes)
    if (f.has("devices")) {
        std::stringstream ss(f.str("devices"));
        std::string tok;
        while (std::getline(ss, tok, ',')) opts.devices.push_back(std::stoi(tok));
    } else if (f.u64("gpus", 1) > 1) {
        for (std::uint64_t d = 0; d < f.u64("gpus", 1); ++d) opts.devices.push_back(static_cast<int>(d));
    }
    if (opts.devices.size() > 1)
        std::cerr << "hsaw: multi-device solve over " << opts.devices.size() << " devices, transport: "
                  << multi_device_transport(opts.devices) << '\n';
    const double eps = f.real("epsilon", 0.1), delta = f.real("delta", 0.1);
    InterdictionResult res = kind == ItemKind::Edge
                                 ? esia(g, vi, cand, static_cast<std::uint32_t>(k), eps, delta, opts)
                                 : nsia(g, vi, cand, static_cast<std::uint32_t>(k), eps, delta, opts);
    emit(to_json(res, f.switches.count("omit-timing") == 0), f.str("output"));
    return 0;
}

int cmd_sample(const Flags& f) {  // cli.cpp:267-290
    f.require("graph");
    f.require("target");
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = load_graph(f, seed);
    SuspectSet vi = load_suspect_args(f, g, seed);
    SamplerConfig cfg;
    cfg.max_attempts = f.u64("max-attempts", 100'000'000);
    const std::uint64_t target = f.u64("target", 0);
    DeviceGraph dg(g, vi, static_cast<int>(f.u64("device", 0)));
    SampleStream stream(dg, seed, cfg);
    stream.ensure(target);
    std::ostringstream j;
    if (f.has("dump")) {  // only the dump needs the walks on the host
        SamplePool pool = stream.to_pool(target);
        std::ofstream df(f.str("dump"));
        if (!df) throw DataError("cannot write dump: " + f.str("dump"));
        dump_walks(pool, df);
    }
    const auto c = stream.counters_for(target);
    if (c.attempts == 0) throw std::invalid_argument("estimate_influence: no attempts");
    const double rate = static_cast<double>(c.accepted) / static_cast<double>(c.attempts);
    j << "{\n  \"acceptance_rate\": " << json_real(rate) << ",\n  \"accepted\": " << c.accepted
      << ",\n  \"attempts\": " << c.attempts << ",\n  \"est_influence\": "
      << json_real(static_cast<double>(g.n) * static_cast<double>(c.accepted) /
                   static_cast<double>(c.attempts))
      << ",\n  \"target\": " << target << "\n}";
    emit(j.str(), f.str("output"));
    return 0;
}

int cmd_estimate(const Flags& f) {  // cli.cpp:162-185
    f.require("graph");
    f.require("removal");
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = load_graph(f, seed);
    SuspectSet vi = load_suspect_args(f, g, seed);
    const std::string mode = f.str("mode", "edge");
    if (mode != "edge" && mode != "node") throw UsageError("--mode: expected edge|node");
    RemovalSet removal;
    removal.kind = mode == "edge" ? ItemKind::Edge : ItemKind::Node;
    removal.ids = read_item_file(f.str("removal"), removal.kind, g);
    removal.validate(g);
    const double eps = f.real("epsilon", 0.1), delta = f.real("delta", 0.1);
    PrgState s = seed_from_worker(seed);
    SuspensionEstimate est;
    // argument checks first, as the reference does before any simulation (evaluation.cpp:214-218)
    if (!(eps > 0.0) || eps >= 1.0) throw std::invalid_argument("epsilon must be in (0,1)");
    if (!(delta > 0.0) || delta >= 1.0) throw std::invalid_argument("delta must be in (0,1)");
    if (!removal.ids.empty()) {
        DeviceGraph dg(g, vi, static_cast<int>(f.u64("device", 0)));
        est = estimate_suspension(dg, removal, eps, delta, s);
    }
    std::ostringstream j;  // nlohmann object: keys sorted, dump(2)
    j << "{\n  \"capped\": " << (est.capped ? "true" : "false") << ",\n  \"delta\": "
      << json_shortest(delta) << ",\n  \"epsilon\": " << json_shortest(eps) << ",\n  \"kind\": \""
      << to_string(removal.kind) << "\",\n  \"removed\": " << removal.ids.size()
      << ",\n  \"runs\": " << est.runs << ",\n  \"suspension\": " << json_shortest(est.value)
      << "\n}";
    emit(j.str(), f.str("output"));
    return 0;
}

int cmd_synth(const Flags& f) {  // cli.cpp:335-348
    f.require("nodes");
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = synth_graph(static_cast<NodeId>(f.u64("nodes", 0)),
                              static_cast<std::uint32_t>(f.u64("density", 10)), seed);
    if (f.has("out")) save_edge_list(g, f.str("out"));
    if (f.has("cache")) save_cache(g, f.str("cache"));
    std::cout << "{\n  \"edges\": " << g.m << ",\n  \"nodes\": " << g.n << ",\n  \"seed\": " << seed
              << "\n}\n";
    return 0;
}

int cmd_bench(const Flags& f) {  // cli.cpp:350-379, one device run instead of 1 / N workers
    f.require("target");
    const std::uint64_t seed = f.u64("seed", 0);
    const std::uint64_t synth_nodes = f.u64("synth-nodes", 0);
    ProbGraph g = synth_nodes > 0
                      ? synth_graph(static_cast<NodeId>(synth_nodes),
                                    static_cast<std::uint32_t>(f.u64("synth-density", 10)), seed)
                      : (f.require("graph"), load_graph(f, seed));
    SuspectSet vi = load_suspect_args(f, g, seed);
    const std::uint64_t target = f.u64("target", 0);
    DeviceGraph dg(g, vi, static_cast<int>(f.u64("device", 0)));
    const auto t0 = std::chrono::steady_clock::now();
    SampleStream stream(dg, seed);
    stream.ensure(target);
    const auto c = stream.counters_for(target);
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::ostringstream j;
    j << "{\n  \"edges\": " << g.m << ",\n  \"nodes\": " << g.n << ",\n  \"runs\": [\n    {\n"
      << "      \"accepted\": " << c.accepted << ",\n      \"attempts\": " << c.attempts
      << ",\n      \"attempts_per_sec\": " << json_real(static_cast<double>(c.attempts) / secs)
      << ",\n      \"device\": " << f.u64("device", 0) << ",\n      \"seconds\": " << json_real(secs)
      << "\n    }\n  ],\n  \"target\": " << target << "\n}";
    emit(j.str(), f.str("output"));
    return 0;
}

// nlohmann dump(2) of an integer array value at nesting depth 1
template <class T>
std::string json_int_array(const std::vector<T>& xs) {
    if (xs.empty()) return "[]";
    std::ostringstream o;
    o << "[";
    for (std::size_t i = 0; i < xs.size(); ++i) o << (i ? ",\n    " : "\n    ") << xs[i];
    o << "\n  ]";
    return o.str();
}

ItemKind parse_item_mode(const std::string& mode) {
    if (mode == "edge") return ItemKind::Edge;
    if (mode == "node") return ItemKind::Node;
    throw UsageError("--mode: expected edge|node");
}

BaselineKind parse_baseline_kind(const std::string& name) {  // cli.cpp:187-195
    if (name == "pagerank") return BaselineKind::Pagerank;
    if (name == "maxdegree") return BaselineKind::MaxDegree;
    if (name == "randomized") return BaselineKind::Randomized;
    if (name == "infmax-v") return BaselineKind::InfMaxV;
    if (name == "infmax-vi") return BaselineKind::InfMaxVI;
    throw UsageError("--method: expected pagerank|maxdegree|randomized|infmax-v|infmax-vi");
}

int cmd_baseline(const Flags& f) {  // cli.cpp:197-265
    f.require("graph");
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = load_graph(f, seed);
    SuspectSet vi = load_suspect_args(f, g, seed);
    const ItemKind kind = parse_item_mode(f.str("mode", "edge"));
    const double eps = f.real("epsilon", 0.1), delta = f.real("delta", 0.1);
    DeviceGraph dg(g, vi, static_cast<int>(f.u64("device", 0)));
    if (f.has("sweep")) {  // suspension curves: every baseline plus the interdiction algorithm
        std::vector<std::uint32_t> ks;
        std::stringstream ss(f.str("sweep"));
        std::string tok;
        while (std::getline(ss, tok, ',')) ks.push_back(static_cast<std::uint32_t>(std::stoul(tok)));
        const std::pair<const char*, BaselineKind> methods[] = {
            {"pagerank", BaselineKind::Pagerank},     {"maxdegree", BaselineKind::MaxDegree},
            {"randomized", BaselineKind::Randomized}, {"infmax-v", BaselineKind::InfMaxV},
            {"infmax-vi", BaselineKind::InfMaxVI}};
        const std::string csv = f.str("csv").empty() ? "sweep.csv" : f.str("csv");
        std::ofstream out(csv);
        if (!out) throw DataError("cannot write csv");
        out << "method,k,suspension\n";
        for (std::uint32_t kk : ks) {
            for (const auto& [name, bk] : methods) {
                PrgState s = seed_from_worker(seed);
                RemovalSet r = baseline(dg, g, vi, bk, kind, kk, s);
                out << name << ',' << kk << ',' << estimate_suspension(dg, r, eps, delta, s).value
                    << '\n';
            }
            InterdictionOptions opts;
            opts.seed = seed;
            const CandidateSet cand = CandidateSet::all(kind);
            const InterdictionResult res = kind == ItemKind::Edge
                                               ? esia(dg, g, cand, kk, eps, delta, opts)
                                               : nsia(dg, g, cand, kk, eps, delta, opts);
            RemovalSet r{kind, res.solution};
            PrgState s = seed_from_worker(seed);
            out << (kind == ItemKind::Edge ? "esia" : "nsia") << ',' << kk << ','
                << estimate_suspension(dg, r, eps, delta, s).value << '\n';
        }
        return 0;
    }
    const std::string method = f.str("method", "pagerank");
    const auto k = static_cast<std::uint32_t>(f.u64("k", 1));
    PrgState s = seed_from_worker(seed);
    RemovalSet r = baseline(dg, g, vi, parse_baseline_kind(method), kind, k, s);
    const SuspensionEstimate est = estimate_suspension(dg, r, eps, delta, s);
    std::ostringstream j;  // nlohmann object: keys sorted, dump(2)
    j << "{\n";
    if (kind == ItemKind::Node) {
        const SolutionAnalysis a = analyze_solution(g, vi, r);
        j << "  \"cost\": " << json_shortest(a.cost) << ",\n";
    }
    j << "  \"ids\": " << json_int_array(r.ids) << ",\n  \"k\": " << k << ",\n  \"kind\": \""
      << to_string(kind) << "\",\n  \"method\": \"" << method << "\"";
    if (kind == ItemKind::Node) j << ",\n  \"ssr\": " << json_shortest(analyze_solution(g, vi, r).ssr);
    j << ",\n  \"suspension\": " << json_shortest(est.value) << "\n}";
    emit(j.str(), f.str("output"));
    return 0;
}

int cmd_partition(const Flags& f) {  // cli.cpp:292-335
    f.require("graph");
    f.require("parts");
    const std::uint64_t seed = f.u64("seed", 0);
    ProbGraph g = load_graph(f, seed, /*on_host=*/f.u64("target", 0) == 0);
    const std::string method = f.str("method", "hash");
    PartitionMethod pm;
    if (method == "hash")
        pm = PartitionMethod::Hash;
    else if (method == "labelprop")
        pm = PartitionMethod::LabelProp;
    else if (method == "external")
        pm = PartitionMethod::ExternalFile;
    else
        throw UsageError("--method: expected hash|labelprop|external");
    const auto p = static_cast<std::uint32_t>(f.u64("parts", 1));
    const auto hops = static_cast<std::uint32_t>(f.u64("hops", 0));
    Partitioning part = extend_partition(g, partition_graph(g, p, pm, seed, f.str("part-file")), hops);
    if (f.has("save")) save_partition(part, f.str("save"));
    std::vector<std::uint64_t> sizes, ext_sizes;
    for (std::uint32_t i = 0; i < part.p; ++i) {
        sizes.push_back(part.base[i].size());
        ext_sizes.push_back(part.extended_size(i));
    }
    const std::uint64_t target = f.u64("target", 0);
    std::ostringstream j;
    j << "{\n";
    DistributedResult res;
    if (target > 0) {
        SuspectSet vi = load_suspect_args(f, g, seed);
        DeviceGraph dg(g, vi, static_cast<int>(f.u64("device", 0)));
        res = distributed_sample(dg, part, target, seed);
        j << "  \"accepted\": " << res.pool.accepted() << ",\n  \"attempts\": " << res.attempts
          << ",\n  \"crossing_fraction\": " << json_shortest(res.crossing_fraction)
          << ",\n  \"crossings\": " << res.crossings << ",\n";
    }
    j << "  \"extended_sizes\": " << json_int_array(ext_sizes) << ",\n  \"hops\": " << hops
      << ",\n  \"method\": \"" << method << "\",\n  \"part_sizes\": " << json_int_array(sizes)
      << ",\n  \"parts\": " << p;
    if (target > 0)
        j << ",\n  \"per_part_targets\": " << json_int_array(res.targets) << ",\n  \"target\": "
          << target;
    j << "\n}";
    emit(j.str(), f.str("output"));
    return 0;
}

}  // namespace

int run_cli(std::vector<std::string> args) {
    try {
        if (args.empty()) throw UsageError("a subcommand is required: interdict|sample|estimate|baseline|partition|synth|bench");
        const std::string& cmd = args[0];
        if (cmd == "--help" || cmd == "-h") {
            std::cout << "usage: hsaw interdict|sample|estimate|baseline|partition|synth|bench [--flags]\n";
            return 0;
        }
        if (cmd == "interdict")
            return cmd_interdict(parse_flags(
                args, 1,
                with(kGraphFlags, {"mode", "k", "epsilon", "delta", "candidates", "workers", "seed",
                                   "max-attempts", "output", "device", "gpus", "devices"}),
                {"symmetrize", "omit-timing"}));
        if (cmd == "sample")
            return cmd_sample(parse_flags(
                args, 1,
                with(kGraphFlags, {"target", "workers", "seed", "max-attempts", "dump", "output",
                                   "device"}),
                {"symmetrize"}));
        if (cmd == "synth")
            return cmd_synth(
                parse_flags(args, 1, {"nodes", "density", "seed", "out", "cache"}, {}));
        if (cmd == "bench")
            return cmd_bench(parse_flags(
                args, 1,
                with(kGraphFlags, {"synth-nodes", "synth-density", "target", "workers", "seed",
                                   "output", "device"}),
                {}));
        if (cmd == "estimate")
            return cmd_estimate(parse_flags(
                args, 1,
                with(kGraphFlags, {"mode", "removal", "epsilon", "delta", "seed", "output", "device"}),
                {"symmetrize"}));
        if (cmd == "baseline")
            return cmd_baseline(parse_flags(
                args, 1,
                with(kGraphFlags, {"method", "mode", "k", "epsilon", "delta", "seed", "workers",
                                   "sweep", "csv", "output", "device"}),
                {"symmetrize"}));
        if (cmd == "partition")
            return cmd_partition(parse_flags(
                args, 1,
                with(kGraphFlags, {"parts", "method", "hops", "part-file", "target", "workers", "seed",
                                   "save", "output", "device"}),
                {"symmetrize"}));
        throw UsageError("unknown subcommand '" + cmd + "'");
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << '\n';
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cerr << "usage error: " << e.what() << '\n';
        return 1;
    } catch (const DataError& e) {
        std::cerr << "data error: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "runtime error: " << e.what() << '\n';
        return 3;
    }
}

}  // namespace hsaw
