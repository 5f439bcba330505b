// Partitioned sampling, host side: the reference's partition.hpp interface.
// partition_graph / extend_partition / save_partition restate proj/src/partition.cpp:29-151 on the
// host (they are setup code over the CSR; the label propagation is a sequential, order-dependent
// sweep by definition). distributed_sample keeps the reference's quota and cut logic
// (partition.cpp:153-279) and runs every part's restricted batches on the device through a
// restricted SampleStream (hsaw_gpu_stream_restrict).
#include <algorithm>
#include <fstream>
#include <numeric>

#include "hsaw_b200.hpp"

namespace hsaw {

namespace {

constexpr std::uint64_t kPartStride = 1ull << 40;  // worker-id window per part (partition.cpp:14)

void fill_base(NodeId n, Partitioning& part) {
    part.base.assign(part.p, {});
    for (NodeId v = 0; v < n; ++v) part.base[part.assign[v]].push_back(v);
}

// LabelProp, partition.cpp:43-111: ten synchronous sweeps over the undirected view; every node
// adopts the most frequent label among itself and its neighbours (ties: smaller label) among the
// labels that still have room (capacity ~1.15 n / p, filled in node order within a sweep).
std::vector<std::uint32_t> propagate_labels(const ProbGraph& g, std::uint32_t p, std::uint64_t seed) {
    const NodeId n = g.n;
    std::vector<std::uint32_t> label(n), next(n);
    for (NodeId v = 0; v < n; ++v)
        label[v] = static_cast<std::uint32_t>(
            splitmix_next(seed * 0x9E3779B97F4A7C15ULL + v).output % p);
    // undirected adjacency with antiparallel edges merged (each neighbour votes once)
    std::vector<std::uint64_t> deg(static_cast<std::size_t>(n) + 1, 0);
    for (EdgeId e = 0; e < g.m; ++e) {
        ++deg[g.in_src[e] + 1];
        ++deg[g.edge_dst[e] + 1];
    }
    std::partial_sum(deg.begin(), deg.end(), deg.begin());
    std::vector<NodeId> adj(deg[n]);
    std::vector<std::uint64_t> at(deg.begin(), deg.end() - 1);
    for (EdgeId e = 0; e < g.m; ++e) {
        adj[at[g.in_src[e]]++] = g.edge_dst[e];
        adj[at[g.edge_dst[e]]++] = g.in_src[e];
    }
    std::vector<std::uint64_t> end(n);
    for (NodeId v = 0; v < n; ++v) {
        auto first = adj.begin() + static_cast<std::ptrdiff_t>(deg[v]);
        auto last = adj.begin() + static_cast<std::ptrdiff_t>(deg[v + 1]);
        std::sort(first, last);
        end[v] = static_cast<std::uint64_t>(std::unique(first, last) - adj.begin());
    }
    const std::uint64_t cap = std::max<std::uint64_t>(
        (static_cast<std::uint64_t>(n) * 115 + 100ull * p - 1) / (100ull * p), 1);
    std::vector<std::uint32_t> votes(p);
    std::vector<std::uint64_t> load(p);
    for (int sweep = 0; sweep < 10; ++sweep) {
        std::fill(load.begin(), load.end(), 0);
        for (NodeId v = 0; v < n; ++v) {
            std::fill(votes.begin(), votes.end(), 0);
            votes[label[v]] = 1;
            for (std::uint64_t i = deg[v]; i < end[v]; ++i) ++votes[label[adj[i]]];
            std::uint32_t pick = p;
            for (std::uint32_t c = 0; c < p; ++c) {
                if (load[c] >= cap) continue;
                if (pick == p || votes[c] > votes[pick]) pick = c;
            }
            next[v] = pick;
            ++load[pick];
        }
        label.swap(next);
    }
    // a label can starve: every empty part takes the highest-numbered node of the largest part
    std::fill(load.begin(), load.end(), 0);
    for (NodeId v = 0; v < n; ++v) ++load[label[v]];
    for (std::uint32_t c = 0; c < p; ++c) {
        if (load[c] > 0) continue;
        const auto donor =
            static_cast<std::uint32_t>(std::max_element(load.begin(), load.end()) - load.begin());
        for (NodeId v = n; v-- > 0;) {
            if (label[v] != donor) continue;
            label[v] = c;
            --load[donor];
            ++load[c];
            break;
        }
    }
    return label;
}

}  // namespace

std::size_t Partitioning::extended_size(std::uint32_t part) const {
    const auto& mask = extended[part];
    return static_cast<std::size_t>(std::count(mask.begin(), mask.end(), std::uint8_t{1}));
}

Partitioning partition_graph(const ProbGraph& g, std::uint32_t p, PartitionMethod method,
                             std::uint64_t seed, const std::string& part_file) {
    if (p < 1 || p > g.n) throw DataError("part count must be in [1, n]");
    Partitioning part;
    part.p = p;
    part.assign.resize(g.n);
    if (method == PartitionMethod::Hash) {
        for (NodeId v = 0; v < g.n; ++v) part.assign[v] = v % p;
    } else if (method == PartitionMethod::LabelProp) {
        part.assign = propagate_labels(g, p, seed);
    } else {  // one part id per node, whitespace separated, in node order
        std::ifstream in(part_file);
        if (!in) throw DataError("cannot open part file: " + part_file);
        std::uint64_t id = 0;
        NodeId v = 0;
        while (in >> id) {
            if (v >= g.n) throw DataError("part file longer than n");
            if (id >= p) throw DataError("part id " + std::to_string(id) + " out of range");
            part.assign[v++] = static_cast<std::uint32_t>(id);
        }
        if (v != g.n) throw DataError("part file shorter than n");
    }
    fill_base(g.n, part);
    return extend_partition(g, std::move(part), 0);
}

Partitioning extend_partition(const ProbGraph& g, Partitioning part, std::uint32_t h) {
    part.hops = h;
    part.extended.assign(part.p, std::vector<std::uint8_t>(g.n, 0));
    std::vector<NodeId> frontier, found;
    for (std::uint32_t i = 0; i < part.p; ++i) {
        auto& mask = part.extended[i];
        frontier = part.base[i];
        for (NodeId v : frontier) mask[v] = 1;
        for (std::uint32_t hop = 0; hop < h && !frontier.empty(); ++hop) {
            found.clear();
            for (NodeId v : frontier)
                for (std::uint64_t e = g.in_offsets[v]; e < g.in_offsets[v + 1]; ++e) {
                    const NodeId u = g.in_src[e];
                    if (mask[u]) continue;
                    mask[u] = 1;
                    found.push_back(u);
                }
            frontier.swap(found);
        }
    }
    return part;
}

void save_partition(const Partitioning& part, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw DataError("cannot write part file: " + path);
    for (std::uint32_t id : part.assign) out << id << '\n';
}

DistributedResult distributed_sample(const DeviceGraph& dg, const Partitioning& part,
                                     std::uint64_t total_target, std::uint64_t seed,
                                     const SamplerConfig& cfg) {
    if (part.assign.size() != dg.n() || part.base.size() != part.p || part.extended.size() != part.p)
        throw std::invalid_argument("partitioning does not match the graph");
    for (std::uint32_t i = 0; i < part.p; ++i)
        if (part.base[i].empty()) throw DataError("part " + std::to_string(i) + " is empty");

    // quotas proportional to |part i|, largest remainders first (partition.cpp:163-181)
    DistributedResult res;
    res.targets.assign(part.p, 0);
    std::vector<std::pair<double, std::uint32_t>> rema(part.p);
    std::uint64_t assigned = 0;
    for (std::uint32_t i = 0; i < part.p; ++i) {
        const double share = static_cast<double>(total_target) *
                             static_cast<double>(part.base[i].size()) / static_cast<double>(dg.n());
        res.targets[i] = static_cast<std::uint64_t>(share);
        assigned += res.targets[i];
        rema[i] = {share - static_cast<double>(res.targets[i]), i};
    }
    std::sort(rema.begin(), rema.end(), [](const auto& a, const auto& b) {
        return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    for (std::uint64_t r = 0; r < total_target - assigned; ++r) ++res.targets[rema[r % part.p].second];

    for (std::uint32_t i = 0; i < part.p; ++i) {
        if (res.targets[i] == 0) continue;  // nothing sampled, nothing counted (partition.cpp:245-262)
        SampleStream stream(dg, seed + i * kPartStride, cfg);
        stream.restrict(part.base[i], part.extended[i].data());
        try {
            stream.ensure(res.targets[i]);
        } catch (const SamplingError&) {
            throw SamplingError("attempt budget exhausted in partitioned sampling");
        }
        // whole batches up to the minimal prefix reaching the quota: all of its samples are kept
        SamplePool piece = stream.to_pool(res.targets[i]);
        res.crossings += stream.crossings_for(res.targets[i]);
        res.attempts += piece.attempts;
        for (std::size_t w = 0; w < piece.samples.size(); ++w) {
            res.pool.samples.push_back(std::move(piece.samples[w]));
            res.pool.tags.push_back(piece.tags[w]);
        }
    }
    res.pool.attempts = res.attempts;
    res.crossing_fraction = res.attempts == 0 ? 0.0
                                              : static_cast<double>(res.crossings) /
                                                    static_cast<double>(res.attempts);
    return res;
}

DistributedResult distributed_sample(const ProbGraph& g, const SuspectSet& vi,
                                     const Partitioning& part, std::uint64_t total_target,
                                     std::uint64_t seed, std::uint32_t /*workers*/,
                                     const SamplerConfig& cfg) {
    DeviceGraph dg(g, vi);
    return distributed_sample(dg, part, total_target, seed, cfg);
}

}  // namespace hsaw
