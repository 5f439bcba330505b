// Ranking baselines: the reference's baseline() interface
// (proj/include/hsaw/evaluation.hpp:45-50, proj/src/evaluation.cpp:110-191,310-395). The InfMax
// kinds — reverse-reachable node sets + greedy max-cover over them — run on the device
// (hsaw_gpu_rr_node_sets, hsaw_gpu_greedy); the three score rankings and the node -> in-edge mapping
// are host code as in the reference.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_set>

#include "hsaw_b200.hpp"
#include "hsaw_gpu.h"

namespace hsaw {

namespace {

[[noreturn]] void bad(const std::string& msg) { throw DataError(msg); }

// score descending, ties by ascending id (evaluation.cpp:110-119)
std::vector<std::uint32_t> rank_by(const std::vector<double>& score) {
    std::vector<std::uint32_t> order(score.size());
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
        return score[a] != score[b] ? score[a] > score[b] : a < b;
    });
    return order;
}

// k distinct uniform draws below `limit` (evaluation.cpp:153-165)
std::vector<std::uint32_t> uniform_distinct(PrgState& s, std::uint32_t limit, std::uint32_t k) {
    if (k > limit) bad("k exceeds candidate count");
    std::unordered_set<std::uint32_t> seen;
    std::vector<std::uint32_t> out;
    while (out.size() < k) {
        auto x = static_cast<std::uint32_t>(u01(prg_next(s)) * limit);
        if (x >= limit) x = limit - 1;
        if (seen.insert(x).second) out.push_back(x);
    }
    return out;
}

// The k heaviest in-edges of the ranked nodes, one per node per pass (evaluation.cpp:121-151).
std::vector<std::uint32_t> heaviest_in_edges(const ProbGraph& g,
                                             const std::vector<std::uint32_t>& nodes,
                                             std::uint32_t k) {
    // rows are only sorted when the round-robin actually reaches them
    std::vector<std::vector<EdgeId>> sorted(nodes.size());
    std::vector<std::uint8_t> ready(nodes.size(), 0);
    std::vector<std::size_t> taken(nodes.size(), 0);
    std::vector<std::uint32_t> out;
    while (out.size() < k) {
        bool advanced = false;
        for (std::size_t i = 0; i < nodes.size() && out.size() < k; ++i) {
            const NodeId v = nodes[i];
            const std::uint64_t lo = g.in_offsets[v], hi = g.in_offsets[v + 1];
            if (taken[i] >= hi - lo) continue;
            if (!ready[i]) {
                sorted[i].resize(hi - lo);
                std::iota(sorted[i].begin(), sorted[i].end(), static_cast<EdgeId>(lo));
                std::sort(sorted[i].begin(), sorted[i].end(), [&](EdgeId a, EdgeId b) {
                    return g.weight[a] != g.weight[b] ? g.weight[a] > g.weight[b] : a < b;
                });
                ready[i] = 1;
            }
            out.push_back(sorted[i][taken[i]++]);
            advanced = true;
        }
        if (!advanced) bad("not enough incoming edges among ranked nodes");
    }
    return out;
}

}  // namespace

std::vector<std::vector<std::uint32_t>> rr_node_sets(const DeviceGraph& dg, PrgState& s,
                                                     std::uint32_t count) {
    hsaw_gpu_walkset* ws = nullptr;
    std::uint64_t total = 0;
    if (hsaw_gpu_rr_node_sets(dg.ctx(), &s.state, count, &ws, &total) != HSAW_OK)
        throw DeviceError(std::string("rr_node_sets: ") + hsaw_gpu_last_error(dg.ctx()));
    std::vector<std::uint64_t> off(static_cast<std::size_t>(count) + 1);
    std::vector<std::uint32_t> items(total + 1);
    const int rc = hsaw_gpu_walkset_export(ws, off.data(), items.data());
    hsaw_gpu_walkset_destroy(ws);
    if (rc != HSAW_OK) throw DeviceError("rr_node_sets: export failed");
    std::vector<std::vector<std::uint32_t>> sets(count);
    for (std::uint32_t i = 0; i < count; ++i)
        sets[i].assign(items.begin() + static_cast<std::ptrdiff_t>(off[i]),
                       items.begin() + static_cast<std::ptrdiff_t>(off[i + 1]));
    return sets;
}

std::vector<double> pagerank_scores(const ProbGraph& g, double damping, double tol, int max_iters) {
    // evaluation.cpp:310-328, same accumulation order (edges in id order) so the scores — and
    // the ranking, ties included — are the reference's
    const auto out_deg = g.out_degrees();
    std::vector<double> pr(g.n, 1.0 / g.n), next(g.n, 0.0);
    for (int it = 0; it < max_iters; ++it) {
        double dangling = 0.0;
        for (NodeId v = 0; v < g.n; ++v)
            if (out_deg[v] == 0) dangling += pr[v];
        const double base = (1.0 - damping) / g.n + damping * dangling / g.n;
        std::fill(next.begin(), next.end(), base);
        for (EdgeId e = 0; e < g.m; ++e)
            next[g.edge_dst[e]] += damping * pr[g.in_src[e]] / out_deg[g.in_src[e]];
        double diff = 0.0;
        for (NodeId v = 0; v < g.n; ++v) diff += std::abs(next[v] - pr[v]);
        pr.swap(next);
        if (diff < tol) break;
    }
    return pr;
}

RemovalSet baseline(const DeviceGraph& dg, const ProbGraph& g, const SuspectSet& vi,
                    BaselineKind kind, ItemKind mode, std::uint32_t k, PrgState& s,
                    std::uint32_t infmax_samples) {
    RemovalSet r;
    r.kind = mode;
    if (kind == BaselineKind::Randomized) {
        r.ids = uniform_distinct(s, mode == ItemKind::Edge ? g.m : g.n, k);
        return r;
    }
    std::vector<std::uint32_t> ranked;
    if (kind == BaselineKind::Pagerank) {
        ranked = rank_by(pagerank_scores(g));
    } else if (kind == BaselineKind::MaxDegree) {
        const auto out_deg = g.out_degrees();
        std::vector<double> deg(g.n);
        for (NodeId v = 0; v < g.n; ++v) deg[v] = static_cast<double>(out_deg[v]) + g.in_degree(v);
        ranked = rank_by(deg);
    } else {  // InfMaxV / InfMaxVI: greedy max-cover over reverse-reachable node sets
        CandidateSet cand = CandidateSet::all(ItemKind::Node);
        if (kind == BaselineKind::InfMaxVI) {
            std::vector<std::uint32_t> ids;
            for (const auto& member : vi.members) ids.push_back(member.first);
            if (ids.empty()) bad("suspect set is empty");
            cand = CandidateSet::of(ItemKind::Node, std::move(ids));
        }
        hsaw_gpu_walkset* ws = nullptr;
        if (hsaw_gpu_rr_node_sets(dg.ctx(), &s.state, infmax_samples, &ws, nullptr) != HSAW_OK)
            throw DeviceError(std::string("rr_node_sets: ") + hsaw_gpu_last_error(dg.ctx()));
        CoverageIndex idx(dg, ws, infmax_samples, cand, g);  // owns the walk set from here on
        const auto budget = static_cast<std::uint32_t>(std::min<std::uint64_t>(
            idx.num_candidates(), mode == ItemKind::Edge ? std::max<std::uint32_t>(k, 64) : k));
        ranked = greedy_max_cover(idx, budget).solution;
    }
    if (mode == ItemKind::Node) {
        if (k > ranked.size()) bad("k exceeds candidate count");
        r.ids.assign(ranked.begin(), ranked.begin() + k);
        return r;
    }
    if (k > g.m) bad("k exceeds edge count");
    // the ranked pool may not carry k in-edges: every other node follows in id order
    std::vector<std::uint8_t> listed(g.n, 0);
    for (std::uint32_t v : ranked) listed[v] = 1;
    for (NodeId v = 0; v < g.n; ++v)
        if (!listed[v]) ranked.push_back(v);
    r.ids = heaviest_in_edges(g, ranked, k);
    return r;
}

RemovalSet baseline(const ProbGraph& g, const SuspectSet& vi, BaselineKind kind, ItemKind mode,
                    std::uint32_t k, PrgState& s, std::uint32_t infmax_samples) {
    if (kind == BaselineKind::InfMaxV || kind == BaselineKind::InfMaxVI) {
        DeviceGraph dg(g, vi);
        return baseline(dg, g, vi, kind, mode, k, s, infmax_samples);
    }
    // the score rankings never touch the device: a null DeviceGraph reference is never used
    RemovalSet r;
    r.kind = mode;
    if (kind == BaselineKind::Randomized) {
        r.ids = uniform_distinct(s, mode == ItemKind::Edge ? g.m : g.n, k);
        return r;
    }
    std::vector<std::uint32_t> ranked;
    if (kind == BaselineKind::Pagerank) {
        ranked = rank_by(pagerank_scores(g));
    } else {
        const auto out_deg = g.out_degrees();
        std::vector<double> deg(g.n);
        for (NodeId v = 0; v < g.n; ++v) deg[v] = static_cast<double>(out_deg[v]) + g.in_degree(v);
        ranked = rank_by(deg);
    }
    if (mode == ItemKind::Node) {
        if (k > ranked.size()) bad("k exceeds candidate count");
        r.ids.assign(ranked.begin(), ranked.begin() + k);
        return r;
    }
    if (k > g.m) bad("k exceeds edge count");
    r.ids = heaviest_in_edges(g, ranked, k);
    return r;
}

SolutionAnalysis analyze_solution(const ProbGraph& g, const SuspectSet& vi,
                                  const RemovalSet& removal) {
    if (removal.kind != ItemKind::Node)
        throw std::invalid_argument("analysis requires a node removal set");
    if (removal.ids.empty()) throw std::invalid_argument("removal set is empty");
    removal.validate(g);
    SolutionAnalysis a;
    std::size_t in_vi = 0;
    for (std::uint32_t v : removal.ids) {
        if (vi.is_suspect(v)) ++in_vi;
        a.cost += (1.0 - vi.p_of[v]) * std::log(g.in_degree(v) + 1.0);
    }
    a.ssr = static_cast<double>(in_vi) / static_cast<double>(removal.ids.size());
    return a;
}

}  // namespace hsaw
