// hsaw_b200.hpp — C++ host layer of the B200 HSAW path.
//
// Mirrors the public interface of the reference library (/root/reference/proj/include/hsaw/*.hpp)
// for the eSIA/nSIA hot path — same names, argument meaning and error behaviour — so that code and
// tests written against the reference read the same here. Everything that samples walks or runs
// greedy max-cover executes on the GPU through the C-ABI in include/hsaw_gpu.h; loaders, the
// sample-size schedule, the stopping rule and the doubling loop stay on the host, as north_star
// item (4) asks. There is no CPU fallback: without a CUDA device the sampling entry points throw.
//
// Reference interface -> this header
//   types.hpp        NodeId, EdgeId, ItemKind, DataError, SamplingError
//   prng.hpp         PrgState, splitmix_next, prg_next, u01, pick_uniform_node, seed_from_worker
//   graph.hpp        ProbGraph, SuspectSet, CandidateSet, WeightMode, LoadOptions, build_graph,
//                    load_edge_list, load_suspects, random_suspects, synth_graph, save_edge_list,
//                    save_cache, load_cache
//   sampler.hpp      EncodedWalk, HsawSample, WalkTag, SamplePool, SamplerConfig, thread_sample,
//                    DecodeContext, SampleStream, stream_samples, estimate_influence, dump_walks
//   coverage.hpp     CoverageIndex, GreedyResult, greedy_max_cover, Schedule, ln_choose,
//                    compute_schedule(_m), CheckResult, check_solution
//   interdiction.hpp InterdictionResult, InterdictionOptions, esia, nsia, to_json
//   evaluation.hpp   RemovalSet, SuspensionEstimate, lt_forward_simulate, estimate_suspension
//                    (the paired forward simulation; baselines / brute force are out of scope)
//   cli.hpp          run_cli
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

struct hsaw_gpu_ctx;
struct hsaw_gpu_stream;
struct hsaw_gpu_walkset;

namespace hsaw {

// ---- types (proj/include/hsaw/types.hpp) --------------------------------------------------------
using NodeId = std::uint32_t;
using EdgeId = std::uint32_t;
inline constexpr NodeId kInvalidNode = ~NodeId(0);

enum class ItemKind { Edge, Node };
inline const char* to_string(ItemKind k) { return k == ItemKind::Edge ? "edge" : "node"; }

struct DataError : std::runtime_error {
    explicit DataError(const std::string& m) : std::runtime_error(m) {}
};
struct SamplingError : std::runtime_error {
    explicit SamplingError(const std::string& m) : std::runtime_error(m) {}
};
// Not in the reference: the device path failed (no GPU, CUDA error). Maps to CLI exit code 3.
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// ---- prng (proj/include/hsaw/prng.hpp) — host copies used by the loaders and generators --------
struct PrgState {
    std::uint64_t state = 0x853C49E6748FEA9BULL;
    friend bool operator==(const PrgState& a, const PrgState& b) { return a.state == b.state; }
};
struct SplitMixResult {
    std::uint64_t state, output;
};
SplitMixResult splitmix_next(std::uint64_t state);
std::uint64_t prg_next(PrgState& s);
double u01(std::uint64_t output);
NodeId pick_uniform_node(PrgState& s, NodeId n);
PrgState seed_from_worker(std::uint64_t worker_id);

// ---- graph (proj/include/hsaw/graph.hpp) --------------------------------------------------------
struct ProbGraph {
    NodeId n = 0;
    EdgeId m = 0;
    std::vector<std::uint64_t> in_offsets;  // n + 1
    std::vector<NodeId> in_src;             // m, ascending per target
    std::vector<double> in_cum;             // m, sequential per-row cumulative weights
    std::vector<double> weight;             // m
    std::vector<NodeId> edge_dst;           // m

    std::pair<NodeId, NodeId> endpoints(EdgeId e) const { return {in_src[e], edge_dst[e]}; }
    std::uint32_t in_degree(NodeId v) const {
        return static_cast<std::uint32_t>(in_offsets[v + 1] - in_offsets[v]);
    }
    double total_in_weight(NodeId v) const {
        return in_offsets[v + 1] > in_offsets[v] ? in_cum[in_offsets[v + 1] - 1] : 0.0;
    }
    void validate() const;  // throws DataError
    std::vector<std::uint32_t> out_degrees() const;
};

struct SuspectSet {
    std::vector<std::pair<NodeId, double>> members;  // sorted by node id
    std::vector<double> p_of;                        // n, 0 = not a suspect
    double p(NodeId v) const { return p_of[v]; }
    bool is_suspect(NodeId v) const { return p_of[v] > 0.0; }
    std::size_t size() const { return members.size(); }
    static SuspectSet from_members(std::vector<std::pair<NodeId, double>> mem, const ProbGraph& g);
    static SuspectSet from_members(std::vector<std::pair<NodeId, double>> mem, NodeId n);
};

struct CandidateSet {
    ItemKind kind = ItemKind::Edge;
    std::optional<std::vector<std::uint32_t>> ids;  // nullopt = all items of the kind
    static CandidateSet all(ItemKind k) { return CandidateSet{k, std::nullopt}; }
    static CandidateSet of(ItemKind k, std::vector<std::uint32_t> v) {
        return CandidateSet{k, std::move(v)};
    }
    std::size_t size(const ProbGraph& g) const {
        return ids ? ids->size() : (kind == ItemKind::Edge ? g.m : g.n);
    }
    void validate(const ProbGraph& g) const;
};

enum class WeightMode { Given, InDegree, RandomNormalized };

struct LoadOptions {
    bool symmetrize = false;
    std::string mapping_out;
};

ProbGraph build_graph(NodeId n, std::vector<std::tuple<NodeId, NodeId, double>> edges,
                      WeightMode mode, std::uint64_t seed);
ProbGraph load_edge_list(const std::string& path, WeightMode mode, std::uint64_t seed,
                         const LoadOptions& opts = {});
SuspectSet load_suspects(const std::string& path, const ProbGraph& g);
SuspectSet random_suspects(const ProbGraph& g, NodeId count, std::uint64_t seed);
SuspectSet random_suspects(NodeId n, NodeId count, std::uint64_t seed);  // same draws, no graph needed
ProbGraph synth_graph(NodeId n, std::uint32_t density, std::uint64_t seed);
void save_edge_list(const ProbGraph& g, const std::string& path);
void save_cache(const ProbGraph& g, const std::string& path);
ProbGraph load_cache(const std::string& path);

// Bench tooling (not in the reference): R-MAT(a,b,c,d) graph with 1/in-degree weights, built
// without validate() because hub rows exceed its 1e-12 tolerance.
ProbGraph rmat_graph(std::uint32_t scale, double edge_factor, std::uint64_t seed, double a = 0.57,
                     double b = 0.19, double c = 0.19);
// Same generator for any node count (the named shapes are not powers of two: 41.7 M, 65.6 M):
// ceil(log2 n) quadrant draws per raw edge, raw edges with an endpoint >= n dropped like
// self-loops and duplicates. rmat_graph(scale, f, ...) == rmat_graph_n(2^scale, floor(f 2^scale), ...).
ProbGraph rmat_graph_n(NodeId n, std::uint64_t raw_edges, std::uint64_t seed, double a = 0.57,
                       double b = 0.19, double c = 0.19);
// The generator's relabelling (seeded Fisher-Yates, n-1 draws) and the PrgState after it: the
// sequential part of the stream, computed on the host for the device generator too.
struct RmatLabels {
    std::vector<NodeId> label;
    PrgState state;
};
RmatLabels rmat_labels(NodeId n, std::uint64_t seed);
void fill_indegree_weights(ProbGraph& g);  // weight = 1/d + sequential in_cum from in_offsets
// rmat_graph_n generated, sorted, deduplicated and summed on the GPU (hsaw_gpu_rmat_build): the
// same ProbGraph bit for bit in seconds at the 1.47 G-edge shape. lean: leave weight / edge_dst
// empty (the sampling path never reads them; 12 bytes per edge of host memory saved).
ProbGraph rmat_graph_device(NodeId n, std::uint64_t raw_edges, std::uint64_t seed, double a = 0.57,
                            double b = 0.19, double c = 0.19, int device = 0, bool lean = false);
// Direct CSR fill (in_offsets, in_src, in_cum given); weight/edge_dst derived; no validate().
ProbGraph graph_from_csr(NodeId n, EdgeId m, const std::uint64_t* in_offsets, const NodeId* in_src,
                         const double* in_cum);

// ---- device binding (new: the reference has no device) -----------------------------------------
// Owns one hsaw_gpu_ctx with the graph + suspects uploaded. Every sampling object below borrows it.
// build_graph (proj/include/hsaw/graph.hpp:123-125) with the sort, the per-row sequential sums and
// the validation run on the GPU (hsaw_gpu_csr_build): same ProbGraph, bit for bit, same DataError
// messages, for WeightMode::Given and ::InDegree. RandomNormalized falls through to build_graph's
// host loop (one global draw stream). Throws DeviceError without a CUDA device.
ProbGraph build_graph_device(NodeId n, const std::vector<std::tuple<NodeId, NodeId, double>>& edges,
                             WeightMode mode, std::uint64_t seed = 0, int device = 0);
// Same from flat arrays (w may be null unless mode == Given).
ProbGraph build_graph_device(NodeId n, std::uint64_t nedges, const NodeId* u, const NodeId* v,
                             const double* w, WeightMode mode, int device = 0);

// load_edge_list (proj/include/hsaw/graph.hpp:126-128) with the text parse, the id remap, the sort,
// the per-row sums and the validation on the GPU (hsaw_gpu_edge_text_parse + hsaw_gpu_csr_build).
// Same ProbGraph, same node-map file, same DataErrors: a file with any line outside the device
// parser's plain grammar (or opts.symmetrize, or WeightMode::RandomNormalized's host draw stream)
// is handed to load_edge_list / build_graph unchanged.
ProbGraph load_edge_list_device(const std::string& path, WeightMode mode, std::uint64_t seed,
                                const LoadOptions& opts = {}, int device = 0);

// load_cache (proj/include/hsaw/graph.hpp:139-141) with the decode, the per-row cumulative sums and
// validate() on the GPU (hsaw_gpu_cache_decode): the file is mapped and shipped as it lies on disk.
// Same ProbGraph bit for bit, same DataError messages.
ProbGraph load_cache_device(const std::string& path, int device = 0);

class DeviceGraph {
public:
    DeviceGraph(const ProbGraph& g, const SuspectSet& vi, int device = 0,
                void* cuda_stream = nullptr);
    // HSAW1 cache file -> graph resident on the device, no host CSR (hsaw_gpu_graph_cache_upload).
    // No suspects yet: call set_suspects() before sampling.
    static std::unique_ptr<DeviceGraph> from_cache(const std::string& path, int device = 0,
                                                   void* cuda_stream = nullptr);
    // Edge-list text file -> graph resident on the device (parse, re-rank, sort, sum and layout
    // all on the GPU; hsaw_gpu_edge_text_parse + hsaw_gpu_edge_text_install), for
    // WeightMode::Given / ::InDegree files within the device parser's plain grammar. Returns null
    // when the file needs the host loader (load_edge_list_device + the constructor above).
    static std::unique_ptr<DeviceGraph> from_edge_list(const std::string& path, WeightMode mode,
                                                       int device = 0, void* cuda_stream = nullptr);
    // rmat_graph_n generated on the device and installed where it lies: no host CSR at all unless
    // host_copy is given (filled lean: in_offsets / in_src / in_cum only). vi may be null (no
    // suspects yet).
    static std::unique_ptr<DeviceGraph> from_rmat(NodeId n, std::uint64_t raw_edges,
                                                  std::uint64_t seed, const SuspectSet* vi,
                                                  double a = 0.57, double b = 0.19, double c = 0.19,
                                                  int device = 0, void* cuda_stream = nullptr,
                                                  ProbGraph* host_copy = nullptr);
    ~DeviceGraph();
    DeviceGraph(const DeviceGraph&) = delete;
    DeviceGraph& operator=(const DeviceGraph&) = delete;

    void set_suspects(const SuspectSet& vi);  // new SuspectSet on the same graph
    hsaw_gpu_ctx* ctx() const { return ctx_; }
    NodeId n() const { return n_; }
    EdgeId m() const { return m_; }
    std::uint64_t device_bytes() const;
    std::uint64_t launches() const;
    // {encode, decode, distinct, compact, index, rounds, coverage, upload} milliseconds on device
    std::vector<double> stage_ms(bool reset = false) const;

private:
    DeviceGraph() = default;
    hsaw_gpu_ctx* ctx_ = nullptr;
    NodeId n_ = 0;
    EdgeId m_ = 0;
};

// ---- sampler (proj/include/hsaw/sampler.hpp) ----------------------------------------------------
struct EncodedWalk {
    PrgState seed;
    std::uint32_t len = 0;
    std::uint64_t worker_id = 0;
    std::uint32_t seq = 0;
};
struct HsawSample {
    std::vector<NodeId> nodes;
    std::vector<EdgeId> edge_ids;
    NodeId source() const { return nodes.front(); }
    NodeId hit() const { return nodes.back(); }
};
struct WalkTag {
    std::uint64_t worker_id = 0;
    std::uint32_t seq = 0;
};
struct SamplePool {
    std::vector<HsawSample> samples;
    std::vector<WalkTag> tags;
    std::uint64_t attempts = 0;
    std::uint64_t accepted() const { return samples.size(); }
};

enum class CycleHeuristic { Brent, Floyd, None };  // proj/include/hsaw/sampler.hpp:46

// Reference: the reference's xorshift64* stream, every result bit-exact (the default, always).
// PhiloxPerWalk: the device's throughput mode — an independent counter-based substream per walk
// index; same walk law, different walks (statistical parity only). Never chosen implicitly.
enum class WalkRng { Reference, PhiloxPerWalk };

struct SamplerConfig {
    CycleHeuristic heuristic = CycleHeuristic::Brent;
    std::uint32_t window = 2;
    std::uint32_t batch_size = 10;
    std::uint64_t max_attempts = 100'000'000;
    WalkRng rng = WalkRng::Reference;  // not in the reference's SamplerConfig (sampler.hpp:48-55)
};

// thread_sample (proj/src/sampler.cpp:267-290) on the device.
std::vector<EncodedWalk> thread_sample(const DeviceGraph& dg, std::uint64_t worker_id,
                                       std::uint32_t l, const SamplerConfig& cfg = {});
std::vector<EncodedWalk> thread_sample(const ProbGraph& g, const SuspectSet& vi,
                                       std::uint64_t worker_id, std::uint32_t l,
                                       const SamplerConfig& cfg = {});

// DecodeContext (proj/include/hsaw/sampler.hpp:85-100) on the device.
class DecodeContext {
public:
    explicit DecodeContext(const DeviceGraph& dg) : dg_(dg) {}
    std::optional<HsawSample> decode(const EncodedWalk& ew);  // throws DataError on mismatch
    // Batched form: nullopt entries are walks dropped by the exact recheck.
    std::vector<std::optional<HsawSample>> decode(std::span<const EncodedWalk> walks);

private:
    const DeviceGraph& dg_;
};

// SampleStream (proj/include/hsaw/sampler.hpp:133-163): decoded walks stay on the device.
class SampleStream {
public:
    // Which item lists of each walk the device pool keeps (hsaw_gpu_stream_keep). The drivers
    // ask for the one their candidate kind indexes; prefix() / to_pool() need Both.
    enum class Items { Both, EdgesOnly, NodesOnly };
    SampleStream(const DeviceGraph& dg, std::uint64_t seed, SamplerConfig cfg = {},
                 Items items = Items::Both);
    ~SampleStream();
    SampleStream(const SampleStream&) = delete;
    SampleStream& operator=(const SampleStream&) = delete;

    void ensure(std::uint64_t min_accepted);  // throws SamplingError on budget exhaustion
    // Host copy of samples [offset, offset + count); throws std::out_of_range like the reference.
    std::vector<HsawSample> prefix(std::uint64_t offset, std::uint64_t count) const;
    struct Counters {
        std::uint64_t attempts = 0, accepted = 0;
    };
    Counters counters_for(std::uint64_t min_accepted) const;
    SamplePool to_pool(std::uint64_t min_accepted) const;

    // Partitioned sampling: start domain + allowed mask (before sampling), and the crossings of
    // the minimal batch prefix reaching min_accepted.
    void restrict(std::span<const NodeId> start_domain, const std::uint8_t* allowed);
    std::uint64_t crossings_for(std::uint64_t min_accepted) const;
    std::uint64_t materialized() const;
    hsaw_gpu_stream* handle() const { return s_; }
    const DeviceGraph& device() const { return dg_; }
    std::vector<std::uint64_t> stats() const;  // u64[8], see hsaw_gpu.h

private:
    const DeviceGraph& dg_;
    hsaw_gpu_stream* s_ = nullptr;
};

SamplePool stream_samples(const DeviceGraph& dg, std::uint64_t target, std::uint64_t seed = 0,
                          const SamplerConfig& cfg = {});
// Reference signature; `workers` is accepted and ignored (the GPU is the worker pool).
SamplePool stream_samples(const ProbGraph& g, const SuspectSet& vi, std::uint32_t workers,
                          std::uint64_t target, std::uint64_t seed = 0,
                          const SamplerConfig& cfg = {});
double estimate_influence(const SamplePool& pool, NodeId n);
void dump_walks(const SamplePool& pool, std::ostream& out);

// ---- partitioned sampling (proj/include/hsaw/partition.hpp) ---------------------------------------
// Node partition plus, per part, the h-hop in-neighbourhood closure walks may enter; a walk that
// steps outside it is aborted and counted as a crossing.
struct Partitioning {
    std::uint32_t p = 1;
    std::uint32_t hops = 0;
    std::vector<std::uint32_t> assign;                 // node -> part
    std::vector<std::vector<NodeId>> base;             // part -> owned nodes, ascending
    std::vector<std::vector<std::uint8_t>> extended;   // part -> byte mask over nodes
    std::size_t extended_size(std::uint32_t part) const;
};
enum class PartitionMethod { Hash, LabelProp, ExternalFile };
Partitioning partition_graph(const ProbGraph& g, std::uint32_t p, PartitionMethod method,
                             std::uint64_t seed, const std::string& part_file = "");
Partitioning extend_partition(const ProbGraph& g, Partitioning part, std::uint32_t h);
void save_partition(const Partitioning& part, const std::string& path);

struct DistributedResult {
    SamplePool pool;
    std::uint64_t crossings = 0;
    std::uint64_t attempts = 0;
    double crossing_fraction = 0;
    std::vector<std::uint64_t> targets;  // per-part quotas
};
// distributed_sample (proj/src/partition.cpp:153-279) with every part's restricted batches run on
// the device: quotas by largest remainder, part i samples worker ids seed + i * 2^40 + b with
// starts in base[i] and the extended[i] mask, cut at the minimal batch prefix reaching its quota.
// `workers` is accepted and ignored. Results equal the reference's for every worker count.
DistributedResult distributed_sample(const DeviceGraph& dg, const Partitioning& part,
                                     std::uint64_t total_target, std::uint64_t seed = 0,
                                     const SamplerConfig& cfg = {});
DistributedResult distributed_sample(const ProbGraph& g, const SuspectSet& vi,
                                     const Partitioning& part, std::uint64_t total_target,
                                     std::uint64_t seed = 0, std::uint32_t workers = 1,
                                     const SamplerConfig& cfg = {});

// ---- coverage (proj/include/hsaw/coverage.hpp) --------------------------------------------------
// Device-resident coverage index: a range of a SampleStream (edge ids or nodes of each walk) or a
// raw collection of item sets (the fixed-walk-set parity mode), restricted to the candidates.
class CoverageIndex {
public:
    CoverageIndex(ItemKind kind, const SampleStream& stream, std::uint64_t offset,
                  std::uint64_t count, const CandidateSet& cand, const ProbGraph& g);
    CoverageIndex(const DeviceGraph& dg, std::span<const std::vector<std::uint32_t>> item_sets,
                  const CandidateSet& cand, const ProbGraph& g);
    // Takes over a device-resident walk set (e.g. the reverse-reachable sets of rr_node_sets).
    CoverageIndex(const DeviceGraph& dg, hsaw_gpu_walkset* adopted, std::uint64_t nsets,
                  const CandidateSet& cand, const ProbGraph& g);
    ~CoverageIndex();
    CoverageIndex(const CoverageIndex&) = delete;
    CoverageIndex& operator=(const CoverageIndex&) = delete;

    ItemKind kind() const { return kind_; }
    std::uint32_t num_samples() const { return static_cast<std::uint32_t>(count_); }
    std::uint64_t num_candidates() const { return ncand_; }
    std::uint64_t coverage_of(std::span<const std::uint32_t> items) const;
    // Upper bound of coverage_of over every set of at most k candidates (sum of the k largest
    // per-item occurrence counts); lets the doubling loop skip iterations that cannot pass.
    std::uint64_t coverage_upper_bound(std::uint32_t k) const;

private:
    friend struct GreedyAccess;
    ItemKind kind_;
    hsaw_gpu_ctx* ctx_ = nullptr;
    hsaw_gpu_stream* stream_ = nullptr;
    hsaw_gpu_walkset* walkset_ = nullptr;
    std::uint64_t offset_ = 0, count_ = 0, ncand_ = 0;
    std::optional<std::vector<std::uint32_t>> cand_;
};

struct GreedyResult {
    std::vector<std::uint32_t> solution;
    std::uint64_t coverage = 0;
};
GreedyResult greedy_max_cover(const CoverageIndex& idx, std::uint32_t k);

struct Schedule {
    double epsilon = 0, delta = 0;
    std::uint32_t k = 0;
    double lambda = 0, lambda1 = 0, n_max = 0;
    std::uint32_t t_max = 1;
    std::uint64_t lambda_samples() const;
};
double ln_choose(std::uint64_t M, std::uint64_t k);
Schedule compute_schedule_m(std::uint64_t M, std::uint32_t k, double epsilon, double delta);
Schedule compute_schedule(const ProbGraph& g, ItemKind kind, std::uint32_t k, double epsilon,
                          double delta);

struct CheckResult {
    bool pass = false;
    double eps_t = 0;
};
CheckResult check_solution(std::span<const std::uint32_t> solution, const CoverageIndex& idx_r,
                           const CoverageIndex& idx_r_prime, const Schedule& sched,
                           std::uint32_t t);
// The arithmetic of check_solution on two coverage counts (used by both overloads and by tests).
CheckResult check_counts(double cov_r, double cov_rp, double n_rp, const Schedule& sched,
                         std::uint32_t t);

// ---- interdiction (proj/include/hsaw/interdiction.hpp) ------------------------------------------
struct InterdictionResult {
    ItemKind kind = ItemKind::Edge;
    std::uint32_t k = 0;
    double epsilon = 0, delta = 0;
    std::vector<std::uint32_t> solution;
    double est_suspension = 0;
    std::uint64_t coverage = 0, samples_used = 0, attempts = 0;
    std::uint32_t iterations = 0;
    bool passed_check = false;
    double wall_time_s = 0;
    // device-side breakdown (not serialised): sampling / greedy / check seconds of host wall time
    double sample_s = 0, greedy_s = 0, check_s = 0;
};

struct InterdictionOptions {
    std::uint32_t workers = 1;  // accepted for source compatibility; unused on the device path
    std::uint64_t seed = 0;
    SamplerConfig sampler;
    int device = 0;
    // More than one entry: the multi-device solve (host/multi.cpp) — the graph is replicated on
    // every listed device, each round's batch range is split into contiguous blocks (one per
    // device), marginal-gain counts are combined with an all-reduce (NCCL over NVLink when the
    // devices are distinct; an in-process exchange when a device id repeats, which is how the
    // path is tested on a single GPU). Same InterdictionResult for every device list.
    std::vector<int> devices;
};

// The multi-device doubling loop behind esia / nsia when opts.devices lists more than one device
// (host/multi.cpp), and the transport it would use for a device list ("nccl", "in-process
// exchange", "single device").
InterdictionResult run_interdiction_multi(const ProbGraph& g, const SuspectSet& vi,
                                          const CandidateSet& cand, std::uint32_t k, double epsilon,
                                          double delta, const InterdictionOptions& opts);
std::string multi_device_transport(const std::vector<int>& devices);

InterdictionResult esia(const ProbGraph& g, const SuspectSet& vi, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts = {});
InterdictionResult nsia(const ProbGraph& g, const SuspectSet& vi, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts = {});
// Same, on an already uploaded graph (upload excluded from wall_time_s).
InterdictionResult esia(const DeviceGraph& dg, const ProbGraph& g, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts = {});
InterdictionResult nsia(const DeviceGraph& dg, const ProbGraph& g, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts = {});

// A double as nlohmann::json::dump prints it (fixed notation for decimal exponents in (-4, 15]).
std::string json_number(double x);
std::string to_json(const InterdictionResult& r, bool include_timing = true);

// ---- evaluation (proj/include/hsaw/evaluation.hpp:16-39) ----------------------------------------
// The step after the path: forward LT simulation of a removal set, paired runs on the original and
// the residual graph sharing one realisation. Every run executes on the device
// (hsaw_gpu_paired_runs / hsaw_gpu_estimate_suspension) and reproduces the reference's single
// sequential PRG stream bit for bit; `s` is advanced exactly as the reference advances it.
struct RemovalSet {
    ItemKind kind = ItemKind::Edge;
    std::vector<std::uint32_t> ids;
    void validate(const ProbGraph& g) const;  // throws DataError("removal id out of range: ...")
};
struct SuspensionEstimate {
    double value = 0;
    bool capped = false;  // draw cap hit before the stopping rule fired
    std::uint64_t runs = 0;
};
std::uint32_t lt_forward_simulate(const DeviceGraph& dg, PrgState& s);
std::uint32_t lt_forward_simulate(const ProbGraph& g, const SuspectSet& vi, PrgState& s);
SuspensionEstimate estimate_suspension(const DeviceGraph& dg, const RemovalSet& removal,
                                       double epsilon, double delta, PrgState& s);
SuspensionEstimate estimate_suspension(const ProbGraph& g, const SuspectSet& vi,
                                       const RemovalSet& removal, double epsilon, double delta,
                                       PrgState& s);
// The paired runs themselves (not in the reference's interface; its loop body,
// proj/src/evaluation.cpp:233-236): infected counts of `runs` consecutive runs.
struct PairedRuns {
    std::vector<std::uint32_t> full, residual;
};
PairedRuns paired_runs(const DeviceGraph& dg, const RemovalSet& removal, std::uint64_t runs,
                       PrgState& s);

// ---- ranking baselines (proj/include/hsaw/evaluation.hpp:45-50) -----------------------------------
enum class BaselineKind { Pagerank, MaxDegree, Randomized, InfMaxV, InfMaxVI };
// Reverse-reachable node sets (rr_node_sets, proj/src/evaluation.cpp:169-191) drawn on the device
// from the caller's sequential stream, bit-exact (hsaw_gpu_rr_node_sets); s is advanced.
std::vector<std::vector<std::uint32_t>> rr_node_sets(const DeviceGraph& dg, PrgState& s,
                                                     std::uint32_t count);
std::vector<double> pagerank_scores(const ProbGraph& g, double damping = 0.85, double tol = 1e-10,
                                    int max_iters = 200);
// baseline() (evaluation.cpp:330-395). The InfMax kinds draw their sets and run greedy on the
// device (the sets never visit the host); Pagerank / MaxDegree / Randomized are host rankings as
// in the reference. Edge mode maps the ranked nodes to their heaviest in-edges round-robin.
RemovalSet baseline(const DeviceGraph& dg, const ProbGraph& g, const SuspectSet& vi,
                    BaselineKind kind, ItemKind mode, std::uint32_t k, PrgState& s,
                    std::uint32_t infmax_samples = 100000);
RemovalSet baseline(const ProbGraph& g, const SuspectSet& vi, BaselineKind kind, ItemKind mode,
                    std::uint32_t k, PrgState& s, std::uint32_t infmax_samples = 100000);
struct SolutionAnalysis {
    double ssr = 0;   // fraction of the solution drawn from the suspect set
    double cost = 0;  // sum (1 - p(v)) ln(d_in(v) + 1)
};
SolutionAnalysis analyze_solution(const ProbGraph& g, const SuspectSet& vi,
                                  const RemovalSet& removal);  // evaluation.cpp:397-412

// ---- cli (proj/include/hsaw/cli.hpp) ------------------------------------------------------------
int run_cli(std::vector<std::string> args);

}  // namespace hsaw
