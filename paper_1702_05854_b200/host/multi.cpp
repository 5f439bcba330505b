// Multi-device eSIA / nSIA in the C++ host layer: one host thread per device, the
// graph replicated, walks sharded by batch range, marginal-gain counts combined with an all-reduce.
//
//  * batches (worker id = seed + b) are independent pure functions (proj/src/sampler.cpp:267-290,
//    430): every ensure() round's batch range is split into `world` contiguous blocks, rank r
//    samples block r on its device and keeps its walks. The global (batch, seq) order is
//    round-major / rank-major — the single-stream order of sampler.cpp:452-460 — so R_t and R'_t
//    (interdiction.cpp:38-41) are contiguous local ranges on every rank.
//  * exchange steps: per round an all-gather of `world` accepted counts; per upper bound one
//    all-reduce of the count vector; per greedy call one all-reduce of the count vector and one
//    all-gather of the walks restricted to the items that can still win, after which every rank
//    runs the single-device greedy redundantly (hsaw_gpu.h, "sharded solve"); scalar all-gathers
//    for coverage_of and counters_for. No walk crosses NVLink unreduced, no per-round exchange.
//  * transport: NCCL (libnccl.so.2, resolved at run time so the library loads without it):
//    ncclCommInitAll over the device list, ncclAllReduce / grouped ncclBroadcast on each
//    context's stream. When a device id repeats in the list — the only way to exercise this path
//    on a one-GPU box, NCCL refuses duplicate devices — the same steps run over an in-process
//    exchange (device-to-device copies + an add kernel).
//  * schedule, stopping rule and est_suspension are the single-device host functions
//    (solver.cpp), so InterdictionResult is identical for every device list.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "hsaw_b200.hpp"
#include "hsaw_gpu.h"

namespace hsaw {

namespace {

using Clock = std::chrono::steady_clock;

// ---- minimal NCCL surface, resolved with dlsym (types as in nccl.h 2.x) ---------------------------
using ncclComm_t = struct ncclComm*;
enum { kNcclSuccess = 0, kNcclUint32 = 3, kNcclSum = 0 };  // ncclUint32 = 3, ncclSum = 0 (nccl.h)
struct NcclApi {
    int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, void*) = nullptr;
    int (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, void*) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    int (*GetVersion)(int*) = nullptr;
    bool ok = false;
    static const NcclApi& get() {
        static const NcclApi api = [] {
            NcclApi a;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return a;
            auto sym = [&](const char* name, auto& fn) {
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
                return fn != nullptr;
            };
            a.ok = sym("ncclCommInitAll", a.CommInitAll) && sym("ncclCommDestroy", a.CommDestroy) &&
                   sym("ncclAllReduce", a.AllReduce) && sym("ncclBroadcast", a.Broadcast) &&
                   sym("ncclGroupStart", a.GroupStart) && sym("ncclGroupEnd", a.GroupEnd) &&
                   sym("ncclGetErrorString", a.GetErrorString) && sym("ncclGetVersion", a.GetVersion);
            return a;
        }();
        return api;
    }
};

// ---- rendezvous of the rank threads ----------------------------------------------------------------
// A barrier that can be poisoned: a rank that fails wakes everyone, who then throw too instead of
// waiting forever for a peer that is gone.
class Rendezvous {
public:
    explicit Rendezvous(int world) : world_(world) {}
    void arrive() {
        std::unique_lock<std::mutex> lock(mu_);
        if (failed_) throw DeviceError("a peer device failed");
        const std::uint64_t gen = generation_;
        if (++waiting_ == world_) {
            waiting_ = 0;
            ++generation_;
            cv_.notify_all();
            return;
        }
        cv_.wait(lock, [&] { return generation_ != gen || failed_; });
        if (failed_) throw DeviceError("a peer device failed");
    }
    void poison() {
        std::lock_guard<std::mutex> lock(mu_);
        failed_ = true;
        cv_.notify_all();
    }

private:
    const int world_;
    int waiting_ = 0;
    std::uint64_t generation_ = 0;
    bool failed_ = false;
    std::mutex mu_;
    std::condition_variable cv_;
};

void chk(int status, hsaw_gpu_ctx* ctx, const char* where) {
    if (status == HSAW_OK) return;
    const std::string msg = std::string(where) + ": " + hsaw_gpu_last_error(ctx);
    switch (status) {
        case HSAW_EINVAL: throw std::invalid_argument(msg);
        case HSAW_EDATA: throw DataError(msg);
        case HSAW_EBUDGET: throw SamplingError(msg);
        case HSAW_ERANGE: throw std::out_of_range(msg);
        default: throw DeviceError(msg);
    }
}

// ---- the collective steps -----------------------------------------------------------------------
class Exchange {
public:
    Exchange(const std::vector<int>& devices, std::vector<hsaw_gpu_ctx*> ctxs)
        : world_(static_cast<int>(devices.size())), ctxs_(std::move(ctxs)), meet_(world_),
          slots_u64_(world_), slots_ptr_(world_, nullptr) {
        std::vector<int> sorted = devices;
        std::sort(sorted.begin(), sorted.end());
        const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
        if (distinct && world_ > 1) {
            const NcclApi& nccl = NcclApi::get();
            if (!nccl.ok) throw DeviceError("multi-device solve: libnccl.so.2 not found");
            comms_.assign(world_, nullptr);
            const int rc = nccl.CommInitAll(comms_.data(), world_, devices.data());
            if (rc != kNcclSuccess)
                throw DeviceError(std::string("ncclCommInitAll: ") + nccl.GetErrorString(rc));
            int version = 0;
            nccl.GetVersion(&version);
            transport_ = "NCCL " + std::to_string(version) + " (ncclCommInitAll over " +
                         std::to_string(world_) + " devices)";
        } else {
            transport_ = "in-process exchange (a device id repeats: NCCL refuses duplicate devices)";
        }
    }
    ~Exchange() {
        for (ncclComm_t c : comms_)
            if (c) NcclApi::get().CommDestroy(c);
    }
    int world() const { return world_; }
    const std::string& transport() const { return transport_; }
    void poison() { meet_.poison(); }

    // every rank contributes `mine`; returns all contributions in rank order
    std::vector<std::vector<std::uint64_t>> all_gather_u64(int rank, std::vector<std::uint64_t> mine) {
        slots_u64_[rank] = std::move(mine);
        meet_.arrive();
        std::vector<std::vector<std::uint64_t>> all = slots_u64_;
        meet_.arrive();
        return all;
    }

    // in-place sum over ranks of `count` u32 counters on each rank's device
    void all_reduce_sum_u32(int rank, std::uint32_t* d_buf, std::uint64_t count) {
        if (world_ == 1) return;
        hsaw_gpu_ctx* ctx = ctxs_[rank];
        if (!comms_.empty()) {
            const NcclApi& nccl = NcclApi::get();
            const int rc = nccl.AllReduce(d_buf, d_buf, count, kNcclUint32, kNcclSum, comms_[rank],
                                          hsaw_gpu_ctx_cuda_stream(ctx));
            if (rc != kNcclSuccess)
                throw DeviceError(std::string("ncclAllReduce: ") + nccl.GetErrorString(rc));
            chk(hsaw_gpu_ctx_sync(ctx), ctx, "all_reduce");
            return;
        }
        slots_ptr_[rank] = d_buf;
        meet_.arrive();
        if (rank == 0) {  // rank 0 accumulates, everyone copies the sum back
            void* tmp = nullptr;
            chk(hsaw_gpu_device_alloc(ctx, count * 4, &tmp), ctx, "all_reduce");
            for (int r = 1; r < world_; ++r) {
                chk(hsaw_gpu_device_copy(ctx, tmp, slots_ptr_[r], count * 4), ctx, "all_reduce");
                chk(hsaw_gpu_counts_add(ctx, d_buf, static_cast<std::uint32_t*>(tmp), count), ctx,
                    "all_reduce");
            }
            hsaw_gpu_device_free(ctx, tmp);
        }
        meet_.arrive();
        if (rank != 0) chk(hsaw_gpu_device_copy(ctx, d_buf, slots_ptr_[0], count * 4), ctx, "all_reduce");
        meet_.arrive();
    }

    // concatenation, in rank order, of every rank's `n` u32 values -> a fresh buffer on this
    // rank's device (caller frees with hsaw_gpu_device_free); sizes[r] = rank r's length
    std::uint32_t* all_gather_u32(int rank, const std::uint32_t* d_mine, std::uint64_t n,
                                  std::vector<std::uint64_t>& sizes) {
        hsaw_gpu_ctx* ctx = ctxs_[rank];
        const auto lens = all_gather_u64(rank, {n});
        sizes.assign(world_, 0);
        std::uint64_t total = 0;
        for (int r = 0; r < world_; ++r) total += sizes[r] = lens[r][0];
        void* out = nullptr;
        chk(hsaw_gpu_device_alloc(ctx, (total ? total : 1) * 4, &out), ctx, "all_gather");
        auto* dst = static_cast<std::uint32_t*>(out);
        if (!comms_.empty()) {
            const NcclApi& nccl = NcclApi::get();
            nccl.GroupStart();
            std::uint64_t at = 0;
            for (int r = 0; r < world_; ++r) {
                if (sizes[r]) {
                    const int rc = nccl.Broadcast(r == rank ? d_mine : nullptr, dst + at, sizes[r],
                                                  kNcclUint32, r, comms_[rank],
                                                  hsaw_gpu_ctx_cuda_stream(ctx));
                    if (rc != kNcclSuccess)
                        throw DeviceError(std::string("ncclBroadcast: ") + nccl.GetErrorString(rc));
                }
                at += sizes[r];
            }
            nccl.GroupEnd();
            chk(hsaw_gpu_ctx_sync(ctx), ctx, "all_gather");
            return dst;
        }
        slots_ptr_[rank] = const_cast<std::uint32_t*>(d_mine);
        meet_.arrive();
        std::uint64_t at = 0;
        for (int r = 0; r < world_; ++r) {
            if (sizes[r]) chk(hsaw_gpu_device_copy(ctx, dst + at, slots_ptr_[r], sizes[r] * 4), ctx, "all_gather");
            at += sizes[r];
        }
        meet_.arrive();  // pieces may be released once everyone has copied them
        return dst;
    }

private:
    const int world_;
    std::vector<hsaw_gpu_ctx*> ctxs_;
    Rendezvous meet_;
    std::vector<std::vector<std::uint64_t>> slots_u64_;
    std::vector<void*> slots_ptr_;
    std::vector<ncclComm_t> comms_;
    std::string transport_;
};

// ---- where the global (batch, seq) order lives: per round, per rank ---------------------------------
struct Round {
    std::uint64_t first_batch = 0;
    std::vector<std::uint64_t> sizes, accepted;
    std::uint64_t block_start(int r) const {
        std::uint64_t at = first_batch;
        for (int i = 0; i < r; ++i) at += sizes[i];
        return at;
    }
};

struct Layout {
    int world = 1;
    std::vector<Round> rounds;
    std::uint64_t accepted() const {
        std::uint64_t a = 0;
        for (const Round& rd : rounds)
            for (std::uint64_t x : rd.accepted) a += x;
        return a;
    }
    // number of `rank`'s walks whose global position is below x
    std::uint64_t count_below(int rank, std::uint64_t x) const {
        std::uint64_t g = 0, total = 0;
        for (const Round& rd : rounds)
            for (int r = 0; r < world; ++r) {
                const std::uint64_t a = rd.accepted[r];
                if (r == rank) total += std::min(x > g ? x - g : 0, a);
                g += a;
            }
        return total;
    }
    std::pair<std::uint64_t, std::uint64_t> local_range(int rank, std::uint64_t off,
                                                        std::uint64_t cnt) const {
        const std::uint64_t lo = count_below(rank, off);
        return {lo, count_below(rank, off + cnt) - lo};
    }
};

struct Device {  // one rank: context + local stream
    std::unique_ptr<DeviceGraph> dg;
    hsaw_gpu_stream* stream = nullptr;
    ~Device() {
        if (stream) hsaw_gpu_stream_destroy(stream);
    }
};

class RankSolver {
public:
    RankSolver(int rank, Exchange& ex, Device& dev, const ProbGraph& g, const InterdictionOptions& opts)
        : rank_(rank), ex_(ex), dev_(dev), ctx_(dev.dg->ctx()), g_(g), opts_(opts) {
        layout_.world = ex.world();
    }

    // SampleStream::ensure (proj/src/sampler.cpp:388-463), sharded
    void ensure(std::uint64_t min_accepted) {
        const std::uint64_t bs = opts_.sampler.batch_size;
        const int w = ex_.world();
        while (layout_.accepted() < min_accepted) {
            const std::uint64_t attempts_so_far = next_batch_ * bs;
            const std::uint64_t budget_left = opts_.sampler.max_attempts > attempts_so_far
                                                  ? opts_.sampler.max_attempts - attempts_so_far
                                                  : 0;
            const std::uint64_t max_batches = budget_left / bs;
            if (max_batches == 0)
                throw SamplingError("attempt budget exhausted while sampling walks; suspects may be "
                                    "unreachable");
            const std::uint64_t have = layout_.accepted();
            std::uint64_t batches;
            if (have == 0) {
                batches = grow_;
                grow_ = std::min<std::uint64_t>(grow_ * 8, 1ull << 22);
            } else {  // only a speed knob: results are cut at whole-batch prefixes
                const double rate = static_cast<double>(have) / static_cast<double>(attempts_so_far);
                batches = static_cast<std::uint64_t>(
                              static_cast<double>(min_accepted - have) / (rate * static_cast<double>(bs)) * 1.02) +
                          64;
            }
            batches = std::max<std::uint64_t>(std::min(batches, max_batches), 1);
            Round rd;
            rd.first_batch = next_batch_;
            rd.sizes.assign(w, batches / w);
            for (std::uint64_t r = 0; r < batches % w; ++r) ++rd.sizes[r];
            std::uint64_t got = 0;
            if (rd.sizes[rank_])
                chk(hsaw_gpu_stream_sample_range(dev_.stream, rd.block_start(rank_), rd.sizes[rank_], &got),
                    ctx_, "sample_range");
            const auto all = ex_.all_gather_u64(rank_, {got});
            rd.accepted.resize(w);
            for (int r = 0; r < w; ++r) rd.accepted[r] = all[r][0];
            layout_.rounds.push_back(std::move(rd));
            next_batch_ += batches;
        }
    }

    // SampleStream::counters_for (sampler.cpp:472-482), sharded: the owner of the block in which
    // the cumulative count reaches the target answers for everyone
    void counters_for(std::uint64_t min_accepted, std::uint64_t& attempts, std::uint64_t& accepted) {
        attempts = accepted = 0;
        if (min_accepted == 0) return;
        std::uint64_t g = 0;
        for (std::size_t j = 0; j < layout_.rounds.size(); ++j) {
            const Round& rd = layout_.rounds[j];
            for (int r = 0; r < layout_.world; ++r) {
                if (g + rd.accepted[r] < min_accepted) {
                    g += rd.accepted[r];
                    continue;
                }
                std::vector<std::uint64_t> mine{0, 0};
                if (r == rank_) {
                    std::uint64_t local_before = 0, batches_before = 0;
                    for (std::size_t i = 0; i < j; ++i) {
                        local_before += layout_.rounds[i].accepted[r];
                        batches_before += layout_.rounds[i].sizes[r];
                    }
                    std::uint64_t nb = 0, acc = 0;
                    chk(hsaw_gpu_stream_local_cut(dev_.stream, local_before + (min_accepted - g), &nb, &acc),
                        ctx_, "local_cut");
                    const std::uint64_t global_batches = rd.block_start(r) + (nb - batches_before);
                    mine = {global_batches * opts_.sampler.batch_size, g + (acc - local_before)};
                }
                const auto all = ex_.all_gather_u64(rank_, mine);
                attempts = all[r][0];
                accepted = all[r][1];
                return;
            }
        }
        throw std::out_of_range("sample stream target not materialized");
    }

    std::uint64_t coverage_of(const std::vector<std::uint32_t>& items, int kind, std::uint64_t off,
                              std::uint64_t cnt, const CandidateSet& cand) {
        const auto [lo, n] = layout_.local_range(rank_, off, cnt);
        std::uint64_t local = 0;
        if (n)
            chk(hsaw_gpu_coverage_of(ctx_, dev_.stream, nullptr, kind, lo, n,
                                     cand.ids ? cand.ids->data() : nullptr,
                                     cand.ids ? cand.ids->size() : 0, items.data(), items.size(), &local),
                ctx_, "coverage_of");
        std::uint64_t total = 0;
        for (const auto& v : ex_.all_gather_u64(rank_, {local})) total += v[0];
        return total;
    }

    // all-reduced counts of global walks [off, off + cnt) on this rank's device (caller frees)
    std::uint32_t* global_counts(int kind, std::uint64_t off, std::uint64_t cnt, const CandidateSet& cand,
                                 std::uint32_t limit) {
        const auto [lo, n] = layout_.local_range(rank_, off, cnt);
        void* buf = nullptr;
        chk(hsaw_gpu_device_alloc(ctx_, static_cast<std::uint64_t>(limit) * 4, &buf), ctx_, "counts");
        auto* counts = static_cast<std::uint32_t*>(buf);
        chk(hsaw_gpu_stream_histogram(ctx_, dev_.stream, kind, lo, n, cand.ids ? cand.ids->data() : nullptr,
                                      cand.ids ? cand.ids->size() : 0, counts),
            ctx_, "stream_histogram");
        ex_.all_reduce_sum_u32(rank_, counts, limit);
        return counts;
    }

    std::uint64_t coverage_upper_bound(std::uint32_t k, int kind, std::uint64_t off, std::uint64_t cnt,
                                       const CandidateSet& cand, std::uint32_t limit) {
        std::uint32_t* counts = global_counts(kind, off, cnt, cand, limit);
        std::uint64_t bound = 0;
        const int rc = hsaw_gpu_counts_bound(ctx_, counts, limit, k, cnt, &bound);
        hsaw_gpu_device_free(ctx_, counts);
        chk(rc, ctx_, "counts_bound");
        return bound;
    }

    // greedy_max_cover on global walks [0, size): gather-and-replicate (see the file header)
    GreedyResult greedy(std::uint32_t k, int kind, std::uint64_t size, const CandidateSet& cand,
                        std::uint32_t limit) {
        const auto [lo, n] = layout_.local_range(rank_, 0, size);
        std::uint32_t* counts = global_counts(kind, 0, size, cand, limit);
        GreedyResult res;
        res.solution.resize(k);
        try {
            // thresholds from bold to safe: 60 %, 30 % of the k-th largest count, the 1/8-mass rule,
            // then everything; a run whose smallest gain stays at or above its threshold is exact
            std::vector<std::uint32_t> ladder;
            for (std::uint32_t pct : {60u, 30u, 0u}) {
                std::uint32_t mc = 1;
                chk(hsaw_gpu_counts_threshold_for(ctx_, counts, limit, k, pct, &mc), ctx_,
                    "counts_threshold");
                if (ladder.empty() || mc < ladder.back()) ladder.push_back(mc);
            }
            if (ladder.back() > 1) ladder.push_back(1);
            std::size_t rung = 0;
            std::uint32_t min_count = ladder[rung];
            for (;;) {
                hsaw_gpu_walkset* mine = nullptr;
                std::uint64_t nsets = 0, nitems = 0;
                chk(hsaw_gpu_reduced_walks(ctx_, dev_.stream, kind, lo, n, counts, min_count, &mine, &nsets,
                                           &nitems),
                    ctx_, "reduced_walks");
                void *d_lens = nullptr, *d_items = nullptr;
                chk(hsaw_gpu_device_alloc(ctx_, (nsets ? nsets : 1) * 4, &d_lens), ctx_, "greedy");
                chk(hsaw_gpu_device_alloc(ctx_, (nitems ? nitems : 1) * 4, &d_items), ctx_, "greedy");
                const int rc = hsaw_gpu_walkset_copy_device(mine, static_cast<std::uint32_t*>(d_lens),
                                                            static_cast<std::uint32_t*>(d_items));
                hsaw_gpu_walkset_destroy(mine);
                chk(rc, ctx_, "walkset_copy_device");
                std::vector<std::uint64_t> len_sizes, item_sizes;
                std::uint32_t* all_lens =
                    ex_.all_gather_u32(rank_, static_cast<std::uint32_t*>(d_lens), nsets, len_sizes);
                std::uint32_t* all_items =
                    ex_.all_gather_u32(rank_, static_cast<std::uint32_t*>(d_items), nitems, item_sizes);
                hsaw_gpu_device_free(ctx_, d_lens);
                hsaw_gpu_device_free(ctx_, d_items);
                std::uint64_t tot_sets = 0, tot_items = 0;
                for (std::uint64_t x : len_sizes) tot_sets += x;
                for (std::uint64_t x : item_sizes) tot_items += x;
                hsaw_gpu_walkset* all = nullptr;
                const int rc2 = hsaw_gpu_walkset_from_device(ctx_, limit, tot_sets, all_lens, all_items,
                                                             tot_items, &all);
                hsaw_gpu_device_free(ctx_, all_lens);
                hsaw_gpu_device_free(ctx_, all_items);
                chk(rc2, ctx_, "walkset_from_device");
                const int rc3 = hsaw_gpu_greedy(ctx_, nullptr, all, kind, 0, tot_sets,
                                                cand.ids ? cand.ids->data() : nullptr,
                                                cand.ids ? cand.ids->size() : 0, k, res.solution.data(),
                                                &res.coverage);
                hsaw_gpu_walkset_destroy(all);
                chk(rc3, ctx_, "greedy");
                if (min_count <= 1 || hsaw_gpu_last_greedy_min_gain(ctx_) >= min_count) break;
                min_count = ladder[++rung];  // the k-th gain fell below the threshold: next rung
            }
        } catch (...) {
            hsaw_gpu_device_free(ctx_, counts);
            throw;
        }
        hsaw_gpu_device_free(ctx_, counts);
        return res;
    }

    // run_interdiction (proj/src/interdiction.cpp:12-67), sharded
    InterdictionResult solve(const CandidateSet& cand, std::uint32_t k, double epsilon, double delta) {
        const auto t0 = Clock::now();
        const int kind = cand.kind == ItemKind::Edge ? HSAW_KIND_EDGE : HSAW_KIND_NODE;
        const std::uint32_t limit = cand.kind == ItemKind::Edge ? g_.m : g_.n;
        const Schedule sched = compute_schedule(g_, cand.kind, k, epsilon, delta);
        const std::uint64_t base = sched.lambda_samples();
        InterdictionResult res;
        res.kind = cand.kind;
        res.k = k;
        res.epsilon = epsilon;
        res.delta = delta;
        std::uint64_t size = 0;
        GreedyResult picked;
        CheckResult verdict;
        std::uint32_t t = 0;
        bool bound_can_skip = true;
        auto since = [](Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); };
        for (;;) {
            ++t;
            size = base << (t - 1);
            auto ts = Clock::now();
            ensure(2 * size);
            res.sample_s += since(ts);
            if (bound_can_skip && static_cast<double>(size) < sched.n_max) {  // same skips as the single-device loop
                if (static_cast<double>(size) < sched.lambda1) continue;
                ts = Clock::now();
                const auto bound = static_cast<double>(coverage_upper_bound(k, kind, size, size, cand, limit));
                res.check_s += since(ts);
                if (bound < sched.lambda1) continue;
                bound_can_skip = false;  // reached once: later (larger) R' will reach it too
            }
            ts = Clock::now();
            picked = greedy(k, kind, size, cand, limit);
            res.greedy_s += since(ts);
            ts = Clock::now();
            const std::uint64_t cov_r = coverage_of(picked.solution, kind, 0, size, cand);
            const std::uint64_t cov_rp = coverage_of(picked.solution, kind, size, size, cand);
            verdict = check_counts(static_cast<double>(cov_r), static_cast<double>(cov_rp),
                                   static_cast<double>(size), sched, t);
            res.check_s += since(ts);
            if (verdict.pass || static_cast<double>(size) >= sched.n_max) break;
        }
        res.solution = picked.solution;
        res.coverage = picked.coverage;
        res.samples_used = 2 * size;
        res.iterations = t;
        res.passed_check = verdict.pass;
        std::uint64_t attempts = 0, accepted = 0;
        counters_for(2 * size, attempts, accepted);
        res.attempts = attempts;
        const double influence =
            static_cast<double>(g_.n) * static_cast<double>(accepted) / static_cast<double>(attempts);
        res.est_suspension = influence * static_cast<double>(picked.coverage) / static_cast<double>(size);
        res.wall_time_s = since(t0);
        return res;
    }

private:
    const int rank_;
    Exchange& ex_;
    Device& dev_;
    hsaw_gpu_ctx* ctx_;
    const ProbGraph& g_;
    const InterdictionOptions& opts_;
    Layout layout_;
    std::uint64_t next_batch_ = 0, grow_ = 4096;
};

}  // namespace

std::string multi_device_transport(const std::vector<int>& devices) {
    std::vector<int> sorted = devices;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (devices.size() < 2) return "single device";
    if (!distinct) return "in-process exchange";
    return NcclApi::get().ok ? "nccl" : "nccl (libnccl.so.2 not found)";
}

InterdictionResult run_interdiction_multi(const ProbGraph& g, const SuspectSet& vi,
                                          const CandidateSet& cand, std::uint32_t k, double epsilon,
                                          double delta, const InterdictionOptions& opts) {
    cand.validate(g);
    if (k < 1 || k > cand.size(g)) throw std::invalid_argument("budget k must be in [1, |C|]");
    const int world = static_cast<int>(opts.devices.size());
    const auto t0 = Clock::now();
    // replicate the graph: one context per listed device, uploads in parallel
    std::vector<Device> devs(world);
    {
        std::vector<std::thread> up;
        std::vector<std::exception_ptr> err(world);
        for (int r = 0; r < world; ++r)
            up.emplace_back([&, r] {
                try {
                    devs[r].dg = std::make_unique<DeviceGraph>(g, vi, opts.devices[r]);
                } catch (...) {
                    err[r] = std::current_exception();
                }
            });
        for (auto& t : up) t.join();
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
    }
    hsaw_sampler_cfg cfg{};
    cfg.heuristic = opts.sampler.heuristic == CycleHeuristic::Brent   ? 0
                    : opts.sampler.heuristic == CycleHeuristic::Floyd ? 1
                                                                      : 2;
    cfg.window = opts.sampler.window;
    cfg.batch_size = opts.sampler.batch_size;
    cfg.max_attempts = ~0ull >> 2;  // the budget is enforced globally (RankSolver::ensure)
    cfg.rng_mode = opts.sampler.rng == WalkRng::PhiloxPerWalk ? 1u : 0u;
    std::vector<hsaw_gpu_ctx*> ctxs(world);
    const bool edges = cand.kind == ItemKind::Edge;
    for (int r = 0; r < world; ++r) {
        ctxs[r] = devs[r].dg->ctx();
        chk(hsaw_gpu_stream_create(ctxs[r], opts.seed, &cfg, &devs[r].stream), ctxs[r], "stream_create");
        chk(hsaw_gpu_stream_keep(devs[r].stream, edges ? 0 : 1, edges ? 1 : 0), ctxs[r], "stream_keep");
    }
    Exchange ex(opts.devices, ctxs);
    std::vector<InterdictionResult> results(world);
    std::vector<std::exception_ptr> err(world);
    std::vector<std::thread> ranks;
    for (int r = 0; r < world; ++r)
        ranks.emplace_back([&, r] {
            try {
                RankSolver solver(r, ex, devs[r], g, opts);
                results[r] = solver.solve(cand, k, epsilon, delta);
            } catch (...) {
                err[r] = std::current_exception();
                ex.poison();
            }
        });
    for (auto& t : ranks) t.join();
    // report the first real failure (peers that were only woken up by it come later)
    for (auto& e : err) {
        if (!e) continue;
        try {
            std::rethrow_exception(e);
        } catch (const DeviceError& d) {
            if (std::string(d.what()) == "a peer device failed") continue;
            throw;
        }
    }
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
    InterdictionResult res = results[0];
    res.wall_time_s = std::chrono::duration<double>(Clock::now() - t0).count();
    return res;
}

}  // namespace hsaw
