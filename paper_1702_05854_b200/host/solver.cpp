// Host side of eSIA / nSIA: the sample-size schedule, the out-of-sample stopping rule and the
// doubling loop (north_star item 4 keeps these on the host). Sampling, greedy max-cover and the two
// coverage counts of every iteration run on the device through DeviceGraph / SampleStream /
// CoverageIndex. Follows /root/reference/proj/src/coverage.cpp:168-231 and interdiction.cpp:12-104;
// the FP64 expressions keep the reference's operation order so that ceil(lambda), t_max and eps_t
// come out bit-identical with the same libm.
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <sstream>

#include "hsaw_b200.hpp"

namespace hsaw {

// ---- schedule -----------------------------------------------------------------------------------
double ln_choose(std::uint64_t M, std::uint64_t k) {  // coverage.cpp:168-173
    double acc = 0.0;
    for (std::uint64_t i = 1; i <= k; ++i)
        acc += std::log(static_cast<double>(M - k + i) / static_cast<double>(i));
    return acc;
}

std::uint64_t Schedule::lambda_samples() const {
    return static_cast<std::uint64_t>(std::ceil(lambda));
}

Schedule compute_schedule_m(std::uint64_t M, std::uint32_t k, double epsilon, double delta) {
    if (!(epsilon > 0.0) || epsilon >= 1.0) throw std::invalid_argument("epsilon must be in (0,1)");
    if (!(delta > 0.0) || delta >= 1.0) throw std::invalid_argument("delta must be in (0,1)");
    if (k < 1 || k > M) throw std::invalid_argument("budget k out of range");
    Schedule out;
    out.epsilon = epsilon;
    out.delta = delta;
    out.k = k;
    const double two_minus_inv_e = 2.0 - 1.0 / std::exp(1.0);
    const double c = two_minus_inv_e * two_minus_inv_e;
    const double a = 2.0 + 2.0 * epsilon / 3.0;
    const double eps_sq = epsilon * epsilon;
    out.n_max = c * a * static_cast<double>(M) * (std::log(6.0 / delta) + ln_choose(M, k)) /
                (static_cast<double>(k) * eps_sq);
    const double lambda0 = a * std::log(3.0 / delta) / eps_sq;
    const double rounds = std::ceil(std::log2(2.0 * out.n_max / lambda0));
    out.t_max = rounds < 1.0 ? 1u : static_cast<std::uint32_t>(rounds);
    out.lambda = a * std::log(3.0 * out.t_max / delta) / eps_sq;
    out.lambda1 = 1.0 + (1.0 + epsilon) * a * std::log(3.0 * out.t_max / delta) / eps_sq;
    return out;
}

Schedule compute_schedule(const ProbGraph& g, ItemKind kind, std::uint32_t k, double epsilon,
                          double delta) {
    return compute_schedule_m(kind == ItemKind::Edge ? g.m : g.n, k, epsilon, delta);
}

// ---- stopping rule ------------------------------------------------------------------------------
CheckResult check_counts(double cov_r, double cov_rp, double n_rp, const Schedule& sched,
                         std::uint32_t t) {  // coverage.cpp:218-230
    if (cov_rp < sched.lambda1) return {false, std::numeric_limits<double>::infinity()};
    const double eps = sched.epsilon;
    const double doubling = std::ldexp(1.0, static_cast<int>(t) - 1);
    const double one_me = 1.0 - 1.0 / std::exp(1.0);
    const double eps1 = cov_r / cov_rp - 1.0;
    const double eps2 = eps * std::sqrt(n_rp * (1.0 + eps) / (doubling * cov_rp));
    const double eps3 = eps * std::sqrt(n_rp * (1.0 + eps) * (one_me - eps) /
                                        ((1.0 + eps / 3.0) * doubling * cov_rp));
    const double eps_t = (eps1 + eps2 + eps1 * eps2) * (one_me - eps) + one_me * eps3;
    return {eps_t <= eps, eps_t};
}

CheckResult check_solution(std::span<const std::uint32_t> solution, const CoverageIndex& idx_r,
                           const CoverageIndex& idx_r_prime, const Schedule& sched,
                           std::uint32_t t) {
    const auto cov_r = static_cast<double>(idx_r.coverage_of(solution));
    const auto cov_rp = static_cast<double>(idx_r_prime.coverage_of(solution));
    return check_counts(cov_r, cov_rp, static_cast<double>(idx_r_prime.num_samples()), sched, t);
}

// ---- doubling loop ------------------------------------------------------------------------------
namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

InterdictionResult run_on_device(const DeviceGraph& dg, const ProbGraph& g,
                                 const CandidateSet& cand, std::uint32_t k, double epsilon,
                                 double delta, const InterdictionOptions& opts) {
    cand.validate(g);
    if (k < 1 || k > cand.size(g))  // interdiction.cpp:17-18
        throw std::invalid_argument("budget k must be in [1, |C|]");
    const auto t0 = Clock::now();
    const Schedule sched = compute_schedule(g, cand.kind, k, epsilon, delta);
    const std::uint64_t base = sched.lambda_samples();

    // the pool keeps only the item lists this candidate kind indexes (coverage.cpp:49-53)
    SampleStream stream(dg, opts.seed, opts.sampler,
                        cand.kind == ItemKind::Edge ? SampleStream::Items::EdgesOnly
                                                    : SampleStream::Items::NodesOnly);
    InterdictionResult res;
    res.kind = cand.kind;
    res.k = k;
    res.epsilon = epsilon;
    res.delta = delta;

    std::uint64_t size = 0;
    GreedyResult picked;
    CheckResult verdict;
    std::uint32_t t = 0;
    const char* skip_env = std::getenv("HSAW_SKIP_BOUND");
    const bool skip_by_bound = !(skip_env && std::atoi(skip_env) == 0);
    bool bound_can_skip = true;
    for (;;) {  // interdiction.cpp:36-47
        ++t;
        size = base << (t - 1);
        auto ts = Clock::now();
        stream.ensure(2 * size);
        res.sample_s += seconds_since(ts);
        // R_t = samples [0, size), R'_t = [size, 2 size): two views of the device-resident pool
        CoverageIndex in_sample(cand.kind, stream, 0, size, cand, g);
        CoverageIndex out_of_sample(cand.kind, stream, size, size, cand, g);
        // check_solution fails whenever Cov_R'(solution) < Lambda_1 (coverage.cpp:216-217). If
        // even the k most frequent candidates of R'_t cannot reach Lambda_1 — and this is not the
        // last iteration N_max allows — the iteration cannot pass whatever greedy picks: skip its
        // greedy run and coverage counts. Only the final iteration's solution is ever reported
        // (interdiction.cpp:49-61), so the result is unchanged. HSAW_SKIP_BOUND=0 disables.
        if (skip_by_bound && bound_can_skip && static_cast<double>(size) < sched.n_max) {
            // Cov_R'(S) <= |R'_t| = size for every S: while size < Lambda_1 (always the case at
            // t = 1, where size = ceil(Lambda) and Lambda_1 = 1 + (1 + eps) Lambda) no histogram
            // is needed to know the answer
            if (static_cast<double>(size) < sched.lambda1) continue;
            ts = Clock::now();
            const auto bound = static_cast<double>(out_of_sample.coverage_upper_bound(k));
            res.check_s += seconds_since(ts);
            if (bound < sched.lambda1) continue;
            // The k largest counts of R'_t grow with its size (each R' is a fresh sample twice as
            // large) while Lambda_1 is fixed: once the bound has reached it, later iterations
            // will not be skipped either, and computing their bound only costs a histogram of
            // R'_t - half of all walk items in the final iteration, whose R' is never needed
            // again if the check passes. (Purely a cost decision: a bound is never required.)
            bound_can_skip = false;
        }
        ts = Clock::now();
        picked = greedy_max_cover(in_sample, k);
        res.greedy_s += seconds_since(ts);
        ts = Clock::now();
        // check_solution (coverage.cpp:212-231) with Cov_R(S) taken from the greedy run instead of
        // a second pass over R_t: the walks of a stream are self-avoiding (K2b), so no item occurs
        // twice in a walk and the sum of the marginal gains IS the number of walks S covers (the
        // zero-gain padding covers nothing new). HSAW_RECOUNT_COVERAGE=1 keeps the second pass.
        const char* recount_env = std::getenv("HSAW_RECOUNT_COVERAGE");  // (read per call: tests)
        const bool recount = recount_env && std::atoi(recount_env) != 0;
        if (recount) {
            verdict = check_solution(picked.solution, in_sample, out_of_sample, sched, t);
        } else {
            const auto cov_rp = static_cast<double>(out_of_sample.coverage_of(picked.solution));
            verdict = check_counts(static_cast<double>(picked.coverage), cov_rp,
                                   static_cast<double>(out_of_sample.num_samples()), sched, t);
        }
        res.check_s += seconds_since(ts);
        if (verdict.pass || static_cast<double>(size) >= sched.n_max) break;
    }

    res.solution = picked.solution;
    res.coverage = picked.coverage;
    res.samples_used = 2 * size;
    res.iterations = t;
    res.passed_check = verdict.pass;
    const auto counters = stream.counters_for(2 * size);
    res.attempts = counters.attempts;
    const double influence = static_cast<double>(g.n) * static_cast<double>(counters.accepted) /
                             static_cast<double>(counters.attempts);
    res.est_suspension =
        influence * static_cast<double>(picked.coverage) / static_cast<double>(size);
    res.wall_time_s = seconds_since(t0);
    return res;
}

void require_kind(const CandidateSet& cand, ItemKind want, const char* msg) {
    if (cand.kind != want) throw std::invalid_argument(msg);
}

}  // namespace

InterdictionResult esia(const DeviceGraph& dg, const ProbGraph& g, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts) {
    require_kind(cand, ItemKind::Edge, "esia requires an edge candidate set");
    return run_on_device(dg, g, cand, k, epsilon, delta, opts);
}

InterdictionResult nsia(const DeviceGraph& dg, const ProbGraph& g, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts) {
    require_kind(cand, ItemKind::Node, "nsia requires a node candidate set");
    return run_on_device(dg, g, cand, k, epsilon, delta, opts);
}

InterdictionResult esia(const ProbGraph& g, const SuspectSet& vi, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts) {
    require_kind(cand, ItemKind::Edge, "esia requires an edge candidate set");
    if (opts.devices.size() > 1) return run_interdiction_multi(g, vi, cand, k, epsilon, delta, opts);
    const auto t0 = Clock::now();
    DeviceGraph dg(g, vi, opts.devices.size() == 1 ? opts.devices[0] : opts.device);
    InterdictionResult res = run_on_device(dg, g, cand, k, epsilon, delta, opts);
    res.wall_time_s = seconds_since(t0);  // upload included, like a host-to-result call
    return res;
}

InterdictionResult nsia(const ProbGraph& g, const SuspectSet& vi, const CandidateSet& cand,
                        std::uint32_t k, double epsilon, double delta,
                        const InterdictionOptions& opts) {
    require_kind(cand, ItemKind::Node, "nsia requires a node candidate set");
    if (opts.devices.size() > 1) return run_interdiction_multi(g, vi, cand, k, epsilon, delta, opts);
    const auto t0 = Clock::now();
    DeviceGraph dg(g, vi, opts.devices.size() == 1 ? opts.devices[0] : opts.device);
    InterdictionResult res = run_on_device(dg, g, cand, k, epsilon, delta, opts);
    res.wall_time_s = seconds_since(t0);
    return res;
}

// ---- JSON ---------------------------------------------------------------------------------------
// Same document as nlohmann::json::dump(2) produces for the reference (interdiction.cpp:89-104):
// keys in alphabetical order, two-space indent, one array element per line, doubles in shortest
// round-trip form with a ".0" suffix when integral. tests/golden/interdict12.json is byte-stable.
// nlohmann::json::dump formats doubles with its Grisu2 "to_chars": shortest round-trip digits laid
// out in FIXED notation while the decimal exponent n satisfies -4 < n <= 15 ("0.0001",
// "100000.0", "1000000.0"; integral values get ".0"), otherwise d[.ddd]e[+-]XX with at least two
// exponent digits. std::to_chars alone would pick whichever form is shorter ("1e-04", "1e+05").
std::string json_number(double x) {
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    if (!std::isfinite(x)) return "null";  // nlohmann dumps non-finite numbers as null
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    std::string sci(buf, res.ptr);  // [-]d[.ddd]e[+-]XX, shortest round-trip digits
    std::string out;
    std::size_t pos = 0;
    if (sci[0] == '-') {
        out = "-";
        pos = 1;
    }
    const std::size_t epos = sci.find('e');
    std::string digits;
    for (std::size_t i = pos; i < epos; ++i)
        if (sci[i] != '.') digits += sci[i];
    const int exp10 = std::stoi(sci.substr(epos + 1));
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point relative to the digit string
    if (k <= n && n <= 15) {  // integral: digits, zero padding, ".0"
        out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {  // dig.its
        out += digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
    } else if (-4 < n && n <= 0) {  // 0.[000]digits
        out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {  // d[.igits]e+-XX
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

std::string to_json(const InterdictionResult& r, bool include_timing) {
    std::ostringstream out;
    out << "{\n";
    out << "  \"attempts\": " << r.attempts << ",\n";
    out << "  \"coverage\": " << r.coverage << ",\n";
    out << "  \"delta\": " << json_number(r.delta) << ",\n";
    out << "  \"epsilon\": " << json_number(r.epsilon) << ",\n";
    out << "  \"est_suspension\": " << json_number(r.est_suspension) << ",\n";
    out << "  \"iterations\": " << r.iterations << ",\n";
    out << "  \"k\": " << r.k << ",\n";
    out << "  \"kind\": \"" << to_string(r.kind) << "\",\n";
    out << "  \"passed_check\": " << (r.passed_check ? "true" : "false") << ",\n";
    out << "  \"samples_used\": " << r.samples_used << ",\n";
    out << "  \"solution\": [";
    if (r.solution.empty()) {
        out << "]";
    } else {
        for (std::size_t i = 0; i < r.solution.size(); ++i)
            out << (i ? ",\n    " : "\n    ") << r.solution[i];
        out << "\n  ]";
    }
    if (include_timing) out << ",\n  \"wall_time_s\": " << json_number(r.wall_time_s);
    out << "\n}";
    return out.str();
}

}  // namespace hsaw
