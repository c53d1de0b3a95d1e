// plse_b200.hpp -- the C++ host API above the C ABI (header-only, C++17).
//
// Mirrors the reference's public C++ interface (/root/reference/proj/include/plse)
// with the same names, argument meaning and error behaviour, so code written
// against the reference switches by changing the namespace:
//
//   reference                                   here
//   instance.hpp  PlsInstance, generate_instance,  PlsInstance, generate_instance,
//                 parse_instance, serialize_..,     parse_instance, serialize_instance,
//                 load_instance, save_instance      load_instance, save_instance
//   rng.hpp       derive_seed                       derive_seed
//   lsgraph.hpp   preprocess(build_graph(..))       preprocess -> ReducedGraph
//   engine.hpp    SolverConfig, RunLimits,          SolverConfig, RunLimits,
//                 GenerationStats, RunResult, run   GenerationStats, RunResult, run
//   coloring.hpp  to_grid                           to_grid
//   verify.hpp    verify_certificate                verify_certificate
//   oracle.hpp    solve_exact                       solve_exact
//   report.hpp    variant_name/parse_*, result_to_json(..).dump(2)
//                                                   the same names; result_to_json returns the dump(2) text
//
// run() executes on one B200 through plse_solve (no CPU fallback: without an
// sm_100 device it throws CudaError).  SolverConfig gains two device fields:
// `device` and `tie_mode` (PLSE_TIE_REF reproduces the reference's trajectories
// bit for bit; PLSE_TIE_CANON is the throughput mode).  Errors: invalid
// arguments throw std::invalid_argument, parse / runtime failures
// std::runtime_error, device failures CudaError, requests outside the device
// envelope Unsupported.
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "plse_b200.h"

namespace plse_b200 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc, const plse_ctx* ctx = nullptr) {
    if (rc == PLSE_OK) return;
    const std::string msg = plse_last_error(ctx);
    if (rc == PLSE_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == PLSE_ERR_CUDA) throw CudaError(msg);
    if (rc == PLSE_ERR_UNSUPPORTED) throw Unsupported(msg);
    throw std::runtime_error(msg);
}

// ------------------------------------------------------------------ instance.hpp
class PlsInstance {
public:
    PlsInstance() = default;
    explicit PlsInstance(int n) : n_(n), cells_(static_cast<size_t>(n) * n, 0) {
        if (n <= 0) throw std::invalid_argument("order must be positive");
    }
    int order() const { return n_; }
    uint16_t at(int r, int c) const { return cells_[static_cast<size_t>(r) * n_ + c]; }
    void set(int r, int c, uint16_t s) {
        if (s > n_) throw std::invalid_argument("symbol out of range");
        cells_[static_cast<size_t>(r) * n_ + c] = s;
    }
    int filled_count() const {
        int k = 0;
        for (uint16_t s : cells_) k += s != 0;
        return k;
    }
    double fill_ratio() const { return static_cast<double>(filled_count()) / (static_cast<double>(n_) * n_); }
    const uint16_t* data() const { return cells_.data(); }
    uint16_t* data() { return cells_.data(); }
    bool operator==(const PlsInstance& o) const { return n_ == o.n_ && cells_ == o.cells_; }

private:
    int n_ = 0;
    std::vector<uint16_t> cells_;
};

inline PlsInstance generate_instance(int n, double r, uint64_t seed) {
    PlsInstance g(n);
    check(plse_generate_instance(n, r, seed, g.data()));
    return g;
}

inline PlsInstance parse_instance(const std::string& text) {
    int32_t n = 0;
    check(plse_parse_instance(text.c_str(), &n, nullptr, 0));
    PlsInstance g(n);
    check(plse_parse_instance(text.c_str(), &n, g.data(), n * n));
    return g;
}

inline std::string serialize_instance(const PlsInstance& g) {
    std::ostringstream out;
    const int n = g.order();
    out << n << '\n';
    for (int r = 0; r < n; ++r) {
        for (int c = 0; c < n; ++c) {
            if (c) out << ' ';
            out << g.at(r, c);
        }
        out << '\n';
    }
    return out.str();
}

inline PlsInstance load_instance(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open instance file: " + path);
    std::ostringstream buffer;
    buffer << in.rdbuf();
    return parse_instance(buffer.str());
}

inline void save_instance(const PlsInstance& g, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write file: " + path);
    out << serialize_instance(g);
}

// ----------------------------------------------------------------------- rng.hpp
inline uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
    uint64_t s = master;
    uint64_t h = splitmix64(s);
    s = h ^ (tag * 0xD1B54A32D192ED03ULL);
    h = splitmix64(s);
    s = h ^ (index * 0x8CB92BA72F3D8DD7ULL);
    return splitmix64(s);
}

namespace stream_tag {
inline constexpr uint64_t kInitPopulation = 1, kImprove = 2, kCrossover = 3, kInstanceGen = 4, kBench = 5, kMatch = 6;
}

// ------------------------------------------------------------------- lsgraph.hpp
class ReducedGraph {
public:
    explicit ReducedGraph(const PlsInstance& g) {
        check(plse_preprocess(g.order(), g.data(), &h_));
        check(plse_graph_view(h_, &view_));
    }
    ~ReducedGraph() { plse_graph_free(h_); }
    ReducedGraph(const ReducedGraph&) = delete;
    ReducedGraph& operator=(const ReducedGraph&) = delete;
    ReducedGraph(ReducedGraph&& o) noexcept : h_(o.h_), view_(o.view_) { o.h_ = nullptr; }

    int order() const { return view_.order; }
    int vertex_count() const { return view_.vertex_count; }
    int l() const { return view_.l; }
    const plse_graph& view() const { return view_; }
    const plse_graph_h* handle() const { return h_; }

private:
    plse_graph_h* h_ = nullptr;
    plse_graph view_{};
};

inline ReducedGraph preprocess(const PlsInstance& g) { return ReducedGraph(g); }

// lsgraph.hpp:220-225 compute_bounds
struct InstanceBounds {
    int l = 0;
    int upper_bound = 0;
};
inline InstanceBounds compute_bounds(const ReducedGraph& g) {
    const int n = g.order();
    return {g.l(), g.l() == 1 ? n * n - 2 : n * n - g.l()};
}

// -------------------------------------------------------------------- engine.hpp
enum class Variant { MPMA, PartialMPMA };
enum class CrossoverMode { AUX, UX, None };
enum class MatchingStrategy { NearestNeighbor, Random };
enum class ExclusionScope { Run, Generation, Off };

struct CrossoverConfig {
    CrossoverMode mode = CrossoverMode::AUX;
    double beta = 20.0;
    MatchingStrategy matching = MatchingStrategy::NearestNeighbor;
    ExclusionScope exclusion = ExclusionScope::Run;
};

struct RunLimits {
    double time_seconds = 0;
    int64_t total_iterations = 0;
    int64_t generations = 0;
};

struct SolverConfig {
    int p = 12288;
    double alpha = 0.6;
    int64_t phase1_iters = 0;
    int64_t phase2_iters = 0;
    double gamma = 10.0;
    Variant variant = Variant::MPMA;
    CrossoverConfig crossover;
    RunLimits limits;
    uint64_t master_seed = 0;
    int workers = 1;
    // device path
    int device = 0;
    int tie_mode = PLSE_TIE_CANON;

    void validate() const {
        if (p < 2) throw std::invalid_argument("population size must be at least 2");
        if (!(gamma > 1.0)) throw std::invalid_argument("gamma must exceed 1");
        if (crossover.mode == CrossoverMode::AUX && !(crossover.beta > gamma))
            throw std::invalid_argument("beta must exceed gamma");
        if (!(alpha >= 0.0)) throw std::invalid_argument("alpha must be non-negative");
        if (phase1_iters < 0 || phase2_iters < 0) throw std::invalid_argument("phase budgets must be positive");
        if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    }

    plse_params params() const {
        plse_params q{};
        q.p = p;
        q.alpha = alpha;
        q.gamma = gamma;
        q.beta = crossover.beta;
        q.phase1_iters = phase1_iters;
        q.crossover = static_cast<int32_t>(crossover.mode);
        q.matching = static_cast<int32_t>(crossover.matching);
        q.exclusion = static_cast<int32_t>(crossover.exclusion);
        q.tie_mode = tie_mode;
        q.master_seed = master_seed;
        q.p_total = 0;
        q.offset = 0;
        q.variant = variant == Variant::MPMA ? PLSE_V_MPMA : PLSE_V_PARTIAL;
        q.phase2_iters = phase2_iters;
        return q;
    }
};

struct GenerationStats {
    int64_t generation = 0;
    int best_f = 0;
    double mean_f = 0;
    double mean_distance = 0;
    int64_t iterations = 0;
    double elapsed_seconds = 0;
    int shortfall = 0;
};

using GenerationCallback = std::function<void(const GenerationStats&)>;

struct RunResult {
    int best_score = 0;
    int best_f = 0;
    int l = 0;
    int upper_bound = 0;
    int vertex_count = 0;
    bool proven_optimal = false;
    int64_t generations = 0;
    int64_t total_iterations = 0;
    double elapsed_seconds = 0;
    double time_to_best_seconds = 0;
    std::string stop_reason;
    std::vector<uint16_t> best_solution;  // |V| colours
};

inline const char* stop_reason_name(int code) {
    static const char* names[] = {"optimal", "time_limit", "iteration_limit", "generation_limit", "trivial", "target"};
    return code >= 0 && code < 6 ? names[code] : "unknown";
}

// engine.hpp:114-262 on one device
inline RunResult run(const PlsInstance& instance, const SolverConfig& config, const GenerationCallback& on_generation = {}) {
    config.validate();
    plse_solver_config cfg{};
    cfg.params = config.params();
    cfg.variant = cfg.params.variant;
    cfg.time_limit = config.limits.time_seconds;
    cfg.iteration_limit = config.limits.total_iterations;
    cfg.generation_limit = config.limits.generations;
    cfg.device = config.device;
    plse_run_result res{};
    std::vector<uint16_t> best(static_cast<size_t>(instance.order()) * instance.order() + 1, 0);
    struct Ctx {
        const GenerationCallback* cb;
        std::exception_ptr err;
    } ctx{&on_generation, nullptr};
    auto tramp = [](const plse_generation_stats* s, void* user) {
        auto* c = static_cast<Ctx*>(user);
        if (c->err) return;
        try {
            GenerationStats g;
            g.generation = s->generation;
            g.best_f = s->best_f;
            g.mean_f = s->mean_f;
            g.mean_distance = s->mean_distance;
            g.iterations = s->iterations;
            g.elapsed_seconds = s->elapsed_seconds;
            g.shortfall = s->shortfall;
            (*c->cb)(g);
        } catch (...) {
            c->err = std::current_exception();
        }
    };
    check(plse_solve(instance.order(), instance.data(), &cfg, &res, best.data(),
                     on_generation ? +tramp : nullptr, &ctx));
    if (ctx.err) std::rethrow_exception(ctx.err);
    RunResult r;
    r.best_score = res.best_score;
    r.best_f = res.best_f;
    r.l = res.l;
    r.upper_bound = res.upper_bound;
    r.vertex_count = res.vertex_count;
    r.proven_optimal = res.proven_optimal != 0;
    r.generations = res.generations;
    r.total_iterations = res.total_iterations;
    r.elapsed_seconds = res.elapsed_seconds;
    r.time_to_best_seconds = res.time_to_best_seconds;
    r.stop_reason = stop_reason_name(res.stop_reason);
    r.best_solution.assign(best.begin(), best.begin() + res.vertex_count);
    return r;
}

// ------------------------------------------------------- coloring / verify / oracle
inline PlsInstance to_grid(const PlsInstance& instance, const ReducedGraph& reduced,
                           const std::vector<uint16_t>& solution) {
    if (static_cast<int>(solution.size()) != reduced.vertex_count())
        throw std::invalid_argument("solution size differs from the graph's vertex count");
    PlsInstance out(instance.order());
    check(plse_to_grid(reduced.handle(), solution.data(), out.data()));
    return out;
}

struct VerifyReport {
    bool legal = false;
    int score = 0;
    std::vector<std::string> problems;
};

inline VerifyReport verify_certificate(const PlsInstance& instance, const PlsInstance& certificate) {
    int32_t legal = 0, score = 0;
    int64_t len = 0;
    check(plse_verify_certificate(instance.order(), instance.data(), certificate.order(), certificate.data(), &legal,
                                  &score, nullptr, 0, &len));
    std::string text(static_cast<size_t>(len) + 1, '\0');
    check(plse_verify_certificate(instance.order(), instance.data(), certificate.order(), certificate.data(), &legal,
                                  &score, text.data(), static_cast<int64_t>(text.size()), &len));
    text.resize(static_cast<size_t>(len));
    VerifyReport r;
    r.legal = legal != 0;
    r.score = score;
    size_t at = 0;
    while (!text.empty() && at <= text.size()) {
        const size_t nl = text.find('\n', at);
        r.problems.push_back(text.substr(at, nl == std::string::npos ? std::string::npos : nl - at));
        if (nl == std::string::npos) break;
        at = nl + 1;
    }
    return r;
}

struct OracleResult {
    int optimum_f = 0;
    std::vector<uint16_t> certificate;
    bool exact = true;
    int64_t nodes = 0;
};

inline OracleResult solve_exact(const ReducedGraph& reduced, int64_t node_budget = 50'000'000) {
    OracleResult r;
    r.certificate.assign(static_cast<size_t>(reduced.vertex_count()) + 1, 0);
    int32_t f = 0, exact = 0;
    check(plse_solve_exact(reduced.handle(), node_budget, &f, &exact, &r.nodes, r.certificate.data()));
    r.certificate.resize(static_cast<size_t>(reduced.vertex_count()));
    r.optimum_f = f;
    r.exact = exact != 0;
    return r;
}

// --------------------------------------------------------------------- report.hpp
inline const char* variant_name(Variant v) { return v == Variant::MPMA ? "mpma" : "partial"; }
inline Variant parse_variant(const std::string& s) {
    if (s == "mpma") return Variant::MPMA;
    if (s == "partial") return Variant::PartialMPMA;
    throw std::invalid_argument("unknown variant: " + s);
}
inline const char* crossover_name(CrossoverMode m) {
    return m == CrossoverMode::AUX ? "aux" : m == CrossoverMode::UX ? "ux" : "none";
}
inline CrossoverMode parse_crossover(const std::string& s) {
    if (s == "aux") return CrossoverMode::AUX;
    if (s == "ux") return CrossoverMode::UX;
    if (s == "none") return CrossoverMode::None;
    throw std::invalid_argument("unknown crossover mode: " + s);
}
inline const char* matching_name(MatchingStrategy m) {
    return m == MatchingStrategy::NearestNeighbor ? "nearest" : "random";
}
inline MatchingStrategy parse_matching(const std::string& s) {
    if (s == "nearest") return MatchingStrategy::NearestNeighbor;
    if (s == "random") return MatchingStrategy::Random;
    throw std::invalid_argument("unknown matching strategy: " + s);
}
inline const char* exclusion_name(ExclusionScope e) {
    return e == ExclusionScope::Run ? "run" : e == ExclusionScope::Generation ? "generation" : "off";
}
inline ExclusionScope parse_exclusion(const std::string& s) {
    if (s == "run") return ExclusionScope::Run;
    if (s == "generation") return ExclusionScope::Generation;
    if (s == "off") return ExclusionScope::Off;
    throw std::invalid_argument("unknown exclusion scope: " + s);
}

// a minimal ordered-JSON printer with nlohmann's dump(2) conventions: 2-space indent, ": ",
// shortest round-trip doubles (with ".0" when integral), non-finite -> null
namespace json_detail {
// shortest round-trip digits, laid out like nlohmann::detail::dtoa_impl::format_buffer
inline std::string number(double x) {
    if (!std::isfinite(x)) return "null";
    if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    std::string sci(buf, res.ptr), out;
    if (sci[0] == '-') {
        out = "-";
        sci.erase(0, 1);
    }
    const size_t epos = sci.find('e');
    std::string digits = sci.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int e10 = std::stoi(sci.substr(epos + 1));
    const int k = static_cast<int>(digits.size()), n = e10 + 1;  // digits d1..dk, value 0.d1..dk * 10^n
    if (k <= n && n <= 15) return out + digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    if (0 < n && n <= 15) return out + digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    if (-4 < n && n <= 0) return out + "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    std::string m = digits.substr(0, 1);
    if (k > 1) m += "." + digits.substr(1);
    const int ex = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    return out + m + eb;
}
inline std::string quote(const std::string& s) {
    std::string o = "\"";
    for (unsigned char ch : s) {
        switch (ch) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (ch < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", ch);
                    o += b;
                } else {
                    o += static_cast<char>(ch);
                }
        }
    }
    return o + "\"";
}
struct Object {
    std::vector<std::pair<std::string, std::string>> kv;  // value already rendered at its depth
    void add(const std::string& k, const std::string& v) { kv.emplace_back(k, v); }
    std::string dump(int depth) const {
        const std::string pad(static_cast<size_t>(2 * (depth + 1)), ' '), end(static_cast<size_t>(2 * depth), ' ');
        std::string o = "{\n";
        for (size_t i = 0; i < kv.size(); ++i)
            o += pad + quote(kv[i].first) + ": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
        return o + end + "}";
    }
};
}  // namespace json_detail

// report.hpp:63-81
inline std::string config_to_json(const SolverConfig& c, int depth = 0) {
    using namespace json_detail;
    Object j;
    j.add("p", std::to_string(c.p));
    j.add("alpha", number(c.alpha));
    j.add("gamma", number(c.gamma));
    j.add("beta", number(c.crossover.beta));
    j.add("phase1_iters", std::to_string(c.phase1_iters));
    j.add("phase2_iters", std::to_string(c.phase2_iters));
    j.add("variant", quote(variant_name(c.variant)));
    j.add("crossover", quote(crossover_name(c.crossover.mode)));
    j.add("matching", quote(matching_name(c.crossover.matching)));
    j.add("exclusion", quote(exclusion_name(c.crossover.exclusion)));
    j.add("seed", std::to_string(c.master_seed));
    j.add("workers", std::to_string(c.workers));
    j.add("time_limit", number(c.limits.time_seconds));
    j.add("iteration_limit", std::to_string(c.limits.total_iterations));
    j.add("generation_limit", std::to_string(c.limits.generations));
    return j.dump(depth);
}

// report.hpp:85-103, as printed by tools/plse.cpp:154 (`j.dump(2)`, without the trailing newline)
inline std::string result_to_json(const std::string& instance_name, int order, const RunResult& r,
                                  const SolverConfig& config, bool include_timing = false) {
    using namespace json_detail;
    Object j;
    j.add("instance", quote(instance_name));
    j.add("n", std::to_string(order));
    j.add("vertices", std::to_string(r.vertex_count));
    j.add("l", std::to_string(r.l));
    j.add("upper_bound", std::to_string(r.upper_bound));
    j.add("best_score", std::to_string(r.best_score));
    j.add("f", std::to_string(r.best_f));
    j.add("proven_optimal", r.proven_optimal ? "true" : "false");
    j.add("stop_reason", quote(r.stop_reason));
    j.add("generations", std::to_string(r.generations));
    j.add("total_iterations", std::to_string(r.total_iterations));
    if (include_timing) j.add("elapsed_seconds", number(r.elapsed_seconds));
    j.add("config", config_to_json(config, 1));
    return j.dump(0);
}

}  // namespace plse_b200
