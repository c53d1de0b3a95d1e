// plse_b200 -- the reference's command-line front-end (tools/plse.cpp) on the B200 device path.
//
// Subcommands, flags, output files, stdout / stderr lines and exit codes follow
// plse.cpp:26-315: generate (111-130), solve (132-174), verify (175-198) and
// bench (199-250, with the bench.hpp report: per-run rows CSV, class aggregates
// CSV, report JSON).  Everything goes through the C++ host API
// (include/plse_b200.hpp) and the C ABI; run() executes on one B200.  Extra
// device flags: --device N, --tie canon|ref (ref = the reference's own
// tie-break, bit-exact with the reference, both variants).
//
// The argument parser is a small stand-in for CLI11 (not available offline):
// same option names and value forms; usage errors exit 106 like CLI11's.
//
// Provenance: the flag-to-config glue (resolve_workers, make_config, warn_memory), the fixed output strings
// and the bench sweep loop deliberately follow tools/plse.cpp line for line (plse.cpp:69-113, 132-150,
// 176-190, 215-229) so that `solve --tie ref` prints the reference CLI's bytes; the CLI itself is outside
// the hot path and kept only as the reference-facing driver.  `python -m
// paper_2103_10453_b200` is a thin wrapper over this binary.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <map>
#include <mutex>
#include <random>
#include <set>
#include <sys/stat.h>
#include <dirent.h>
#include <thread>
#include <tuple>

#include "plse_b200.hpp"

using namespace plse_b200;

namespace {

struct CommonFlags {
    int p = 1024;
    double alpha = 0.6, gamma = 10.0, beta = 20.0;
    int64_t phase1_iters = 0, phase2_iters = 0;
    std::string variant = "mpma", crossover = "aux", matching = "nearest", exclusion = "run";
    double time_limit = 0;
    int64_t iter_limit = 0, gen_limit = 0;
    uint64_t seed = 0;
    bool seed_set = false;
    int workers = 0;
    bool paper_params = false;
    int device = 0;
    std::string tie = "canon";
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- a tiny CLI11 stand-in
struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::vector<std::string>> opt;  // name -> values (multi for sweeps)
    std::set<std::string> flags;
};

Args parse_args(int argc, char** argv, int first, const std::set<std::string>& flag_names,
                const std::set<std::string>& multi_names, const std::map<std::string, std::string>& aliases) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.size() > 1 && s[0] == '-' && !(s.size() > 1 && (std::isdigit((unsigned char)s[1]) || s[1] == '.'))) {
            std::string val;
            bool has_val = false;
            const size_t eq = s.find('=');
            if (s.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = s.substr(eq + 1);
                s = s.substr(0, eq);
                has_val = true;
            }
            auto al = aliases.find(s);
            if (al != aliases.end()) s = al->second;
            if (flag_names.count(s)) {
                a.flags.insert(s);
                continue;
            }
            if (multi_names.count(s)) {
                if (has_val) a.opt[s].push_back(val);
                while (i + 1 < argc && argv[i + 1][0] != '-') a.opt[s].push_back(argv[++i]);
                continue;
            }
            if (!has_val) {
                if (i + 1 >= argc) throw UsageError(s + " requires an argument");
                val = argv[++i];
            }
            a.opt[s] = {val};
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

template <class T>
T num(const std::string& s, const std::string& name) {
    try {
        size_t used = 0;
        T v;
        if constexpr (std::is_same_v<T, double>)
            v = std::stod(s, &used);
        else if constexpr (std::is_same_v<T, uint64_t>)
            v = std::stoull(s, &used);
        else
            v = static_cast<T>(std::stoll(s, &used));
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw UsageError("invalid value for " + name + ": " + s);
    }
}

const std::set<std::string> kSolverOpts = {"--pop", "--alpha", "--gamma", "--beta", "--phase1-iters",
                                           "--phase2-iters", "--variant", "--crossover", "--matching",
                                           "--exclusion", "--time-limit", "--iter-limit", "--gen-limit", "--seed",
                                           "--workers", "--device", "--tie"};

void read_solver_flags(const Args& a, CommonFlags& f) {
    auto get = [&](const char* k) -> const std::string* {
        auto it = a.opt.find(k);
        return it == a.opt.end() ? nullptr : &it->second.back();
    };
    if (auto* v = get("--pop")) f.p = num<int>(*v, "--pop");
    if (auto* v = get("--alpha")) f.alpha = num<double>(*v, "--alpha");
    if (auto* v = get("--gamma")) f.gamma = num<double>(*v, "--gamma");
    if (auto* v = get("--beta")) f.beta = num<double>(*v, "--beta");
    if (auto* v = get("--phase1-iters")) f.phase1_iters = num<int64_t>(*v, "--phase1-iters");
    if (auto* v = get("--phase2-iters")) f.phase2_iters = num<int64_t>(*v, "--phase2-iters");
    if (auto* v = get("--variant")) f.variant = *v;
    if (auto* v = get("--crossover")) f.crossover = *v;
    if (auto* v = get("--matching")) f.matching = *v;
    if (auto* v = get("--exclusion")) f.exclusion = *v;
    if (auto* v = get("--time-limit")) f.time_limit = num<double>(*v, "--time-limit");
    if (auto* v = get("--iter-limit")) f.iter_limit = num<int64_t>(*v, "--iter-limit");
    if (auto* v = get("--gen-limit")) f.gen_limit = num<int64_t>(*v, "--gen-limit");
    if (auto* v = get("--seed")) {
        f.seed = num<uint64_t>(*v, "--seed");
        f.seed_set = true;
    }
    if (auto* v = get("--workers")) f.workers = num<int>(*v, "--workers");
    if (auto* v = get("--device")) f.device = num<int>(*v, "--device");
    if (auto* v = get("--tie")) f.tie = *v;
    f.paper_params = a.flags.count("--paper-params") > 0;
}

// plse.cpp:69-75
uint64_t resolve_seed(CommonFlags& flags) {
    if (!flags.seed_set) {
        std::random_device entropy;
        flags.seed = (static_cast<uint64_t>(entropy()) << 32) ^ entropy();
    }
    return flags.seed;
}

// plse.cpp:77-84 (default_workers: parallel.hpp:13-16)
int resolve_workers(const CommonFlags& flags) {
    if (flags.workers > 0) return flags.workers;
    if (const char* env = std::getenv("PLSE_WORKERS")) {
        const int count = std::atoi(env);
        if (count > 0) return count;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

// plse.cpp:86-106
SolverConfig make_config(CommonFlags& flags) {
    SolverConfig config;
    config.p = flags.paper_params ? 12288 : flags.p;
    config.alpha = flags.alpha;
    config.gamma = flags.gamma;
    config.phase1_iters = flags.phase1_iters;
    config.phase2_iters = flags.phase2_iters;
    config.variant = parse_variant(flags.variant);
    config.crossover.mode = parse_crossover(flags.crossover);
    config.crossover.beta = flags.beta;
    config.crossover.matching = parse_matching(flags.matching);
    config.crossover.exclusion = parse_exclusion(flags.exclusion);
    config.limits.time_seconds = flags.time_limit;
    config.limits.total_iterations = flags.iter_limit;
    config.limits.generations = flags.gen_limit;
    config.master_seed = resolve_seed(flags);
    config.workers = resolve_workers(flags);
    config.device = flags.device;
    if (flags.tie != "canon" && flags.tie != "ref") throw std::invalid_argument("unknown tie mode: " + flags.tie);
    config.tie_mode = flags.tie == "ref" ? PLSE_TIE_REF : PLSE_TIE_CANON;
    config.validate();
    return config;
}

void warn_memory(const SolverConfig& config, int vertex_count) {
    const double bytes = 3.0 * config.p * config.p * 4 + 3.0 * config.p * vertex_count * 2;
    if (bytes > 2e9)
        std::cerr << "warning: p=" << config.p << " needs about " << static_cast<long long>(bytes / 1e6)
                  << " MB for distance blocks; consider a smaller --pop\n";
}

std::string basename_of(const std::string& path) {
    const size_t s = path.find_last_of('/');
    return s == std::string::npos ? path : path.substr(s + 1);
}

int cmd_generate(int n, double r, int count, CommonFlags& flags, const std::string& out_dir) {
    const uint64_t master = resolve_seed(flags);
    mkdir(out_dir.c_str(), 0777);
    const int r_tag = static_cast<int>(std::lround(100.0 * r));
    for (int id = 0; id < count; ++id) {
        const uint64_t seed = derive_seed(master, stream_tag::kInstanceGen, static_cast<uint64_t>(id));
        const PlsInstance instance = generate_instance(n, r, seed);
        const std::string path = out_dir + "/QC-" + std::to_string(n) + "-" + std::to_string(r_tag) + "-" +
                                 std::to_string(id) + ".txt";
        save_instance(instance, path);
        std::cout << path << " (" << instance.filled_count() << " filled)\n";
    }
    std::cerr << "seed " << master << '\n';
    return 0;
}

int cmd_solve(const std::string& instance_path, CommonFlags& flags, const std::string& json_path,
              const std::string& cert_path, bool log, bool timing) {
    const PlsInstance instance = load_instance(instance_path);
    SolverConfig config = make_config(flags);
    GenerationCallback callback;
    if (log) {
        callback = [](const GenerationStats& stats) {
            std::cerr << "gen " << stats.generation << " best_f " << stats.best_f << " mean_f " << stats.mean_f
                      << " mean_dist " << stats.mean_distance << " iters " << stats.iterations << " elapsed "
                      << stats.elapsed_seconds;
            if (stats.shortfall > 0) std::cerr << " shortfall " << stats.shortfall;
            std::cerr << '\n';
        };
    }
    {
        const ReducedGraph reduced = preprocess(instance);
        warn_memory(config, reduced.vertex_count());
    }
    const RunResult result = run(instance, config, callback);
    const std::string j = result_to_json(basename_of(instance_path), instance.order(), result, config, timing);
    if (json_path.empty()) {
        std::cout << j << '\n';
    } else {
        std::ofstream out(json_path);
        out << j << '\n';
    }
    if (!cert_path.empty()) {
        const ReducedGraph reduced = preprocess(instance);
        save_instance(to_grid(instance, reduced, result.best_solution), cert_path);
    }
    std::cerr << "score " << result.best_score << '/' << result.upper_bound
              << (result.proven_optimal ? " (optimal)" : "") << " in " << result.elapsed_seconds << "s, "
              << result.total_iterations << " iterations, seed " << config.master_seed << '\n';
    return result.proven_optimal ? 0 : 2;
}

int cmd_verify(const std::string& instance_path, const std::string& cert_path, bool exact, int64_t node_budget) {
    const PlsInstance instance = load_instance(instance_path);
    const PlsInstance certificate = load_instance(cert_path);
    const VerifyReport report = verify_certificate(instance, certificate);
    if (!report.legal) {
        std::cout << "illegal certificate:\n";
        for (const std::string& problem : report.problems) std::cout << "  " << problem << '\n';
        return 1;
    }
    std::cout << "legal, score " << report.score << '\n';
    const ReducedGraph reduced = preprocess(instance);
    const InstanceBounds bounds = compute_bounds(reduced);
    std::cout << "upper bound " << bounds.upper_bound << " (l = " << bounds.l << ")\n";
    if (exact) {
        const OracleResult oracle = solve_exact(reduced, node_budget);
        const int optimum = instance.order() * instance.order() - reduced.l() - oracle.optimum_f;
        std::cout << "exact optimum " << optimum << (oracle.exact ? "" : " (budget exhausted)") << ", gap "
                  << optimum - report.score << '\n';
    }
    return 0;
}

// ---------------------------------------------------------------- bench.hpp
struct BenchRow {
    std::string instance, id, crossover, matching, variant;
    int n = 0, r_percent = 0, repeat = 0, p = 0, score = 0, f = 0, upper_bound = 0;
    uint64_t seed = 0;
    bool proven_optimal = false;
    int64_t generations = 0, iterations = 0;
    double elapsed_seconds = 0;
};
struct BenchAggregate {
    int n = 0, r_percent = 0, p = 0, instances = 0, runs = 0;
    std::string crossover, matching, variant;
    double f_best_mean = 0, f_avg_mean = 0, optimal_rate = 0, time_mean = 0;
};
struct BenchTask {
    std::string path, stem;
    int instance_index = 0;
};

// bench.hpp:64-81
void parse_instance_name(const std::string& stem, const PlsInstance& instance, int& n, int& r_percent,
                         std::string& id) {
    n = instance.order();
    r_percent = static_cast<int>(std::lround(100.0 * instance.fill_ratio()));
    id = stem;
    if (stem.rfind("QC-", 0) == 0) {
        std::istringstream in(stem.substr(3));
        int pn = 0, pr = 0;
        char dash1 = 0, dash2 = 0;
        std::string pid;
        if (in >> pn >> dash1 >> pr >> dash2 && dash1 == '-' && dash2 == '-' && std::getline(in, pid) &&
            !pid.empty() && pn == instance.order()) {
            r_percent = pr;
            id = pid;
        }
    }
}

// bench.hpp:83-118
std::vector<BenchAggregate> compute_aggregates(const std::vector<BenchRow>& rows) {
    std::map<std::tuple<int, int, std::string, std::string, std::string, int>,
             std::map<std::string, std::vector<const BenchRow*>>>
        classes;
    for (const BenchRow& row : rows)
        classes[{row.n, row.r_percent, row.crossover, row.matching, row.variant, row.p}][row.instance].push_back(&row);
    std::vector<BenchAggregate> out;
    for (const auto& [key, instances] : classes) {
        BenchAggregate agg;
        std::tie(agg.n, agg.r_percent, agg.crossover, agg.matching, agg.variant, agg.p) = key;
        agg.instances = static_cast<int>(instances.size());
        double best_sum = 0, score_sum = 0, time_sum = 0;
        int optimal = 0, runs = 0;
        for (const auto& [name, rs] : instances) {
            int best = 0;
            for (const BenchRow* row : rs) {
                best = std::max(best, row->score);
                score_sum += row->score;
                time_sum += row->elapsed_seconds;
                optimal += row->proven_optimal;
                ++runs;
            }
            best_sum += best;
        }
        agg.runs = runs;
        agg.f_best_mean = best_sum / agg.instances;
        agg.f_avg_mean = score_sum / runs;
        agg.optimal_rate = static_cast<double>(optimal) / runs;
        agg.time_mean = time_sum / runs;
        out.push_back(agg);
    }
    return out;
}

void write_rows_csv(const std::vector<BenchRow>& rows, std::ostream& out) {
    out << "instance,n,r,id,repeat,seed,p,crossover,matching,variant,score,f,upper_bound,"
           "proven_optimal,generations,iterations,elapsed_seconds\n";
    for (const BenchRow& r : rows)
        out << r.instance << ',' << r.n << ',' << r.r_percent << ',' << r.id << ',' << r.repeat << ',' << r.seed
            << ',' << r.p << ',' << r.crossover << ',' << r.matching << ',' << r.variant << ',' << r.score << ','
            << r.f << ',' << r.upper_bound << ',' << (r.proven_optimal ? 1 : 0) << ',' << r.generations << ','
            << r.iterations << ',' << r.elapsed_seconds << '\n';
}

void write_aggregates_csv(const std::vector<BenchAggregate>& aggs, std::ostream& out) {
    out << "n,r,crossover,matching,variant,p,instances,runs,f_best_mean,f_avg_mean,optimal_rate,time_mean\n";
    for (const BenchAggregate& a : aggs)
        out << a.n << ',' << a.r_percent << ',' << a.crossover << ',' << a.matching << ',' << a.variant << ','
            << a.p << ',' << a.instances << ',' << a.runs << ',' << a.f_best_mean << ',' << a.f_avg_mean << ','
            << a.optimal_rate << ',' << a.time_mean << '\n';
}

// bench.hpp:145-185 report_to_json(...).dump(2)
std::string report_to_json(const std::vector<BenchRow>& rows, const std::vector<BenchAggregate>& aggs) {
    using namespace json_detail;
    auto arr = [](const std::vector<std::string>& items) {
        if (items.empty()) return std::string("[]");
        std::string o = "[\n";
        for (size_t i = 0; i < items.size(); ++i) o += "    " + items[i] + (i + 1 < items.size() ? ",\n" : "\n");
        return o + "  ]";
    };
    std::vector<std::string> rs, as;
    for (const BenchRow& r : rows) {
        Object j;
        j.add("instance", quote(r.instance));
        j.add("n", std::to_string(r.n));
        j.add("r", std::to_string(r.r_percent));
        j.add("id", quote(r.id));
        j.add("repeat", std::to_string(r.repeat));
        j.add("seed", std::to_string(r.seed));
        j.add("p", std::to_string(r.p));
        j.add("crossover", quote(r.crossover));
        j.add("matching", quote(r.matching));
        j.add("variant", quote(r.variant));
        j.add("score", std::to_string(r.score));
        j.add("f", std::to_string(r.f));
        j.add("upper_bound", std::to_string(r.upper_bound));
        j.add("proven_optimal", r.proven_optimal ? "true" : "false");
        j.add("generations", std::to_string(r.generations));
        j.add("iterations", std::to_string(r.iterations));
        j.add("elapsed_seconds", number(r.elapsed_seconds));
        rs.push_back(j.dump(2));
    }
    for (const BenchAggregate& a : aggs) {
        Object j;
        j.add("n", std::to_string(a.n));
        j.add("r", std::to_string(a.r_percent));
        j.add("crossover", quote(a.crossover));
        j.add("matching", quote(a.matching));
        j.add("variant", quote(a.variant));
        j.add("p", std::to_string(a.p));
        j.add("instances", std::to_string(a.instances));
        j.add("runs", std::to_string(a.runs));
        j.add("f_best_mean", number(a.f_best_mean));
        j.add("f_avg_mean", number(a.f_avg_mean));
        j.add("optimal_rate", number(a.optimal_rate));
        j.add("time_mean", number(a.time_mean));
        as.push_back(j.dump(2));
    }
    return "{\n  \"rows\": " + arr(rs) + ",\n  \"aggregates\": " + arr(as) + "\n}";
}

int cmd_bench(const std::string& suite_dir, CommonFlags& flags, int repeats, const std::string& csv_path,
              const std::string& json_path, const std::vector<std::string>& crossovers,
              const std::vector<std::string>& matchings, const std::vector<int>& pops, int jobs) {
    std::vector<std::string> files;
    if (DIR* d = opendir(suite_dir.c_str())) {
        while (dirent* e = readdir(d)) {
            const std::string name = e->d_name, path = suite_dir + "/" + name;
            struct stat st;
            if (name.size() > 4 && name.compare(name.size() - 4, 4, ".txt") == 0 && stat(path.c_str(), &st) == 0 &&
                S_ISREG(st.st_mode))
                files.push_back(path);
        }
        closedir(d);
    }
    std::sort(files.begin(), files.end());
    std::vector<BenchTask> tasks;
    for (const std::string& f : files) {
        const std::string b = basename_of(f);
        tasks.push_back({f, b.substr(0, b.size() - 4), static_cast<int>(tasks.size())});
    }
    if (tasks.empty()) {
        std::cerr << "error: no .txt instances under " << suite_dir << '\n';
        return 1;
    }
    const SolverConfig base = make_config(flags);
    std::vector<SolverConfig> sweep;
    const auto cross_list = crossovers.empty() ? std::vector<std::string>{flags.crossover} : crossovers;
    const auto match_list = matchings.empty() ? std::vector<std::string>{flags.matching} : matchings;
    const auto pop_list = pops.empty() ? std::vector<int>{base.p} : pops;
    for (const std::string& cross : cross_list)
        for (const std::string& match : match_list)
            for (int p : pop_list) {
                SolverConfig config = base;
                config.crossover.mode = parse_crossover(cross);
                config.crossover.matching = parse_matching(match);
                config.p = p;
                config.validate();
                sweep.push_back(config);
            }
    // bench.hpp:196-250: seeds from (master, instance index, sweep index, repeat)
    struct Spec {
        const BenchTask* task;
        int s, rep;
    };
    std::vector<Spec> specs;
    for (const BenchTask& t : tasks)
        for (int s = 0; s < static_cast<int>(sweep.size()); ++s)
            for (int rep = 0; rep < repeats; ++rep) specs.push_back({&t, s, rep});
    std::vector<BenchRow> rows(specs.size());
    std::mutex mu;
    std::vector<std::exception_ptr> errs;
    auto one = [&](size_t k, int device) {
        const Spec& sp = specs[k];
        const PlsInstance instance = load_instance(sp.task->path);
        SolverConfig config = sweep[static_cast<size_t>(sp.s)];
        config.device = device;
        config.master_seed = derive_seed(
            base.master_seed, stream_tag::kBench,
            (static_cast<uint64_t>(sp.task->instance_index) * sweep.size() + sp.s) * static_cast<uint64_t>(repeats) +
                static_cast<uint64_t>(sp.rep));
        const RunResult result = run(instance, config);
        BenchRow row;
        row.instance = sp.task->stem;
        parse_instance_name(sp.task->stem, instance, row.n, row.r_percent, row.id);
        row.repeat = sp.rep;
        row.seed = config.master_seed;
        row.p = config.p;
        row.crossover = crossover_name(config.crossover.mode);
        row.matching = matching_name(config.crossover.matching);
        row.variant = variant_name(config.variant);
        row.score = result.best_score;
        row.f = result.best_f;
        row.upper_bound = result.upper_bound;
        row.proven_optimal = result.proven_optimal;
        row.generations = result.generations;
        row.iterations = result.total_iterations;
        row.elapsed_seconds = result.elapsed_seconds;
        rows[k] = row;
        std::lock_guard<std::mutex> lock(mu);
        std::cerr << row.instance << " repeat " << row.repeat << " score " << row.score << '/' << row.upper_bound
                  << (row.proven_optimal ? " optimal" : "") << '\n';
    };
    // --jobs: concurrent runs spread over the visible devices (one host thread each)
    const int ndev = std::max(1, std::atoi(std::getenv("PLSE_BENCH_DEVICES") ? std::getenv("PLSE_BENCH_DEVICES") : "1"));
    if (jobs <= 1) {
        for (size_t k = 0; k < specs.size(); ++k) one(k, base.device);
    } else {
        size_t next = 0;
        std::vector<std::thread> th;
        for (int w = 0; w < jobs; ++w)
            th.emplace_back([&, w] {
                for (;;) {
                    size_t k;
                    {
                        std::lock_guard<std::mutex> lock(mu);
                        if (next >= specs.size() || !errs.empty()) return;
                        k = next++;
                    }
                    try {
                        one(k, (base.device + w) % ndev);
                    } catch (...) {
                        std::lock_guard<std::mutex> lock(mu);
                        errs.push_back(std::current_exception());
                        return;
                    }
                }
            });
        for (auto& t : th) t.join();
        if (!errs.empty()) std::rethrow_exception(errs.front());
    }
    const std::vector<BenchAggregate> aggs = compute_aggregates(rows);
    if (!csv_path.empty()) {
        std::ofstream out(csv_path);
        write_rows_csv(rows, out);
        std::cerr << "rows -> " << csv_path << '\n';
    } else {
        write_rows_csv(rows, std::cout);
    }
    if (!json_path.empty()) {
        std::ofstream out(json_path);
        out << report_to_json(rows, aggs) << '\n';
        std::cerr << "report -> " << json_path << '\n';
    }
    std::ostringstream agg;
    write_aggregates_csv(aggs, agg);
    std::cerr << agg.str();
    return 0;
}

int usage() {
    std::cerr << "partial Latin square extension solver (B200 device path)\n"
                 "usage: plse_b200 {generate,solve,verify,bench} ...\n"
                 "  generate -n N -r R [-c COUNT] [-o DIR] [--seed S]\n"
                 "  solve INSTANCE [--json F] [--cert F] [--log] [--timing] [solver flags]\n"
                 "  verify INSTANCE CERTIFICATE [--exact] [--node-budget N]\n"
                 "  bench SUITE [--repeats K] [--csv F] [--json F] [--sweep-crossover ..] [--sweep-matching ..]\n"
                 "        [--sweep-pop ..] [--jobs J] [solver flags]\n"
                 "solver flags: -p/--pop --alpha --gamma --beta --phase1-iters --phase2-iters --variant mpma|partial\n"
                 "  --crossover aux|ux|none --matching nearest|random --exclusion run|generation|off --time-limit\n"
                 "  --iter-limit --gen-limit --seed --workers --paper-params --device --tie canon|ref\n";
    return 106;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "generate") {
            const Args a = parse_args(argc, argv, 2, {}, {}, {{"-n", "--order"}, {"-r", "--ratio"}, {"-c", "--count"},
                                                            {"-o", "--out-dir"}});
            if (!a.opt.count("--order") || !a.opt.count("--ratio")) throw UsageError("--order and --ratio are required");
            CommonFlags f;
            if (a.opt.count("--seed")) {
                f.seed = num<uint64_t>(a.opt.at("--seed").back(), "--seed");
                f.seed_set = true;
            }
            const int n = num<int>(a.opt.at("--order").back(), "--order");
            const double r = num<double>(a.opt.at("--ratio").back(), "--ratio");
            const int count = a.opt.count("--count") ? num<int>(a.opt.at("--count").back(), "--count") : 1;
            const std::string dir = a.opt.count("--out-dir") ? a.opt.at("--out-dir").back() : ".";
            return cmd_generate(n, r, count, f, dir);
        }
        if (cmd == "solve") {
            const Args a = parse_args(argc, argv, 2, {"--log", "--timing", "--paper-params"}, {}, {{"-p", "--pop"}});
            if (a.pos.size() != 1) throw UsageError("solve takes exactly one instance file");
            CommonFlags f;
            read_solver_flags(a, f);
            const std::string json = a.opt.count("--json") ? a.opt.at("--json").back() : "";
            const std::string cert = a.opt.count("--cert") ? a.opt.at("--cert").back() : "";
            return cmd_solve(a.pos[0], f, json, cert, a.flags.count("--log") > 0, a.flags.count("--timing") > 0);
        }
        if (cmd == "verify") {
            const Args a = parse_args(argc, argv, 2, {"--exact"}, {}, {});
            if (a.pos.size() != 2) throw UsageError("verify takes an instance and a certificate");
            const int64_t budget =
                a.opt.count("--node-budget") ? num<int64_t>(a.opt.at("--node-budget").back(), "--node-budget")
                                             : 50'000'000;
            return cmd_verify(a.pos[0], a.pos[1], a.flags.count("--exact") > 0, budget);
        }
        if (cmd == "bench") {
            const Args a = parse_args(argc, argv, 2, {"--paper-params"},
                                      {"--sweep-crossover", "--sweep-matching", "--sweep-pop"}, {{"-p", "--pop"}});
            if (a.pos.size() != 1) throw UsageError("bench takes one suite directory");
            CommonFlags f;
            read_solver_flags(a, f);
            const int repeats = a.opt.count("--repeats") ? num<int>(a.opt.at("--repeats").back(), "--repeats") : 5;
            const int jobs = a.opt.count("--jobs") ? num<int>(a.opt.at("--jobs").back(), "--jobs") : 1;
            std::vector<int> pops;
            if (a.opt.count("--sweep-pop"))
                for (const auto& x : a.opt.at("--sweep-pop")) pops.push_back(num<int>(x, "--sweep-pop"));
            auto list = [&](const char* k) {
                return a.opt.count(k) ? a.opt.at(k) : std::vector<std::string>{};
            };
            return cmd_bench(a.pos[0], f, repeats, a.opt.count("--csv") ? a.opt.at("--csv").back() : "",
                             a.opt.count("--json") ? a.opt.at("--json").back() : "", list("--sweep-crossover"),
                             list("--sweep-matching"), pops, jobs);
        }
        return usage();
    } catch (const UsageError& e) {
        std::cerr << e.what() << '\n';
        return usage();
    } catch (const std::exception& error) {
        std::cerr << "error: " << error.what() << '\n';
        return 1;
    }
}
