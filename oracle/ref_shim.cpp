// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY.  Compiled by oracle/Makefile with
// -I/root/reference/proj/include -I/root/reference/proj/tests straight from
// the read-only reference tree; the output goes to oracle/_ref/ (git-ignored).
// No reference source is copied into this repository: this file only calls
// the reference's public functions (cited per entry point) so that tests can
// pin the C oracle and bench.py can time the reference's own CPU path.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "plse/engine.hpp"
#include "plse/plits.hpp"
#if __has_include(<json.hpp>)
#include "plse/bench.hpp"
#include "plse/report.hpp"
#define PLSE_REF_HAVE_JSON 1
#endif
#include <dirent.h>
#include <sys/stat.h>

#include <sstream>
#include "plse/verify.hpp"
#include "plse/oracle.hpp"
#include "support/builders.hpp"

using namespace plse;

struct ref_graph {
    ReducedGraph g;
};

struct ref_excl {
    MatchingExclusion e;
};

static Coloring make(const ReducedGraph& g, const uint16_t* c) {
    Coloring s(g);
    s.assign(std::vector<Color>(c, c + g.vertex_count()));
    return s;
}

extern "C" {

// instance.hpp:204 generate_instance
int ref_generate_instance(int n, double r, uint64_t seed, uint16_t* grid) {
    try {
        PlsInstance inst = generate_instance(n, r, seed);
        std::memcpy(grid, inst.cells().data(), sizeof(uint16_t) * n * n);
        return 0;
    } catch (...) {
        return -1;
    }
}

// tests/support/builders.hpp:46 lsc_instance
void ref_lsc_instance(int n, double r, uint64_t seed, uint16_t* grid) {
    PlsInstance inst = builders::lsc_instance(n, r, seed);
    std::memcpy(grid, inst.cells().data(), sizeof(uint16_t) * n * n);
}

static PlsInstance grid_instance(int n, const uint16_t* grid) {
    PlsInstance inst(n);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) inst.set(a, b, grid[a * n + b]);
    return inst;
}

// lsgraph.hpp:115 preprocess(build_graph(...))
ref_graph* ref_preprocess(int n, const uint16_t* grid) {
    auto* h = new ref_graph;
    h->g = preprocess(build_graph(grid_instance(n, grid)));
    return h;
}
void ref_graph_free(ref_graph* h) { delete h; }
int ref_graph_nv(const ref_graph* h) { return h->g.vertex_count(); }
int ref_graph_l(const ref_graph* h) { return h->g.l; }
int ref_graph_adj_len(const ref_graph* h) { return (int)h->g.adj.size(); }
int ref_graph_dom_len(const ref_graph* h) { return (int)h->g.dom.size(); }
void ref_graph_export(const ref_graph* h, int32_t* cell_row, int32_t* cell_col, int32_t* adj_off,
                      int32_t* adj, int32_t* dom_off, uint16_t* dom) {
    const ReducedGraph& g = h->g;
    const int nv = g.vertex_count();
    for (int v = 0; v < nv; ++v) {
        if (cell_row) cell_row[v] = g.cells[v].row;
        if (cell_col) cell_col[v] = g.cells[v].col;
    }
    if (adj_off) std::memcpy(adj_off, g.adj_offsets.data(), sizeof(int32_t) * (nv + 1));
    if (adj) std::memcpy(adj, g.adj.data(), sizeof(int32_t) * g.adj.size());
    if (dom_off) std::memcpy(dom_off, g.dom_offsets.data(), sizeof(int32_t) * (nv + 1));
    if (dom) std::memcpy(dom, g.dom.data(), sizeof(uint16_t) * g.dom.size());
}

// coloring.hpp:59-73
void ref_eval(const ref_graph* h, const uint16_t* colors, int* f, int* c) {
    Coloring s = make(h->g, colors);
    *f = s.f();
    *c = s.c();
}

// coloring.hpp:105 ConflictTable::build
void ref_gamma_build(const ref_graph* h, const uint16_t* colors, int32_t* gamma) {
    ConflictTable t;
    t.build(make(h->g, colors));
    std::memcpy(gamma, t.gamma.data(), sizeof(int32_t) * t.gamma.size());
}

// partial.hpp:41 repair(Coloring)
void ref_repair(const ref_graph* h, uint16_t* colors) {
    Coloring out = repair(make(h->g, colors));
    std::memcpy(colors, out.colors().data(), sizeof(uint16_t) * h->g.vertex_count());
}

// partial.hpp:156 partial_mpma_improve with Rng(stream_seed)
int64_t ref_improve(const ref_graph* h, const uint16_t* input, uint16_t* out_best, uint64_t stream_seed,
                    int64_t budget, double alpha, int stop_f, int* best_f) {
    PartialColScratch scratch;
    Rng rng(stream_seed);
    SearchStats st;
    Coloring out = partial_mpma_improve(scratch, make(h->g, input), rng, budget, &st, alpha, stop_f);
    std::memcpy(out_best, out.colors().data(), sizeof(uint16_t) * h->g.vertex_count());
    if (best_f) *best_f = out.f();
    return st.iterations;
}

// partial.hpp:76-143: drive PartialColSearch step by step and record the
// current colouring after every step (nv*steps uint16) plus best f per step.
int64_t ref_improve_states(const ref_graph* h, const uint16_t* input, uint64_t stream_seed, int64_t steps,
                           double alpha, uint16_t* repaired, uint16_t* states, int32_t* best_f) {
    PartialColScratch scratch;
    Rng rng(stream_seed);
    Coloring cur = make(h->g, input);
    PartialColSearch search(scratch, cur, rng, alpha);
    const int nv = h->g.vertex_count();
    std::memcpy(repaired, search.current().colors().data(), sizeof(uint16_t) * nv);
    int64_t t = 0;
    for (; t < steps; ++t) {
        if (!search.step()) break;
        std::memcpy(states + (size_t)t * nv, search.current().colors().data(), sizeof(uint16_t) * nv);
        best_f[t] = search.best().f();
    }
    return t;
}

// plits.hpp:276 plits_run(scratch, input, Rng(stream_seed), params, &stats).  A scratch is
// reused across calls on the same thread, as engine.hpp:176 does per worker.
int64_t ref_plits(const ref_graph* h, const uint16_t* input, uint16_t* out, uint64_t stream_seed, int64_t iters1,
                  int64_t iters2, double alpha, int stop_f) {
    thread_local PlitsScratch scratch;
    Rng rng(stream_seed);
    PlitsParams params;
    params.phase1_iters = iters1;
    params.phase2_iters = iters2;
    params.alpha = alpha;
    params.stop_f = stop_f;
    SearchStats stats;
    Coloring res = plits_run(scratch, make(h->g, input), rng, params, &stats);
    std::memcpy(out, res.colors().data(), sizeof(uint16_t) * h->g.vertex_count());
    return stats.iterations;
}

// plits_run's two phases (plits.hpp:255-292) driven step by step through
// PlitsSearch::step(&applied), recording every step: (phase, v, to, df, dc,
// current f, c, best_scaled).  Returns the number of steps recorded.
int64_t ref_plits_trace(const ref_graph* h, const uint16_t* input, uint64_t stream_seed, int64_t iters1,
                        int64_t iters2, double alpha, int stop_f, int32_t* rec /* 7 per step */,
                        int64_t* best_scaled, int64_t cap, uint16_t* out) {
    const int nv = h->g.vertex_count();
    PlitsScratch scratch;
    Rng rng(stream_seed);
    Coloring col = make(h->g, input);
    if (iters1 <= 0) iters1 = phase1_default(nv);
    if (iters2 <= 0) iters2 = phase2_default(nv);
    int64_t n = 0;
    auto phase = [&](int ph, PhaseWeights w, int64_t budget) {
        PlitsSearch search(scratch, col, w, rng, alpha);
        int64_t it = 0;
        bool hit = false;
        while (it < budget) {
            if (search.best().legal() && search.best().f() <= stop_f) {
                hit = true;
                break;
            }
            CandidateMove m;
            const StepResult r = search.step(&m);
            if (r == StepResult::Exhausted) break;
            if (n < cap) {
                int32_t* q = rec + 7 * n;
                q[0] = ph;
                q[1] = r == StepResult::Moved ? m.v : -1;
                q[2] = r == StepResult::Moved ? m.to : 0;
                q[3] = r == StepResult::Moved ? m.df : 0;
                q[4] = r == StepResult::Moved ? m.dc : 0;
                q[5] = search.current().f();
                q[6] = search.current().c();
                best_scaled[n] = search.best_scaled();
            }
            ++n;
            ++it;
        }
        hit = hit || (search.best().legal() && search.best().f() <= stop_f);
        col = search.best();
        return hit;
    };
    if (!phase(1, PhaseWeights::from_phi(0.5), iters1)) phase(2, PhaseWeights::from_phi((double)nv), iters2);
    if (!col.legal()) col = repair(std::move(col));
    std::memcpy(out, col.colors().data(), sizeof(uint16_t) * nv);
    return n;
}

// population.hpp:41 compute_cross_distances
void ref_cross_distances(const ref_graph* h, int p, const uint16_t* members, const uint16_t* improved,
                         int32_t* cross, int32_t* fresh) {
    const int nv = h->g.vertex_count();
    std::vector<Coloring> a, b;
    for (int i = 0; i < p; ++i) {
        a.push_back(make(h->g, members + (size_t)i * nv));
        b.push_back(make(h->g, improved + (size_t)i * nv));
    }
    DistanceBlocks blocks = compute_cross_distances(a, b, 1);
    std::memcpy(cross, blocks.cross.data.data(), sizeof(int32_t) * p * p);
    std::memcpy(fresh, blocks.fresh.data.data(), sizeof(int32_t) * p * p);
}

// population.hpp:103 update_population (members/dist in-out)
void ref_update(const ref_graph* h, int p, double gamma, uint16_t* members, int32_t* dist,
                const uint16_t* improved, const int32_t* cross, const int32_t* fresh, int32_t* pool_best_f,
                int32_t* shortfall_slots, int32_t* n_shortfall) {
    const int nv = h->g.vertex_count();
    Population pop;
    pop.spacing_gamma = gamma;
    std::vector<Coloring> imp;
    for (int i = 0; i < p; ++i) {
        pop.members.push_back(make(h->g, members + (size_t)i * nv));
        imp.push_back(make(h->g, improved + (size_t)i * nv));
    }
    pop.dist.resize(p, p);
    std::memcpy(pop.dist.data.data(), dist, sizeof(int32_t) * p * p);
    DistanceBlocks blocks;
    blocks.cross.resize(p, p);
    blocks.fresh.resize(p, p);
    std::memcpy(blocks.cross.data.data(), cross, sizeof(int32_t) * p * p);
    std::memcpy(blocks.fresh.data.data(), fresh, sizeof(int32_t) * p * p);
    UpdateInfo info = update_population(pop, std::move(imp), blocks);
    for (int i = 0; i < p; ++i)
        std::memcpy(members + (size_t)i * nv, pop.members[i].colors().data(), sizeof(uint16_t) * nv);
    std::memcpy(dist, pop.dist.data.data(), sizeof(int32_t) * p * p);
    *pool_best_f = info.pool_best_f;
    *n_shortfall = (int32_t)info.shortfall_slots.size();
    for (size_t k = 0; k < info.shortfall_slots.size(); ++k) shortfall_slots[k] = info.shortfall_slots[k];
}

ref_excl* ref_excl_new(int p) {
    auto* e = new ref_excl;
    e->e.reset(p);
    return e;
}
void ref_excl_free(ref_excl* e) { delete e; }
void ref_excl_reset(ref_excl* e, int p) { e->e.reset(p); }

// crossover.hpp:54 build_offspring
void ref_offspring(const ref_graph* h, int p, const uint16_t* members, const int32_t* dist, int crossover,
                   double beta, int matching, int exclusion, ref_excl* ex, uint64_t master_seed,
                   uint64_t generation, uint16_t* offspring) {
    const int nv = h->g.vertex_count();
    Population pop;
    for (int i = 0; i < p; ++i) pop.members.push_back(make(h->g, members + (size_t)i * nv));
    pop.dist.resize(p, p);
    std::memcpy(pop.dist.data.data(), dist, sizeof(int32_t) * p * p);
    CrossoverConfig cc;
    cc.mode = crossover == 0 ? CrossoverMode::AUX : crossover == 1 ? CrossoverMode::UX : CrossoverMode::None;
    cc.beta = beta;
    cc.matching = matching == 0 ? MatchingStrategy::NearestNeighbor : MatchingStrategy::Random;
    cc.exclusion = exclusion == 0 ? ExclusionScope::Run : exclusion == 1 ? ExclusionScope::Generation : ExclusionScope::Off;
    std::vector<Coloring> off = build_offspring(pop, cc, ex->e, master_seed, generation, 1);
    for (int i = 0; i < p; ++i)
        std::memcpy(offspring + (size_t)i * nv, off[i].colors().data(), sizeof(uint16_t) * nv);
}

// engine.hpp:88 initialize_population (members + full distance matrix)
void ref_init_population(const ref_graph* h, int p, uint64_t master_seed, uint16_t* members, int32_t* dist) {
    SolverConfig cfg;
    cfg.p = p;
    cfg.master_seed = master_seed;
    cfg.workers = 1;
    Population pop = initialize_population(h->g, cfg);
    const int nv = h->g.vertex_count();
    for (int i = 0; i < p; ++i)
        std::memcpy(members + (size_t)i * nv, pop.members[i].colors().data(), sizeof(uint16_t) * nv);
    if (dist) std::memcpy(dist, pop.dist.data.data(), sizeof(int32_t) * p * p);
}

// oracle.hpp:134 solve_exact / 141 enumerate_exact with node counts and certificates
int ref_solve_exact_full(const ref_graph* h, int64_t budget, int enumerate, int* exact, int64_t* nodes,
                         uint16_t* cert) {
    OracleResult r = enumerate ? enumerate_exact(h->g) : solve_exact(h->g, budget);
    if (exact) *exact = r.exact ? 1 : 0;
    if (nodes) *nodes = r.nodes;
    if (cert) std::memcpy(cert, r.certificate.colors().data(), sizeof(uint16_t) * h->g.vertex_count());
    return r.optimum_f;
}

// oracle.hpp:134 solve_exact
int ref_solve_exact(const ref_graph* h, int* exact) {
    OracleResult r = solve_exact(h->g);
    if (exact) *exact = r.exact ? 1 : 0;
    return r.optimum_f;
}

// GenerationStats capture for the next ref_run (engine.hpp:49-57)
struct ref_gen_log {
    int64_t generation;
    int32_t best_f, shortfall;
    int64_t iterations;
    double mean_f, mean_distance;
};
static ref_gen_log* g_log = nullptr;
static int64_t g_log_cap = 0, g_log_n = 0;

void ref_set_log(ref_gen_log* log, int64_t cap) {
    g_log = log;
    g_log_cap = cap;
    g_log_n = 0;
}
int64_t ref_log_count(void) { return g_log_n; }

struct ref_run_result {
    int32_t best_f, best_score, proven_optimal, stop_reason, l, upper_bound, vertex_count;
    int64_t generations, total_iterations;
    double elapsed_seconds;
    double first_best_seconds;  // elapsed when best_f first reached its final value
};

// engine.hpp:114 run(), Partial-MPMA or MPMA, optional limits
int ref_run(int n, const uint16_t* grid, int p, double alpha, double gamma, double beta, int64_t phase1,
            int64_t phase2, int variant, int crossover, int matching, int exclusion, uint64_t seed, int workers,
            double time_limit, int64_t iteration_limit, int64_t generation_limit, ref_run_result* out,
            uint16_t* best_colors) {
    SolverConfig cfg;
    cfg.p = p;
    cfg.alpha = alpha;
    cfg.gamma = gamma;
    cfg.crossover.beta = beta;
    cfg.phase1_iters = phase1;
    cfg.phase2_iters = phase2;
    cfg.variant = variant == 1 ? Variant::PartialMPMA : Variant::MPMA;
    cfg.crossover.mode = crossover == 0 ? CrossoverMode::AUX : crossover == 1 ? CrossoverMode::UX : CrossoverMode::None;
    cfg.crossover.matching = matching == 0 ? MatchingStrategy::NearestNeighbor : MatchingStrategy::Random;
    cfg.crossover.exclusion =
        exclusion == 0 ? ExclusionScope::Run : exclusion == 1 ? ExclusionScope::Generation : ExclusionScope::Off;
    cfg.master_seed = seed;
    cfg.workers = workers > 0 ? workers : default_workers();
    cfg.limits.time_seconds = time_limit;
    cfg.limits.total_iterations = iteration_limit;
    cfg.limits.generations = generation_limit;
    int last_best = -1;
    double first_at = 0;
    RunResult r = run(grid_instance(n, grid), cfg, [&](const GenerationStats& s) {
        if (g_log && g_log_n < g_log_cap)
            g_log[g_log_n++] = {s.generation, s.best_f, s.shortfall, s.iterations, s.mean_f, s.mean_distance};
        if (s.best_f != last_best) {
            last_best = s.best_f;
            first_at = s.elapsed_seconds;
        }
    });
    out->best_f = r.best_f;
    out->best_score = r.best_score;
    out->proven_optimal = r.proven_optimal;
    out->stop_reason = r.stop_reason == "optimal" ? 0 : r.stop_reason == "time_limit" ? 1
                       : r.stop_reason == "iteration_limit" ? 2 : r.stop_reason == "generation_limit" ? 3 : 4;
    out->l = r.l;
    out->upper_bound = r.upper_bound;
    out->vertex_count = r.vertex_count;
    out->generations = r.generations;
    out->total_iterations = r.total_iterations;
    out->elapsed_seconds = r.elapsed_seconds;
    out->first_best_seconds = (last_best == r.best_f) ? first_at : r.elapsed_seconds;
    if (best_colors && r.best_solution.size() == r.vertex_count)
        std::memcpy(best_colors, r.best_solution.colors().data(), sizeof(uint16_t) * r.vertex_count);
    return 0;
}

// engine.hpp:184-206: the reference's own improve phase (parallel_for over
// `workers` threads, per-worker scratch, stream (seed, 2, gen*p+i)).  Returns
// total iterations; *seconds receives the phase wall time.
int64_t ref_improve_phase(const ref_graph* h, int p, const uint16_t* offspring, uint16_t* improved,
                          uint64_t master_seed, uint64_t generation, int64_t budget, double alpha, int stop_f,
                          int workers, double* seconds) {
    const int nv = h->g.vertex_count();
    if (workers <= 0) workers = default_workers();
    std::vector<PartialColScratch> scratch((size_t)workers);
    std::vector<int64_t> iters((size_t)p, 0);
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t chunk = (p + workers - 1) / workers;
    parallel_for(0, workers, workers, [&](int64_t w) {
        const int64_t lo = w * chunk;
        const int64_t hi = std::min<int64_t>(p, lo + chunk);
        for (int64_t i = lo; i < hi; ++i) {
            Rng rng = derive_stream(master_seed, stream_tag::kImprove, generation * (uint64_t)p + (uint64_t)i);
            SearchStats st;
            Coloring out = partial_mpma_improve(scratch[(size_t)w], make(h->g, offspring + (size_t)i * nv), rng,
                                                budget, &st, alpha, stop_f);
            if (improved) std::memcpy(improved + (size_t)i * nv, out.colors().data(), sizeof(uint16_t) * nv);
            iters[(size_t)i] = st.iterations;
        }
    });
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    int64_t total = 0;
    for (int64_t x : iters) total += x;
    return total;
}

// engine.hpp:184-199 for the MPMA variant: plits_run per individual, per-worker PlitsScratch
int64_t ref_plits_phase(const ref_graph* h, int p, const uint16_t* offspring, uint16_t* improved,
                        uint64_t master_seed, uint64_t generation, int64_t iters1, int64_t iters2, double alpha,
                        int stop_f, int workers, double* seconds) {
    const int nv = h->g.vertex_count();
    if (workers <= 0) workers = default_workers();
    std::vector<PlitsScratch> scratch((size_t)workers);
    std::vector<int64_t> iters((size_t)p, 0);
    PlitsParams params;
    params.phase1_iters = iters1;
    params.phase2_iters = iters2;
    params.alpha = alpha;
    params.stop_f = stop_f;
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t chunk = (p + workers - 1) / workers;
    parallel_for(0, workers, workers, [&](int64_t w) {
        const int64_t lo = w * chunk;
        const int64_t hi = std::min<int64_t>(p, lo + chunk);
        for (int64_t i = lo; i < hi; ++i) {
            Rng rng = derive_stream(master_seed, stream_tag::kImprove, generation * (uint64_t)p + (uint64_t)i);
            SearchStats st;
            Coloring out = plits_run(scratch[(size_t)w], make(h->g, offspring + (size_t)i * nv), rng, params, &st);
            if (improved) std::memcpy(improved + (size_t)i * nv, out.colors().data(), sizeof(uint16_t) * nv);
            iters[(size_t)i] = st.iterations;
        }
    });
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    int64_t total = 0;
    for (int64_t x : iters) total += x;
    return total;
}

int ref_default_workers() { return default_workers(); }


static void copy_out(const std::string& s, char* out, int cap) {
    if (!out || cap <= 0) return;
    const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(out, s.data(), n);
    out[n] = 0;
}

// verify.hpp:20 verify_certificate; problems joined by '\n'.  Returns legal.
int ref_verify_certificate(int n, const uint16_t* instance, int m, const uint16_t* certificate, int* score,
                           char* problems, int cap) {
    VerifyReport r = verify_certificate(grid_instance(n, instance), grid_instance(m, certificate));
    std::string joined;
    for (std::size_t i = 0; i < r.problems.size(); ++i) joined += (i ? "\n" : "") + r.problems[i];
    copy_out(joined, problems, cap);
    if (score) *score = r.score;
    return r.legal ? 1 : 0;
}

// coloring.hpp:171 to_grid
int ref_to_grid(int n, const uint16_t* grid, const uint16_t* colors, uint16_t* out) {
    PlsInstance inst = grid_instance(n, grid);
    ReducedGraph g = preprocess(build_graph(inst));
    Coloring c(g);
    c.assign(std::vector<Color>(colors, colors + g.vertex_count()));
    PlsInstance res = to_grid(inst, g, c);
    for (int r = 0; r < n; ++r)
        for (int col = 0; col < n; ++col) out[r * n + col] = res.at(r, col);
    return 0;
}

#ifdef PLSE_REF_HAVE_JSON
// report.hpp:85 result_to_json, printed as plse.cpp:154 does (dump(2)).
int ref_result_json(const char* name, int order, const ref_run_result* res, const char* stop_reason, int p,
                    double alpha, double gamma, double beta, int64_t phase1, int64_t phase2, int variant,
                    int crossover, int matching, int exclusion, uint64_t seed, int workers, double time_limit,
                    int64_t iteration_limit, int64_t generation_limit, int timing, char* out, int cap) {
    SolverConfig cfg;
    cfg.p = p;
    cfg.alpha = alpha;
    cfg.gamma = gamma;
    cfg.crossover.beta = beta;
    cfg.phase1_iters = phase1;
    cfg.phase2_iters = phase2;
    cfg.variant = variant == 1 ? Variant::PartialMPMA : Variant::MPMA;
    cfg.crossover.mode = crossover == 0 ? CrossoverMode::AUX : crossover == 1 ? CrossoverMode::UX : CrossoverMode::None;
    cfg.crossover.matching = matching == 0 ? MatchingStrategy::NearestNeighbor : MatchingStrategy::Random;
    cfg.crossover.exclusion =
        exclusion == 0 ? ExclusionScope::Run : exclusion == 1 ? ExclusionScope::Generation : ExclusionScope::Off;
    cfg.master_seed = seed;
    cfg.workers = workers;
    cfg.limits.time_seconds = time_limit;
    cfg.limits.total_iterations = iteration_limit;
    cfg.limits.generations = generation_limit;
    RunResult r;
    r.best_f = res->best_f;
    r.best_score = res->best_score;
    r.proven_optimal = res->proven_optimal != 0;
    r.stop_reason = stop_reason;
    r.l = res->l;
    r.upper_bound = res->upper_bound;
    r.vertex_count = res->vertex_count;
    r.generations = res->generations;
    r.total_iterations = res->total_iterations;
    r.elapsed_seconds = res->elapsed_seconds;
    copy_out(result_to_json(name, order, r, cfg, timing != 0).dump(2), out, cap);
    return 0;
}

static std::vector<std::string> split_csv(const char* s) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* q = s; q && *q; ++q) {
        if (*q == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *q;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

// plse.cpp:199-250 cmd_bench through bench.hpp run_bench (CPU reference), all outputs as text
int ref_bench(const char* suite_dir, int repeats, uint64_t master_seed, int p, int64_t gen_limit, int64_t phase1,
              int variant, const char* crossovers, const char* matchings, const char* pops, int jobs, int workers,
              char* rows_csv, int cap1, char* agg_csv, int cap2, char* json_out, int cap3) {
    // plse.cpp:203-211 with POSIX directory calls (std::filesystem clashes with the libstdc++ some
    // Python extensions preload)
    std::vector<BenchTask> tasks;
    std::vector<std::string> files;
    if (DIR* d = opendir(suite_dir)) {
        while (dirent* e = readdir(d)) {
            const std::string name = e->d_name;
            const std::string path = std::string(suite_dir) + "/" + name;
            struct stat st;
            if (name.size() > 4 && name.compare(name.size() - 4, 4, ".txt") == 0 && stat(path.c_str(), &st) == 0 &&
                S_ISREG(st.st_mode))
                files.push_back(path);
        }
        closedir(d);
    }
    std::sort(files.begin(), files.end());
    for (const std::string& file : files) {
        const std::string base = file.substr(file.rfind('/') + 1);
        tasks.push_back({file, base.substr(0, base.size() - 4), static_cast<int>(tasks.size())});
    }
    SolverConfig base;
    base.p = p;
    base.phase1_iters = phase1;
    base.variant = variant == 1 ? Variant::PartialMPMA : Variant::MPMA;
    base.limits.generations = gen_limit;
    base.master_seed = master_seed;
    base.workers = workers;
    std::vector<SolverConfig> sweep;
    auto cl = split_csv(crossovers), ml = split_csv(matchings), pl = split_csv(pops);
    if (cl.empty()) cl = {"aux"};
    if (ml.empty()) ml = {"nearest"};
    std::vector<int> pv;
    for (auto& x : pl) pv.push_back(std::stoi(x));
    if (pv.empty()) pv = {p};
    for (auto& c : cl)
        for (auto& m : ml)
            for (int pp : pv) {
                SolverConfig config = base;
                config.crossover.mode = parse_crossover(c);
                config.crossover.matching = parse_matching(m);
                config.p = pp;
                config.validate();
                sweep.push_back(config);
            }
    const BenchReport report = run_bench(tasks, sweep, repeats, master_seed, jobs, nullptr);
    std::ostringstream a, b;
    write_rows_csv(report, a);
    write_aggregates_csv(report, b);
    copy_out(a.str(), rows_csv, cap1);
    copy_out(b.str(), agg_csv, cap2);
    copy_out(report_to_json(report).dump(2), json_out, cap3);
    return 0;
}
#endif

}  // extern "C"
