/*
 * plse_oracle.h -- CPU restatement of the reference's Partial-MPMA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2103_10453_b200/,
 * include/, the C-ABI library) links, loads or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may use it, and only as the checker / the CPU baseline.
 *
 * It restates, in plain C, the reference headers under
 * /root/reference/proj/include/plse (each function cites the file:line it
 * follows).  Two tie-break policies for the PartialCol step are provided:
 *
 *   OR_TIE_REF   -- the reference's own rule: reservoir sampling in IndexSet
 *                   order with sequential xoshiro256++ draws
 *                   (partial.hpp:100-117).  Pinned bit-exact against the
 *                   compiled reference (oracle/_ref) and the committed golden
 *                   trajectories in tests/golden/.
 *   OR_TIE_CANON -- the order-free canonical rule the GPU implements (see
 *                   DESIGN.md "Canonical tie-break"): the r-th admissible
 *                   minimum-delta candidate in ascending (v, k) order with
 *                   r = floor(u32 * N / 2^32), u32 from a counter-based
 *                   fmix32 hash keyed (stream seed, step).  Everything
 *                   else in the step (gamma, aspiration, tabu, eviction,
 *                   tenure formula, best snapshot) is shared code with
 *                   OR_TIE_REF, so pinning the REF policy pins it.
 *
 * Parity pinned: yes -- see tests/test_oracle_vs_reference.py and
 * tests/test_oracle_golden.py.
 */
#ifndef PLSE_ORACLE_H
#define PLSE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_TIE_CANON = 0, OR_TIE_REF = 1 };
enum { OR_X_AUX = 0, OR_X_UX = 1, OR_X_NONE = 2 };
enum { OR_M_NEAREST = 0, OR_M_RANDOM = 1 };
enum { OR_E_RUN = 0, OR_E_GENERATION = 1, OR_E_OFF = 2 };
enum { OR_STOP_OPTIMAL = 0, OR_STOP_TIME = 1, OR_STOP_ITERS = 2, OR_STOP_GENS = 3, OR_STOP_TRIVIAL = 4 };

/* ---- rng.hpp:14-92 ---------------------------------------------------- */
typedef struct { uint64_t s[4]; } or_rng;
uint64_t or_splitmix64(uint64_t* state);
void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
uint64_t or_rng_below(or_rng* r, uint64_t bound);
double or_rng_double(or_rng* r);
uint64_t or_derive_seed(uint64_t master, uint64_t tag, uint64_t index);
/* counter-based draw used by OR_TIE_CANON for step j (hi: move rank, lo: tenure offset) */
uint64_t or_canon_draw(uint64_t s, uint64_t j);

/* ---- instance.hpp:204-262, builders.hpp:30-58 ------------------------- */
int or_generate_instance(int n, double r, uint64_t seed, uint16_t* grid);
void or_lsc_instance(int n, double r, uint64_t seed, uint16_t* grid);

/* ---- lsgraph.hpp:67-211 ----------------------------------------------- */
typedef struct {
    int n, nv, l;
    int32_t* cell_row;    /* nv */
    int32_t* cell_col;    /* nv */
    int32_t* vertex_at;   /* n*n, -1 if removed */
    int32_t* adj_off;     /* nv+1 */
    int32_t* adj;         /* adj_off[nv] */
    int32_t* dom_off;     /* nv+1 */
    uint16_t* dom;        /* dom_off[nv], ascending, starts with 0 */
} or_graph;

or_graph* or_preprocess(int n, const uint16_t* grid);
void or_graph_free(or_graph* g);
int or_graph_nv(const or_graph* g);
int or_graph_l(const or_graph* g);
int or_graph_adj_len(const or_graph* g);
int or_graph_dom_len(const or_graph* g);
int or_graph_order(const or_graph* g);
/* copies the CSR arrays out (caller-sized buffers, any may be NULL) */
void or_graph_export(const or_graph* g, int32_t* cell_row, int32_t* cell_col, int32_t* adj_off,
                     int32_t* adj, int32_t* dom_off, uint16_t* dom);

/* ---- coloring.hpp:59-167 ---------------------------------------------- */
void or_eval(const or_graph* g, const uint16_t* colors, int* f, int* c);
void or_gamma_build(const or_graph* g, const uint16_t* colors, int32_t* gamma /* nv*(n+1) */);
int or_hamming(int nv, const uint16_t* a, const uint16_t* b);

/* ---- partial.hpp:22-39 ------------------------------------------------- */
void or_repair(const or_graph* g, uint16_t* colors);

/* ---- partial.hpp:76-169 ------------------------------------------------ */
typedef struct {
    int64_t step;      /* 0-based step index (tabu clock) */
    int32_t v, k;      /* chosen move; -1, 0 on an all-tabu step */
    int32_t e;         /* evictions */
    int32_t ev0, ev1;  /* evicted vertices (-1 if none), in CSR order */
    int32_t f_before, f_after, best_f;
    int32_t tenure;    /* -1 on an all-tabu step */
    int32_t n_adm;     /* CANON: admissible candidates at the min level; REF: ties */
    int32_t level;     /* min admissible delta (-1, 0, 1), 2 if none */
} or_step;

typedef struct {
    int64_t iterations;
    int32_t repaired_f, best_f;
    double alg_bytes; /* sum of SURVEY 8(d) algorithmic bytes B_t over the run */
} or_improve_stats;

/* partial_mpma_improve(scratch, input, Rng(stream_seed), budget, ..., alpha, stop_f)
 * out_best receives best(); trace (optional) receives up to trace_cap steps. */
/* state probe of or_improve (the per-step parity contract): before each listed step */
typedef struct {
    int n;                 /* probe points, ascending steps */
    const int64_t* steps;
    int32_t* gamma;        /* n x nv x (order+1) */
    int32_t* tabu;         /* n x cap x 3: v, k, until */
    int32_t* n_tabu;       /* n */
    int32_t* dumped;       /* [1] */
    int cap;
} or_probe;
int or_plits_probe(const or_graph* g, const uint16_t* input, uint64_t stream_seed, int64_t iters1, int64_t iters2,
                   double alpha, int stop_f, int tie_mode, const or_probe* probe);
int or_improve_probe(const or_graph* g, const uint16_t* input, uint64_t stream_seed, int64_t budget, double alpha,
                     int stop_f, int tie_mode, const or_probe* probe);
int or_improve(const or_graph* g, const uint16_t* input, uint16_t* out_best, uint64_t stream_seed,
               int64_t budget, double alpha, int stop_f, int tie_mode, or_improve_stats* st,
               or_step* trace, int64_t trace_cap);

/* ---- plits.hpp:96-292 (the MPMA variant's improve operator) ------------ */
typedef struct {
    int64_t step;       /* 0-based step index over both phases (the CANON draw key) */
    int32_t phase;      /* 1 or 2 */
    int32_t v, k, from; /* chosen move; v = -1 on an all-tabu step */
    int32_t df, dc;
    int64_t delta;      /* wf*df + wc*dc */
    int64_t cur_scaled, best_scaled; /* after the step */
    int32_t n_adm;      /* CANON: admissible candidates at the minimum; REF: ties */
    int32_t tenure;     /* -1 on an all-tabu step */
    int32_t active;     /* |uncoloured| + |conflicting| after the step */
    int32_t f, c;       /* after the step */
} or_plits_step;

typedef struct {
    int64_t iterations;        /* both phases (SearchStats::iterations) */
    int64_t phase1_iterations;
    int32_t hit_target;        /* phase 1 reached a legal best with f <= stop_f */
    int32_t repaired;          /* the final greedy repair ran (phase 2 ended illegal) */
    int32_t final_f;           /* f of the returned (legal) colouring */
    double alg_bytes;          /* DESIGN.md "PLITS" byte model */
} or_plits_stats;

/* plits_run(scratch, input, Rng(stream_seed), {iters1, iters2, alpha, stop_f}, &stats):
 * phase 1 (phi = 0.5: 2F = 2f + c) then, unless it hit the target, phase 2
 * (phi = |V|: 2F = 2f + 2|V|c) from phase 1's best with a fresh tabu table,
 * then the greedy repair if the result still conflicts.  iters <= 0 take the
 * defaults 100|V| and 2|V| (plits.hpp:243-244).  OR_TIE_REF = the reference's
 * reservoir sampling over IndexSet order; OR_TIE_CANON = the GPU's rule, with
 * the draw keyed by the step index over both phases. */
int or_plits(const or_graph* g, const uint16_t* input, uint16_t* out, uint64_t stream_seed, int64_t iters1,
             int64_t iters2, double alpha, int stop_f, int tie_mode, or_plits_stats* st,
             or_plits_step* trace, int64_t trace_cap);

/* ---- oracle.hpp:24-179 (exact optimum; recursive, for small |V|) ---------- */
typedef struct {
    int32_t optimum_f;
    int32_t exact;   /* 0 when the node budget ran out */
    int64_t nodes;
} or_exact_result;
/* solve_exact: fail-first branch and bound with pruning; certificate = |V| colours */
int or_solve_exact(const or_graph* g, int64_t node_budget, or_exact_result* res, uint16_t* certificate);
/* enumerate_exact: every legal colouring, vertices in index order, no pruning */
int or_enumerate_exact(const or_graph* g, or_exact_result* res, uint16_t* certificate);

/* ---- population.hpp:41-228, crossover.hpp:26-104, engine.hpp:88-106 --- */
void or_cross_distances(int nv, int p, const uint16_t* members, const uint16_t* improved,
                        int32_t* cross, int32_t* fresh);
void or_full_distances(int nv, int p, const uint16_t* members, int32_t* dist);
/* or_update with m migrant rows as extra pool candidates (ids 2p..2p+m-1; island exchange) */
int or_update_ex(const or_graph* g, int p, double spacing_gamma, uint16_t* members, int32_t* dist,
                 const uint16_t* improved, const int32_t* cross, const int32_t* fresh, int m,
                 const uint16_t* migrants, int32_t* pool_best_f, int32_t* shortfall_slots,
                 int32_t* n_shortfall, int32_t* selected_ids);
int or_update(const or_graph* g, int p, double spacing_gamma, uint16_t* members, int32_t* dist,
              const uint16_t* improved, const int32_t* cross, const int32_t* fresh,
              int32_t* pool_best_f, int32_t* shortfall_slots, int32_t* n_shortfall,
              int32_t* selected_ids);
int or_nearest_neighbor(int p, const int32_t* dist, int i, uint8_t* excl /* p*p or NULL */);
int or_offspring(const or_graph* g, int p, const uint16_t* members, const int32_t* dist,
                 int crossover, double beta, int matching, int exclusion, uint8_t* excl,
                 uint64_t master_seed, uint64_t generation, uint16_t* offspring, int32_t* partner);
void or_init_population(const or_graph* g, int p, uint64_t master_seed, uint16_t* members);
/* island forms: stream indices offset+i and stream_base+i */
int or_offspring_ex(const or_graph* g, int p, const uint16_t* members, const int32_t* dist,
                    int crossover, double beta, int matching, int exclusion, uint8_t* excl,
                    uint64_t master_seed, uint64_t stream_base, uint16_t* offspring, int32_t* partner);
void or_init_population_ex(const or_graph* g, int p, uint64_t master_seed, uint64_t offset, uint16_t* members);

/* ---- engine.hpp:114-262 (partial variant) ------------------------------ */
typedef struct {
    int32_t p;
    double alpha, gamma, beta;
    int64_t phase1_iters; /* 0 -> 100|V| */
    int32_t crossover, matching, exclusion;
    uint64_t master_seed;
    int64_t iteration_limit, generation_limit;
    int32_t tie_mode;
    int32_t disable_optimal_stop; /* harness flag */
    int32_t variant;              /* 0 = MPMA (PLITS improve), 1 = Partial-MPMA (engine.hpp:193-203) */
    int64_t phase2_iters;         /* MPMA phase-2 budget, 0 -> 2|V| */
} or_config;

typedef struct {
    int32_t best_f, best_score, proven_optimal, stop_reason, l, upper_bound, vertex_count;
    int64_t generations, total_iterations;
} or_result;

/* per-generation log (GenerationStats, engine.hpp:49-57 / emit_stats 214-233): best_f after the
   improve phase, iterations so far, and the population's mean f and mean pairwise distance */
typedef struct {
    int64_t generation;
    int32_t best_f;
    int32_t shortfall;
    int64_t iterations;
    double mean_f;
    double mean_distance;
} or_gen_log;

int or_run(int n, const uint16_t* grid, const or_config* cfg, or_result* res, uint16_t* best_colors,
           or_gen_log* log, int64_t log_cap);

#ifdef __cplusplus
}
#endif
#endif
