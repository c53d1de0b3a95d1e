/*
 * plse_b200.h -- C ABI of the B200-native Partial-MPMA hot path.
 *
 * The reference (/root/reference/proj, header-only C++20) has no plugin or FFI
 * layer: its seam is five C++ calls inside run().  Each entry
 * point below replaces one of them with a batched, device-resident version:
 *
 *   plse_init_population  <- initialize_population      engine.hpp:88-106
 *   plse_improve          <- partial_mpma_improve x p    partial.hpp:156-169,
 *                            driven by the improve phase engine.hpp:184-209
 *                            (+ best tracking engine.hpp:211-217)
 *   plse_distances        <- compute_cross_distances    population.hpp:41-61
 *   plse_update           <- update_population          population.hpp:103-183
 *   plse_offspring        <- build_offspring            crossover.hpp:54-104
 *   plse_solve            <- run (Partial-MPMA)         engine.hpp:114-262
 *
 * plus the reference's host helpers kept on the host side of the boundary:
 *   plse_generate_instance <- generate_instance         instance.hpp:204-262
 *   plse_parse_instance    <- parse_instance            instance.hpp:107-170
 *   plse_preprocess        <- preprocess(build_graph()) lsgraph.hpp:115-211
 *
 * Conventions (mirroring the reference's C++ contract):
 *   - every entry point returns PLSE_OK (0) or a plse_status; the message of
 *     the last failure is available from plse_last_error().  Status codes map
 *     onto the reference's exception types (std::invalid_argument ->
 *     PLSE_ERR_INVALID, std::runtime_error / GenerationError / ParseError ->
 *     PLSE_ERR_RUNTIME).
 *   - colours are uint16_t on the host side of the ABI (Color = Symbol =
 *     uint16_t, instance.hpp:15 / lsgraph.hpp:14); distances are int32_t
 *     (DistanceMatrix, population.hpp:19-32).
 *   - a plse_ctx owns one device and is not thread-safe (one host thread or
 *     process per GPU).  The population stays device-resident between calls.
 *   - there is NO CPU fallback: without a usable sm_100 device plse_create
 *     fails with PLSE_ERR_CUDA.
 */
#ifndef PLSE_B200_H
#define PLSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLSE_ABI_VERSION 2

typedef enum {
    PLSE_OK = 0,
    PLSE_ERR_INVALID = 1,     /* std::invalid_argument in the reference */
    PLSE_ERR_CUDA = 2,        /* device / driver failure, or no sm_100 device */
    PLSE_ERR_UNSUPPORTED = 3, /* outside the device path's envelope (e.g. n > 127) */
    PLSE_ERR_RUNTIME = 4      /* std::runtime_error, GenerationError, ParseError */
} plse_status;

/* population buffers addressed by plse_set_colors / plse_get_colors */
enum { PLSE_MEMBERS = 0, PLSE_OFFSPRING = 1, PLSE_IMPROVED = 2 };
/* distance matrices addressed by plse_get_dist / plse_set_dist */
enum { PLSE_DIST = 0, PLSE_CROSS = 1, PLSE_FRESH = 2 };
/* SolverConfig enums (crossover.hpp:17-19, engine.hpp:18) */
enum { PLSE_X_AUX = 0, PLSE_X_UX = 1, PLSE_X_NONE = 2 };
enum { PLSE_M_NEAREST = 0, PLSE_M_RANDOM = 1 };
enum { PLSE_E_RUN = 0, PLSE_E_GENERATION = 1, PLSE_E_OFF = 2 };
enum { PLSE_V_MPMA = 0, PLSE_V_PARTIAL = 1 };
enum { PLSE_TIE_CANON = 0, PLSE_TIE_REF = 1 };
enum { PLSE_STOP_OPTIMAL = 0, PLSE_STOP_TIME = 1, PLSE_STOP_ITERS = 2, PLSE_STOP_GENS = 3, PLSE_STOP_TRIVIAL = 4,
       PLSE_STOP_TARGET = 5 /* harness: target_score reached */ };

typedef struct plse_ctx plse_ctx;
typedef struct plse_graph_h plse_graph_h; /* host-side ReducedGraph handle */

/* ReducedGraph (lsgraph.hpp:67-109) as plain arrays. */
typedef struct {
    int32_t order;              /* n */
    int32_t vertex_count;       /* |V| */
    int32_t l;                  /* cells impossible to fill */
    const int32_t* cell_row;    /* [|V|] */
    const int32_t* cell_col;    /* [|V|] */
    const int32_t* dom_offsets; /* [|V|+1] CSR domains, ascending, starting with 0 */
    const uint16_t* dom;        /* [dom_offsets[|V|]] */
    int32_t n_prefilled;        /* ReducedGraph::prefilled (lsgraph.hpp:85) */
    const int32_t* prefilled;   /* [3*n_prefilled]: row, col, symbol */
} plse_graph;

/* SolverConfig (engine.hpp:26-47) + the island coordinates of this shard. */
typedef struct {
    int32_t p;              /* population (of this shard) */
    double alpha;           /* tenure factor (partial.hpp:136-137) */
    double gamma;           /* spacing divisor (population.hpp:74) */
    double beta;            /* AUX divisor (crossover.hpp:26-30) */
    int64_t phase1_iters;   /* 0 -> 100|V| (engine.hpp:173-174) */
    int32_t crossover;      /* PLSE_X_* */
    int32_t matching;       /* PLSE_M_* */
    int32_t exclusion;      /* PLSE_E_* */
    int32_t tie_mode;       /* PLSE_TIE_CANON (throughput) or PLSE_TIE_REF (the reference's reservoir
                               draws: bit-exact trajectories, both variants) */
    uint64_t master_seed;
    int64_t p_total;        /* stream index space: gen*p_total + offset + i; 0 -> p */
    int64_t offset;         /* first global individual of this shard */
    int32_t variant;        /* PLSE_V_PARTIAL (PartialCol improve) or PLSE_V_MPMA (PLITS improve, plits.hpp) */
    int64_t phase2_iters;   /* MPMA phase-2 budget, 0 -> 2|V| (plits.hpp:244) */
} plse_params;

/* One PartialCol step, for the per-step parity probe (partial.hpp:92-143). */
typedef struct {
    int64_t step;
    int32_t v, k, e, ev0, ev1;
    int32_t f_before, f_after, best_f;
    int32_t tenure, n_adm, level;
} plse_step;

/* Timings / counters of the last plse_improve (device-side CUDA events). */
typedef struct {
    double improve_ms;          /* improve kernel */
    double alg_bytes;           /* sum of SURVEY 8(d) algorithmic bytes over the launch */
    int64_t moves;              /* iterations (tabu moves) of the launch */
    int32_t grid, threads, warps_per_sm, slots;
    int64_t smem_bytes;
    int64_t kernel_launches;    /* this context's kernel launches so far */
    double distances_ms;        /* last plse_distances (K3: one-hot expansion + tcgen05 GEMM) */
    double update_ms;           /* last plse_update */
    double offspring_ms;        /* last plse_offspring */
    double k3_ops;              /* 2 * M * N * Kpad summed over the last plse_distances GEMMs */
    int32_t k3_tensor_cores;    /* 1 if K3 ran on tcgen05 */
} plse_counters;

/* RunResult (engine.hpp:59-71) */
typedef struct {
    int32_t best_f, best_score, proven_optimal, stop_reason, l, upper_bound, vertex_count;
    int64_t generations, total_iterations;
    double elapsed_seconds;
    double time_to_best_seconds; /* elapsed when best_f first reached its final value */
} plse_run_result;

/* SolverConfig + RunLimits for plse_solve */
typedef struct {
    plse_params params;
    int32_t variant;            /* PLSE_V_PARTIAL or PLSE_V_MPMA (overrides params.variant) */
    double time_limit;          /* seconds, 0 = unlimited */
    int64_t iteration_limit;    /* 0 = unlimited */
    int64_t generation_limit;   /* 0 = unlimited */
    int32_t device;
    int32_t disable_optimal_stop; /* harness flag */
    double target_score;        /* >0: stop as soon as best_score >= target (time-to-target) */
    int32_t race;               /* with target_score: end the improve phase as soon as ANY individual
                                   reaches the target (device-global early exit; not parity mode) */
} plse_solver_config;

/* per-generation statistics (GenerationStats, engine.hpp:49-57) */
typedef struct {
    int64_t generation;
    int32_t best_f;          /* best f ever seen (legal) */
    double mean_f;           /* mean f of the (updated) population */
    double mean_distance;    /* mean pairwise Hamming distance over i < j */
    int64_t iterations;      /* total tabu iterations so far */
    double elapsed_seconds;
    int32_t shortfall;       /* slots the pool update could not fill */
} plse_generation_stats;

/* per-generation callback (GenerationCallback, engine.hpp:108) */
typedef void (*plse_generation_cb)(const plse_generation_stats* stats, void* user);

int plse_abi_version(void);
const char* plse_last_error(const plse_ctx* ctx); /* ctx may be NULL: last global error */

/* ---- host helpers (C++ host library, instance.hpp / lsgraph.hpp semantics) */
int plse_generate_instance(int32_t n, double r, uint64_t seed, uint16_t* grid /* n*n */);
int plse_parse_instance(const char* text, int32_t* n, uint16_t* grid /* cap n*n */, int32_t grid_cap);
int plse_preprocess(int32_t n, const uint16_t* grid, plse_graph_h** out);
void plse_graph_free(plse_graph_h* g);
int plse_graph_view(const plse_graph_h* g, plse_graph* view); /* borrowed arrays, valid until free */
/* coloring.hpp:171 to_grid: certificate grid [n*n] from a |V|-colouring (colours are symbols, 0 = empty) */
int plse_to_grid(const plse_graph_h* g, const uint16_t* colors, uint16_t* grid);
/* oracle.hpp:134 solve_exact (host, CPU): exact minimum f by branch and bound, one optimal certificate
   (|V| colours), exact = 0 when the node budget ran out (default budget in the reference: 50'000'000) */
int plse_solve_exact(const plse_graph_h* g, int64_t node_budget, int32_t* optimum_f, int32_t* exact, int64_t* nodes,
                     uint16_t* certificate /* |V| */);
/* verify.hpp:20 verify_certificate: problems joined by '\n' (NUL-terminated, truncated to cap;
   *problems_len = full length); legal = no problems, score = filled cells of the certificate */
int plse_verify_certificate(int32_t n, const uint16_t* instance, int32_t m, const uint16_t* certificate,
                            int32_t* legal, int32_t* score, char* problems, int64_t problems_cap,
                            int64_t* problems_len);

/* ---- device context */
int plse_create(const plse_graph* graph, const plse_params* params, int32_t device, plse_ctx** out);
void plse_destroy(plse_ctx* ctx);
/* colourings as u16 rows [p][|V|] (vertex order of plse_preprocess).  set: the rows are copied as they are
   and checked on the device (every colour 0 or in the vertex's domain, lsgraph.hpp:152-156); an invalid
   colouring returns PLSE_ERR_INVALID ("assignment leaves vertex domain") and leaves the buffer unchanged.
   Pinned host rows (cudaHostAlloc / cudaHostRegister) copy at the full link rate; pageable ones work too. */
int plse_set_colors(plse_ctx* ctx, int32_t which, const uint16_t* host, int64_t count /* p*|V| */);
int plse_get_colors(plse_ctx* ctx, int32_t which, uint16_t* host);
/* one row (individual `index`) of a population buffer: |V| u16 colours (the run's best without the whole
   population crossing the link) */
int plse_get_row(plse_ctx* ctx, int32_t which, int32_t index, uint16_t* host /* |V| */);
int plse_get_dist(plse_ctx* ctx, int32_t which, int32_t* host /* p*p */);
int plse_set_dist(plse_ctx* ctx, int32_t which, const int32_t* host);
/* f, c (conflicting edges) and the last improve's iterations per individual; any may be NULL */
int plse_get_stats(plse_ctx* ctx, int32_t which, int32_t* f, int32_t* c, int64_t* iters);
int plse_get_partners(plse_ctx* ctx, int32_t* host /* p */);
int plse_get_counters(plse_ctx* ctx, plse_counters* out);
/* device-side timing on the context's stream (CUDA events): start, then stop -> elapsed ms */
int plse_timer_start(plse_ctx* ctx);
int plse_timer_stop(plse_ctx* ctx, double* ms);
/* device pointer of a u8 population buffer (row stride = |V| rounded up to 16), for NCCL / torch interop */
int plse_device_colors(plse_ctx* ctx, int32_t which, void** dev_ptr, int64_t* row_stride);

int plse_init_population(plse_ctx* ctx);
int plse_full_distances(plse_ctx* ctx); /* dist <- D(members, members) */
int plse_improve(plse_ctx* ctx, uint64_t generation, int64_t* iters_total, int32_t* best_f, int32_t* best_idx);
int plse_distances(plse_ctx* ctx);
/* the whole update runs on the device; the outputs (each optional, NULL = not read back, no host
   synchronisation) are UpdateInfo's fields */
int plse_update(plse_ctx* ctx, int32_t* pool_best_f, int32_t* n_shortfall, int32_t* shortfall_slots /* cap p */);
int plse_reset_exclusion(plse_ctx* ctx);
int plse_offspring(plse_ctx* ctx, uint64_t generation);
/* run individual idx of OFFSPRING through improve with a per-step trace (parity probe) */
int plse_trace(plse_ctx* ctx, int32_t idx, uint64_t generation, int64_t max_steps, plse_step* out, int64_t* n_out);

/* per-step state probe (the north star's "gamma tables ... tabu lists bit-exact per step"): run
   individual idx of OFFSPRING through improve and, before each listed step j (ascending; j = 0 is the
   post-repair state), dump gamma[v][k] (coloring.hpp:105-116; n_steps x |V| x (order+1)) and the live
   tabu entries (v, k, until) on the reference's iteration clock (search_util.hpp:54-81; n_steps x tabu_cap
   x 3, count per step in n_tabu_out).  n_dumped = probe points the search reached; cache_mismatch =
   vertices whose tabu cache disagreed with the dense table (0 on a correct kernel).  Canonical policy;
   with variant MPMA (PLITS) the steps are counted over both phases, colour 0 can be tabu, and until is on
   the phase's own clock (plits.hpp:81). */
int plse_probe(plse_ctx* ctx, int32_t idx, uint64_t generation, int32_t n_steps, const int64_t* steps,
               int32_t* gamma_out, int32_t tabu_cap, int32_t* tabu_out, int32_t* n_tabu_out, int32_t* n_dumped,
               int32_t* cache_mismatch);

/* ---- island exchange (multi-GPU): the driver moves the bytes (NCCL all-gather) */
/* the n_elite best members ((illegal, f, slot) ascending) as u8 rows [n_elite * row_stride] into dev_out,
   written on the context's stream (plse_stream); f_out (host, optional) synchronises */
int plse_export_elites(plse_ctx* ctx, int32_t n_elite, void* dev_out, int32_t* f_out);
/* stage n_in u8 rows [n_in * row_stride] (device pointer, read on the context's stream) as extra
   candidates -- pool ids 2p..2p+n_in-1 -- of the next plse_update (update_population with a 2p+n_in
   pool, population.hpp:103-183); call between plse_improve and plse_update */
int plse_import_migrants(plse_ctx* ctx, int32_t n_in, const void* dev_in);
/* the cudaStream_t every phase of this context is enqueued on (for event / collective ordering) */
int plse_stream(plse_ctx* ctx, void** stream_out);

/* ---- the whole run() (engine.hpp:114-262) on one device */
int plse_solve(int32_t n, const uint16_t* grid, const plse_solver_config* cfg, plse_run_result* res,
               uint16_t* best_colors /* |V| */, plse_generation_cb cb, void* user);

#ifdef __cplusplus
}
#endif
#endif
