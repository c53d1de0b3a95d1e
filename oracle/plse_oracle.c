/*
 * plse_oracle.c -- CPU restatement of the reference's Partial-MPMA hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see plse_oracle.h).  Every function cites the
 * reference file:line (paths relative to /root/reference/proj/include/plse)
 * whose behaviour it restates.  Written for clarity, not speed: it keeps the
 * reference's dense int32 gamma table and dense tabu table so that it is an
 * independent check of the GPU's row/column-occupancy formulation.
 */
#include "plse_oracle.h"

#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

/* ------------------------------------------------------------------ rng */

/* rng.hpp:14-19 */
uint64_t or_splitmix64(uint64_t* state) {
    uint64_t z = (*state += GOLDEN);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.hpp:25-28 */
void or_rng_seed(or_rng* r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = or_splitmix64(&sm);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:30-40 (xoshiro256++) */
uint64_t or_rng_next(or_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* rng.hpp:43-49 (unbiased by rejection) */
uint64_t or_rng_below(or_rng* r, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t x = or_rng_next(r);
        if (x >= threshold) return x % bound;
    }
}

/* rng.hpp:56-58 */
double or_rng_double(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:81-88 */
uint64_t or_derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
    uint64_t s = master;
    uint64_t h = or_splitmix64(&s);
    s = h ^ (tag * 0xD1B54A32D192ED03ULL);
    h = or_splitmix64(&s);
    s = h ^ (index * 0x8CB92BA72F3D8DD7ULL);
    return or_splitmix64(&s);
}

/* Canonical counter-based draw for step j of the stream seeded s (not in the
 * reference): SplitMix64's (j+1)-th output from
 * state s (rng.hpp:14-19's generator, evaluated at a counter), i.e. keyed by the
 * full 64-bit stream seed.  hi 32 bits select the move (r = floor(hi * N / 2^32)),
 * lo 32 bits the tenure offset (L = floor(lo * 10 / 2^32)). */
uint64_t or_canon_draw(uint64_t s, uint64_t j) {
    uint64_t z = s + (j + 1) * GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------- instance */

/* instance.hpp:204-262: random partial Latin square at fill ratio r. */
int or_generate_instance(int n, double r, uint64_t seed, uint16_t* grid) {
    if (n <= 0 || !(r > 0.0 && r < 1.0)) return -1;
    const int total = n * n;
    const int target = (int)(r * total);
    const int max_failures = 50 * total;
    const int words = (n + 64) / 64;
    uint64_t* used = (uint64_t*)malloc(sizeof(uint64_t) * 2 * n * words);
    int* empty = (int*)malloc(sizeof(int) * total);
    uint16_t* adm = (uint16_t*)malloc(sizeof(uint16_t) * (n + 1));
    int ok = -1;
    for (int restart = 0; restart < 100 && ok != 0; ++restart) {
        or_rng rng;
        or_rng_seed(&rng, or_derive_seed(seed, 4, (uint64_t)restart));
        memset(grid, 0, sizeof(uint16_t) * total);
        memset(used, 0, sizeof(uint64_t) * 2 * n * words);
        for (int i = 0; i < total; ++i) empty[i] = i;
        int empty_count = total, filled = 0, failures = 0;
        while (filled < target && failures < max_failures) {
            const int pick = (int)or_rng_below(&rng, (uint64_t)empty_count);
            const int cell = empty[pick];
            const int row = cell / n, col = cell % n;
            int na = 0;
            for (int s = 1; s <= n; ++s) {
                const int ur = (int)((used[(size_t)row * words + s / 64] >> (s % 64)) & 1);
                const int uc = (int)((used[(size_t)(n + col) * words + s / 64] >> (s % 64)) & 1);
                if (!ur && !uc) adm[na++] = (uint16_t)s;
            }
            if (na == 0) {
                ++failures;
                continue;
            }
            const uint16_t sym = adm[or_rng_below(&rng, (uint64_t)na)];
            grid[cell] = sym;
            used[(size_t)row * words + sym / 64] |= 1ULL << (sym % 64);
            used[(size_t)(n + col) * words + sym / 64] |= 1ULL << (sym % 64);
            empty[pick] = empty[--empty_count];
            ++filled;
            failures = 0;
        }
        if (filled == target) ok = 0;
    }
    free(used);
    free(empty);
    free(adm);
    return ok;
}

/* builders.hpp:19-26 */
static void random_permutation(int n, or_rng* rng, int* perm) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = n - 1; i > 0; --i) {
        const int j = (int)or_rng_below(rng, (uint64_t)(i + 1));
        const int t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
}

/* builders.hpp:30-58: complete cyclic square, permuted, then cells deleted. */
void or_lsc_instance(int n, double r, uint64_t seed, uint16_t* grid) {
    or_rng rng;
    or_rng_seed(&rng, seed);
    int* rows = (int*)malloc(sizeof(int) * n);
    int* cols = (int*)malloc(sizeof(int) * n);
    int* syms = (int*)malloc(sizeof(int) * n);
    random_permutation(n, &rng, rows);
    random_permutation(n, &rng, cols);
    random_permutation(n, &rng, syms);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) grid[a * n + b] = (uint16_t)(syms[(rows[a] + cols[b]) % n] + 1);
    or_rng_seed(&rng, seed ^ 0x5DEECE66DULL);
    const int keep = (int)(r * n * n);
    int* cells = (int*)malloc(sizeof(int) * n * n);
    random_permutation(n * n, &rng, cells);
    for (int i = keep; i < n * n; ++i) grid[cells[i]] = 0;
    free(rows);
    free(cols);
    free(syms);
    free(cells);
}

/* ---------------------------------------------------------------- graph */

/* lsgraph.hpp:115-211 (Alg. 1 reduction). */
or_graph* or_preprocess(int n, const uint16_t* grid) {
    const int total = n * n;
    const int words = (n + 64) / 64;
    or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
    g->n = n;
    g->vertex_at = (int32_t*)malloc(sizeof(int32_t) * total);
    for (int i = 0; i < total; ++i) g->vertex_at[i] = -1;
    uint64_t* line = (uint64_t*)calloc((size_t)2 * n * words, sizeof(uint64_t));
    for (int v = 0; v < total; ++v) {
        const int k = grid[v];
        if (!k) continue;
        line[(size_t)(v / n) * words + k / 64] |= 1ULL << (k % 64);
        line[(size_t)(n + v % n) * words + k / 64] |= 1ULL << (k % 64);
    }
    /* survivors in row-major order, domains {0} u free symbols (149-165) */
    int nv = 0, ndom = 0;
    for (int v = 0; v < total; ++v) {
        if (grid[v]) continue;
        int sz = 0;
        for (int k = 1; k <= n; ++k) {
            const int m = (int)(((line[(size_t)(v / n) * words + k / 64] |
                                  line[(size_t)(n + v % n) * words + k / 64]) >>
                                 (k % 64)) & 1);
            sz += !m;
        }
        if (sz == 0) {
            g->l++;
            continue;
        }
        g->vertex_at[v] = nv++;
        ndom += sz + 1;
    }
    g->nv = nv;
    g->cell_row = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    g->cell_col = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    g->dom_off = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    g->dom = (uint16_t*)malloc(sizeof(uint16_t) * (ndom + 1));
    g->dom_off[0] = 0;
    for (int v = 0; v < total; ++v) {
        const int id = g->vertex_at[v];
        if (id < 0) continue;
        g->cell_row[id] = v / n;
        g->cell_col[id] = v % n;
        int at = g->dom_off[id];
        g->dom[at++] = 0;
        for (int k = 1; k <= n; ++k) {
            const int m = (int)(((line[(size_t)(v / n) * words + k / 64] |
                                  line[(size_t)(n + v % n) * words + k / 64]) >>
                                 (k % 64)) & 1);
            if (!m) g->dom[at++] = (uint16_t)k;
        }
        g->dom_off[id + 1] = at;
    }
    /* adjacency: fill order of 185-209 (per line index: row group, then column group) */
    int* row_cnt = (int*)calloc(n, sizeof(int));
    int* col_cnt = (int*)calloc(n, sizeof(int));
    for (int v = 0; v < nv; ++v) {
        row_cnt[g->cell_row[v]]++;
        col_cnt[g->cell_col[v]]++;
    }
    g->adj_off = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    g->adj_off[0] = 0;
    for (int v = 0; v < nv; ++v)
        g->adj_off[v + 1] = g->adj_off[v] + row_cnt[g->cell_row[v]] + col_cnt[g->cell_col[v]] - 2;
    g->adj = (int32_t*)malloc(sizeof(int32_t) * (g->adj_off[nv] + 1));
    int* fill = (int*)malloc(sizeof(int) * (nv + 1));
    for (int v = 0; v < nv; ++v) fill[v] = g->adj_off[v];
    /* by_row / by_col lists in ascending vertex order */
    int* by_row_start = (int*)calloc(n + 1, sizeof(int));
    int* by_col_start = (int*)calloc(n + 1, sizeof(int));
    for (int i = 0; i < n; ++i) {
        by_row_start[i + 1] = by_row_start[i] + row_cnt[i];
        by_col_start[i + 1] = by_col_start[i] + col_cnt[i];
    }
    int* by_row = (int*)malloc(sizeof(int) * (nv + 1));
    int* by_col = (int*)malloc(sizeof(int) * (nv + 1));
    int* rp = (int*)malloc(sizeof(int) * n);
    int* cp = (int*)malloc(sizeof(int) * n);
    for (int i = 0; i < n; ++i) {
        rp[i] = by_row_start[i];
        cp[i] = by_col_start[i];
    }
    for (int v = 0; v < nv; ++v) {
        by_row[rp[g->cell_row[v]]++] = v;
        by_col[cp[g->cell_col[v]]++] = v;
    }
    for (int ln = 0; ln < n; ++ln) {
        for (int a = by_row_start[ln]; a < by_row_start[ln + 1]; ++a)
            for (int b = by_row_start[ln]; b < by_row_start[ln + 1]; ++b)
                if (a != b) g->adj[fill[by_row[a]]++] = by_row[b];
        for (int a = by_col_start[ln]; a < by_col_start[ln + 1]; ++a)
            for (int b = by_col_start[ln]; b < by_col_start[ln + 1]; ++b)
                if (a != b) g->adj[fill[by_col[a]]++] = by_col[b];
    }
    free(line);
    free(row_cnt);
    free(col_cnt);
    free(fill);
    free(by_row_start);
    free(by_col_start);
    free(by_row);
    free(by_col);
    free(rp);
    free(cp);
    return g;
}

void or_graph_free(or_graph* g) {
    if (!g) return;
    free(g->cell_row);
    free(g->cell_col);
    free(g->vertex_at);
    free(g->adj_off);
    free(g->adj);
    free(g->dom_off);
    free(g->dom);
    free(g);
}

int or_graph_nv(const or_graph* g) { return g->nv; }
int or_graph_l(const or_graph* g) { return g->l; }
int or_graph_adj_len(const or_graph* g) { return g->adj_off[g->nv]; }
int or_graph_dom_len(const or_graph* g) { return g->dom_off[g->nv]; }
int or_graph_order(const or_graph* g) { return g->n; }

void or_graph_export(const or_graph* g, int32_t* cell_row, int32_t* cell_col, int32_t* adj_off,
                     int32_t* adj, int32_t* dom_off, uint16_t* dom) {
    const int nv = g->nv;
    if (cell_row) memcpy(cell_row, g->cell_row, sizeof(int32_t) * nv);
    if (cell_col) memcpy(cell_col, g->cell_col, sizeof(int32_t) * nv);
    if (adj_off) memcpy(adj_off, g->adj_off, sizeof(int32_t) * (nv + 1));
    if (adj) memcpy(adj, g->adj, sizeof(int32_t) * g->adj_off[nv]);
    if (dom_off) memcpy(dom_off, g->dom_off, sizeof(int32_t) * (nv + 1));
    if (dom) memcpy(dom, g->dom, sizeof(uint16_t) * g->dom_off[nv]);
}

/* ------------------------------------------------------------- coloring */

/* coloring.hpp:59-73 */
void or_eval(const or_graph* g, const uint16_t* colors, int* f, int* c) {
    int ff = 0, cc = 0;
    for (int v = 0; v < g->nv; ++v) {
        const int k = colors[v];
        if (!k) {
            ++ff;
            continue;
        }
        for (int a = g->adj_off[v]; a < g->adj_off[v + 1]; ++a)
            if (g->adj[a] > v && colors[g->adj[a]] == k) ++cc;
    }
    if (f) *f = ff;
    if (c) *c = cc;
}

/* coloring.hpp:105-116 */
void or_gamma_build(const or_graph* g, const uint16_t* colors, int32_t* gamma) {
    const int w = g->n + 1;
    memset(gamma, 0, sizeof(int32_t) * (size_t)g->nv * w);
    for (int v = 0; v < g->nv; ++v) {
        const int k = colors[v];
        if (!k) continue;
        for (int a = g->adj_off[v]; a < g->adj_off[v + 1]; ++a) gamma[(size_t)g->adj[a] * w + k] += 1;
    }
}

/* coloring.hpp:159-167 */
int or_hamming(int nv, const uint16_t* a, const uint16_t* b) {
    int d = 0;
    for (int i = 0; i < nv; ++i) d += a[i] != b[i];
    return d;
}

/* Mutable coloring state: colours + f/c caches + gamma (coloring.hpp:20-156). */
typedef struct {
    const or_graph* g;
    int w;
    uint16_t* col;
    int32_t* gamma;
    int f, c;
} state;

/* coloring.hpp:139-156 (apply_move; the domain checks of 141-143 are the
 * caller's contract and hold by construction here) */
static void apply_move(state* s, int v, int to) {
    const int from = s->col[v];
    const int32_t* row = s->gamma + (size_t)v * s->w;
    s->f += (to == 0) - (from == 0);
    s->c += (to ? row[to] : 0) - (from ? row[from] : 0);
    s->col[v] = (uint16_t)to;
    const or_graph* g = s->g;
    for (int a = g->adj_off[v]; a < g->adj_off[v + 1]; ++a) {
        int32_t* r = s->gamma + (size_t)g->adj[a] * s->w;
        if (from) r[from] -= 1;
        if (to) r[to] += 1;
    }
}

/* partial.hpp:22-39: uncolor argmax gamma[v][col(v)] (strict >, lowest index) until c = 0 */
static void repair_state(state* s) {
    while (s->c > 0) {
        int worst = -1;
        int32_t wc = 0;
        for (int v = 0; v < s->g->nv; ++v) {
            const int k = s->col[v];
            if (!k) continue;
            const int32_t cnt = s->gamma[(size_t)v * s->w + k];
            if (cnt > wc) {
                wc = cnt;
                worst = v;
            }
        }
        apply_move(s, worst, 0);
    }
}

static void state_init(state* s, const or_graph* g, const uint16_t* colors) {
    s->g = g;
    s->w = g->n + 1;
    s->col = (uint16_t*)malloc(sizeof(uint16_t) * (g->nv + 1));
    memcpy(s->col, colors, sizeof(uint16_t) * g->nv);
    s->gamma = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->nv * s->w + 1));
    or_gamma_build(g, s->col, s->gamma);
    or_eval(g, s->col, &s->f, &s->c);
}

static void state_free(state* s) {
    free(s->col);
    free(s->gamma);
}

void or_repair(const or_graph* g, uint16_t* colors) {
    state s;
    state_init(&s, g, colors);
    repair_state(&s);
    memcpy(colors, s.col, sizeof(uint16_t) * g->nv);
    state_free(&s);
}

/* ------------------------------------------------------------ partialcol */

/* search_util.hpp:12-49 (IndexSet: erase swaps in the last element) */
typedef struct {
    int32_t* pos;
    int32_t* el;
    int size;
} indexset;

static void is_insert(indexset* x, int v) {
    if (x->pos[v] >= 0) return;
    x->pos[v] = x->size;
    x->el[x->size++] = v;
}

static void is_erase(indexset* x, int v) {
    const int p = x->pos[v];
    if (p < 0) return;
    const int last = x->el[x->size - 1];
    x->el[p] = last;
    x->pos[last] = p;
    x->size--;
    x->pos[v] = -1;
}

/* the state probe of the per-step parity contract: gamma (|V| x (n+1)) and the live tabu entries
   (until > j, colours kmin..n, (v, k) order) into probe point q */
static void probe_dump_state(const or_probe* probe, int q, const int32_t* gamma, const int64_t* until, int nv, int w,
                             int64_t j, int kmin) {
    memcpy(probe->gamma + (size_t)q * nv * w, gamma, sizeof(int32_t) * (size_t)nv * w);
    int cnt = 0;
    int32_t* tb = probe->tabu + (size_t)q * probe->cap * 3;
    for (int v = 0; v < nv; ++v)
        for (int k = kmin; k < w; ++k)
            if (until[(size_t)v * w + k] > j) {
                if (cnt < probe->cap) {
                    tb[3 * cnt] = v;
                    tb[3 * cnt + 1] = k;
                    tb[3 * cnt + 2] = (int32_t)until[(size_t)v * w + k];
                }
                ++cnt;
            }
    probe->n_tabu[q] = cnt;
    *probe->dumped = q + 1;
}

/* partial.hpp:76-169 + 8(d) byte counter.  Tabu state is fresh per call,
 * which equals the reference's skip_past reuse (partial.hpp:60) for alpha <= 1.
 * probe (optional): before each listed step j, the incremental gamma table
 * (coloring.hpp:139-156) and the live tabu entries until > j in (v, k) order
 * (search_util.hpp:69-75). */
static int improve_core(const or_graph* g, const uint16_t* input, uint16_t* out_best, uint64_t stream_seed,
                        int64_t budget, double alpha, int stop_f, int tie_mode, or_improve_stats* st,
                        or_step* trace, int64_t trace_cap, const or_probe* probe) {
    const int nv = g->nv;
    state s;
    state_init(&s, g, input);
    repair_state(&s);
    const int w = s.w;
    indexset un;
    un.pos = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    un.el = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    un.size = 0;
    for (int v = 0; v < nv; ++v) un.pos[v] = -1;
    for (int v = 0; v < nv; ++v)
        if (s.col[v] == 0) is_insert(&un, v);
    int64_t* until = (int64_t*)calloc((size_t)nv * w + 1, sizeof(int64_t));
    uint16_t* best = (uint16_t*)malloc(sizeof(uint16_t) * (nv + 1));
    memcpy(best, s.col, sizeof(uint16_t) * nv);
    int bestf = s.f;
    const int repaired_f = s.f;
    or_rng rng;
    or_rng_seed(&rng, stream_seed);
    double bytes = 0.0;

    int64_t it = 0;
    int probe_next = 0;
    if (probe) *probe->dumped = 0;
    while (it < budget && bestf > stop_f) {
        if (s.f == 0) break; /* step() returns false: not counted (partial.hpp:93, 163) */
        const int64_t j = it; /* tabu clock of this step's scan */
        if (probe && probe_next < probe->n && probe->steps[probe_next] == j)
            probe_dump_state(probe, probe_next++, s.gamma, until, nv, w, j, 1);
        const int f_before = s.f;
        int bv = -1, bk = 0, level = 2, nadm = 0;
        uint64_t x = 0;
        if (tie_mode == OR_TIE_REF) {
            /* partial.hpp:100-119 */
            int32_t bd = 0;
            uint64_t ties = 0;
            for (int idx = 0; idx < un.size; ++idx) {
                const int v = un.el[idx];
                const int32_t* row = s.gamma + (size_t)v * w;
                for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
                    const int k = g->dom[a];
                    if (!k) continue;
                    const int32_t d = -1 + row[k];
                    if (bv >= 0 && d > bd) continue;
                    const int asp = s.f + d < bestf;
                    if (!asp && until[(size_t)v * w + k] > j) continue;
                    if (bv < 0 || d < bd) {
                        bv = v;
                        bk = k;
                        bd = d;
                        ties = 1;
                    } else if (or_rng_below(&rng, ++ties) == 0) {
                        bv = v;
                        bk = k;
                    }
                }
            }
            if (bv >= 0) level = bd;
            nadm = (int)ties;
        } else {
            /* canonical rule: count admissible per level in ascending (v,k), pick the r-th */
            int cnt[3] = {0, 0, 0};
            for (int v = 0; v < nv; ++v) {
                if (s.col[v]) continue;
                const int32_t* row = s.gamma + (size_t)v * w;
                for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
                    const int k = g->dom[a];
                    if (!k) continue;
                    const int32_t d = -1 + row[k];
                    const int asp = s.f + d < bestf;
                    if (!asp && until[(size_t)v * w + k] > j) continue;
                    cnt[d + 1]++;
                }
            }
            x = or_canon_draw(stream_seed, (uint64_t)j);
            for (int lv = 0; lv < 3; ++lv)
                if (cnt[lv]) {
                    level = lv - 1;
                    nadm = cnt[lv];
                    break;
                }
            if (level != 2) {
                const uint32_t hi = (uint32_t)(x >> 32);
                int64_t r = (int64_t)(((uint64_t)hi * (uint64_t)nadm) >> 32);
                for (int v = 0; v < nv && bv < 0; ++v) {
                    if (s.col[v]) continue;
                    const int32_t* row = s.gamma + (size_t)v * w;
                    for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
                        const int k = g->dom[a];
                        if (!k) continue;
                        const int32_t d = -1 + row[k];
                        if (d != level) continue;
                        const int asp = s.f + d < bestf;
                        if (!asp && until[(size_t)v * w + k] > j) continue;
                        if (r == 0) {
                            bv = v;
                            bk = k;
                            break;
                        }
                        --r;
                    }
                }
            }
        }
        /* tick (partial.hpp:121) is implicit: the next scan uses clock j+1 */
        double bt = 2.0 * w * f_before;
        or_step rec;
        rec.step = j;
        rec.v = bv;
        rec.k = bk;
        rec.e = 0;
        rec.ev0 = rec.ev1 = -1;
        rec.f_before = f_before;
        rec.tenure = -1;
        rec.n_adm = nadm;
        rec.level = level;
        if (bv >= 0) {
            /* partial.hpp:124-141 */
            int ev[2] = {-1, -1}, e = 0;
            bt += 4.0 * (g->adj_off[bv + 1] - g->adj_off[bv]);
            apply_move(&s, bv, bk);
            is_erase(&un, bv);
            if (s.c > 0) {
                for (int a = g->adj_off[bv]; a < g->adj_off[bv + 1]; ++a) {
                    const int u = g->adj[a];
                    if (s.col[u] == bk) {
                        apply_move(&s, u, 0);
                        is_insert(&un, u);
                        if (e < 2) ev[e] = u;
                        ++e;
                        bt += 4.0 * (g->adj_off[u + 1] - g->adj_off[u]);
                    }
                }
            }
            const uint64_t lpart = (tie_mode == OR_TIE_REF)
                                       ? or_rng_below(&rng, 10)
                                       : ((uint64_t)(uint32_t)x * 10ULL) >> 32;
            const uint64_t tenure = lpart + (uint64_t)(alpha * (double)un.size);
            for (int q = 0; q < e && q < 2; ++q) until[(size_t)ev[q] * w + bk] = j + 1 + (int64_t)tenure;
            bt += 2.0 * (1 + e);
            if (s.f < bestf) {
                memcpy(best, s.col, sizeof(uint16_t) * nv);
                bestf = s.f;
                bt += 2.0 * nv;
            }
            rec.e = e;
            rec.ev0 = ev[0];
            rec.ev1 = ev[1];
            rec.tenure = (int32_t)tenure;
        }
        rec.f_after = s.f;
        rec.best_f = bestf;
        bytes += bt;
        if (trace && j < trace_cap) trace[j] = rec;
        ++it;
    }
    if (out_best) memcpy(out_best, best, sizeof(uint16_t) * nv);
    if (st) {
        st->iterations = it;
        st->repaired_f = repaired_f;
        st->best_f = bestf;
        st->alg_bytes = bytes;
    }
    free(un.pos);
    free(un.el);
    free(until);
    free(best);
    state_free(&s);
    return 0;
}

int or_improve(const or_graph* g, const uint16_t* input, uint16_t* out_best, uint64_t stream_seed,
               int64_t budget, double alpha, int stop_f, int tie_mode, or_improve_stats* st,
               or_step* trace, int64_t trace_cap) {
    return improve_core(g, input, out_best, stream_seed, budget, alpha, stop_f, tie_mode, st, trace, trace_cap,
                        NULL);
}

int or_improve_probe(const or_graph* g, const uint16_t* input, uint64_t stream_seed, int64_t budget, double alpha,
                     int stop_f, int tie_mode, const or_probe* probe) {
    return improve_core(g, input, NULL, stream_seed, budget, alpha, stop_f, tie_mode, NULL, NULL, 0, probe);
}


/* ----------------------------------------------------------------- plits */

typedef struct {
    const or_graph* g;
    state s;
    indexset un, cf;   /* uncoloured / conflicting sets (plits.hpp:74-75), REF iteration order */
    int64_t* until;    /* phase-local tabu clock: until > j <=> tabu at step j */
    int64_t wf, wc;
} plits_phase_state;

/* plits.hpp:193-212 update_membership_around */
static void plits_membership(plits_phase_state* ps, int v, int from, int to) {
    const or_graph* g = ps->g;
    const int w = ps->s.w;
    if (from == 0) is_erase(&ps->un, v);
    if (to == 0) {
        is_insert(&ps->un, v);
        is_erase(&ps->cf, v);
    } else if (ps->s.gamma[(size_t)v * w + to] > 0) {
        is_insert(&ps->cf, v);
    } else {
        is_erase(&ps->cf, v);
    }
    for (int a = g->adj_off[v]; a < g->adj_off[v + 1]; ++a) {
        const int u = g->adj[a];
        const int cu = ps->s.col[u];
        if (cu == 0 || (cu != from && cu != to)) continue;
        if (ps->s.gamma[(size_t)u * w + cu] > 0)
            is_insert(&ps->cf, u);
        else
            is_erase(&ps->cf, u);
    }
}

/* plits.hpp:255-270 detail::run_phase with PlitsSearch (96-191) inlined.
 * col is the phase input and receives search.best(). Returns hit_target. */
static int plits_phase(const or_graph* g, uint16_t* col, int phase, int64_t wf, int64_t wc, int64_t budget,
                       double alpha, int stop_f, int tie_mode, or_rng* rng, uint64_t seed, int64_t* J,
                       int64_t* iters, double* bytes, or_plits_step* trace, int64_t trace_cap,
                       const or_probe* probe, int* probe_next) {
    const int nv = g->nv;
    plits_phase_state ps;
    ps.g = g;
    ps.wf = wf;
    ps.wc = wc;
    state_init(&ps.s, g, col);
    const int w = ps.s.w;
    ps.un.pos = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    ps.un.el = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    ps.cf.pos = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    ps.cf.el = (int32_t*)malloc(sizeof(int32_t) * (nv + 1));
    ps.un.size = ps.cf.size = 0;
    for (int v = 0; v < nv; ++v) ps.un.pos[v] = ps.cf.pos[v] = -1;
    /* plits.hpp:109-115 */
    for (int v = 0; v < nv; ++v) {
        const int k = ps.s.col[v];
        if (k == 0)
            is_insert(&ps.un, v);
        else if (ps.s.gamma[(size_t)v * w + k] > 0)
            is_insert(&ps.cf, v);
    }
    /* fresh tabu per phase == PlitsScratch::prepare's skip_past(16 + 2|V|) (plits.hpp:81)
       whenever every tenure 9 + alpha*active stays below 17 + 2|V| (alpha < 2) */
    ps.until = (int64_t*)calloc((size_t)nv * w + 1, sizeof(int64_t));
    uint16_t* best = (uint16_t*)malloc(sizeof(uint16_t) * (nv + 1));
    memcpy(best, ps.s.col, sizeof(uint16_t) * nv);
    int best_f = ps.s.f, best_c = ps.s.c;
    int64_t best_scaled = wf * ps.s.f + wc * ps.s.c;
    int64_t it = 0;
    int hit = 0;
    while (it < budget) {
        if (best_c == 0 && best_f <= stop_f) {
            hit = 1;
            break;
        }
        if (ps.un.size == 0 && ps.cf.size == 0) break; /* StepResult::Exhausted, not counted */
        const int64_t j = it;                           /* tabu clock of this step's scan */
        /* probe points are keyed by the step index over both phases; tabu entries on the phase clock */
        if (probe && *probe_next < probe->n && probe->steps[*probe_next] == *J)
            probe_dump_state(probe, (*probe_next)++, ps.s.gamma, ps.until, nv, w, j, 0);
        const int64_t cur_scaled = wf * ps.s.f + wc * ps.s.c;
        int bv = -1, bk = 0, bdf = 0, bdc = 0;
        int64_t bd = 0;
        int64_t nadm = 0;
        uint64_t x = 0;
        double bt = 2.0 * w * (ps.un.size + ps.cf.size);
        if (tie_mode == OR_TIE_REF) {
            /* plits.hpp:135-176: uncoloured set, then conflicting set, each in IndexSet order */
            uint64_t ties = 0;
            for (int pass = 0; pass < 2; ++pass) {
                const indexset* set = pass == 0 ? &ps.un : &ps.cf;
                for (int idx = 0; idx < set->size; ++idx) {
                    const int v = set->el[idx];
                    const int cur = ps.s.col[v];
                    const int32_t* row = ps.s.gamma + (size_t)v * w;
                    for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
                        const int k = g->dom[a];
                        if (pass == 0 ? (k == 0) : (k == cur)) continue;
                        const int df = (k == 0) - (cur == 0);
                        const int dc = (k ? row[k] : 0) - (cur ? row[cur] : 0);
                        const int64_t d = wf * df + wc * dc;
                        if (bv >= 0 && d > bd) continue;
                        if (ps.until[(size_t)v * w + k] > j && cur_scaled + d >= best_scaled) continue;
                        if (bv < 0 || d < bd) {
                            bv = v, bk = k, bdf = df, bdc = dc, bd = d;
                            ties = 1;
                        } else if (or_rng_below(rng, ++ties) == 0) {
                            bv = v, bk = k, bdf = df, bdc = dc;
                        }
                    }
                }
            }
            nadm = (int64_t)ties;
        } else {
            /* canonical rule: minimum admissible delta, count N, the r-th in ascending (v, k) */
            int64_t dmin = INT64_MAX;
            for (int pass = 0; pass < 2; ++pass) {
                int64_t r = 0;
                if (pass == 1) {
                    if (nadm == 0) break;
                    x = or_canon_draw(seed, (uint64_t)*J);
                    r = (int64_t)(((x >> 32) * (uint64_t)nadm) >> 32);
                }
                for (int v = 0; v < nv && bv < 0; ++v) {
                    const int cur = ps.s.col[v];
                    const int32_t* row = ps.s.gamma + (size_t)v * w;
                    if (cur != 0 && row[cur] == 0) continue; /* not in the neighbourhood (plits.hpp:47-63) */
                    for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
                        const int k = g->dom[a];
                        if (k == cur) continue;
                        const int df = (k == 0) - (cur == 0);
                        const int dc = (k ? row[k] : 0) - (cur ? row[cur] : 0);
                        const int64_t d = wf * df + wc * dc;
                        if (ps.until[(size_t)v * w + k] > j && cur_scaled + d >= best_scaled) continue;
                        if (pass == 0) {
                            if (d < dmin) {
                                dmin = d;
                                nadm = 1;
                            } else if (d == dmin) {
                                ++nadm;
                            }
                        } else if (d == dmin) {
                            if (r == 0) {
                                bv = v, bk = k, bdf = df, bdc = dc, bd = d;
                                break;
                            }
                            --r;
                        }
                    }
                }
            }
        }
        /* tick (plits.hpp:178): the next scan uses clock j+1 */
        or_plits_step rec;
        memset(&rec, 0, sizeof(rec));
        rec.step = *J;
        rec.phase = phase;
        rec.v = bv;
        rec.k = bk;
        rec.from = bv >= 0 ? ps.s.col[bv] : 0;
        rec.n_adm = (int32_t)nadm;
        rec.tenure = -1;
        if (bv >= 0) {
            const int from = ps.s.col[bv];
            apply_move(&ps.s, bv, bk);
            plits_membership(&ps, bv, from, bk);
            const uint64_t active = (uint64_t)ps.un.size + (uint64_t)ps.cf.size;
            const uint64_t lpart = (tie_mode == OR_TIE_REF) ? or_rng_below(rng, 10)
                                                            : (((uint64_t)(uint32_t)x * 10ULL) >> 32);
            const uint64_t tenure = lpart + (uint64_t)(alpha * (double)active);
            ps.until[(size_t)bv * w + from] = j + 1 + (int64_t)tenure;
            const int64_t now = cur_scaled + bd;
            bt += 4.0 * (g->adj_off[bv + 1] - g->adj_off[bv]) + 2.0;
            if (now < best_scaled) {
                best_scaled = now;
                memcpy(best, ps.s.col, sizeof(uint16_t) * nv);
                best_f = ps.s.f;
                best_c = ps.s.c;
                bt += 2.0 * nv;
            }
            rec.df = bdf;
            rec.dc = bdc;
            rec.delta = bd;
            rec.tenure = (int32_t)tenure;
        }
        rec.cur_scaled = wf * ps.s.f + wc * ps.s.c;
        rec.best_scaled = best_scaled;
        rec.active = ps.un.size + ps.cf.size;
        rec.f = ps.s.f;
        rec.c = ps.s.c;
        if (trace && *J < trace_cap) trace[*J] = rec;
        *bytes += bt;
        ++it;
        ++*J;
    }
    if (best_c == 0 && best_f <= stop_f) hit = 1;
    memcpy(col, best, sizeof(uint16_t) * nv);
    *iters += it;
    free(best);
    free(ps.until);
    free(ps.un.pos);
    free(ps.un.el);
    free(ps.cf.pos);
    free(ps.cf.el);
    state_free(&ps.s);
    return hit;
}

/* plits.hpp:276-292 plits_run */
static int plits_core(const or_graph* g, const uint16_t* input, uint16_t* out, uint64_t stream_seed, int64_t iters1,
                      int64_t iters2, double alpha, int stop_f, int tie_mode, or_plits_stats* st,
                      or_plits_step* trace, int64_t trace_cap, const or_probe* probe) {
    int probe_next = 0;
    if (probe) *probe->dumped = 0;
    const int nv = g->nv;
    or_plits_stats z;
    memset(&z, 0, sizeof(z));
    if (nv == 0) {
        if (st) *st = z;
        return 0;
    }
    if (iters1 <= 0) iters1 = 100LL * nv;
    if (iters2 <= 0) iters2 = 2LL * nv;
    uint16_t* col = (uint16_t*)malloc(sizeof(uint16_t) * (nv + 1));
    memcpy(col, input, sizeof(uint16_t) * nv);
    or_rng rng;
    or_rng_seed(&rng, stream_seed);
    int64_t J = 0, iters = 0;
    double bytes = 0;
    const int done = plits_phase(g, col, 1, 2, 1, iters1, alpha, stop_f, tie_mode, &rng, stream_seed, &J, &iters,
                                 &bytes, trace, trace_cap, probe, &probe_next);
    z.phase1_iterations = iters;
    z.hit_target = done;
    if (!done)
        plits_phase(g, col, 2, 2, 2LL * nv, iters2, alpha, stop_f, tie_mode, &rng, stream_seed, &J, &iters, &bytes,
                    trace, trace_cap, probe, &probe_next);
    int f, c;
    or_eval(g, col, &f, &c);
    if (c > 0) {
        or_repair(g, col);
        or_eval(g, col, &f, &c);
        z.repaired = 1;
        bytes += 2.0 * nv;
    }
    if (out) memcpy(out, col, sizeof(uint16_t) * nv);
    z.iterations = iters;
    z.final_f = f;
    z.alg_bytes = bytes;
    if (st) *st = z;
    free(col);
    return 0;
}

int or_plits(const or_graph* g, const uint16_t* input, uint16_t* out, uint64_t stream_seed, int64_t iters1,
             int64_t iters2, double alpha, int stop_f, int tie_mode, or_plits_stats* st,
             or_plits_step* trace, int64_t trace_cap) {
    return plits_core(g, input, out, stream_seed, iters1, iters2, alpha, stop_f, tie_mode, st, trace, trace_cap,
                      NULL);
}

/* the state probe of or_plits: before each listed step J (counted over both phases) the gamma table and
   the live tabu entries (v, k >= 0, until) on the phase's own clock (plits.hpp:81: a fresh table per phase) */
int or_plits_probe(const or_graph* g, const uint16_t* input, uint64_t stream_seed, int64_t iters1, int64_t iters2,
                   double alpha, int stop_f, int tie_mode, const or_probe* probe) {
    return plits_core(g, input, NULL, stream_seed, iters1, iters2, alpha, stop_f, tie_mode, NULL, NULL, 0, probe);
}


/* ---------------------------------------------------------------- exact */

typedef struct {
    const or_graph* g;
    int64_t budget, nodes;
    int exhausted, best_f, prune;
    int16_t* assign;
    int32_t* used; /* [nv][n+1]: neighbours of v coloured k */
    int16_t* best;
} exact_state;

static void exact_adjust(exact_state* x, int v, int k, int d) {
    if (k == 0) return;
    const or_graph* g = x->g;
    for (int a = g->adj_off[v]; a < g->adj_off[v + 1]; ++a) x->used[(size_t)g->adj[a] * (g->n + 1) + k] += d;
}

/* oracle.hpp:64-119 ExactSolver::descend */
static void exact_descend(exact_state* x, int zeros) {
    const or_graph* g = x->g;
    if (x->exhausted) return;
    if (++x->nodes > x->budget) {
        x->exhausted = 1;
        return;
    }
    int pick = -1, pick_feasible = 0, forced = 0;
    for (int v = 0; v < g->nv; ++v) {
        if (x->assign[v] != -1) continue;
        int feasible = 0;
        for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a)
            if (g->dom[a] != 0 && x->used[(size_t)v * (g->n + 1) + g->dom[a]] == 0) ++feasible;
        if (feasible == 0) {
            ++forced;
            continue;
        }
        if (pick < 0 || feasible < pick_feasible) {
            pick = v;
            pick_feasible = feasible;
        }
    }
    if (x->prune && zeros + forced >= x->best_f) return;
    if (pick < 0) {
        const int f = zeros + forced;
        if (f < x->best_f) {
            x->best_f = f;
            for (int v = 0; v < g->nv; ++v) x->best[v] = x->assign[v] == -1 ? 0 : x->assign[v];
        }
        return;
    }
    for (int a = g->dom_off[pick]; a < g->dom_off[pick + 1]; ++a) {
        const int k = g->dom[a];
        if (k == 0 || x->used[(size_t)pick * (g->n + 1) + k] != 0) continue;
        x->assign[pick] = (int16_t)k;
        exact_adjust(x, pick, k, +1);
        exact_descend(x, zeros);
        exact_adjust(x, pick, k, -1);
        if (x->exhausted) break;
    }
    if (!x->exhausted) {
        x->assign[pick] = 0;
        exact_descend(x, zeros + 1);
    }
    x->assign[pick] = -1;
}

int or_solve_exact(const or_graph* g, int64_t node_budget, or_exact_result* res, uint16_t* certificate) {
    exact_state x;
    memset(&x, 0, sizeof(x));
    x.g = g;
    x.budget = node_budget;
    x.prune = 1;
    x.best_f = g->nv;
    x.assign = (int16_t*)malloc(sizeof(int16_t) * (g->nv + 1));
    x.best = (int16_t*)calloc((size_t)g->nv + 1, sizeof(int16_t));
    x.used = (int32_t*)calloc((size_t)g->nv * (g->n + 1) + 1, sizeof(int32_t));
    for (int v = 0; v < g->nv; ++v) x.assign[v] = -1;
    exact_descend(&x, 0);
    res->optimum_f = x.best_f;
    res->exact = !x.exhausted;
    res->nodes = x.nodes;
    for (int v = 0; v < g->nv; ++v) certificate[v] = (uint16_t)x.best[v];
    free(x.assign);
    free(x.best);
    free(x.used);
    return 0;
}

/* oracle.hpp:141-177 enumerate_exact */
static void enum_rec(const or_graph* g, int v, int zeros, uint16_t* asg, uint16_t* best, int* best_f, int64_t* nodes) {
    ++*nodes;
    if (v == g->nv) {
        if (zeros < *best_f) {
            *best_f = zeros;
            memcpy(best, asg, sizeof(uint16_t) * g->nv);
        }
        return;
    }
    for (int a = g->dom_off[v]; a < g->dom_off[v + 1]; ++a) {
        const int k = g->dom[a];
        if (k != 0) {
            int ok = 1;
            for (int b = g->adj_off[v]; b < g->adj_off[v + 1] && ok; ++b)
                if (g->adj[b] < v && asg[g->adj[b]] == k) ok = 0;
            if (!ok) continue;
        }
        asg[v] = (uint16_t)k;
        enum_rec(g, v + 1, zeros + (k == 0), asg, best, best_f, nodes);
    }
    asg[v] = 0;
}

int or_enumerate_exact(const or_graph* g, or_exact_result* res, uint16_t* certificate) {
    uint16_t* asg = (uint16_t*)calloc((size_t)g->nv + 1, sizeof(uint16_t));
    uint16_t* best = (uint16_t*)calloc((size_t)g->nv + 1, sizeof(uint16_t));
    int best_f = g->nv + 1;
    int64_t nodes = 0;
    enum_rec(g, 0, 0, asg, best, &best_f, &nodes);
    res->optimum_f = best_f;
    res->exact = 1;
    res->nodes = nodes;
    memcpy(certificate, best, sizeof(uint16_t) * g->nv);
    free(asg);
    free(best);
    return 0;
}

/* ----------------------------------------------------------- population */

/* population.hpp:41-61 */
void or_cross_distances(int nv, int p, const uint16_t* members, const uint16_t* improved,
                        int32_t* cross, int32_t* fresh) {
    for (int i = 0; i < p; ++i) {
        for (int j = 0; j < p; ++j)
            cross[(size_t)i * p + j] = or_hamming(nv, members + (size_t)i * nv, improved + (size_t)j * nv);
        fresh[(size_t)i * p + i] = 0;
        for (int j = i + 1; j < p; ++j)
            fresh[(size_t)i * p + j] = or_hamming(nv, improved + (size_t)i * nv, improved + (size_t)j * nv);
    }
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < i; ++j) fresh[(size_t)i * p + j] = fresh[(size_t)j * p + i];
}

/* population.hpp:76-87 */
void or_full_distances(int nv, int p, const uint16_t* members, int32_t* dist) {
    for (int i = 0; i < p; ++i) {
        dist[(size_t)i * p + i] = 0;
        for (int j = i + 1; j < p; ++j)
            dist[(size_t)i * p + j] = or_hamming(nv, members + (size_t)i * nv, members + (size_t)j * nv);
    }
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < i; ++j) dist[(size_t)i * p + j] = dist[(size_t)j * p + i];
}

typedef struct {
    int illegal, f, id;
} pool_key;

static int cmp_key(const void* a, const void* b) {
    const pool_key* x = (const pool_key*)a;
    const pool_key* y = (const pool_key*)b;
    if (x->illegal != y->illegal) return x->illegal - y->illegal;
    if (x->f != y->f) return x->f - y->f;
    return x->id - y->id;
}

/* population.hpp:103-183, with the island exchange's migrants as extra pool candidates:
   pool ids 0..p-1 members, p..2p-1 improved, 2p..2p+m-1 migrants; a migrant's distances are Hamming
   distances computed here (coloring.hpp:159-167).  m = 0 is the reference's update exactly. */
int or_update_ex(const or_graph* g, int p, double spacing_gamma, uint16_t* members, int32_t* dist,
                 const uint16_t* improved, const int32_t* cross, const int32_t* fresh, int m,
                 const uint16_t* migrants, int32_t* pool_best_f, int32_t* shortfall_slots,
                 int32_t* n_shortfall, int32_t* selected_ids) {
    const int nv = g->nv;
    const double threshold = nv / spacing_gamma;
    const int pool = 2 * p + m;
    pool_key* keys = (pool_key*)malloc(sizeof(pool_key) * pool);
    int* legal = (int*)malloc(sizeof(int) * pool);
    int* fval = (int*)calloc(pool, sizeof(int));
#define ROW(id)                                                   \
    ((id) < p       ? members + (size_t)(id) * nv                 \
     : (id) < 2 * p ? improved + (size_t)((id) - p) * nv          \
                    : migrants + (size_t)((id) - 2 * p) * nv)
    for (int id = 0; id < pool; ++id) {
        int f, cc;
        or_eval(g, ROW(id), &f, &cc);
        legal[id] = cc == 0;
        fval[id] = f;
        keys[id].illegal = cc == 0 ? 0 : 1;
        keys[id].f = f;
        keys[id].id = id;
    }
    qsort(keys, pool, sizeof(pool_key), cmp_key);
#define PD(a, b)                                                                          \
    ((a) == (b) ? 0                                                                       \
     : ((a) >= 2 * p || (b) >= 2 * p) ? or_hamming(nv, ROW(a), ROW(b))                    \
     : ((a) < p && (b) < p)   ? dist[(size_t)(a) * p + (b)]                               \
     : ((a) >= p && (b) >= p) ? fresh[(size_t)((a) - p) * p + ((b) - p)]                  \
     : ((a) < p)              ? cross[(size_t)(a) * p + ((b) - p)]                        \
                              : cross[(size_t)(b) * p + ((a) - p)])
    *pool_best_f = fval[keys[0].id];
    int* sel = (int*)malloc(sizeof(int) * p);
    int* skipped = (int*)malloc(sizeof(int) * pool);
    int ns = 0, nk = 0;
    sel[ns++] = keys[0].id;
    for (int k = 1; k < pool && ns < p; ++k) {
        const int cnd = keys[k].id;
        if (!legal[cnd]) {
            skipped[nk++] = cnd;
            continue;
        }
        int32_t md = 0x7fffffff;
        for (int q = 0; q < ns; ++q) {
            const int32_t d = PD(cnd, sel[q]);
            if (d < md) md = d;
        }
        if ((double)md > threshold)
            sel[ns++] = cnd;
        else
            skipped[nk++] = cnd;
    }
    int nsf = 0;
    for (int k = 0; k < nk && ns < p; ++k) {
        shortfall_slots[nsf++] = ns;
        sel[ns++] = skipped[k];
    }
    *n_shortfall = nsf;
    int32_t* nd = (int32_t*)malloc(sizeof(int32_t) * (size_t)p * p);
    for (int i = 0; i < p; ++i) {
        nd[(size_t)i * p + i] = 0;
        for (int j = i + 1; j < p; ++j) {
            const int32_t d = PD(sel[i], sel[j]);
            nd[(size_t)i * p + j] = d;
            nd[(size_t)j * p + i] = d;
        }
    }
#undef PD
    uint16_t* nm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)p * nv);
    for (int i = 0; i < p; ++i) {
        const int id = sel[i];
        memcpy(nm + (size_t)i * nv, ROW(id), sizeof(uint16_t) * nv);
        if (selected_ids) selected_ids[i] = id;
    }
#undef ROW
    memcpy(members, nm, sizeof(uint16_t) * (size_t)p * nv);
    memcpy(dist, nd, sizeof(int32_t) * (size_t)p * p);
    free(nm);
    free(nd);
    free(sel);
    free(skipped);
    free(keys);
    free(legal);
    free(fval);
    return 0;
}

/* population.hpp:103-183 */
int or_update(const or_graph* g, int p, double spacing_gamma, uint16_t* members, int32_t* dist,
              const uint16_t* improved, const int32_t* cross, const int32_t* fresh,
              int32_t* pool_best_f, int32_t* shortfall_slots, int32_t* n_shortfall,
              int32_t* selected_ids) {
    return or_update_ex(g, p, spacing_gamma, members, dist, improved, cross, fresh, 0, NULL, pool_best_f,
                        shortfall_slots, n_shortfall, selected_ids);
}

/* population.hpp:209-228 (excl: p*p bytes, slot-keyed; NULL = no exclusion) */
int or_nearest_neighbor(int p, const int32_t* dist, int i, uint8_t* excl) {
    int best = -1, bu = -1;
    const int32_t* row = dist + (size_t)i * p;
    for (int j = 0; j < p; ++j) {
        if (j == i) continue;
        const int32_t d = row[j];
        if (bu < 0 || d < row[bu]) bu = j;
        if (excl && excl[(size_t)i * p + j]) continue;
        if (best < 0 || d < row[best]) best = j;
    }
    if (best < 0) {
        memset(excl + (size_t)i * p, 0, p);
        return bu;
    }
    return best;
}

/* crossover.hpp:54-104 (+ mixing_probability 26-30, aux_crossover 34-46) */
int or_offspring(const or_graph* g, int p, const uint16_t* members, const int32_t* dist,
                 int crossover, double beta, int matching, int exclusion, uint8_t* excl,
                 uint64_t master_seed, uint64_t generation, uint16_t* offspring, int32_t* partner) {
    return or_offspring_ex(g, p, members, dist, crossover, beta, matching, exclusion, excl, master_seed,
                           generation * (uint64_t)p, offspring, partner);
}

/* island form: stream index = stream_base + i (stream_base = gen*p_total + offset) */
int or_offspring_ex(const or_graph* g, int p, const uint16_t* members, const int32_t* dist,
                    int crossover, double beta, int matching, int exclusion, uint8_t* excl,
                    uint64_t master_seed, uint64_t stream_base, uint16_t* offspring, int32_t* partner) {
    const int nv = g->nv;
    if (crossover == OR_X_NONE) {
        memcpy(offspring, members, sizeof(uint16_t) * (size_t)p * nv);
        if (partner)
            for (int i = 0; i < p; ++i) partner[i] = -1;
        return 0;
    }
    int* part = (int*)malloc(sizeof(int) * p);
    for (int i = 0; i < p; ++i) {
        int j;
        if (matching == OR_M_RANDOM) {
            or_rng m;
            or_rng_seed(&m, or_derive_seed(master_seed, 6, stream_base + (uint64_t)i));
            j = (int)or_rng_below(&m, (uint64_t)(p - 1));
            if (j >= i) ++j;
        } else {
            j = or_nearest_neighbor(p, dist, i, exclusion == OR_E_OFF ? NULL : excl);
        }
        if (exclusion != OR_E_OFF) excl[(size_t)i * p + j] = 1;
        part[i] = j;
    }
    for (int i = 0; i < p; ++i) {
        or_rng st;
        or_rng_seed(&st, or_derive_seed(master_seed, 3, stream_base + (uint64_t)i));
        const uint16_t* first = members + (size_t)i * nv;
        const uint16_t* second = members + (size_t)part[i] * nv;
        uint16_t* child = offspring + (size_t)i * nv;
        double pij = 0.5;
        if (crossover == OR_X_AUX) {
            const int32_t d = dist[(size_t)i * p + part[i]];
            if ((double)d * beta <= (double)nv) {
                memcpy(child, first, sizeof(uint16_t) * nv);
                continue;
            }
            pij = 1.0 - (double)nv / (beta * (double)d);
        }
        for (int v = 0; v < nv; ++v) child[v] = (or_rng_double(&st) < pij) ? first[v] : second[v];
    }
    if (partner)
        for (int i = 0; i < p; ++i) partner[i] = part[i];
    free(part);
    return 0;
}

/* engine.hpp:88-106 (distances are separate: or_full_distances) */
void or_init_population(const or_graph* g, int p, uint64_t master_seed, uint16_t* members) {
    or_init_population_ex(g, p, master_seed, 0, members);
}

void or_init_population_ex(const or_graph* g, int p, uint64_t master_seed, uint64_t offset, uint16_t* members) {
    const int nv = g->nv;
    for (int i = 0; i < p; ++i) {
        or_rng r;
        or_rng_seed(&r, or_derive_seed(master_seed, 1, offset + (uint64_t)i));
        for (int v = 0; v < nv; ++v) {
            const int begin = g->dom_off[v] + 1;
            const int choices = g->dom_off[v + 1] - begin;
            members[(size_t)i * nv + v] = g->dom[begin + (int)or_rng_below(&r, (uint64_t)choices)];
        }
    }
}

/* ---------------------------------------------------------------- engine */

/* engine.hpp:76-84 */
static int is_optimal_fc(int f, int c, int l) {
    if (c != 0) return 0;
    return (f == 0 && l != 1) || (f == 1 && l == 1);
}

/* engine.hpp:114-262, partial variant, no wall-clock limit */
int or_run(int n, const uint16_t* grid, const or_config* cfg, or_result* res, uint16_t* best_colors,
           or_gen_log* log, int64_t log_cap) {
    or_graph* g = or_preprocess(n, grid);
    const int nv = g->nv, p = cfg->p;
    memset(res, 0, sizeof(*res));
    res->l = g->l;
    res->upper_bound = (g->l == 1) ? n * n - 2 : n * n - g->l;
    res->vertex_count = nv;
    uint16_t* best = (uint16_t*)calloc((size_t)nv + 1, sizeof(uint16_t));
    res->best_f = nv;
    const int target_f = g->l == 1 ? 1 : 0;
    int reason = OR_STOP_TRIVIAL;
    if (nv == 0) {
        res->best_f = 0;
        goto finalize;
    }
    {
        uint16_t* members = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)p * nv);
        uint16_t* offspring = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)p * nv);
        uint16_t* improved = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)p * nv);
        int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * (size_t)p * p);
        int32_t* cross = (int32_t*)malloc(sizeof(int32_t) * (size_t)p * p);
        int32_t* fresh = (int32_t*)malloc(sizeof(int32_t) * (size_t)p * p);
        uint8_t* excl = (uint8_t*)calloc((size_t)p * p, 1);
        int32_t* sfs = (int32_t*)malloc(sizeof(int32_t) * p);
        or_init_population(g, p, cfg->master_seed, members);
        or_full_distances(nv, p, members, dist);
        for (int i = 0; i < p; ++i) {
            int f, c;
            or_eval(g, members + (size_t)i * nv, &f, &c);
            if (c == 0 && f < res->best_f) {
                res->best_f = f;
                memcpy(best, members + (size_t)i * nv, sizeof(uint16_t) * nv);
            }
        }
        {
            int f, c;
            or_eval(g, best, &f, &c);
            if (!cfg->disable_optimal_stop && is_optimal_fc(f, c, g->l)) {
                reason = OR_STOP_OPTIMAL;
                goto done;
            }
        }
        memcpy(offspring, members, sizeof(uint16_t) * (size_t)p * nv);
        const int64_t budget = cfg->phase1_iters > 0 ? cfg->phase1_iters : 100LL * nv;
        int64_t nlog = 0;
        for (int64_t gen = 1;; ++gen) {
            for (int i = 0; i < p; ++i) {
                const uint64_t sd = or_derive_seed(cfg->master_seed, 2, (uint64_t)gen * p + i);
                if (cfg->variant == 0) {
                    or_plits_stats ps;
                    or_plits(g, offspring + (size_t)i * nv, improved + (size_t)i * nv, sd, cfg->phase1_iters,
                             cfg->phase2_iters, cfg->alpha, target_f, cfg->tie_mode, &ps, NULL, 0);
                    res->total_iterations += ps.iterations;
                } else {
                    or_improve_stats st;
                    or_improve(g, offspring + (size_t)i * nv, improved + (size_t)i * nv, sd, budget, cfg->alpha,
                               target_f, cfg->tie_mode, &st, NULL, 0);
                    res->total_iterations += st.iterations;
                }
            }
            res->generations = gen;
            for (int i = 0; i < p; ++i) {
                int f, c;
                or_eval(g, improved + (size_t)i * nv, &f, &c);
                if (f < res->best_f) {
                    res->best_f = f;
                    memcpy(best, improved + (size_t)i * nv, sizeof(uint16_t) * nv);
                }
            }
            const int optimal = !cfg->disable_optimal_stop && is_optimal_fc(res->best_f, 0, g->l);
            const int iters_up = cfg->iteration_limit > 0 && res->total_iterations >= cfg->iteration_limit;
            const int gens_up = cfg->generation_limit > 0 && gen >= cfg->generation_limit;
            int32_t pbf = 0, nsf = 0;
            if (!(optimal || iters_up || gens_up)) {
                or_cross_distances(nv, p, members, improved, cross, fresh);
                or_update(g, p, cfg->gamma, members, dist, improved, cross, fresh, &pbf, sfs, &nsf, NULL);
                if (cfg->exclusion == OR_E_GENERATION) memset(excl, 0, (size_t)p * p);
                or_offspring(g, p, members, dist, cfg->crossover, cfg->beta, cfg->matching, cfg->exclusion,
                             excl, cfg->master_seed, (uint64_t)gen, offspring, NULL);
            }
            if (log && nlog < log_cap) {
                log[nlog].generation = gen;
                log[nlog].best_f = res->best_f;
                log[nlog].shortfall = nsf;
                log[nlog].iterations = res->total_iterations;
                /* engine.hpp:219-225: f over members, distance over i < j */
                double f_sum = 0, d_sum = 0;
                for (int i = 0; i < p; ++i) {
                    int f, c;
                    or_eval(g, members + (size_t)i * nv, &f, &c);
                    f_sum += f;
                    for (int j = i + 1; j < p; ++j) d_sum += dist[(size_t)i * p + j];
                }
                log[nlog].mean_f = f_sum / p;
                log[nlog].mean_distance = d_sum / (0.5 * p * (p - 1));
                ++nlog;
            }
            if (optimal || iters_up || gens_up) {
                reason = optimal ? OR_STOP_OPTIMAL : iters_up ? OR_STOP_ITERS : OR_STOP_GENS;
                break;
            }
        }
    done:
        free(members);
        free(offspring);
        free(improved);
        free(dist);
        free(cross);
        free(fresh);
        free(excl);
        free(sfs);
    }
finalize:
    res->best_score = n * n - g->l - res->best_f;
    {
        int f, c;
        or_eval(g, best, &f, &c);
        res->proven_optimal = is_optimal_fc(f, c, g->l);
    }
    res->stop_reason = res->proven_optimal ? OR_STOP_OPTIMAL : reason;
    if (best_colors) memcpy(best_colors, best, sizeof(uint16_t) * nv);
    free(best);
    or_graph_free(g);
    return 0;
}
