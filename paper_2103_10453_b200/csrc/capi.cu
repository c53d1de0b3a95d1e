// capi.cu -- the C ABI (include/plse_b200.h): device context, buffer
// management, the host halves of the population phases, and plse_solve, the
// generational driver that mirrors engine.hpp:114-262 on top of the kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "device_api.h"
#include "host_internal.h"
#include "plse_b200.h"

using namespace plse_dev;

namespace plse_dev {
cudaError_t set_plits_list_cap(int cap, cudaStream_t st);  // plits.cu: the instrumented kernel's list capacity
// population.cu: u16 host-format rows <-> u8 device rows, with the domain check
cudaError_t launch_unpack_colors(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad, int n, int W,
                                 const uint16_t* cell, const uint64_t* pr, const uint64_t* pc, int* bad,
                                 cudaStream_t st);
cudaError_t launch_pack_colors(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad, cudaStream_t st);
}

namespace {

thread_local std::string g_last_error;

// NVTX range per phase (header-only NVTX v3: no library dependency; a no-op without a tool attached), so
// ncu --nvtx / any NVTX-aware profiler can attribute the generation's kernels to run()'s phases
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// run()'s deadline on the device clock: now + remaining (engine.hpp:148-151)
__global__ void k_set_deadline(unsigned long long* deadline, unsigned long long remaining_ns) {
    *deadline = globaltimer_ns() + remaining_ns;
}

// sum of dist(i, j) over i < j (engine.hpp:222-225)
__global__ void k_upper_sum(const uint16_t* __restrict__ d, int p, unsigned long long* out) {
    unsigned long long s = 0;
    for (int i = blockIdx.x; i < p; i += gridDim.x)
        for (int j = i + 1 + threadIdx.x; j < p; j += blockDim.x) s += d[(size_t)i * p + j];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e__ = (x);                                                                  \
        if (e__ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e__)); \
    } while (0)

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct plse_ctx {
    int device = 0, nsm = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int n = 0, nv = 0, nvpad = 0, W = 1, lane_words = 1, l = 0;
    plse_params prm{};
    int64_t budget = 0;
    int stop_f = 0;
    // graph
    uint16_t *d_cell = nullptr, *d_rs = nullptr, *d_cs = nullptr, *d_cl = nullptr;
    uint64_t *d_pr = nullptr, *d_pc = nullptr, *d_below = nullptr;
    int32_t* d_dom_off = nullptr;
    uint8_t* d_dom = nullptr;
    std::vector<uint64_t> h_dommask;  // nv * W, bit k set iff k in D(v) (incl. 0)
    // population
    uint8_t *d_members = nullptr, *d_offspring = nullptr, *d_improved = nullptr, *d_next = nullptr;
    uint16_t *d_dist = nullptr, *d_cross = nullptr, *d_fresh = nullptr, *d_dnext = nullptr;
    int32_t *d_best_f = nullptr, *d_rep_f = nullptr, *d_mf = nullptr, *d_mc = nullptr, *d_tmpf = nullptr,
            *d_tmpc = nullptr;
    int64_t* d_iters = nullptr;
    unsigned long long* d_bytes = nullptr;
    int32_t* d_imc = nullptr;  // c of the improved individuals (0 after improve; set by plse_set_colors)
    int32_t *d_nf = nullptr, *d_nc = nullptr;  // next members' f / c (gathered by the update)
    uint32_t* d_excl = nullptr;
    int excl_words = 0;
    // K3 on tcgen05: one-hot operands (p x Kpad u8) and the column tables of the domain CSR
    bool use_tc = true;
    int kdom = 0, kpad = 0;
    uint16_t* d_colvert = nullptr;
    // k_improve's padded row / column colour copies (device_api.h ImproveArgs)
    uint16_t *d_rpos = nullptr, *d_cpos = nullptr;
    uint64_t *d_rinfo = nullptr, *d_cinfo = nullptr;
    int rp_bytes = 0, cp_bytes = 0;
    uint8_t *d_hA = nullptr, *d_hB = nullptr;
    int32_t* d_partner = nullptr;
    // improve launch
    void* d_rec = nullptr;
    uint32_t* d_until = nullptr;
    uint32_t* d_slot_clock = nullptr;
    uint8_t* d_conf_scratch = nullptr;
    uint32_t tenure_cap = 0;
    size_t rec_stride = 0, until_stride = 0;
    int grid = 0, threads = 0, wpc = 0, slots = 0, warps_per_sm = 0;
    bool plits = false;      // variant MPMA: k_plits (plits.cu) is the improve kernel
    bool ref_ties = false;   // tie_mode REF: k_improve_ref (improve_ref.cu)
    int64_t budget2 = 0;     // PLITS phase-2 budget
    int lane_words16 = 1;
    size_t smem = 0;
    int* d_work = nullptr;
    unsigned long long* d_prof = nullptr;  // PLSE_PROFILE instrumentation counters
    int* d_race = nullptr;                 // race-mode flag (plse_solve with race)
    int race_f = -1;
    unsigned long long* d_deadline = nullptr;  // %globaltimer deadline of plse_solve's time limit
    unsigned long long* d_dsum = nullptr;      // GenerationStats::mean_distance reduction
    // pool update scratch (pool.cu)
    PoolScratch ps{};
    int pool_cap = 0;  // pool positions the scratch holds (2p + migrant capacity)
    // island exchange: migrants staged as extra pool candidates of the next update
    uint8_t* d_migr = nullptr;
    int32_t *d_gf = nullptr, *d_gc = nullptr;
    uint16_t* d_migd = nullptr;  // n_mig x (2p + n_mig)
    uint8_t* d_hM = nullptr;     // one-hot rows of the migrants
    int mig_cap = 0, n_mig = 0;
    bool onehot_valid = false;  // d_hA / d_hB hold onehot(members) / onehot(improved) of this generation
    ImproveSummary* d_sum = nullptr;
    ImproveSummary* h_sum = nullptr;  // pinned
    int32_t* h_info = nullptr;        // pinned: pool_best_f, shortfall count
    // phase timers: events recorded on the stream, resolved when the counters are read
    cudaEvent_t ph_ev[3][2] = {};
    bool ph_pending[3] = {false, false, false};
    // host staging (pinned, so host<->device copies run at full PCIe rate)
    uint8_t* stage = nullptr;
    size_t stage_bytes = 0;
    // device copies of a host-format colouring (u16 rows) and its u8 form, allocated on first use
    uint16_t* d_c16 = nullptr;
    uint8_t* d_c8 = nullptr;
    int* d_bad = nullptr;
    cudaEvent_t tm0 = nullptr, tm1 = nullptr;
    plse_counters ctr{};
    std::string err;

    ~plse_ctx() {
        if (device >= 0) cudaSetDevice(device);
        void* bufs[] = {d_cell, d_rs, d_cs, d_cl, d_pr, d_pc, d_below, d_dom_off, d_dom, d_members, d_offspring,
                        d_improved, d_next, d_dist, d_cross, d_fresh, d_dnext, d_best_f, d_rep_f, d_mf, d_mc,
                        d_tmpf, d_tmpc, d_iters, d_bytes, d_excl, d_partner, d_rec, d_until, d_slot_clock,
                        d_conf_scratch, d_work, d_prof, d_race, d_deadline, d_dsum, d_colvert, d_hA, d_hB, d_imc,
                        d_rpos, d_cpos, d_rinfo, d_cinfo,
                        d_nf, d_nc, ps.keys0, ps.keys1, ps.order, ps.sel, ps.nsel, ps.slots, ps.info, ps.legal,
                        ps.admitted, ps.ok, ps.conf, d_migr, d_gf, d_gc, d_migd, d_hM, d_sum, d_c16, d_c8, d_bad};
        for (void* b : bufs)
            if (b) cudaFree(b);
        if (stage) cudaFreeHost(stage);
        if (h_sum) cudaFreeHost(h_sum);
        if (h_info) cudaFreeHost(h_info);
        for (auto& pr : ph_ev)
            for (cudaEvent_t e : pr)
                if (e) cudaEventDestroy(e);
        if (tm0) cudaEventDestroy(tm0);
        if (tm1) cudaEventDestroy(tm1);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (st) cudaStreamDestroy(st);
    }

    PopGraph pop_graph() const {
        PopGraph g;
        g.n = n;
        g.nv = nv;
        g.nvpad = nvpad;
        g.cell = d_cell;
        g.row_start = d_rs;
        g.col_start = d_cs;
        g.col_list = d_cl;
        g.dom_off = d_dom_off;
        g.dom = d_dom;
        g.below_thr = d_below;
        return g;
    }
    uint8_t* colors(int which) {
        if (which == PLSE_MEMBERS) return d_members;
        if (which == PLSE_OFFSPRING) return d_offspring;
        if (which == PLSE_IMPROVED) return d_improved;
        throw std::invalid_argument("unknown population buffer");
    }
    uint16_t* distbuf(int which) {
        if (which == PLSE_DIST) return d_dist;
        if (which == PLSE_CROSS) return d_cross;
        if (which == PLSE_FRESH) return d_fresh;
        throw std::invalid_argument("unknown distance matrix");
    }
    void launched(cudaError_t e, int count = 1) {
        CK(e);
        ctr.kernel_launches += count;
    }
    uint64_t stream_base(uint64_t gen) const { return gen * (uint64_t)prm.p_total + (uint64_t)prm.offset; }
    uint8_t* staging(size_t bytes) {
        if (bytes > stage_bytes) {
            if (stage) cudaFreeHost(stage);
            stage = nullptr;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&stage), bytes, cudaHostAllocDefault));
            stage_bytes = bytes;
        }
        return stage;
    }
};

namespace {

int finish(plse_ctx* ctx, int code, const char* what) {
    g_last_error = what;
    if (ctx) ctx->err = what;
    return code;
}

template <class F>
int guard(plse_ctx* ctx, F&& f) {
    try {
        f();
        return PLSE_OK;
    } catch (const std::invalid_argument& e) {
        return finish(ctx, PLSE_ERR_INVALID, e.what());
    } catch (const CudaError& e) {
        return finish(ctx, PLSE_ERR_CUDA, e.what());
    } catch (const Unsupported& e) {
        return finish(ctx, PLSE_ERR_UNSUPPORTED, e.what());
    } catch (const std::exception& e) {
        return finish(ctx, PLSE_ERR_RUNTIME, e.what());
    } catch (...) {
        return finish(ctx, PLSE_ERR_RUNTIME, "unknown error");
    }
}

// engine.hpp:38-46
void validate_params(const plse_params& p) {
    if (p.p < 2) throw std::invalid_argument("population size must be at least 2");
    if (!(p.gamma > 1.0)) throw std::invalid_argument("gamma must exceed 1");
    if (p.crossover == PLSE_X_AUX && !(p.beta > p.gamma)) throw std::invalid_argument("beta must exceed gamma");
    if (!(p.alpha >= 0.0)) throw std::invalid_argument("alpha must be non-negative");
    if (p.phase1_iters < 0 || p.phase2_iters < 0) throw std::invalid_argument("phase budgets must be positive");
    if (p.variant != PLSE_V_PARTIAL && p.variant != PLSE_V_MPMA) throw std::invalid_argument("unknown variant");
    if (p.crossover < 0 || p.crossover > 2) throw std::invalid_argument("unknown crossover mode");
    if (p.matching < 0 || p.matching > 1) throw std::invalid_argument("unknown matching strategy");
    if (p.exclusion < 0 || p.exclusion > 2) throw std::invalid_argument("unknown exclusion scope");
    if (p.tie_mode != PLSE_TIE_CANON && p.tie_mode != PLSE_TIE_REF) throw std::invalid_argument("unknown tie mode");
    if (p.p_total < 0 || p.offset < 0) throw std::invalid_argument("negative island coordinates");
}

// f / c of p colour rows into device arrays (coloring.hpp:59-73)
void eval_into(plse_ctx* c, const uint8_t* colors, int32_t* df, int32_t* dc, int rows = -1) {
    c->launched(launch_eval_fc(c->pop_graph(), rows < 0 ? c->prm.p : rows, colors, df, dc, c->st));
}

// K3: D = hamming(A rows, B rows) -- tcgen05 one-hot GEMM over precomputed one-hot operands, or the
// CUDA-core kernel (PLSE_TC=0) over the colour rows.  upper: A == B, only tiles on or above the diagonal.
void sim_block(plse_ctx* c, const uint8_t* hA, const uint8_t* A, int na, const uint8_t* hB, const uint8_t* B, int nb,
               uint16_t* D, int ldd, int upper) {
    if (!c->use_tc) {
        c->launched(launch_hamming(A, na, B, nb, c->nv, c->nvpad, D, ldd, c->st, upper));
        return;
    }
    c->launched(launch_similarity_tc(hA, na, hB, nb, c->kpad, c->nv, D, ldd, c->st, upper));
    c->ctr.k3_ops += upper ? (double)na * (na - 1) * c->kpad : 2.0 * na * (double)nb * c->kpad;
}

void onehot(plse_ctx* c, const uint8_t* X, int rows, uint8_t* H) {
    if (c->use_tc) c->launched(launch_onehot(X, rows, c->nvpad, c->d_colvert, c->d_dom, c->kdom, c->kpad, H, c->st));
}

// the full members x members matrix (population.hpp:76-87)
void full_distances(plse_ctx* c) {
    const int p = c->prm.p;
    onehot(c, c->d_members, p, c->d_hA);
    sim_block(c, c->d_hA, c->d_members, p, c->d_hA, c->d_members, p, c->d_dist, p, 0);
    c->onehot_valid = false;  // d_hB does not hold onehot(improved)
}

// migrant rows vs members | improved | migrants (the extra candidates of the next pool); needs the
// one-hot operands of this generation's members and improved in d_hA / d_hB
void migrant_distances(plse_ctx* c) {
    const int p = c->prm.p, m = c->n_mig, ld = 2 * p + m;
    if (!m) return;
    onehot(c, c->d_migr, m, c->d_hM);
    sim_block(c, c->d_hM, c->d_migr, m, c->d_hA, c->d_members, p, c->d_migd, ld, 0);
    sim_block(c, c->d_hM, c->d_migr, m, c->d_hB, c->d_improved, p, c->d_migd + p, ld, 0);
    sim_block(c, c->d_hM, c->d_migr, m, c->d_hM, c->d_migr, m, c->d_migd + 2 * p, ld, 0);
}

// population.hpp:41-61: cross = D(members, improved); fresh = D(improved, improved), upper triangle only
// (the pool update reads fresh[min][max]); onehot(improved) is expanded once for both
void cross_distances(plse_ctx* c) {
    const int p = c->prm.p;
    onehot(c, c->d_members, p, c->d_hA);
    onehot(c, c->d_improved, p, c->d_hB);
    sim_block(c, c->d_hA, c->d_members, p, c->d_hB, c->d_improved, p, c->d_cross, p, 0);
    sim_block(c, c->d_hB, c->d_improved, p, c->d_hB, c->d_improved, p, c->d_fresh, p, 1);
    c->onehot_valid = true;
    migrant_distances(c);
}

// pool-position scratch for 2p + m candidates (m = staged migrants)
void ensure_pool_scratch(plse_ctx* c, int m) {
    const int P = 2 * c->prm.p + m;
    if (P <= c->pool_cap) return;
    for (void* b : {(void*)c->ps.keys0, (void*)c->ps.keys1, (void*)c->ps.order, (void*)c->ps.legal,
                    (void*)c->ps.admitted})
        if (b) CK(cudaFree(b));
    c->ps.keys0 = dalloc<uint64_t>(P);
    c->ps.keys1 = dalloc<uint64_t>(P);
    c->ps.order = dalloc<int32_t>(P);
    c->ps.legal = dalloc<uint8_t>(P);
    c->ps.admitted = dalloc<uint8_t>(P);
    c->pool_cap = P;
}

// the f / c of a population buffer, read back from the device
void fetch_fc(plse_ctx* c, int which, std::vector<int32_t>& f, std::vector<int32_t>& cc) {
    const int p = c->prm.p;
    f.resize(p);
    cc.resize(p);
    const int32_t* df = which == PLSE_MEMBERS ? c->d_mf : c->d_best_f;
    const int32_t* dc = which == PLSE_MEMBERS ? c->d_mc : c->d_imc;
    CK(cudaMemcpyAsync(f.data(), df, 4 * p, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(cc.data(), dc, 4 * p, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
}

// phase timers: PH_DIST, PH_UPDATE, PH_OFFSPRING
enum { PH_DIST = 0, PH_UPDATE = 1, PH_OFFSPRING = 2 };
void phase_begin(plse_ctx* c, int ph) { CK(cudaEventRecord(c->ph_ev[ph][0], c->st)); }
void phase_end(plse_ctx* c, int ph) {
    CK(cudaEventRecord(c->ph_ev[ph][1], c->st));
    c->ph_pending[ph] = true;
}
void resolve_phase_timers(plse_ctx* c) {
    double* out[3] = {&c->ctr.distances_ms, &c->ctr.update_ms, &c->ctr.offspring_ms};
    for (int ph = 0; ph < 3; ++ph) {
        if (!c->ph_pending[ph]) continue;
        CK(cudaEventSynchronize(c->ph_ev[ph][1]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ph_ev[ph][0], c->ph_ev[ph][1]));
        *out[ph] = ms;
        c->ph_pending[ph] = false;
    }
}

void create_impl(const plse_graph* gr, const plse_params* pp, int device, plse_ctx** out) {
    if (!gr || !pp || !out) throw std::invalid_argument("null argument");
    validate_params(*pp);
    const int n = gr->order, nv = gr->vertex_count;
    if (n <= 0) throw std::invalid_argument("order must be positive");
    if (n > 127) throw Unsupported("device path supports n <= 127 (u8 colours, <= 2 mask words)");
    if (nv <= 0) throw Unsupported("empty reduced graph: nothing to search (trivial instance)");
    if (nv > 65535) throw Unsupported("device path supports |V| <= 65535");
    auto ctx = std::make_unique<plse_ctx>();
    plse_ctx* c = ctx.get();
    c->device = -1;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw CudaError("no CUDA device " + std::to_string(device));
    CK(cudaSetDevice(device));
    c->device = device;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError(std::string("device is not sm_100 (B200): ") + prop.name);
    c->nsm = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    c->n = n;
    c->nv = nv;
    c->l = gr->l;
    c->prm = *pp;
    if (c->prm.p_total == 0) c->prm.p_total = c->prm.p;
    c->budget = pp->phase1_iters > 0 ? pp->phase1_iters : 100LL * nv;
    c->budget2 = pp->phase2_iters > 0 ? pp->phase2_iters : 2LL * nv;
    c->plits = pp->variant == PLSE_V_MPMA;
    c->ref_ties = pp->tie_mode == PLSE_TIE_REF;
    if (c->budget + (c->plits ? c->budget2 : 0) >= (1LL << 30)) throw Unsupported("budget must be < 2^30 iterations");
    if (pp->alpha * nv >= (double)(1 << 29)) throw Unsupported("alpha * |V| must be < 2^29 (tabu tenure range)");
    c->tenure_cap = 10u + (uint32_t)(pp->alpha * (double)nv);
    c->stop_f = gr->l == 1 ? 1 : 0;
    c->W = n < 64 ? 1 : 2;
    c->nvpad = (int)up((size_t)nv, 16);
    const int nwords = (nv + 31) / 32;
    c->lane_words = (nwords + 31) / 32;
    const int W = c->W;

    // ---- graph: cells must be row-major (lsgraph.hpp:149-165)
    std::vector<uint16_t> cell(nv), rs(n + 1, 0), cs(n + 1, 0), cl(nv);
    std::vector<int> ccount(n, 0);
    for (int v = 0; v < nv; ++v) {
        const int r = gr->cell_row[v], col = gr->cell_col[v];
        if (r < 0 || r >= n || col < 0 || col >= n) throw std::invalid_argument("cell out of range");
        if (v && (r < gr->cell_row[v - 1] || (r == gr->cell_row[v - 1] && col <= gr->cell_col[v - 1])))
            throw std::invalid_argument("vertices must be in row-major cell order");
        cell[v] = (uint16_t)(r << 8 | col);
        ccount[col]++;
    }
    for (int r = 0, v = 0; r <= n; ++r) {
        while (v < nv && gr->cell_row[v] < r) ++v;
        rs[r] = (uint16_t)v;
    }
    for (int col = 0; col < n; ++col) cs[col + 1] = (uint16_t)(cs[col] + ccount[col]);
    {
        std::vector<int> fill(cs.begin(), cs.end() - 1);
        for (int v = 0; v < nv; ++v) cl[fill[gr->cell_col[v]]++] = (uint16_t)v;
    }
    std::vector<uint64_t> pr((size_t)n * W, 0), pc((size_t)n * W, 0);
    for (int q = 0; q < gr->n_prefilled; ++q) {
        const int r = gr->prefilled[3 * q], col = gr->prefilled[3 * q + 1], s = gr->prefilled[3 * q + 2];
        if (r < 0 || r >= n || col < 0 || col >= n || s < 1 || s > n) throw std::invalid_argument("bad prefilled cell");
        pr[(size_t)r * W + s / 64] |= 1ULL << (s % 64);
        pc[(size_t)col * W + s / 64] |= 1ULL << (s % 64);
    }
    // domains must be exactly {0} u {k : k not prefilled in row or column} (lsgraph.hpp:152-156)
    c->h_dommask.assign((size_t)nv * W, 0);
    std::vector<uint8_t> dom8(gr->dom_offsets[nv]);
    for (int v = 0; v < nv; ++v) {
        const int r = gr->cell_row[v], col = gr->cell_col[v];
        int expect = 1;
        for (int k = 1; k <= n; ++k) expect += !(((pr[(size_t)r * W + k / 64] | pc[(size_t)col * W + k / 64]) >> (k % 64)) & 1);
        const int b = gr->dom_offsets[v], e = gr->dom_offsets[v + 1];
        if (e - b != expect || gr->dom[b] != 0) throw std::invalid_argument("domain does not match the prefilled cells");
        for (int a = b; a < e; ++a) {
            const int k = gr->dom[a];
            if (a > b && (k <= gr->dom[a - 1] ||
                          (((pr[(size_t)r * W + k / 64] | pc[(size_t)col * W + k / 64]) >> (k % 64)) & 1)))
                throw std::invalid_argument("domain does not match the prefilled cells");
            c->h_dommask[(size_t)v * W + k / 64] |= 1ULL << (k % 64);
            dom8[a] = (uint8_t)k;
        }
    }
    c->kdom = gr->dom_offsets[nv];
    c->kpad = (int)up((size_t)c->kdom, 128);
    std::vector<uint16_t> colvert(c->kdom);
    for (int v = 0; v < nv; ++v)
        for (int a = gr->dom_offsets[v]; a < gr->dom_offsets[v + 1]; ++a) colvert[a] = (uint16_t)v;
    if (const char* env = std::getenv("PLSE_TC")) c->use_tc = env[0] != '0';
    if (c->use_tc) CK(prepare_similarity_tc());
    std::vector<uint64_t> below(n + 1, 0);
    for (int b = 1; b <= n; ++b) below[b] = (0 - (uint64_t)b) % (uint64_t)b;

    c->d_cell = dalloc<uint16_t>(nv);
    c->d_rs = dalloc<uint16_t>(n + 1);
    c->d_cs = dalloc<uint16_t>(n + 1);
    c->d_cl = dalloc<uint16_t>(nv);
    c->d_pr = dalloc<uint64_t>((size_t)n * W);
    c->d_pc = dalloc<uint64_t>((size_t)n * W);
    c->d_below = dalloc<uint64_t>(n + 1);
    c->d_dom_off = dalloc<int32_t>(nv + 1);
    c->d_dom = dalloc<uint8_t>(dom8.size());
    CK(cudaMemcpy(c->d_cell, cell.data(), 2 * nv, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_rs, rs.data(), 2 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_cs, cs.data(), 2 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_cl, cl.data(), 2 * nv, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_pr, pr.data(), 8 * pr.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_pc, pc.data(), 8 * pc.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_below, below.data(), 8 * below.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_dom_off, gr->dom_offsets, 4 * (nv + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_dom, dom8.data(), dom8.size(), cudaMemcpyHostToDevice));
    {  // padded row / column copies: each line starts on an 8-byte boundary, 0xFF between lines
        std::vector<uint16_t> rpos(nv), cpos(nv);
        std::vector<uint64_t> rinfo(n), cinfo(n);
        size_t ro = 0, co = 0;
        for (int r = 0; r < n; ++r) {
            const int len = rs[r + 1] - rs[r];
            rinfo[r] = (uint64_t)ro | (uint64_t)((len + 7) / 8) << 16 | (uint64_t)rs[r] << 32;
            for (int x = 0; x < len; ++x) rpos[rs[r] + x] = (uint16_t)(ro + x);
            ro += up((size_t)len, 8);
        }
        for (int col = 0; col < n; ++col) {
            const int len = cs[col + 1] - cs[col];
            cinfo[col] = (uint64_t)co | (uint64_t)((len + 7) / 8) << 16 | (uint64_t)cs[col] << 32;
            for (int x = 0; x < len; ++x) cpos[cl[cs[col] + x]] = (uint16_t)(co + x);
            co += up((size_t)len, 8);
        }
        c->rp_bytes = (int)up(ro, 16);
        c->cp_bytes = (int)up(co, 16);
        if (c->rp_bytes + c->cp_bytes > 65535) throw Unsupported("padded colour copies exceed 64 KB");
        c->d_rpos = dalloc<uint16_t>(nv);
        c->d_cpos = dalloc<uint16_t>(nv);
        c->d_rinfo = dalloc<uint64_t>(n);
        c->d_cinfo = dalloc<uint64_t>(n);
        CK(cudaMemcpy(c->d_rpos, rpos.data(), 2 * nv, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_cpos, cpos.data(), 2 * nv, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_rinfo, rinfo.data(), 8 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_cinfo, cinfo.data(), 8 * n, cudaMemcpyHostToDevice));
    }
    c->d_colvert = dalloc<uint16_t>(c->kdom);
    CK(cudaMemcpy(c->d_colvert, colvert.data(), 2 * colvert.size(), cudaMemcpyHostToDevice));

    // ---- population buffers
    const size_t p = (size_t)c->prm.p;
    const size_t rows = p * c->nvpad;
    c->d_members = dalloc<uint8_t>(rows);
    c->d_offspring = dalloc<uint8_t>(rows);
    c->d_improved = dalloc<uint8_t>(rows);
    c->d_next = dalloc<uint8_t>(rows);
    CK(cudaMemset(c->d_members, 0, rows));
    CK(cudaMemset(c->d_offspring, 0, rows));
    CK(cudaMemset(c->d_improved, 0, rows));
    CK(cudaMemset(c->d_next, 0, rows));
    c->d_dist = dalloc<uint16_t>(p * p);
    c->d_cross = dalloc<uint16_t>(p * p);
    c->d_fresh = dalloc<uint16_t>(p * p);
    c->d_dnext = dalloc<uint16_t>(p * p);
    if (c->use_tc) {
        c->d_hA = dalloc<uint8_t>(p * (size_t)c->kpad);
        c->d_hB = dalloc<uint8_t>(p * (size_t)c->kpad);
    }
    CK(cudaMemset(c->d_dist, 0, 2 * p * p));
    c->d_best_f = dalloc<int32_t>(p);
    c->d_rep_f = dalloc<int32_t>(p);
    c->d_mf = dalloc<int32_t>(p);
    c->d_mc = dalloc<int32_t>(p);
    c->d_tmpf = dalloc<int32_t>(p);
    c->d_tmpc = dalloc<int32_t>(p);
    c->d_iters = dalloc<int64_t>(p);
    c->d_bytes = dalloc<unsigned long long>(p);
    c->d_imc = dalloc<int32_t>(p);
    c->d_nf = dalloc<int32_t>(p);
    c->d_nc = dalloc<int32_t>(p);
    {  // members start uncoloured (f = |V|, c = 0) until initialised or uploaded
        std::vector<int32_t> fv(p, nv);
        CK(cudaMemcpy(c->d_mf, fv.data(), 4 * p, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_best_f, fv.data(), 4 * p, cudaMemcpyHostToDevice));
        CK(cudaMemset(c->d_mc, 0, 4 * p));
        CK(cudaMemset(c->d_imc, 0, 4 * p));
        CK(cudaMemset(c->d_iters, 0, 8 * p));
    }
    c->excl_words = (int)((p + 31) / 32);
    c->d_excl = dalloc<uint32_t>(p * c->excl_words);
    CK(cudaMemset(c->d_excl, 0, 4 * p * c->excl_words));
    c->d_partner = dalloc<int32_t>(p);
    ensure_pool_scratch(c, 0);
    c->ps.sel = dalloc<int32_t>(p);
    c->ps.nsel = dalloc<int32_t>(1);
    c->ps.slots = dalloc<int32_t>(p);
    c->ps.info = dalloc<int32_t>(2);
    c->ps.ok = dalloc<uint8_t>(1024);
    c->ps.conf = dalloc<uint32_t>(1024 * 32);
    CK(prepare_pool_update());
    c->d_sum = dalloc<ImproveSummary>(1);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_sum), sizeof(ImproveSummary), cudaHostAllocDefault));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_info), 2 * sizeof(int32_t), cudaHostAllocDefault));
    for (auto& pr : c->ph_ev)
        for (cudaEvent_t& e : pr) CK(cudaEventCreate(&e));
    c->d_work = dalloc<int>(1);

    // ---- improve launch shape: maximise resident individuals per SM
    c->lane_words16 = (nwords + 15) / 16;
    const void* kern = c->plits       ? (c->ref_ties ? plits_ref_kernel_ptr(W, false) : plits_kernel_ptr(W, false))
                       : c->ref_ties  ? improve_ref_kernel_ptr(W, false)
                                      : improve_kernel_ptr(W, false);
    const void* kern_dbg = c->plits       ? (c->ref_ties ? plits_ref_kernel_ptr(W, true) : plits_kernel_ptr(W, true))
                           : c->ref_ties  ? improve_ref_kernel_ptr(W, true)
                                          : improve_kernel_ptr(W, true);
    size_t graph_bytes = 0, warp_bytes = 0;
    if (c->plits && c->ref_ties) {
        const PlitsRefSmemLayout L = plits_ref_smem_layout(n, nv, c->nvpad, c->lane_words, W);
        graph_bytes = L.graph_bytes;
        warp_bytes = L.warp_bytes;
    } else if (c->ref_ties) {
        const RefSmemLayout L = improve_ref_smem_layout(n, nv, c->nvpad, c->lane_words, W);
        graph_bytes = L.graph_bytes;
        warp_bytes = L.warp_bytes;
    } else if (c->plits) {
        const PlitsSmemLayout L = plits_smem_layout(n, nv, c->nvpad, c->lane_words, W);
        graph_bytes = L.graph_bytes;
        warp_bytes = L.warp_bytes;
    } else {
        const PadSmemLayout L = pad_smem_layout(n, nv, c->lane_words, W, c->rp_bytes, c->cp_bytes);
        graph_bytes = L.graph_bytes;
        warp_bytes = L.warp_bytes;
    }
    // k_improve runs up to 28 warps in one CTA per SM (the graph tables staged once per SM)
    const bool big_ctas = !c->plits && !c->ref_ties;
    const int per_warp = 1;
    int best_ind = 0;
    int force_wpc = 0;
    if (const char* env = std::getenv("PLSE_IMPROVE_WPC")) force_wpc = std::atoi(env);
    int max_optin = 0;
    CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    for (int wpc : {28, 16, 8, 4, 2, 1}) {
        if (force_wpc && wpc != force_wpc) continue;
        if (wpc > 8 && !big_ctas) continue;
        const size_t smem = graph_bytes + (size_t)wpc * warp_bytes;
        if (smem > (size_t)max_optin) continue;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int bps = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 32 * wpc, smem));
        if (bps * wpc * per_warp > best_ind) {
            best_ind = bps * wpc * per_warp;
            c->wpc = wpc;
            c->smem = smem;
            c->grid = bps * c->nsm;
        }
    }
    if (best_ind == 0) throw Unsupported("instance too large for the shared-memory resident search");
    // a population that fits one warp per block everywhere runs one individual per block: the block
    // scheduler then spreads the individuals evenly over the SMs (a latency-bound small population
    // otherwise lands on whichever warps win the work counter)
    if (!force_wpc && c->wpc != 1) {
        const size_t smem1 = graph_bytes + warp_bytes;
        if (smem1 <= (size_t)max_optin) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
            int bps1 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps1, kern, 32, smem1));
            if (bps1 > 0 && c->prm.p <= bps1 * c->nsm) {
                best_ind = bps1;
                c->wpc = 1;
                c->smem = smem1;
                c->grid = bps1 * c->nsm;
            }
        }
    }
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem));
    CK(cudaFuncSetAttribute(kern_dbg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem));
    c->threads = 32 * c->wpc;
    c->warps_per_sm = best_ind / per_warp;
    c->slots = c->grid * c->wpc * per_warp;
    // PLITS (canonical) keeps W words of possibly-tabu colours and an until bound per vertex there (plits.cu)
    const size_t rec_bytes = std::max(tabu_rec_bytes(W), c->plits && !c->ref_ties ? (size_t)8 * (W + 1) : (size_t)0);
    c->rec_stride = up((size_t)nv * rec_bytes, 256);
    c->until_stride = up((size_t)nv * (n + 1), 64);
    c->d_rec = dalloc<uint8_t>((size_t)c->slots * c->rec_stride);
    c->d_until = dalloc<uint32_t>((size_t)c->slots * c->until_stride);
    CK(cudaMemset(c->d_until, 0, sizeof(uint32_t) * (size_t)c->slots * c->until_stride));
    c->d_conf_scratch = dalloc<uint8_t>((size_t)c->slots * c->nvpad);
    c->d_slot_clock = dalloc<uint32_t>(c->slots);
    CK(cudaMemset(c->d_slot_clock, 0, sizeof(uint32_t) * c->slots));
    c->ctr.grid = c->grid;
    c->ctr.threads = c->threads;
    c->ctr.warps_per_sm = c->warps_per_sm;
    c->ctr.slots = c->slots;
    c->ctr.smem_bytes = (int64_t)c->smem;
    *out = ctx.release();
}

void ensure_color_buffers(plse_ctx* c) {
    if (c->d_c16) return;
    c->d_c16 = dalloc<uint16_t>((size_t)c->prm.p * c->nv);
    c->d_c8 = dalloc<uint8_t>((size_t)c->prm.p * c->nvpad);
    c->d_bad = dalloc<int>(1);
}

// the caller's u16 rows go to the device as they are; a kernel narrows them to the u8 rows and checks
// every colour against its vertex's domain, and only a valid colouring replaces the target buffer
void upload_colors(plse_ctx* c, int which, const uint16_t* host, int64_t count) {
    const int p = c->prm.p, nv = c->nv, nvpad = c->nvpad;
    if (!host) throw std::invalid_argument("null colours");
    if (count != (int64_t)p * nv) throw std::invalid_argument("assignment size mismatch");
    ensure_color_buffers(c);
    CK(cudaMemcpyAsync(c->d_c16, host, (size_t)count * sizeof(uint16_t), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(c->d_bad, 0, sizeof(int), c->st));
    c->launched(launch_unpack_colors(c->d_c16, c->d_c8, p, nv, nvpad, c->n, c->W, c->d_cell, c->d_pr, c->d_pc,
                                     c->d_bad, c->st));
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (bad) throw std::invalid_argument("assignment leaves vertex domain");
    uint8_t* dst = c->colors(which);
    CK(cudaMemcpyAsync(dst, c->d_c8, (size_t)p * nvpad, cudaMemcpyDeviceToDevice, c->st));
    if (which == PLSE_MEMBERS) eval_into(c, dst, c->d_mf, c->d_mc);
    if (which == PLSE_IMPROVED) eval_into(c, dst, c->d_best_f, c->d_imc);
    c->onehot_valid = false;
    CK(cudaStreamSynchronize(c->st));
}

void download_colors(plse_ctx* c, int which, uint16_t* host) {
    const int p = c->prm.p, nv = c->nv, nvpad = c->nvpad;
    if (!host) throw std::invalid_argument("null output");
    ensure_color_buffers(c);
    c->launched(launch_pack_colors(c->colors(which), c->d_c16, p, nv, nvpad, c->st));
    CK(cudaMemcpyAsync(host, c->d_c16, (size_t)p * nv * sizeof(uint16_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
}

void improve_impl(plse_ctx* c, uint64_t gen, int trace_idx, int64_t trace_cap, plse_step* d_trace, int p_eff,
                  int first, const StateProbe* probe = nullptr) {
    ImproveArgs a{};
    if (probe) a.probe = *probe;
    a.n = c->n;
    a.nv = c->nv;
    a.nvpad = c->nvpad;
    a.lane_words = c->lane_words;
    a.lane_words16 = c->lane_words16;
    a.cell = c->d_cell;
    a.row_start = c->d_rs;
    a.col_start = c->d_cs;
    a.col_list = c->d_cl;
    a.pre_row = c->d_pr;
    a.pre_col = c->d_pc;
    a.p = p_eff;
    a.offspring = c->d_offspring;
    a.improved = c->d_improved;
    a.best_f = c->d_best_f;
    a.repaired_f = c->d_rep_f;
    a.iters = c->d_iters;
    a.bytes = c->d_bytes;
    a.tabu_rec = c->d_rec;
    a.rec_stride = c->rec_stride;
    a.until = c->d_until;
    a.until_stride = c->until_stride;
    a.slot_clock = c->d_slot_clock;
    a.conf_scratch = c->d_conf_scratch;
    a.conf_stride = (size_t)c->nvpad;
    a.tenure_cap = c->tenure_cap;
    a.work_counter = c->d_work;
    a.master = c->prm.master_seed;
    a.generation = gen;
    a.p_total = (uint64_t)c->prm.p_total;
    a.offset = (uint64_t)c->prm.offset;
    a.budget = c->budget;
    a.budget2 = c->budget2;
    a.stop_f = c->stop_f;
    a.alpha = c->prm.alpha;
    a.trace_idx = trace_idx;
    a.trace_cap = trace_cap;
    a.trace = d_trace;
    a.prof = nullptr;
    a.race_flag = c->race_f >= 0 ? c->d_race : nullptr;
    a.race_f = c->race_f;
    a.deadline = c->d_deadline;
    a.rpos = c->d_rpos;
    a.cpos = c->d_cpos;
    a.rinfo = c->d_rinfo;
    a.cinfo = c->d_cinfo;
    a.rp_bytes = c->rp_bytes;
    a.cp_bytes = c->cp_bytes;
    if (const char* env = std::getenv("PLSE_PROFILE")) {
        if (env[0] == '1') {
            if (!c->d_prof) c->d_prof = dalloc<unsigned long long>(16);
            CK(cudaMemsetAsync(c->d_prof, 0, 16 * 8, c->st));
            a.prof = c->d_prof;
        }
    }
    a.first = first;
    {  // balanced rounds: every active slot searches the same number of individuals
        const int todo = std::max(1, p_eff - first);
        const int resident = c->wpc == 1 ? std::min(c->grid, todo) : c->slots;
        const int rounds = (todo + resident - 1) / resident;
        a.nslots = (todo + rounds - 1) / rounds;
    }
    CK(cudaMemsetAsync(c->d_work, 0, sizeof(int), c->st));
    CK(cudaEventRecord(c->ev0, c->st));
    // one individual per block when the blocks are single warps (see create): the first blocks, spread
    // round-robin over the SMs by the block scheduler, take the individuals
    const int grid = c->wpc == 1 ? std::max(1, std::min(c->grid, p_eff - first)) : c->grid;
    if (c->plits && c->ref_ties)
        c->launched(launch_plits_ref(a, c->W, grid, c->threads, c->smem, c->st));
    else if (c->plits) {
        // the instrumented kernel (traces, probes, PLSE_PROFILE) reads its register-list capacity
        const bool debug = a.trace != nullptr || a.prof != nullptr || a.probe.n > 0;
        const char* cap = a.prof ? std::getenv("PLSE_PLITS_CAP") : nullptr;
        if (debug) CK(set_plits_list_cap(cap ? std::atoi(cap) : 32, c->st));
        c->launched(launch_plits(a, c->W, grid, c->threads, c->smem, c->st));
    } else if (c->ref_ties)
        c->launched(launch_improve_ref(a, c->W, grid, c->threads, c->smem, c->st));
    else
        c->launched(launch_improve(a, c->W, grid, c->threads, c->smem, c->st));
    CK(cudaEventRecord(c->ev1, c->st));
}

void collect_improve(plse_ctx* c, int64_t* iters_total, int32_t* best_f, int32_t* best_idx) {
    const int p = c->prm.p;
    // engine.hpp:207-217 on the device: total iterations, lowest-index argmin of f (strict <); the
    // improved individuals are legal (repair / PLITS' final repair), so their c is 0
    CK(cudaMemsetAsync(c->d_imc, 0, 4 * p, c->st));
    c->launched(launch_improve_reduce(c->d_best_f, c->d_iters, c->d_bytes, p, c->d_sum, c->st));
    CK(cudaMemcpyAsync(c->h_sum, c->d_sum, sizeof(ImproveSummary), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->onehot_valid = false;
    const int64_t tot = c->h_sum->iters;
    const double by = (double)c->h_sum->bytes;
    const int bf = c->h_sum->best_f, bi = c->h_sum->best_idx;
    if (c->d_prof && std::getenv("PLSE_PROFILE") && c->ref_ties && c->plits) {
        unsigned long long pr[16];
        CK(cudaMemcpy(pr, c->d_prof, sizeof(pr), cudaMemcpyDeviceToHost));
        const double st = pr[0] ? (double)pr[0] : 1.0;
        std::fprintf(stderr,
                     "[plse-prof plits-ref] steps %llu | cyc/step: stage %.0f walk %.0f fast %.0f | mean sequence "
                     "%.1f, walked vertices %.2f considered %.2f T-hits %.2f | fast: moves+tabu %.0f scan+early %.0f "
                     "segment %.0f generate %.0f select %.0f outputs/step %.2f | long sequences %llu, long segments %llu\n",
                     pr[0], pr[1] / st, pr[2] / st, pr[3] / st, pr[4] / st, pr[5] / st, pr[6] / st, pr[7] / st,
                     pr[8] / st, pr[9] / st, pr[10] / st, pr[11] / st, pr[12] / st, pr[13] / st, pr[14], pr[15]);
    } else if (c->d_prof && std::getenv("PLSE_PROFILE") && c->ref_ties) {
        unsigned long long pr[16];
        CK(cudaMemcpy(pr, c->d_prof, sizeof(pr), cudaMemcpyDeviceToHost));
        const double st = pr[0] ? (double)pr[0] : 1.0;
        std::fprintf(stderr,
                     "[plse-prof ref] steps %llu | cyc/step: masks %.0f walk %.0f apply %.0f | draws/step %.2f | "
                     "mean f %.1f | fast path (|V0| > 32): masks %.0f scans %.0f stream %.0f owner %.0f | early draws/step %.2f\n",
                     pr[0], pr[1] / st, pr[2] / st, pr[3] / st, pr[4] / st, pr[5] / st, pr[6] / st, pr[7] / st,
                     pr[8] / st, pr[9] / st, pr[10] / st);
    } else if (c->d_prof && std::getenv("PLSE_PROFILE") && c->plits) {
        unsigned long long pr[16];
        CK(cudaMemcpy(pr, c->d_prof, sizeof(pr), cudaMemcpyDeviceToHost));
        const double st = pr[0] ? (double)pr[0] : 1.0;
        std::fprintf(stderr,
                     "[plse-prof plits] indiv %llu steps %llu | cyc/step: list %.0f level %.0f select %.0f move %.0f "
                     "total %.0f | extra level passes %.3f/step | mean active %.1f | move: select->membership %.0f "
                     "membership %.0f tail %.0f | level: minimum %.0f admissible %.0f extra passes %.0f | register "
                     "mode: %llu entries, %llu exits\n",
                     pr[8], pr[0], pr[1] / st, pr[2] / st, pr[3] / st, pr[4] / st, pr[5] / st, pr[6] / st, pr[7] / st,
                     pr[9] / st, pr[10] / st, pr[11] / st, pr[12] / st, pr[13] / st, pr[14] / st, pr[15] & 0xFFFFFFFFull,
                     pr[15] >> 32);
    } else if (c->d_prof && std::getenv("PLSE_PROFILE")) {
        unsigned long long pr[16];
        CK(cudaMemcpy(pr, c->d_prof, sizeof(pr), cudaMemcpyDeviceToHost));
        std::fprintf(stderr,
                     "[plse-prof] indiv %llu prologue %.0f cyc/indiv | dense %llu steps %.0f cyc/step mean f %.1f | "
                     "sparse %llu steps %.0f cyc/step | enter %llu | total %.3g cyc/indiv | f<=8 %llu f<=16 %llu "
                     "f<=24 %llu f<=32 %llu\n",
                     pr[0], (double)pr[1] / pr[0], pr[2], pr[2] ? (double)pr[3] / pr[2] : 0.0,
                     pr[2] ? (double)pr[6] / pr[2] : 0.0, pr[4], pr[4] ? (double)pr[5] / pr[4] : 0.0, pr[7],
                     (double)pr[8] / pr[0], pr[9], pr[10], pr[11], pr[12]);
    }
    c->ctr.improve_ms = ms;
    c->ctr.alg_bytes = by;
    c->ctr.moves = tot;
    if (iters_total) *iters_total = tot;
    if (best_f) *best_f = bf;
    if (best_idx) *best_idx = bi;
}

// population.hpp:103-183 on the device (pool.cu): key sort, admission chain, shortfall fill and the
// gathers are enqueued on the stream with no host round trip; the UpdateInfo outputs are read back only
// when the caller asks for them.  Staged migrants (island exchange) join the pool as ids 2p..2p+m-1.
void update_impl(plse_ctx* c, int32_t* pool_best_f, int32_t* n_shortfall, int32_t* slots_out) {
    const int p = c->prm.p, m = c->n_mig;
    ensure_pool_scratch(c, m);
    const double thr = c->nv / c->prm.gamma;  // population.hpp:74 spacing threshold, compared as double
    const int dthr = (int)std::floor(thr);    // integer d > thr  <=>  d > floor(thr)
    PoolView pv{p, m, c->d_dist, c->d_cross, c->d_fresh, c->d_migd};
    PoolFC fc{p, m, c->d_mf, c->d_mc, c->d_best_f, c->d_imc, c->d_gf, c->d_gc};
    int64_t nl = 0;
    CK(launch_pool_update(pv, fc, c->ps, c->nv, dthr, c->d_members, c->d_improved, c->d_migr, c->d_next, c->d_dnext,
                          c->d_nf, c->d_nc, c->nvpad, c->st, &nl));
    c->ctr.kernel_launches += nl;
    std::swap(c->d_members, c->d_next);
    std::swap(c->d_dist, c->d_dnext);
    std::swap(c->d_mf, c->d_nf);
    std::swap(c->d_mc, c->d_nc);
    c->n_mig = 0;
    c->onehot_valid = false;
    if (pool_best_f || n_shortfall || slots_out) {
        CK(cudaMemcpyAsync(c->h_info, c->ps.info, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (pool_best_f) *pool_best_f = c->h_info[0];
        if (n_shortfall) *n_shortfall = c->h_info[1];
        if (slots_out && c->h_info[1] > 0) {
            CK(cudaMemcpyAsync(slots_out, c->ps.slots, 4 * (size_t)c->h_info[1], cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
    }
}

void offspring_impl(plse_ctx* c, uint64_t gen) {
    const int p = c->prm.p;
    if (c->prm.crossover == PLSE_X_NONE) {
        CK(cudaMemcpyAsync(c->d_offspring, c->d_members, (size_t)p * c->nvpad, cudaMemcpyDeviceToDevice, c->st));
    } else {
        c->launched(launch_match(c->d_dist, p, c->prm.matching, c->prm.exclusion, c->d_excl, c->excl_words,
                                 c->prm.master_seed, c->stream_base(gen), c->d_partner, c->st));
        c->launched(launch_crossover(c->d_members, c->d_dist, c->d_partner, p, c->nv, c->nvpad, c->prm.crossover,
                                     c->prm.beta, c->prm.master_seed, c->stream_base(gen), c->d_offspring, c->st));
    }
}

void init_impl(plse_ctx* c) {
    c->launched(launch_init_population(c->pop_graph(), c->prm.p, c->prm.master_seed, (uint64_t)c->prm.offset,
                                       c->d_members, c->st));
    eval_into(c, c->d_members, c->d_mf, c->d_mc);
    full_distances(c);
    CK(cudaStreamSynchronize(c->st));
}

}  // namespace

extern "C" {

int plse_abi_version(void) { return PLSE_ABI_VERSION; }

const char* plse_last_error(const plse_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int plse_generate_instance(int32_t n, double r, uint64_t seed, uint16_t* grid) {
    return guard(nullptr, [&] {
        if (!grid) throw std::invalid_argument("null grid");
        auto g = plse_host::generate_instance(n, r, seed);
        std::memcpy(grid, g.data(), 2 * g.size());
    });
}

int plse_parse_instance(const char* text, int32_t* n, uint16_t* grid, int32_t grid_cap) {
    return guard(nullptr, [&] {
        if (!text || !n) throw std::invalid_argument("null argument");
        int nn = 0;
        auto g = plse_host::parse_instance(text, nn);
        *n = nn;
        if (grid) {
            if ((int64_t)g.size() > grid_cap) throw std::invalid_argument("grid buffer too small");
            std::memcpy(grid, g.data(), 2 * g.size());
        }
    });
}

int plse_preprocess(int32_t n, const uint16_t* grid, plse_graph_h** out) {
    return guard(nullptr, [&] {
        if (!grid || !out || n <= 0) throw std::invalid_argument("bad arguments");
        for (int q = 0; q < n * n; ++q)
            if (grid[q] > n) throw std::invalid_argument("symbol out of range");
        auto* h = new plse_graph_h;
        h->g = plse_host::preprocess(n, grid);
        *out = h;
    });
}

void plse_graph_free(plse_graph_h* g) { delete g; }

int plse_graph_view(const plse_graph_h* h, plse_graph* v) {
    return guard(nullptr, [&] {
        if (!h || !v) throw std::invalid_argument("null argument");
        const auto& g = h->g;
        v->order = g.n;
        v->vertex_count = g.nv;
        v->l = g.l;
        v->cell_row = g.cell_row.data();
        v->cell_col = g.cell_col.data();
        v->dom_offsets = g.dom_off.data();
        v->dom = g.dom.data();
        v->n_prefilled = (int32_t)(g.prefilled.size() / 3);
        v->prefilled = g.prefilled.data();
    });
}

int plse_to_grid(const plse_graph_h* h, const uint16_t* colors, uint16_t* grid) {
    return guard(nullptr, [&] {
        if (!h || !colors || !grid) throw std::invalid_argument("null argument");
        auto g = plse_host::to_grid(h->g, colors);
        std::memcpy(grid, g.data(), 2 * g.size());
    });
}

int plse_solve_exact(const plse_graph_h* h, int64_t node_budget, int32_t* optimum_f, int32_t* exact, int64_t* nodes,
                     uint16_t* certificate) {
    return guard(nullptr, [&] {
        if (!h || node_budget < 0) throw std::invalid_argument("bad arguments");
        auto r = plse_host::solve_exact(h->g, node_budget);
        if (optimum_f) *optimum_f = r.optimum_f;
        if (exact) *exact = r.exact ? 1 : 0;
        if (nodes) *nodes = r.nodes;
        if (certificate && !r.certificate.empty()) std::memcpy(certificate, r.certificate.data(), 2 * r.certificate.size());
    });
}

int plse_verify_certificate(int32_t n, const uint16_t* instance, int32_t m, const uint16_t* certificate,
                            int32_t* legal, int32_t* score, char* problems, int64_t problems_cap,
                            int64_t* problems_len) {
    return guard(nullptr, [&] {
        if (!instance || !certificate || n <= 0 || m <= 0) throw std::invalid_argument("bad arguments");
        auto r = plse_host::verify_certificate(n, instance, m, certificate);
        std::string joined;
        for (size_t i = 0; i < r.problems.size(); ++i) joined += (i ? "\n" : "") + r.problems[i];
        if (legal) *legal = r.legal ? 1 : 0;
        if (score) *score = r.score;
        if (problems_len) *problems_len = (int64_t)joined.size();
        if (problems && problems_cap > 0) {
            const size_t k = std::min<size_t>(joined.size(), (size_t)(problems_cap - 1));
            std::memcpy(problems, joined.data(), k);
            problems[k] = 0;
        }
    });
}

int plse_create(const plse_graph* graph, const plse_params* params, int32_t device, plse_ctx** out) {
    return guard(nullptr, [&] { create_impl(graph, params, device, out); });
}

void plse_destroy(plse_ctx* ctx) { delete ctx; }

int plse_set_colors(plse_ctx* c, int32_t which, const uint16_t* host, int64_t count) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        upload_colors(c, which, host, count);
    });
}

int plse_get_colors(plse_ctx* c, int32_t which, uint16_t* host) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        download_colors(c, which, host);
    });
}

int plse_get_row(plse_ctx* c, int32_t which, int32_t index, uint16_t* host) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!host) throw std::invalid_argument("null output");
        if (index < 0 || index >= c->prm.p) throw std::invalid_argument("individual index out of range");
        std::vector<uint8_t> row((size_t)c->nvpad);
        CK(cudaMemcpyAsync(row.data(), c->colors(which) + (size_t)index * c->nvpad, (size_t)c->nvpad,
                           cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        for (int v = 0; v < c->nv; ++v) host[v] = row[v];
    });
}

int plse_get_dist(plse_ctx* c, int32_t which, int32_t* host) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!host) throw std::invalid_argument("null output");
        const size_t pp = (size_t)c->prm.p * c->prm.p;
        std::vector<uint16_t> tmp(pp);
        CK(cudaMemcpyAsync(tmp.data(), c->distbuf(which), 2 * pp, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        const int p = c->prm.p;
        if (which == PLSE_FRESH) {  // the device keeps fresh's upper triangle; mirror it (population.hpp:84-86)
            for (int i = 0; i < p; ++i)
                for (int j = 0; j < i; ++j) tmp[(size_t)i * p + j] = tmp[(size_t)j * p + i];
        }
        for (size_t q = 0; q < pp; ++q) host[q] = tmp[q];
    });
}

int plse_set_dist(plse_ctx* c, int32_t which, const int32_t* host) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!host) throw std::invalid_argument("null input");
        const size_t pp = (size_t)c->prm.p * c->prm.p;
        std::vector<uint16_t> tmp(pp);
        for (size_t q = 0; q < pp; ++q) {
            if (host[q] < 0 || host[q] > c->nv) throw std::invalid_argument("distance out of range");
            tmp[q] = (uint16_t)host[q];
        }
        CK(cudaMemcpyAsync(c->distbuf(which), tmp.data(), 2 * pp, cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    });
}

int plse_get_stats(plse_ctx* c, int32_t which, int32_t* f, int32_t* cc, int64_t* iters) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        const int p = c->prm.p;
        std::vector<int32_t> ff, cv;
        if (which == PLSE_MEMBERS || which == PLSE_IMPROVED) {
            fetch_fc(c, which, ff, cv);
        } else {
            c->colors(which);  // validates `which`
            eval_into(c, c->colors(which), c->d_tmpf, c->d_tmpc);
            ff.resize(p);
            cv.resize(p);
            CK(cudaMemcpyAsync(ff.data(), c->d_tmpf, 4 * p, cudaMemcpyDeviceToHost, c->st));
            CK(cudaMemcpyAsync(cv.data(), c->d_tmpc, 4 * p, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
        if (f) std::memcpy(f, ff.data(), 4 * p);
        if (cc) std::memcpy(cc, cv.data(), 4 * p);
        if (iters) {
            CK(cudaMemcpyAsync(iters, c->d_iters, 8 * p, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
    });
}

int plse_get_partners(plse_ctx* c, int32_t* host) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(host, c->d_partner, 4 * c->prm.p, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
    });
}

int plse_get_counters(plse_ctx* c, plse_counters* out) {
    if (!c || !out) return finish(c, PLSE_ERR_INVALID, "null argument");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        resolve_phase_timers(c);
        *out = c->ctr;
    });
}

int plse_timer_start(plse_ctx* c) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!c->tm0) CK(cudaEventCreate(&c->tm0));
        if (!c->tm1) CK(cudaEventCreate(&c->tm1));
        CK(cudaEventRecord(c->tm0, c->st));
    });
}

int plse_timer_stop(plse_ctx* c, double* ms) {
    if (!c || !ms) return finish(c, PLSE_ERR_INVALID, "null argument");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!c->tm0) throw std::invalid_argument("timer not started");
        CK(cudaEventRecord(c->tm1, c->st));
        CK(cudaEventSynchronize(c->tm1));
        float f = 0;
        CK(cudaEventElapsedTime(&f, c->tm0, c->tm1));
        *ms = f;
    });
}

int plse_device_colors(plse_ctx* c, int32_t which, void** dev_ptr, int64_t* row_stride) {
    if (!c || !dev_ptr) return finish(c, PLSE_ERR_INVALID, "null argument");
    return guard(c, [&] {
        *dev_ptr = c->colors(which);
        if (row_stride) *row_stride = c->nvpad;
    });
}

int plse_init_population(plse_ctx* c) {
    NvtxRange nvtx_("plse.init_population");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        init_impl(c);
    });
}

int plse_full_distances(plse_ctx* c) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        full_distances(c);
        CK(cudaStreamSynchronize(c->st));
    });
}

int plse_improve(plse_ctx* c, uint64_t generation, int64_t* iters_total, int32_t* best_f, int32_t* best_idx) {
    NvtxRange nvtx_("plse.improve");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        improve_impl(c, generation, -1, 0, nullptr, c->prm.p, 0);
        collect_improve(c, iters_total, best_f, best_idx);
    });
}

int plse_distances(plse_ctx* c) {
    NvtxRange nvtx_("plse.distances");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        c->ctr.k3_ops = 0;
        c->ctr.k3_tensor_cores = c->use_tc ? 1 : 0;
        phase_begin(c, PH_DIST);
        cross_distances(c);
        phase_end(c, PH_DIST);
    });
}

int plse_update(plse_ctx* c, int32_t* pool_best_f, int32_t* n_shortfall, int32_t* shortfall_slots) {
    NvtxRange nvtx_("plse.update");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        phase_begin(c, PH_UPDATE);
        update_impl(c, pool_best_f, n_shortfall, shortfall_slots);
        phase_end(c, PH_UPDATE);
    });
}

int plse_reset_exclusion(plse_ctx* c) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemsetAsync(c->d_excl, 0, 4ull * c->prm.p * c->excl_words, c->st));
        CK(cudaStreamSynchronize(c->st));
    });
}

int plse_offspring(plse_ctx* c, uint64_t generation) {
    NvtxRange nvtx_("plse.offspring");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        phase_begin(c, PH_OFFSPRING);
        offspring_impl(c, generation);
        phase_end(c, PH_OFFSPRING);
    });
}

int plse_trace(plse_ctx* c, int32_t idx, uint64_t generation, int64_t max_steps, plse_step* out, int64_t* n_out) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (idx < 0 || idx >= c->prm.p) throw std::invalid_argument("individual out of range");
        if (max_steps < 0 || (max_steps && !out)) throw std::invalid_argument("bad trace buffer");
        plse_step* d_tr = nullptr;
        if (max_steps) d_tr = dalloc<plse_step>((size_t)max_steps);
        try {
            improve_impl(c, generation, idx, max_steps, d_tr, idx + 1, idx);
            CK(cudaStreamSynchronize(c->st));
            int64_t it = 0;
            CK(cudaMemcpy(&it, c->d_iters + idx, 8, cudaMemcpyDeviceToHost));
            const int64_t m = std::min(it, max_steps);
            if (m) CK(cudaMemcpy(out, d_tr, sizeof(plse_step) * m, cudaMemcpyDeviceToHost));
            if (n_out) *n_out = it;
        } catch (...) {
            if (d_tr) cudaFree(d_tr);
            throw;
        }
        if (d_tr) cudaFree(d_tr);
    });
}

int plse_probe(plse_ctx* c, int32_t idx, uint64_t generation, int32_t n_steps, const int64_t* steps,
               int32_t* gamma_out, int32_t tabu_cap, int32_t* tabu_out, int32_t* n_tabu_out, int32_t* n_dumped,
               int32_t* cache_mismatch) {
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (c->ref_ties) throw Unsupported("the state probe covers the canonical kernels (PartialCol, PLITS)");
        if (idx < 0 || idx >= c->prm.p) throw std::invalid_argument("individual out of range");
        if (n_steps < 0 || tabu_cap < 0 || (n_steps && (!steps || !gamma_out || !n_tabu_out)) ||
            (tabu_cap && !tabu_out))
            throw std::invalid_argument("bad probe buffers");
        for (int q = 1; q < n_steps; ++q)
            if (steps[q] <= steps[q - 1]) throw std::invalid_argument("probe steps must ascend");
        const size_t gsz = (size_t)n_steps * c->nv * (c->n + 1);
        StateProbe pr{};
        pr.n = n_steps;
        pr.cap = tabu_cap;
        int64_t* d_steps = dalloc<int64_t>(std::max(n_steps, 1));
        int32_t* d_gamma = dalloc<int32_t>(std::max<size_t>(gsz, 1));
        int32_t* d_tabu = dalloc<int32_t>(std::max<size_t>((size_t)n_steps * tabu_cap * 3, 1));
        int32_t* d_small = dalloc<int32_t>(n_steps + 2);
        auto cleanup = [&] {
            cudaFree(d_steps);
            cudaFree(d_gamma);
            cudaFree(d_tabu);
            cudaFree(d_small);
        };
        try {
            if (n_steps) CK(cudaMemcpy(d_steps, steps, 8 * n_steps, cudaMemcpyHostToDevice));
            CK(cudaMemset(d_small, 0, 4 * (n_steps + 2)));
            pr.steps = d_steps;
            pr.gamma = d_gamma;
            pr.tabu = d_tabu;
            pr.n_tabu = d_small + 2;
            pr.dumped = d_small;
            pr.mismatch = d_small + 1;
            improve_impl(c, generation, idx, 0, nullptr, idx + 1, idx, &pr);
            CK(cudaStreamSynchronize(c->st));
            std::vector<int32_t> small(n_steps + 2);
            CK(cudaMemcpy(small.data(), d_small, 4 * (n_steps + 2), cudaMemcpyDeviceToHost));
            if (gsz) CK(cudaMemcpy(gamma_out, d_gamma, 4 * gsz, cudaMemcpyDeviceToHost));
            if (n_steps && tabu_cap)
                CK(cudaMemcpy(tabu_out, d_tabu, 12ull * n_steps * tabu_cap, cudaMemcpyDeviceToHost));
            if (n_steps) std::memcpy(n_tabu_out, small.data() + 2, 4 * n_steps);
            if (n_dumped) *n_dumped = small[0];
            if (cache_mismatch) *cache_mismatch = small[1];
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int plse_export_elites(plse_ctx* c, int32_t n_elite, void* dev_out, int32_t* f_out) {
    NvtxRange nvtx_("plse.export_elites");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        const int p = c->prm.p;
        if (n_elite < 0 || n_elite > p || (n_elite && !dev_out)) throw std::invalid_argument("bad elite count");
        // members in (illegal, f, slot) order on the device; the rows are written on the context's stream
        int32_t* d_f = nullptr;
        if (f_out && n_elite) d_f = c->d_tmpf;
        CK(launch_export_elites(c->d_mf, c->d_mc, c->nv, p, n_elite, c->d_members, c->nvpad, c->ps,
                                static_cast<uint8_t*>(dev_out), d_f, c->st));
        c->ctr.kernel_launches += 2 + (n_elite > 0);
        if (d_f) {
            CK(cudaMemcpyAsync(f_out, d_f, 4 * (size_t)n_elite, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
    });
}

int plse_import_migrants(plse_ctx* c, int32_t n_in, const void* dev_in) {
    NvtxRange nvtx_("plse.import_migrants");
    if (!c) return finish(nullptr, PLSE_ERR_INVALID, "null context");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        const int p = c->prm.p;
        if (n_in < 0 || n_in > 4 * p || (n_in && !dev_in)) throw std::invalid_argument("bad migrant count");
        if (n_in > c->mig_cap) {
            for (void* b : {(void*)c->d_migr, (void*)c->d_gf, (void*)c->d_gc, (void*)c->d_migd, (void*)c->d_hM})
                if (b) CK(cudaFree(b));
            c->d_migr = dalloc<uint8_t>((size_t)n_in * c->nvpad);
            c->d_gf = dalloc<int32_t>(n_in);
            c->d_gc = dalloc<int32_t>(n_in);
            c->d_migd = dalloc<uint16_t>((size_t)n_in * (2 * p + n_in));
            if (c->use_tc) c->d_hM = dalloc<uint8_t>((size_t)n_in * c->kpad);
            c->mig_cap = n_in;
        }
        c->n_mig = n_in;
        if (!n_in) return;
        CK(cudaMemcpyAsync(c->d_migr, dev_in, (size_t)n_in * c->nvpad, cudaMemcpyDeviceToDevice, c->st));
        eval_into(c, c->d_migr, c->d_gf, c->d_gc, n_in);
        // after this generation's plse_distances the one-hot operands are still in place: the migrant
        // block is computed now; otherwise plse_distances computes it
        if (c->onehot_valid || !c->use_tc) migrant_distances(c);
    });
}

int plse_stream(plse_ctx* c, void** stream_out) {
    if (!c || !stream_out) return finish(c, PLSE_ERR_INVALID, "null argument");
    *stream_out = c->st;
    return PLSE_OK;
}

// engine.hpp:114-262 (Partial-MPMA) on one device.
int plse_solve(int32_t n, const uint16_t* grid, const plse_solver_config* cfg, plse_run_result* res,
               uint16_t* best_colors, plse_generation_cb cb, void* user) {
    plse_ctx* ctx = nullptr;
    const int rc = guard(nullptr, [&] {
        if (!grid || !cfg || !res) throw std::invalid_argument("null argument");
        plse_params prm = cfg->params;
        prm.variant = cfg->variant;  // plse_solver_config::variant selects the improve operator
        validate_params(prm);
        const auto t0 = std::chrono::steady_clock::now();
        auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
        const plse_host::GraphH g = plse_host::preprocess(n, grid);
        std::memset(res, 0, sizeof(*res));
        res->l = g.l;
        res->upper_bound = g.l == 1 ? n * n - 2 : n * n - g.l;
        res->vertex_count = g.nv;
        res->best_f = g.nv;
        std::vector<uint16_t> best(g.nv, 0);
        double ttb = 0;
        auto finalize = [&](int reason) {
            res->best_score = n * n - g.l - res->best_f;
            res->proven_optimal = (res->best_f == 0 && g.l != 1) || (res->best_f == 1 && g.l == 1);
            res->stop_reason = res->proven_optimal ? PLSE_STOP_OPTIMAL : reason;
            res->elapsed_seconds = elapsed();
            res->time_to_best_seconds = ttb;
            if (best_colors) std::memcpy(best_colors, best.data(), 2 * best.size());
        };
        if (g.nv == 0) {
            res->best_f = 0;
            finalize(PLSE_STOP_TRIVIAL);
            return;
        }
        plse_graph view;
        view.order = g.n;
        view.vertex_count = g.nv;
        view.l = g.l;
        view.cell_row = g.cell_row.data();
        view.cell_col = g.cell_col.data();
        view.dom_offsets = g.dom_off.data();
        view.dom = g.dom.data();
        view.n_prefilled = (int32_t)(g.prefilled.size() / 3);
        view.prefilled = g.prefilled.data();
        create_impl(&view, &prm, cfg->device, &ctx);
        plse_ctx* c = ctx;
        const int p = c->prm.p;
        const bool opt_stop = !cfg->disable_optimal_stop;
        auto is_opt = [&](int f) { return (f == 0 && g.l != 1) || (f == 1 && g.l == 1); };
        auto fetch_row = [&](uint8_t* buf, int i) {
            std::vector<uint8_t> row(c->nvpad);
            CK(cudaMemcpy(row.data(), buf + (size_t)i * c->nvpad, c->nvpad, cudaMemcpyDeviceToHost));
            for (int v = 0; v < g.nv; ++v) best[v] = row[v];
        };
        init_impl(c);
        {
            std::vector<int32_t> mf, mc;
            fetch_fc(c, PLSE_MEMBERS, mf, mc);
            for (int i = 0; i < p; ++i)
                if (mc[i] == 0 && mf[i] < res->best_f) {
                    res->best_f = mf[i];
                    fetch_row(c->d_members, i);
                    ttb = elapsed();
                }
        }
        if (opt_stop && is_opt(res->best_f)) {
            finalize(PLSE_STOP_OPTIMAL);
            return;
        }
        CK(cudaMemcpy(c->d_offspring, c->d_members, (size_t)p * c->nvpad, cudaMemcpyDeviceToDevice));
        CK(cudaMemset(c->d_excl, 0, 4ull * p * c->excl_words));
        if (cfg->race && cfg->target_score > 0) {
            c->d_race = dalloc<int>(1);
            CK(cudaMemset(c->d_race, 0, sizeof(int)));
            c->race_f = std::max(0, (int)std::floor((double)(n * n - g.l) - cfg->target_score));
        }
        if (cfg->time_limit > 0) {
            // partial.hpp:165: each search checks the deadline every 4096 steps
            c->d_deadline = dalloc<unsigned long long>(1);
            const double remaining = std::max(0.0, cfg->time_limit - elapsed());
            k_set_deadline<<<1, 1, 0, c->st>>>(c->d_deadline, (unsigned long long)(remaining * 1e9));
            CK(cudaGetLastError());
        }
        auto emit_stats = [&](int64_t gen, int shortfall) {
            if (!cb) return;
            plse_generation_stats st{};
            st.generation = gen;
            st.best_f = res->best_f;
            std::vector<int32_t> mf, mc;
            fetch_fc(c, PLSE_MEMBERS, mf, mc);
            double fs = 0;
            for (int i = 0; i < p; ++i) fs += mf[i];
            st.mean_f = fs / p;
            if (!c->d_dsum) c->d_dsum = dalloc<unsigned long long>(1);
            CK(cudaMemsetAsync(c->d_dsum, 0, 8, c->st));
            k_upper_sum<<<std::min(p, 4 * 148), 256, 0, c->st>>>(c->d_dist, p, c->d_dsum);
            CK(cudaGetLastError());
            unsigned long long ds = 0;
            CK(cudaMemcpyAsync(&ds, c->d_dsum, 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
            st.mean_distance = (double)ds / (0.5 * p * (p - 1));
            st.iterations = res->total_iterations;
            st.elapsed_seconds = elapsed();
            st.shortfall = shortfall;
            cb(&st, user);
        };
        for (int64_t gen = 1;; ++gen) {
            int64_t it = 0;
            int32_t bf = 0, bi = -1;
            {
                NvtxRange r_("plse.solve.improve");
                improve_impl(c, (uint64_t)gen, -1, 0, nullptr, p, 0);
                collect_improve(c, &it, &bf, &bi);
            }
            res->total_iterations += it;
            res->generations = gen;
            if (bi >= 0 && bf < res->best_f) {
                res->best_f = bf;
                fetch_row(c->d_improved, bi);
                ttb = elapsed();
            }
            const bool optimal = opt_stop && is_opt(res->best_f);
            const bool time_up = cfg->time_limit > 0 && elapsed() >= cfg->time_limit;
            const bool iters_up = cfg->iteration_limit > 0 && res->total_iterations >= cfg->iteration_limit;
            const bool gens_up = cfg->generation_limit > 0 && gen >= cfg->generation_limit;
            const bool target = cfg->target_score > 0 && (n * n - g.l - res->best_f) >= cfg->target_score;
            if (optimal || time_up || iters_up || gens_up || target) {
                emit_stats(gen, 0);
                finalize(optimal ? PLSE_STOP_OPTIMAL
                         : time_up ? PLSE_STOP_TIME
                         : iters_up ? PLSE_STOP_ITERS
                         : gens_up ? PLSE_STOP_GENS
                                   : PLSE_STOP_TARGET);
                return;
            }
            int32_t nsf = 0;
            {
                NvtxRange r_("plse.solve.population");
                cross_distances(c);
                update_impl(c, nullptr, cb ? &nsf : nullptr, nullptr);
            }
            if (c->prm.exclusion == PLSE_E_GENERATION) CK(cudaMemset(c->d_excl, 0, 4ull * p * c->excl_words));
            offspring_impl(c, (uint64_t)gen);
            emit_stats(gen, nsf);
        }
    });
    delete ctx;
    return rc;
}

}  // extern "C"
