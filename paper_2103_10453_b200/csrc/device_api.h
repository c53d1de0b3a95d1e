// device_api.h -- internal interface between the host context (capi.cu) and
// the sm_100a kernels.  Not part of the public C ABI (include/plse_b200.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "plse_b200.h"

namespace plse_dev {

constexpr int kImproveMaxThreads = 256;
constexpr int kImproveMinBlocks = 4;  // 32 resident warps per SM -> <= 64 registers
// k_improve: up to 28 warps in ONE CTA per SM, so the graph tables are staged once per SM
constexpr int kPadMaxThreads = 896;  // 28 warps per SM: 72 registers per thread (32 warps cap them at 64)

// state probe of the per-step parity contract (plse_probe): gamma table and live tabu entries of the
// traced individual at chosen steps
struct StateProbe {
    int n;                 // probe points (0 = off)
    const int64_t* steps;  // ascending step indices (the state before step j; j = 0 is the post-repair state)
    int32_t* gamma;        // n x nv x (order+1)
    int32_t* tabu;         // n x cap x 3: (v, k, until on the reference's iteration clock)
    int32_t* n_tabu;       // n: live entries (may exceed cap)
    int32_t* dumped;       // [1] probe points reached
    int32_t* mismatch;     // [1] vertices whose tabu cache disagrees with the dense table
    int cap;
};

struct ImproveArgs {
    // graph (global copies; the kernel stages them in shared memory)
    int n, nv, nvpad, lane_words, lane_words16;
    const uint16_t* cell;       // [nv] row << 8 | col
    const uint16_t* row_start;  // [n+1] survivors of row r are ids [row_start[r], row_start[r+1])
    const uint16_t* col_start;  // [n+1]
    const uint16_t* col_list;   // [nv] survivors grouped by column, ascending
    const uint64_t* pre_row;    // [n*W] prefilled symbols per row
    const uint64_t* pre_col;    // [n*W]
    // population
    int p;
    const uint8_t* offspring;   // [p*nvpad]
    uint8_t* improved;          // [p*nvpad]
    int32_t* best_f;
    int32_t* repaired_f;
    int64_t* iters;
    unsigned long long* bytes;
    // per-warp-slot tabu scratch
    void* tabu_rec;
    size_t rec_stride;          // bytes per slot
    uint32_t* until;
    size_t until_stride;        // u32 per slot (multiple of 4)
    uint32_t* slot_clock;       // per slot: tabu clock base of its next individual
    uint32_t tenure_cap;        // 10 + floor(alpha*|V|) > any tenure
    int* work_counter;          // zeroed per launch; individuals past the first per slot are pulled from it
    int first;                  // individuals [first, p) are searched
    int nslots;                 // warp slots that search (<= resident slots; balanced rounds)
    // streams (engine.hpp:189-191): seed = derive(master, 2, gen*p_total + offset + i)
    uint64_t master, generation, p_total, offset;
    int64_t budget;
    int64_t budget2;            // PLITS phase-2 budget (plits.hpp:244); unused by PartialCol
    int stop_f;
    double alpha;
    // per-slot repair counters (nvpad bytes each; the warp kernel keeps them out of shared memory)
    uint8_t* conf_scratch;
    size_t conf_stride;
    // race mode (time-to-target): stop every search once any individual reaches best f <= race_f
    int* race_flag;             // nullptr = off
    int race_f;
    // time limit (partial.hpp:165): after every 4096th step, stop once %globaltimer >= *deadline
    const unsigned long long* deadline;  // nullptr = no limit
    // optional clock64 instrumentation (PLSE_PROFILE=1): 16 counters, see capi.cu
    unsigned long long* prof;
    // parity probe
    int trace_idx;
    int64_t trace_cap;
    void* trace;
    StateProbe probe;
    // k_improve's padded colour copies (host-built tables, staged in shared memory): each row (column) of
    // the grid starts on an 8-byte boundary of the row-padded (column-padded) copy, 0xFF in the gaps, so
    // the holder of a colour in a row or column is one aligned 8-byte load per lane
    const uint16_t* rpos;   // [nv] byte of v in the row-padded copy
    const uint16_t* cpos;   // [nv] byte of v in the column-padded copy (column lists' order)
    const uint64_t* rinfo;  // [n] offset | 8-byte words << 16 | first vertex << 32
    const uint64_t* cinfo;  // [n] offset | 8-byte words << 16 | column-list base << 32
    int rp_bytes, cp_bytes; // sizes of the two copies (multiples of 16)
};

struct PadSmemLayout {
    size_t cell, rs, cs, cl, rpos, cpos, deg, rinfo, cinfo, pr, pc, graph_bytes;
    size_t warp0, warp_bytes, w_rp, w_cp, w_list, w_seed, w_R, w_C, w_U;
};

__host__ __device__ inline size_t align_up_(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline PadSmemLayout pad_smem_layout(int n, int nv, int lane_words, int W, int rp_bytes,
                                                         int cp_bytes) {
    PadSmemLayout L;
    size_t o = 0;
    L.cell = o;
    o += (size_t)nv * 2;
    L.rs = o;
    o += (size_t)(n + 1) * 2;
    L.cs = o;
    o += (size_t)(n + 1) * 2;
    L.cl = o;
    o += (size_t)nv * 2;
    L.rpos = o;
    o += (size_t)nv * 2;
    L.cpos = o;
    o += (size_t)nv * 2;
    L.deg = o;
    o += (size_t)nv;
    o = align_up_(o, 16);
    L.rinfo = o;
    o += (size_t)n * 8;
    L.cinfo = o;
    o += (size_t)n * 8;
    L.pr = o;  // n + 1 lines: line n is the all-prefilled dummy line of the empty slot-list lanes
    o += (size_t)(n + 1) * W * 8;
    L.pc = o;
    o += (size_t)(n + 1) * W * 8;
    o = align_up_(o, 16);
    L.graph_bytes = o;
    L.warp0 = o;
    size_t w = 0;
    L.w_rp = w;
    w += (size_t)rp_bytes;
    L.w_cp = w;
    w += (size_t)cp_bytes;
    L.w_list = w;
    w += 64;
    L.w_seed = w;  // the individual's 64-bit stream seed (read when a 32-step draw window is refilled)
    w += 16;
    w = align_up_(w, 16);
    L.w_R = w;  // n + 1 lines (line n: the dummy line, always empty)
    w += (size_t)(n + 1) * W * 8;
    L.w_C = w;
    w += (size_t)(n + 1) * W * 8;
    L.w_U = w;
    w += (size_t)32 * lane_words * 4;
    L.warp_bytes = align_up_(w, 16);
    return L;
}

struct ImproveSmemLayout {
    size_t cell, rs, cs, cl, colpos, deg, pr, pc, graph_bytes;
    size_t warp0, warp_bytes, w_col, w_colT, w_list, w_R, w_C, w_U;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline ImproveSmemLayout improve_smem_layout(int n, int nv, int nvpad, int lane_words, int W) {
    ImproveSmemLayout L;
    size_t o = 0;
    L.cell = o;
    o += (size_t)nv * 2;
    L.rs = o;
    o += (size_t)(n + 1) * 2;
    L.cs = o;
    o += (size_t)(n + 1) * 2;
    L.cl = o;
    o += (size_t)nv * 2;
    L.colpos = o;
    o += (size_t)nv * 2;
    L.deg = o;
    o += (size_t)nv;
    o = align_up(o, 16);
    L.pr = o;
    o += (size_t)n * W * 8;
    L.pc = o;
    o += (size_t)n * W * 8;
    o = align_up(o, 16);
    L.graph_bytes = o;
    L.warp0 = o;
    size_t w = 0;
    L.w_col = w;
    w += (size_t)nvpad;
    L.w_colT = w;  // column-major colour copy (ordered like the column lists)
    w += (size_t)nvpad;
    L.w_list = w;  // the 32-entry u16 list that seeds sparse mode (repair counters live in HBM scratch)
    w += 64;
    w = align_up(w, 16);
    L.w_R = w;
    w += (size_t)n * W * 8;
    L.w_C = w;
    w += (size_t)n * W * 8;
    L.w_U = w;
    w += (size_t)32 * lane_words * 4;
    L.warp_bytes = align_up(w, 16);
    return L;
}

// PLITS (plits.cu): graph part as improve_smem_layout, per warp: colours, bit-sliced row /
// column colour counts ((5 + W) planes of W words per line), the active-vertex bitmask, the
// compacted active list and a per-listed-vertex scratch word
constexpr int kPlitsMaxThreads = 256;
constexpr int kPlitsMinBlocks = 2;  // <= 128 registers

struct PlitsSmemLayout {
    size_t graph_bytes, warp0, warp_bytes, w_col, w_rp, w_cp, w_A, w_list, w_vmin, w_vcnt;
};

__host__ __device__ inline PlitsSmemLayout plits_smem_layout(int n, int nv, int nvpad, int lane_words, int W) {
    const ImproveSmemLayout G = improve_smem_layout(n, nv, nvpad, lane_words, W);
    PlitsSmemLayout L;
    L.graph_bytes = G.graph_bytes;
    L.warp0 = G.warp0;
    const size_t planes = (size_t)n * (5 + W) * W * 8;
    size_t w = 0;
    L.w_col = w;
    w += (size_t)nvpad;
    w = align_up(w, 16);
    L.w_rp = w;
    w += planes;
    L.w_cp = w;
    w += planes;
    L.w_A = w;
    w += (size_t)32 * lane_words * 4;
    L.w_list = w;
    w += align_up((size_t)nv * 2, 16);
    L.w_vmin = w;
    w += (size_t)nv * 4;
    L.w_vcnt = w;
    w += (size_t)nv;
    L.warp_bytes = align_up(w, 16);
    return L;
}

// PLITS with the reference's tie-break (plits_ref.cu): colours, count planes, the two IndexSets,
// possibly-tabu masks, a 32-vertex staging area and a neighbour scratch list per warp
struct PlitsRefSmemLayout {
    size_t graph_bytes, warp0, warp_bytes, w_col, w_rp, w_cp, w_un_el, w_un_pos, w_cf_el, w_cf_pos, w_T, w_stage,
        w_stage_i, w_evl;
};

__host__ __device__ inline PlitsRefSmemLayout plits_ref_smem_layout(int n, int nv, int nvpad, int lane_words, int W) {
    const ImproveSmemLayout G = improve_smem_layout(n, nv, nvpad, lane_words, W);
    PlitsRefSmemLayout L;
    L.graph_bytes = G.graph_bytes;
    L.warp0 = G.warp0;
    const size_t planes = (size_t)n * (5 + W) * W * 8, ids = align_up((size_t)nv * 2, 16);
    size_t w = 0;
    L.w_col = w;
    w += (size_t)nvpad;
    w = align_up(w, 16);
    L.w_rp = w;
    w += planes;
    L.w_cp = w;
    w += planes;
    L.w_un_el = w;
    w += ids;
    L.w_un_pos = w;
    w += ids;
    L.w_cf_el = w;
    w += ids;
    L.w_cf_pos = w;
    w += ids;
    L.w_T = 0;  // the possibly-tabu mask lives in global memory (plits_ref.cu)
    L.w_stage = w;
    w += (size_t)32 * (5 + W + 2) * W * 8;
    L.w_stage_i = w;
    w += 32 * 5 * 4;
    L.w_evl = w;
    w += align_up((size_t)2 * n * 2, 16);
    L.warp_bytes = align_up(w, 16);
    return L;
}

const void* plits_ref_kernel_ptr(int W, bool debug);
cudaError_t launch_plits_ref(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st);

const void* plits_kernel_ptr(int W, bool debug);
cudaError_t launch_plits(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st);

// PartialCol with the reference's tie-break (improve_ref.cu): improve's layout plus the IndexSet-ordered
// uncoloured list and a 32-vertex mask staging area per warp
struct RefSmemLayout {
    size_t graph_bytes, warp0, warp_bytes, w_col, w_colT, w_R, w_C, w_U, w_el, w_msk;
};

__host__ __device__ inline RefSmemLayout improve_ref_smem_layout(int n, int nv, int nvpad, int lane_words, int W) {
    const ImproveSmemLayout G = improve_smem_layout(n, nv, nvpad, lane_words, W);
    RefSmemLayout L;
    L.graph_bytes = G.graph_bytes;
    L.warp0 = G.warp0;
    size_t w = 0;
    L.w_col = w;
    w += (size_t)nvpad;
    L.w_colT = w;
    w += (size_t)nvpad;
    w = align_up(w, 16);
    L.w_R = w;
    w += (size_t)n * W * 8;
    L.w_C = w;
    w += (size_t)n * W * 8;
    L.w_U = w;
    w += (size_t)32 * lane_words * 4;
    w = align_up(w, 16);
    L.w_el = w;
    w += align_up((size_t)nv * 2, 16);
    L.w_msk = w;
    w += (size_t)32 * 3 * W * 8;
    L.warp_bytes = align_up(w, 16);
    return L;
}

const void* improve_ref_kernel_ptr(int W, bool debug);
cudaError_t launch_improve_ref(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st);

size_t tabu_rec_bytes(int W);
const void* improve_kernel_ptr(int W, bool debug);
cudaError_t launch_improve(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st);

// ---- distances (K3)
// D[i][j] = #{v : A_i[v] != B_j[v]} for u8 rows with stride nvpad (pad bytes equal)
// upper != 0 (A == B, square): tiles strictly below the diagonal are skipped (the consumer reads [min][max])
cudaError_t launch_hamming(const uint8_t* A, int na, const uint8_t* B, int nb, int nv, int nvpad, uint16_t* D,
                           int ldd, cudaStream_t st, int upper = 0);

// K3 on tcgen05 (similarity_tc.cu): one-hot expansion + i8 UMMA GEMM, D = |V| - A.B^T
cudaError_t launch_onehot(const uint8_t* X, int rows, int nvpad, const uint16_t* col_vert, const uint8_t* col_color,
                          int K, int Kpad, uint8_t* H, cudaStream_t st);
cudaError_t prepare_similarity_tc();
cudaError_t launch_similarity_tc(const uint8_t* HA, int M, const uint8_t* HB, int N, int Kpad, int nv, uint16_t* D,
                                 int ldd, cudaStream_t st, int upper = 0);

// ---- population kernels (population.cu)
struct PopGraph {
    int n, nv, nvpad;
    const uint16_t* cell;
    const uint16_t* row_start;
    const uint16_t* col_start;
    const uint16_t* col_list;
    const int32_t* dom_off;
    const uint8_t* dom;
    const uint64_t* below_thr;  // [n+1] (2^64 - b) % b for b = 1..n
};
cudaError_t launch_init_population(const PopGraph& g, int p, uint64_t master, uint64_t offset, uint8_t* members,
                                   cudaStream_t st);
cudaError_t launch_eval_fc(const PopGraph& g, int p, const uint8_t* colors, int32_t* f, int32_t* c,
                           cudaStream_t st);
cudaError_t launch_match(const uint16_t* dist, int p, int matching, int exclusion, uint32_t* excl, int excl_words,
                         uint64_t master, uint64_t stream_base, int32_t* partner, cudaStream_t st);
cudaError_t launch_crossover(const uint8_t* members, const uint16_t* dist, const int32_t* partner, int p, int nv,
                             int nvpad, int mode, double beta, uint64_t master, uint64_t stream_base,
                             uint8_t* offspring, cudaStream_t st);
// ---- pool update (pool.cu): population.hpp:103-183 on the device
struct PoolView {
    int p, m;               // members = improved count, migrant count
    const uint16_t* dist;   // members x members (full)
    const uint16_t* cross;  // members x improved
    const uint16_t* fresh;  // improved x improved, upper triangle (i <= j) valid
    const uint16_t* migd;   // m x (2p + m): migrant vs members | improved | migrants
};
struct PoolFC {             // f and c of every pool id
    int p, m;
    const int32_t *mf, *mc, *imf, *imc, *gf, *gc;
};
struct PoolScratch {
    uint64_t *keys0, *keys1;
    int32_t *order, *sel, *nsel, *slots, *info;  // info[0] = pool_best_f, info[1] = shortfall count
    uint8_t *legal, *admitted, *ok;
    uint32_t* conf;
};
struct ImproveSummary {
    int64_t iters;
    unsigned long long bytes;
    int32_t best_f, best_idx;
};
cudaError_t prepare_pool_update();
cudaError_t launch_pool_update(const PoolView& pv, const PoolFC& fc, const PoolScratch& w, int nv, int dthr,
                               const uint8_t* members, const uint8_t* improved, const uint8_t* migrants,
                               uint8_t* next_members, uint16_t* next_dist, int32_t* next_f, int32_t* next_c,
                               int nvpad, cudaStream_t st, int64_t* launches);
cudaError_t launch_improve_reduce(const int32_t* best_f, const int64_t* iters, const unsigned long long* bytes,
                                  int p, ImproveSummary* out, cudaStream_t st);
cudaError_t launch_export_elites(const int32_t* mf, const int32_t* mc, int nv, int p, int n_elite,
                                 const uint8_t* members, int nvpad, const PoolScratch& w, uint8_t* out,
                                 int32_t* fout, cudaStream_t st);
cudaError_t launch_u16_to_i32(const uint16_t* in, int32_t* out, size_t count, cudaStream_t st);
cudaError_t launch_i32_to_u16(const int32_t* in, uint16_t* out, size_t count, cudaStream_t st);
cudaError_t launch_colors_u16_to_u8(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad, cudaStream_t st);
cudaError_t launch_colors_u8_to_u16(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad, cudaStream_t st);

}  // namespace plse_dev
