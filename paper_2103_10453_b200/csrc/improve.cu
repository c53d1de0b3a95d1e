// improve.cu -- K1 + K1b + K2: the Partial-MPMA improve phase on sm_100a.
//
// Replaces the reference's per-individual loop
//   engine.hpp:184-209 -> partial_mpma_improve (partial.hpp:156-169)
//     -> PartialColSearch ctor (76-85: gamma build coloring.hpp:105-116,
//        repair partial.hpp:22-39) -> step() (92-143)
// with ONE WARP PER INDIVIDUAL, persistent over a work counter.
//
// Data layout:
//   * The individual's colours (u8) live in shared memory for the whole
//     search, together with per-row / per-column colour-occupancy bitmasks
//     R[r], C[c] (W x u64 each) and the uncoloured set U as a bitmask.
//     In a legal colouring gamma[v][k] = [k in R[row v]] + [k in C[col v]]
//     for every uncoloured v, so the three move classes of an uncoloured
//     vertex (delta -1 / 0 / +1) are three W-word mask expressions -- the
//     int16 gamma rows of the north star are never materialised.
//   * The domain of v is ~(PR[row] | PC[col]) over the prefilled-symbol masks
//     (lsgraph.hpp:152-156), shared by the CTA in shared memory.
//   * Tabu state (search_util.hpp:54-81) is per warp slot in HBM/L2: a dense
//     u32 `until[v][k]` table (the reference layout) plus a 16/32-byte record
//     per vertex {tabu-bit mask, max until, exact flag} so that the common
//     case costs one vector load per uncoloured vertex per step.
//   * Selection is the canonical order-free rule: count the
//     admissible candidates per delta level per lane, warp-scan the counts of
//     the lowest non-empty level, draw r = floor(u32 * N / 2^32) from the
//     counter-based stream, and let the lane holding the r-th candidate (in
//     ascending (v, k) order) recover it with a popcount search.
#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

template <int W>
struct alignas(16) TabuRec {
    uint64_t tm[W];
    uint32_t umax;
    uint32_t exact;
};

struct WarpSmem {
    uint8_t* col;
    uint8_t* conf;
    uint64_t* R;
    uint64_t* C;
    uint32_t* U;
};

template <int W>
struct Graph {
    int n, nv, nvpad, lane_words;
    const uint16_t* cell;
    const uint16_t* rs;
    const uint16_t* cs;
    const uint16_t* cl;
    const uint64_t* pr;
    const uint64_t* pc;
    uint64_t full[W];
};

template <int W>
__device__ __forceinline__ void tabu_mask(TabuRec<W>* rec, const uint32_t* until, int w1, int v, uint32_t j,
                                          uint64_t (&T)[W]) {
    TabuRec<W> r = rec[v];
    if (r.umax <= j) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < W; ++q) {
            any |= r.tm[q] != 0;
            T[q] = 0;
        }
        if (any) {
            TabuRec<W> z;
#pragma unroll
            for (int q = 0; q < W; ++q) z.tm[q] = 0;
            z.umax = 0;
            z.exact = 1;
            rec[v] = z;
        }
        return;
    }
    int pc = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) pc += __popcll(r.tm[q]);
    if (r.exact && pc == 1) {
#pragma unroll
        for (int q = 0; q < W; ++q) T[q] = r.tm[q];
        return;
    }
    // slow path: verify every set bit against the dense until table, recompute umax
    uint32_t um = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t m = r.tm[q];
        uint64_t keep = 0;
        while (m) {
            const int b = __ffsll((long long)m) - 1;
            m &= m - 1;
            const uint32_t u = until[(size_t)v * w1 + q * 64 + b];
            if (u > j) {
                keep |= 1ULL << b;
                um = max(um, u);
            }
        }
        r.tm[q] = keep;
        T[q] = keep;
    }
    r.umax = um;
    r.exact = 1;
    rec[v] = r;
}

// Admissible candidate masks of an uncoloured vertex v at the three delta levels.
template <int W>
__device__ __forceinline__ void cand_masks(const Graph<W>& g, const WarpSmem& s, TabuRec<W>* rec,
                                           const uint32_t* until, int v, uint32_t j, bool asp,
                                           uint64_t (&m0)[W], uint64_t (&m1)[W], uint64_t (&m2)[W]) {
    const uint16_t rc = g.cell[v];
    const int r = rc >> 8, c = rc & 0xFF;
    uint64_t T[W];
    tabu_mask<W>(rec, until, g.n + 1, v, j, T);
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const uint64_t dom = ~(g.pr[r * W + q] | g.pc[c * W + q]) & g.full[q];
        const uint64_t Rr = s.R[r * W + q], Cc = s.C[c * W + q];
        const uint64_t fr = dom & ~Rr & ~Cc;
        m0[q] = asp ? fr : (fr & ~T[q]);
        m1[q] = dom & (Rr ^ Cc) & ~T[q];
        m2[q] = dom & Rr & Cc & ~T[q];
    }
}

template <int W>
__device__ __forceinline__ int popc_w(const uint64_t (&m)[W]) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) c += __popcll(m[q]);
    return c;
}

__device__ __forceinline__ void snapshot(const uint8_t* col, uint8_t* dst, int nvpad, int lane) {
    const uint4* s4 = reinterpret_cast<const uint4*>(col);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int t = lane; t < nvpad / 16; t += 32) d4[t] = s4[t];
}

template <int W>
__device__ void improve_one(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, TabuRec<W>* rec,
                            uint32_t* until, int i, int lane) {
    const int n = g.n, nv = g.nv, w1 = n + 1;
    const int B = 32 * g.lane_words;
    const int v_lo = lane * B;
    const int v_hi = min(nv, v_lo + B);
    uint8_t* col = s.col;
    uint8_t* conf = s.conf;

    // ---- load the offspring (u8, row stride nvpad) and reset this slot's tabu records
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.offspring + (size_t)i * g.nvpad);
        uint4* d4 = reinterpret_cast<uint4*>(col);
        for (int t = lane; t < g.nvpad / 16; t += 32) d4[t] = src[t];
        TabuRec<W> z;
#pragma unroll
        for (int q = 0; q < W; ++q) z.tm[q] = 0;
        z.umax = 0;
        z.exact = 1;
        for (int t = lane; t < nv; t += 32) rec[t] = z;
    }
    __syncwarp();

    // ---- K1: conflict counts gamma[v][col v] of coloured vertices (coloring.hpp:105-116)
    for (int v = v_lo; v < v_hi; ++v) {
        const int k = col[v];
        int cnt = 0;
        if (k) {
            const uint16_t rc = g.cell[v];
            const int r = rc >> 8, c = rc & 0xFF;
            for (int u = g.rs[r]; u < g.rs[r + 1]; ++u) cnt += col[u] == k;
            for (int t = g.cs[c]; t < g.cs[c + 1]; ++t) cnt += col[g.cl[t]] == k;
            cnt -= 2;  // v itself in its row and its column
        }
        conf[v] = (uint8_t)cnt;
    }
    __syncwarp();

    // ---- K1b: greedy repair, argmax conflicts with lowest-index ties (partial.hpp:22-39)
    for (;;) {
        int bc = 0, bv = -1;
        for (int v = v_lo; v < v_hi; ++v) {
            const int c = conf[v];
            if (c > bc) {
                bc = c;
                bv = v;
            }
        }
        const int mx = __reduce_max_sync(kFull, (unsigned)bc);
        if (mx == 0) break;
        const int wl = __ffs(__ballot_sync(kFull, bc == mx)) - 1;
        const int w = __shfl_sync(kFull, bv, wl);
        const int k = col[w];
        const uint16_t rc = g.cell[w];
        const int r = rc >> 8, c = rc & 0xFF;
        for (int u = g.rs[r] + lane; u < g.rs[r + 1]; u += 32)
            if (u != w && col[u] == k) conf[u] -= 1;
        for (int t = g.cs[c] + lane; t < g.cs[c + 1]; t += 32) {
            const int u = g.cl[t];
            if (u != w && col[u] == k) conf[u] -= 1;
        }
        __syncwarp();
        if (lane == 0) {
            col[w] = 0;
            conf[w] = 0;
        }
        __syncwarp();
    }

    // ---- occupancy masks R/C and uncoloured bitmask U of the (now legal) colouring
    for (int t = lane; t < n * W; t += 32) {
        s.R[t] = 0;
        s.C[t] = 0;
    }
    __syncwarp();
    int fl = 0;
    for (int q = 0; q < g.lane_words; ++q) {
        const int base = v_lo + 32 * q;
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            const int v = base + b;
            if (v >= nv) break;
            const int k = col[v];
            if (!k) {
                bits |= 1u << b;
            } else {
                const uint16_t rc = g.cell[v];
                atomicOr((unsigned long long*)&s.R[(rc >> 8) * W + (k >> 6)], 1ULL << (k & 63));
                atomicOr((unsigned long long*)&s.C[(rc & 0xFF) * W + (k >> 6)], 1ULL << (k & 63));
            }
        }
        s.U[lane * g.lane_words + q] = bits;
        fl += __popc(bits);
    }
    int f = (int)__reduce_add_sync(kFull, (unsigned)fl);
    __syncwarp();

    const int repaired_f = f;
    int bestf = f;
    bool pending = true;  // best_ == current (partial.hpp:84)
    uint32_t j = 0;
    unsigned long long bytes = 0;
    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    const bool tracing = (i == a.trace_idx) && a.trace != nullptr;

    while ((int64_t)j < a.budget && bestf > a.stop_f && f > 0) {
        const bool asp = (f == bestf);
        // ---- phase A: admissible counts per level over this lane's uncoloured vertices
        int c0 = 0, c1 = 0, c2 = 0;
        for (int q = 0; q < g.lane_words; ++q) {
            uint32_t bits = s.U[lane * g.lane_words + q];
            while (bits) {
                const int v = v_lo + 32 * q + __ffs(bits) - 1;
                bits &= bits - 1;
                uint64_t m0[W], m1[W], m2[W];
                cand_masks<W>(g, s, rec, until, v, j, asp, m0, m1, m2);
                c0 += popc_w<W>(m0);
                c1 += popc_w<W>(m1);
                c2 += popc_w<W>(m2);
            }
        }
        const unsigned b0 = __ballot_sync(kFull, c0 > 0);
        const unsigned b1 = __ballot_sync(kFull, c1 > 0);
        const unsigned b2 = __ballot_sync(kFull, c2 > 0);
        const int lvl = b0 ? -1 : b1 ? 0 : b2 ? 1 : 2;
        const int cnt = lvl == -1 ? c0 : lvl == 0 ? c1 : lvl == 1 ? c2 : 0;
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += t;
        }
        const int N = __shfl_sync(kFull, incl, 31);
        const uint64_t x = canon_draw(seed, j);
        const int f_before = f;
        unsigned long long bt = 2ULL * (unsigned)w1 * (unsigned)f_before;
        if (N == 0) {
            // every candidate tabu: no move, the clock still advances (partial.hpp:121-122)
            if (tracing && lane == 0 && (int64_t)j < a.trace_cap) {
                plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + j;
                tr->step = j;
                tr->v = -1;
                tr->k = 0;
                tr->e = 0;
                tr->ev0 = tr->ev1 = -1;
                tr->f_before = tr->f_after = f;
                tr->best_f = bestf;
                tr->tenure = -1;
                tr->n_adm = 0;
                tr->level = 2;
            }
            bytes += bt;
            ++j;
            continue;
        }
        const uint32_t r = (uint32_t)(((x >> 32) * (uint64_t)(uint32_t)N) >> 32);
        const unsigned wb = __ballot_sync(kFull, (uint32_t)(incl - cnt) <= r && r < (uint32_t)incl);
        const int wl = __ffs(wb) - 1;
        // ---- phase B: the winner lane recovers its (r - prefix)-th candidate in (v, k) order
        int vs = -1, ks = 0;
        if (lane == wl) {
            int rr = (int)r - (incl - cnt);
            for (int q = 0; q < g.lane_words && vs < 0; ++q) {
                uint32_t bits = s.U[lane * g.lane_words + q];
                while (bits) {
                    const int v = v_lo + 32 * q + __ffs(bits) - 1;
                    bits &= bits - 1;
                    uint64_t m0[W], m1[W], m2[W];
                    cand_masks<W>(g, s, rec, until, v, j, asp, m0, m1, m2);
                    uint64_t m[W];
#pragma unroll
                    for (int z = 0; z < W; ++z) m[z] = lvl == -1 ? m0[z] : lvl == 0 ? m1[z] : m2[z];
                    const int pc = popc_w<W>(m);
                    if (rr < pc) {
#pragma unroll
                        for (int z = 0; z < W; ++z) {
                            const int pz = __popcll(m[z]);
                            if (vs < 0) {
                                if (rr < pz) {
                                    ks = z * 64 + nth_bit64(m[z], rr);
                                    vs = v;
                                } else {
                                    rr -= pz;
                                }
                            }
                        }
                        break;
                    }
                    rr -= pc;
                }
            }
        }
        vs = __shfl_sync(kFull, vs, wl);
        ks = __shfl_sync(kFull, ks, wl);

        // ---- apply (partial.hpp:124-141)
        if (pending && lvl >= 0) {
            // the current colouring is the best one and is about to change without improving
            snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
            pending = false;
        }
        const uint16_t rcs = g.cell[vs];
        const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
        const int kw = ks >> 6;
        const uint64_t bitk = 1ULL << (ks & 63);
        const bool inR = (s.R[rs_ * W + kw] & bitk) != 0;
        const bool inC = (s.C[cs_ * W + kw] & bitk) != 0;
        int ur = -1, uc = -1;
        if (inR) {
            for (int base = g.rs[rs_]; base < g.rs[rs_ + 1]; base += 32) {
                const int u = base + lane;
                const unsigned hit = __ballot_sync(kFull, u < g.rs[rs_ + 1] && col[u] == ks);
                if (hit) {
                    ur = base + __ffs(hit) - 1;
                    break;
                }
            }
        }
        if (inC) {
            for (int base = g.cs[cs_]; base < g.cs[cs_ + 1]; base += 32) {
                const int t = base + lane;
                const int u = t < g.cs[cs_ + 1] ? g.cl[t] : 0;
                const unsigned hit = __ballot_sync(kFull, t < g.cs[cs_ + 1] && col[u] == ks);
                if (hit) {
                    uc = __shfl_sync(kFull, u, __ffs(hit) - 1);
                    break;
                }
            }
        }
        const int e = (ur >= 0) + (uc >= 0);
        int deg_bytes = 0;
        {
            auto deg = [&](int v) {
                const uint16_t rc = g.cell[v];
                const int r_ = rc >> 8, c_ = rc & 0xFF;
                return (g.rs[r_ + 1] - g.rs[r_] - 1) + (g.cs[c_ + 1] - g.cs[c_] - 1);
            };
            deg_bytes = deg(vs) + (ur >= 0 ? deg(ur) : 0) + (uc >= 0 ? deg(uc) : 0);
        }
        __syncwarp();
        if (lane == 0) {
            col[vs] = (uint8_t)ks;
            s.U[vs >> 5] &= ~(1u << (vs & 31));
            if (ur >= 0) {
                col[ur] = 0;
                s.U[ur >> 5] |= 1u << (ur & 31);
                s.C[(g.cell[ur] & 0xFF) * W + kw] &= ~bitk;
            }
            if (uc >= 0) {
                col[uc] = 0;
                s.U[uc >> 5] |= 1u << (uc & 31);
                s.R[(g.cell[uc] >> 8) * W + kw] &= ~bitk;
            }
            s.R[rs_ * W + kw] |= bitk;
            s.C[cs_ * W + kw] |= bitk;
        }
        f = f - 1 + e;
        const uint32_t lpart = (uint32_t)(((x & 0xFFFFFFFFULL) * 10ULL) >> 32);
        const uint32_t tenure = lpart + (uint32_t)(a.alpha * (double)f);
        const uint32_t ut = j + 1 + tenure;
        if ((lane == 1 && ur >= 0) || (lane == 2 && uc >= 0)) {
            const int u = lane == 1 ? ur : uc;
            until[(size_t)u * w1 + ks] = ut;
            TabuRec<W> rr = rec[u];
            if (rr.tm[kw] & bitk) rr.exact = 0;
            rr.tm[kw] |= bitk;
            rr.umax = max(rr.umax, ut);
            rec[u] = rr;
        }
        bt += 4ULL * (unsigned)deg_bytes + 2ULL * (unsigned)(1 + e);
        const bool improved = f < bestf;
        if (improved) {
            bestf = f;
            pending = true;
            bt += 2ULL * (unsigned)nv;
        }
        bytes += bt;
        if (tracing && lane == 0 && (int64_t)j < a.trace_cap) {
            plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + j;
            // CSR order of N(v*): row-mates first iff row <= col (lsgraph.hpp:202-209)
            const bool row_first = rs_ <= cs_;
            const int e0 = row_first ? (ur >= 0 ? ur : uc) : (uc >= 0 ? uc : ur);
            const int e1 = e == 2 ? (row_first ? uc : ur) : -1;
            tr->step = j;
            tr->v = vs;
            tr->k = ks;
            tr->e = e;
            tr->ev0 = e0;
            tr->ev1 = e1;
            tr->f_before = f_before;
            tr->f_after = f;
            tr->best_f = bestf;
            tr->tenure = (int32_t)tenure;
            tr->n_adm = N;
            tr->level = lvl;
        }
        __syncwarp();
        ++j;
    }
    if (pending) snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
    if (lane == 0) {
        a.best_f[i] = bestf;
        a.repaired_f[i] = repaired_f;
        a.iters[i] = (int64_t)j;
        a.bytes[i] = bytes;
    }
    __syncwarp();
}

template <int W>
__global__ void __launch_bounds__(kImproveMaxThreads) k_improve(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, nv = a.nv;
    const ImproveSmemLayout L = improve_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + L.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + L.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + L.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + L.cl);
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + L.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + L.pc);
    for (int t = threadIdx.x; t < nv; t += blockDim.x) {
        s_cell[t] = a.cell[t];
        s_cl[t] = a.col_list[t];
    }
    for (int t = threadIdx.x; t <= n; t += blockDim.x) {
        s_rs[t] = a.row_start[t];
        s_cs[t] = a.col_start[t];
    }
    for (int t = threadIdx.x; t < n * W; t += blockDim.x) {
        s_pr[t] = a.pre_row[t];
        s_pc[t] = a.pre_col[t];
    }
    __syncthreads();

    Graph<W> g;
    g.n = n;
    g.nv = nv;
    g.nvpad = a.nvpad;
    g.lane_words = a.lane_words;
    g.cell = s_cell;
    g.rs = s_rs;
    g.cs = s_cs;
    g.cl = s_cl;
    g.pr = s_pr;
    g.pc = s_pc;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t m = 0;
        for (int b = 0; b < 64; ++b) {
            const int k = q * 64 + b;
            if (k >= 1 && k <= n) m |= 1ULL << b;
        }
        g.full[q] = m;
    }

    uint8_t* wbase = smem + L.warp0 + (size_t)warp * L.warp_bytes;
    WarpSmem s;
    s.col = wbase + L.w_col;
    s.conf = wbase + L.w_conf;
    s.R = reinterpret_cast<uint64_t*>(wbase + L.w_R);
    s.C = reinterpret_cast<uint64_t*>(wbase + L.w_C);
    s.U = reinterpret_cast<uint32_t*>(wbase + L.w_U);

    const int slot = blockIdx.x * nwarps + warp;
    TabuRec<W>* rec = reinterpret_cast<TabuRec<W>*>(reinterpret_cast<char*>(a.tabu_rec) + (size_t)slot * a.rec_stride);
    uint32_t* until = a.until + (size_t)slot * a.until_stride;

    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(a.work_counter, 1);
        i = __shfl_sync(kFull, i, 0);
        if (i >= a.p) break;
        improve_one<W>(a, g, s, rec, until, i, lane);
    }
}

// W = 64-bit words per colour mask: 1 for n <= 63, 2 for n <= 127 (the u8 conflict
// counters of the repair bound n at 127; capi.cu rejects larger orders).
size_t tabu_rec_bytes(int W) { return W == 1 ? sizeof(TabuRec<1>) : sizeof(TabuRec<2>); }

const void* improve_kernel_ptr(int W) {
    if (W == 1) return reinterpret_cast<const void*>(&k_improve<1>);
    return reinterpret_cast<const void*>(&k_improve<2>);
}

cudaError_t launch_improve(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    if (W == 1)
        k_improve<1><<<grid, threads, smem, st>>>(a);
    else
        k_improve<2><<<grid, threads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace plse_dev
