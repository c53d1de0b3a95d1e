// improve_hw.cu -- the improve phase with TWO INDIVIDUALS PER WARP.
//
// Same algorithm, data layout and canonical rule as improve.cu (see its
// header); the difference is the execution mapping.  Lanes 0-15 search one
// individual and lanes 16-31 another, so every warp instruction of the
// per-step plumbing (level vote, prefix scan, draws, the 3-lane update, the
// slot re-sort) advances two searches.  In sparse mode (|V0| <= 32) each lane
// holds two consecutive slots of its half's sorted uncoloured list.  All
// collectives take the half's lane mask (width-16 shuffles, masked votes /
// reductions), so the halves may diverge (dense mode, repair, finishing) and
// re-converge without deadlock.  The row / column holder of k* is found with
// one 64-byte word-parallel pass over a row-major and a column-major copy of
// the colours (the column copy is ordered like the graph's column lists).
#include "improve_common.cuh"

namespace plse_dev {

struct HalfSmem {
    uint8_t* col;   // [nvpad] colour of vertex v
    uint8_t* colT;  // [nvpad] colour of vertex cl[x] (column-major copy); repair counters before that
    uint64_t* R;
    uint64_t* C;
    uint32_t* U;
    uint16_t* list;  // 32-entry seed list of sparse mode
};

struct HSlot {
    uint32_t vc, u1, u2, kk;  // vertex | row << 16 | col << 24, tabu cache
};

__device__ __forceinline__ void hslot_clear(HSlot& s) {
    s.vc = 0xFFFFu;
    s.u1 = s.u2 = s.kk = 0;
}

__device__ __forceinline__ uint32_t hsel(uint32_t a0, uint32_t a1, int sel) { return sel ? a1 : a0; }

// position of the unique byte == k in bytes [a, b) of buf (word-parallel over the 16 lanes of a half)
__device__ __forceinline__ int half_find_byte(const uint8_t* buf, int a, int b, int k, int hl, unsigned hm, int hshift) {
    const uint32_t kk4 = (uint32_t)k * 0x01010101u;
    for (int base = a & ~3; base < b; base += 64) {
        const int wpos = base + 4 * hl;
        uint32_t hit = 0;
        if (wpos < b) {
            const uint32_t w = reinterpret_cast<const uint32_t*>(buf)[wpos >> 2] ^ kk4;
            uint32_t z = ~(((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;  // 0x80 where the byte == k
            uint32_t valid = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (wpos + q >= a && wpos + q < b) valid |= 0x80u << (8 * q);
            hit = z & valid;
        }
        const unsigned bal = (__ballot_sync(hm, hit != 0) >> hshift) & 0xFFFFu;
        if (bal) {
            const int src = __ffs(bal) - 1;
            const int byte = (__ffs(hit) - 1) >> 3;  // meaningful on the source lane only
            return __shfl_sync(hm, base + 4 * hl + byte, src, 16);
        }
    }
    return -1;
}

template <int W>
__device__ __forceinline__ void half_snapshot(const uint8_t* col, uint8_t* dst, int nvpad, int hl) {
    const uint4* s4 = reinterpret_cast<const uint4*>(col);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int x = hl; x < nvpad / 16; x += 16) d4[x] = s4[x];
}

template <int W, bool kDebug>
__global__ void __launch_bounds__(kHwMaxThreads, kHwMinBlocks) k_improve_hw(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int h = lane >> 4, hl = lane & 15, hshift = 16 * h;
    const unsigned hm = 0xFFFFu << hshift;
    const int n = a.n, nv = a.nv, w1 = n + 1, nvpad = a.nvpad;
    const HwSmemLayout L = improve_hw_smem_layout(n, nv, nvpad, a.lane_words16, W);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + L.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + L.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + L.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + L.cl);
    uint16_t* s_cp = reinterpret_cast<uint16_t*>(smem + L.colpos);
    uint8_t* s_deg = smem + L.deg;
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + L.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + L.pc);
    for (int x = threadIdx.x; x < nv; x += blockDim.x) {
        s_cell[x] = a.cell[x];
        const uint16_t v = a.col_list[x];
        s_cl[x] = v;
        s_cp[v] = (uint16_t)x;
    }
    for (int x = threadIdx.x; x <= n; x += blockDim.x) {
        s_rs[x] = a.row_start[x];
        s_cs[x] = a.col_start[x];
    }
    for (int x = threadIdx.x; x < n * W; x += blockDim.x) {
        s_pr[x] = a.pre_row[x];
        s_pc[x] = a.pre_col[x];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nv; x += blockDim.x) {
        const int r = s_cell[x] >> 8, c = s_cell[x] & 0xFF;
        s_deg[x] = (uint8_t)((s_rs[r + 1] - s_rs[r] - 1) + (s_cs[c + 1] - s_cs[c] - 1));
    }
    __syncthreads();

    Graph<W> g;
    g.n = n;
    g.nv = nv;
    g.nvpad = nvpad;
    g.lane_words = a.lane_words16;
    g.cell = s_cell;
    g.deg = s_deg;
    g.rs = s_rs;
    g.cs = s_cs;
    g.cl = s_cl;
    g.colpos = s_cp;
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
    uint8_t* hb = smem + L.warp0 + (size_t)warp * L.warp_bytes + (size_t)h * L.half_bytes;
    HalfSmem s;
    s.col = hb + L.h_col;
    s.colT = hb + L.h_colT;
    s.R = reinterpret_cast<uint64_t*>(hb + L.h_R);
    s.C = reinterpret_cast<uint64_t*>(hb + L.h_C);
    s.U = reinterpret_cast<uint32_t*>(hb + L.h_U);
    s.list = reinterpret_cast<uint16_t*>(hb + L.h_list);
    WarpSmem ws;  // view for level_masks
    ws.col = s.col;
    ws.conf = s.colT;
    ws.R = s.R;
    ws.C = s.C;
    ws.U = s.U;

    const int hslot = (blockIdx.x * nwarps + warp) * 2 + h;
    TabuRec* rec = reinterpret_cast<TabuRec*>(reinterpret_cast<char*>(a.tabu_rec) + (size_t)hslot * a.rec_stride);
    uint32_t* until = a.until + (size_t)hslot * a.until_stride;
    uint32_t* slot_clock = a.slot_clock + hslot;
    const int LW = a.lane_words16;
    const int B = 32 * LW;
    const int v_lo = hl * B;
    const int v_hi = min(nv, v_lo + B);
    uint8_t* col = s.col;

    unsigned long long* prof = kDebug ? a.prof : nullptr;
    long long t_start = 0, t_step = 0, t_prologue = 0;
    unsigned long long pc_dense = 0, pc_sparse = 0, pn_dense = 0, pn_sparse = 0, pf_dense = 0, pn_enter = 0;

    int state = 0;  // 0 = needs an individual, 1 = searching, 2 = no work left
    int i = 0;
    int f = 0, bestf = 0, repaired_f = 0;
    bool pending = false, sparse = false, tracing = false;
    uint32_t j = 0, base = 0, s32 = 0;
    unsigned long long acc = 0;
    HSlot sl0, sl1;
    hslot_clear(sl0);
    hslot_clear(sl1);

    for (;;) {
        if (state == 0) {
            // ---------------------------------------------------------- fetch + prologue
            int ii = 0;
            if (hl == 0) ii = atomicAdd(a.work_counter, 1);
            ii = __shfl_sync(hm, ii, 0, 16);
            if (ii >= a.p) {
                state = 2;
            } else {
                i = ii;
                if (prof) t_start = clock64();
                base = *slot_clock;
                if ((uint64_t)base + (uint64_t)a.budget + a.tenure_cap + 2 >= 0xFFFFFFFFull) {
                    uint4* u4 = reinterpret_cast<uint4*>(until);
                    for (size_t x = hl; x < a.until_stride / 4; x += 16) u4[x] = make_uint4(0, 0, 0, 0);
                    base = 0;
                }
                {
                    const uint4* src = reinterpret_cast<const uint4*>(a.offspring + (size_t)i * nvpad);
                    uint4* d4 = reinterpret_cast<uint4*>(col);
                    for (int x = hl; x < nvpad / 16; x += 16) d4[x] = src[x];
                    const TabuRec z{0, 0, 0, 0};
                    for (int x = hl; x < nv; x += 16) rec[x] = z;
                }
                __syncwarp(hm);
                uint8_t* conf = s.colT;
                // K1: same-coloured neighbours of every coloured vertex (coloring.hpp:105-116)
                for (int v = v_lo; v < v_hi; ++v) {
                    const int k = col[v];
                    int cnt = 0;
                    if (k) {
                        const uint16_t rc = g.cell[v];
                        const int r = rc >> 8, c = rc & 0xFF;
                        for (int u = g.rs[r]; u < g.rs[r + 1]; ++u) cnt += col[u] == k;
                        for (int x = g.cs[c]; x < g.cs[c + 1]; ++x) cnt += col[g.cl[x]] == k;
                        cnt -= 2;
                    }
                    conf[v] = (uint8_t)cnt;
                }
                __syncwarp(hm);
                // K1b: repair (partial.hpp:22-39), argmax with lowest-index ties
                for (;;) {
                    int bc = 0, bv = -1;
                    for (int v = v_lo; v < v_hi; ++v) {
                        const int c = conf[v];
                        if (c > bc) {
                            bc = c;
                            bv = v;
                        }
                    }
                    const int mx = (int)__reduce_max_sync(hm, (unsigned)bc);
                    if (mx == 0) break;
                    const int wl = __ffs((__ballot_sync(hm, bc == mx) >> hshift) & 0xFFFFu) - 1;
                    const int w = __shfl_sync(hm, bv, wl, 16);
                    const int k = col[w];
                    const uint16_t rc = g.cell[w];
                    const int r = rc >> 8, c = rc & 0xFF;
                    for (int u = g.rs[r] + hl; u < g.rs[r + 1]; u += 16)
                        if (u != w && col[u] == k) conf[u] -= 1;
                    for (int x = g.cs[c] + hl; x < g.cs[c + 1]; x += 16) {
                        const int u = g.cl[x];
                        if (u != w && col[u] == k) conf[u] -= 1;
                    }
                    __syncwarp(hm);
                    if (hl == 0) {
                        col[w] = 0;
                        conf[w] = 0;
                    }
                    __syncwarp(hm);
                }
                // occupancy masks, uncoloured bitmask, column-major colour copy
                for (int x = hl; x < n * W; x += 16) {
                    s.R[x] = 0;
                    s.C[x] = 0;
                }
                __syncwarp(hm);
                int fl = 0;
                for (int q = 0; q < LW; ++q) {
                    const int vb = v_lo + 32 * q;
                    uint32_t bits = 0;
                    for (int b = 0; b < 32; ++b) {
                        const int v = vb + b;
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
                    s.U[hl * LW + q] = bits;
                    fl += __popc(bits);
                }
                __syncwarp(hm);
                for (int x = hl; x < nv; x += 16) s.colT[x] = col[g.cl[x]];
                f = (int)__reduce_add_sync(hm, (unsigned)fl);
                __syncwarp(hm);
                repaired_f = f;
                bestf = f;
                pending = true;
                sparse = false;
                j = 0;
                acc = 0;
                const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
                s32 = (uint32_t)(seed ^ (seed >> 32));
                tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
                if (prof) t_prologue = clock64() - t_start;
                state = 1;
            }
        }
        if (__ballot_sync(kFull, state == 2) == kFull) break;
        if (state != 1) continue;

        bool raced = a.race_flag && (j & 63) == 0 && *reinterpret_cast<volatile int*>(a.race_flag);
        if (a.deadline && j != 0 && (j & 0xFFFu) == 0) {  // partial.hpp:165, decided by the half's lane 0
            const int hit = hl == 0 ? (globaltimer_ns() >= *a.deadline) : 0;
            raced |= __shfl_sync(hm, hit, 0, 16) != 0;
        }
        if (raced || !((int64_t)j < a.budget && bestf > a.stop_f && f > 0)) {
            // ---------------------------------------------------------- finish the individual
            if (pending) half_snapshot<W>(col, a.improved + (size_t)i * nvpad, nvpad, hl);
            const unsigned long long a1 = __shfl_sync(hm, acc, 1, 16), a2 = __shfl_sync(hm, acc, 2, 16);
            if (hl == 0) {
                a.best_f[i] = bestf;
                a.repaired_f[i] = repaired_f;
                a.iters[i] = (int64_t)j;
                a.bytes[i] = acc + a1 + a2;
                *slot_clock = base + j + 2 + a.tenure_cap;
                if (prof) {
                    atomicAdd(prof + 0, 1ULL);
                    atomicAdd(prof + 1, (unsigned long long)t_prologue);
                    atomicAdd(prof + 2, pn_dense);
                    atomicAdd(prof + 3, pc_dense);
                    atomicAdd(prof + 4, pn_sparse);
                    atomicAdd(prof + 5, pc_sparse);
                    atomicAdd(prof + 6, pf_dense);
                    atomicAdd(prof + 7, pn_enter);
                    atomicAdd(prof + 8, (unsigned long long)(clock64() - t_start));
                }
            }
            pc_dense = pc_sparse = pn_dense = pn_sparse = pf_dense = pn_enter = 0;
            __syncwarp(hm);
            state = 0;
            continue;
        }

        // -------------------------------------------------------------- one PartialCol step
        if (prof) t_step = clock64();
        const bool step_sparse = f <= 32;
        const bool asp = (f == bestf);
        const uint32_t t = base + j;
        if (f <= 32 && !sparse) {
            if (prof) ++pn_enter;
            int cnt = 0;
            for (int q = 0; q < LW; ++q) cnt += __popc(s.U[hl * LW + q]);
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 16; d <<= 1) {
                const int x = __shfl_up_sync(hm, incl, d, 16);
                if (hl >= d) incl += x;
            }
            int at = incl - cnt;
            for (int q = 0; q < LW; ++q) {
                uint32_t bits = s.U[hl * LW + q];
                while (bits) {
                    s.list[at++] = (uint16_t)(v_lo + 32 * q + __ffs(bits) - 1);
                    bits &= bits - 1;
                }
            }
            __syncwarp(hm);
#pragma unroll
            for (int z = 0; z < 2; ++z) {
                HSlot& sl = z ? sl1 : sl0;
                const int idx = 2 * hl + z;
                if (idx < f) {
                    const int v = s.list[idx];
                    const TabuRec tr = rec[v];
                    const uint16_t rc = g.cell[v];
                    sl.vc = (uint32_t)v | ((uint32_t)(rc >> 8) << 16) | ((uint32_t)(rc & 0xFF) << 24);
                    sl.u1 = tr.u1;
                    sl.u2 = tr.u2;
                    sl.kk = tr.kk;
                } else {
                    hslot_clear(sl);
                }
            }
            __syncwarp(hm);
            sparse = true;
        }
        const uint32_t h1 = fmix32(s32 + (j + 1) * 0x9E3779B9u);
        const uint32_t h2 = fmix32(h1 + 0x632BE5ABu);
        int lvl, N, vs = 0, ks = 0, wi = 0;
        if (sparse) {
            // ---- score both slots of this lane: packed counts c(-1) | c(0) << 8 | c(+1) << 16
            uint32_t pk0 = 0, pk1 = 0;
#pragma unroll
            for (int z = 0; z < 2; ++z) {
                HSlot& sl = z ? sl1 : sl0;
                if (2 * hl + z < f) {
                    const int r = (sl.vc >> 16) & 0xFF, c = sl.vc >> 24;
                    uint64_t dom[W], T[W], m0[W], m1[W], m2[W];
                    dom_mask<W>(g, r, c, dom);
                    tabu_of<W>(sl.u1, sl.u2, sl.kk, until + (size_t)(sl.vc & 0xFFFFu) * w1, dom, t, T);
                    level_masks<W>(ws, r, c, dom, T, asp, m0, m1, m2);
                    const uint32_t pk = (uint32_t)popc_w<W>(m0) | ((uint32_t)popc_w<W>(m1) << 8) |
                                        ((uint32_t)popc_w<W>(m2) << 16);
                    if (z)
                        pk1 = pk;
                    else
                        pk0 = pk;
                }
            }
            const uint32_t pk = pk0 + pk1;
            const unsigned b0 = (__ballot_sync(hm, (pk & 0xFFu) != 0) >> hshift) & 0xFFFFu;
            const unsigned b1 = (__ballot_sync(hm, (pk & 0xFF00u) != 0) >> hshift) & 0xFFFFu;
            const unsigned b2 = (__ballot_sync(hm, (pk & 0xFF0000u) != 0) >> hshift) & 0xFFFFu;
            const int lc = b0 ? 0 : b1 ? 1 : b2 ? 2 : 3;
            lvl = lc - 1;
            const int sh = 8 * (lc & 3);
            const int cnt = lc == 3 ? 0 : (int)((pk >> sh) & 0xFFu);
            const int nl = (f + 1) >> 1;  // lanes holding slots
            int incl = cnt;
            for (int d = 1; d < nl; d <<= 1) {
                const int x = __shfl_up_sync(hm, incl, d, 16);
                if (hl >= d) incl += x;
            }
            N = __shfl_sync(hm, incl, nl - 1, 16);
            if (N > 0) {
                const uint32_t r = __umulhi(h1, (uint32_t)N);
                const int wl = __ffs((__ballot_sync(hm, (uint32_t)(incl - cnt) <= r && r < (uint32_t)incl) >> hshift) &
                                     0xFFFFu) - 1;
                if (hl == wl) {
                    int rr = (int)r - (incl - cnt);
                    const int c0 = lc == 3 ? 0 : (int)((pk0 >> sh) & 0xFFu);
                    const int z = rr < c0 ? 0 : 1;
                    rr -= z ? c0 : 0;
                    // re-derive the chosen slot's masks (its tabu cache was already normalised above)
                    const uint32_t vc = z ? sl1.vc : sl0.vc;
                    uint32_t u1 = z ? sl1.u1 : sl0.u1, u2 = z ? sl1.u2 : sl0.u2, kk = z ? sl1.kk : sl0.kk;
                    const int r_ = (vc >> 16) & 0xFF, c_ = vc >> 24;
                    uint64_t dom[W], T[W], m0[W], m1[W], m2[W];
                    dom_mask<W>(g, r_, c_, dom);
                    tabu_of<W>(u1, u2, kk, until + (size_t)(vc & 0xFFFFu) * w1, dom, t, T);
                    level_masks<W>(ws, r_, c_, dom, T, asp, m0, m1, m2);
                    uint64_t m[W];
#pragma unroll
                    for (int q = 0; q < W; ++q) m[q] = lc == 0 ? m0[q] : lc == 1 ? m1[q] : m2[q];
                    ks = nth_bit_w<W>(m, rr);
                    vs = (int)(vc & 0xFFFFu);
                    wi = 2 * hl + z;
                }
                vs = __shfl_sync(hm, vs, wl, 16);
                ks = __shfl_sync(hm, ks, wl, 16);
                wi = __shfl_sync(hm, wi, wl, 16);
            }
        } else {
            // ---- dense: each lane scans its bitmask words
            int c0 = 0, c1 = 0, c2 = 0;
            for (int q = 0; q < LW; ++q) {
                uint32_t bits = s.U[hl * LW + q];
                while (bits) {
                    const int v = v_lo + 32 * q + __ffs(bits) - 1;
                    bits &= bits - 1;
                    uint64_t x0[W], x1[W], x2[W];
                    dense_masks<W>(g, ws, rec, until, v, t, asp, x0, x1, x2);
                    c0 += popc_w<W>(x0);
                    c1 += popc_w<W>(x1);
                    c2 += popc_w<W>(x2);
                }
            }
            const unsigned b0 = (__ballot_sync(hm, c0 > 0) >> hshift) & 0xFFFFu;
            const unsigned b1 = (__ballot_sync(hm, c1 > 0) >> hshift) & 0xFFFFu;
            const unsigned b2 = (__ballot_sync(hm, c2 > 0) >> hshift) & 0xFFFFu;
            lvl = b0 ? -1 : b1 ? 0 : b2 ? 1 : 2;
            const int cnt = lvl == -1 ? c0 : lvl == 0 ? c1 : lvl == 1 ? c2 : 0;
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 16; d <<= 1) {
                const int x = __shfl_up_sync(hm, incl, d, 16);
                if (hl >= d) incl += x;
            }
            N = __shfl_sync(hm, incl, 15, 16);
            if (N > 0) {
                const uint32_t r = __umulhi(h1, (uint32_t)N);
                const int wl = __ffs((__ballot_sync(hm, (uint32_t)(incl - cnt) <= r && r < (uint32_t)incl) >> hshift) &
                                     0xFFFFu) - 1;
                vs = -1;
                if (hl == wl) {
                    int rr = (int)r - (incl - cnt);
                    for (int q = 0; q < LW && vs < 0; ++q) {
                        uint32_t bits = s.U[hl * LW + q];
                        while (bits) {
                            const int v = v_lo + 32 * q + __ffs(bits) - 1;
                            bits &= bits - 1;
                            uint64_t x0[W], x1[W], x2[W];
                            dense_masks<W>(g, ws, rec, until, v, t, asp, x0, x1, x2);
                            uint64_t mm[W];
#pragma unroll
                            for (int z = 0; z < W; ++z) mm[z] = lvl == -1 ? x0[z] : lvl == 0 ? x1[z] : x2[z];
                            const int pc = popc_w<W>(mm);
                            if (rr < pc) {
                                ks = nth_bit_w<W>(mm, rr);
                                vs = v;
                                break;
                            }
                            rr -= pc;
                        }
                    }
                }
                vs = __shfl_sync(hm, vs, wl, 16);
                ks = __shfl_sync(hm, ks, wl, 16);
            }
        }
        const int f_before = f;
        if (N == 0) {
            // every candidate tabu: no move, the clock still advances (partial.hpp:121-122)
            if (hl == 0) acc += 2ULL * (unsigned)w1 * (unsigned)f;
            if (tracing && hl == 0 && (int64_t)j < a.trace_cap) {
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
            ++j;
            continue;
        }

        // -------------------------------------------------------------- apply (partial.hpp:124-141)
        if (pending && lvl >= 0) {
            half_snapshot<W>(col, a.improved + (size_t)i * nvpad, nvpad, hl);
            pending = false;
        }
        const uint16_t rcs = g.cell[vs];
        const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
        const int kw = ks >> 6;
        const uint64_t bitk = 1ULL << (ks & 63);
        int ur = -1, uc = -1;
        if (lvl >= 0) {
            const bool inR = (s.R[rs_ * W + kw] & bitk) != 0;
            const bool inC = (s.C[cs_ * W + kw] & bitk) != 0;
            if (inR) ur = half_find_byte(col, g.rs[rs_], g.rs[rs_ + 1], ks, hl, hm, hshift);
            if (inC) {
                const int x = half_find_byte(s.colT, g.cs[cs_], g.cs[cs_ + 1], ks, hl, hm, hshift);
                uc = g.cl[x];
            }
        }
        const int e = (ur >= 0) + (uc >= 0);
        const int f_new = f - 1 + e;
        const uint32_t tenure = __umulhi(h2, 10u) + (uint32_t)(a.alpha * (double)f_new);
        const uint32_t ut = t + 1 + tenure;
        const bool improved = f_new < bestf;
        __syncwarp(hm);
        const int my_u = hl == 1 ? ur : hl == 2 ? uc : -1;
        TabuRec nr{0, 0, 0, 0};
        if (my_u >= 0) nr = rec[my_u];
        if (hl == 0) {
            col[vs] = (uint8_t)ks;
            s.colT[g.colpos[vs]] = (uint8_t)ks;
            atomicAnd(&s.U[vs >> 5], ~(1u << (vs & 31)));
            s.R[rs_ * W + kw] |= bitk;
            s.C[cs_ * W + kw] |= bitk;
            acc += 2ULL * (unsigned)w1 * (unsigned)f_before + 4ULL * g.deg[vs] + 2ULL +
                   (improved ? 2ULL * (unsigned)nv : 0ULL);
        } else if (my_u >= 0) {
            col[my_u] = 0;
            s.colT[g.colpos[my_u]] = 0;
            atomicOr(&s.U[my_u >> 5], 1u << (my_u & 31));
            if (hl == 1)
                s.C[(g.cell[my_u] & 0xFF) * W + kw] &= ~bitk;  // row holder leaves its column
            else
                s.R[(g.cell[my_u] >> 8) * W + kw] &= ~bitk;    // column holder leaves its row
            until[(size_t)my_u * w1 + ks] = ut;
            acc += 4ULL * g.deg[my_u] + 2ULL;
        }
        if (sparse) {
            if (f_new > 32) {
                sparse = false;
            } else {
                // new sorted list = old list - {v*} + {ur, uc}; lane hl takes new slots 2hl, 2hl+1
                const int v0 = (int)(sl0.vc & 0xFFFFu), v1 = (int)(sl1.vc & 0xFFFFu);
                const bool ok0 = 2 * hl < f && 2 * hl != wi, ok1 = 2 * hl + 1 < f && 2 * hl + 1 != wi;
                int pr_ = -1, pc_ = -1;
                if (ur >= 0)
                    pr_ = (int)__reduce_add_sync(hm, (unsigned)((ok0 && v0 < ur) + (ok1 && v1 < ur))) +
                          (uc >= 0 && uc < ur);
                if (uc >= 0)
                    pc_ = (int)__reduce_add_sync(hm, (unsigned)((ok0 && v0 < uc) + (ok1 && v1 < uc))) +
                          (ur >= 0 && ur < uc);
                if (my_u >= 0) {
                    cache_forbid(nr, ks, ut, t);
                    rec[my_u] = nr;
                }
                const uint32_t ru1 = __shfl_sync(hm, nr.u1, 1, 16), ru2 = __shfl_sync(hm, nr.u2, 1, 16),
                               rkk = __shfl_sync(hm, nr.kk, 1, 16);
                const uint32_t cu1 = __shfl_sync(hm, nr.u1, 2, 16), cu2 = __shfl_sync(hm, nr.u2, 2, 16),
                               ckk = __shfl_sync(hm, nr.kk, 2, 16);
                HSlot nsl[2];
#pragma unroll
                for (int z = 0; z < 2; ++z) {
                    const int x = 2 * hl + z;
                    const int y = x - (pr_ >= 0 && pr_ < x) - (pc_ >= 0 && pc_ < x);
                    const int src = (y >= wi ? y + 1 : y) & 31;
                    const int sl_ = (src >> 1) & 15, sel = src & 1;
                    const uint32_t vc = hsel(__shfl_sync(hm, sl0.vc, sl_, 16), __shfl_sync(hm, sl1.vc, sl_, 16), sel);
                    const uint32_t u1 = hsel(__shfl_sync(hm, sl0.u1, sl_, 16), __shfl_sync(hm, sl1.u1, sl_, 16), sel);
                    const uint32_t u2 = hsel(__shfl_sync(hm, sl0.u2, sl_, 16), __shfl_sync(hm, sl1.u2, sl_, 16), sel);
                    const uint32_t kk = hsel(__shfl_sync(hm, sl0.kk, sl_, 16), __shfl_sync(hm, sl1.kk, sl_, 16), sel);
                    if (x == pr_ || x == pc_) {
                        const int u = x == pr_ ? ur : uc;
                        const uint16_t rc = g.cell[u];
                        nsl[z].vc = (uint32_t)u | ((uint32_t)(rc >> 8) << 16) | ((uint32_t)(rc & 0xFF) << 24);
                        nsl[z].u1 = x == pr_ ? ru1 : cu1;
                        nsl[z].u2 = x == pr_ ? ru2 : cu2;
                        nsl[z].kk = x == pr_ ? rkk : ckk;
                    } else {
                        nsl[z].vc = vc;
                        nsl[z].u1 = u1;
                        nsl[z].u2 = u2;
                        nsl[z].kk = kk;
                    }
                }
                sl0 = nsl[0];
                sl1 = nsl[1];
            }
        }
        if (!sparse && my_u >= 0) {
            cache_forbid(nr, ks, ut, t);
            rec[my_u] = nr;
        }
        f = f_new;
        if (improved) {
            bestf = f;
            pending = true;
            if (a.race_flag && bestf <= a.race_f && hl == 0) atomicExch(a.race_flag, 1);
        }
        if (tracing && hl == 0 && (int64_t)j < a.trace_cap) {
            plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + j;
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
        __syncwarp(hm);
        ++j;
        if (prof) {
            const unsigned long long dt = (unsigned long long)(clock64() - t_step);
            if (step_sparse) {
                pc_sparse += dt;
                ++pn_sparse;
            } else {
                pc_dense += dt;
                ++pn_dense;
                pf_dense += (unsigned)f_before;
            }
        }
    }
}

const void* improve_hw_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_improve_hw<1, true>)
                             : reinterpret_cast<const void*>(&k_improve_hw<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_improve_hw<2, true>)
                 : reinterpret_cast<const void*>(&k_improve_hw<2, false>);
}

cudaError_t launch_improve_hw(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr || a.prof != nullptr;
    if (W == 1) {
        if (debug)
            k_improve_hw<1, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve_hw<1, false><<<grid, threads, smem, st>>>(a);
    } else {
        if (debug)
            k_improve_hw<2, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve_hw<2, false><<<grid, threads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace plse_dev
