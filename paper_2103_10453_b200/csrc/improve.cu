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
//     search -- row-major (col) and column-major (colT, ordered like the
//     graph's column lists) -- with per-row / per-column colour-occupancy
//     bitmasks R[r], C[c] (W x u64) and the uncoloured set U as a bitmask.
//     In a legal colouring gamma[v][k] = [k in R[row v]] + [k in C[col v]]
//     for every uncoloured v, so the three move classes of an uncoloured
//     vertex (delta -1 / 0 / +1) are three W-word mask expressions: the gamma
//     rows the north star puts in HBM are never materialised.
//   * The domain of v is ~(PR[row] | PC[col]) over the prefilled-symbol masks
//     (lsgraph.hpp:152-156), shared by the CTA in shared memory.
//   * Tabu state (search_util.hpp:54-81): the reference's dense until[v][k]
//     table lives per warp slot in HBM, on a monotone per-slot clock so it is
//     never cleared (the reference's skip_past, partial.hpp:60).  A 16-byte
//     record per vertex caches its two most recent (colour, until) pairs plus
//     an overflow flag; only a vertex with three or more live tabu colours
//     reads the dense table.
//   * Sparse mode (|V0| <= 32, i.e. everything after the first ~1% of the
//     descent) is a tight, branch-light inner loop: lane l holds the l-th
//     uncoloured vertex (ascending id, with its row / column packed in) and
//     its tabu pairs in registers, so scoring costs four shared loads per
//     lane; the row / column holder of k* is one word-parallel pass over the
//     row-major / column-major colour copies; the update is a predicated
//     five-lane XOR (colour bytes, U bits, R / C bits) and the slot list is
//     re-sorted with one computed-source shuffle per field.  Dense mode
//     (|V0| > 32) scans the U bitmask (lane-owned 32*lane_words blocks).
//   * Selection is the canonical order-free rule: the lowest
//     admissible delta level, per-lane counts, a warp prefix sum, and
//     r = floor(h1 * N / 2^32) from a counter-based draw keyed by (stream seed, step); the
//     lane holding the r-th candidate in ascending (v, k) order recovers it
//     with a popcount search.
#include "improve_common.cuh"

namespace plse_dev {

template <int W, bool kDebug>
__device__ void improve_one(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                            uint32_t* until, uint32_t* slot_clock, uint8_t* conf, int i, int lane) {
    const int n = g.n, nv = g.nv, w1 = n + 1;
    const int B = 32 * g.lane_words;
    const int v_lo = lane * B;
    const int v_hi = min(nv, v_lo + B);
    uint8_t* col = s.col;
    uint8_t* colT = s.colT;
    unsigned long long* prof = kDebug ? a.prof : nullptr;
    long long t_start = prof ? clock64() : 0, t_step = 0;
    unsigned long long pc_dense = 0, pc_sparse = 0, pn_dense = 0, pn_sparse = 0, pf_dense = 0, pn_enter = 0;

    // ---- tabu clock of this warp slot: every until[][] left by earlier individuals is <= base
    uint32_t base = *slot_clock;
    if ((uint64_t)base + (uint64_t)a.budget + a.tenure_cap + 2 >= 0xFFFFFFFFull) {
        uint4* u4 = reinterpret_cast<uint4*>(until);
        for (size_t x = lane; x < a.until_stride / 4; x += 32) u4[x] = make_uint4(0, 0, 0, 0);
        base = 0;
    }

    int f = partial_prologue<W>(a, g, s, rec, conf, i, lane);
    __syncwarp();

    const long long t_prologue = prof ? clock64() - t_start : 0;
    const int repaired_f = f;
    int bestf = f;
    bool pending = true;  // best_ == current (partial.hpp:84)
    uint32_t j = 0;
    // SURVEY 8(d) algorithmic bytes: lane 0 accounts the scan, v*'s RMW and the
    // snapshots, lanes 1/2 the evictees' RMW; summed over the warp at the end.
    unsigned long long acc = 0;
    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    CanonDraws draws{seed, 0u, 0u, -1};
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
    const bool probing = kDebug && (i == a.trace_idx) && a.probe.n > 0;
    int probe_next = 0;
    // the state before step jj, at the probe points (plse_probe)
    auto probe_at = [&](uint32_t jj) {
        if (probing && probe_next < a.probe.n && (int64_t)jj == a.probe.steps[probe_next]) {
            __syncwarp();
            probe_dump<W>(a, g, s, rec, until, base, base + jj, probe_next, lane);
            ++probe_next;
        }
    };
    const int64_t budget = a.budget;
    const int stop_f = a.stop_f;
    const double alpha = a.alpha;
    const int* race_flag = a.race_flag;
    const int race_f = a.race_f;
    // partial.hpp:164-165: `++iterations; if ((iterations & 0xFFF) == 0 && deadline_passed) break;`
    // lane 0 reads the clock so the whole warp takes the same decision
    const unsigned long long* deadline = a.deadline;
    // polled every 64 steps: the race flag, and the deadline at multiples of 4096
    auto poll_stop = [race_flag, deadline](uint32_t jj) -> bool {
        if (race_flag && *reinterpret_cast<const volatile int*>(race_flag)) return true;
        if (!deadline || jj == 0 || (jj & 0xFFFu)) return false;
        return __shfl_sync(kFull, globaltimer_ns() >= *deadline ? 1 : 0, 0) != 0;
    };

    // step record of the parity probe
    auto trace_step = [&](uint32_t jj, int vs, int ks, int ur, int uc, int rs_, int cs_, int fb, int fa, int bf,
                          int ten, int N, int lvl) {
        plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + jj;
        const int e = (ur >= 0) + (uc >= 0);
        // CSR order of N(v*): row-mates first iff row <= col (lsgraph.hpp:202-209)
        const bool row_first = rs_ <= cs_;
        tr->step = jj;
        tr->v = vs;
        tr->k = ks;
        tr->e = e;
        tr->ev0 = vs < 0 ? -1 : row_first ? (ur >= 0 ? ur : uc) : (uc >= 0 ? uc : ur);
        tr->ev1 = e == 2 ? (row_first ? uc : ur) : -1;
        tr->f_before = fb;
        tr->f_after = fa;
        tr->best_f = bf;
        tr->tenure = ten;
        tr->n_adm = N;
        tr->level = lvl;
    };

    for (;;) {
        if (!((int64_t)j < budget && bestf > stop_f && f > 0)) break;
        if ((j & 63) == 0 && poll_stop(j)) break;
        if (kDebug) probe_at(j);
        const int f_before = f;
        const bool asp = (f == bestf);
        const uint32_t t = base + j;
        uint32_t h1, h2;
        draws.at(j, lane, h1, h2);
        if (f > 32) {
            // ============================================== dense step (start of the descent)
            if (prof) t_step = clock64();
            int c0 = 0, c1 = 0, c2 = 0;
            for (int q = 0; q < g.lane_words; ++q) {
                uint32_t bits = s.U[lane * g.lane_words + q];
                while (bits) {
                    const int v = v_lo + 32 * q + __ffs(bits) - 1;
                    bits &= bits - 1;
                    uint64_t x0[W], x1[W], x2[W];
                    dense_masks<W>(g, s, rec, until, v, t, asp, x0, x1, x2);
                    c0 += popc_w<W>(x0);
                    c1 += popc_w<W>(x1);
                    c2 += popc_w<W>(x2);
                }
            }
            const unsigned b0 = __ballot_sync(kFull, c0 > 0);
            const unsigned b1 = __ballot_sync(kFull, c1 > 0);
            const unsigned b2 = __ballot_sync(kFull, c2 > 0);
            const int lvl = b0 ? -1 : b1 ? 0 : b2 ? 1 : 2;
            const int cnt = lvl == -1 ? c0 : lvl == 0 ? c1 : lvl == 1 ? c2 : 0;
            int incl = warp_incl_sum(cnt);
            const int N = __shfl_sync(kFull, incl, 31);
            if (N == 0) {
                if (lane == 0) acc += 2ULL * (unsigned)w1 * (unsigned)f;
                if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                    trace_step(j, -1, 0, -1, -1, 0, 0, f, f, bestf, -1, 0, 2);
                ++j;
                continue;
            }
            const uint32_t r = __umulhi(h1, (uint32_t)N);
            const int wl = __ffs(__ballot_sync(kFull, (uint32_t)(incl - cnt) <= r && r < (uint32_t)incl)) - 1;
            int vs = -1, ks = 0;
            if (lane == wl) {
                int rr = (int)r - (incl - cnt);
                for (int q = 0; q < g.lane_words && vs < 0; ++q) {
                    uint32_t bits = s.U[lane * g.lane_words + q];
                    while (bits) {
                        const int v = v_lo + 32 * q + __ffs(bits) - 1;
                        bits &= bits - 1;
                        uint64_t x0[W], x1[W], x2[W];
                        dense_masks<W>(g, s, rec, until, v, t, asp, x0, x1, x2);
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
            vs = __shfl_sync(kFull, vs, wl);
            ks = __shfl_sync(kFull, ks, wl);
            if (pending && lvl >= 0) {
                snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
                pending = false;
            }
            const uint16_t rcs = g.cell[vs];
            const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
            const int kw = ks >> 6;
            const uint64_t bitk = 1ULL << (ks & 63);
            const bool inR = (s.R[rs_ * W + kw] & bitk) != 0;
            const bool inC = (s.C[cs_ * W + kw] & bitk) != 0;
            const int ur = warp_find_byte(col, g.rs[rs_], g.rs[rs_ + 1], ks, inR, lane);
            const int xc = warp_find_byte(colT, g.cs[cs_], g.cs[cs_ + 1], ks, inC, lane);
            const int uc = xc >= 0 ? (int)g.cl[xc] : -1;
            const int e = (ur >= 0) + (uc >= 0);
            const int f_new = f - 1 + e;
            const uint32_t tenure = __umulhi(h2, 10u) + (uint32_t)(alpha * (double)f_new);
            const uint32_t ut = t + 1 + tenure;
            const bool improved = f_new < bestf;
            apply_move_lanes<W>(g, s, rec, until, vs, ur, uc, ks, rs_, cs_, inR, inC, f_before, improved, ut, t, lane,
                                acc);
            f = f_new;
            if (improved) {
                bestf = f;
                pending = true;
                if (race_flag && bestf <= race_f && lane == 0) atomicExch(const_cast<int*>(race_flag), 1);
            }
            if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                trace_step(j, vs, ks, ur, uc, rs_, cs_, f_before, f, bestf, (int)tenure, N, lvl);
            __syncwarp();
            ++j;
            if (prof) {
                pc_dense += (unsigned long long)(clock64() - t_step);
                ++pn_dense;
                pf_dense += (unsigned)f_before;
            }
            continue;
        }

        // ================================================== sparse phase (|V0| <= 32)
        if (prof) ++pn_enter;
        // lane l takes the l-th uncoloured vertex (ascending v) with its tabu cache
        uint32_t svc = 0xFFFFu, su1 = 0, su2 = 0, skk = 0;
        {
            int cnt = 0;
            for (int q = 0; q < g.lane_words; ++q) cnt += __popc(s.U[lane * g.lane_words + q]);
            int incl = warp_incl_sum(cnt);
            int at = incl - cnt;
            for (int q = 0; q < g.lane_words; ++q) {
                uint32_t bits = s.U[lane * g.lane_words + q];
                while (bits) {
                    s.list[at++] = (uint16_t)(v_lo + 32 * q + __ffs(bits) - 1);
                    bits &= bits - 1;
                }
            }
            __syncwarp();
            if (lane < f) {
                const int v = s.list[lane];
                const TabuRec tr = rec[v];
                const uint16_t rc = g.cell[v];
                svc = (uint32_t)v | ((uint32_t)(rc >> 8) << 16) | ((uint32_t)(rc & 0xFF) << 24);
                su1 = tr.u1;
                su2 = tr.u2;
                skk = tr.kk;
            }
            __syncwarp();
        }
        for (;;) {
            if (prof) t_step = clock64();
            if (kDebug) probe_at(j);
            const int fb = f;
            const bool asp_s = (f == bestf);
            const uint32_t ts = base + j;
            uint32_t g1, g2;
            draws.at(j, lane, g1, g2);
            // ---- score this lane's slot
            const int r = (svc >> 16) & 0xFF, c = svc >> 24;
            const bool mine = lane < f;
            uint64_t dom[W], T[W], m0[W], m1[W], m2[W];
            dom_mask<W>(g, r, c, dom);
#pragma unroll
            for (int z = 0; z < W; ++z) dom[z] = mine ? dom[z] : 0ULL;  // an empty slot has no candidates
            tabu_of<W>(su1, su2, skk, until + (size_t)(svc & 0xFFFFu) * w1, dom, ts, T);
            level_masks<W>(s, r, c, dom, T, asp_s, m0, m1, m2);
            uint64_t o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
            for (int z = 0; z < W; ++z) {
                o0 |= m0[z];
                o1 |= m1[z];
                o2 |= m2[z];
            }
            const unsigned lv = o0 ? 0u : o1 ? 1u : o2 ? 2u : 3u;
            const int lc = (int)__reduce_min_sync(kFull, lv);
            uint64_t m[W];
#pragma unroll
            for (int z = 0; z < W; ++z) m[z] = lc == 0 ? m0[z] : lc == 1 ? m1[z] : m2[z];
            const int cnt = popc_w<W>(m);
            int incl = warp_incl_sum(cnt);
            const int N = __shfl_sync(kFull, incl, 31);
            if (N == 0) {
                // every candidate tabu: no move, the clock still advances (partial.hpp:121-122)
                if (lane == 0) acc += 2ULL * (unsigned)w1 * (unsigned)f;
                if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                    trace_step(j, -1, 0, -1, -1, 0, 0, f, f, bestf, -1, 0, 2);
                ++j;
                if (!((int64_t)j < budget) ||
                    ((j & 63) == 0 && poll_stop(j)))
                    break;
                continue;
            }
            const uint32_t rnk = __umulhi(g1, (uint32_t)N);
            const int excl = incl - cnt;
            const int wl = __ffs(__ballot_sync(kFull, (uint32_t)excl <= rnk && rnk < (uint32_t)incl)) - 1;
            const int ks = warp_nth_bit<W>(m, (int)rnk - __shfl_sync(kFull, excl, wl), wl, lane);
            const uint32_t vcs = __shfl_sync(kFull, svc, wl);
            const int vs = (int)(vcs & 0xFFFFu), rs_ = (vcs >> 16) & 0xFF, cs_ = vcs >> 24;
            const int lvl = lc - 1;
            if (pending && lvl >= 0) {
                // the current colouring is the best one and is about to change without improving
                snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
                pending = false;
            }
            const int kw = ks >> 6;
            const uint64_t bitk = 1ULL << (ks & 63);
            const bool inR = (s.R[rs_ * W + kw] & bitk) != 0;
            const bool inC = (s.C[cs_ * W + kw] & bitk) != 0;
            // ---- the row / column holder of k* (at most one each: the colouring is legal)
            const int ur = warp_find_byte(col, g.rs[rs_], g.rs[rs_ + 1], ks, inR, lane);
            const int xc = warp_find_byte(colT, g.cs[cs_], g.cs[cs_ + 1], ks, inC, lane);
            const int uc = xc >= 0 ? (int)g.cl[xc] : -1;
            const int e = (ur >= 0) + (uc >= 0);
            const int f_new = f - 1 + e;
            const uint32_t tenure = __umulhi(g2, 10u) + (uint32_t)(alpha * (double)f_new);
            const uint32_t ut = ts + 1 + tenure;
            const bool improved = f_new < bestf;
            // ---- the move: predicated five-lane update (improve_common.cuh apply_move_lanes)
            const TabuRec nr = apply_move_lanes<W>(g, s, rec, until, vs, ur, uc, ks, rs_, cs_, inR, inC, fb, improved,
                                                   ut, ts, lane, acc);
            f = f_new;
            if (improved) {
                bestf = f;
                pending = true;
                if (race_flag && bestf <= race_f && lane == 0) atomicExch(const_cast<int*>(race_flag), 1);
            }
            if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                trace_step(j, vs, ks, ur, uc, rs_, cs_, fb, f, bestf, (int)tenure, N, lvl);
            ++j;
            if (f_new > 32) {
                __syncwarp();
                if (prof) {
                    pc_sparse += (unsigned long long)(clock64() - t_step);
                    ++pn_sparse;
                }
                break;  // back to dense mode; the slot list is rebuilt on re-entry
            }
            // ---- re-sort the slot list: new = old - {v*} + {ur, uc}
            {
                const int vl = (int)(svc & 0xFFFFu);
                const bool old_ok = mine && lane != wl;
                const unsigned br = __ballot_sync(kFull, old_ok && vl < ur);
                const unsigned bc = __ballot_sync(kFull, old_ok && vl < uc);
                // new lanes of ur / uc (64 = absent; -1 compares as the largest unsigned id)
                const int pr_ = ur >= 0 ? __popc(br) + ((unsigned)uc < (unsigned)ur) : 64;
                const int pc_ = uc >= 0 ? __popc(bc) + ((unsigned)ur < (unsigned)uc) : 64;
                const int y = lane - (pr_ < lane) - (pc_ < lane);
                const int src = (y >= wl ? y + 1 : y) & 31;
                const uint32_t mvc = __shfl_sync(kFull, svc, src);
                const uint32_t mu1 = __shfl_sync(kFull, su1, src);
                const uint32_t mu2 = __shfl_sync(kFull, su2, src);
                const uint32_t mkk = __shfl_sync(kFull, skk, src);
                const int from = lane == pr_ ? 1 : 2;  // evictee caches come from lanes 1 / 2
                const uint32_t nu1 = __shfl_sync(kFull, nr.u1, from);
                const uint32_t nu2 = __shfl_sync(kFull, nr.u2, from);
                const uint32_t nkk = __shfl_sync(kFull, nr.kk, from);
                const bool take_new = lane == pr_ || lane == pc_;
                const int u = lane == pr_ ? ur : uc;
                const uint16_t rc = g.cell[take_new ? u : 0];
                svc = take_new ? ((uint32_t)u | ((uint32_t)(rc >> 8) << 16) | ((uint32_t)(rc & 0xFF) << 24)) : mvc;
                su1 = take_new ? nu1 : mu1;
                su2 = take_new ? nu2 : mu2;
                skk = take_new ? nkk : mkk;
            }
            __syncwarp();
            if (prof) {
                pc_sparse += (unsigned long long)(clock64() - t_step);
                ++pn_sparse;
            }
            if (!((int64_t)j < budget && bestf > stop_f)) break;
            if ((j & 63) == 0 && poll_stop(j)) break;
        }
    }
    if (pending) snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
    {
        // lanes 0..2 hold the byte-counter parts
        const unsigned long long a1 = __shfl_sync(kFull, acc, 1), a2 = __shfl_sync(kFull, acc, 2);
        acc += a1 + a2;
    }
    if (lane == 0) {
        a.best_f[i] = bestf;
        a.repaired_f[i] = repaired_f;
        a.iters[i] = (int64_t)j;
        a.bytes[i] = acc;
        // every until written by this individual is < base + j + 1 + tenure_cap
        *slot_clock = base + j + 2 + a.tenure_cap;
    }
    if (prof && lane == 0) {
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
    __syncwarp();
}

template <int W, bool kDebug>
__global__ void __launch_bounds__(kImproveMaxThreads, kImproveMinBlocks) k_improve(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, nv = a.nv;
    const ImproveSmemLayout L = improve_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + L.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + L.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + L.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + L.cl);
    uint16_t* s_cp = reinterpret_cast<uint16_t*>(smem + L.colpos);
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + L.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + L.pc);
    uint8_t* s_deg = smem + L.deg;
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
    g.nvpad = a.nvpad;
    g.lane_words = a.lane_words;
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

    uint8_t* wbase = smem + L.warp0 + (size_t)warp * L.warp_bytes;
    WarpSmem s;
    s.col = wbase + L.w_col;
    s.conf = nullptr;
    s.colT = wbase + L.w_colT;
    s.list = reinterpret_cast<uint16_t*>(wbase + L.w_list);
    s.R = reinterpret_cast<uint64_t*>(wbase + L.w_R);
    s.C = reinterpret_cast<uint64_t*>(wbase + L.w_C);
    s.U = reinterpret_cast<uint32_t*>(wbase + L.w_U);

    const int slot = blockIdx.x * nwarps + warp;
    TabuRec* rec = reinterpret_cast<TabuRec*>(reinterpret_cast<char*>(a.tabu_rec) + (size_t)slot * a.rec_stride);
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    uint8_t* conf = a.conf_scratch + (size_t)slot * a.conf_stride;

    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(a.work_counter, 1);
        i = __shfl_sync(kFull, i, 0);
        if (i >= a.p) break;
        improve_one<W, kDebug>(a, g, s, rec, until, a.slot_clock + slot, conf, i, lane);
    }
}

// W = 64-bit words per colour mask: 1 for n <= 63, 2 for n <= 127 (the u8 conflict
// counters of the repair bound n at 127; capi.cu rejects larger orders).
size_t tabu_rec_bytes(int) { return sizeof(TabuRec); }

const void* improve_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_improve<1, true>)
                             : reinterpret_cast<const void*>(&k_improve<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_improve<2, true>)
                 : reinterpret_cast<const void*>(&k_improve<2, false>);
}

cudaError_t launch_improve(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr || a.prof != nullptr || a.probe.n > 0;
    if (W == 1) {
        if (debug)
            k_improve<1, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve<1, false><<<grid, threads, smem, st>>>(a);
    } else {
        if (debug)
            k_improve<2, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve<2, false><<<grid, threads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace plse_dev
