// plits.cu -- the MPMA variant's improve operator: PLITS, the two-phase
// partial legal and illegal tabu search (plits.hpp:96-292), on sm_100a.
//
// Replaces engine.hpp:193-197 (plits_run per individual) with ONE WARP PER
// INDIVIDUAL, persistent over a work counter, like the PartialCol kernel
// (improve.cu).  Data layout:
//   * colours (u8) in shared memory; gamma is never materialised: for a
//     vertex v in row r / column c and any colour k != col(v),
//       gamma[v][k] = rcnt[r][k] + ccnt[c][k]
//     and gamma[v][col(v)] = rcnt[r][col v] + ccnt[c][col v] - 2, over the
//     per-row / per-column colour counts (u8 [n][n+1] each, shared memory).
//     PLITS colourings are illegal, so counts (not the occupancy bits of the
//     legal PartialCol state) are what the step needs.
//   * the neighbourhood N0 u Nc (plits.hpp:47-63) is an active-vertex
//     bitmask A: v is active iff col(v) = 0 or its row / column holds col(v)
//     twice.  A move changes counts in one row and one column only, so only
//     those cells are re-classified.
//   * tabu: the reference's dense until[v][k] (search_util.hpp:54-81) per
//     warp slot in HBM on the slot's monotone clock; a phase switch (fresh
//     table, plits.hpp:81) advances the clock past every live entry.  The scan
//     reads until[][] only for candidates at or below the lane's running
//     minimum, so the table costs a handful of loads per step.
//   * the objective is the integer 2F = wf*f + wc*c (plits.hpp:22-36):
//     (2, 1) in phase 1, (2, 2|V|) in phase 2; aspiration compares against
//     the phase best (plits.hpp:147).
//   * selection is the canonical order-free rule: the
//     minimum admissible delta, N candidates at it, r = floor(h1 * N / 2^32)
//     from the counter hash keyed by (stream seed, step over both phases),
//     the r-th candidate in ascending (v, k) order with k = 0 first; tenure
//     floor(h2 * 10 / 2^32) + floor(alpha * active) (plits.hpp:182-185).
//   * best tracking: deferred snapshot into the improved row (the row is
//     written only before a move that does not improve on the phase best).
#include <climits>

#include "improve_common.cuh"

namespace plse_dev {

struct PlitsWarp {
    uint8_t* col;   // [nvpad]
    uint8_t* rcnt;  // [n][n+1] colour counts per row (index 0 counts uncoloured cells)
    uint8_t* ccnt;  // [n][n+1] per column
    uint32_t* A;    // [32 * lane_words] active vertices; word v >> 5 (lane-owned blocks)
};

template <int W>
__device__ __forceinline__ bool plits_is_active(const Graph<W>& g, const PlitsWarp& s, int u, int w1) {
    const int k = s.col[u];
    if (!k) return true;
    const uint16_t rc = g.cell[u];
    return s.rcnt[(rc >> 8) * w1 + k] >= 2 || s.ccnt[(rc & 0xFF) * w1 + k] >= 2;
}

// counts, active set, f and c of the colouring in s.col (plits.hpp:104-116, coloring.hpp:59-73)
template <int W>
__device__ void plits_build(const Graph<W>& g, const PlitsWarp& s, int cnt_bytes, int lane, int& f, int& c,
                            int& active) {
    const int n = g.n, nv = g.nv, w1 = n + 1;
    uint4* z = reinterpret_cast<uint4*>(s.rcnt);
    for (int x = lane; x < cnt_bytes / 16; x += 32) z[x] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    for (int r = lane; r < n; r += 32) {
        uint8_t* row = s.rcnt + r * w1;
        for (int u = g.rs[r]; u < g.rs[r + 1]; ++u) row[s.col[u]] += 1;
    }
    for (int cc = lane; cc < n; cc += 32) {
        uint8_t* row = s.ccnt + cc * w1;
        for (int x = g.cs[cc]; x < g.cs[cc + 1]; ++x) row[s.col[g.cl[x]]] += 1;
    }
    __syncwarp();
    const int v_lo = lane * 32 * g.lane_words;
    int fl = 0, cl2 = 0, al = 0;
    for (int q = 0; q < g.lane_words; ++q) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            const int v = v_lo + 32 * q + b;
            if (v >= nv) break;
            const int k = s.col[v];
            if (!k) {
                bits |= 1u << b;
                ++fl;
            } else {
                const uint16_t rc = g.cell[v];
                const int gv = s.rcnt[(rc >> 8) * w1 + k] + s.ccnt[(rc & 0xFF) * w1 + k] - 2;
                cl2 += gv;
                if (gv) bits |= 1u << b;
            }
        }
        s.A[lane * g.lane_words + q] = bits;
        al += __popc(bits);
    }
    f = (int)__reduce_add_sync(kFull, (unsigned)fl);
    c = (int)__reduce_add_sync(kFull, (unsigned)cl2) / 2;
    active = (int)__reduce_add_sync(kFull, (unsigned)al);
    __syncwarp();
}

template <int W, bool kDebug>
__device__ void plits_one(const ImproveArgs& a, const Graph<W>& g, const PlitsWarp& s, int cnt_bytes,
                          uint32_t* until, uint32_t* slot_clock, int i, int lane) {
    const int n = g.n, nv = g.nv, w1 = n + 1;
    const int v_lo = lane * 32 * g.lane_words;
    const int v_hi = min(nv, v_lo + 32 * g.lane_words);
    uint8_t* col = s.col;
    uint8_t* best_row = a.improved + (size_t)i * g.nvpad;
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;

    // ---- tabu clock of this warp slot (two phases, each followed by a skip of tenure_cap + 2)
    uint32_t base = *slot_clock;
    if ((uint64_t)base + (uint64_t)a.budget + (uint64_t)a.budget2 + 2ull * (a.tenure_cap + 4) >= 0xFFFFFFFFull) {
        uint4* u4 = reinterpret_cast<uint4*>(until);
        for (size_t x = lane; x < a.until_stride / 4; x += 32) u4[x] = make_uint4(0, 0, 0, 0);
        base = 0;
    }

    {
        const uint4* src = reinterpret_cast<const uint4*>(a.offspring + (size_t)i * g.nvpad);
        uint4* d4 = reinterpret_cast<uint4*>(col);
        for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
    }
    __syncwarp();

    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    const uint32_t s32 = (uint32_t)(seed ^ (seed >> 32));
    const int stop_f = a.stop_f;
    const double alpha = a.alpha;
    const int* race_flag = a.race_flag;
    const unsigned long long* deadline = a.deadline;
    // per phase: race flag every 64 steps, deadline after every 4096th (plits.hpp:262)
    auto poll_stop = [race_flag, deadline](uint32_t jj) -> bool {
        if (race_flag && *reinterpret_cast<const volatile int*>(race_flag)) return true;
        if (!deadline || jj == 0 || (jj & 0xFFFu)) return false;
        return __shfl_sync(kFull, globaltimer_ns() >= *deadline ? 1 : 0, 0) != 0;
    };

    int f = 0, c = 0, active = 0;
    plits_build<W>(g, s, cnt_bytes, lane, f, c, active);
    const int initial_f = f;
    uint32_t J = 0;        // step index over both phases: the canonical draw's key
    int64_t iters = 0;
    bool hit = false;
    bool pending = true;   // the phase best equals the current colouring
    int best_f = f, best_c = c;
    unsigned long long acc = 0;

    for (int phase = 1; phase <= 2; ++phase) {
        const int wf = 2;
        const int wc = phase == 1 ? 1 : 2 * nv;  // PhaseWeights::from_phi(0.5 / |V|), plits.hpp:27-33
        const int64_t budget = phase == 1 ? a.budget : a.budget2;
        if (phase == 2) {
            // plits.hpp:285-288: phase 2 starts from phase 1's best with a fresh tabu table
            if (!pending) {
                const uint4* src = reinterpret_cast<const uint4*>(best_row);
                uint4* d4 = reinterpret_cast<uint4*>(col);
                for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
                __syncwarp();
            }
            plits_build<W>(g, s, cnt_bytes, lane, f, c, active);
        }
        int64_t best_scaled = (int64_t)wf * f + (int64_t)wc * c;
        best_f = f;
        best_c = c;
        pending = true;
        uint32_t j = 0;
        for (;;) {
            if (best_c == 0 && best_f <= stop_f) {
                hit = true;
                break;
            }
            if (!((int64_t)j < budget)) break;
            if (active == 0) break;  // StepResult::Exhausted: not counted
            if ((j & 63) == 0 && poll_stop(j)) break;
            const uint32_t t = base + j;
            const uint32_t h1 = fmix32(s32 + (J + 1) * 0x9E3779B9u);
            const uint32_t h2 = fmix32(h1 + 0x632BE5ABu);
            const int64_t cur_scaled = (int64_t)wf * f + (int64_t)wc * c;
            const int64_t thr64 = best_scaled - cur_scaled;  // tabu move admissible iff delta < thr
            const int thr = (int)max(min(thr64, (int64_t)INT_MAX), (int64_t)INT_MIN);
            const int active_before = active;

            // ---- pass 1: each lane's minimum admissible delta and its multiplicity
            int lmin = INT_MAX, lcnt = 0;
            for (int q = 0; q < g.lane_words; ++q) {
                uint32_t bits = s.A[lane * g.lane_words + q];
                while (bits) {
                    const int v = v_lo + 32 * q + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const uint16_t rc = g.cell[v];
                    const int r = rc >> 8, cc = rc & 0xFF;
                    const int cur = col[v];
                    const uint8_t* rrow = s.rcnt + r * w1;
                    const uint8_t* crow = s.ccnt + cc * w1;
                    const uint32_t* urow = until + (size_t)v * w1;
                    const int gcur = cur ? rrow[cur] + crow[cur] - 2 : 0;
                    if (cur) {
                        const int d = wf - wc * gcur;  // to 0: df = +1, dc = -gamma[v][cur]
                        if (d <= lmin && !(urow[0] > t && !(d < thr))) {
                            if (d < lmin) {
                                lmin = d;
                                lcnt = 1;
                            } else {
                                ++lcnt;
                            }
                        }
                    }
                    const int dbase = (cur ? 0 : -wf) - wc * gcur;
                    uint64_t dom[W];
                    dom_mask<W>(g, r, cc, dom);
                    if (cur) dom[cur >> 6] &= ~(1ULL << (cur & 63));
#pragma unroll
                    for (int qq = 0; qq < W; ++qq) {
                        uint64_t m = dom[qq];
                        while (m) {
                            const int k = qq * 64 + __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const int d = dbase + wc * (rrow[k] + crow[k]);
                            if (d > lmin) continue;
                            if (urow[k] > t && !(d < thr)) continue;
                            if (d < lmin) {
                                lmin = d;
                                lcnt = 1;
                            } else {
                                ++lcnt;
                            }
                        }
                    }
                }
            }
            const int dmin = __reduce_min_sync(kFull, lmin);
            if (dmin == INT_MAX) {
                // every candidate tabu: the clock still advances (plits.hpp:178-179)
                if (lane == 0) acc += 2ULL * (unsigned)w1 * (unsigned)active_before;
                if (tracing && lane == 0 && (int64_t)J < a.trace_cap) {
                    plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + J;
                    *tr = plse_step{(int64_t)J, -1, 0, phase, 0, active, f, c, (int32_t)best_scaled, -1, 0, 0};
                }
                ++j;
                ++J;
                continue;
            }
            const int cnt = lmin == dmin ? lcnt : 0;
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(kFull, incl, d);
                incl += lane >= d ? x : 0;
            }
            const int N = __shfl_sync(kFull, incl, 31);
            const uint32_t rnk = __umulhi(h1, (uint32_t)N);
            const int excl = incl - cnt;
            const bool owner = (uint32_t)excl <= rnk && rnk < (uint32_t)incl;
            int sv = -1, sk = 0, sdc = 0;
            if (owner) {
                // ---- pass 2 (one lane): the (rnk - excl)-th admissible candidate at dmin, ascending (v, k)
                int left = (int)rnk - excl;
                for (int q = 0; q < g.lane_words && sv < 0; ++q) {
                    uint32_t bits = s.A[lane * g.lane_words + q];
                    while (bits && sv < 0) {
                        const int v = v_lo + 32 * q + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const uint16_t rc = g.cell[v];
                        const int r = rc >> 8, cc = rc & 0xFF;
                        const int cur = col[v];
                        const uint8_t* rrow = s.rcnt + r * w1;
                        const uint8_t* crow = s.ccnt + cc * w1;
                        const uint32_t* urow = until + (size_t)v * w1;
                        const int gcur = cur ? rrow[cur] + crow[cur] - 2 : 0;
                        if (cur) {
                            const int d = wf - wc * gcur;
                            if (d == dmin && !(urow[0] > t && !(d < thr))) {
                                if (left == 0) {
                                    sv = v;
                                    sk = 0;
                                    sdc = -gcur;
                                    break;
                                }
                                --left;
                            }
                        }
                        const int dbase = (cur ? 0 : -wf) - wc * gcur;
                        uint64_t dom[W];
                        dom_mask<W>(g, r, cc, dom);
                        if (cur) dom[cur >> 6] &= ~(1ULL << (cur & 63));
                        for (int qq = 0; qq < W && sv < 0; ++qq) {
                            uint64_t m = dom[qq];
                            while (m) {
                                const int k = qq * 64 + __ffsll((long long)m) - 1;
                                m &= m - 1;
                                const int gk = rrow[k] + crow[k];
                                const int d = dbase + wc * gk;
                                if (d != dmin) continue;
                                if (urow[k] > t && !(d < thr)) continue;
                                if (left == 0) {
                                    sv = v;
                                    sk = k;
                                    sdc = gk - gcur;
                                    break;
                                }
                                --left;
                            }
                        }
                    }
                }
            }
            const int wl = __ffs(__ballot_sync(kFull, owner)) - 1;
            const int vs = __shfl_sync(kFull, sv, wl);
            const int ks = __shfl_sync(kFull, sk, wl);
            const int dcs = __shfl_sync(kFull, sdc, wl);
            const int from = col[vs];
            const int dfs = (ks == 0) - (from == 0);
            const int64_t now = cur_scaled + dmin;
            if (now >= best_scaled && pending) {
                // deferred snapshot: the colouring about to change is the phase best
                const uint4* src = reinterpret_cast<const uint4*>(col);
                uint4* d4 = reinterpret_cast<uint4*>(best_row);
                for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
                pending = false;
            }
            __syncwarp();
            const uint16_t rcs = g.cell[vs];
            const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
            if (lane == 0) {
                col[vs] = (uint8_t)ks;
                s.rcnt[rs_ * w1 + from] -= 1;
                s.ccnt[cs_ * w1 + from] -= 1;
                s.rcnt[rs_ * w1 + ks] += 1;
                s.ccnt[cs_ * w1 + ks] += 1;
            }
            __syncwarp();
            // ---- membership around the move (plits.hpp:193-212): re-classify v's row and column
            for (int u = g.rs[rs_] + lane; u < g.rs[rs_ + 1]; u += 32) {
                const uint32_t bit = 1u << (u & 31);
                if (plits_is_active<W>(g, s, u, w1))
                    atomicOr(&s.A[u >> 5], bit);
                else
                    atomicAnd(&s.A[u >> 5], ~bit);
            }
            for (int x = g.cs[cs_] + lane; x < g.cs[cs_ + 1]; x += 32) {
                const int u = g.cl[x];
                const uint32_t bit = 1u << (u & 31);
                if (plits_is_active<W>(g, s, u, w1))
                    atomicOr(&s.A[u >> 5], bit);
                else
                    atomicAnd(&s.A[u >> 5], ~bit);
            }
            __syncwarp();
            {
                int al = 0;
                for (int q = 0; q < g.lane_words; ++q) al += __popc(s.A[lane * g.lane_words + q]);
                active = (int)__reduce_add_sync(kFull, (unsigned)al);
            }
            f += dfs;
            c += dcs;
            const uint32_t tenure = __umulhi(h2, 10u) + (uint32_t)(alpha * (double)active);
            if (lane == 0) {
                until[(size_t)vs * w1 + from] = t + 1 + tenure;
                acc += 2ULL * (unsigned)w1 * (unsigned)active_before + 4ULL * g.deg[vs] + 2ULL;
            }
            if (now < best_scaled) {
                best_scaled = now;
                best_f = f;
                best_c = c;
                pending = true;
                if (lane == 0) acc += 2ULL * (unsigned)nv;
                if (race_flag && best_c == 0 && best_f <= a.race_f && lane == 0)
                    atomicExch(const_cast<int*>(race_flag), 1);
            }
            if (tracing && lane == 0 && (int64_t)J < a.trace_cap) {
                plse_step* tr = reinterpret_cast<plse_step*>(a.trace) + J;
                *tr = plse_step{(int64_t)J, vs, ks, phase, from, active, f, c, (int32_t)best_scaled, (int32_t)tenure,
                                N, dmin};
            }
            __syncwarp();
            ++j;
            ++J;
        }
        if (best_c == 0 && best_f <= stop_f) hit = true;
        iters += j;
        // the phase's result is its best colouring (plits.hpp:268)
        if (!pending) {
            const uint4* src = reinterpret_cast<const uint4*>(best_row);
            uint4* d4 = reinterpret_cast<uint4*>(col);
            for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
            __syncwarp();
            pending = true;
        }
        base += j + 2 + a.tenure_cap;  // every until written in this phase is < base
        if (hit) break;                // plits.hpp:284: phase 2 only when phase 1 missed the target
    }

    // ---- final greedy repair when the result still conflicts (plits.hpp:289, partial.hpp:22-39)
    if (best_c > 0) {
        plits_build<W>(g, s, cnt_bytes, lane, f, c, active);
        for (;;) {
            int bc = 0, bv = -1;
            for (int v = v_lo; v < v_hi; ++v) {
                const int k = col[v];
                if (!k) continue;
                const uint16_t rc = g.cell[v];
                const int gv = s.rcnt[(rc >> 8) * w1 + k] + s.ccnt[(rc & 0xFF) * w1 + k] - 2;
                if (gv > bc) {
                    bc = gv;
                    bv = v;
                }
            }
            const int mx = (int)__reduce_max_sync(kFull, (unsigned)bc);
            if (mx == 0) break;
            const int wl = __ffs(__ballot_sync(kFull, bc == mx)) - 1;
            const int w = __shfl_sync(kFull, bv, wl);
            if (lane == 0) {
                const uint16_t rc = g.cell[w];
                const int k = col[w];
                col[w] = 0;
                s.rcnt[(rc >> 8) * w1 + k] -= 1;
                s.ccnt[(rc & 0xFF) * w1 + k] -= 1;
                s.rcnt[(rc >> 8) * w1] += 1;
                s.ccnt[(rc & 0xFF) * w1] += 1;
            }
            ++f;
            __syncwarp();
        }
        best_f = f;
        if (lane == 0) acc += 2ULL * (unsigned)nv;
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(col);
        uint4* d4 = reinterpret_cast<uint4*>(best_row);
        for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
    }
    if (lane == 0) {
        a.best_f[i] = best_f;
        a.repaired_f[i] = initial_f;
        a.iters[i] = iters;
        a.bytes[i] = acc;
        *slot_clock = base;
        if (race_flag && best_f <= a.race_f) atomicExch(const_cast<int*>(race_flag), 1);
    }
    __syncwarp();
}

template <int W, bool kDebug>
__global__ void __launch_bounds__(kImproveMaxThreads, kImproveMinBlocks) k_plits(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, nv = a.nv;
    const ImproveSmemLayout G = improve_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    const PlitsSmemLayout L = plits_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + G.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + G.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + G.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + G.cl);
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + G.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + G.pc);
    uint8_t* s_deg = smem + G.deg;
    for (int x = threadIdx.x; x < nv; x += blockDim.x) {
        s_cell[x] = a.cell[x];
        s_cl[x] = a.col_list[x];
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
    g.colpos = nullptr;
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
    PlitsWarp s;
    s.col = wbase + L.w_col;
    s.rcnt = wbase + L.w_rcnt;
    s.ccnt = wbase + L.w_ccnt;
    s.A = reinterpret_cast<uint32_t*>(wbase + L.w_A);
    const int cnt_bytes = (int)(L.w_A - L.w_rcnt);

    const int slot = blockIdx.x * nwarps + warp;
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(a.work_counter, 1);
        i = __shfl_sync(kFull, i, 0);
        if (i >= a.p) break;
        plits_one<W, kDebug>(a, g, s, cnt_bytes, until, a.slot_clock + slot, i, lane);
    }
}

const void* plits_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_plits<1, true>)
                             : reinterpret_cast<const void*>(&k_plits<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_plits<2, true>)
                 : reinterpret_cast<const void*>(&k_plits<2, false>);
}

cudaError_t launch_plits(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr;
    if (W == 1) {
        if (debug)
            k_plits<1, true><<<grid, threads, smem, st>>>(a);
        else
            k_plits<1, false><<<grid, threads, smem, st>>>(a);
    } else {
        if (debug)
            k_plits<2, true><<<grid, threads, smem, st>>>(a);
        else
            k_plits<2, false><<<grid, threads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace plse_dev
