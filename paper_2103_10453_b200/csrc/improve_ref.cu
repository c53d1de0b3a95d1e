// improve_ref.cu -- PartialCol with the REFERENCE's own tie-break (PLSE_TIE_REF) on sm_100a.
//
// The canonical kernel (improve.cu) replaces the reference's reservoir
// sampling by an order-free counter-hash rule.  This kernel reproduces the
// reference bit for bit instead (partial.hpp:92-143): the uncoloured set is
// kept in IndexSet order (search_util.hpp:12-49: insert appends, erase moves
// the last element into the hole), the candidates are visited in that order
// with colours ascending, and every tie with the running best draws
// next_below(++ties) from the individual's xoshiro256++ stream (rng.hpp:43-49)
// -- so the draws are a serial chain, which one lane walks while the warp
// computes the move masks 32 vertices at a time.  The tenure draw
// next_below(10) follows the move (partial.hpp:136-137).  Everything else --
// repair, gamma from the occupancy masks, tabu records, eviction, deferred
// best snapshot, the byte counter -- is the canonical kernel's.
//
// With this kernel the whole device run() equals the reference's run() (the
// population phases are bit-exact already); it is the parity mode, the
// canonical kernel the throughput mode.
#include "improve_common.cuh"
#include "ref_draws.cuh"

namespace plse_dev {

// ---- the same selection computed in parallel when the uncoloured set fits one warp (|V0| <= 32).
// Levels are -1 / 0 / +1 (index 0 / 1 / 2), so the reservoir's history is a handful of segments:
// the prefix minimum of the per-vertex minimum level says where each vertex enters; a vertex's draws
// are the candidates at the running level between the events where the level drops; the final
// segment is every admissible candidate at the global minimum level D from its first one c* on, and
// its j-th member (j >= 2) draws next_below(j).  Lane 0 only generates the stream (one next() per
// draw); the lanes test their own final-segment draws.  Any output below 2^32 (a possible rejection,
// probability 2^-32 per draw) or an oversized final segment falls back to the serial walk.

template <int W>
__device__ __forceinline__ uint64_t word_sel(const uint64_t (&x)[W], int q) {
    return (W == 1 || q == 0) ? x[0] : x[W - 1];
}

// first set bit of a W-word mask after position pos (-1: from the start), or -1
template <int W>
__device__ __forceinline__ int next_bit(const uint64_t (&m)[W], int pos) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const int lo = pos + 1 - 64 * q;
        uint64_t x = m[q];
        if (lo >= 64) continue;
        if (lo > 0) x &= ~0ULL << lo;
        if (x) return 64 * q + __ffsll((long long)x) - 1;
    }
    return -1;
}

// set bits of m in the open range (pos, e) (e = -1: to the end)
template <int W>
__device__ __forceinline__ int popc_range(const uint64_t (&m)[W], int pos, int e) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t x = m[q];
        const int lo = pos + 1 - 64 * q, hi = e < 0 ? 64 : e - 64 * q;  // keep bits [lo, hi)
        if (lo >= 64 || hi <= 0) continue;
        if (lo > 0) x &= ~0ULL << lo;
        if (hi < 64) x &= (1ULL << hi) - 1;
        c += __popcll(x);
    }
    return c;
}

// dense_masks with the vertex's tabu record held by the lane (the fast path |V0| <= 32 keeps each IndexSet
// position's record in its lane across steps: no vertex that stays uncoloured is written by anyone else);
// a cache rebuild is still written back, so HBM stays authoritative for the vertex's next owner
template <int W>
__device__ __forceinline__ void dense_masks_held(const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                                                 const uint32_t* until, int v, uint32_t t, bool asp, TabuRec& tr,
                                                 uint64_t (&m0)[W], uint64_t (&m1)[W], uint64_t (&m2)[W]) {
    const uint16_t rc = g.cell[v];
    const int r = rc >> 8, c = rc & 0xFF;
    uint64_t dom[W], T[W];
    dom_mask<W>(g, r, c, dom);
    const uint32_t kk0 = tr.kk;
    tabu_of<W>(tr.u1, tr.u2, tr.kk, until + (size_t)v * (g.n + 1), dom, t, T);
    if (tr.kk != kk0) rec[v] = tr;
    level_masks<W>(s, r, c, dom, T, asp, m0, m1, m2);
}

// draws the reference makes inside one vertex entered at running level cur (3 = nothing found yet),
// stopping at its first level-`stop` candidate when stop < 3
template <int W>
__device__ __forceinline__ int vertex_draws(const uint64_t (&a0)[W], const uint64_t (&a1)[W], const uint64_t (&a2)[W],
                                            int cur, int stop) {
    int draws = 0, pos = -1;
    for (int it = 0; it < 4; ++it) {
        uint64_t lower[W], atcur[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
            lower[q] = cur == 3 ? (a0[q] | a1[q] | a2[q]) : cur == 2 ? (a0[q] | a1[q]) : cur == 1 ? a0[q] : 0ULL;
            atcur[q] = cur == 0 ? a0[q] : cur == 1 ? a1[q] : cur == 2 ? a2[q] : 0ULL;
        }
        const int e = next_bit<W>(lower, pos);
        if (cur != 3) draws += popc_range<W>(atcur, pos, e);
        if (e < 0) break;
        const uint64_t bit = 1ULL << (e & 63);
        const int q = e >> 6;
        const int lvl = (word_sel<W>(a0, q) & bit) ? 0 : (word_sel<W>(a1, q) & bit) ? 1 : 2;
        if (lvl == stop) break;  // c*, the first candidate of the final level
        cur = lvl;
        pos = e;
    }
    return draws;
}

struct RefScan {
    int found, bd, cv, ck, cpos;
    uint32_t ties;
};

// partial.hpp:100-117 over one vertex's admissible candidates (x0: delta -1, x1: 0, x2: +1), k ascending
template <int W>
__device__ __forceinline__ void ref_walk(RefScan& st, Xoshiro& rng, const uint64_t* x0, const uint64_t* x1,
                                         const uint64_t* x2, int v, int pos) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const uint64_t a0 = x0[q], a1 = x1[q], a2 = x2[q];
        // `if (found && d > bd) continue;` -- only levels <= bd are visited
        uint64_t rel = !st.found ? (a0 | a1 | a2) : st.bd < 0 ? a0 : st.bd == 0 ? (a0 | a1) : (a0 | a1 | a2);
        while (rel) {
            const int b = __ffsll((long long)rel) - 1;
            const uint64_t bit = 1ULL << b;
            rel &= rel - 1;
            const int l = (a0 & bit) ? -1 : (a1 & bit) ? 0 : 1;
            if (!st.found || l < st.bd) {
                st.found = 1;
                st.bd = l;
                st.ties = 1;
                st.cv = v;
                st.ck = q * 64 + b;
                st.cpos = pos;
                rel &= l < 0 ? a0 : l == 0 ? (a0 | a1) : (a0 | a1 | a2);
            } else if (ref_below_is_zero(rng, ++st.ties)) {
                st.cv = v;
                st.ck = q * 64 + b;
                st.cpos = pos;
            }
        }
    }
}

// the same scan for |V0| > 32: 32 vertices per round, lane p owning vertex 32 c + p, the masks
// recomputed per pass (minimum, counts, owner)
template <int W>
__device__ __forceinline__ bool partial_ref_fast(const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                                                 const uint32_t* until, const uint16_t* el, uint64_t* msk, int f,
                                                 uint32_t t, bool asp, int lane, Xoshiro& rng, RefScan& st,
                                                 unsigned long long* pc) {
    long long tf = pc ? clock64() : 0;
    auto fstamp = [&](int z) {
        if (pc) {
            const long long x = clock64();
            pc[z] += (unsigned long long)(x - tf);
            tf = x;
        }
    };
    const int nch = (f + 31) >> 5;
    uint64_t a0[W], a1[W], a2[W];
    auto masks_of = [&](int c) {
#pragma unroll
        for (int q = 0; q < W; ++q) a0[q] = a1[q] = a2[q] = 0;
        const int p = 32 * c + lane;
        if (p < f) dense_masks<W>(g, s, rec, until, el[p], t, asp, a0, a1, a2);
    };
    auto level_of = [&](int c) -> int {
        return (32 * c + lane >= f) ? 3 : popc_w<W>(a0) ? 0 : popc_w<W>(a1) ? 1 : popc_w<W>(a2) ? 2 : 3;
    };
    // ---- pass 1: the global minimum level
    int D = 3;
    for (int c = 0; c < nch; ++c) {
        masks_of(c);
        D = min(D, (int)__reduce_min_sync(kFull, (unsigned)level_of(c)));
    }
    fstamp(6);
    if (D == 3) return true;  // no admissible candidate: no draw at all
    // ---- pass 2: early draws up to the first level-D candidate, the size of the final segment
    int E = 0, ND = 0, Rc = 3, cD1 = 0, incl1 = 0;
    bool seen = false;
    for (int c = 0; c < nch; ++c) {
        if (nch > 1) masks_of(c);
        const int m = level_of(c);
        const int pm = warp_incl_min(m);  // inclusive prefix minimum of the per-vertex minimum level
        if (!seen) {
            int R = __shfl_up_sync(kFull, pm, 1);
            if (lane == 0) R = 3;
            R = min(R, Rc);
            const unsigned bal = __ballot_sync(kFull, m == D);
            const int istar = bal ? __ffs(bal) - 1 : 32;
            int early = 0;
            if (lane <= istar && 32 * c + lane < f) early = vertex_draws<W>(a0, a1, a2, R, lane == istar ? D : 3);
            E += (int)__reduce_add_sync(kFull, (unsigned)early);
            seen = bal != 0;
        }
        uint64_t aD[W];
#pragma unroll
        for (int q = 0; q < W; ++q) aD[q] = D == 0 ? a0[q] : D == 1 ? a1[q] : a2[q];
        cD1 = popc_w<W>(aD);
        incl1 = warp_incl_sum(cD1);  // inclusive prefix sum of the level-D counts (kept for a one-round set)
        ND += __shfl_sync(kFull, incl1, 31);
        Rc = min(Rc, __shfl_sync(kFull, pm, 31));
    }
    fstamp(7);
    // ---- final-segment member j (1-based; the first is j = 1) keeps the choice iff next_below(j) == 0,
    // draw E + j - 2 of the stream (ref_stream_draws)
    const Xoshiro saved = rng;
    bool bad = false;
    const int bestj = ref_stream_draws(rng, msk, E, E + ND - 1, lane, bad);
    fstamp(8);
    if (bad) {
        if (lane == 0) rng = saved;  // take the exact path
        return false;
    }
    int J = (int)__reduce_max_sync(kFull, (unsigned)bestj);
    if (J == 0) J = 1;
    // ---- pass 3: the owner of member J
    int based = 0;
    for (int c = 0; c < nch; ++c) {
        if (nch > 1) masks_of(c);
        uint64_t aD[W];
#pragma unroll
        for (int q = 0; q < W; ++q) aD[q] = (32 * c + lane >= f) ? 0ULL : D == 0 ? a0[q] : D == 1 ? a1[q] : a2[q];
        int cD = cD1, incl = incl1;
        if (nch > 1) {
            cD = popc_w<W>(aD);
            incl = warp_incl_sum(cD);
        }
        const int tot = nch > 1 ? __shfl_sync(kFull, incl, 31) : ND;
        if (J > based + tot) {
            based += tot;
            continue;
        }
        const int sD = based + incl - cD;
        const bool own = sD < J && J <= sD + cD;
        int cv = 0, ck = 0, cpos = 0;
        if (own) {
            cpos = 32 * c + lane;
            cv = el[cpos];
            ck = nth_bit_w<W>(aD, J - sD - 1);
        }
        const int wl = __ffs(__ballot_sync(kFull, own)) - 1;
        st.found = 1;
        st.bd = D - 1;
        st.ties = (uint32_t)ND;
        st.cv = __shfl_sync(kFull, cv, wl);
        st.ck = __shfl_sync(kFull, ck, wl);
        st.cpos = __shfl_sync(kFull, cpos, wl);
        break;
    }
    __syncwarp();
    fstamp(9);
    return true;
}

template <int W, bool kDebug>
__device__ void improve_ref_one(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, uint16_t* el,
                                uint64_t* msk, TabuRec* rec, uint32_t* until, uint32_t* slot_clock, uint8_t* conf, int i,
                                int lane) {
    const int nv = g.nv, w1 = g.n + 1;
    uint8_t* col = s.col;
    uint8_t* colT = s.colT;
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
    unsigned long long* prof = kDebug ? a.prof : nullptr;
    // steps, mask cycles, walk cycles, apply cycles, draws, sum f | fast path: masks, scans, stream, owner
    unsigned long long pc[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

    long long tq = 0;

    uint32_t base = *slot_clock;
    if ((uint64_t)base + (uint64_t)a.budget + a.tenure_cap + 2 >= 0xFFFFFFFFull) {
        uint4* u4 = reinterpret_cast<uint4*>(until);
        for (size_t x = lane; x < a.until_stride / 4; x += 32) u4[x] = make_uint4(0, 0, 0, 0);
        base = 0;
    }
    int f = partial_prologue<W>(a, g, s, rec, conf, i, lane);

    // IndexSet order of the uncoloured set: ids ascending after the repair (partial.hpp:80-82)
    {
        int cnt = 0;
        for (int q = 0; q < g.lane_words; ++q) cnt += __popc(s.U[lane * g.lane_words + q]);
        const int incl = warp_incl_sum(cnt);
        int at = incl - cnt;
        const int v_lo = lane * 32 * g.lane_words;
        for (int q = 0; q < g.lane_words; ++q) {
            uint32_t bits = s.U[lane * g.lane_words + q];
            while (bits) {
                el[at++] = (uint16_t)(v_lo + 32 * q + __ffs(bits) - 1);
                bits &= bits - 1;
            }
        }
    }
    __syncwarp();

    // the tabu record of IndexSet position `lane` while |V0| <= 32 (held_v: its vertex, -1 = not held)
    TabuRec held{0, 0, 0, 0};
    int held_v = -1;

    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    Xoshiro rng(seed);  // the stream of Rng(derive_stream(master, kImprove, gen*p + i)), engine.hpp:189-191
    const int repaired_f = f;
    int bestf = f;
    bool pending = true;
    uint32_t j = 0;
    unsigned long long acc = 0;
    const int64_t budget = a.budget;
    const int stop_f = a.stop_f;
    const double alpha = a.alpha;
    const int* race_flag = a.race_flag;
    const unsigned long long* deadline = a.deadline;
    auto poll_stop = [race_flag, deadline](uint32_t jj) -> bool {
        if (race_flag && *reinterpret_cast<const volatile int*>(race_flag)) return true;
        if (!deadline || jj == 0 || (jj & 0xFFFu)) return false;
        return __shfl_sync(kFull, globaltimer_ns() >= *deadline ? 1 : 0, 0) != 0;
    };

    for (;;) {
        if (!((int64_t)j < budget && bestf > stop_f)) break;
        if (f == 0) break;  // step() == false: not counted (partial.hpp:93, 163)
        if ((j & 63) == 0 && poll_stop(j)) break;
        const uint32_t t = base + j;
        const bool asp = (f == bestf);
        const int f_before = f;

        // ---- the reservoir scan (partial.hpp:100-119)
        RefScan st{0, 2, -1, 0, -1, 0};
        if (prof) {
            tq = clock64();
            ++pc[0];
            pc[5] += (unsigned)f;
        }
        bool fast_done = false;
        if (f <= 32) {
            // one round: the masks of position `lane` stay in registers
            uint64_t a0[W], a1[W], a2[W];
#pragma unroll
            for (int q = 0; q < W; ++q) a0[q] = a1[q] = a2[q] = 0;
            if (lane < f) {
                const int v = el[lane];
                if (v != held_v) {
                    held = rec[v];
                    held_v = v;
                }
                dense_masks_held<W>(g, s, rec, until, v, t, asp, held, a0, a1, a2);
            }
            const int m = (lane >= f) ? 3 : popc_w<W>(a0) ? 0 : popc_w<W>(a1) ? 1 : popc_w<W>(a2) ? 2 : 3;
            const int D = (int)__reduce_min_sync(kFull, (unsigned)m);
            if (D == 3) {
                fast_done = true;  // no admissible candidate: no draw at all
            } else {
                const int pm = warp_incl_min(m);  // inclusive prefix minimum of the per-vertex minimum level
                int R = __shfl_up_sync(kFull, pm, 1);
                if (lane == 0) R = 3;
                const int istar = __ffs(__ballot_sync(kFull, m == D)) - 1;
                int early = 0;
                if (lane <= istar && lane < f) early = vertex_draws<W>(a0, a1, a2, R, lane == istar ? D : 3);
                uint64_t aD[W];
#pragma unroll
                for (int q = 0; q < W; ++q) aD[q] = D == 0 ? a0[q] : D == 1 ? a1[q] : a2[q];
                const int cD = popc_w<W>(aD);
                const int E = (int)__reduce_add_sync(kFull, (unsigned)early);
                int sD = warp_incl_sum(cD);  // inclusive prefix sum of the level-D counts
                const int ND = __shfl_sync(kFull, sD, 31);
                sD -= cD;  // exclusive: index (0-based) of this lane's first level-D candidate
                const Xoshiro saved = rng;
                if (prof) pc[10] += (unsigned)E;
                bool bad = false;
                const int bestj = ref_stream_draws(rng, msk, E, E + ND - 1, lane, bad);
                if (!bad) {
                    int J = (int)__reduce_max_sync(kFull, (unsigned)bestj);
                    if (J == 0) J = 1;
                    const bool own = sD < J && J <= sD + cD;
                    if (own) {
                        st.cv = el[lane];
                        st.ck = nth_bit_w<W>(aD, J - sD - 1);
                        st.cpos = lane;
                    }
                    const int wl = __ffs(__ballot_sync(kFull, own)) - 1;
                    st.found = 1;
                    st.bd = D - 1;
                    st.ties = (uint32_t)ND;
                    st.cv = __shfl_sync(kFull, st.cv, wl);
                    st.ck = __shfl_sync(kFull, st.ck, wl);
                    st.cpos = __shfl_sync(kFull, st.cpos, wl);
                    fast_done = true;
                } else if (lane == 0) {
                    rng = saved;  // take the exact path
                }
                __syncwarp();
            }
        } else {
            held_v = -1;  // the rounds of 32 read (and may rebuild) the records in HBM
            fast_done = partial_ref_fast<W>(g, s, rec, until, el, msk, f, t, asp, lane, rng, st, prof ? pc : nullptr);
        }
        if (!fast_done) held_v = -1;  // the serial walk reads the records in HBM
        if (prof) {
            const long long x = clock64();
            pc[2] += (unsigned long long)(x - tq);
            tq = x;
        }
        for (int c0 = 0; c0 < f && !fast_done; c0 += 32) {
            const int p = c0 + lane;
            if (p < f) {
                uint64_t x0[W], x1[W], x2[W];
                dense_masks<W>(g, s, rec, until, el[p], t, asp, x0, x1, x2);
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    msk[(lane * 3 + 0) * W + q] = x0[q];
                    msk[(lane * 3 + 1) * W + q] = x1[q];
                    msk[(lane * 3 + 2) * W + q] = x2[q];
                }
            }
            __syncwarp();
            if (prof) {
                const long long x = clock64();
                pc[1] += (unsigned long long)(x - tq);
                tq = x;
            }
            if (lane == 0) {
                const int m = min(32, f - c0);
                for (int q = 0; q < m; ++q)
                    ref_walk<W>(st, rng, msk + (q * 3 + 0) * W, msk + (q * 3 + 1) * W, msk + (q * 3 + 2) * W,
                                el[c0 + q], c0 + q);
            }
            __syncwarp();
            if (prof) {
                const long long x = clock64();
                pc[2] += (unsigned long long)(x - tq);
                tq = x;
            }
        }
        if (prof) pc[4] += st.found ? st.ties - 1 : 0;
        const int found = __shfl_sync(kFull, st.found, 0);
        const uint32_t ties = __shfl_sync(kFull, st.ties, 0);
        if (!found) {
            // every candidate tabu: tick only (partial.hpp:121-122)
            if (lane == 0) acc += 2ULL * (unsigned)w1 * (unsigned)f;
            if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                *(reinterpret_cast<plse_step*>(a.trace) + j) = plse_step{(int64_t)j, -1, 0, 0, -1, -1, f, f, bestf,
                                                                        -1, 0, 2};
            ++j;
            continue;
        }
        const int vs = __shfl_sync(kFull, st.cv, 0);
        const int ks = __shfl_sync(kFull, st.ck, 0);
        const int ps = __shfl_sync(kFull, st.cpos, 0);
        const int lvl = __shfl_sync(kFull, st.bd, 0);
        if (pending && lvl >= 0) {
            snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
            pending = false;
        }
        // ---- apply (partial.hpp:124-141): the row / column holder of k* are the neighbours coloured k*
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
        // displaced vertices join the IndexSet in CSR order: row-mates first iff row <= col (lsgraph.hpp:201-209)
        const bool row_first = rs_ <= cs_;
        const int ev0 = row_first ? (ur >= 0 ? ur : uc) : (uc >= 0 ? uc : ur);
        const int ev1 = e == 2 ? (row_first ? uc : ur) : -1;
        uint32_t tenure = 0;
        if (lane == 0) {
            tenure = (uint32_t)ref_below(rng, 10) + (uint32_t)(alpha * (double)f_new);
            const uint16_t last = el[f - 1];
            el[ps] = last;  // IndexSet::erase(v*)
            int sz = f - 1;
            if (ev0 >= 0) el[sz++] = (uint16_t)ev0;
            if (ev1 >= 0) el[sz++] = (uint16_t)ev1;
        }
        tenure = __shfl_sync(kFull, tenure, 0);
        const uint32_t ut = t + 1 + tenure;
        const bool improved = f_new < bestf;
        __syncwarp();
        const TabuRec evr = apply_move_lanes<W>(g, s, rec, until, vs, ur, uc, ks, rs_, cs_, inR, inC, f_before,
                                                improved, ut, t, lane, acc);
        {
            // the held records follow the IndexSet: position ps takes the last position's, the evictees'
            // (appended at f - 1, f) are the records the move just wrote (lanes 1 / 2)
            const int lv = __shfl_sync(kFull, held_v, f - 1);
            const uint32_t l1 = __shfl_sync(kFull, held.u1, f - 1), l2 = __shfl_sync(kFull, held.u2, f - 1);
            const uint32_t lk = __shfl_sync(kFull, held.kk, f - 1);
            const int src0 = ev0 == ur ? 1 : 2, src1 = ev1 == ur ? 1 : 2;
            const int srcl = lane == f - 1 ? src0 : src1;
            const uint32_t e1 = __shfl_sync(kFull, evr.u1, srcl), e2 = __shfl_sync(kFull, evr.u2, srcl);
            const uint32_t ek = __shfl_sync(kFull, evr.kk, srcl);
            if (lane == ps) {
                held_v = lv;
                held = TabuRec{l1, l2, lk, 0};
            }
            if ((lane == f - 1 && ev0 >= 0) || (lane == f && ev1 >= 0)) {
                held_v = lane == f - 1 ? ev0 : ev1;
                held = TabuRec{e1, e2, ek, 0};
            }
        }
        f = f_new;
        if (improved) {
            bestf = f;
            pending = true;
            if (race_flag && bestf <= a.race_f && lane == 0) atomicExch(const_cast<int*>(race_flag), 1);
        }
        if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
            *(reinterpret_cast<plse_step*>(a.trace) + j) =
                plse_step{(int64_t)j, vs, ks, e, ev0, ev1, f_before, f, bestf, (int)tenure, (int32_t)ties, lvl};
        __syncwarp();
        if (prof) pc[3] += (unsigned long long)(clock64() - tq);
        ++j;
    }
    if (pending) snapshot(col, a.improved + (size_t)i * g.nvpad, g.nvpad, lane);
    {
        const unsigned long long a1 = __shfl_sync(kFull, acc, 1), a2 = __shfl_sync(kFull, acc, 2);
        acc += a1 + a2;
    }
    if (lane == 0) {
        a.best_f[i] = bestf;
        a.repaired_f[i] = repaired_f;
        a.iters[i] = (int64_t)j;
        a.bytes[i] = acc;
        *slot_clock = base + j + 2 + a.tenure_cap;
        if (prof) {
#pragma unroll
            for (int z = 0; z < 11; ++z) atomicAdd(prof + z, pc[z]);
        }
    }
    __syncwarp();
}

template <int W, bool kDebug>
__global__ void __launch_bounds__(kImproveMaxThreads, 2) k_improve_ref(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, nv = a.nv;
    const ImproveSmemLayout G = improve_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    const RefSmemLayout L = improve_ref_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + G.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + G.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + G.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + G.cl);
    uint16_t* s_cp = reinterpret_cast<uint16_t*>(smem + G.colpos);
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + G.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + G.pc);
    uint8_t* s_deg = smem + G.deg;
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
    s.list = nullptr;
    s.R = reinterpret_cast<uint64_t*>(wbase + L.w_R);
    s.C = reinterpret_cast<uint64_t*>(wbase + L.w_C);
    s.U = reinterpret_cast<uint32_t*>(wbase + L.w_U);
    uint16_t* el = reinterpret_cast<uint16_t*>(wbase + L.w_el);
    uint64_t* msk = reinterpret_cast<uint64_t*>(wbase + L.w_msk);

    const int slot = blockIdx.x * nwarps + warp;
    TabuRec* rec = reinterpret_cast<TabuRec*>(reinterpret_cast<char*>(a.tabu_rec) + (size_t)slot * a.rec_stride);
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    uint8_t* conf = a.conf_scratch + (size_t)slot * a.conf_stride;
    for (int i = first_individual(a.first, a.nslots, a.p, warp); i < a.p;
         i = next_individual(a.first, a.nslots, a.work_counter, lane))
        improve_ref_one<W, kDebug>(a, g, s, el, msk, rec, until, a.slot_clock + slot, conf, i, lane);
}

const void* improve_ref_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_improve_ref<1, true>)
                             : reinterpret_cast<const void*>(&k_improve_ref<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_improve_ref<2, true>)
                 : reinterpret_cast<const void*>(&k_improve_ref<2, false>);
}

cudaError_t launch_improve_ref(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr || a.prof != nullptr;
    if (W == 1) {
        if (debug)
            k_improve_ref<1, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve_ref<1, false><<<grid, threads, smem, st>>>(a);
    } else {
        if (debug)
            k_improve_ref<2, true><<<grid, threads, smem, st>>>(a);
        else
            k_improve_ref<2, false><<<grid, threads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace plse_dev
