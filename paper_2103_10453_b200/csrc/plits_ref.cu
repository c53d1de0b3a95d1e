// plits_ref.cu -- PLITS with the REFERENCE's own tie-break (PLSE_TIE_REF) on sm_100a.
//
// Reproduces plits.hpp:96-292 bit for bit: the uncoloured and conflicting sets
// are kept as the reference's IndexSets (search_util.hpp:12-49: insert appends,
// erase moves the last element into the hole; membership re-decided in the
// order of plits.hpp:193-212, neighbours in CSR order), the candidates are
// visited uncoloured set first, then conflicting set, colours ascending (k = 0
// first for a conflicting vertex), and every tie with the running best draws
// next_below(++ties) from the individual's xoshiro256++ stream -- one stream
// over both phases, as in plits_run -- followed by next_below(10) for the
// tenure.  The warp computes the move classes of 32 vertices at a time from
// the bit-sliced colour counts (plits_common.cuh) into shared memory; lane 0
// walks them in order, reading until[][] only for colours in the vertex's
// possibly-tabu mask.  Everything else -- the phases and their weights, the
// fresh tabu table per phase, best tracking, the final repair, the byte model
// -- is the canonical kernel's (plits.cu).
#include "plits_common.cuh"
#include "ref_draws.cuh"

namespace plse_dev {

namespace {

constexpr uint16_t kNone = 0xFFFF;

struct PlitsRefWarp {
    uint8_t* col;
    uint64_t* rp;
    uint64_t* cp;
    uint16_t *un_el, *un_pos, *cf_el, *cf_pos;  // IndexSets (plits.hpp:74-75)
    uint64_t* T;                                // [nv][W] colours possibly tabu (GLOBAL, per warp slot)
    uint64_t* stage;                            // 32 staged vertices: S planes and candidate mask
    int32_t* stage_i;                           // 32 staged vertices: v, cur, dbase, d0
    uint16_t* evl;                              // neighbours whose membership is re-decided, CSR order
};

__device__ __forceinline__ void is_insert(uint16_t* el, uint16_t* pos, int& size, int x) {
    if (pos[x] != kNone) return;
    pos[x] = (uint16_t)size;
    el[size++] = (uint16_t)x;
}

__device__ __forceinline__ void is_erase(uint16_t* el, uint16_t* pos, int& size, int x) {
    const int p = pos[x];
    if (p == kNone) return;
    const int last = el[size - 1];
    el[p] = (uint16_t)last;
    pos[last] = (uint16_t)p;
    --size;
    pos[x] = kNone;
}

template <int W>
__device__ __forceinline__ int gamma_of(const Graph<W>& g, const PlitsRefWarp& s, int u, int k) {
    constexpr int NP = PlitsK<W>::NP;
    const uint16_t rc = g.cell[u];
    return plane_val<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k) + plane_val<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k);
}

// planes, f, c and the two IndexSets in ascending id order (plits.hpp:104-116)
template <int W>
__device__ void plits_ref_build(const Graph<W>& g, const PlitsRefWarp& s, int lane, int& f, int& c, int& nu, int& ncf) {
    const int nv = g.nv;
    plits_build_planes<W>(g, s, lane);
    for (int x = lane; x < nv; x += 32) {
        s.un_pos[x] = kNone;
        s.cf_pos[x] = kNone;
    }
    const int B = 32 * g.lane_words, v_lo = lane * B, v_hi = min(nv, v_lo + B);
    int cu = 0, cc = 0, cl2 = 0;
    for (int v = v_lo; v < v_hi; ++v) {
        const int k = s.col[v];
        if (!k) {
            ++cu;
        } else {
            const int gv = gamma_of<W>(g, s, v, k) - 2;
            cl2 += gv;
            cc += gv > 0;
        }
    }
    const int iu = warp_incl_sum(cu), ic = warp_incl_sum(cc);
    nu = __shfl_sync(kFull, iu, 31);
    ncf = __shfl_sync(kFull, ic, 31);
    int pu = iu - cu, pc = ic - cc;
    __syncwarp();
    for (int v = v_lo; v < v_hi; ++v) {
        const int k = s.col[v];
        if (!k) {
            s.un_el[pu] = (uint16_t)v;
            s.un_pos[v] = (uint16_t)pu++;
        } else if (gamma_of<W>(g, s, v, k) > 2) {
            s.cf_el[pc] = (uint16_t)v;
            s.cf_pos[v] = (uint16_t)pc++;
        }
    }
    f = nu;
    c = (int)__reduce_add_sync(kFull, (unsigned)cl2) / 2;
    __syncwarp();
}

struct RefChoice {
    int found, delta, v, k, dc, df;
    uint32_t ties;
};

// plits.hpp:135-176 consider() over one staged vertex, lane 0
template <int W>
__device__ __forceinline__ void ref_walk_vertex(RefChoice& ch, Xoshiro& rng, const uint64_t* S_, const uint64_t* M_,
                                                int v, int cur, int dbase, int d0, bool conflicting, int wf, int wc,
                                                const uint32_t* urow, uint64_t* Tv, uint32_t t, int64_t cur_scaled,
                                                int64_t best_scaled, unsigned long long* pc) {
    constexpr int NB = PlitsK<W>::NB;
    const int gcur = cur ? (wf - d0) / wc : 0;
    auto consider = [&](int k, int delta, int dc, int df) {
        if (ch.found && delta > ch.delta) return;
        if (pc) ++pc[6];
        const uint64_t bit = 1ULL << (k & 63);
        if (Tv[k >> 6] & bit) {
            if (pc) ++pc[7];
            if (urow[k] > t) {
                if (!(cur_scaled + delta < best_scaled)) return;  // tabu and not aspirating
            } else {
                Tv[k >> 6] &= ~bit;  // expired: the mask is a superset of the live entries
            }
        }
        if (!ch.found || delta < ch.delta) {
            ch.found = 1;
            ch.delta = delta;
            ch.ties = 1;
            ch.v = v;
            ch.k = k;
            ch.dc = dc;
            ch.df = df;
        } else if (ref_below_is_zero(rng, ++ch.ties)) {
            ch.v = v;
            ch.k = k;
            ch.dc = dc;
            ch.df = df;
        }
    };
    if (conflicting) consider(0, d0, -gcur, 1);  // k = 0 comes first in D(v)
    uint64_t S[NB][W];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < W; ++q) S[b][q] = S_[b * W + q];
    uint64_t rel[W];
#pragma unroll
    for (int q = 0; q < W; ++q) rel[q] = M_[q];
    if (ch.found) {  // only candidates with delta <= the running best can matter
        const int th = floor_div(ch.delta - dbase, wc);  // gamma <= th
        uint64_t above[W];
#pragma unroll
        for (int q = 0; q < W; ++q) above[q] = ~0ULL;
        sliced_ge<W, NB>(S, th + 1, above);
#pragma unroll
        for (int q = 0; q < W; ++q) rel[q] &= ~above[q];
    }
    for (int q = 0; q < W; ++q) {
        uint64_t x = word_of<W>(rel, q);
        while (x) {
            const int b = __ffsll((long long)x) - 1;
            x &= x - 1;
            const int k = q * 64 + b;
            const int gk = sliced_val<W, NB>(S, k);
            consider(k, dbase + wc * gk, gk - gcur, cur ? 0 : -1);
        }
    }
}

// ---- the same reservoir scan computed in parallel, 32 vertices of the sequence per round.
// Every quantity the serial walk branches on -- the candidate deltas, which candidates are tabu and not
// aspirating -- is fixed before the walk starts, so its history is determined by the deltas alone: the
// global minimum D, the prefix minimum of the per-vertex minima (where each vertex enters the walk), the
// ties at levels above D before the first D-candidate (E early draws, whose values are irrelevant), and
// the final segment -- every admissible candidate at D, the j-th of which (j >= 2) keeps the choice iff
// next_below(j) == 0.  Lane p owns vertex 32 c + p of round c; lane 0 only generates the stream, 32
// outputs at a time into shared memory, and the lanes test those draws.  A sequence of one round keeps
// its vertex in registers; longer ones recompute it per pass (minimum, counts, owner) -- the until[][]
// reads repeat only for the live entries of the possibly-tabu mask.  Any output below 2^32 (a possible
// rejection, probability 2^-32 per draw) falls back to the serial walk.

template <int W>
struct LaneView {
    VertexMoves<W> m;
    int v;
    uint64_t al[W];  // admissible colours k != 0
    bool a0;         // the move to 0 admissible (conflicting vertices only)
    int vmin;        // minimum delta over the admissible moves (INT_MAX: none)
};

template <int W>
__device__ __forceinline__ void view_min(LaneView<W>& x, int wc) {
    constexpr int NB = PlitsK<W>::NB;
    x.vmin = x.a0 ? x.m.d0 : INT_MAX;
    if (popc_w<W>(x.al)) {
        uint64_t sel[W];
#pragma unroll
        for (int q = 0; q < W; ++q) sel[q] = x.al[q];
        x.vmin = min(x.vmin, x.m.dbase + wc * sliced_min<W, NB>(x.m.S, sel));
    }
}

// the admissible moves of sequence position p (tabu moves are admissible iff delta < asp = best - cur);
// expired entries leave the possibly-tabu mask on the way
template <int W>
__device__ __forceinline__ void view_admissible(const Graph<W>& g, const PlitsRefWarp& s, int p, int nu, int wf,
                                                int wc, const uint32_t* until, int w1, uint32_t t, int asp,
                                                LaneView<W>& x) {
    constexpr int NB = PlitsK<W>::NB;
    const bool conflicting = p >= nu;
    x.v = conflicting ? s.cf_el[p - nu] : s.un_el[p];
    uint64_t* Tv = s.T + (size_t)x.v * W;
    uint64_t tv[W];  // global: issued ahead of the move classes so the load overlaps them
#pragma unroll
    for (int q = 0; q < W; ++q) tv[q] = Tv[q];
    vertex_moves<W>(g, s, x.v, wf, wc, x.m);
    uint64_t live[W];
#pragma unroll
    for (int q = 0; q < W; ++q) live[q] = 0;
    const uint32_t* urow = until + (size_t)x.v * w1;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t y = tv[q] & (x.m.M[q] | ((q == 0 && conflicting) ? 1ULL : 0ULL));
        uint64_t expired = 0;
        while (y) {
            const int b = __ffsll((long long)y) - 1;
            y &= y - 1;
            if (urow[q * 64 + b] > t)
                live[q] |= 1ULL << b;
            else
                expired |= 1ULL << b;
        }
        if (expired) Tv[q] = tv[q] & ~expired;  // the mask stays a superset of the live entries
    }
    x.a0 = conflicting && (!(live[0] & 1ULL) || x.m.d0 < asp);
    live[0] &= ~1ULL;
    // tabu colours admissible only with gamma <= floor((asp - 1 - dbase) / wc)
    uint64_t hi[W];
#pragma unroll
    for (int q = 0; q < W; ++q) hi[q] = live[q];
    sliced_ge<W, NB>(x.m.S, floor_div(asp - 1 - x.m.dbase, wc) + 1, hi);
#pragma unroll
    for (int q = 0; q < W; ++q) x.al[q] = x.m.M[q] & ~hi[q];
    view_min<W>(x, wc);
}

// early draws of one vertex: ties at levels above D, counted per level from the incoming running
// minimum rin -- a candidate at level L ties iff it precedes every candidate below L and the running
// minimum already is L (an earlier candidate at L, or the incoming one)
template <int W>
__device__ __forceinline__ int view_early(const LaneView<W>& x, int rin, int D, int wc) {
    constexpr int NB = PlitsK<W>::NB;
    constexpr int kInf = INT_MAX;
    int early = 0;
    int r = rin;
    uint64_t G[W];
#pragma unroll
    for (int q = 0; q < W; ++q) G[q] = x.al[q];
    if (x.a0) {  // k = 0 comes first
        if (x.m.d0 < r)
            r = x.m.d0;
        else if (x.m.d0 == r)
            ++early;
    }
    if (r == kInf && popc_w<W>(G)) {  // nothing before this vertex: its first colour resets
        const int k1 = first_bit_w<W>(G);
        r = x.m.dbase + wc * sliced_val<W, NB>(x.m.S, k1);
#pragma unroll
        for (int q = 0; q < W; ++q)
            if ((k1 >> 6) == q) G[q] &= ~(1ULL << (k1 & 63));
    }
    if (r == kInf || r <= D || !popc_w<W>(G)) return early;
    const int gr = floor_div(r - x.m.dbase, wc);
    {
        uint64_t hi[W];
#pragma unroll
        for (int q = 0; q < W; ++q) hi[q] = G[q];
        sliced_ge<W, NB>(x.m.S, gr + 1, hi);
#pragma unroll
        for (int q = 0; q < W; ++q) G[q] &= ~hi[q];
    }
    // the levels present, lowest first (each one's count only depends on the candidates below it)
    uint64_t lower[W];
#pragma unroll
    for (int q = 0; q < W; ++q) lower[q] = 0;
    while (popc_w<W>(G)) {
        uint64_t sel[W];
#pragma unroll
        for (int q = 0; q < W; ++q) sel[q] = G[q];
        const int L = x.m.dbase + wc * sliced_min<W, NB>(x.m.S, sel);  // sel: the candidates at L
        if (L > D) {
            const int cnt = popc_below_w<W>(sel, first_bit_w<W>(lower));
            early += (L == r) ? cnt : max(cnt - 1, 0);
        }
#pragma unroll
        for (int q = 0; q < W; ++q) {
            lower[q] |= sel[q];
            G[q] &= ~sel[q];
        }
    }
    return early;
}

// the vertex's members of the final segment: k = 0 first (z0), then the colours aD ascending
template <int W>
__device__ __forceinline__ int view_final(const LaneView<W>& x, int D, int wc, uint64_t (&aD)[W], bool& z0) {
    constexpr int NB = PlitsK<W>::NB;
#pragma unroll
    for (int q = 0; q < W; ++q) aD[q] = 0;
    z0 = false;
    if (x.vmin != D) return 0;
    z0 = x.a0 && x.m.d0 == D;
    const int num = D - x.m.dbase;
    if (num >= 0 && num % wc == 0) {
#pragma unroll
        for (int q = 0; q < W; ++q) aD[q] = x.al[q];
        sliced_eq<W, NB>(x.m.S, num / wc, aD);
    }
    return (int)z0 + popc_w<W>(aD);
}

template <int W>
__device__ __forceinline__ bool plits_ref_fast(const Graph<W>& g, const PlitsRefWarp& s, int lane, int nseq, int nu,
                                               int wf, int wc, uint32_t* until, int w1, uint32_t t,
                                               int64_t cur_scaled, int64_t best_scaled, Xoshiro& rng,
                                               RefChoice& ch, unsigned long long* tp) {
    constexpr int kInf = INT_MAX;
    long long t0 = tp ? clock64() : 0;
    auto stamp = [&](int z) {
        if (tp) {
            const long long x = clock64();
            tp[z] += (unsigned long long)(x - t0);
            t0 = x;
        }
    };
    const int nch = (nseq + 31) >> 5;
    uint64_t* out = s.stage;  // the inputs of 32 stream outputs at a time (ref_stream_draws)
    const int64_t asp64 = best_scaled - cur_scaled;
    const int asp = (int)max((int64_t)INT_MIN / 4, min((int64_t)INT_MAX / 4, asp64));
    auto empty = [](LaneView<W>& x) {
#pragma unroll
        for (int q = 0; q < W; ++q) x.al[q] = 0;
        x.a0 = false;
        x.vmin = kInf;
        x.v = 0;
        x.m.cur = x.m.dbase = x.m.d0 = 0;
    };
    auto view_of = [&](int c, LaneView<W>& x) {
        const int p = 32 * c + lane;
        if (p < nseq)
            view_admissible<W>(g, s, p, nu, wf, wc, until, w1, t, asp, x);
        else
            empty(x);
    };

    // ---- pass 1: admissible moves, their minimum
    LaneView<W> x;
    int D = kInf;
    for (int c = 0; c < nch; ++c) {
        view_of(c, x);
        D = min(D, __reduce_min_sync(kFull, x.vmin));
    }
    stamp(0);
    if (D == kInf) {  // every candidate tabu: nothing found, no draw
        ch.found = 0;
        return true;
    }
    // ---- pass 2: early draws up to the first D-candidate, the size of the final segment
    int E = 0, ND = 0, rcarry = kInf;
    bool seen = false;
    for (int c = 0; c < nch; ++c) {
        if (nch > 1) view_of(c, x);
        const int pm = warp_incl_min(x.vmin);  // inclusive prefix minimum of the per-vertex minima
        if (!seen) {
            int rin = __shfl_up_sync(kFull, pm, 1);
            if (lane == 0) rin = kInf;
            rin = min(rin, rcarry);
            const unsigned bal = __ballot_sync(kFull, x.vmin == D);
            const int istar = bal ? __ffs(bal) - 1 : 32;
            const int early = (32 * c + lane < nseq && lane <= istar) ? view_early<W>(x, rin, D, wc) : 0;
            E += (int)__reduce_add_sync(kFull, (unsigned)early);
            seen = bal != 0;
        }
        uint64_t aD[W];
        bool z0;
        ND += (int)__reduce_add_sync(kFull, (unsigned)view_final<W>(x, D, wc, aD, z0));
        rcarry = min(rcarry, __shfl_sync(kFull, pm, 31));
    }
    stamp(1);
    // member j (1-based, in walk order) of the final segment keeps the choice iff next_below(j) == 0
    // (j >= 2): draw E + j - 2 of the stream
    const Xoshiro before = rng;
    if (tp) tp[5] += (unsigned)(E + ND - 1);
    bool bad = false;  // an output below 2^32: a rejection is possible, take the exact path
    const int bestj = ref_stream_draws(rng, out, E, E + ND - 1, lane, bad);
    stamp(3);
    if (bad) {
        if (lane == 0) rng = before;
        return false;
    }
    int J = (int)__reduce_max_sync(kFull, (unsigned)bestj);
    if (J == 0) J = 1;
    // ---- pass 3: the owner of member J
    int based = 0;
    for (int c = 0; c < nch; ++c) {
        if (nch > 1) view_of(c, x);
        uint64_t aD[W];
        bool z0;
        const int cD = view_final<W>(x, D, wc, aD, z0);
        const int incl = warp_incl_sum(cD);
        const int tot = __shfl_sync(kFull, incl, 31);
        if (J > based + tot) {
            based += tot;
            continue;
        }
        const int sD = based + incl - cD;
        const bool own = sD < J && J <= sD + cD;
        int kk = 0, dc = 0, df = 0;
        if (own) {
            const int li = J - sD - 1;
            const int gcur = x.m.cur ? (wf - x.m.d0) / wc : 0;
            if (z0 && li == 0) {
                kk = 0;
                dc = -gcur;
                df = 1;
            } else {
                kk = nth_bit_w<W>(aD, li - (int)z0);
                dc = (D - x.m.dbase) / wc - gcur;
                df = x.m.cur ? 0 : -1;
            }
        }
        const int wl = __ffs(__ballot_sync(kFull, own)) - 1;
        ch.found = 1;
        ch.delta = D;
        ch.ties = (uint32_t)ND;
        ch.v = __shfl_sync(kFull, x.v, wl);
        ch.k = __shfl_sync(kFull, kk, wl);
        ch.dc = __shfl_sync(kFull, dc, wl);
        ch.df = __shfl_sync(kFull, df, wl);
        break;
    }
    __syncwarp();
    stamp(4);
    return true;
}

template <int W, bool kDebug>
__device__ void plits_ref_one(const ImproveArgs& a, const Graph<W>& g, const PlitsRefWarp& s, uint32_t* until,
                              uint32_t* slot_clock, int i, int lane) {
    constexpr int NP = PlitsK<W>::NP;
    constexpr int NB = PlitsK<W>::NB;
    const int nv = g.nv, w1 = g.n + 1;
    uint8_t* col = s.col;
    uint8_t* best_row = a.improved + (size_t)i * g.nvpad;
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
    unsigned long long* prof = kDebug ? a.prof : nullptr;
    unsigned long long pc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // steps, stage, walk, apply, sum nseq, walked vertices
    long long tq = 0;

    uint32_t base = *slot_clock;
    if ((uint64_t)base + (uint64_t)a.budget + (uint64_t)a.budget2 + 2ull * (a.tenure_cap + 4) >= 0xFFFFFFFFull) {
        uint4* u4 = reinterpret_cast<uint4*>(until);
        for (size_t x = lane; x < a.until_stride / 4; x += 32) u4[x] = make_uint4(0, 0, 0, 0);
        base = 0;
    }
    snapshot(a.offspring + (size_t)i * g.nvpad, col, g.nvpad, lane);
    __syncwarp();

    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    Xoshiro rng(seed);  // one stream for both phases (plits.hpp:276-292)
    const int stop_f = a.stop_f;
    const double alpha = a.alpha;
    const int* race_flag = a.race_flag;
    const unsigned long long* deadline = a.deadline;
    auto poll_stop = [race_flag, deadline](uint32_t jj) -> bool {
        if (race_flag && *reinterpret_cast<const volatile int*>(race_flag)) return true;
        if (!deadline || jj == 0 || (jj & 0xFFFu)) return false;
        return __shfl_sync(kFull, globaltimer_ns() >= *deadline ? 1 : 0, 0) != 0;
    };

    int f = 0, c = 0, nu = 0, ncf = 0;
    plits_ref_build<W>(g, s, lane, f, c, nu, ncf);
    const int initial_f = f;
    uint32_t J = 0;
    int64_t iters = 0;
    bool hit = false, pending = true;
    int best_f = f, best_c = c;
    unsigned long long acc = 0;

    for (int phase = 1; phase <= 2; ++phase) {
        const int wf = 2;
        const int wc = phase == 1 ? 1 : 2 * nv;
        const int64_t budget = phase == 1 ? a.budget : a.budget2;
        if (phase == 2) plits_ref_build<W>(g, s, lane, f, c, nu, ncf);  // PlitsScratch::prepare, plits.hpp:79-91
        for (int x = lane; x < nv * W; x += 32) s.T[x] = 0;            // fresh tabu table
        __syncwarp();
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
            const int nseq = nu + ncf;
            if (nseq == 0) break;  // StepResult::Exhausted: not counted
            if ((j & 63) == 0 && poll_stop(j)) break;
            const uint32_t t = base + j;
            const int64_t cur_scaled = (int64_t)wf * f + (int64_t)wc * c;
            const int active_before = nseq;

            // ---- the reservoir scan: uncoloured set, then conflicting set, in IndexSet order
            RefChoice ch{0, 0, -1, 0, 0, 0, 0};
            if (prof) {
                tq = clock64();
                ++pc[0];
                pc[4] += (unsigned)nseq;
            }
            bool fast_done = false;
            {
                fast_done = plits_ref_fast<W>(g, s, lane, nseq, nu, wf, wc, until, w1, t, cur_scaled, best_scaled,
                                              rng, ch, prof ? pc + 8 : nullptr);
                if (prof) {
                    const long long x = clock64();
                    pc[3] += (unsigned long long)(x - tq);
                    tq = x;
                }
            }
            for (int c0 = 0; c0 < nseq && !fast_done; c0 += 32) {
                const int p = c0 + lane;
                if (p < nseq) {
                    const int v = p < nu ? s.un_el[p] : s.cf_el[p - nu];
                    VertexMoves<W> m;
                    vertex_moves<W>(g, s, v, wf, wc, m);
                    uint64_t* st = s.stage + (size_t)lane * (NB + 1) * W;
#pragma unroll
                    for (int b = 0; b < NB; ++b)
#pragma unroll
                        for (int q = 0; q < W; ++q) st[b * W + q] = m.S[b][q];
#pragma unroll
                    for (int q = 0; q < W; ++q) st[NB * W + q] = m.M[q];
                    s.stage_i[lane * 5 + 0] = v;
                    s.stage_i[lane * 5 + 1] = m.cur;
                    s.stage_i[lane * 5 + 2] = m.dbase;
                    s.stage_i[lane * 5 + 3] = m.d0;
                    // tabu-blind minimum delta: a vertex whose every move is above the running best
                    // cannot win or draw, so lane 0 skips it
                    int vm = p >= nu ? m.d0 : INT_MAX;
                    uint64_t sel[W];
#pragma unroll
                    for (int q = 0; q < W; ++q) sel[q] = m.M[q];
                    if (popc_w<W>(sel)) vm = min(vm, m.dbase + wc * sliced_min<W, NB>(m.S, sel));
                    s.stage_i[lane * 5 + 4] = vm;
                }
                __syncwarp();
                if (prof) {
                    const long long x = clock64();
                    pc[1] += (unsigned long long)(x - tq);
                    tq = x;
                }
                if (lane == 0) {
                    const int mcount = min(32, nseq - c0);
                    for (int q = 0; q < mcount; ++q) {
                        if (ch.found && s.stage_i[q * 5 + 4] > ch.delta) continue;
                        if (prof) ++pc[5];
                        const int v = s.stage_i[q * 5 + 0];
                        const uint64_t* st = s.stage + (size_t)q * (NB + 1) * W;
                        ref_walk_vertex<W>(ch, rng, st, st + NB * W, v, s.stage_i[q * 5 + 1], s.stage_i[q * 5 + 2],
                                           s.stage_i[q * 5 + 3], c0 + q >= nu, wf, wc, until + (size_t)v * w1,
                                           s.T + (size_t)v * W, t, cur_scaled, best_scaled, prof ? pc : nullptr);
                    }
                }
                __syncwarp();
                if (prof) {
                    const long long x = clock64();
                    pc[2] += (unsigned long long)(x - tq);
                    tq = x;
                }
            }
            const int found = __shfl_sync(kFull, ch.found, 0);
            if (!found) {
                // every candidate tabu: the clock still advances (plits.hpp:178-179)
                if (lane == 0) acc += 2ULL * (unsigned)w1 * (unsigned)active_before;
                if (tracing && lane == 0 && (int64_t)J < a.trace_cap)
                    *(reinterpret_cast<plse_step*>(a.trace) + J) =
                        plse_step{(int64_t)J, -1, 0, phase, 0, nseq, f, c, (int32_t)best_scaled, -1, 0, 0};
                ++j;
                ++J;
                continue;
            }
            const int vs = __shfl_sync(kFull, ch.v, 0);
            const int ks = __shfl_sync(kFull, ch.k, 0);
            const int dl = __shfl_sync(kFull, ch.delta, 0);
            const int dcs = __shfl_sync(kFull, ch.dc, 0);
            const int dfs = __shfl_sync(kFull, ch.df, 0);
            const uint32_t ties = __shfl_sync(kFull, ch.ties, 0);
            const int from = col[vs];
            const int64_t now = cur_scaled + dl;
            if (now >= best_scaled && pending) {
                snapshot(col, best_row, g.nvpad, lane);
                pending = false;
            }
            __syncwarp();
            const uint16_t rcs = g.cell[vs];
            const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
            if (lane == 0) {
                col[vs] = (uint8_t)ks;
                plane_move<W, NP>(s.rp + (size_t)rs_ * NP * W, from, ks);
            }
            if (lane == 1) plane_move<W, NP>(s.cp + (size_t)cs_ * NP * W, from, ks);
            __syncwarp();
            // ---- membership (plits.hpp:193-212): neighbours coloured `from` or `to`, CSR order
            int nev = 0;
            {
                const bool row_first = rs_ <= cs_;
                const int nr = g.rs[rs_ + 1] - g.rs[rs_], ncol = g.cs[cs_ + 1] - g.cs[cs_];
                const int tot = nr + ncol;
                for (int x0 = 0; x0 < tot; x0 += 32) {
                    const int x = x0 + lane;
                    int u = -1;
                    if (x < tot) {
                        const bool first = x < (row_first ? nr : ncol);
                        const int xx = first ? x : x - (row_first ? nr : ncol);
                        const bool in_row = first == row_first;
                        u = in_row ? g.rs[rs_] + xx : g.cl[g.cs[cs_] + xx];
                    }
                    const int cu = u >= 0 ? col[u] : 0;
                    const bool take = u >= 0 && u != vs && cu != 0 && (cu == from || cu == ks);
                    const unsigned bal = __ballot_sync(kFull, take);
                    if (take) s.evl[nev + __popc(bal & ((1u << lane) - 1))] = (uint16_t)u;
                    nev += __popc(bal);
                }
            }
            __syncwarp();
            uint32_t tenure = 0;
            if (lane == 0) {
                if (from == 0) is_erase(s.un_el, s.un_pos, nu, vs);
                if (ks == 0) {
                    is_insert(s.un_el, s.un_pos, nu, vs);
                    is_erase(s.cf_el, s.cf_pos, ncf, vs);
                } else if (gamma_of<W>(g, s, vs, ks) > 2) {
                    is_insert(s.cf_el, s.cf_pos, ncf, vs);
                } else {
                    is_erase(s.cf_el, s.cf_pos, ncf, vs);
                }
                for (int e = 0; e < nev; ++e) {
                    const int u = s.evl[e];
                    if (gamma_of<W>(g, s, u, col[u]) > 2)
                        is_insert(s.cf_el, s.cf_pos, ncf, u);
                    else
                        is_erase(s.cf_el, s.cf_pos, ncf, u);
                }
                tenure = (uint32_t)ref_below(rng, 10) + (uint32_t)(alpha * (double)(nu + ncf));
                until[(size_t)vs * w1 + from] = t + 1 + tenure;
                s.T[(size_t)vs * W + (from >> 6)] |= 1ULL << (from & 63);
                acc += 2ULL * (unsigned)w1 * (unsigned)active_before + 4ULL * g.deg[vs] + 2ULL;
            }
            nu = __shfl_sync(kFull, nu, 0);
            ncf = __shfl_sync(kFull, ncf, 0);
            tenure = __shfl_sync(kFull, tenure, 0);
            f += dfs;
            c += dcs;
            if (now < best_scaled) {
                best_scaled = now;
                best_f = f;
                best_c = c;
                pending = true;
                if (lane == 0) acc += 2ULL * (unsigned)nv;
                if (race_flag && best_c == 0 && best_f <= a.race_f && lane == 0)
                    atomicExch(const_cast<int*>(race_flag), 1);
            }
            if (tracing && lane == 0 && (int64_t)J < a.trace_cap)
                *(reinterpret_cast<plse_step*>(a.trace) + J) = plse_step{
                    (int64_t)J, vs, ks, phase, from, nu + ncf, f, c, (int32_t)best_scaled, (int32_t)tenure,
                    (int32_t)ties, dl};
            __syncwarp();

            ++j;
            ++J;
        }
        if (best_c == 0 && best_f <= stop_f) hit = true;
        iters += j;
        if (!pending) {
            snapshot(best_row, col, g.nvpad, lane);
            __syncwarp();
            pending = true;
        }
        base += j + 2 + a.tenure_cap;
        if (hit) break;
    }

    // ---- final greedy repair (plits.hpp:289, partial.hpp:22-39): argmax gamma[v][col v], lowest id
    if (best_c > 0) {
        plits_ref_build<W>(g, s, lane, f, c, nu, ncf);
        for (;;) {
            int bc = 0, bv = nv;
            for (int x = lane; x < ncf; x += 32) {
                const int v = s.cf_el[x];
                const int gv = gamma_of<W>(g, s, v, col[v]) - 2;
                if (gv > bc || (gv == bc && gv > 0 && v < bv)) {
                    bc = gv;
                    bv = v;
                }
            }
            const int mx = (int)__reduce_max_sync(kFull, (unsigned)bc);
            if (mx == 0) break;
            const int w = (int)__reduce_min_sync(kFull, (unsigned)(bc == mx ? bv : nv));
            const int k = col[w];
            const uint16_t rc = g.cell[w];
            __syncwarp();
            if (lane == 0) {
                col[w] = 0;
                plane_move<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k, 0);
            }
            if (lane == 1) plane_move<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k, 0);
            __syncwarp();
            // re-decide the conflicting set around w (order is irrelevant to the argmax)
            if (lane == 0) {
                is_erase(s.cf_el, s.cf_pos, ncf, w);
                const int r = rc >> 8, cc = rc & 0xFF;
                for (int u = g.rs[r]; u < g.rs[r + 1]; ++u)
                    if (col[u] == k && gamma_of<W>(g, s, u, k) <= 2) is_erase(s.cf_el, s.cf_pos, ncf, u);
                for (int x = g.cs[cc]; x < g.cs[cc + 1]; ++x) {
                    const int u = g.cl[x];
                    if (col[u] == k && gamma_of<W>(g, s, u, k) <= 2) is_erase(s.cf_el, s.cf_pos, ncf, u);
                }
            }
            ncf = __shfl_sync(kFull, ncf, 0);
            ++f;
            __syncwarp();
        }
        best_f = f;
        if (lane == 0) acc += 2ULL * (unsigned)nv;
    }
    snapshot(col, best_row, g.nvpad, lane);
    if (lane == 0) {
        a.best_f[i] = best_f;
        a.repaired_f[i] = initial_f;
        a.iters[i] = iters;
        a.bytes[i] = acc;
        *slot_clock = base;
        if (race_flag && best_f <= a.race_f) atomicExch(const_cast<int*>(race_flag), 1);
        if (prof) {
#pragma unroll
            for (int z = 0; z < 16; ++z) atomicAdd(prof + z, pc[z]);
        }
    }
    __syncwarp();
}

}  // namespace

template <int W, bool kDebug>
__global__ void __launch_bounds__(kPlitsMaxThreads, 1) k_plits_ref(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, nv = a.nv;
    const ImproveSmemLayout G = improve_smem_layout(n, nv, a.nvpad, a.lane_words, W);
    const PlitsRefSmemLayout L = plits_ref_smem_layout(n, nv, a.nvpad, a.lane_words, W);
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
    PlitsRefWarp s;
    s.col = wbase + L.w_col;
    s.rp = reinterpret_cast<uint64_t*>(wbase + L.w_rp);
    s.cp = reinterpret_cast<uint64_t*>(wbase + L.w_cp);
    s.un_el = reinterpret_cast<uint16_t*>(wbase + L.w_un_el);
    s.un_pos = reinterpret_cast<uint16_t*>(wbase + L.w_un_pos);
    s.cf_el = reinterpret_cast<uint16_t*>(wbase + L.w_cf_el);
    s.cf_pos = reinterpret_cast<uint16_t*>(wbase + L.w_cf_pos);
    s.stage = reinterpret_cast<uint64_t*>(wbase + L.w_stage);
    s.stage_i = reinterpret_cast<int32_t*>(wbase + L.w_stage_i);
    s.evl = reinterpret_cast<uint16_t*>(wbase + L.w_evl);

    const int slot = blockIdx.x * nwarps + warp;
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    // the possibly-tabu mask lives in the slot's tabu-record area in global memory (nv * 16 >= nv * 8 W
    // bytes): shared memory stays for the colouring, the count planes and the IndexSets, which doubles
    // the resident warps
    s.T = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(a.tabu_rec) + (size_t)slot * a.rec_stride);
    for (int i = first_individual(a.first, a.nslots, a.p, warp); i < a.p;
         i = next_individual(a.first, a.nslots, a.work_counter, lane))
        plits_ref_one<W, kDebug>(a, g, s, until, a.slot_clock + slot, i, lane);
}

const void* plits_ref_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_plits_ref<1, true>)
                             : reinterpret_cast<const void*>(&k_plits_ref<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_plits_ref<2, true>)
                 : reinterpret_cast<const void*>(&k_plits_ref<2, false>);
}

cudaError_t launch_plits_ref(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr || a.prof != nullptr;
    if (W == 1) {
        if (debug)
            k_plits_ref<1, true><<<grid, threads, smem, st>>>(a);
        else
            k_plits_ref<1, false><<<grid, threads, smem, st>>>(a);
    } else {
        if (debug)
            k_plits_ref<2, true><<<grid, threads, smem, st>>>(a);
        else
            k_plits_ref<2, false><<<grid, threads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace plse_dev
