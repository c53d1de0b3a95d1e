// plits.cu -- the MPMA variant's improve operator: PLITS, the two-phase
// partial legal and illegal tabu search (plits.hpp:96-292), on sm_100a.
//
// Replaces engine.hpp:193-197 (plits_run per individual) with ONE WARP PER
// INDIVIDUAL, persistent over a work counter, like the PartialCol kernel
// (improve.cu).  Data layout:
//   * colours (u8) in shared memory.  gamma is never materialised: for a
//     vertex v in row r / column c and any colour k != col(v)
//       gamma[v][k] = cnt_row[r][k] + cnt_col[c][k]
//     and gamma[v][col v] is the same sum minus 2.  The colour counts are kept
//     BIT-SLICED: plane b of row r is the W-word mask of colours whose count
//     has bit b set (NP = 5 + W planes, counts <= n).  One ripple-carry add of
//     the row and column planes gives gamma for all colours of v at once, and
//     a bit-sliced minimum over the candidate mask gives v's best move class
//     and its multiplicity -- about 80 word ops per vertex instead of a loop
//     over its domain.
//   * the neighbourhood N0 u Nc (plits.hpp:47-63) is an active-vertex bitmask:
//     v is active iff col(v) = 0 or col(v) occurs twice in its row or column.
//     Every step compacts it into an ascending id list dealt round-robin to
//     the lanes, so the scan is balanced however the active set clusters.
//   * tabu: the reference's dense until[v][k] (search_util.hpp:54-81) per warp
//     slot in HBM on the slot's monotone clock; a phase switch (fresh table,
//     plits.hpp:81) advances the clock past every live entry.  The step finds
//     the lowest delta LEVEL with an admissible candidate: the level minimum
//     is computed tabu-blind from shared memory, then only the candidates AT
//     that level read until[][] (batched, independent loads); when all of them
//     are tabu and not aspirating (plits.hpp:147) the next level is tried.
//   * objective: the integer 2F = wf*f + wc*c (plits.hpp:22-36), (2, 1) in
//     phase 1 and (2, 2|V|) in phase 2; aspiration against the phase best.
//   * selection: the canonical order-free rule: N
//     admissible candidates at the level, r = floor(h1 * N / 2^32) from the
//     counter hash keyed by (stream seed, step over both phases), the r-th in
//     ascending (v, k) order with k = 0 first; tenure floor(h2 * 10 / 2^32) +
//     floor(alpha * active) (plits.hpp:182-185).
//   * best tracking: deferred snapshot into the improved row (written only
//     before a move that does not improve on the phase best).
#include "plits_common.cuh"

namespace plse_dev {

struct PlitsWarp {
    uint8_t* col;     // [nvpad]
    uint64_t* rp;     // [n][NP][W] row colour-count planes
    uint64_t* cp;     // [n][NP][W] column colour-count planes
    uint32_t* A;      // [32 * lane_words] active vertices; word v >> 5 (lane-owned blocks)
    uint16_t* list;   // [nv] the step's active ids (ascending); after the selection: scratch for the
                      //      cells whose cached minimum is refreshed
    int32_t* vmin;    // [nv] per active vertex: tabu-blind minimum delta of its moves (refreshed when its
                      //      row or column changes)
    uint8_t* vcnt;    // [nv] per active vertex at the step's level: its admissible moves
    uint64_t* T;      // [nv][W + 1] GLOBAL (the slot's tabu-record area, L1-resident for a lone warp): W words
                      //         of colours possibly tabu -- a superset of the live until[][] entries, so only
                      //         those colours read until[][] -- and the largest until ever written for v
                      //         (low half of word W)
    uint8_t* X;       // [2n][n+1] register mode only, over list / vmin / vcnt (which only the bitmask mode
                      //         uses): per row and colour the XOR of the row offsets (u - rs[r]) of its cells
                      //         holding that colour, per column the XOR of their row indices -- the one cell
                      //         when the count is 1
};

// tabu-blind minimum delta over v's candidates (plits.hpp:135-176 without the tabu test)
template <int W>
__device__ __forceinline__ int vertex_min(const Graph<W>& g, const PlitsWarp& s, int v, int wf, int wc) {
    constexpr int NB = PlitsK<W>::NB;
    VertexMoves<W> m;
    vertex_moves<W>(g, s, v, wf, wc, m);
    int vm = m.cur ? m.d0 : INT_MAX;
    if (popc_w<W>(m.M)) vm = min(vm, m.dbase + wc * sliced_min<W, NB>(m.S, m.M));
    return vm;
}

// after a move of colour `from` -> `to` in row r / column c: re-classify those cells
// (plits.hpp:193-212) and refresh the cached minimum of each active one whose moves could have
// changed: it was inactive, or its own colour or a colour of its domain is `from` or `to` (only the
// counts of those two colours changed, and only in its row or column).  Nothing else moved.
template <int W>
__device__ __forceinline__ void plits_membership(const Graph<W>& g, const PlitsWarp& s, int r, int c, int from, int to,
                                                 int wf, int wc, int lane) {
    const int nr = g.rs[r + 1] - g.rs[r];
    const int tot = nr + g.cs[c + 1] - g.cs[c];
    uint64_t ft[W];
#pragma unroll
    for (int q = 0; q < W; ++q)
        ft[q] = ((from >> 6) == q && from ? 1ULL << (from & 63) : 0ULL) | ((to >> 6) == q && to ? 1ULL << (to & 63) : 0ULL);
    // classify every cell, collect the ones whose cached minimum must be refreshed ...
    int nredo = 0;
    for (int x0 = 0; x0 < tot; x0 += 32) {
        const int x = x0 + lane;
        bool need = false;
        int u = -1;
        if (x < tot) {
            u = x < nr ? g.rs[r] + x : g.cl[g.cs[c] + x - nr];
            const uint32_t bit = 1u << (u & 31);
            if (plits_is_active<W>(g, s, u)) {
                const bool was = (s.A[u >> 5] & bit) != 0;
                const int cu = s.col[u];
                need = !was || (cu && (cu == from || cu == to));
                if (!need) {
                    const uint16_t rc = g.cell[u];
                    uint64_t d[W];
                    dom_mask<W>(g, rc >> 8, rc & 0xFF, d);
#pragma unroll
                    for (int q = 0; q < W; ++q) need |= (d[q] & ft[q]) != 0;
                }
                if (!was) atomicOr(&s.A[u >> 5], bit);
            } else {
                atomicAnd(&s.A[u >> 5], ~bit);
            }
        }
        const unsigned bal = __ballot_sync(kFull, need);
        if (need) s.list[nredo + __popc(bal & ((1u << lane) - 1))] = (uint16_t)u;
        nredo += __popc(bal);
    }
    __syncwarp();
    // ... and refresh them in one round (the moved vertex may appear twice: same value)
    for (int x = lane; x < nredo; x += 32) {
        const int u = s.list[x];
        s.vmin[u] = vertex_min<W>(g, s, u, wf, wc);
    }
}

// count planes, active set, f and c of the colouring in s.col (plits.hpp:104-116, coloring.hpp:59-73)
template <int W>
__device__ void plits_build(const Graph<W>& g, const PlitsWarp& s, int lane, int wf, int wc, int& f, int& c,
                            int& active) {
    constexpr int NP = PlitsK<W>::NP;
    const int nv = g.nv;
    plits_build_planes<W>(g, s, lane);
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
                const int gv = plane_val<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k) +
                               plane_val<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k) - 2;
                cl2 += gv;
                if (gv) bits |= 1u << b;
            }
        }
        s.A[lane * g.lane_words + q] = bits;
        al += __popc(bits);
        while (bits) {
            const int v = v_lo + 32 * q + __ffs(bits) - 1;
            bits &= bits - 1;
            s.vmin[v] = vertex_min<W>(g, s, v, wf, wc);
        }
    }
    f = (int)__reduce_add_sync(kFull, (unsigned)fl);
    c = (int)__reduce_add_sync(kFull, (unsigned)cl2) / 2;
    active = (int)__reduce_add_sync(kFull, (unsigned)al);
    __syncwarp();
}

// x / wc with the phase-1 weight wc = 1 kept off the integer-division path
__device__ __forceinline__ int div_wc(int x, int wc) { return wc == 1 ? x : x / wc; }

// the xor tables of the colouring in s.col (register mode): lane l builds lines l, l + 32, ... (rows, then
// columns)
template <int W>
__device__ void plits_build_xor(const Graph<W>& g, const PlitsWarp& s, int lane) {
    const int n = g.n, w1 = n + 1;
    for (int line = lane; line < 2 * n; line += 32) {
        const bool is_row = line < n;
        const int idx = is_row ? line : line - n;
        uint8_t* X = s.X + (size_t)line * w1;
        for (int k = 0; k <= n; ++k) X[k] = 0;
        const int lo = is_row ? g.rs[idx] : g.cs[idx], hi = is_row ? g.rs[idx + 1] : g.cs[idx + 1];
        for (int x = lo; x < hi; ++x) {
            const int u = is_row ? x : g.cl[x];
            const int k = s.col[u];
            if (k) X[k] ^= (uint8_t)(is_row ? x - lo : g.cell[u] >> 8);
        }
    }
    __syncwarp();
}

// plane_move that also returns the line's counts of `from` and `to` after the move (0 for colour 0)
template <int W, int NP>
__device__ __forceinline__ void plane_move_count(uint64_t* P, int from, int to, int& cf, int& ct) {
    cf = 0;
    ct = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const bool hf = from && (from >> 6) == q, ht = to && (to >> 6) == q;
        if (!hf && !ht) continue;
        uint64_t borrow = hf ? 1ULL << (from & 63) : 0ULL;
        uint64_t carry = ht ? 1ULL << (to & 63) : 0ULL;
#pragma unroll
        for (int b = 0; b < NP; ++b) {
            const uint64_t old = P[b * W + q];
            const uint64_t mid = old ^ borrow;
            borrow &= ~old;
            const uint64_t x = mid ^ carry;
            carry &= mid;
            P[b * W + q] = x;
            if (hf) cf |= (int)((x >> (from & 63)) & 1ULL) << b;
            if (ht) ct |= (int)((x >> (to & 63)) & 1ULL) << b;
        }
    }
}

// the admissible moves of one vertex at delta level dl (plits.hpp:146-147): adm = colours k != 0,
// adm0 = the move to 0.  Only colours in the possibly-tabu mask tv (loaded by the caller ahead of the
// move classes so the load overlaps them) read until[][] (independent pairs of loads); expired ones
// leave tv (tv_changed tells the caller to store it back).
// v's moves at delta level dl, tabu-blind: adm = colours k != 0, adm0 = the move to 0
template <int W>
__device__ __forceinline__ void level_class(const VertexMoves<W>& m, int dl, int wc, uint64_t (&adm)[W], bool& adm0) {
    constexpr int NB = PlitsK<W>::NB;
    const int qv = dl - m.dbase;
#pragma unroll
    for (int q = 0; q < W; ++q) adm[q] = m.M[q];
    if (qv < 0 || (wc != 1 && qv % wc)) {
#pragma unroll
        for (int q = 0; q < W; ++q) adm[q] = 0;
    } else {
        sliced_eq<W, NB>(m.S, div_wc(qv, wc), adm);
    }
    adm0 = m.cur && m.d0 == dl;
}

template <int W>
__device__ __forceinline__ int level_adm(const VertexMoves<W>& m, int dl, int wc, bool asp_all, const uint32_t* urow,
                                         uint64_t (&tv)[W], uint32_t t, uint64_t (&adm)[W], bool& adm0,
                                         bool& tv_changed) {
    tv_changed = false;
    level_class<W>(m, dl, wc, adm, adm0);
    if (!asp_all && (adm0 || popc_w<W>(adm))) {
#pragma unroll
        for (int q = 0; q < W; ++q) {
            uint64_t x = adm[q] & tv[q];
            if (q == 0 && adm0) x |= tv[0] & 1ULL;
            uint64_t expired = 0;
            while (x) {
                int ks[2];
                uint32_t us[2];
#pragma unroll
                for (int z = 0; z < 2; ++z) {
                    ks[z] = x ? __ffsll((long long)x) - 1 : -1;
                    x &= x - 1;
                }
#pragma unroll
                for (int z = 0; z < 2; ++z) us[z] = ks[z] >= 0 ? urow[q * 64 + ks[z]] : 0u;
#pragma unroll
                for (int z = 0; z < 2; ++z) {
                    if (ks[z] < 0) continue;
                    if (us[z] > t) {
                        if (q == 0 && ks[z] == 0)
                            adm0 = false;
                        else
                            adm[q] &= ~(1ULL << ks[z]);
                    } else {
                        expired |= 1ULL << ks[z];
                    }
                }
            }
            if (expired) {
                tv[q] &= ~expired;
                tv_changed = true;
            }
        }
    }
    return popc_w<W>(adm) + (adm0 ? 1 : 0);
}

// ---- register-resident mode: while |active| <= 32 lane L holds the L-th active vertex (ascending id)
// with its move classes, tabu-blind minimum and tabu entries in registers, and a move updates the list
// in place: only the cells of the moved vertex's row and column whose colour is the old or the new one
// can change membership (their counts are the only ones that moved), so no re-classification scan and
// no compaction run per step.  The shared-memory active bitmask and minima are not maintained in this
// mode (their space holds the xor tables); they are rebuilt from the list when the set outgrows a warp.
constexpr int kNoV = 0xFFFF;        // an empty lane: sorts after every vertex id
constexpr int kListHysteresis = 4;  // enter at <= cap - 4 active vertices, leave above cap
// the list capacity: 32 (one vertex per lane); the instrumented kernel takes a smaller one from
// PLSE_PLITS_CAP so that tests drive the mode transitions often
__device__ int g_plits_list_cap = 32;

template <int W>
struct LaneVertex {
    int v, rc;  // vertex (kNoV: empty lane), its cell row << 8 | column
    VertexMoves<W> m;
    int vmin;  // tabu-blind minimum delta over v's moves
    // v's live tabu entries: exactly {k1 if u1 > t, k2 if u2 > t} (tk = k1 | k2 << 8), or, with the
    // overflow flag (tk bit 16), a superset tv read through until[][]; umax bounds every until of v
    uint32_t u1, u2, tk, umax;
    uint64_t tv[W];
};
constexpr uint32_t kTabuOvf = 1u << 16;

// level_adm on the lane's cached tabu entries (no memory access)
template <int W>
__device__ __forceinline__ int level_adm_cached(const LaneVertex<W>& L, int dl, int wc, bool asp_all, uint32_t t,
                                                uint64_t (&adm)[W], bool& adm0) {
    level_class<W>(L.m, dl, wc, adm, adm0);
    if (!asp_all) {
#pragma unroll
        for (int z = 0; z < 2; ++z) {
            const int k = z ? (L.tk >> 8) & 0xFF : L.tk & 0xFF;
            const bool live = (z ? L.u2 : L.u1) > t;
            if (live && k == 0) adm0 = false;
            // a select per word (a conditional update per word would be folded into adm[k >> 6], which
            // puts the array in local memory for W = 2)
            const uint64_t clear = (live && k) ? 1ULL << (k & 63) : 0ULL;
#pragma unroll
            for (int q = 0; q < W; ++q) adm[q] &= ((k >> 6) == q) ? ~clear : ~0ULL;
        }
    }
    return popc_w<W>(adm) + (adm0 ? 1 : 0);
}

// the lane's vertex got the tabu entry (k, un) (until[v][k] = un overwrites any earlier entry)
template <int W>
__device__ __forceinline__ void lane_tabu_write(LaneVertex<W>& L, int k, uint32_t un, uint32_t t) {
    L.umax = max(L.umax, un);
    if (L.tk & kTabuOvf) {
#pragma unroll
        for (int q = 0; q < W; ++q)
            if ((k >> 6) == q) L.tv[q] |= 1ULL << (k & 63);
        return;
    }
    const int k1 = L.tk & 0xFF, k2 = (L.tk >> 8) & 0xFF;
    if (k1 == k) {
        L.u1 = un;
    } else if (k2 == k) {
        L.u2 = un;
    } else if (L.u1 <= t) {
        L.tk = (L.tk & ~0xFFu) | (uint32_t)k;
        L.u1 = un;
    } else if (L.u2 <= t) {
        L.tk = (L.tk & ~0xFF00u) | (uint32_t)k << 8;
        L.u2 = un;
    } else {
        // three live entries: the superset {k1, k2, k} is read through until[][] from now on
#pragma unroll
        for (int q = 0; q < W; ++q) {
            uint64_t m = 0;
            if ((k1 >> 6) == q) m |= 1ULL << (k1 & 63);
            if ((k2 >> 6) == q) m |= 1ULL << (k2 & 63);
            if ((k >> 6) == q) m |= 1ULL << (k & 63);
            L.tv[q] = m;
        }
        L.tk |= kTabuOvf;
    }
}

// a vertex entering the list starts in overflow mode on its stored possibly-tabu mask and until bound
// (loaded here, first used at the next step: the bound usually shows that nothing is live any more)
template <int W>
__device__ __forceinline__ void lane_tabu_load(const PlitsWarp& s, LaneVertex<W>& L, int u) {
    const uint64_t* rec = s.T + (size_t)u * (W + 1);
#pragma unroll
    for (int q = 0; q < W; ++q) L.tv[q] = rec[q];
    L.umax = (uint32_t)rec[W];
    L.tk = kTabuOvf;
    L.u1 = 0;
    L.u2 = 0;
}

template <int W>
__device__ __forceinline__ int moves_min(const VertexMoves<W>& m, int wc) {
    constexpr int NB = PlitsK<W>::NB;
    int vm = m.cur ? m.d0 : INT_MAX;
    if (popc_w<W>(m.M)) {
        uint64_t sel[W];
#pragma unroll
        for (int q = 0; q < W; ++q) sel[q] = m.M[q];
        vm = min(vm, m.dbase + wc * sliced_min<W, NB>(m.S, sel));
    }
    return vm;
}

// the lane's move classes and minimum from the planes (L.v and L.rc set)
template <int W>
__device__ __forceinline__ void lane_load(const Graph<W>& g, const PlitsWarp& s, LaneVertex<W>& L, int wf, int wc) {
    if (L.v == kNoV) {
        L.rc = 0xFFFF;  // no row or column n <= 127 matches 0xFF
        L.m.cur = 0;
#pragma unroll
        for (int q = 0; q < W; ++q) L.m.M[q] = 0;
        L.vmin = INT_MAX;
        return;
    }
    vertex_moves_rc<W>(g, s, L.v, L.rc, wf, wc, L.m);
    L.vmin = moves_min<W>(L.m, wc);
}

// enter the register mode from the bitmask s.A (|active| = na <= 32)
template <int W>
__device__ __forceinline__ void sparse_enter(const Graph<W>& g, const PlitsWarp& s, LaneVertex<W>& L, int wf, int wc,
                                             int lane) {
    const int v_lo = lane * 32 * g.lane_words;
    int my = 0;
    for (int q = 0; q < g.lane_words; ++q) my += __popc(s.A[lane * g.lane_words + q]);
    int pos = warp_incl_sum(my) - my;
    for (int q = 0; q < g.lane_words; ++q) {
        uint32_t bits = s.A[lane * g.lane_words + q];
        while (bits) {
            s.list[pos++] = (uint16_t)(v_lo + 32 * q + __ffs(bits) - 1);
            bits &= bits - 1;
        }
    }
    const int na = __shfl_sync(kFull, pos, 31);
    __syncwarp();
    L.v = lane < na ? s.list[lane] : kNoV;
    __syncwarp();
    plits_build_xor<W>(g, s, lane);  // over the list
    if (L.v != kNoV) {
        L.rc = g.cell[L.v];
        lane_tabu_load<W>(s, L, L.v);
    } else {
        L.tk = 0;
        L.u1 = L.u2 = L.umax = 0;
    }
    lane_load<W>(g, s, L, wf, wc);
    __syncwarp();
}

// leave it: the bitmask and the cached minima of every member (the list plus up to two vertices that
// did not fit), from the planes as they are after the move
template <int W>
__device__ __forceinline__ void sparse_leave(const Graph<W>& g, const PlitsWarp& s, int lv, int lvmin, int x1, int x2,
                                             int wf, int wc, int lane) {
    for (int q = lane; q < 32 * g.lane_words; q += 32) s.A[q] = 0;
    __syncwarp();
    if (lv != kNoV) {
        atomicOr(&s.A[lv >> 5], 1u << (lv & 31));
        s.vmin[lv] = lvmin;
    }
    const int x = lane == 0 ? x1 : lane == 1 ? x2 : -1;
    if (x >= 0) {
        atomicOr(&s.A[x >> 5], 1u << (x & 31));
        s.vmin[x] = vertex_min<W>(g, s, x, wf, wc);
    }
    __syncwarp();
}

// lanes >= pos take the next lane's vertex (pos: the lane of a deleted vertex)
template <int W>
__device__ __forceinline__ void list_delete(LaneVertex<W>& L, int pos, int lane, bool& dirty) {
    const int v = __shfl_down_sync(kFull, L.v, 1);
    const int rc = __shfl_down_sync(kFull, L.rc, 1);
    const uint32_t u1 = __shfl_down_sync(kFull, L.u1, 1), u2 = __shfl_down_sync(kFull, L.u2, 1);
    const uint32_t tk = __shfl_down_sync(kFull, L.tk, 1), um = __shfl_down_sync(kFull, L.umax, 1);
    uint64_t tv[W];
#pragma unroll
    for (int q = 0; q < W; ++q) tv[q] = __shfl_down_sync(kFull, L.tv[q], 1);
    if (lane >= pos) {
        L.v = lane == 31 ? kNoV : v;
        L.rc = rc;
        L.u1 = u1;
        L.u2 = u2;
        L.tk = tk;
        L.umax = um;
#pragma unroll
        for (int q = 0; q < W; ++q) L.tv[q] = tv[q];
        dirty = true;
    }
}

// insert u (cell rcu) at its ascending position (the list holds < 32 vertices, not u); its possibly-tabu
// mask is loaded here and first used in the next step's level search
template <int W>
__device__ __forceinline__ void list_insert(const PlitsWarp& s, LaneVertex<W>& L, int u, int rcu, int lane,
                                            bool& dirty) {
    const int pos = __popc(__ballot_sync(kFull, L.v < u));
    const int v = __shfl_up_sync(kFull, L.v, 1);
    const int rc = __shfl_up_sync(kFull, L.rc, 1);
    const uint32_t u1 = __shfl_up_sync(kFull, L.u1, 1), u2 = __shfl_up_sync(kFull, L.u2, 1);
    const uint32_t tk = __shfl_up_sync(kFull, L.tk, 1), um = __shfl_up_sync(kFull, L.umax, 1);
    uint64_t tv[W];
#pragma unroll
    for (int q = 0; q < W; ++q) tv[q] = __shfl_up_sync(kFull, L.tv[q], 1);
    if (lane > pos) {
        L.v = v;
        L.rc = rc;
        L.u1 = u1;
        L.u2 = u2;
        L.tk = tk;
        L.umax = um;
#pragma unroll
        for (int q = 0; q < W; ++q) L.tv[q] = tv[q];
        dirty = true;
    } else if (lane == pos) {
        L.v = u;
        L.rc = rcu;
        lane_tabu_load<W>(s, L, u);
        dirty = true;
    }
}

// what one line (lane 0: the moved vertex's row, lane 1: its column) reports after the move
struct LineChange {
    int rcF;     // cell of the one left with `from` (its count fell to 1), or -1
    bool keepF;  // ... stays active: its other line repeats `from`
    int rcT;     // cell of the other one with `to` (its count rose to 2), or -1
    int uT;      // its vertex id (the row's lane; -1 for the column's: resolved by the warp)
    int ct;      // the line's count of `to` after the move
};

// lanes 0 (row r of vs) and 1 (column c) apply the move from colour `from` to `to` to their line: count
// planes, and in the register mode the xor table, reporting the membership changes the move can cause
// (plits.hpp:193-212): only cells of this line with colour `from` or `to` change their counts.  The two
// lanes touch different lines, and each reads only lines the other does not write.
template <int W>
__device__ __forceinline__ void line_move(const Graph<W>& g, const PlitsWarp& s, int vs, int r, int c, int from, int to,
                                          bool xor_tables, int lane, LineChange& lc) {
    constexpr int NP = PlitsK<W>::NP;
    const int n = g.n, w1 = n + 1;
    lc.rcF = -1;
    lc.keepF = false;
    lc.rcT = -1;
    lc.uT = -1;
    lc.ct = 0;
    if (lane < 2) {
        if (lane == 0) s.col[vs] = (uint8_t)to;
        uint64_t* P = lane ? s.cp + (size_t)c * NP * W : s.rp + (size_t)r * NP * W;
        int cf, ct;
        plane_move_count<W, NP>(P, from, to, cf, ct);
        lc.ct = ct;
        if (xor_tables) {
            const int r0 = g.rs[r];
            uint8_t* X = s.X + (size_t)(lane ? n + c : r) * w1;
            const int key = lane ? r : vs - r0;  // vs's entry: its row offset / its row index
            int xf = 0, xt = 0;
            if (from) {
                xf = X[from] ^ key;
                X[from] = (uint8_t)xf;
            }
            if (to) {
                xt = X[to] ^ key;
                X[to] = (uint8_t)xt;
            }
            if (from && cf == 1) {
                lc.rcF = lane ? (xf << 8 | c) : g.cell[r0 + xf];
                lc.keepF = plane_multi<W, NP>(lane ? s.rp + (size_t)xf * NP * W
                                                   : s.cp + (size_t)(lc.rcF & 0xFF) * NP * W, from);
            }
            if (to && ct == 2) {
                const int o = xt ^ key;
                if (lane) {
                    lc.rcT = o << 8 | c;
                } else {
                    lc.uT = r0 + o;
                    lc.rcT = g.cell[lc.uT];
                }
            }
        }
    }
}

// the register list after the move of vs (row r, column c) to colour `to`, from the two lines' reports:
// deletions of the cells left alone with `from` (unless their other line repeats it) and of vs when it no
// longer conflicts; insertions of the cells that now share `to` with vs.  Then every lane whose vertex
// changed or lies in row r or column c reloads its move classes.  Returns false when the set outgrew the
// warp (the bitmask mode is set up instead); na is the new |active|.
template <int W>
__device__ __forceinline__ bool sparse_membership(const Graph<W>& g, const PlitsWarp& s, LaneVertex<W>& L, int vs,
                                                  int r, int c, int to, const LineChange& lc, int wf, int wc,
                                                  int lane, int cap, int& na) {
    const int rcF0 = __shfl_sync(kFull, lc.rcF, 0), rcF1 = __shfl_sync(kFull, lc.rcF, 1);
    const unsigned keep = __ballot_sync(kFull, lc.keepF);
    const int rcT0 = __shfl_sync(kFull, lc.rcT, 0), rcT1 = __shfl_sync(kFull, lc.rcT, 1);
    const int uT0 = __shfl_sync(kFull, lc.uT, 0);
    const int ct0 = __shfl_sync(kFull, lc.ct, 0), ct1 = __shfl_sync(kFull, lc.ct, 1);
    const int d1 = (rcF0 >= 0 && !(keep & 1u)) ? rcF0 : -1;
    const int d2 = (rcF1 >= 0 && !(keep & 2u)) ? rcF1 : -1;
    const int d3 = (to && ct0 < 2 && ct1 < 2) ? (r << 8 | c) : -1;
    bool dirty = false;
    int cnt = na;
#pragma unroll
    for (int z = 0; z < 3; ++z) {
        const int d = z == 0 ? d1 : z == 1 ? d2 : d3;
        if (d < 0) continue;
        const unsigned b = __ballot_sync(kFull, L.v != kNoV && L.rc == d);
        list_delete<W>(L, __ffs(b) - 1, lane, dirty);
        --cnt;
    }
    const bool in1 = rcT0 >= 0 && !__any_sync(kFull, L.v != kNoV && L.rc == rcT0);
    const bool in2 = rcT1 >= 0 && !__any_sync(kFull, L.v != kNoV && L.rc == rcT1);
    int uT1 = -1;
    if (in2) {
        // the column's cell: its id from its row (cells of a row are consecutive ids, in column order)
        const int rr = rcT1 >> 8, lo = g.rs[rr], nr = g.rs[rr + 1] - lo;
        for (int x0 = 0; x0 < nr; x0 += 32) {
            const unsigned b = __ballot_sync(kFull, x0 + lane < nr && g.cell[lo + x0 + lane] == rcT1);
            if (b) uT1 = lo + x0 + __ffs(b) - 1;
        }
    }
    const int nins = (int)in1 + (int)in2;
    if (cnt + nins > cap) {
        // refresh the listed vertices in row r / column c, then hand over to the bitmask mode
        if (dirty || (L.rc >> 8) == r || (L.rc & 0xFF) == c) lane_load<W>(g, s, L, wf, wc);
        __syncwarp();
        sparse_leave<W>(g, s, L.v, L.vmin, in1 ? uT0 : -1, in2 ? uT1 : -1, wf, wc, lane);
        na = cnt + nins;
        return false;
    }
    if (in1) list_insert<W>(s, L, uT0, rcT0, lane, dirty);
    if (in2) list_insert<W>(s, L, uT1, rcT1, lane, dirty);
    na = cnt + nins;
    if (dirty || (L.rc >> 8) == r || (L.rc & 0xFF) == c) lane_load<W>(g, s, L, wf, wc);
    return true;
}

// plse_probe on PLITS: gamma[v][k] = cnt_row[r][k] + cnt_col[c][k] - 2 [k = col v] for k >= 1 (the
// incremental table of coloring.hpp:139-156, here from the bit-sliced counts), column 0 zero; the live tabu
// entries (v, k >= 0, until) of the dense table on the phase's own clock (plits.hpp:81)
template <int W>
__device__ void plits_probe_dump(const ImproveArgs& a, const Graph<W>& g, const PlitsWarp& s, const uint32_t* until,
                                 uint32_t base, uint32_t t, int q, int lane) {
    constexpr int NP = PlitsK<W>::NP;
    const int nv = g.nv, w1 = g.n + 1;
    int32_t* gam = a.probe.gamma + (size_t)q * nv * w1;
    for (int v = lane; v < nv; v += 32) {
        const uint16_t rc = g.cell[v];
        const int kv = s.col[v];
        gam[(size_t)v * w1] = 0;
        for (int k = 1; k <= g.n; ++k)
            gam[(size_t)v * w1 + k] = plane_val<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k) +
                                      plane_val<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k) - 2 * (k == kv);
    }
    int32_t* tb = a.probe.tabu + (size_t)q * a.probe.cap * 3;
    int total = 0;
    for (int v0 = 0; v0 < nv; v0 += 32) {
        const int v = v0 + lane;
        int nl = 0;
        if (v < nv)
            for (int k = 0; k <= g.n; ++k) nl += until[(size_t)v * w1 + k] > t;
        const int incl = warp_incl_sum(nl);
        int at = total + incl - nl;
        if (v < nv)
            for (int k = 0; k <= g.n; ++k)
                if (until[(size_t)v * w1 + k] > t) {
                    if (at < a.probe.cap) {
                        tb[3 * at] = v;
                        tb[3 * at + 1] = k;
                        tb[3 * at + 2] = (int32_t)(until[(size_t)v * w1 + k] - base);
                    }
                    ++at;
                }
        total += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) {
        a.probe.n_tabu[q] = total;
        *a.probe.dumped = q + 1;
    }
    __syncwarp();
}

template <int W, bool kDebug>
__device__ void plits_one(const ImproveArgs& a, const Graph<W>& g, const PlitsWarp& s, uint32_t* until,
                          uint32_t* slot_clock, int i, int lane, bool sparse_ok) {
    constexpr int NP = PlitsK<W>::NP;
    constexpr int NB = PlitsK<W>::NB;
    const int n = g.n, nv = g.nv, w1 = n + 1;
    const int v_lo = lane * 32 * g.lane_words;
    uint8_t* col = s.col;
    uint8_t* best_row = a.improved + (size_t)i * g.nvpad;
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
    const bool probing = kDebug && (i == a.trace_idx) && a.probe.n > 0;
    int probe_next = 0;
    unsigned long long* prof = kDebug ? a.prof : nullptr;
    // steps, list, level, select, move, step, level iters, sum na | move: plane, membership, tail
    unsigned long long pc[14] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long modes = 0;  // register-mode entries (low half) and exits (high half)
    const int cap = kDebug ? min(max(g_plits_list_cap, kListHysteresis + 1), 32) : 32;
    long long tp0 = 0, tp1 = 0;

    // ---- tabu clock of this warp slot (two phases, each followed by a skip of tenure_cap + 2)
    uint32_t base = *slot_clock;
    if ((uint64_t)base + (uint64_t)a.budget + (uint64_t)a.budget2 + 2ull * (a.tenure_cap + 4) >= 0xFFFFFFFFull) {
        uint4* u4 = reinterpret_cast<uint4*>(until);
        for (size_t x = lane; x < a.until_stride / 4; x += 32) u4[x] = make_uint4(0, 0, 0, 0);
        base = 0;
    }
    snapshot(a.offspring + (size_t)i * g.nvpad, col, g.nvpad, lane);
    __syncwarp();

    const uint64_t seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    CanonDraws draws{seed, 0u, 0u, -1};
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
    plits_build<W>(g, s, lane, 2, 1, f, c, active);
    const int initial_f = f;
    uint32_t J = 0;  // step index over both phases: the canonical draw's key
    int64_t iters = 0;
    bool hit = false;
    bool pending = true;  // the phase best equals the current colouring
    int best_f = f, best_c = c;
    unsigned long long acc = 0;
    bool sparse = false;  // the register-resident active list is in use
    LaneVertex<W> L;

    for (int phase = 1; phase <= 2; ++phase) {
        const int wf = 2;
        const int wc = phase == 1 ? 1 : 2 * nv;  // PhaseWeights::from_phi(0.5 / |V|), plits.hpp:27-33
        const int64_t budget = phase == 1 ? a.budget : a.budget2;
        if (phase == 2) plits_build<W>(g, s, lane, wf, wc, f, c, active);  // from phase 1's best
        sparse = sparse_ok && active <= cap;
        if (sparse) {
            sparse_enter<W>(g, s, L, wf, wc, lane);
            if (prof) ++modes;
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
            if (kDebug && probing && probe_next < a.probe.n && (int64_t)J == a.probe.steps[probe_next]) {
                __syncwarp();
                plits_probe_dump<W>(a, g, s, until, base, base + j, probe_next++, lane);
            }
            const uint32_t t = base + j;
            uint32_t h1, h2;
            draws.at(J, lane, h1, h2);
            const int64_t cur_scaled = (int64_t)wf * f + (int64_t)wc * c;
            const int64_t thr64 = best_scaled - cur_scaled;  // a tabu move is admissible iff delta < thr
            const int thr = (int)max(min(thr64, (int64_t)INT_MAX), (int64_t)INT_MIN);
            const int active_before = active;
            if (prof) tp0 = tp1 = clock64();
            auto tick = [&](int slot) {
                if (prof) {
                    const long long x = clock64();
                    pc[slot] += (unsigned long long)(x - tp1);
                    tp1 = x;
                }
            };

            if (prof) pc[7] += (unsigned)active;
            int N = 0, dl = INT_MAX, vs = -1, ks = 0, dcs = 0;
            if (sparse) {
                tick(1);
                // ---- the lowest level with an admissible candidate, all from registers (until[][] only
                // for possibly-tabu colours at the level)
                bool hp = false;
                int prev = 0, cnt = 0;
                uint64_t adm[W];
                bool adm0 = false;
                if ((L.tk & kTabuOvf) && L.umax <= t) {  // every entry of v has expired
                    L.tk = 0;
                    L.u1 = L.u2 = 0;
                }
                for (;;) {
                    int lm = L.vmin;
                    if (hp) {
                        uint64_t M2[W];
#pragma unroll
                        for (int q = 0; q < W; ++q) M2[q] = L.m.M[q];
                        lm = INT_MAX;
                        if (L.v != kNoV) {
                            const int x = prev - L.m.dbase;
                            sliced_ge<W, NB>(L.m.S, (wc == 1 ? x : floor_div(x, wc)) + 1, M2);
                            if (L.m.cur && L.m.d0 > prev) lm = L.m.d0;
                            if (popc_w<W>(M2)) lm = min(lm, L.m.dbase + wc * sliced_min<W, NB>(L.m.S, M2));
                        }
                    }
                    dl = __reduce_min_sync(kFull, lm);
                    if (dl == INT_MAX) break;  // every candidate tabu
                    const bool asp_all = dl < thr;
                    cnt = 0;
                    adm0 = false;
#pragma unroll
                    for (int q = 0; q < W; ++q) adm[q] = 0;
                    if (L.v != kNoV && (hp || L.vmin <= dl)) {
                        if (L.tk & kTabuOvf) {
                            bool ch;
                            cnt = level_adm<W>(L.m, dl, wc, asp_all, until + (size_t)L.v * w1, L.tv, t, adm, adm0,
                                               ch);
                        } else {
                            cnt = level_adm_cached<W>(L, dl, wc, asp_all, t, adm, adm0);
                        }
                    }
                    N = (int)__reduce_add_sync(kFull, (unsigned)cnt);
                    if (N > 0) break;
                    hp = true;
                    prev = dl;
                    if (prof) ++pc[6];
                }
                tick(2);
                if (N > 0) {
                    // ---- the r-th admissible candidate in ascending (v, k): lanes are in ascending v
                    const uint32_t rnk = __umulhi(h1, (uint32_t)N);
                    const int incl = warp_incl_sum(cnt);
                    const bool owner = (uint32_t)(incl - cnt) <= rnk && rnk < (uint32_t)incl;
                    int sk = 0, sdc = 0;
                    if (owner) {
                        const int local = (int)rnk - (incl - cnt);
                        sk = (adm0 && local == 0) ? 0 : nth_bit_w<W>(adm, local - (adm0 ? 1 : 0));
                        const int gcur = L.m.cur ? div_wc(wf - L.m.d0, wc) : 0;
                        sdc = (sk ? div_wc(dl - L.m.dbase, wc) : 0) - gcur;
                    }
                    const int wl = __ffs(__ballot_sync(kFull, owner)) - 1;
                    vs = __shfl_sync(kFull, L.v, wl);
                    ks = __shfl_sync(kFull, sk, wl);
                    dcs = __shfl_sync(kFull, sdc, wl);
                }
                tick(3);
            } else {
                // ---- compact the active set into ascending ids; lane L takes the L-th contiguous block, so
                // lanes in order then list order is the ascending (v, k) order of the canonical rule
                int na = 0;
                {
                    int my = 0;
                    for (int q = 0; q < g.lane_words; ++q) my += __popc(s.A[lane * g.lane_words + q]);
                    const int incl = warp_incl_sum(my);
                    na = __shfl_sync(kFull, incl, 31);
                    int pos = incl - my;
                    for (int q = 0; q < g.lane_words; ++q) {
                        uint32_t bits = s.A[lane * g.lane_words + q];
                        while (bits) {
                            s.list[pos++] = (uint16_t)(v_lo + 32 * q + __ffs(bits) - 1);
                            bits &= bits - 1;
                        }
                    }
                }
                __syncwarp();
                const int per = (na + 31) >> 5;
                const int i_lo = min(na, lane * per), i_hi = min(na, i_lo + per);
                tick(1);
                // ---- the lowest delta level holding an admissible candidate: its tabu-blind minimum from
                // the cached per-vertex minima, then the until[][] reads of the candidates at that level only
                bool has_prev = false;
                int prev = 0, lc = 0;
                bool asp_all = false;
                int c_v = -1, c_d0 = 0, c_dbase = 0;  // this lane's first vertex with admissible moves at dl
                uint64_t c_adm[W];
                bool c_adm0 = false;
                for (;;) {
                    int lmin = INT_MAX;
                    for (int idx = i_lo; idx < i_hi; ++idx) {
                        {
                            const int v = s.list[idx];
                            int vm;
                            if (!has_prev) {
                                vm = s.vmin[v];
                            } else {
                                VertexMoves<W> m;
                                vertex_moves<W>(g, s, v, wf, wc, m);
                                sliced_ge<W, NB>(m.S, floor_div(prev - m.dbase, wc) + 1, m.M);
                                vm = (m.cur && m.d0 > prev) ? m.d0 : INT_MAX;
                                if (popc_w<W>(m.M)) vm = min(vm, m.dbase + wc * sliced_min<W, NB>(m.S, m.M));
                            }
                            lmin = min(lmin, vm);
                        }
                    }
                    dl = __reduce_min_sync(kFull, lmin);
                    long long tl0 = prof ? clock64() : 0;
                    if (prof) pc[has_prev ? 13 : 11] += (unsigned long long)(tl0 - tp1);
                    if (dl == INT_MAX) break;  // every candidate tabu
                    asp_all = dl < thr;
                    lc = 0;
                    c_v = -1;
                    for (int idx = i_lo; idx < i_hi; ++idx) {
                        {
                            const int v = s.list[idx];
                            if (!has_prev && s.vmin[v] > dl) continue;
                            uint64_t tv[W];
#pragma unroll
                            for (int q = 0; q < W; ++q) tv[q] = s.T[(size_t)v * (W + 1) + q];
                            VertexMoves<W> m;
                            vertex_moves<W>(g, s, v, wf, wc, m);
                            uint64_t adm[W];
                            bool adm0;
                            bool ch;
                            const int cnt = level_adm<W>(m, dl, wc, asp_all, until + (size_t)v * w1, tv, t, adm, adm0, ch);
                            if (ch) {
#pragma unroll
                                for (int q = 0; q < W; ++q) s.T[(size_t)v * (W + 1) + q] = tv[q];
                            }
                            if (cnt && c_v < 0) {
                                c_v = v;
                                c_adm0 = adm0;
                                c_d0 = m.d0;
                                c_dbase = m.dbase;
#pragma unroll
                                for (int qq = 0; qq < W; ++qq) c_adm[qq] = adm[qq];
                            }
                            s.vcnt[v] = (uint8_t)cnt;
                            lc += cnt;
                        }
                    }
                    N = (int)__reduce_add_sync(kFull, (unsigned)lc);
                    if (prof) {
                        const long long x = clock64();
                        pc[has_prev ? 13 : 12] += (unsigned long long)(x - tl0);
                        tp1 = x;
                    }
                    if (N > 0) break;
                    has_prev = true;
                    prev = dl;
                    if (prof) ++pc[6];
                }
                __syncwarp();
                tick(2);
                if (N > 0) {
                    // ---- the r-th admissible candidate in ascending (v, k)
                    const uint32_t rnk = __umulhi(h1, (uint32_t)N);
                    const int incl = warp_incl_sum(lc);
                    const bool owner = (uint32_t)(incl - lc) <= rnk && rnk < (uint32_t)incl;
                    int sv = -1, sk = 0, sdc = 0;
                    if (owner) {
                        int local = (int)rnk - (incl - lc);
                        for (int idx = i_lo; idx < i_hi && sv < 0; ++idx) {
                            {
                                const int v = s.list[idx];
                                if (!has_prev && s.vmin[v] > dl) continue;
                                const int cnt = s.vcnt[v];
                                if (local < cnt) {
                                    sv = v;
                                    break;
                                }
                                local -= cnt;
                            }
                        }
                        uint64_t adm[W];
                        bool adm0;
                        int d0, dbase, cur;
                        if (sv == c_v) {
                            adm0 = c_adm0;
                            d0 = c_d0;
                            dbase = c_dbase;
#pragma unroll
                            for (int q = 0; q < W; ++q) adm[q] = c_adm[q];
                        } else {
                            VertexMoves<W> m;
                            vertex_moves<W>(g, s, sv, wf, wc, m);
                            uint64_t tv[W];
#pragma unroll
                            for (int q = 0; q < W; ++q) tv[q] = s.T[(size_t)sv * (W + 1) + q];
                            bool ch;
                            level_adm<W>(m, dl, wc, asp_all, until + (size_t)sv * w1, tv, t, adm, adm0, ch);
                            if (ch) {
#pragma unroll
                                for (int q = 0; q < W; ++q) s.T[(size_t)sv * (W + 1) + q] = tv[q];
                            }
                            d0 = m.d0;
                            dbase = m.dbase;
                        }
                        cur = col[sv];
                        if (adm0 && local == 0)
                            sk = 0;
                        else
                            sk = nth_bit_w<W>(adm, local - (adm0 ? 1 : 0));
                        // every candidate at level dl has gamma[v][k] = (dl - dbase) / wc; gamma[v][cur] from d0
                        const int gcur = cur ? (wf - d0) / wc : 0;
                        sdc = (sk ? (dl - dbase) / wc : 0) - gcur;
                    }
                    tick(3);
                    const int wl = __ffs(__ballot_sync(kFull, owner)) - 1;
                    vs = __shfl_sync(kFull, sv, wl);
                    ks = __shfl_sync(kFull, sk, wl);
                    dcs = __shfl_sync(kFull, sdc, wl);
                }
            }
            if (N == 0) {
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

            const int from = col[vs];
            const int dfs = (ks == 0) - (from == 0);
            const int64_t now = cur_scaled + dl;
            if (now >= best_scaled && pending) {
                // deferred snapshot: the colouring about to change is the phase best
                snapshot(col, best_row, g.nvpad, lane);
                pending = false;
            }
            __syncwarp();
            const uint16_t rcs = g.cell[vs];
            const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
            LineChange lch;
            line_move<W>(g, s, vs, rs_, cs_, from, ks, sparse, lane, lch);
            __syncwarp();
            long long tm0 = prof ? clock64() : 0;
            if (prof) pc[8] += (unsigned long long)(tm0 - tp1);
            if (sparse) {
                sparse = sparse_membership<W>(g, s, L, vs, rs_, cs_, ks, lch, wf, wc, lane, cap, active);
                if (prof && !sparse) modes += 1ULL << 32;
            } else {
                plits_membership<W>(g, s, rs_, cs_, from, ks, wf, wc, lane);
                __syncwarp();
                int al = 0;
                for (int q = 0; q < g.lane_words; ++q) al += __popc(s.A[lane * g.lane_words + q]);
                active = (int)__reduce_add_sync(kFull, (unsigned)al);
            }
            if (prof) {
                const long long x = clock64();
                pc[9] += (unsigned long long)(x - tm0);
                tm0 = x;
            }
            f += dfs;
            c += dcs;
            const uint32_t tenure = __umulhi(h2, 10u) + (uint32_t)(alpha * (double)active);
            if (lane == 0) {
                until[(size_t)vs * w1 + from] = t + 1 + tenure;
                // fire-and-forget reductions: nothing in the step waits for them
                uint64_t* rec = s.T + (size_t)vs * (W + 1);
                atomicOr(reinterpret_cast<unsigned long long*>(rec + (from >> 6)), 1ULL << (from & 63));
                atomicMax(reinterpret_cast<unsigned int*>(rec + W), t + 1 + tenure);
                acc += 2ULL * (unsigned)w1 * (unsigned)active_before + 4ULL * g.deg[vs] + 2ULL;
            }
            if (sparse && L.v == vs) lane_tabu_write<W>(L, from, t + 1 + tenure, t);
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
                                N, dl};
            }
            __syncwarp();
            if (!sparse && sparse_ok && active <= cap - kListHysteresis) {
                sparse_enter<W>(g, s, L, wf, wc, lane);
                sparse = true;
                if (prof) ++modes;
            }
            if (prof) pc[10] += (unsigned long long)(clock64() - tm0);
            tick(4);
            if (prof) {
                pc[5] += (unsigned long long)(clock64() - tp0);
                ++pc[0];
            }
            ++j;
            ++J;
        }
        if (best_c == 0 && best_f <= stop_f) hit = true;
        iters += j;
        // the phase's result is its best colouring (plits.hpp:268)
        if (!pending) {
            snapshot(best_row, col, g.nvpad, lane);
            __syncwarp();
            pending = true;
        }
        base += j + 2 + a.tenure_cap;  // every until written in this phase is < base
        if (hit) break;                // plits.hpp:284: phase 2 only when phase 1 missed the target
    }

    // ---- final greedy repair when the result still conflicts (plits.hpp:289, partial.hpp:22-39):
    // argmax gamma[v][col v] over the conflicting (active, coloured) vertices, lowest id on ties
    if (best_c > 0) {
        plits_build<W>(g, s, lane, 2, 2 * nv, f, c, active);
        for (;;) {
            int bc = 0, bv = -1;
            for (int q = 0; q < g.lane_words; ++q) {
                uint32_t bits = s.A[lane * g.lane_words + q];
                while (bits) {
                    const int v = v_lo + 32 * q + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int k = col[v];
                    if (!k) continue;
                    const uint16_t rc = g.cell[v];
                    const int gv = plane_val<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k) +
                                   plane_val<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k) - 2;
                    if (gv > bc) {
                        bc = gv;
                        bv = v;
                    }
                }
            }
            const int mx = (int)__reduce_max_sync(kFull, (unsigned)bc);
            if (mx == 0) break;
            const int wl = __ffs(__ballot_sync(kFull, bc == mx)) - 1;
            const int w = __shfl_sync(kFull, bv, wl);
            const int k = col[w];
            const uint16_t rc = g.cell[w];
            __syncwarp();
            if (lane == 0) {
                col[w] = 0;
                plane_move<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k, 0);
            }
            if (lane == 1) plane_move<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k, 0);
            __syncwarp();
            plits_membership<W>(g, s, rc >> 8, rc & 0xFF, k, 0, 2, 2 * nv, lane);
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
            for (int z = 0; z < 8; ++z) atomicAdd(prof + z, pc[z]);
            atomicAdd(prof + 8, 1ULL);
            for (int z = 8; z < 14; ++z) atomicAdd(prof + z + 1, pc[z]);
            atomicAdd(prof + 15, modes);
        }
    }
    __syncwarp();
}

template <int W, bool kDebug>
// one CTA per SM: the register-resident active list needs more than 128 registers per thread
__global__ void __launch_bounds__(kPlitsMaxThreads, 1) k_plits(const ImproveArgs a) {
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
    s.rp = reinterpret_cast<uint64_t*>(wbase + L.w_rp);
    s.cp = reinterpret_cast<uint64_t*>(wbase + L.w_cp);
    s.A = reinterpret_cast<uint32_t*>(wbase + L.w_A);
    s.list = reinterpret_cast<uint16_t*>(wbase + L.w_list);
    s.vmin = reinterpret_cast<int32_t*>(wbase + L.w_vmin);
    s.vcnt = wbase + L.w_vcnt;
    s.X = wbase + L.w_list;
    // the register mode needs its xor tables to fit over list / vmin / vcnt (|V| >= ~0.3 n^2)
    const bool sparse_ok = (size_t)2 * n * (n + 1) <= L.warp_bytes - L.w_list;

    const int slot = blockIdx.x * nwarps + warp;
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    // the possibly-tabu masks and until bounds live in the slot's tabu-record area (capi.cu sizes it for
    // nv * 8 (W + 1) bytes); stale content is harmless: a superset mask, and every until[][] entry of an
    // earlier individual is below its clock
    s.T = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(a.tabu_rec) + (size_t)slot * a.rec_stride);

    for (int i = first_individual(a.first, a.nslots, a.p, warp); i < a.p;
         i = next_individual(a.first, a.nslots, a.work_counter, lane))
        plits_one<W, kDebug>(a, g, s, until, a.slot_clock + slot, i, lane, sparse_ok);
}

cudaError_t set_plits_list_cap(int cap, cudaStream_t st) {
    return cudaMemcpyToSymbolAsync(g_plits_list_cap, &cap, sizeof(int), 0, cudaMemcpyHostToDevice, st);
}

const void* plits_kernel_ptr(int W, bool debug) {
    if (W == 1) return debug ? reinterpret_cast<const void*>(&k_plits<1, true>)
                             : reinterpret_cast<const void*>(&k_plits<1, false>);
    return debug ? reinterpret_cast<const void*>(&k_plits<2, true>)
                 : reinterpret_cast<const void*>(&k_plits<2, false>);
}

cudaError_t launch_plits(const ImproveArgs& a, int W, int grid, int threads, size_t smem, cudaStream_t st) {
    const bool debug = a.trace != nullptr || a.prof != nullptr || a.probe.n > 0;
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
