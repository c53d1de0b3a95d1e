// improve_common.cuh -- device helpers shared by the improve kernels
// (improve.cu and improve_ref.cu: one individual per warp).
#pragma once
#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

// per-vertex tabu cache: (k1, u1), (k2, u2) exact until values of the two
// most recently forbidden colours; kk = k1 | k2 << 8 | ovf << 16.  ovf: a
// third colour was forbidden while both pairs were live -> consult until[][].
struct alignas(16) TabuRec {
    uint32_t u1, u2, kk, pad;
};

struct WarpSmem {
    uint8_t* col;    // colour of vertex v
    uint8_t* conf;   // repair counters
    uint64_t* R;
    uint64_t* C;
    uint32_t* U;
    uint8_t* colT;   // improve: colour of vertex cl[x] (column-major copy)
    uint16_t* list;  // improve: 32-entry seed list of sparse mode
    uint64_t* seed = nullptr;  // k_improve: the individual's stream seed
};

template <int W>
struct Graph {
    int n, nv, nvpad, lane_words;
    const uint16_t* cell;
    const uint8_t* deg;  // |N(v)| = row-mates + column-mates (for the 8(d) byte counter)
    const uint16_t* rs;
    const uint16_t* cs;
    const uint16_t* cl;
    const uint16_t* colpos;  // position of v in the column-major copy (k_improve: the column-padded copy)
    const uint64_t* pr;
    const uint64_t* pc;
    uint64_t full[W];
    // k_improve's padded layouts (nullptr in the other kernels): s.col / s.colT are then the row- / column-
    // padded copies, v's colour is s.col[rpos[v]]
    const uint16_t* rpos = nullptr;
    const uint64_t* rinfo = nullptr;  // [n] offset | 8-byte words << 16 | first vertex << 32
    const uint64_t* cinfo = nullptr;  // [n] offset | 8-byte words << 16 | column-list base << 32
};

// Work distribution of the persistent improve kernels.  Only `nslots` warp slots search (the host picks
// nslots = ceil(p / rounds) with rounds = ceil(p / resident warps), so every slot gets the same number of
// individuals and no round runs half empty); slot (CTA b, warp w) is number b + gridDim.x * w, so the active
// slots are spread evenly over the SMs and their schedulers.  A slot's first individual is first + its
// number, the rest are pulled from the work counter (load balance for the very different per-individual
// step counts).
__device__ __forceinline__ int first_individual(int first, int nslots, int p, int warp) {
    const int s = (int)blockIdx.x + (int)gridDim.x * warp;
    return s < nslots ? first + s : p;
}
__device__ __forceinline__ int next_individual(int first, int nslots, int* counter, int lane) {
    int k = 0;
    if (lane == 0) k = atomicAdd(counter, 1);
    return first + nslots + __shfl_sync(0xFFFFFFFFu, k, 0);
}

// colour of vertex v in either layout
template <int W>
__device__ __forceinline__ int col_of(const Graph<W>& g, const WarpSmem& s, int v) {
    return g.rpos ? s.col[g.rpos[v]] : s.col[v];
}

template <int W>
__device__ __forceinline__ void dom_mask(const Graph<W>& g, int r, int c, uint64_t (&d)[W]) {
#pragma unroll
    for (int q = 0; q < W; ++q) d[q] = ~(g.pr[r * W + q] | g.pc[c * W + q]) & g.full[q];
}

// exact tabu mask at clock t from a (u1, u2, kk) cache; the overflow case reads
// the dense table for every colour of D(v) and rebuilds the cache when <= 2 remain
template <int W>
__device__ __forceinline__ void tabu_of(uint32_t& u1, uint32_t& u2, uint32_t& kk, const uint32_t* until_row,
                                        const uint64_t (&dom)[W], uint32_t t, uint64_t (&T)[W]) {
#pragma unroll
    for (int q = 0; q < W; ++q) T[q] = 0;
    if (!(kk >> 16)) {
        const int k1 = kk & 0xFF, k2 = (kk >> 8) & 0xFF;
        if (u1 > t) T[k1 >> 6] |= 1ULL << (k1 & 63);
        if (u2 > t) T[k2 >> 6] |= 1ULL << (k2 & 63);
        return;
    }
    int n_live = 0, ka = 0, kb = 0;
    uint32_t ua = 0, ub = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t m = dom[q];
        while (m) {
            const int b = __ffsll((long long)m) - 1;
            m &= m - 1;
            const int k = q * 64 + b;
            const uint32_t u = until_row[k];
            if (u > t) {
                T[q] |= 1ULL << b;
                if (n_live == 0) {
                    ka = k;
                    ua = u;
                } else if (n_live == 1) {
                    kb = k;
                    ub = u;
                }
                ++n_live;
            }
        }
    }
    if (n_live <= 2) {
        u1 = ua;
        u2 = ub;
        kk = (uint32_t)ka | ((uint32_t)kb << 8);
    }
}

// forbid (k, until = ut) in a vertex's cache (search_util.hpp:73-75 overwrite semantics)
__device__ __forceinline__ void cache_forbid(TabuRec& r, int k, uint32_t ut, uint32_t t) {
    const int k1 = r.kk & 0xFF, k2 = (r.kk >> 8) & 0xFF;
    uint32_t ovf = r.kk & 0xFF0000u;
    int n1 = k1, n2 = k2;
    if (k1 == k && r.u1) {
        r.u1 = ut;
    } else if (k2 == k && r.u2) {
        r.u2 = ut;
    } else if (r.u1 <= t) {
        n1 = k;
        r.u1 = ut;
    } else if (r.u2 <= t) {
        n2 = k;
        r.u2 = ut;
    } else {
        ovf = 1u << 16;  // both cached colours still tabu: the dense table is now authoritative
        if (r.u1 <= r.u2) {
            n1 = k;
            r.u1 = ut;
        } else {
            n2 = k;
            r.u2 = ut;
        }
    }
    r.kk = (uint32_t)n1 | ((uint32_t)n2 << 8) | ovf;
}

// cache_forbid as straight-line selects (the sparse loop's evictee lanes run it every step)
__device__ __forceinline__ void cache_forbid_nb(TabuRec& r, int k, uint32_t ut, uint32_t t) {
    const int k1 = r.kk & 0xFF, k2 = (r.kk >> 8) & 0xFF;
    const bool A = k1 == k && r.u1 != 0;  // k already cached in pair 1
    const bool B = k2 == k && r.u2 != 0;  // ... in pair 2
    const bool l1 = r.u1 > t, l2 = r.u2 > t;
    const bool ov = !A && !B && l1 && l2;  // both pairs live: the dense table becomes authoritative
    const bool s1 = A || (!B && (!l1 || (l2 && r.u1 <= r.u2)));
    const uint32_t n1 = s1 ? (uint32_t)k : (uint32_t)k1, n2 = s1 ? (uint32_t)k2 : (uint32_t)k;
    r.u1 = s1 ? ut : r.u1;
    r.u2 = s1 ? r.u2 : ut;
    r.kk = n1 | (n2 << 8) | (ov ? (1u << 16) : (r.kk & 0xFF0000u));
}

// The move of partial.hpp:124-141 on the occupancy state, as one straight-line predicated pass (no
// reconvergence blocks): lanes 0-2 write the colour byte (row- and column-major) and the U bit of v*, ur,
// uc; lane 1 clears k* from C[col ur], lane 2 from R[row uc]; lane 3 sets it in R[row v*] unless ur held
// it, lane 4 in C[col v*] unless uc did; lanes 1/2 forbid (evictee, k*) until ut (search_util.hpp:73-75)
// and return the evictee's updated tabu cache.  Adds the SURVEY 8(d) bytes of the step to acc (lanes 0-2).
template <int W>
__device__ __forceinline__ TabuRec apply_move_lanes(const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                                                    uint32_t* until, int vs, int ur, int uc, int ks, int rs_,
                                                    int cs_, bool inR, bool inC, int f_before, bool improved,
                                                    uint32_t ut, uint32_t t, int lane, unsigned long long& acc) {
    const int w1 = g.n + 1, kw = ks >> 6;
    const uint64_t bitk = 1ULL << (ks & 63);
    (void)rs_;
    (void)cs_;
    // lane 1 addresses ur, lane 2 uc, every other lane v* (lanes 3/4 take v*'s row / column from its cell)
    const bool l1 = lane == 1, l2 = lane == 2;
    const int u = l1 ? ur : l2 ? uc : vs;
    const bool act = lane < 3 && u >= 0;
    const int uu = max(u, 0);
    TabuRec nr = rec[uu];  // issued early, consumed after the updates (lanes 1/2 only)
    const uint16_t cu = g.cell[uu];
    const int cpos = g.colpos[uu];
    const uint32_t dg = g.deg[uu];
    __syncwarp();
    const uint8_t nc = lane == 0 ? (uint8_t)ks : (uint8_t)0;
    if (act) {
        s.col[uu] = nc;
        s.colT[cpos] = nc;
        atomicXor(&s.U[uu >> 5], 1u << (uu & 31));
    }
    const bool on_c = l1 || lane == 4;
    const int line_no = on_c ? (cu & 0xFF) : (cu >> 8);
    const bool lx = lane == 3 ? !inR : lane == 4 ? !inC : (l1 || l2) && act;
    uint64_t* line = (on_c ? s.C : s.R) + line_no * W + kw;
    if (lx) *line ^= bitk;
    acc += (act ? 4u * dg + 2u : 0u) +
           (lane == 0 ? 2u * (uint32_t)w1 * (uint32_t)f_before + (improved ? 2u * (uint32_t)g.nv : 0u) : 0u);
    if (act && lane > 0) {
        until[(size_t)uu * w1 + ks] = ut;
        cache_forbid_nb(nr, ks, ut, t);
        rec[uu] = nr;
    }
    return nr;
}

// inclusive warp prefix sum: per round one shfl.up whose in-range predicate guards the add (no lane test,
// no select)
__device__ __forceinline__ int warp_incl_sum(int x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm volatile("{\n\t.reg .s32 r0;\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 r0|p, %0, %1, 0x0, 0xffffffff;\n\t"
            "@p add.s32 %0, r0, %0;\n\t}"
            : "+r"(x)
            : "r"(d));
    return x;
}

// inclusive warp prefix minimum, same scheme
__device__ __forceinline__ int warp_incl_min(int x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm volatile("{\n\t.reg .s32 r0;\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 r0|p, %0, %1, 0x0, 0xffffffff;\n\t"
            "@p min.s32 %0, r0, %0;\n\t}"
            : "+r"(x)
            : "r"(d));
    return x;
}

// rr-th set bit (0-based) of lane src's W-word mask, found by the whole warp: lane src's words are
// broadcast and lane l tests bit l of the word holding the answer (warp-uniform result)
template <int W>
__device__ __forceinline__ int warp_nth_bit(const uint64_t (&m)[W], int rr, int src, int lane) {
    if (W == 1) {
        // one 64-bit mask: pick its half by the low half's popcount, then lane l tests bit l of that half
        const uint32_t lo = __shfl_sync(kFull, (uint32_t)m[0], src), hi = __shfl_sync(kFull, (uint32_t)(m[0] >> 32), src);
        const int clo = __popc(lo);
        const bool up = rr >= clo;
        const uint32_t word = up ? hi : lo;
        const int r2 = up ? rr - clo : rr;
        const bool hit = ((word >> lane) & 1u) && __popc(word & ((1u << lane) - 1u)) == r2;
        return (up ? 32 : 0) + __ffs(__ballot_sync(kFull, hit)) - 1;
    }
    uint32_t word = 0;
    int wbase = 0, r2 = 0;
#pragma unroll
    for (int z = 0; z < 2 * W; ++z) {
        const uint32_t x = __shfl_sync(kFull, (uint32_t)(m[z >> 1] >> (32 * (z & 1))), src);
        const int pc = __popc(x);
        const bool here = rr >= 0 && rr < pc;
        word = here ? x : word;
        wbase = here ? 32 * z : wbase;
        r2 = here ? rr : r2;
        rr -= pc;
    }
    const bool hit = ((word >> lane) & 1u) && __popc(word & ((1u << lane) - 1u)) == r2;
    return wbase + __ffs(__ballot_sync(kFull, hit)) - 1;
}

// admissible candidate masks of an uncoloured vertex at the three delta levels
template <int W>
__device__ __forceinline__ void level_masks(const WarpSmem& s, int r, int c, const uint64_t (&dom)[W],
                                            const uint64_t (&T)[W], bool asp, uint64_t (&m0)[W], uint64_t (&m1)[W],
                                            uint64_t (&m2)[W]) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const uint64_t Rr = s.R[r * W + q], Cc = s.C[c * W + q];
        const uint64_t fr = dom[q] & ~Rr & ~Cc;
        m0[q] = asp ? fr : (fr & ~T[q]);
        m1[q] = dom[q] & (Rr ^ Cc) & ~T[q];
        m2[q] = dom[q] & Rr & Cc & ~T[q];
    }
}

// dense mode: masks of vertex v with its tabu cache read from (and written back to) HBM
template <int W>
__device__ __forceinline__ void dense_masks(const Graph<W>& g, const WarpSmem& s, TabuRec* rec, const uint32_t* until,
                                            int v, uint32_t t, bool asp, uint64_t (&m0)[W], uint64_t (&m1)[W],
                                            uint64_t (&m2)[W]) {
    const uint16_t rc = g.cell[v];
    const int r = rc >> 8, c = rc & 0xFF;
    uint64_t dom[W], T[W];
    dom_mask<W>(g, r, c, dom);
    TabuRec tr = rec[v];
    const uint32_t kk0 = tr.kk;
    tabu_of<W>(tr.u1, tr.u2, tr.kk, until + (size_t)v * (g.n + 1), dom, t, T);
    if (tr.kk != kk0) rec[v] = tr;
    level_masks<W>(s, r, c, dom, T, asp, m0, m1, m2);
}

template <int W>
__device__ __forceinline__ int popc_w(const uint64_t (&m)[W]) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) c += __popcll(m[q]);
    return c;
}

// lowest set bit of a W-word mask (64 W if empty)
template <int W>
__device__ __forceinline__ int first_bit_w(const uint64_t (&m)[W]) {
    int k = 64 * W;
#pragma unroll
    for (int z = W - 1; z >= 0; --z)
        if (m[z]) k = z * 64 + __ffsll((long long)m[z]) - 1;
    return k;
}

// set bits of a W-word mask below bit position pos
template <int W>
__device__ __forceinline__ int popc_below_w(const uint64_t (&m)[W], int pos) {
    int c = 0;
#pragma unroll
    for (int z = 0; z < W; ++z) {
        const int lo = z * 64;
        const uint64_t mk = pos >= lo + 64 ? ~0ULL : pos <= lo ? 0ULL : (1ULL << (pos - lo)) - 1;
        c += __popcll(m[z] & mk);
    }
    return c;
}

// 0-based rr-th set bit of a W-word mask (rr < popc)
template <int W>
__device__ __forceinline__ int nth_bit_w(const uint64_t (&m)[W], int rr) {
    int k = 0;
#pragma unroll
    for (int z = 0; z < W; ++z) {
        const int pz = __popcll(m[z]);
        if (rr >= 0 && rr < pz) k = z * 64 + nth_bit64(m[z], rr);
        rr -= pz;
    }
    return k;
}

__device__ __forceinline__ void snapshot(const uint8_t* col, uint8_t* dst, int nvpad, int lane) {
    const uint4* s4 = reinterpret_cast<const uint4*>(col);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int t = lane; t < nvpad / 16; t += 32) d4[t] = s4[t];
}

// position of the unique byte == k in bytes [a, b) of buf, or -1 (warp-uniform result)
__device__ __forceinline__ int warp_find_byte(const uint8_t* buf, int a, int b, int k, bool enable, int lane) {
    if (!enable) return -1;
    const uint32_t k4 = (uint32_t)k * 0x01010101u;
    for (int base = a & ~3; base < b; base += 128) {
        const int wpos = base + 4 * lane;
        uint32_t hit = 0;
        if (wpos < b) {
            const uint32_t w = reinterpret_cast<const uint32_t*>(buf)[wpos >> 2] ^ k4;
            const uint32_t z = ~(((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;  // 0x80 where byte == k
            const int lo = a - wpos, hi = b - wpos;  // valid bytes q: lo <= q < hi
            uint32_t valid = 0x80808080u;
            if (lo > 0) valid &= 0x80808080u << (8 * min(lo, 4));
            if (hi < 4) valid &= 0x80808080u >> (8 * (4 - max(hi, 0)));
            hit = z & valid;
        }
        const unsigned bal = __ballot_sync(kFull, hit != 0);
        if (bal) {
            const int src = __ffs(bal) - 1;
            return __shfl_sync(kFull, wpos + ((__ffs(hit) - 1) >> 3), src);
        }
    }
    return -1;
}

// plse_probe: materialise the state the step reads, as the reference holds it (coloring.hpp:105-116,
// search_util.hpp:54-81).  gamma[v][k]: 0 for k = 0; for k = col(v) the conflict count (same-coloured
// neighbours, what the repair counters hold); otherwise [k in R[row v]] + [k in C[col v]] from the
// occupancy masks the kernel decides with.  Tabu: every dense-table entry live at clock t, in (v, k) order,
// reported on the reference's iteration clock (until - base); the per-vertex caches are checked against it.
template <int W>
__device__ void probe_dump(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, const TabuRec* rec,
                           const uint32_t* until, uint32_t base, uint32_t t, int q, int lane) {
    const int nv = g.nv, w1 = g.n + 1;
    int32_t* gam = a.probe.gamma + (size_t)q * nv * w1;
    for (int v = lane; v < nv; v += 32) {
        const uint16_t rc = g.cell[v];
        const int r = rc >> 8, c = rc & 0xFF;
        const int kv = col_of<W>(g, s, v);
        int same = 0;
        if (kv) {
            for (int u = g.rs[r]; u < g.rs[r + 1]; ++u) same += u != v && col_of<W>(g, s, u) == kv;
            for (int x = g.cs[c]; x < g.cs[c + 1]; ++x) same += g.cl[x] != v && col_of<W>(g, s, g.cl[x]) == kv;
        }
        gam[(size_t)v * w1] = 0;
        for (int k = 1; k <= g.n; ++k) {
            const int inr = (int)((s.R[r * W + (k >> 6)] >> (k & 63)) & 1);
            const int inc = (int)((s.C[c * W + (k >> 6)] >> (k & 63)) & 1);
            gam[(size_t)v * w1 + k] = k == kv ? same : inr + inc;
        }
    }
    int32_t* tb = a.probe.tabu + (size_t)q * a.probe.cap * 3;
    int total = 0, mism = 0;
    for (int v0 = 0; v0 < nv; v0 += 32) {
        const int v = v0 + lane;
        // the kernel's effective tabu view: a non-overflowed cache is exact on its own; an overflowed one
        // defers to the dense table (which k_improve writes only then)
        uint64_t live[W];
#pragma unroll
        for (int z = 0; z < W; ++z) live[z] = 0;
        uint32_t lu[2] = {0, 0};
        int lk[2] = {0, 0};
        bool dense_view = false;
        if (v < nv) {
            const TabuRec tr = rec[v];
            dense_view = (tr.kk >> 16) != 0;
            if (!dense_view) {
                lk[0] = tr.kk & 0xFF;
                lk[1] = (tr.kk >> 8) & 0xFF;
                lu[0] = tr.u1;
                lu[1] = tr.u2;
                for (int z = 0; z < 2; ++z)
                    if (lu[z] > t) live[lk[z] >> 6] |= 1ULL << (lk[z] & 63);
                mism += (lu[0] > t && lu[1] > t && lk[0] == lk[1]);  // a colour cached twice
            } else {
                for (int k = 1; k <= g.n; ++k)
                    if (until[(size_t)v * w1 + k] > t) live[k >> 6] |= 1ULL << (k & 63);
            }
        }
        int nl = 0;
#pragma unroll
        for (int z = 0; z < W; ++z) nl += __popcll(live[z]);
        const int incl = warp_incl_sum(nl);
        int at = total + incl - nl;
        if (v < nv)
            for (int k = 1; k <= g.n; ++k)
                if ((live[k >> 6] >> (k & 63)) & 1) {
                    const uint32_t u = dense_view ? until[(size_t)v * w1 + k] : (k == lk[0] && lu[0] > t ? lu[0] : lu[1]);
                    if (at < a.probe.cap) {
                        tb[3 * at] = v;
                        tb[3 * at + 1] = k;
                        tb[3 * at + 2] = (int32_t)(u - base);
                    }
                    ++at;
                }
        total += __shfl_sync(kFull, incl, 31);
    }
    mism = (int)__reduce_add_sync(kFull, (unsigned)mism);
    if (lane == 0) {
        a.probe.n_tabu[q] = total;
        *a.probe.dumped = q + 1;
        *a.probe.mismatch += mism;
    }
    __syncwarp();
}

// Shared by the PartialCol kernels (improve.cu canonical policy, improve_ref.cu reference policy):
// load offspring i, reset the slot's tabu caches, K1 conflict counts (coloring.hpp:105-116), K1b greedy
// repair (partial.hpp:22-39), occupancy masks R/C, uncoloured bitmask U and the column-major copy.
// Returns f after the repair.
template <int W>
__device__ int partial_prologue(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                                uint8_t* conf, int i, int lane) {
    const int n = g.n, nv = g.nv;
    const int B = 32 * g.lane_words;
    const int v_lo = lane * B;
    const int v_hi = min(nv, v_lo + B);
    uint8_t* col = s.col;
    uint8_t* colT = s.colT;
    // ---- load the offspring (u8, row stride nvpad) and reset this slot's tabu caches
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.offspring + (size_t)i * g.nvpad);
        uint4* d4 = reinterpret_cast<uint4*>(col);
        for (int x = lane; x < g.nvpad / 16; x += 32) d4[x] = src[x];
        const TabuRec z{0, 0, 0, 0};
        for (int x = lane; x < nv; x += 32) rec[x] = z;
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
            for (int x = g.cs[c]; x < g.cs[c + 1]; ++x) cnt += col[g.cl[x]] == k;
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
        for (int x = g.cs[c] + lane; x < g.cs[c + 1]; x += 32) {
            const int u = g.cl[x];
            if (u != w && col[u] == k) conf[u] -= 1;
        }
        __syncwarp();
        if (lane == 0) {
            col[w] = 0;
            conf[w] = 0;
        }
        __syncwarp();
    }

    // ---- occupancy masks R/C, uncoloured bitmask U and the column-major copy
    for (int x = lane; x < n * W; x += 32) {
        s.R[x] = 0;
        s.C[x] = 0;
    }
    __syncwarp();
    int fl = 0;
    for (int q = 0; q < g.lane_words; ++q) {
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
        s.U[lane * g.lane_words + q] = bits;
        fl += __popc(bits);
    }
    for (int x = lane; x < nv; x += 32) colT[x] = col[g.cl[x]];
    int f = (int)__reduce_add_sync(kFull, (unsigned)fl);
    __syncwarp();
    return f;
}

}  // namespace plse_dev
