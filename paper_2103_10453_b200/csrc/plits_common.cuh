// plits_common.cuh -- bit-sliced colour-count helpers shared by the PLITS kernels
// (plits.cu: canonical tie-break; plits_ref.cu: the reference's reservoir draws).
// A state type St provides col (u8 colours), rp / cp (row / column count planes).
#pragma once
#include <climits>

#include "improve_common.cuh"

namespace plse_dev {

template <int W>
struct PlitsK {
    static constexpr int NP = 5 + W;  // count bits: counts <= n <= 63 (W = 1) or 127 (W = 2)
    static constexpr int NB = NP + 1; // bits of gamma = row count + column count
};

// count of colour k in a plane stack
template <int W, int NP>
__device__ __forceinline__ int plane_val(const uint64_t* P, int k) {
    int v = 0;
#pragma unroll
    for (int b = 0; b < NP; ++b) v |= (int)((P[b * W + (k >> 6)] >> (k & 63)) & 1ULL) << b;
    return v;
}

// mask of colours whose count is >= 2 (any plane above bit 0)
template <int W, int NP>
__device__ __forceinline__ bool plane_multi(const uint64_t* P, int k) {
    uint64_t m = 0;
#pragma unroll
    for (int b = 1; b < NP; ++b) m |= P[b * W + (k >> 6)];
    return (m >> (k & 63)) & 1ULL;
}

// S = R + C, bit-sliced (gamma of every colour against a vertex in that row / column)
template <int W, int NP>
__device__ __forceinline__ void plane_sum(const uint64_t* R, const uint64_t* C, uint64_t (&S)[NP + 1][W]) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t carry = 0;
#pragma unroll
        for (int b = 0; b < NP; ++b) {
            const uint64_t x = R[b * W + q], y = C[b * W + q], t = x ^ y;
            S[b][q] = t ^ carry;
            carry = (x & y) | (carry & t);
        }
        S[NP][q] = carry;
    }
}

// word q of a register array without dynamic indexing (W <= 2)
template <int W>
__device__ __forceinline__ uint64_t word_of(const uint64_t (&x)[W], int q) {
    return (W == 1 || q == 0) ? x[0] : x[W - 1];
}

template <int W, int NB>
__device__ __forceinline__ int sliced_val(const uint64_t (&S)[NB][W], int k) {
    int v = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b) v |= (int)((word_of<W>(S[b], k >> 6) >> (k & 63)) & 1ULL) << b;
    return v;
}

// minimum of S over a non-empty mask; sel becomes the argmin set
template <int W, int NB>
__device__ __forceinline__ int sliced_min(const uint64_t (&S)[NB][W], uint64_t (&sel)[W]) {
    int val = 0;
#pragma unroll
    for (int b = NB - 1; b >= 0; --b) {
        uint64_t z[W], any = 0;
#pragma unroll
        for (int q = 0; q < W; ++q) {
            z[q] = sel[q] & ~S[b][q];
            any |= z[q];
        }
#pragma unroll
        for (int q = 0; q < W; ++q) sel[q] = any ? z[q] : sel[q];
        val |= any ? 0 : (1 << b);
    }
    return val;
}

// m &= {k : S_k >= th}
template <int W, int NB>
__device__ __forceinline__ void sliced_ge(const uint64_t (&S)[NB][W], int th, uint64_t (&m)[W]) {
    if (th <= 0) return;
    if (th >= (1 << NB)) {
#pragma unroll
        for (int q = 0; q < W; ++q) m[q] = 0;
        return;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t lt = 0, eq = ~0ULL;
#pragma unroll
        for (int b = NB - 1; b >= 0; --b) {
            const uint64_t tb = ((th >> b) & 1) ? ~0ULL : 0ULL;
            lt |= eq & ~S[b][q] & tb;
            eq &= ~(S[b][q] ^ tb);
        }
        m[q] &= ~lt;
    }
}

// m &= {k : S_k == val}
template <int W, int NB>
__device__ __forceinline__ void sliced_eq(const uint64_t (&S)[NB][W], int val, uint64_t (&m)[W]) {
    if (val < 0 || val >= (1 << NB)) {
#pragma unroll
        for (int q = 0; q < W; ++q) m[q] = 0;
        return;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t eq = ~0ULL;
#pragma unroll
        for (int b = 0; b < NB; ++b) eq &= ~(S[b][q] ^ (((val >> b) & 1) ? ~0ULL : 0ULL));
        m[q] &= eq;
    }
}

__device__ __forceinline__ int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// one vertex's move classes: gamma planes, current-colour gamma, delta offsets, candidate mask
template <int W>
struct VertexMoves {
    static constexpr int NB = PlitsK<W>::NB;
    uint64_t S[NB][W];
    uint64_t M[W];  // colours k != col(v) of D(v) \ {0}
    int cur, dbase, d0;
};

template <int W, class St>
__device__ __forceinline__ void vertex_moves_rc(const Graph<W>& g, const St& s, int v, int rc, int wf, int wc,
                                                VertexMoves<W>& m) {
    constexpr int NP = PlitsK<W>::NP;
    const int r = rc >> 8, c = rc & 0xFF;
    plane_sum<W, NP>(s.rp + (size_t)r * NP * W, s.cp + (size_t)c * NP * W, m.S);
    m.cur = s.col[v];
    const int gcur = m.cur ? sliced_val<W, NP + 1>(m.S, m.cur) - 2 : 0;
    m.dbase = (m.cur ? 0 : -wf) - wc * gcur;  // to k != 0: delta = dbase + wc * gamma[v][k]
    m.d0 = wf - wc * gcur;                    // to 0 (coloured v only): df = +1, dc = -gamma[v][cur]
    dom_mask<W>(g, r, c, m.M);
#pragma unroll
    for (int q = 0; q < W; ++q)
        if (m.cur && (m.cur >> 6) == q) m.M[q] &= ~(1ULL << (m.cur & 63));
}

template <int W, class St>
__device__ __forceinline__ void vertex_moves(const Graph<W>& g, const St& s, int v, int wf, int wc,
                                             VertexMoves<W>& m) {
    vertex_moves_rc<W>(g, s, v, g.cell[v], wf, wc, m);
}

// one lane moves a cell of this line from colour `from` to `to`: the two single-bit ripples (-1 at
// `from`, +1 at `to`; 0 = uncoloured is not counted) computed in registers, NP x W words stored back
template <int W, int NP>
__device__ __forceinline__ void plane_move(uint64_t* P, int from, int to) {
    uint64_t x[NP][W];
#pragma unroll
    for (int b = 0; b < NP; ++b)
#pragma unroll
        for (int q = 0; q < W; ++q) x[b][q] = P[b * W + q];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        uint64_t borrow = (from && (from >> 6) == q) ? 1ULL << (from & 63) : 0ULL;
        uint64_t carry = (to && (to >> 6) == q) ? 1ULL << (to & 63) : 0ULL;
#pragma unroll
        for (int b = 0; b < NP; ++b) {
            const uint64_t old = x[b][q];
            x[b][q] = old ^ borrow;
            borrow &= ~old;
            const uint64_t mid = x[b][q];
            x[b][q] = mid ^ carry;
            carry &= mid;
        }
    }
#pragma unroll
    for (int b = 0; b < NP; ++b)
#pragma unroll
        for (int q = 0; q < W; ++q) P[b * W + q] = x[b][q];
}

template <int W, class St>
__device__ __forceinline__ bool plits_is_active(const Graph<W>& g, const St& s, int u) {
    constexpr int NP = PlitsK<W>::NP;
    const int k = s.col[u];
    if (!k) return true;
    const uint16_t rc = g.cell[u];
    return plane_multi<W, NP>(s.rp + (size_t)(rc >> 8) * NP * W, k) ||
           plane_multi<W, NP>(s.cp + (size_t)(rc & 0xFF) * NP * W, k);
}

// the row / column count planes of the colouring in s.col: lane l builds lines l, l + 32, ... in registers
template <int W, class St>
__device__ void plits_build_planes(const Graph<W>& g, const St& s, int lane) {
    constexpr int NP = PlitsK<W>::NP;
    const int n = g.n;
    for (int line = lane; line < 2 * n; line += 32) {
        const bool is_row = line < n;
        const int idx = is_row ? line : line - n;
        uint64_t P[NP][W];
#pragma unroll
        for (int b = 0; b < NP; ++b)
#pragma unroll
            for (int q = 0; q < W; ++q) P[b][q] = 0;
        const int lo = is_row ? g.rs[idx] : g.cs[idx], hi = is_row ? g.rs[idx + 1] : g.cs[idx + 1];
        for (int x = lo; x < hi; ++x) {
            const int k = s.col[is_row ? x : g.cl[x]];
            if (!k) continue;
#pragma unroll
            for (int q = 0; q < W; ++q) {
                uint64_t carry = (k >> 6) == q ? 1ULL << (k & 63) : 0ULL;
#pragma unroll
                for (int b = 0; b < NP; ++b) {
                    const uint64_t t = P[b][q] & carry;
                    P[b][q] ^= carry;
                    carry = t;
                }
            }
        }
        uint64_t* dst = (is_row ? s.rp : s.cp) + (size_t)idx * NP * W;
#pragma unroll
        for (int b = 0; b < NP; ++b)
#pragma unroll
            for (int q = 0; q < W; ++q) dst[b * W + q] = P[b][q];
    }
    __syncwarp();
}

}  // namespace plse_dev
