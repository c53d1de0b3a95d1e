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
//   * Sparse mode (|V0| <= 31, i.e. everything after the first ~1% of the
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

// ============================================================ padded colour layout helpers
// s.col is the ROW-PADDED copy (row r at rinfo[r] & 0xFFFF, on an 8-byte boundary, its cells in vertex
// order, 0xFF up to the next row), s.colT the COLUMN-PADDED copy (column c in column-list order).  Pad bytes
// are 0xFF, never a colour, and are written once per warp; only real cells are ever stored.

__device__ __forceinline__ uint64_t zero_bytes64(uint64_t x) {  // 0x80 in every byte of x that is 0
    return ~(((x & 0x7F7F7F7F7F7F7F7FULL) + 0x7F7F7F7F7F7F7F7FULL) | x) & 0x8080808080808080ULL;
}

// the row holder ur and the column holder uc of colour k in the row / column of v* (partial.hpp:124-135:
// the neighbours coloured k*; at most one each since the colouring is legal), -1 if none: lanes 0-15 load
// the row's 8-byte words, lanes 16-31 the column's, one ballot answers both (n <= 127: <= 16 words each)
template <int W>
__device__ __forceinline__ void holders(const Graph<W>& g, const WarpSmem& s, int ks, int rs_, int cs_, int lane,
                                        int& ur, int& uc) {
    const bool colhalf = lane >= 16;
    const int l16 = lane & 15;
    // one table for both halves: rinfo[0, n) rows, rinfo[n, 2n) columns (their offsets already include the
    // row-padded copy's size, so both halves address s.col)
    const uint64_t info = g.rinfo[colhalf ? g.n + cs_ : rs_];
    const int off = (int)(info & 0xFFFFu), nw = (int)((info >> 16) & 0xFFFFu), vb = (int)(info >> 32);
    // every lane loads a word of its line (clamped into it) and drops the hit if past the end; the line holds k
    // at most once (legal colouring), so a lane sees at most one zero byte
    const uint2 w = *reinterpret_cast<const uint2*>(s.col + off + 8 * min(l16, nw - 1));
    const uint32_t k4 = (uint32_t)ks * 0x01010101u;
    const uint32_t live = l16 < nw ? 0x80808080u : 0u;
    const uint32_t xl = w.x ^ k4, xh = w.y ^ k4;
    const uint32_t zl = ~(((xl & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | xl) & live;
    const uint32_t zh = ~(((xh & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | xh) & live;
    const unsigned bal = __ballot_sync(kFull, (zl | zh) != 0);
    // byte of the single hit: the leading one of its half sits at bit 8b + 7
    const uint32_t zz = zl ? zl : zh;
    const int idx = 8 * l16 + (zl ? 0 : 4) + ((31 - __clz(zz)) >> 3);
    int cand = vb + idx;
    if (colhalf) cand = g.cl[cand];
    const int lr = __ffs(bal & 0xFFFFu) - 1, lc = __ffs(bal >> 16) - 1;
    const int a_ = __shfl_sync(kFull, cand, lr & 31);
    const int b_ = __shfl_sync(kFull, cand, (lc + 16) & 31);
    ur = lr >= 0 ? a_ : -1;
    uc = lc >= 0 ? b_ : -1;
}

// number of bytes equal to k (1 <= k <= n) in a row / column window
__device__ __forceinline__ int count_eq(const uint8_t* buf, uint64_t info, int k) {
    const int off = (int)(info & 0xFFFFu), nw = (int)((info >> 16) & 0xFFFFu);
    const uint64_t k8 = (uint64_t)k * 0x0101010101010101ULL;
    int cnt = 0;
    for (int q = 0; q < nw; ++q) cnt += __popcll(zero_bytes64(*reinterpret_cast<const uint64_t*>(buf + off + 8 * q) ^ k8));
    return cnt;
}

// the vertex-ordered u8 row (stride nvpad, zero pad) of the current colouring, 4 bytes per lane store
template <int W>
__device__ __forceinline__ void pad_snapshot(const Graph<W>& g, const WarpSmem& s, uint8_t* dst, int lane) {
    for (int b = 4 * lane; b < g.nvpad; b += 128) {
        uint32_t w = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (b + q < g.nv) w |= (uint32_t)s.col[g.rpos[b + q]] << (8 * q);
        *reinterpret_cast<uint32_t*>(dst + b) = w;
    }
}

// the uncoloured bitmask U from the colours (sparse mode does not maintain it)
template <int W>
__device__ __forceinline__ int rebuild_U(const Graph<W>& g, const WarpSmem& s, int lane) {
    const int v_lo = lane * 32 * g.lane_words;
    int fl = 0;
    for (int q = 0; q < g.lane_words; ++q) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            const int v = v_lo + 32 * q + b;
            if (v < g.nv && s.col[g.rpos[v]] == 0) bits |= 1u << b;
        }
        s.U[lane * g.lane_words + q] = bits;
        fl += __popc(bits);
    }
    __syncwarp();
    return fl;
}

// partial_prologue (improve_common.cuh) on the padded layout: load offspring i, reset the slot's tabu caches,
// K1 conflict counts (coloring.hpp:105-116), K1b greedy repair with lowest-index ties (partial.hpp:22-39),
// occupancy masks R / C and the uncoloured bitmask U.  Returns f after the repair.
template <int W>
__device__ int pad_prologue(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, TabuRec* rec, uint8_t* conf,
                            int i, int lane) {
    const int n = g.n, nv = g.nv;
    const int B = 32 * g.lane_words;
    const int v_lo = lane * B;
    const int v_hi = min(nv, v_lo + B);
    {
        const uint8_t* src = a.offspring + (size_t)i * g.nvpad;
        for (int v = lane; v < nv; v += 32) {
            const uint8_t k = src[v];
            s.col[g.rpos[v]] = k;
            s.colT[g.colpos[v]] = k;
        }
        const TabuRec z{0, 0, 0, 0};
        for (int x = lane; x < nv; x += 32) rec[x] = z;
    }
    __syncwarp();
    // ---- K1: gamma[v][col v] of the coloured vertices: equal bytes in v's row and column windows, minus v
    for (int v = v_lo; v < v_hi; ++v) {
        const int k = s.col[g.rpos[v]];
        int cnt = 0;
        if (k) {
            const uint16_t rc = g.cell[v];
            cnt = count_eq(s.col, g.rinfo[rc >> 8], k) + count_eq(s.col, g.cinfo[rc & 0xFF], k) - 2;
        }
        conf[v] = (uint8_t)cnt;
    }
    __syncwarp();
    // ---- K1b: uncolour argmax conflicts (strict >, lowest index) until none (partial.hpp:22-39)
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
        const uint16_t rc = g.cell[w];
        const int r = rc >> 8, c = rc & 0xFF;
        const int k = s.col[g.rpos[w]];
        const uint64_t ri = g.rinfo[r], ci = g.cinfo[c];
        const int roff = (int)(ri & 0xFFFFu), rv0 = (int)(ri >> 32);
        const int coff = (int)(ci & 0xFFFFu), cb = (int)(ci >> 32);
        for (int x = lane; x < g.rs[r + 1] - g.rs[r]; x += 32)
            if (rv0 + x != w && s.col[roff + x] == k) conf[rv0 + x] -= 1;
        for (int x = lane; x < g.cs[c + 1] - g.cs[c]; x += 32) {
            const int u = g.cl[cb + x];
            if (u != w && s.col[coff + x] == k) conf[u] -= 1;
        }
        __syncwarp();
        if (lane == 0) {
            s.col[g.rpos[w]] = 0;
            s.colT[g.colpos[w]] = 0;
            conf[w] = 0;
        }
        __syncwarp();
    }
    // ---- occupancy masks R / C and the uncoloured bitmask U
    for (int x = lane; x < (n + 1) * W; x += 32) {
        s.R[x] = 0;
        s.C[x] = 0;
    }
    __syncwarp();
    for (int v = lane; v < nv; v += 32) {
        const int k = s.col[g.rpos[v]];
        if (k) {
            const uint16_t rc = g.cell[v];
            atomicOr((unsigned long long*)&s.R[(rc >> 8) * W + (k >> 6)], 1ULL << (k & 63));
            atomicOr((unsigned long long*)&s.C[(rc & 0xFF) * W + (k >> 6)], 1ULL << (k & 63));
        }
    }
    const int fl = rebuild_U<W>(g, s, lane);
    return (int)__reduce_add_sync(kFull, (unsigned)fl);
}

// apply_move_lanes (improve_common.cuh) on the padded layout: lanes 0-2 store the colour byte of v*, ur, uc
// in both copies (and, in dense mode, flip their U bits); lane 1 clears k* from C[col ur], lane 2 from
// R[row uc]; lane 3 sets it in R[row v*] unless ur held it, lane 4 in C[col v*] unless uc did; lanes 1/2
// forbid (evictee, k*) until ut (search_util.hpp:73-75) and return the evictee's updated tabu cache.
template <int W, bool kDense>
__device__ __forceinline__ TabuRec apply_move_pad(const Graph<W>& g, const WarpSmem& s, TabuRec* rec, uint32_t* until,
                                                  int vs, int ur, int uc, int ks, bool inR, bool inC, int f_before,
                                                  bool improved, uint32_t ut, uint32_t t, int lane,
                                                  uint32_t& acc) {
    const int w1 = g.n + 1, kw = ks >> 6;
    const uint64_t bitk = 1ULL << (ks & 63);
    const bool l1 = lane == 1, l2 = lane == 2;
    const int u = l1 ? ur : l2 ? uc : vs;
    const bool act = lane < 3 && u >= 0;
    const int uu = max(u, 0);
    TabuRec nr = rec[uu];  // issued early, consumed after the updates (lanes 1/2 only)
    const uint16_t cu = g.cell[uu];
    const int rpp = g.rpos[uu], cpp = g.colpos[uu];
    const uint32_t dg = g.deg[uu];
    __syncwarp();
    const uint8_t nc = lane == 0 ? (uint8_t)ks : (uint8_t)0;
    if (act) {
        s.col[rpp] = nc;
        s.colT[cpp] = nc;
        if (kDense) atomicXor(&s.U[uu >> 5], 1u << (uu & 31));
    }
    const bool on_c = l1 || lane == 4;
    const int line_no = on_c ? (cu & 0xFF) : (cu >> 8);
    const bool lx = ((lane == 3) & !inR) | ((lane == 4) & !inC) | ((l1 | l2) & act);
    uint64_t* line = (on_c ? s.C : s.R) + line_no * W + kw;
    if (lx) *line ^= bitk;
    acc += (act ? 4u * dg + 2u : 0u) +
           (lane == 0 ? 2u * (uint32_t)w1 * (uint32_t)f_before + (improved ? 2u * (uint32_t)g.nv : 0u) : 0u);
    if (act && lane > 0) {
        // the dense until[][] row is only read while the vertex's cache is overflowed (three or more live
        // colours), so it is only written then: the new entry while overflowed, plus the two cached pairs at
        // the moment the cache overflows.  Colours outside a non-overflowed cache hold untils <= t there.
        const uint32_t kk0 = nr.kk, u10 = nr.u1, u20 = nr.u2;
        cache_forbid_nb(nr, ks, ut, t);
        if (nr.kk >> 16) {
            uint32_t* row = until + (size_t)uu * w1;
            row[ks] = ut;
            if (!(kk0 >> 16)) {
                row[kk0 & 0xFF] = u10;
                row[(kk0 >> 8) & 0xFF] = u20;
            }
        }
        rec[uu] = nr;
    }
    return nr;
}

template <int W, bool kDebug>
__device__ void improve_one(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, TabuRec* rec,
                            uint32_t* until, uint32_t* slot_clock, uint8_t* conf, int i, int lane) {
    const int n = g.n, nv = g.nv, w1 = n + 1;
    const int B = 32 * g.lane_words;
    const int v_lo = lane * B;
    const int v_hi = min(nv, v_lo + B);
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

    int f = pad_prologue<W>(a, g, s, rec, conf, i, lane);
    __syncwarp();

    const long long t_prologue = prof ? clock64() - t_start : 0;
    const int repaired_f = f;
    int bestf = f;
    bool pending = true;  // best_ == current (partial.hpp:84)
    uint32_t j = 0;
    // SURVEY 8(d) algorithmic bytes: lane 0 accounts the scan, v*'s RMW and the
    // snapshots, lanes 1/2 the evictees' RMW; summed over the warp at the end.
    // 32-bit partial byte counts (lanes 0-2), flushed into a.bytes[i] every 64 steps
    uint32_t acc = 0;
    if (lane == 0) a.bytes[i] = 0;
    __syncwarp();
    auto flush_bytes = [&]() {
        if (lane < 3 && acc) atomicAdd(a.bytes + i, (unsigned long long)acc);
        acc = 0;
    };
    // canonical draws, 32 steps per refill (CanonDraws in common.cuh, with the seed parked in shared memory
    // and a 32-bit window to spare registers)
    if (lane == 0) *s.seed = derive_seed(a.master, 2, a.generation * a.p_total + a.offset + (uint64_t)i);
    __syncwarp();
    uint32_t dwin = 1u, dhi = 0, dlo = 0;  // window 1: no 32-step window yet
    auto draw = [&](uint32_t jj, uint32_t& h1, uint32_t& h2) {
        const uint32_t w = jj & ~31u;
        if (w != dwin) {  // warp-uniform
            const uint64_t z = canon_draw(*s.seed, (uint64_t)w + (uint64_t)lane);
            dhi = (uint32_t)(z >> 32);
            dlo = (uint32_t)z;
            dwin = w;
        }
        h1 = __shfl_sync(kFull, dhi, jj & 31);
        h2 = __shfl_sync(kFull, dlo, jj & 31);
    };
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
    const int budget = (int)a.budget;  // < 2^30 (plse_create)
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

    // every 64 steps: flush the byte counts, poll the race flag / deadline
    auto poll64 = [&](uint32_t jj) -> bool {
        flush_bytes();
        return poll_stop(jj);
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
        if (!((int)j < budget && bestf > stop_f && f > 0)) break;
        if ((j & 63) == 0 && poll64(j)) break;
        if (kDebug) probe_at(j);
        const int f_before = f;
        const bool asp = (f == bestf);
        const uint32_t t = base + j;
        uint32_t h1, h2;
        draw(j, h1, h2);
        if (f > 31) {  // sparse mode holds at most 31 so lane 31 is always an empty slot
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
                if (lane == 0) acc += 2u * (unsigned)w1 * (unsigned)f;
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
                pad_snapshot<W>(g, s, a.improved + (size_t)i * g.nvpad, lane);
                pending = false;
            }
            const uint16_t rcs = g.cell[vs];
            const int rs_ = rcs >> 8, cs_ = rcs & 0xFF;
            int ur, uc;
            holders<W>(g, s, ks, rs_, cs_, lane, ur, uc);
            const bool inR = ur >= 0, inC = uc >= 0;
            const int e = (ur >= 0) + (uc >= 0);
            const int f_new = f - 1 + e;
            const uint32_t tenure = __umulhi(h2, 10u) + (uint32_t)(alpha * (double)f_new);
            const uint32_t ut = t + 1 + tenure;
            const bool improved = f_new < bestf;
            apply_move_pad<W, true>(g, s, rec, until, vs, ur, uc, ks, inR, inC, f_before, improved, ut, t, lane, acc);
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

        // ================================================== sparse phase (|V0| <= 31)
        if (prof) ++pn_enter;
        // lane l takes the l-th uncoloured vertex (ascending v) with its tabu cache
        // an empty lane holds the dummy vertex 0xFFFF on the dummy line n: empty domain, no candidates
        const uint32_t kEmpty = 0xFFFFu | ((uint32_t)n << 16) | ((uint32_t)n << 24);
        uint32_t svc = kEmpty, su1 = 0, su2 = 0, skk = 0;
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
        uint32_t jnext = min((uint32_t)budget, (j + 64) & ~63u);  // next budget / poll check point
        for (;;) {
            if (prof) t_step = clock64();
            if (kDebug) probe_at(j);
            const int fb = f;
            const bool asp_s = (f == bestf);
            const uint32_t ts = base + j;
            uint32_t g1, g2;
            draw(j, g1, g2);
            // ---- score this lane's slot
            const int r = (svc >> 16) & 0xFF, c = svc >> 24;
            const bool mine = lane < f;
            uint64_t dom[W], T[W], m0[W], m1[W], m2[W];
            dom_mask<W>(g, r, c, dom);
            tabu_of<W>(su1, su2, skk, until + (size_t)(svc & 0xFFFFu) * w1, dom, ts, T);
            const uint64_t tmask = asp_s ? 0ULL : ~0ULL;
            // delta -1 / 0 masks first; the +1 class (2% of the steps at C3) only when no lane has a move at or
            // below 0 (warp-uniform branch)
            uint64_t o0 = 0, o1 = 0;
#pragma unroll
            for (int z = 0; z < W; ++z) {
                const uint64_t Rr = s.R[r * W + z], Cc = s.C[c * W + z];
                const uint64_t fr = dom[z] & ~Rr & ~Cc;
                m0[z] = fr & ~(T[z] & tmask);  // aspiration (f = best f) admits the tabu delta -1 moves
                m1[z] = dom[z] & (Rr ^ Cc) & ~T[z];
                o0 |= m0[z];
                o1 |= m1[z];
            }
            int lc = __any_sync(kFull, o0 != 0) ? 0 : __any_sync(kFull, o1 != 0) ? 1 : 2;
            uint64_t m[W];
            if (lc == 2) {
                uint64_t o2 = 0;
#pragma unroll
                for (int z = 0; z < W; ++z) {
                    m2[z] = dom[z] & s.R[r * W + z] & s.C[c * W + z] & ~T[z];
                    o2 |= m2[z];
                }
                lc = (int)__reduce_min_sync(kFull, o2 ? 2u : 3u);
#pragma unroll
                for (int z = 0; z < W; ++z) m[z] = m2[z];
            } else {
#pragma unroll
                for (int z = 0; z < W; ++z) m[z] = lc == 0 ? m0[z] : m1[z];
            }
            const int cnt = popc_w<W>(m);
            int incl = warp_incl_sum(cnt);
            const int N = __shfl_sync(kFull, incl, 31);
            if (N == 0) {
                // every candidate tabu: no move, the clock still advances (partial.hpp:121-122)
                if (lane == 0) acc += 2u * (unsigned)w1 * (unsigned)f;
                if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                    trace_step(j, -1, 0, -1, -1, 0, 0, f, f, bestf, -1, 0, 2);
                ++j;
                if (j == jnext) {
                    if (!((int)j < budget) || ((j & 63) == 0 && poll64(j))) break;
                    jnext = min((uint32_t)budget, (j + 64) & ~63u);
                }
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
                pad_snapshot<W>(g, s, a.improved + (size_t)i * g.nvpad, lane);
                pending = false;
            }
            // ---- the row / column holder of k* (at most one each: the colouring is legal)
            int ur, uc;
            holders<W>(g, s, ks, rs_, cs_, lane, ur, uc);
            const bool inR = ur >= 0, inC = uc >= 0;
            const int e = (ur >= 0) + (uc >= 0);
            const int f_new = f - 1 + e;
            const uint32_t tenure = __umulhi(g2, 10u) + (uint32_t)(alpha * (double)f_new);
            const uint32_t ut = ts + 1 + tenure;
            const bool improved = f_new < bestf;
            // ---- the move: predicated five-lane update (improve_common.cuh apply_move_lanes)
            const TabuRec nr =
                apply_move_pad<W, false>(g, s, rec, until, vs, ur, uc, ks, inR, inC, fb, improved, ut, ts, lane, acc);
            f = f_new;
            bestf = improved ? f : bestf;
            pending = pending || improved;
            if (race_flag && improved && f <= race_f && lane == 0) atomicExch(const_cast<int*>(race_flag), 1);
            if (tracing && lane == 0 && (int64_t)j < a.trace_cap)
                trace_step(j, vs, ks, ur, uc, rs_, cs_, fb, f, bestf, (int)tenure, N, lvl);
            ++j;
            if (f_new > 31) {
                __syncwarp();
                rebuild_U<W>(g, s, lane);  // sparse mode leaves U stale; dense mode scans it
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
                const int src = min(y >= wl ? y + 1 : y, 31);  // lanes past the list read the empty lane 31
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
            // the budget, the stop f and the 64-step poll only at the precomputed next check point (or after an
            // improvement, the only time best f changes)
            if (j == jnext || improved) {
                if (!((int)j < budget && bestf > stop_f)) break;
                if ((j & 63) == 0 && poll64(j)) break;
                jnext = min((uint32_t)budget, (j + 64) & ~63u);
            }
        }
    }
    if (pending) pad_snapshot<W>(g, s, a.improved + (size_t)i * g.nvpad, lane);
    flush_bytes();
    if (lane == 0) {
        a.best_f[i] = bestf;
        a.repaired_f[i] = repaired_f;
        a.iters[i] = (int64_t)j;
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
__global__ void __launch_bounds__(kPadMaxThreads, 1) k_improve(const ImproveArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int lane;  // %laneid through volatile asm: kept in a register instead of re-derived from %tid every use
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
    const int n = a.n, nv = a.nv;
    const PadSmemLayout L = pad_smem_layout(n, nv, a.lane_words, W, a.rp_bytes, a.cp_bytes);
    uint16_t* s_cell = reinterpret_cast<uint16_t*>(smem + L.cell);
    uint16_t* s_rs = reinterpret_cast<uint16_t*>(smem + L.rs);
    uint16_t* s_cs = reinterpret_cast<uint16_t*>(smem + L.cs);
    uint16_t* s_cl = reinterpret_cast<uint16_t*>(smem + L.cl);
    uint16_t* s_rpos = reinterpret_cast<uint16_t*>(smem + L.rpos);
    uint16_t* s_cpos = reinterpret_cast<uint16_t*>(smem + L.cpos);
    uint8_t* s_deg = smem + L.deg;
    uint64_t* s_ri = reinterpret_cast<uint64_t*>(smem + L.rinfo);
    uint64_t* s_ci = reinterpret_cast<uint64_t*>(smem + L.cinfo);
    uint64_t* s_pr = reinterpret_cast<uint64_t*>(smem + L.pr);
    uint64_t* s_pc = reinterpret_cast<uint64_t*>(smem + L.pc);
    for (int x = threadIdx.x; x < nv; x += blockDim.x) {
        s_cell[x] = a.cell[x];
        s_cl[x] = a.col_list[x];
        s_rpos[x] = a.rpos[x];
        s_cpos[x] = a.cpos[x];
    }
    for (int x = threadIdx.x; x <= n; x += blockDim.x) {
        s_rs[x] = a.row_start[x];
        s_cs[x] = a.col_start[x];
    }
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
        s_ri[x] = a.rinfo[x];
        s_ci[x] = a.cinfo[x] + (uint64_t)a.rp_bytes;  // column offsets relative to s.col (the copies are adjacent)
    }
    for (int x = threadIdx.x; x < (n + 1) * W; x += blockDim.x) {
        // line n: every symbol prefilled -> the empty domain of the dummy vertex held by empty slot-list lanes
        s_pr[x] = x < n * W ? a.pre_row[x] : ~0ULL;
        s_pc[x] = x < n * W ? a.pre_col[x] : ~0ULL;
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
    g.colpos = s_cpos;
    g.pr = s_pr;
    g.pc = s_pc;
    g.rpos = s_rpos;
    g.rinfo = s_ri;
    g.cinfo = s_ci;
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
    s.col = wbase + L.w_rp;
    s.conf = nullptr;
    s.colT = wbase + L.w_cp;
    s.list = reinterpret_cast<uint16_t*>(wbase + L.w_list);
    s.R = reinterpret_cast<uint64_t*>(wbase + L.w_R);
    s.C = reinterpret_cast<uint64_t*>(wbase + L.w_C);
    s.U = reinterpret_cast<uint32_t*>(wbase + L.w_U);
    s.seed = reinterpret_cast<uint64_t*>(wbase + L.w_seed);
    // the pad bytes of both copies: 0xFF, written once (only real cells are ever stored afterwards)
    for (int x = lane; x < (a.rp_bytes + a.cp_bytes) / 16; x += 32)
        reinterpret_cast<uint4*>(wbase + L.w_rp)[x] = make_uint4(~0u, ~0u, ~0u, ~0u);
    __syncwarp();

    const int slot = blockIdx.x * nwarps + warp;
    TabuRec* rec = reinterpret_cast<TabuRec*>(reinterpret_cast<char*>(a.tabu_rec) + (size_t)slot * a.rec_stride);
    uint32_t* until = a.until + (size_t)slot * a.until_stride;
    uint8_t* conf = a.conf_scratch + (size_t)slot * a.conf_stride;

    for (int i = first_individual(a.first, a.nslots, a.p, warp); i < a.p;
         i = next_individual(a.first, a.nslots, a.work_counter, lane))
        improve_one<W, kDebug>(a, g, s, rec, until, a.slot_clock + slot, conf, i, lane);
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
