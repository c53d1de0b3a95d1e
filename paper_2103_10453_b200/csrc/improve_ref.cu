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

namespace plse_dev {

// rng.hpp:43-49 next_below(bound): rejection below (2^64 - bound) % bound (< bound), then x % bound
__device__ __forceinline__ uint64_t ref_below(Xoshiro& rng, uint64_t bound) {
    for (;;) {
        const uint64_t x = rng.next();
        if (x >= bound || x >= (0 - bound) % bound) return x % bound;
    }
}

// next_below(bound) == 0 without a 64-bit division: x accepted (x >= bound, or x >= the rejection
// threshold, which is < bound), then bound | x <=> the odd part o of bound divides x >> s (s = its
// trailing zeros) and the low s bits of x are 0; o | y <=> y * o^-1 (mod 2^64) times o does not overflow
__device__ __forceinline__ bool ref_below_is_zero(Xoshiro& rng, uint64_t bound) {
    for (;;) {
        const uint64_t x = rng.next();
        if (x < bound && x < (0 - bound) % bound) continue;  // rejected (probability < bound / 2^64)
        const int sh = __ffsll((long long)bound) - 1;
        if (x & ((1ULL << sh) - 1)) return false;
        const uint64_t o = bound >> sh, y = x >> sh;
        uint64_t inv = o;  // Newton: o * inv == 1 (mod 2^64), 3 -> 6 -> 12 -> 24 -> 48 -> 96 correct bits
#pragma unroll
        for (int it = 0; it < 5; ++it) inv *= 2 - o * inv;
        return __umul64hi(y * inv, o) == 0;
    }
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

template <int W, bool kDebug>
__device__ void improve_ref_one(const ImproveArgs& a, const Graph<W>& g, const WarpSmem& s, uint16_t* el,
                                uint64_t* msk, TabuRec* rec, uint32_t* until, uint32_t* slot_clock, uint8_t* conf, int i,
                                int lane) {
    const int nv = g.nv, w1 = g.n + 1;
    uint8_t* col = s.col;
    uint8_t* colT = s.colT;
    const bool tracing = kDebug && (i == a.trace_idx) && a.trace != nullptr;
    unsigned long long* prof = kDebug ? a.prof : nullptr;
    unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};  // steps, mask cycles, walk cycles, apply cycles, draws, sum f
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
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int x = __shfl_up_sync(kFull, incl, d);
            incl += lane >= d ? x : 0;
        }
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

        // ---- the reservoir scan (partial.hpp:100-119): masks in parallel, draws serially on lane 0
        RefScan st{0, 2, -1, 0, -1, 0};
        if (prof) {
            tq = clock64();
            ++pc[0];
            pc[5] += (unsigned)f;
        }
        for (int c0 = 0; c0 < f; c0 += 32) {
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
        if (lane < 3) {
            const int u = lane == 0 ? vs : lane == 1 ? ur : uc;
            if (u >= 0) {
                const uint8_t nc = lane == 0 ? (uint8_t)ks : (uint8_t)0;
                col[u] = nc;
                colT[g.colpos[u]] = nc;
                atomicXor(&s.U[u >> 5], 1u << (u & 31));
                acc += lane == 0 ? 2ULL * (unsigned)w1 * (unsigned)f_before + 4ULL * g.deg[vs] + 2ULL +
                                       (improved ? 2ULL * (unsigned)nv : 0ULL)
                                 : 4ULL * g.deg[u] + 2ULL;
                if (lane > 0) {
                    until[(size_t)u * w1 + ks] = ut;
                    TabuRec nr = rec[u];
                    cache_forbid(nr, ks, ut, t);
                    rec[u] = nr;
                    if (lane == 1)
                        s.C[(g.cell[u] & 0xFF) * W + kw] &= ~bitk;  // row holder leaves its column
                    else
                        s.R[(g.cell[u] >> 8) * W + kw] &= ~bitk;    // column holder leaves its row
                } else {
                    s.R[rs_ * W + kw] |= bitk;
                    s.C[cs_ * W + kw] |= bitk;
                }
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
            for (int z = 0; z < 6; ++z) atomicAdd(prof + z, pc[z]);
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
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(a.work_counter, 1);
        i = __shfl_sync(kFull, i, 0);
        if (i >= a.p) break;
        improve_ref_one<W, kDebug>(a, g, s, el, msk, rec, until, a.slot_clock + slot, conf, i, lane);
    }
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
