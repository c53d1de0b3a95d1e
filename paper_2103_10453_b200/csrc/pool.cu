// pool.cu -- K4a: update_population (population.hpp:103-183) entirely on the
// device, plus the device-side best tracking of the improve phase
// (engine.hpp:211-217) and the elite export of the island exchange.
//
// Pool ids: 0..p-1 current members, p..2p-1 improved, 2p..2p+m-1 migrants of
// the island exchange (migrants enter the next pool as extra
// candidates; m = 0 is the reference's update exactly).
//
//   k_pool_keys      key = bin << 32 | id, bin = illegal * (|V|+1) + f
//   k_sort_keys      one-CTA stable LSD radix sort over the bin bits only (ids
//                    enter in ascending order, so ties stay ordered by id):
//                    the (illegal, f, id) order of population.hpp:121-125
//   k_pool_first     the pool best enters unconditionally (population.hpp:144)
//   k_pool_check     per block of 1024 candidates: "no admitted member within
//                    |V|/gamma" (early exit) + the in-block conflict rows
//   k_pool_resolve   one warp walks the block in pool order with the conflict
//                    rows staged in shared memory (population.hpp:144-156)
//   k_pool_shortfall skipped candidates fill the remaining slots in pool order
//                    (population.hpp:157-160)
//   k_pool_gather_*  next members, next dist, next f / c
// Every kernel reads the running selection count from device memory, so the
// whole update is enqueued without a host round trip.
#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

__device__ __forceinline__ uint32_t pool_dist(const PoolView& v, int a, int b) {
    const int p = v.p, p2 = 2 * v.p;
    if (a == b) return 0;
    if (a >= p2 || b >= p2) {  // migrant row: members | improved | migrants
        const int m = a >= p2 ? a : b, o = a >= p2 ? b : a;
        return v.migd[(size_t)(m - p2) * (p2 + v.m) + o];
    }
    if (a < p && b < p) return v.dist[(size_t)a * p + b];
    if (a >= p && b >= p) {  // fresh holds its upper triangle (population.hpp:76-87 mirrors it)
        const int x = min(a, b) - p, y = max(a, b) - p;
        return v.fresh[(size_t)x * p + y];
    }
    return a < p ? v.cross[(size_t)a * p + (b - p)] : v.cross[(size_t)b * p + (a - p)];
}

__device__ __forceinline__ void pool_fc(const PoolFC& s, int id, int& f, int& c) {
    if (id < s.p) {
        f = s.mf[id];
        c = s.mc[id];
    } else if (id < 2 * s.p) {
        f = s.imf[id - s.p];
        c = s.imc[id - s.p];
    } else {
        f = s.gf[id - 2 * s.p];
        c = s.gc[id - 2 * s.p];
    }
}

__global__ void k_pool_keys(const PoolFC s, int nv, int P, uint64_t* keys, uint8_t* legal) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= P) return;
    int f, c;
    pool_fc(s, id, f, c);
    const uint32_t bin = (c != 0 ? (uint32_t)(nv + 1) : 0u) + (uint32_t)f;
    keys[id] = (uint64_t)bin << 32 | (uint32_t)id;
    legal[id] = c == 0;
}

// One CTA, 32 warps; warp w owns the contiguous key segment w (stability: segments in order, lanes in
// order inside a 32-key chunk).  Each pass: per-warp digit histograms -> digit-major / warp-minor
// exclusive offsets -> stable scatter with __match_any_sync ranks.  order[x] = id of the x-th key.
constexpr int kSortThreads = 1024;

__global__ void __launch_bounds__(kSortThreads) k_sort_keys(uint64_t* a, uint64_t* b, int N, int passes,
                                                             int32_t* order) {
    __shared__ uint32_t hist[32][257];
    __shared__ uint32_t tot[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = (N + 31) / 32;
    const int lo = min(N, warp * seg), hi = min(N, lo + seg);
    uint64_t* src = a;
    uint64_t* dst = b;
    for (int pass = 0; pass < passes; ++pass) {
        const int sh = 32 + 8 * pass;
        for (int t = threadIdx.x; t < 32 * 257; t += kSortThreads) (&hist[0][0])[t] = 0;
        __syncthreads();
        for (int x = lo + lane; x < hi; x += 32) atomicAdd(&hist[warp][(uint32_t)(src[x] >> sh) & 255u], 1u);
        __syncthreads();
        if (threadIdx.x < 256) {
            const int d = threadIdx.x;
            uint32_t s = 0;
            for (int w = 0; w < 32; ++w) {
                const uint32_t c = hist[w][d];
                hist[w][d] = s;
                s += c;
            }
            tot[d] = s;
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t v[8], s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q] = tot[lane * 8 + q];
                s += v[q];
            }
            uint32_t inc = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t run = inc - s;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                tot[lane * 8 + q] = run;
                run += v[q];
            }
        }
        __syncthreads();
        if (threadIdx.x < 256)
            for (int w = 0; w < 32; ++w) hist[w][threadIdx.x] += tot[threadIdx.x];
        __syncthreads();
        for (int base = lo; base < hi; base += 32) {
            const int x = base + lane;
            const bool valid = x < hi;
            const uint64_t k = valid ? src[x] : 0;
            const uint32_t d = valid ? ((uint32_t)(k >> sh) & 255u) : 256u + (uint32_t)lane;
            const uint32_t peers = __match_any_sync(kFull, d);
            const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            if (valid) dst[hist[warp][d] + rank] = k;
            __syncwarp();
            if (valid && rank == 0) hist[warp][d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    for (int x = threadIdx.x; x < N; x += kSortThreads) order[x] = (int32_t)(uint32_t)src[x];
}

// population.hpp:140-145: info.pool_best_f, and the pool best enters first
__global__ void k_pool_first(const PoolFC s, const int32_t* order, int32_t* sel, int32_t* nsel, uint8_t* admitted,
                             int32_t* info) {
    int f, c;
    pool_fc(s, order[0], f, c);
    sel[0] = order[0];
    *nsel = 1;
    admitted[0] = 1;
    info[0] = f;  // pool_best_f
    info[1] = 0;  // shortfall count
}

// One CTA per candidate of the block [blk_lo, blk_lo + blk_n) of pool positions.
__global__ void k_pool_check(const PoolView pv, const int32_t* order, int blk_lo, int blk_n, const int32_t* sel,
                             const int32_t* nsel, int p, int dthr, const uint8_t* legal, uint8_t* ok,
                             uint32_t* conflict, int cwords) {
    const int ns = *nsel;
    if (ns >= p) return;
    const int t = blockIdx.x;
    const int c = order[blk_lo + t];
    __shared__ int found;
    if (threadIdx.x == 0) found = !legal[c];
    __syncthreads();
    if (!found) {
        // min over the admitted set > |V|/gamma  <=>  no admitted s with d(c, s) <= floor(|V|/gamma)
        for (int q = threadIdx.x; q < ns; q += blockDim.x) {
            if (*(volatile int*)&found) break;
            if ((int)pool_dist(pv, c, sel[q]) <= dthr) {
                found = 1;
                break;
            }
        }
    }
    __syncthreads();
    const bool good = !found;
    if (threadIdx.x == 0) ok[t] = good;
    if (!good) return;  // never admitted: its conflict row is never read
    for (int base = 0; base < cwords * 32; base += blockDim.x) {
        const int u = base + threadIdx.x;
        bool hit = false;
        if (u > t && u < blk_n) {
            const int cu = order[blk_lo + u];
            hit = legal[cu] && (int)pool_dist(pv, c, cu) <= dthr;
        }
        const unsigned bal = __ballot_sync(kFull, hit);
        if ((threadIdx.x & 31) == 0 && (u >> 5) < cwords) conflict[(size_t)t * cwords + (u >> 5)] = bal;
    }
}

constexpr int kPoolBlock = 1024;

// The greedy of population.hpp:144-156 over one block: warp 0 walks the candidates that passed the check in
// pool order; lane l holds word l of the "within |V|/gamma of a candidate admitted in this block" mask.
__global__ void __launch_bounds__(kPoolBlock) k_pool_resolve(const int32_t* order, int blk_lo, int blk_n,
                                                             const uint8_t* ok, const uint32_t* conflict, int cwords,
                                                             int32_t* sel, int32_t* nsel, int p, uint8_t* admitted) {
    extern __shared__ uint32_t s_conf[];  // [blk_n][cwords]
    __shared__ uint32_t s_ok[32];
    int ns = *nsel;
    if (ns >= p) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        const int t = threadIdx.x;
        const bool g = t < blk_n && ok[t];
        const unsigned bal = __ballot_sync(kFull, g);
        if (lane == 0) s_ok[warp] = bal;
        for (int t2 = threadIdx.x; t2 < blk_n * cwords; t2 += blockDim.x) {
            // rows of failed candidates were not written: never read below
            const int row = t2 / cwords;
            if (ok[row]) s_conf[t2] = conflict[t2];
        }
    }
    __syncthreads();
    if (warp != 0) return;
    // 32 candidates (one word) at a time: lane j holds the within-word part of candidate j's conflict row
    // (later candidates of the word within |V|/gamma of it), so the greedy in pool order only visits the
    // candidates still available -- the lowest one is admitted and knocks out its later conflicts -- with
    // no shared-memory round trip per candidate; the admitted rows then update the words of the later
    // candidates in one pass (independent loads).
    uint32_t blocked = 0;  // lane l: word l of "within |V|/gamma of a candidate admitted in this block"
    for (int wi = 0; wi < cwords && ns < p; ++wi) {
        const uint32_t okw = s_ok[wi];
        const int t = wi * 32 + lane;
        const uint32_t R = ((okw >> lane) & 1u) ? s_conf[t * cwords + wi] : 0u;
        uint32_t avail = okw & ~__shfl_sync(kFull, blocked, wi);
        uint32_t A = 0;
        while (avail) {
            const int b = __ffs(avail) - 1;
            A |= 1u << b;
            avail &= ~__shfl_sync(kFull, R, b) & (avail - 1);  // drop b and the later ones it conflicts with
        }
        // admission stops at p members (population.hpp:146): keep the first p - ns in pool order
        const int room = p - ns;
        if (__popc(A) > room) {
            uint32_t keep = 0, x = A;
            for (int k = 0; k < room; ++k) {
                keep |= x & (0u - x);
                x &= x - 1;
            }
            A = keep;
        }
        if ((A >> lane) & 1u) {
            sel[ns + __popc(A & ((1u << lane) - 1u))] = order[blk_lo + t];
            admitted[blk_lo + t] = 1;
        }
        ns += __popc(A);
        if (lane < cwords) {
            uint32_t x = A;
            while (x) {
                const int b = __ffs(x) - 1;
                x &= x - 1;
                blocked |= s_conf[(wi * 32 + b) * cwords + lane];
            }
        }
    }
    if (lane == 0) *nsel = ns;
}

// population.hpp:157-160: skipped candidates (every pool position >= 1 not admitted) in pool order
__global__ void __launch_bounds__(1024) k_pool_shortfall(const int32_t* order, int P, const uint8_t* admitted,
                                                         int32_t* sel, int32_t* nsel, int p, int32_t* slots,
                                                         int32_t* info) {
    __shared__ int wsum[32];
    __shared__ int base;
    const int ns0 = *nsel;
    if (ns0 >= p) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int lo = 1; lo < P; lo += 1024) {
        const int pos = lo + threadIdx.x;
        const int fl = pos < P && !admitted[pos];
        const unsigned bal = __ballot_sync(kFull, fl);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int before = base;
        for (int w = 0; w < warp; ++w) before += wsum[w];
        const int r = before + __popc(bal & ((1u << lane) - 1u));
        if (fl && ns0 + r < p) {
            sel[ns0 + r] = order[pos];
            slots[r] = ns0 + r;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 0; w < 32; ++w) base += wsum[w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int nsf = min(base, p - ns0);
        info[1] = nsf;
        *nsel = ns0 + nsf;
    }
}

__global__ void k_pool_gather_dist(const PoolView pv, const int32_t* sel, uint16_t* next_dist) {
    const int p = pv.p;
    const int i = blockIdx.y;
    const int a = sel[i];
    for (int jj = blockIdx.x * blockDim.x + threadIdx.x; jj < p; jj += gridDim.x * blockDim.x)
        next_dist[(size_t)i * p + jj] = (uint16_t)pool_dist(pv, a, sel[jj]);
}

__global__ void k_pool_gather_rows(const int32_t* sel, int p, const uint8_t* members, const uint8_t* improved,
                                   const uint8_t* migrants, uint8_t* next_members, int nvpad) {
    const int i = blockIdx.x;
    const int a = sel[i];
    const uint8_t* s = a < p ? members + (size_t)a * nvpad
                       : a < 2 * p ? improved + (size_t)(a - p) * nvpad
                                   : migrants + (size_t)(a - 2 * p) * nvpad;
    const uint4* src = reinterpret_cast<const uint4*>(s);
    uint4* dst = reinterpret_cast<uint4*>(next_members + (size_t)i * nvpad);
    for (int t = threadIdx.x; t < nvpad / 16; t += blockDim.x) dst[t] = src[t];
}

__global__ void k_pool_gather_fc(const PoolFC s, const int32_t* sel, int32_t* nf, int32_t* nc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.p) return;
    int f, c;
    pool_fc(s, sel[i], f, c);
    nf[i] = f;
    nc[i] = c;
}

cudaError_t launch_pool_update(const PoolView& pv, const PoolFC& fc, const PoolScratch& w, int nv, int dthr,
                               const uint8_t* members, const uint8_t* improved, const uint8_t* migrants,
                               uint8_t* next_members, uint16_t* next_dist, int32_t* next_f, int32_t* next_c,
                               int nvpad, cudaStream_t st, int64_t* launches) {
    const int p = pv.p, P = 2 * p + pv.m;
    int64_t nl = 0;
    k_pool_keys<<<(P + 255) / 256, 256, 0, st>>>(fc, nv, P, w.keys0, w.legal);
    ++nl;
    const uint32_t maxbin = 2u * (uint32_t)(nv + 1);
    int bits = 1;
    while ((1u << bits) < maxbin) ++bits;
    const int passes = (bits + 7) / 8;
    k_sort_keys<<<1, kSortThreads, 0, st>>>(w.keys0, w.keys1, P, passes, w.order);
    ++nl;
    cudaError_t e = cudaMemsetAsync(w.admitted, 0, P, st);
    if (e != cudaSuccess) return e;
    k_pool_first<<<1, 1, 0, st>>>(fc, w.order, w.sel, w.nsel, w.admitted, w.info);
    ++nl;
    // The chain of blocks is launched unconditionally: once p members are admitted every later kernel
    // returns at its first instruction (the count lives in device memory).
    for (int lo = 1; lo < P; lo += kPoolBlock) {
        const int bn = min(kPoolBlock, P - lo);
        const int cw = (bn + 31) / 32;
        k_pool_check<<<bn, 256, 0, st>>>(pv, w.order, lo, bn, w.sel, w.nsel, p, dthr, w.legal, w.ok, w.conf, cw);
        k_pool_resolve<<<1, kPoolBlock, (size_t)bn * cw * 4, st>>>(w.order, lo, bn, w.ok, w.conf, cw, w.sel, w.nsel,
                                                                     p, w.admitted);
        nl += 2;
    }
    k_pool_shortfall<<<1, 1024, 0, st>>>(w.order, P, w.admitted, w.sel, w.nsel, p, w.slots, w.info);
    dim3 grid((p + 255) / 256 < 8 ? (p + 255) / 256 : 8, p);
    k_pool_gather_dist<<<grid, 256, 0, st>>>(pv, w.sel, next_dist);
    k_pool_gather_rows<<<p, 128, 0, st>>>(w.sel, p, members, improved, migrants, next_members, nvpad);
    k_pool_gather_fc<<<(p + 255) / 256, 256, 0, st>>>(fc, w.sel, next_f, next_c);
    nl += 4;
    if (launches) *launches += nl;
    return cudaGetLastError();
}

cudaError_t prepare_pool_update() {
    return cudaFuncSetAttribute(k_pool_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kPoolBlock * (kPoolBlock / 32) * 4);
}

// ---------------------------------------------------------------- best tracking (engine.hpp:211-217)
// sum of iterations and algorithmic bytes, lowest-index argmin of the improved f (strict <)
__global__ void __launch_bounds__(1024) k_best_reduce(const int32_t* best_f, const int64_t* iters,
                                                         const unsigned long long* bytes, int p,
                                                         ImproveSummary* out) {
    __shared__ unsigned long long s_it[32], s_by[32];
    __shared__ unsigned long long s_key[32];
    unsigned long long it = 0, by = 0, key = ~0ull;
    for (int i = threadIdx.x; i < p; i += blockDim.x) {
        it += (unsigned long long)iters[i];
        by += bytes[i];
        const unsigned long long k = (unsigned long long)(uint32_t)best_f[i] << 32 | (uint32_t)i;
        key = k < key ? k : key;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        it += __shfl_down_sync(kFull, it, o);
        by += __shfl_down_sync(kFull, by, o);
        const unsigned long long k2 = __shfl_down_sync(kFull, key, o);
        key = k2 < key ? k2 : key;
    }
    if (lane == 0) {
        s_it[warp] = it;
        s_by[warp] = by;
        s_key[warp] = key;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        it = lane < nw ? s_it[lane] : 0;
        by = lane < nw ? s_by[lane] : 0;
        key = lane < nw ? s_key[lane] : ~0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            it += __shfl_down_sync(kFull, it, o);
            by += __shfl_down_sync(kFull, by, o);
            const unsigned long long k2 = __shfl_down_sync(kFull, key, o);
            key = k2 < key ? k2 : key;
        }
        if (lane == 0) {
            out->iters = (int64_t)it;
            out->bytes = by;
            out->best_f = p > 0 ? (int32_t)(key >> 32) : 0;
            out->best_idx = p > 0 ? (int32_t)(uint32_t)key : -1;
        }
    }
}

cudaError_t launch_improve_reduce(const int32_t* best_f, const int64_t* iters, const unsigned long long* bytes,
                                  int p, ImproveSummary* out, cudaStream_t st) {
    k_best_reduce<<<1, 1024, 0, st>>>(best_f, iters, bytes, p, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- island export
// member slots in (illegal, f, slot) order -- the same key sort as the pool, over the p members
__global__ void k_member_keys(const int32_t* mf, const int32_t* mc, int nv, int p, uint64_t* keys) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= p) return;
    const uint32_t bin = (mc[id] != 0 ? (uint32_t)(nv + 1) : 0u) + (uint32_t)mf[id];
    keys[id] = (uint64_t)bin << 32 | (uint32_t)id;
}

__global__ void k_gather_rows_f(const int32_t* idx, int n, const uint8_t* rows, const int32_t* f, int nvpad,
                                uint8_t* out, int32_t* fout) {
    const int e = blockIdx.x;
    if (e >= n) return;
    const int a = idx[e];
    const uint4* src = reinterpret_cast<const uint4*>(rows + (size_t)a * nvpad);
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)e * nvpad);
    for (int t = threadIdx.x; t < nvpad / 16; t += blockDim.x) dst[t] = src[t];
    if (threadIdx.x == 0 && fout) fout[e] = f[a];
}

cudaError_t launch_export_elites(const int32_t* mf, const int32_t* mc, int nv, int p, int n_elite,
                                 const uint8_t* members, int nvpad, const PoolScratch& w, uint8_t* out,
                                 int32_t* fout, cudaStream_t st) {
    k_member_keys<<<(p + 255) / 256, 256, 0, st>>>(mf, mc, nv, p, w.keys0);
    const uint32_t maxbin = 2u * (uint32_t)(nv + 1);
    int bits = 1;
    while ((1u << bits) < maxbin) ++bits;
    k_sort_keys<<<1, kSortThreads, 0, st>>>(w.keys0, w.keys1, p, (bits + 7) / 8, w.order);
    if (n_elite > 0) k_gather_rows_f<<<n_elite, 128, 0, st>>>(w.order, n_elite, members, mf, nvpad, out, fout);
    return cudaGetLastError();
}

}  // namespace plse_dev
