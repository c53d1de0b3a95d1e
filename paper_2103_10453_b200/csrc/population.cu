// population.cu -- K0 init, f/c evaluation, K4b matching, K4c crossover on
// sm_100a (K4a pool update: pool.cu).  All integer / byte work (HBM-bound); the
// sequential xoshiro streams of the reference are replayed exactly, one
// thread per individual, so these phases are bit-exact with the reference.
#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

// ---------------------------------------------------------------- K0 init
// engine.hpp:88-106: colour = D(v)[1 + next_index(|D(v)|-1)] from stream (seed, 1, i)
__global__ void k_init_population(const PopGraph g, int p, uint64_t master, uint64_t offset, uint8_t* members) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    Xoshiro rng(derive_seed(master, 1, offset + (uint64_t)i));
    uint8_t* row = members + (size_t)i * g.nvpad;
    uint32_t word[4] = {0, 0, 0, 0};
    for (int v = 0; v < g.nvpad; ++v) {
        uint32_t c = 0;
        if (v < g.nv) {
            const int begin = g.dom_off[v] + 1;
            const int b = g.dom_off[v + 1] - begin;
            const uint64_t x = rng.below((uint64_t)b, g.below_thr[b]);
            c = g.dom[begin + (int)x];
        }
        word[(v >> 2) & 3] |= c << (8 * (v & 3));
        if ((v & 15) == 15) {
            *reinterpret_cast<uint4*>(row + v - 15) = make_uint4(word[0], word[1], word[2], word[3]);
            word[0] = word[1] = word[2] = word[3] = 0;
        }
    }
}

cudaError_t launch_init_population(const PopGraph& g, int p, uint64_t master, uint64_t offset, uint8_t* members,
                                   cudaStream_t st) {
    k_init_population<<<(p + 127) / 128, 128, 0, st>>>(g, p, master, offset, members);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- f / c
// coloring.hpp:59-73: f = #zeros, c = #edges with equal non-zero colours.
// One warp per individual; c = sum over coloured v of same-coloured neighbours / 2.
__global__ void k_eval_fc(const PopGraph g, int p, const uint8_t* colors, int32_t* fo, int32_t* co) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= p) return;
    const uint8_t* row = colors + (size_t)i * g.nvpad;
    int zf = 0, cc = 0;
    for (int v = lane; v < g.nv; v += 32) {
        const int k = row[v];
        if (!k) {
            ++zf;
            continue;
        }
        const uint16_t rc = g.cell[v];
        const int r = rc >> 8, c = rc & 0xFF;
        for (int u = g.row_start[r]; u < g.row_start[r + 1]; ++u) cc += (row[u] == k);
        for (int t = g.col_start[c]; t < g.col_start[c + 1]; ++t) cc += (row[g.col_list[t]] == k);
        cc -= 2;
    }
    zf = __reduce_add_sync(kFull, zf);
    cc = __reduce_add_sync(kFull, cc);
    if (lane == 0) {
        if (fo) fo[i] = zf;
        if (co) co[i] = cc / 2;
    }
}

cudaError_t launch_eval_fc(const PopGraph& g, int p, const uint8_t* colors, int32_t* f, int32_t* c, cudaStream_t st) {
    k_eval_fc<<<(p + 7) / 8, 256, 0, st>>>(g, p, colors, f, c);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- host-format colourings
// plse_set_colors / plse_get_colors exchange u16 rows [p][nv] with the caller; the device keeps u8 rows
// [p][nvpad] (zero padding).  The conversion and the domain check (every colour 0 or not prefilled in its
// row or column, lsgraph.hpp:152-156) run here, over the copied u16 rows, instead of a host loop.
__global__ void k_unpack_colors(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad, int n, int W,
                                const uint16_t* cell, const uint64_t* pr, const uint64_t* pc, int* bad) {
    const int quads = nvpad >> 2;
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)p * quads) return;
    const int i = (int)(t / quads), v0 = (int)(t % quads) * 4;
    const uint16_t* row = in + (size_t)i * nv;
    uint32_t word = 0;
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int v = v0 + j;
        if (v >= nv) break;
        const int k = row[v];
        if (k) {
            const uint16_t rc = cell[v];
            const int q = k >> 6;
            const bool taken = q < W && (((pr[(rc >> 8) * W + q] | pc[(rc & 0xFF) * W + q]) >> (k & 63)) & 1ULL);
            ok &= k <= n && !taken;
        }
        word |= (uint32_t)(k & 0xFF) << (8 * j);
    }
    if (!ok) atomicOr(bad, 1);
    reinterpret_cast<uint32_t*>(out + (size_t)i * nvpad)[v0 >> 2] = word;
}

__global__ void k_pack_colors(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)p * nv) return;
    const int i = (int)(t / nv), v = (int)(t % nv);
    out[t] = in[(size_t)i * nvpad + v];
}

cudaError_t launch_unpack_colors(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad, int n, int W,
                                 const uint16_t* cell, const uint64_t* pr, const uint64_t* pc, int* bad,
                                 cudaStream_t st) {
    const size_t threads = (size_t)p * (nvpad >> 2);
    k_unpack_colors<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(in, out, p, nv, nvpad, n, W, cell, pr, pc,
                                                                       bad);
    return cudaGetLastError();
}

cudaError_t launch_pack_colors(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad, cudaStream_t st) {
    const size_t threads = (size_t)p * nv;
    k_pack_colors<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(in, out, p, nv, nvpad);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K4b matching
// crossover.hpp:67-83 + nearest_neighbor population.hpp:209-228.  The partner
// loop is sequential in the reference but every row reads and writes only its
// own (slot-keyed) exclusion row, so rows are independent: one warp per row.
__global__ void k_match(const uint16_t* dist, int p, int matching, int exclusion, uint32_t* excl, int ew,
                        uint64_t master, uint64_t stream_base, int32_t* partner) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= p) return;
    int j;
    if (matching == PLSE_M_RANDOM) {
        if (lane == 0) {
            Xoshiro m(derive_seed(master, 6, stream_base + (uint64_t)i));
            j = (int)m.below((uint64_t)(p - 1));
            if (j >= i) ++j;
        }
        j = __shfl_sync(kFull, j, 0);
    } else {
        const uint16_t* row = dist + (size_t)i * p;
        const uint32_t* ex = excl + (size_t)i * ew;
        const bool use_ex = exclusion != PLSE_E_OFF;
        uint32_t bu = 0xFFFFFFFFu, br = 0xFFFFFFFFu;  // (d << 16 | j) would overflow for p > 65535: keep two keys
        int bju = -1, bjr = -1;
        for (int jj = lane; jj < p; jj += 32) {
            if (jj == i) continue;
            const uint32_t d = row[jj];
            if (d < bu) {
                bu = d;
                bju = jj;
            }
            if (use_ex && ((ex[jj >> 5] >> (jj & 31)) & 1)) continue;
            if (d < br) {
                br = d;
                bjr = jj;
            }
        }
        // warp argmin, lowest index on ties
        const uint32_t mu = __reduce_min_sync(kFull, bu);
        const uint32_t ju = __reduce_min_sync(kFull, bu == mu && bju >= 0 ? (uint32_t)bju : 0xFFFFFFFFu);
        const uint32_t mr = __reduce_min_sync(kFull, br);
        const uint32_t jr = __reduce_min_sync(kFull, br == mr && bjr >= 0 ? (uint32_t)bjr : 0xFFFFFFFFu);
        if (jr == 0xFFFFFFFFu) {
            // every partner excluded: clear the row, return the unrestricted nearest neighbour
            for (int w = lane; w < ew; w += 32) excl[(size_t)i * ew + w] = 0;
            __syncwarp();
            j = (int)ju;
        } else {
            j = (int)jr;
        }
    }
    if (lane == 0) {
        if (exclusion != PLSE_E_OFF) excl[(size_t)i * ew + (j >> 5)] |= 1u << (j & 31);
        partner[i] = j;
    }
}

cudaError_t launch_match(const uint16_t* dist, int p, int matching, int exclusion, uint32_t* excl, int excl_words,
                         uint64_t master, uint64_t stream_base, int32_t* partner, cudaStream_t st) {
    k_match<<<(p + 7) / 8, 256, 0, st>>>(dist, p, matching, exclusion, excl, excl_words, master, stream_base,
                                         partner);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K4c crossover
// crossover.hpp:26-46, 85-102.  keep first parent's colour iff
// next_double() < p_ij  <=>  (x >> 11) < ceil(p_ij * 2^53)  (exact: both sides scaled by 2^53).
__global__ void k_crossover(const uint8_t* members, const uint16_t* dist, const int32_t* partner, int p, int nv,
                            int nvpad, int mode, double beta, uint64_t master, uint64_t stream_base,
                            uint8_t* offspring) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const uint8_t* first = members + (size_t)i * nvpad;
    uint8_t* child = offspring + (size_t)i * nvpad;
    if (mode == PLSE_X_NONE) {
        for (int t = 0; t < nvpad / 16; ++t)
            reinterpret_cast<uint4*>(child)[t] = reinterpret_cast<const uint4*>(first)[t];
        return;
    }
    const int j = partner[i];
    const uint8_t* second = members + (size_t)j * nvpad;
    double pij = 0.5;
    if (mode == PLSE_X_AUX) {
        const int32_t d = dist[(size_t)i * p + j];
        if ((double)d * beta <= (double)nv) {
            for (int t = 0; t < nvpad / 16; ++t)
                reinterpret_cast<uint4*>(child)[t] = reinterpret_cast<const uint4*>(first)[t];
            return;
        }
        pij = 1.0 - (double)nv / (beta * (double)d);
    }
    const uint64_t thr = (uint64_t)ceil(pij * 9007199254740992.0);
    Xoshiro rng(derive_seed(master, 3, stream_base + (uint64_t)i));
    for (int t = 0; t < nvpad / 16; ++t) {
        const uint4 a4 = reinterpret_cast<const uint4*>(first)[t];
        const uint4 b4 = reinterpret_cast<const uint4*>(second)[t];
        uint32_t a[4] = {a4.x, a4.y, a4.z, a4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w}, o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t sel = 0;
#pragma unroll
            for (int by = 0; by < 4; ++by) {
                const int v = t * 16 + q * 4 + by;
                if (v < nv && (rng.next() >> 11) < thr) sel |= 0xFFu << (8 * by);
            }
            o[q] = (a[q] & sel) | (b[q] & ~sel);
        }
        // pad bytes (v >= nv) take the second parent's pad byte, which is 0 like the first's
        reinterpret_cast<uint4*>(child)[t] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

cudaError_t launch_crossover(const uint8_t* members, const uint16_t* dist, const int32_t* partner, int p, int nv,
                             int nvpad, int mode, double beta, uint64_t master, uint64_t stream_base,
                             uint8_t* offspring, cudaStream_t st) {
    k_crossover<<<(p + 63) / 64, 64, 0, st>>>(members, dist, partner, p, nv, nvpad, mode, beta, master, stream_base,
                                             offspring);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- conversions
__global__ void k_u16_to_i32(const uint16_t* in, int32_t* out, size_t n) {
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x)
        out[t] = in[t];
}
__global__ void k_i32_to_u16(const int32_t* in, uint16_t* out, size_t n) {
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x)
        out[t] = (uint16_t)in[t];
}
__global__ void k_c16_to_8(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad) {
    const size_t total = (size_t)p * nvpad;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const size_t i = t / nvpad, v = t % nvpad;
        out[t] = v < (size_t)nv ? (uint8_t)in[i * nv + v] : 0;
    }
}
__global__ void k_c8_to_16(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad) {
    const size_t total = (size_t)p * nv;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const size_t i = t / nv, v = t % nv;
        out[t] = in[i * nvpad + v];
    }
}

static int grid_for(size_t n) {
    size_t g = (n + 255) / 256;
    return (int)(g > 148 * 16 ? 148 * 16 : (g ? g : 1));
}
cudaError_t launch_u16_to_i32(const uint16_t* in, int32_t* out, size_t count, cudaStream_t st) {
    k_u16_to_i32<<<grid_for(count), 256, 0, st>>>(in, out, count);
    return cudaGetLastError();
}
cudaError_t launch_i32_to_u16(const int32_t* in, uint16_t* out, size_t count, cudaStream_t st) {
    k_i32_to_u16<<<grid_for(count), 256, 0, st>>>(in, out, count);
    return cudaGetLastError();
}
cudaError_t launch_colors_u16_to_u8(const uint16_t* in, uint8_t* out, int p, int nv, int nvpad, cudaStream_t st) {
    k_c16_to_8<<<grid_for((size_t)p * nvpad), 256, 0, st>>>(in, out, p, nv, nvpad);
    return cudaGetLastError();
}
cudaError_t launch_colors_u8_to_u16(const uint8_t* in, uint16_t* out, int p, int nv, int nvpad, cudaStream_t st) {
    k_c8_to_16<<<grid_for((size_t)p * nv), 256, 0, st>>>(in, out, p, nv, nvpad);
    return cudaGetLastError();
}

}  // namespace plse_dev
