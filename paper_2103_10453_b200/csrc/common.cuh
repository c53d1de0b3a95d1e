// common.cuh -- device-side primitives shared by the sm_100a kernels.
//
// RNG: the reference keys every stochastic component by a stream derived
// from (master_seed, tag, index) (rng.hpp:81-92) and draws with xoshiro256++
// (rng.hpp:30-58).  The population phases (init, matching, crossover) replay
// those sequential streams exactly, one thread per individual.  The PartialCol
// tie-break uses the canonical counter-based draw: output j of the
// splitmix64 sequence started at the stream seed.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace plse_dev {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr unsigned kFull = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// rng.hpp:14-19
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    s += kGolden;
    return mix64(s);
}

// rng.hpp:81-88
__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
    uint64_t s = master;
    uint64_t h = splitmix64(s);
    s = h ^ (tag * 0xD1B54A32D192ED03ULL);
    h = splitmix64(s);
    s = h ^ (index * 0x8CB92BA72F3D8DD7ULL);
    return splitmix64(s);
}

// The canonical tie-break draw of step j of the stream seeded s: SplitMix64's (j+1)-th output from state
// s (a counter-based generator keyed by the full 64-bit stream seed); h1 = hi32 ranks the move, h2 = lo32
// the tenure offset.
__host__ __device__ __forceinline__ uint64_t canon_draw(uint64_t s, uint64_t j) { return mix64(s + (j + 1) * kGolden); }

// The kernels draw 32 steps at a time: lane l holds the draw of step (j & ~31) + l, broadcast per step.
struct CanonDraws {
    uint64_t seed;
    uint32_t hi, lo;  // this lane's draw of the current 32-step window
    int64_t window = -1;
#ifdef __CUDACC__
    __device__ __forceinline__ void at(uint32_t j, int lane, uint32_t& h1, uint32_t& h2) {
        const int64_t w = (int64_t)(j & ~31u);
        if (w != window) {  // warp-uniform
            const uint64_t z = canon_draw(seed, (uint64_t)w + (uint64_t)lane);
            hi = (uint32_t)(z >> 32);
            lo = (uint32_t)z;
            window = w;
        }
        h1 = __shfl_sync(0xFFFFFFFFu, hi, j & 31);
        h2 = __shfl_sync(0xFFFFFFFFu, lo, j & 31);
    }
#endif
};
#ifdef __CUDACC__
// %globaltimer (ns): the device clock the run's time limit is checked against
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

// xoshiro256++ seeded by splitmix64 (rng.hpp:21-58)
struct Xoshiro {
    uint64_t s0, s1, s2, s3;
    __host__ __device__ __forceinline__ explicit Xoshiro(uint64_t seed) {
        uint64_t sm = seed;
        s0 = splitmix64(sm);
        s1 = splitmix64(sm);
        s2 = splitmix64(sm);
        s3 = splitmix64(sm);
    }
    __host__ __device__ __forceinline__ static uint64_t rotl(uint64_t x, int k) {
#ifdef __CUDA_ARCH__
        // two funnel shifts (SHF.L.W) instead of the four shifts and an OR of the generic form
        const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
        const uint32_t a = k < 32 ? lo : hi, b = k < 32 ? hi : lo;  // k >= 32: swap the halves first
        const uint32_t nhi = __funnelshift_l(a, b, k & 31), nlo = __funnelshift_l(b, a, k & 31);
        return ((uint64_t)nhi << 32) | nlo;
#else
        return (x << k) | (x >> (64 - k));
#endif
    }
    __host__ __device__ __forceinline__ uint64_t next() {
        const uint64_t result = rotl(s0 + s3, 23) + s0;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl(s3, 45);
        return result;
    }
    // rng.hpp:43-49; `threshold` = (2^64 - bound) % bound, precomputed by the caller
    __host__ __device__ __forceinline__ uint64_t below(uint64_t bound, uint64_t threshold) {
        for (;;) {
            const uint64_t x = next();
            if (x >= threshold) return x % bound;
        }
    }
    __host__ __device__ __forceinline__ uint64_t below(uint64_t bound) {
        return below(bound, (0 - bound) % bound);
    }
};

// 0-based r-th set bit of a 64-bit word (r < popc(m))
__device__ __forceinline__ int nth_bit64(uint64_t m, int r) {
    int pos = 0;
    uint32_t x = (uint32_t)m;
    int c = __popc(x);
    if (r >= c) {
        r -= c;
        x = (uint32_t)(m >> 32);
        pos = 32;
    }
    c = __popc(x & 0xFFFFu);
    if (r >= c) { r -= c; x >>= 16; pos += 16; }
    c = __popc(x & 0xFFu);
    if (r >= c) { r -= c; x >>= 8; pos += 8; }
    c = __popc(x & 0xFu);
    if (r >= c) { r -= c; x >>= 4; pos += 4; }
    c = __popc(x & 0x3u);
    if (r >= c) { r -= c; x >>= 2; pos += 2; }
    if (r >= (int)(x & 1u)) pos += 1;
    return pos;
}

}  // namespace plse_dev
