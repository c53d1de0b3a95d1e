// ref_draws.cuh -- the reference's next_below (rng.hpp:43-49) on the device, and the division-free
// "next_below(bound) == 0" test the reference-tie-break kernels (improve_ref.cu, plits_ref.cu) use to
// decide a reservoir draw.
#pragma once
#include "common.cuh"

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
// 64-bit inverses of the odd parts of 0..256 (0 unused), for the common small bounds
// global (L1-cached) rather than __constant__: the lanes of a warp index it divergently
static __device__ uint64_t kOddInv[257] = {
    0x0000000000000000ULL, 0x0000000000000001ULL, 0x0000000000000001ULL, 0xaaaaaaaaaaaaaaabULL,
    0x0000000000000001ULL, 0xcccccccccccccccdULL, 0xaaaaaaaaaaaaaaabULL, 0x6db6db6db6db6db7ULL,
    0x0000000000000001ULL, 0x8e38e38e38e38e39ULL, 0xcccccccccccccccdULL, 0x2e8ba2e8ba2e8ba3ULL,
    0xaaaaaaaaaaaaaaabULL, 0x4ec4ec4ec4ec4ec5ULL, 0x6db6db6db6db6db7ULL, 0xeeeeeeeeeeeeeeefULL,
    0x0000000000000001ULL, 0xf0f0f0f0f0f0f0f1ULL, 0x8e38e38e38e38e39ULL, 0x86bca1af286bca1bULL,
    0xcccccccccccccccdULL, 0xcf3cf3cf3cf3cf3dULL, 0x2e8ba2e8ba2e8ba3ULL, 0xd37a6f4de9bd37a7ULL,
    0xaaaaaaaaaaaaaaabULL, 0x8f5c28f5c28f5c29ULL, 0x4ec4ec4ec4ec4ec5ULL, 0x84bda12f684bda13ULL,
    0x6db6db6db6db6db7ULL, 0x34f72c234f72c235ULL, 0xeeeeeeeeeeeeeeefULL, 0xef7bdef7bdef7bdfULL,
    0x0000000000000001ULL, 0x0f83e0f83e0f83e1ULL, 0xf0f0f0f0f0f0f0f1ULL, 0xaf8af8af8af8af8bULL,
    0x8e38e38e38e38e39ULL, 0x14c1bacf914c1badULL, 0x86bca1af286bca1bULL, 0x6f96f96f96f96f97ULL,
    0xcccccccccccccccdULL, 0x8f9c18f9c18f9c19ULL, 0xcf3cf3cf3cf3cf3dULL, 0x82fa0be82fa0be83ULL,
    0x2e8ba2e8ba2e8ba3ULL, 0x4fa4fa4fa4fa4fa5ULL, 0xd37a6f4de9bd37a7ULL, 0x51b3bea3677d46cfULL,
    0xaaaaaaaaaaaaaaabULL, 0x7d6343eb1a1f58d1ULL, 0x8f5c28f5c28f5c29ULL, 0xfafafafafafafafbULL,
    0x4ec4ec4ec4ec4ec5ULL, 0x21cfb2b78c13521dULL, 0x84bda12f684bda13ULL, 0x6fb586fb586fb587ULL,
    0x6db6db6db6db6db7ULL, 0x823ee08fb823ee09ULL, 0x34f72c234f72c235ULL, 0xcbeea4e1a08ad8f3ULL,
    0xeeeeeeeeeeeeeeefULL, 0x4fbcda3ac10c9715ULL, 0xef7bdef7bdef7bdfULL, 0xefbefbefbefbefbfULL,
    0x0000000000000001ULL, 0x0fc0fc0fc0fc0fc1ULL, 0x0f83e0f83e0f83e1ULL, 0xf0b7672a07a44c6bULL,
    0xf0f0f0f0f0f0f0f1ULL, 0xf128cfc4a33f128dULL, 0xaf8af8af8af8af8bULL, 0x193d4bb7e327a977ULL,
    0x8e38e38e38e38e39ULL, 0x7e3f1f8fc7e3f1f9ULL, 0x14c1bacf914c1badULL, 0x2fc962fc962fc963ULL,
    0x86bca1af286bca1bULL, 0x4fcace213f2b3885ULL, 0x6f96f96f96f96f97ULL, 0x9b8b577e613716afULL,
    0xcccccccccccccccdULL, 0x2c3f35ba781948b1ULL, 0x8f9c18f9c18f9c19ULL, 0xa3784a062b2e43dbULL,
    0xcf3cf3cf3cf3cf3dULL, 0xfcfcfcfcfcfcfcfdULL, 0x82fa0be82fa0be83ULL, 0x66fd0eb66fd0eb67ULL,
    0x2e8ba2e8ba2e8ba3ULL, 0xf47e8fd1fa3f47e9ULL, 0x4fa4fa4fa4fa4fa5ULL, 0x2fd2fd2fd2fd2fd3ULL,
    0xd37a6f4de9bd37a7ULL, 0x4fd3f4fd3f4fd3f5ULL, 0x51b3bea3677d46cfULL, 0x4e25b9efd4e25b9fULL,
    0xaaaaaaaaaaaaaaabULL, 0xa3a0fd5c5f02a3a1ULL, 0x7d6343eb1a1f58d1ULL, 0xafd6a052bf5a814bULL,
    0x8f5c28f5c28f5c29ULL, 0x3a4c0a237c32b16dULL, 0xfafafafafafafafbULL, 0xdab7ec1dd3431b57ULL,
    0x4ec4ec4ec4ec4ec5ULL, 0x8fd8fd8fd8fd8fd9ULL, 0x21cfb2b78c13521dULL, 0x77a04c8f8d28ac43ULL,
    0x84bda12f684bda13ULL, 0xa6c0964fda6c0965ULL, 0x6fb586fb586fb587ULL, 0xb195e8efdb195e8fULL,
    0x6db6db6db6db6db7ULL, 0x90fdbc090fdbc091ULL, 0x823ee08fb823ee09ULL, 0x2a4bafdc61f2a4bbULL,
    0x34f72c234f72c235ULL, 0xcfdcfdcfdcfdcfddULL, 0xcbeea4e1a08ad8f3ULL, 0xd946fdd946fdd947ULL,
    0xeeeeeeeeeeeeeeefULL, 0x1b810ecf56be69c9ULL, 0x4fbcda3ac10c9715ULL, 0x2fdeb2fdeb2fdeb3ULL,
    0xef7bdef7bdef7bdfULL, 0x1cac083126e978d5ULL, 0xefbefbefbefbefbfULL, 0x7efdfbf7efdfbf7fULL,
    0x0000000000000001ULL, 0x80fe03f80fe03f81ULL, 0x0fc0fc0fc0fc0fc1ULL, 0x03e88cb3c9484e2bULL,
    0x0f83e0f83e0f83e1ULL, 0x133f84cfe133f84dULL, 0xf0b7672a07a44c6bULL, 0x1a8c536fe1a8c537ULL,
    0xf0f0f0f0f0f0f0f1ULL, 0xe21a291c077975b9ULL, 0xf128cfc4a33f128dULL, 0x3aef6ca970586723ULL,
    0xaf8af8af8af8af8bULL, 0x70913f8bcd29c245ULL, 0x193d4bb7e327a977ULL, 0xefe35b4cfaa11e6fULL,
    0x8e38e38e38e38e39ULL, 0x70fe3c070fe3c071ULL, 0x7e3f1f8fc7e3f1f9ULL, 0xd4766bf908b51d9bULL,
    0x14c1bacf914c1badULL, 0xdf5b0f768ce2cabdULL, 0x2fc962fc962fc963ULL, 0x6fe4dfc9bf937f27ULL,
    0x86bca1af286bca1bULL, 0x53a8fe53a8fe53a9ULL, 0x4fcace213f2b3885ULL, 0x2fe592fe592fe593ULL,
    0x6f96f96f96f96f97ULL, 0x5b4fe5e92c0685b5ULL, 0x9b8b577e613716afULL, 0xb5efe63d2eb11b5fULL,
    0xcccccccccccccccdULL, 0xf9a3c6c1fcd1e361ULL, 0x2c3f35ba781948b1ULL, 0x1f693a1c451ab30bULL,
    0x8f9c18f9c18f9c19ULL, 0xcfe72cfe72cfe72dULL, 0xa3784a062b2e43dbULL, 0x8d07aa27db35a717ULL,
    0xcf3cf3cf3cf3cf3dULL, 0xf25deacafb74a399ULL, 0xfcfcfcfcfcfcfcfdULL, 0x80bfa02fe80bfa03ULL,
    0x82fa0be82fa0be83ULL, 0x882383b30d516325ULL, 0x66fd0eb66fd0eb67ULL, 0xefe898231bcb564fULL,
    0x2e8ba2e8ba2e8ba3ULL, 0x43fa36f5e02e4851ULL, 0xf47e8fd1fa3f47e9ULL, 0xed6866f8d962ae7bULL,
    0x4fa4fa4fa4fa4fa5ULL, 0x3454dca410f8ed9dULL, 0x2fd2fd2fd2fd2fd3ULL, 0x6fe99e1395aedd07ULL,
    0xd37a6f4de9bd37a7ULL, 0x9dc0588fe9dc0589ULL, 0x4fd3f4fd3f4fd3f5ULL, 0x8a4472fea18a4473ULL,
    0x51b3bea3677d46cfULL, 0xa53fa94fea53fa95ULL, 0x4e25b9efd4e25b9fULL, 0x1d7ca632ee936f3fULL,
    0xaaaaaaaaaaaaaaabULL, 0x70bf015390948f41ULL, 0xa3a0fd5c5f02a3a1ULL, 0xafeafeafeafeafebULL,
    0x7d6343eb1a1f58d1ULL, 0xc96bdb9d3d137e0dULL, 0xafd6a052bf5a814bULL, 0x2697cc8aef46c0f7ULL,
    0x8f5c28f5c28f5c29ULL, 0xfae7cd0e028c1979ULL, 0x3a4c0a237c32b16dULL, 0x99da2ae0791064e3ULL,
    0xfafafafafafafafbULL, 0x4fec04fec04fec05ULL, 0xdab7ec1dd3431b57ULL, 0xfb0d9a96e115062fULL,
    0x4ec4ec4ec4ec4ec5ULL, 0xf4f9e02732385831ULL, 0x8fd8fd8fd8fd8fd9ULL, 0xc0e8f2a76e68575bULL,
    0x21cfb2b78c13521dULL, 0xb3146e92a10d387dULL, 0x77a04c8f8d28ac43ULL, 0xe6fecf2e6fecf2e7ULL,
    0x84bda12f684bda13ULL, 0x8fed1fda3fb47f69ULL, 0xa6c0964fda6c0965ULL, 0xd4bfb52fed4bfb53ULL,
    0x6fb586fb586fb587ULL, 0xd774fed774fed775ULL, 0xb195e8efdb195e8fULL, 0x687763dfdb43bb1fULL,
    0x6db6db6db6db6db7ULL, 0x0fedcba987654321ULL, 0x90fdbc090fdbc091ULL, 0x1b10ea929ba144cbULL,
    0x823ee08fb823ee09ULL, 0x1d10c4c0478bbcedULL, 0x2a4bafdc61f2a4bbULL, 0x6fee44b5bfb912d7ULL,
    0x34f72c234f72c235ULL, 0x63fb9aeb1fdcd759ULL, 0xcfdcfdcfdcfdcfddULL, 0x76bd8c8714b2a7c3ULL,
    0xcbeea4e1a08ad8f3ULL, 0xde83c7d4cb125ce5ULL, 0xd946fdd946fdd947ULL, 0x64afaa4f437b2e0fULL,
    0xeeeeeeeeeeeeeeefULL, 0xf010fef010fef011ULL, 0x1b810ecf56be69c9ULL, 0x641511e8d2b3183bULL,
    0x4fbcda3ac10c9715ULL, 0x1913da62386cab5dULL, 0x2fdeb2fdeb2fdeb3ULL, 0xf6ac0c6fef6ac0c7ULL,
    0xef7bdef7bdef7bdfULL, 0x367d6e020e64c149ULL, 0x1cac083126e978d5ULL, 0x28cbfbeb9a020a33ULL,
    0xefbefbefbefbefbfULL, 0x8796c44ce6b41c55ULL, 0x7efdfbf7efdfbf7fULL, 0xfefefefefefefeffULL,
    0x0000000000000001ULL};

__device__ __forceinline__ bool divides(uint64_t bound, uint64_t x) {
    const int sh = __ffsll((long long)bound) - 1;
    if (x & ((1ULL << sh) - 1)) return false;
    const uint64_t o = bound >> sh, y = x >> sh;
    uint64_t inv;
    if (bound <= 256) {
        inv = __ldg(&kOddInv[bound]);
    } else {
        inv = o;  // Newton: o * inv == 1 (mod 2^64), 3 -> 6 -> 12 -> 24 -> 48 -> 96 correct bits
#pragma unroll
        for (int it = 0; it < 5; ++it) inv *= 2 - o * inv;
    }
    return __umul64hi(y * inv, o) == 0;
}

__device__ __forceinline__ bool ref_below_is_zero(Xoshiro& rng, uint64_t bound) {
    for (;;) {
        const uint64_t x = rng.next();
        if (x < bound && x < (0 - bound) % bound) continue;  // rejected (probability < bound / 2^64)
        return divides(bound, x);
    }
}

// the fast paths' draws (improve_ref.cu, plits_ref.cu): M consecutive outputs of the individual's
// xoshiro256++ stream, 32 at a time.  Only the state update is a serial chain, so lane 0 runs just that (14 word ops per output) and parks
// each output's inputs (s0, s3 before the update) in stage[0, 64); the lanes then form the outputs
// rotl(s0 + s3, 23) + s0 in parallel.  For output d: d < E is an early draw (only its possible rejection
// matters), d >= E is the draw of final-segment member j = d - E + 2, kept iff next_below(j) == 0.
// Returns, per lane, the largest kept member (0: none) and raises `bad` on an output below 2^32 (a
// rejection is possible: the caller takes the exact walk).
__device__ __forceinline__ int ref_stream_draws(Xoshiro& rng, uint64_t* stage, int E, int M, int lane, bool& bad) {
    int bestj = 0;
    bool low = false;
    for (int d0 = 0; d0 < M; d0 += 32) {
        const int cnt = min(32, M - d0);
        if (lane == 0) {
            uint64_t s0 = rng.s0, s1 = rng.s1, s2 = rng.s2, s3 = rng.s3;
            for (int d = 0; d < cnt; ++d) {
                stage[d] = s0;  // two 64-bit stores from the state's own register pairs (no packing moves)
                stage[32 + d] = s3;
                const uint64_t t = s1 << 17;
                s2 ^= s0;
                s3 ^= s1;
                s1 ^= s2;
                s0 ^= s3;
                s2 ^= t;
                s3 = Xoshiro::rotl(s3, 45);
            }
            rng.s0 = s0;
            rng.s1 = s1;
            rng.s2 = s2;
            rng.s3 = s3;
        }
        __syncwarp();
        if (lane < cnt) {
            const uint64_t x0 = stage[lane], x3 = stage[32 + lane];
            const uint64_t y = Xoshiro::rotl(x0 + x3, 23) + x0;
            low |= (y >> 32) == 0;
            const int d = d0 + lane;
            if (d >= E && divides((uint64_t)(d - E + 2), y)) bestj = d - E + 2;
        }
        __syncwarp();
    }
    bad = __any_sync(kFull, low);
    return bestj;
}

}  // namespace plse_dev
