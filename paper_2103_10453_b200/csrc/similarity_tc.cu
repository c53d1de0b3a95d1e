// similarity_tc.cu -- K3 on the 5th-generation tensor cores.
//
// Hamming distance blocks (population.hpp:41-87, coloring.hpp:159-167) as an
// exact integer GEMM:  D(a, b) = |V| - <onehot(a), onehot(b)>,  where
// onehot(x)[kk] = [x[vert(kk)] == dom[kk]] over the K_dom = sum |D(v)| entries
// of the CSR domain list (colour 0 included, so uncoloured == uncoloured
// counts as equal).  K_dom is the minimum inner dimension of an exact
// equality-kernel factorisation (the equality matrix on D(v) has rank |D(v)|).
//
// k_onehot expands u8 colour rows into 0/1 u8 rows (K padded to 128);
// k_sim_tc computes 128x256 output tiles: TMA (128B swizzle) -> 4-stage
// shared-memory ring -> tcgen05.mma.cta_group::1.kind::i8 (K = 32 per
// instruction, s32 accumulators in TMEM, 256 columns) -> tcgen05.ld epilogue
// that writes |V| - S as u16.  One elected thread issues TMA, one issues MMA;
// all four warps drain TMEM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 128, kTcStages = 4;
constexpr int kTcGroupM = 12;  // tile rows per raster group
constexpr int kTcABytes = kTcBM * kTcBK;  // 16 KB
constexpr int kTcBBytes = kTcBN * kTcBK;  // 32 KB
constexpr int kTcStageBytes = kTcABytes + kTcBBytes;
constexpr int kTcSmem = kTcStages * kTcStageBytes + 1024 + 256;
constexpr uint32_t kTcTmemCols = 256;

// ---------------------------------------------------------------- one-hot
__global__ void k_onehot(const uint8_t* __restrict__ X, int nvpad, const uint16_t* __restrict__ col_vert,
                         const uint8_t* __restrict__ col_color, int K, int Kpad, uint8_t* __restrict__ H) {
    extern __shared__ uint8_t row[];
    const int i = blockIdx.x;
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)i * nvpad);
    for (int t = threadIdx.x; t < nvpad / 16; t += blockDim.x) reinterpret_cast<uint4*>(row)[t] = src[t];
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(H + (size_t)i * Kpad);
    for (int c = threadIdx.x; c < Kpad / 16; c += blockDim.x) {
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int kk = c * 16 + b;
            if (kk < K && row[col_vert[kk]] == col_color[kk]) w[b >> 2] |= 1u << (8 * (b & 3));
        }
        dst[c] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address  [0,14)
    d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;         // SBO            [32,46)
    d |= (uint64_t)1 << 46;                   // descriptor version 1 (sm_100)
    d |= (uint64_t)2 << 61;                   // SWIZZLE_128B   [61,64)
    return d;
}

// instruction descriptor: kind::i8, D = s32, A = B = u8, both K-major, M = 128, N = 256
constexpr uint32_t kTcIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(kTcBN >> 3) << 17) |
                              ((uint32_t)(kTcBM >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// ---------------------------------------------------------------- GEMM
__global__ void __launch_bounds__(128, 1)
    k_sim_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
             int num_kb, int nv, uint16_t* __restrict__ D, int ldd, int upper) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kTcStages + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grouped raster: consecutive CTAs walk kTcGroupM tile rows, then the next tile column, so one wave
    // of resident CTAs shares ~12 A tiles and ~12 B tiles per K slab in L2 (row-major order would stream
    // every B tile once per tile row from DRAM)
    const int nt_n = (N + kTcBN - 1) / kTcBN, nt_m = (M + kTcBM - 1) / kTcBM;
    const int lin = blockIdx.x, per_group = kTcGroupM * nt_n;
    const int first_m = (lin / per_group) * kTcGroupM, gm = min(nt_m - first_m, kTcGroupM);
    const int tile_m = first_m + (lin % per_group) % gm, tile_n = (lin % per_group) / gm;
    // symmetric block (A == B): tiles strictly below the diagonal are skipped, the consumer reads [min][max]
    if (upper && (tile_n + 1) * kTcBN <= tile_m * kTcBM) return;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kTcStages), done = smem_u32(bars + 2 * kTcStages);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        for (int kb = 0; kb < num_kb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (uint32_t)(kb / kTcStages) & 1u;
            if (kb >= kTcStages) mbar_wait(empty0 + 8 * s, ph ^ 1u);
            uint8_t* sa = smem + s * kTcStageBytes;
            mbar_expect_tx(full0 + 8 * s, kTcStageBytes);
            tma_load_2d(smem_u32(sa), &tmA, full0 + 8 * s, kb * kTcBK, tile_m * kTcBM);
            tma_load_2d(smem_u32(sa + kTcABytes), &tmB, full0 + 8 * s, kb * kTcBK, tile_n * kTcBN);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer (one thread for the CTA)
        for (int kb = 0; kb < num_kb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (uint32_t)(kb / kTcStages) & 1u;
            mbar_wait(full0 + 8 * s, ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + s * kTcStageBytes);
            const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kTcABytes);
#pragma unroll
            for (int kk = 0; kk < kTcBK / 32; ++kk)
                umma_i8(tmem_d, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), kTcIdesc, (kb | kk) != 0);
            umma_commit(empty0 + 8 * s);  // frees the stage when these MMAs retire
        }
        umma_commit(done);
    }
    __syncwarp();

    // ---- epilogue: warp w drains TMEM lanes [32w, 32w+32) = output rows of this warp
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = tile_m * kTcBM + warp * 32 + lane;
    uint16_t* drow = D + (size_t)row * ldd + (size_t)tile_n * kTcBN;
#pragma unroll 1
    for (int c0 = 0; c0 < kTcBN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
            const int col0 = tile_n * kTcBN + c0;
            if (col0 + 32 <= N) {
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    pk[q] = ((uint32_t)(nv - (int)v[2 * q]) & 0xFFFFu) | ((uint32_t)(nv - (int)v[2 * q + 1]) << 16);
                uint4* d4 = reinterpret_cast<uint4*>(drow + c0);
                if ((reinterpret_cast<uintptr_t>(d4) & 15) == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) d4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 32; ++q) drow[c0 + q] = (uint16_t)(nv - (int)v[q]);
                }
            } else {
                for (int q = 0; q < 32 && col0 + q < N; ++q) drow[c0 + q] = (uint16_t)(nv - (int)v[q]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(kTcTmemCols));
}

// ---------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static bool make_map(CUtensorMap* m, const uint8_t* base, int rows, int Kpad, int box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)Kpad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)Kpad};
    cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_onehot(const uint8_t* X, int rows, int nvpad, const uint16_t* col_vert, const uint8_t* col_color,
                          int K, int Kpad, uint8_t* H, cudaStream_t st) {
    k_onehot<<<rows, 256, nvpad, st>>>(X, nvpad, col_vert, col_color, K, Kpad, H);
    return cudaGetLastError();
}

// the shared-memory opt-in is a per-device function attribute: called by plse_create after cudaSetDevice
cudaError_t prepare_similarity_tc() {
    return cudaFuncSetAttribute(k_sim_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
}

cudaError_t launch_similarity_tc(const uint8_t* HA, int M, const uint8_t* HB, int N, int Kpad, int nv, uint16_t* D,
                                 int ldd, cudaStream_t st, int upper) {
    CUtensorMap ma, mb;
    if (!make_map(&ma, HA, M, Kpad, kTcBM) || !make_map(&mb, HB, N, Kpad, kTcBN)) return cudaErrorInvalidValue;
    const int tiles = ((N + kTcBN - 1) / kTcBN) * ((M + kTcBM - 1) / kTcBM);
    k_sim_tc<<<tiles, 128, kTcSmem, st>>>(ma, mb, M, N, Kpad / kTcBK, nv, D, ldd, upper);
    return cudaGetLastError();
}

}  // namespace plse_dev
