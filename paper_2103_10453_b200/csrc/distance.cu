// distance.cu -- K3 Hamming distance blocks (population.hpp:41-87,
// coloring.hpp:159-167) on sm_100a CUDA cores.
//
// D[i][j] = #{v : A_i[v] != B_j[v]} over u8 colour rows (stride nvpad, pad
// bytes zero in every row, so they never count).  128x128 output tile per
// CTA, 256 threads x (8x8) accumulators, operands staged through shared
// memory in 32-byte K chunks.  Per 32-bit word pair: x = a ^ b marks
// differing bytes non-zero; ((x & 0x7f7f7f7f) + 0x7f7f7f7f) | x has bit 7 set
// exactly in the non-zero bytes; popc of that & 0x80808080 = differences.
// (The tcgen05 one-hot GEMM variant lives in similarity_tc.cu.)
#include "common.cuh"
#include "device_api.h"

namespace plse_dev {

constexpr int kTile = 128;
constexpr int kKw = 8;  // 32-bit words per K chunk (32 bytes)

__device__ __forceinline__ uint32_t ndiff4(uint32_t a, uint32_t b) {
    const uint32_t x = a ^ b;
    const uint32_t t = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;
    return __popc(t & 0x80808080u);
}

__global__ void __launch_bounds__(256) k_hamming(const uint8_t* __restrict__ A, int na, const uint8_t* __restrict__ B,
                                                 int nb, int nwords, int nvpad, uint16_t* __restrict__ D, int ldd,
                                                 int upper) {
    __shared__ uint32_t As[kKw][kTile + 4];
    __shared__ uint32_t Bs[kKw][kTile + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * kTile, j0 = blockIdx.x * kTile;
    if (upper && j0 + kTile <= i0) return;  // strictly below the diagonal: the consumer reads [min][max]
    uint32_t acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0;

    for (int w0 = 0; w0 < nwords; w0 += kKw) {
        // load: 128 rows x 8 words for A and for B = 1024 words each, 4 per thread
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e >> 3, w = e & 7;
            const int gw = w0 + w;
            uint32_t va = 0, vb = 0;
            if (gw < nwords) {
                if (i0 + row < na) va = reinterpret_cast<const uint32_t*>(A + (size_t)(i0 + row) * nvpad)[gw];
                if (j0 + row < nb) vb = reinterpret_cast<const uint32_t*>(B + (size_t)(j0 + row) * nvpad)[gw];
            }
            As[w][row] = va;
            Bs[w][row] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kKw; ++w) {
            uint32_t a[8], b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                a[q] = As[w][ty * 8 + q];
                b[q] = Bs[w][tx * 8 + q];
            }
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y) acc[x][y] += ndiff4(a[x], b[y]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        const int i = i0 + ty * 8 + x;
        if (i >= na) continue;
#pragma unroll
        for (int y = 0; y < 8; ++y) {
            const int j = j0 + tx * 8 + y;
            if (j < nb) D[(size_t)i * ldd + j] = (uint16_t)acc[x][y];
        }
    }
}

cudaError_t launch_hamming(const uint8_t* A, int na, const uint8_t* B, int nb, int nv, int nvpad, uint16_t* D,
                           int ldd, cudaStream_t st, int upper) {
    (void)nv;
    dim3 grid((nb + kTile - 1) / kTile, (na + kTile - 1) / kTile);
    k_hamming<<<grid, 256, 0, st>>>(A, na, B, nb, nvpad / 4, nvpad, D, ldd, upper);
    return cudaGetLastError();
}

}  // namespace plse_dev
